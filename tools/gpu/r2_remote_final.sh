O=gpurun_out/rfinal; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
for i in 1 2; do timeout 600 python -m pytest tests/test_remote_host.py -q -s -p no:cacheprovider > $O/pytest_$i.log 2>&1; echo "remote tests $i: $(tail -1 $O/pytest_$i.log)"; done
timeout 900 python bench.py --steps 20 --warmup 5 --remote-hosts 1 --no-cpu-baseline --sweep "" > $O/bench_r1.log 2>&1
grep '^{' $O/bench_r1.log | tail -1 > $O/bench_r1.json
python -c "import json;d=json.load(open('$O/bench_r1.json'));r=d['remote_hosts'];print({k:d.get(k) for k in ('value','ls_tpot_attainment','ls_tokens','be_tokens_via_cpu_attention','cpu_pool_busy_frac','iteration_ms_p50')}, r['per_host'], r['engine_state']['states'])" || tail -20 $O/bench_r1.log
