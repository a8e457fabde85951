# remote-host bench lines on the final relay (chunked placements and fetches, non-blocking swap-ins)
O=gpurun_out/rbench6; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
for n in 1 2; do
  timeout 900 python bench.py --steps 20 --warmup 5 --remote-hosts $n --no-cpu-baseline --sweep "" > $O/bench_r$n.log 2>&1
  grep '^{' $O/bench_r$n.log | tail -1 > $O/bench_r$n.json
  python -c "import json;d=json.load(open('$O/bench_r$n.json'));r=d['remote_hosts'];print($n, {k:d.get(k) for k in ('value','ls_tpot_attainment','ls_tokens','be_tokens_via_cpu_attention','cpu_pool_busy_frac','iteration_ms_p50')}, r['per_host'], r['engine_state']['states'])" || tail -20 $O/bench_r$n.log
done
