# round-2 final record on the final tree: GPU suite, smoke, bench lines
O=gpurun_out/final2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/gpu.txt
echo "== pytest -m gpu"; timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
echo "== bench 20/5"; timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_20.log 2>&1; grep '^{' $O/bench_20.log | tail -1 > $O/bench_20.json; python -c "import json;d=json.load(open('$O/bench_20.json'));print({k:d.get(k) for k in ('value','ls_tpot_attainment','ls_tpot_p99_ms','iteration_ms_p50','max_be_tok_s_at_slo')}, d['roofline']['frac'])"
echo "== reference 20/5"; timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.log 2>&1; grep '^{' $O/bench_ref.log | tail -1 > $O/bench_ref.json; python -c "import json;d=json.load(open('$O/bench_ref.json'));print({k:d.get(k) for k in ('value','ms_per_step')})"
echo "== longctx"; timeout 1200 python bench.py --workload longctx --steps 20 --warmup 5 --no-cpu-baseline --sweep "" > $O/bench_longctx.log 2>&1; grep '^{' $O/bench_longctx.log | tail -1 > $O/bench_longctx.json; python -c "import json;d=json.load(open('$O/bench_longctx.json'));print({k:d.get(k) for k in ('value','be_prefill_tok_s','ls_tpot_attainment','iteration_ms_p50')})"
echo "== probes"; timeout 300 python tools/probe_prefill.py > $O/probe_prefill.jsonl 2>&1; tail -1 $O/probe_prefill.jsonl
timeout 300 python tools/probe_layer.py 8 29 64 > $O/probe_layer.txt 2>&1; cat $O/probe_layer.txt
