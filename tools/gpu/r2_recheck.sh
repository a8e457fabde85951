# round-2 re-entry check on HEAD: GPU suite, smoke, driver-style bench, K6 probe
O=gpurun_out/recheck; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/gpu.txt
echo "== probe prefill"; timeout 300 python tools/probe_prefill.py > $O/probe_prefill.jsonl 2>&1; cat $O/probe_prefill.jsonl | tail -4
echo "== pytest -m gpu"; timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; tail -5 $O/pytest_gpu.log
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
echo "== bench 20/5"; timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_20.log 2>&1; grep '^{' $O/bench_20.log | tail -1 > $O/bench_20.json; python -c "import json;d=json.load(open('$O/bench_20.json'));print({k:d.get(k) for k in ('value','e2e','ls_tpot_attainment','ls_tpot_p99_ms','iteration_ms_p50','roofline')})"
