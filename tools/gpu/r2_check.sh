# round-2 status check: GPU tests, smoke, driver-style bench
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
lscpu > $O/lscpu.txt; nvidia-smi topo -m > $O/topo.txt 2>&1
echo "== pytest -m gpu"; timeout 1500 python -m pytest tests -q -m gpu ${PYTEST_ARGS:-} -p no:cacheprovider > $O/pytest_gpu.log 2>&1; tail -15 $O/pytest_gpu.log
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
echo "== bench 20/5"; timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_20.log 2>&1; tail -c 2500 $O/bench_20.log
