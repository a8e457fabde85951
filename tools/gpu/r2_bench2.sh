O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
echo "== bench device merges 20/5"; timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_dev.log 2>&1; tail -c 3500 $O/bench_dev.log; echo
echo "== bench host merges 20/5"; timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --merges host --sweep "" > $O/bench_host.log 2>&1; tail -c 1500 $O/bench_host.log
