# the bench line only
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; tail -c 3000 gpurun_out/bench.log
