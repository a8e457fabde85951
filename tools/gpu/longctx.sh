# config 5 bench (32k-token BE prompts)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python bench.py --workload longctx --steps 600 --warmup 100 --no-cpu-baseline > gpurun_out/bench_longctx.log 2>&1
tail -3 gpurun_out/bench_longctx.log | cut -c1-3000
