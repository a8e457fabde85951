# One GPU session: tests, smoke, bench, ncu launch list + full captures.
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
echo "== pytest -m gpu"; timeout 900 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
echo "== bench"; timeout 900 python bench.py > $O/bench.log 2>&1; tail -c 600 $O/bench.log
echo "== ncu launch list (bench)"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_bench.csv python bench.py --steps 8 --warmup 4 --profile-steps 0 --no-cpu-baseline > $O/ncu_launch.log 2>&1
python tools/ncu_summary.py $O/launches_bench.csv > $O/launches_bench.txt; head -14 $O/launches_bench.txt
echo "== ncu full (probe_step 16 rows x 700 ctx, 2 merges)"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 60 -c 8 -o $O/prof_gemm python tools/probe_step.py 16 700 2 2 > $O/ncu_gemm.log 2>&1; tail -1 $O/ncu_gemm.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 20 -c 2 -o $O/prof_dec python tools/probe_step.py 16 700 2 2 > $O/ncu_dec.log 2>&1; tail -1 $O/ncu_dec.log
ls $O
