O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python bench.py > $O/bench_final.log 2>&1; grep '^{' $O/bench_final.log | tail -1 | cut -c1-300
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 60 -c 4 -o $O/prof_gemm2 python tools/probe_step.py 16 700 2 2 > $O/ncu_gemm2.log 2>&1; tail -1 $O/ncu_gemm2.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 1200 -c 700 --csv --log-file $O/launches_iter2.csv python tools/probe_step.py 16 700 2 6 > /dev/null 2>&1
python tools/ncu_summary.py $O/launches_iter2.csv | tee $O/launches_iter2.txt | head -8
