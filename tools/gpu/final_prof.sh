# end-of-round record: bench, reference arm, steady-state ncu launch list
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
echo "== bench"; timeout 1200 python bench.py > $O/bench_final.log 2>&1; tail -c 400 $O/bench_final.log; echo
echo "== bench reference arm"; timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.log 2>&1; tail -c 300 $O/bench_ref.log; echo
echo "== steady-state launch list"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 60000 -c 3000 --csv --log-file $O/launches_steady.csv python bench.py --steps 400 --warmup 220 --profile-steps 0 --no-cpu-baseline > $O/ncu_launch2.log 2>&1
python tools/ncu_summary.py $O/launches_steady.csv > $O/launches_steady.txt; head -16 $O/launches_steady.txt
