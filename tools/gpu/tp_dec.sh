O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
echo "== tp tests"; timeout 600 python -m pytest tests/test_tp.py -q -m gpu -x -s 2>&1 | tail -4
echo "== decode chunk target sweep"
for t in 64 128 296 592; do timeout 300 python tools/probe_decode.py $t 8x700 16x700 32x700 8x9000 2>&1 | grep target; done
echo "== steady-state launch list"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 40000 -c 3000 --csv --log-file $O/launches_steady.csv python bench.py --steps 300 --warmup 140 --profile-steps 0 --no-cpu-baseline > $O/ncu_launch2.log 2>&1
python tools/ncu_summary.py $O/launches_steady.csv > $O/launches_steady.txt; head -16 $O/launches_steady.txt
