python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for a in "8 700 0" "32 700 0" "16 2000 0" "8 700 4"; do timeout 300 python tools/probe_step.py $a 30 2>&1 | grep "device"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 400 --csv --log-file gpurun_out/step_launches.csv python tools/probe_step.py 8 700 2 4 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/step_launches.csv
