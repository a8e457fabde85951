python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
free -g | head -2
for a in "8 700 0 20 llama2-13b" "32 700 4 20 llama2-13b"; do timeout 300 python tools/probe_step.py $a 2>&1 | grep "device"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 1200 -c 700 --csv --log-file gpurun_out/launches_iter.csv python tools/probe_step.py 16 700 2 6 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/launches_iter.csv | tee gpurun_out/launches_iter.txt | head -20
