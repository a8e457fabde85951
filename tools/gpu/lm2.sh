python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
HS_SKIP=511 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --launch-skip 400 -c 40 --csv --log-file gpurun_out/lm.csv python tools/probe_step.py 8 700 0 12 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/lm.csv
