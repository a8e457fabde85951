python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -c 300 gpurun_out/bench.log; echo
for a in "8 700 0" "32 700 0"; do timeout 300 python tools/probe_step.py $a 20 llama3-70b-tp8 2>&1 | grep "device"; done
