python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
HS_BLOCKED=1 timeout 600 python -m pytest tests/test_serving.py tests/test_ops_gpu.py -q -m gpu -x 2>&1 | tail -2
for a in "8 700 0" "32 700 0" "128 700 0"; do for b in 0 1; do printf "blocked %d " $b; HS_BLOCKED=$b timeout 120 python tools/probe_step.py $a 30 2>&1 | grep "device-only\|rror"; done; done
