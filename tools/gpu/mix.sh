python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_ops_gpu.py tests/test_serving.py -q -m gpu -x 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for a in "8 700 0 30" "32 700 4 30" "128 64 0 10" "512 64 0 6"; do timeout 120 python tools/probe_step.py $a 2>&1 | grep -o "device-only.*"; done
