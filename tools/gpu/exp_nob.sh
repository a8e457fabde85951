python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_ops_gpu.py tests/test_serving.py -q -m gpu -x 2>&1 | tail -1
timeout 300 python tools/probe_layer.py 512 256 128 32 16 2>&1 | grep -o "n=.*gemms *[0-9.]*"
for a in "8 700 0" "32 700 0"; do timeout 120 python tools/probe_step.py $a 30 2>&1 | grep "device-only"; done
