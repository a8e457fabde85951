# decode attention: one vs two warp groups (HS_DEC_WG), parity tests first
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_ops_gpu.py tests/test_serving.py -q -m gpu -x 2>&1 | tail -1
HS_DEC_WG=2 timeout 600 python -m pytest tests/test_ops_gpu.py -q -m gpu -x -k decode 2>&1 | tail -1
HS_DEC_WG=1 timeout 600 python -m pytest tests/test_ops_gpu.py -q -m gpu -x -k decode 2>&1 | tail -1
for w in 1 2; do echo "WG=$w"; HS_DEC_WG=$w timeout 300 python tools/probe_decode.py 296 2x700 8x700 16x700 1x9000 2x9000 2>&1 | grep target; done
for a in "8 700 0" "16 700 2" "32 700 0"; do timeout 120 python tools/probe_step.py $a 30 2>&1 | grep "device-only"; done
