python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for e in 0 1; do echo "no_small=$e"; if [ $e = 1 ]; then export HS_NO_SMALL=1; fi; timeout 300 python tools/probe_decode.py 296 1x9000 2x9000 1x2000 4x2000 2x700 8x700 16x700 8x2000 2>&1 | grep target; done
unset HS_NO_SMALL
timeout 600 python -m pytest tests/test_ops_gpu.py tests/test_serving.py -q -m gpu 2>&1 | tail -1
for a in "8 700 0" "16 700 0" "32 700 0"; do timeout 120 python tools/probe_step.py $a 30 2>&1 | grep "device-only"; done
