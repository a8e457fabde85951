O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
echo "== prefill ops parity"; timeout 600 python -m pytest tests/test_ops_gpu.py -q -m gpu -k "prefill" -p no:cacheprovider 2>&1 | grep -E "^E|passed|failed|Error" | head -20
echo "== probe tcgen05"; timeout 300 python tools/probe_prefill.py 2>&1 | tail -8
echo "== probe warp-mma"; HS_PREFILL_MMA=1 timeout 300 python tools/probe_prefill.py 2>&1 | tail -8
echo "== serving"; timeout 900 python -m pytest tests/test_serving.py tests/test_serving_8b.py tests/test_fp32_mode.py -q -m gpu -p no:cacheprovider 2>&1 | grep -E "^E|passed|failed|Error" | head -20
