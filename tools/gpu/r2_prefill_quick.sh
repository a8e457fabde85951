O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
echo "== prefill ops parity"; timeout 300 python -m pytest tests/test_ops_gpu.py -q -m gpu -k "prefill" -p no:cacheprovider 2>&1 | grep -E "^E|passed|failed|Error" | head -20
echo "== probe tcgen05"; timeout 300 python tools/probe_prefill.py 2>&1 | tail -8
