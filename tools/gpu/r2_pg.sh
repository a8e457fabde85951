# device-polled merges: equivalence + live parity, then a bench in that mode
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
echo "== device merges"; timeout 900 python -m pytest tests/test_device_merges.py tests/test_live_parity.py tests/test_profiler.py -q -m gpu -p no:cacheprovider -s 2>&1 | grep -E "^E|passed|failed|merges|live:|accuracy|Error" | head -40
