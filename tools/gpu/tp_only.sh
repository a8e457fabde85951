python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_tp.py -q -m gpu -s 2>&1 | grep -E "Error|error|assert|tp2|passed|failed" | head -20
