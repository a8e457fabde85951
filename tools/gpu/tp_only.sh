# tensor-parallel two-process parity test, repeated
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for i in 1 2 3 4 5; do timeout 900 python -m pytest tests/test_tp.py -q -m gpu 2>&1 | grep -E "^E  |passed|failed" | head -6; done
