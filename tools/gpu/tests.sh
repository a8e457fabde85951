# GPU tests + smoke only
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
echo "== pytest -m gpu"; timeout 1500 python -m pytest tests -q -m gpu -x ${PYTEST_ARGS:-} > $O/pytest_gpu.log 2>&1; tail -5 $O/pytest_gpu.log
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
