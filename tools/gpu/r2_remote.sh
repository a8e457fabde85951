# remote CPU hosts: GPU tests
O=gpurun_out/remote; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
echo "== remote tests"; timeout 900 python -m pytest tests/test_remote_host.py -q -s -p no:cacheprovider ${PYTEST_ARGS:-} > $O/pytest_remote.log 2>&1; tail -15 $O/pytest_remote.log; grep -n "hs " $O/pytest_remote.log | head
