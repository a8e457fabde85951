# remote CPU hosts: the remote tests, the live ones repeated (the host crash
# was a ThreadPool race), then the per-layer in-stream split for the glue work
O=gpurun_out/remote; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 600 python -m pytest tests/test_remote_host.py -q -s -p no:cacheprovider > $O/pytest_remote.log 2>&1; echo "full: $(tail -1 $O/pytest_remote.log)"
for i in 1 2 3 4; do
  timeout 300 python -m pytest tests/test_remote_host.py -q -s -p no:cacheprovider -k "live_engine_with_remote_hosts" > $O/loop_$i.log 2>&1
  echo "run $i: $(tail -1 $O/loop_$i.log)"; grep -n "hs \|(+0x" $O/loop_$i.log | head -10
done
echo "== probe_layer"; timeout 300 python tools/probe_layer.py 8 16 29 64 > $O/probe_layer.txt 2>&1; cat $O/probe_layer.txt
