# live remote tests repeated: streaming fetch (HEAD) vs the previous relay
O=gpurun_out/rab; mkdir -p $O
for v in head prev; do
  if [ $v = prev ]; then git show cd1caf3~1:paper_2603_12831_b200/csrc/cpu_remote.cpp > paper_2603_12831_b200/csrc/cpu_remote.cpp; fi
  python -c "import __graft_entry__ as g; g.build()" > $O/build_$v.log 2>&1 || { tail -20 $O/build_$v.log; exit 1; }
  for i in 1 2 3; do
    timeout 300 python -m pytest tests/test_remote_host.py -q -s -p no:cacheprovider -m gpu -k live > $O/${v}_$i.log 2>&1
    echo "$v $i: $(tail -1 $O/${v}_$i.log) $(grep -c IntegrityFault $O/${v}_$i.log)"
  done
done
