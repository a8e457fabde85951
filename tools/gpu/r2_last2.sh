# stream-ordered tag retract at host-KV release: full GPU suite, live remote loop, smoke
O=gpurun_out/last2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
echo "== pytest -m gpu"; timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
for i in 1 2 3 4; do
  timeout 300 python -m pytest tests/test_remote_host.py -q -s -p no:cacheprovider -m gpu -k live > $O/live_$i.log 2>&1
  echo "live $i: $(tail -1 $O/live_$i.log) $(grep -c IntegrityFault $O/live_$i.log)"
done
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
echo "== bench 20/5"; timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_20.log 2>&1; grep '^{' $O/bench_20.log | tail -1 > $O/bench_20.json; python -c "import json;d=json.load(open('$O/bench_20.json'));print({k:d.get(k) for k in ('value','ls_tpot_attainment','ls_tpot_p99_ms','iteration_ms_p50','max_be_tok_s_at_slo')}, d['roofline']['frac'])"
