# bench (driver-style), reference arm, live parity tests
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
echo "== live parity"; timeout 600 python -m pytest tests/test_live_parity.py -q -m gpu -p no:cacheprovider 2>&1 | tail -3
echo "== bench 20/5"; timeout 900 python bench.py --steps 20 --warmup 5 --write-batch > $O/bench_20.log 2>&1; tail -c 5000 $O/bench_20.log
cp profiles/bench_batch.json $O/ 2>/dev/null
echo "== reference 20/5"; timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.log 2>&1; tail -c 3000 $O/bench_ref.log
