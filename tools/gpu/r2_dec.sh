O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
echo "== decode ops"; timeout 600 python -m pytest tests/test_ops_gpu.py -q -m gpu -k "decode" -p no:cacheprovider 2>&1 | grep -E "^E|passed|failed" | head
echo "== probe decode"; timeout 300 python tools/probe_decode.py 296 2x700 8x700 16x700 32x700 1x9000 8x9000 2>&1 | grep -iE "target|us" | head -20
echo "== longctx"; timeout 1200 python bench.py --workload longctx --steps 20 --warmup 5 --no-cpu-baseline --sweep "" --profile-steps 0 > $O/bench_longctx.log 2>&1
python - $O/bench_longctx.log <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
print({k: d.get(k) for k in ("value","be_prefill_tok_s","ls_tpot_attainment","ls_tpot_p99_ms","merges","be_tokens_via_cpu_attention","iteration_ms_p50","batch")})
PY
tail -3 $O/bench_longctx.log | grep -iE "error|Trace"
