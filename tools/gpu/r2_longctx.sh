O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 1200 python bench.py --workload longctx --steps 20 --warmup 5 --no-cpu-baseline --sweep "" > $O/bench_longctx.log 2>&1
python - $O/bench_longctx.log <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
print({k: d.get(k) for k in ("value","be_prefill_tok_s","ls_tpot_attainment","ls_tpot_p99_ms","merges","be_tokens_via_cpu_attention","iteration_ms_p50","avg_batch_tokens","warmup_iterations","cpu_pool_busy_frac")})
PY
tail -5 $O/bench_longctx.log | grep -iE "error|Trace" 
