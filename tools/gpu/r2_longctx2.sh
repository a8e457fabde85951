O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
for a in "--be-chains 0 --be-rate 1.0" "--be-chains 2 --be-rate 0.5"; do
timeout 1200 python bench.py --workload longctx --steps 20 --warmup 5 --no-cpu-baseline --sweep "" --profile-steps 0 $a > $O/bench_longctx.log 2>&1
python - $O/bench_longctx.log "$a" <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
print(sys.argv[2], {k: d.get(k) for k in ("value","be_prefill_tok_s","ls_tpot_attainment","ls_tpot_p99_ms","merges","be_tokens_via_cpu_attention","iteration_ms_p50","batch")})
PY
tail -5 $O/bench_longctx.log | grep -iE "error|Trace"
done
