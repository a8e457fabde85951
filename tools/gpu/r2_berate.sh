O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
for r in 0 0.25 0.5 1.0; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --sweep "" --profile-steps 0 --be-rate $r > $O/bench_be$r.log 2>&1
  python - $O/bench_be$r.log <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
print(sys.argv[1], {k: d.get(k) for k in ("value","e2e","be_prefill_tok_s","ls_tpot_attainment","ls_tpot_p99_ms","merges","be_tokens_via_cpu_attention","iteration_ms_p50","avg_batch_tokens")})
PY
  tail -3 $O/bench_be$r.log | grep -i error
done
