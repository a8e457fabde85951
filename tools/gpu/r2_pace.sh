O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
summ() { python - "$1" "$2" <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
print(sys.argv[2], {k: d.get(k) for k in ("value","be_prefill_tok_s","ls_tpot_attainment","ls_tpot_p99_ms","merges","be_tokens_via_cpu_attention","iteration_ms_p50","host_ms_per_iteration")}, (d.get("device_breakdown_ms") or {}).get("between_layers"))
PY
}
for a in "--pace 2 --pace-tail 12" "" ; do
  timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --sweep "" $a > $O/b.log 2>&1; summ $O/b.log "headline $a"; tail -3 $O/b.log | grep -iE "error|Trace"
done
timeout 1200 python bench.py --workload longctx --steps 20 --warmup 5 --no-cpu-baseline --sweep "" > $O/b.log 2>&1; summ $O/b.log "longctx"; tail -3 $O/b.log | grep -iE "error|Trace"
