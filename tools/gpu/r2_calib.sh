O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python bench.py --calibrate --calibrate-out $O/b200_llama3-8b_models.json --steps 1 --warmup 1 --no-cpu-baseline --sweep "" --profile-steps 0 > $O/calib.log 2>&1
grep -E "dense|decode attn" $O/calib.log | tail -3
cp $O/b200_llama3-8b_models.json profiles/b200_llama3-8b_models.json
timeout 1200 python bench.py --workload longctx --steps 20 --warmup 5 --no-cpu-baseline --sweep "" --profile-steps 0 > $O/b.log 2>&1
python - $O/b.log <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
print({k: d.get(k) for k in ("value","be_prefill_tok_s","ls_tpot_attainment","ls_tpot_p99_ms","merges","be_tokens_via_cpu_attention","iteration_ms_p50","batch_tokens_p90")})
PY
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --sweep "" --profile-steps 0 > $O/b2.log 2>&1
python - $O/b2.log <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
print({k: d.get(k) for k in ("value","be_prefill_tok_s","ls_tpot_attainment","ls_tpot_p99_ms","merges","be_tokens_via_cpu_attention","iteration_ms_p50","batch_tokens_p90")})
PY
