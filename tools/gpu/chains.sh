python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for n in 16 32 64 96; do
  timeout 600 python bench.py --steps 800 --warmup 150 --profile-steps 0 --no-cpu-baseline --be-chains $n > gpurun_out/bc$n.log 2>&1
  python - "$n" <<'P'
import json, sys
l = [x for x in open(f"gpurun_out/bc{sys.argv[1]}.log") if x.startswith("{")]
d = json.loads(l[-1])
print("chains", sys.argv[1], "value %.1f" % d["value"], "ms %.2f p50 %.2f" % (d["ms_per_step"], d["iteration_ms_p50"]), "cpu_tok", d["be_tokens_via_cpu_attention"], "busy %.2f" % d["cpu_pool_busy_frac"], "merges", d["merges"], "attain %.4f p99 %.1f" % (d["ls_tpot_attainment"], d["ls_tpot_p99_ms"]))
P
done
