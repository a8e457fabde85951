python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for pt in 0 12; do
  timeout 600 python bench.py --steps 400 --warmup 64 --profile-steps 0 --no-cpu-baseline --pace-tail $pt > gpurun_out/bench_pt$pt.log 2>&1
  python - "$pt" <<'P'
import json, sys
l = [x for x in open(f"gpurun_out/bench_pt{sys.argv[1]}.log") if x.startswith("{")]
if not l: print("no line", sys.argv[1]); sys.exit()
d = json.loads(l[-1])
print("pace_tail", sys.argv[1], "value %.1f" % d["value"], "ms/step %.3f" % d["ms_per_step"], "p50 %.3f" % d["iteration_ms_p50"], "attain %.4f" % d["ls_tpot_attainment"], "p99 %.1f" % d["ls_tpot_p99_ms"], "merges", d["merges"], "cpu_tok", d["be_tokens_via_cpu_attention"], "rows %.1f" % d["avg_batch_tokens"], "roof %.3f" % d["roofline"]["frac"], {k: round(v, 3) for k, v in d["host_ms_per_step"].items()})
P
done
