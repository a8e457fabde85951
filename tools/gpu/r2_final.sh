# round-2 record: full GPU suite, smoke, bench lines (default, driver-style,
# reference arm, config 5), launch list and K6 capture
O=gpurun_out/final; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/gpu.txt
echo "== pytest -m gpu"; timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
echo "== bench default"; timeout 1200 python bench.py > $O/bench_default.log 2>&1; grep '^{' $O/bench_default.log | tail -1 > $O/bench_default.json; python -c "import json;d=json.load(open('$O/bench_default.json'));print({k:d.get(k) for k in ('value','ls_tpot_attainment','ls_tpot_p99_ms','max_be_tok_s_at_slo','iteration_ms_p50')})"
echo "== bench 20/5"; timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_20.log 2>&1; grep '^{' $O/bench_20.log | tail -1 > $O/bench_20.json; python -c "import json;d=json.load(open('$O/bench_20.json'));print({k:d.get(k) for k in ('value','ls_tpot_attainment','ls_tpot_p99_ms','iteration_ms_p50')})"
echo "== reference 20/5"; timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.log 2>&1; grep '^{' $O/bench_ref.log | tail -1 > $O/bench_ref.json; python -c "import json;d=json.load(open('$O/bench_ref.json'));print({k:d.get(k) for k in ('value','ms_per_step')})"
echo "== longctx"; timeout 1200 python bench.py --workload longctx --steps 20 --warmup 5 --no-cpu-baseline --sweep "" > $O/bench_longctx.log 2>&1; grep '^{' $O/bench_longctx.log | tail -1 > $O/bench_longctx.json
echo "== launch list (whole iterations, 8 LS decodes x 700 + 2 merges/layer)"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_8x700_m2.csv python tools/probe_step.py 8 700 2 6 > $O/ncu_launch.log 2>&1
python tools/ncu_summary.py $O/launches_8x700_m2.csv > $O/launches_8x700_m2.txt; head -16 $O/launches_8x700_m2.txt
echo "== kernel probes"
timeout 300 python tools/probe_prefill.py > $O/probe_prefill.jsonl 2>&1; tail -1 $O/probe_prefill.jsonl
timeout 300 python tools/probe_decode.py > $O/probe_decode.jsonl 2>&1; grep '"g": 8, "ctx": 700' $O/probe_decode.jsonl | head -1
timeout 300 python tools/probe_gemm_pair.py 256 512 1024 > $O/probe_gemm_pair.jsonl 2>&1; tail -2 $O/probe_gemm_pair.jsonl
echo "== K6 capture (1024-token chunk after 31744)"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prefill_attn_tc -s 74 -c 1 -o $O/ncu_prefill_tc_32k python tools/probe_prefill.py > $O/ncu_prefill.log 2>&1; tail -1 $O/ncu_prefill.log
ls $O
