# recalibrate the latency models on the final kernels (K6 at 0.54 of peak, early PDL release),
# then the driver-style bench and config 5 on them
O=gpurun_out/recal; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
cp profiles/b200_llama3-8b_models.json $O/models_before.json
timeout 900 python bench.py --calibrate --calibrate-out $O/b200_llama3-8b_models.json --steps 20 --warmup 5 --no-cpu-baseline --sweep "" > $O/calib.log 2>&1; grep "dense\|attn" $O/calib.log | head -5
cp $O/b200_llama3-8b_models.json profiles/b200_llama3-8b_models.json
echo "== bench 20/5 (new models)"; timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_20.log 2>&1; grep '^{' $O/bench_20.log | tail -1 > $O/bench_20.json; python -c "import json;d=json.load(open('$O/bench_20.json'));print({k:d.get(k) for k in ('value','ls_tpot_attainment','ls_tpot_p99_ms','iteration_ms_p50','max_be_tok_s_at_slo')}, d['roofline']['frac'])"
echo "== longctx (new models)"; timeout 1200 python bench.py --workload longctx --steps 20 --warmup 5 --no-cpu-baseline --sweep "" > $O/bench_longctx.log 2>&1; grep '^{' $O/bench_longctx.log | tail -1 > $O/bench_longctx.json; python -c "import json;d=json.load(open('$O/bench_longctx.json'));print({k:d.get(k) for k in ('value','be_prefill_tok_s','ls_tpot_attainment','ls_tpot_p99_ms','iteration_ms_p50')})"
