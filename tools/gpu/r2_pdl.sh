# PDL: glue / decode-attention kernels release their dependents before their own wait (A/B)
O=gpurun_out/pdl; mkdir -p $O
for v in 0 1; do
  rm -f build/libhs/elementwise.cu.o build/libhs/attn_decode.cu.o
  HS_NVCC_DEFS="-DHS_PDL_EARLY=$v" python -c "from paper_2603_12831_b200 import _build; _build.build()" > $O/build_$v.log 2>&1 || { tail -20 $O/build_$v.log; exit 1; }
  echo "== early=$v"
  timeout 300 python tools/probe_layer.py 8 29 64 > $O/probe_layer_$v.txt 2>&1; cat $O/probe_layer_$v.txt
  timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --sweep "" > $O/bench_$v.log 2>&1; grep '^{' $O/bench_$v.log | tail -1 > $O/bench_$v.json
  python -c "import json;d=json.load(open('$O/bench_$v.json'));print({k:d.get(k) for k in ('value','ls_tpot_attainment','iteration_ms_p50','host_ms_per_iteration')}, d['roofline']['frac'], d['device_breakdown_ms'])"
done
echo "== tests (early=1)"
timeout 1800 python -m pytest tests/test_ops_gpu.py tests/test_serving.py tests/test_serving_8b.py tests/test_live_parity.py -q -p no:cacheprovider > $O/pytest.log 2>&1; tail -2 $O/pytest.log
