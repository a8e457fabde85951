# K6: share the softmax exponentials between MUFU.EX2 and an FMA-pipe polynomial
O=gpurun_out/k6poly; mkdir -p $O
for v in 0 1 3 2; do
  rm -f build/libhs/attn_prefill_tc.cu.o
  HS_NVCC_DEFS="-DHS_K6_POLY=$v" python -c "from paper_2603_12831_b200 import _build; _build.build()" > $O/build_$v.log 2>&1 || { tail -20 $O/build_$v.log; exit 1; }
  timeout 300 python tools/probe_prefill.py > $O/probe_$v.jsonl 2>&1; echo "poly=$v"; tail -3 $O/probe_$v.jsonl
done
timeout 900 python -m pytest tests/test_ops_gpu.py -q -p no:cacheprovider -k prefill > $O/pytest_prefill.log 2>&1; echo "prefill tests: $(tail -1 $O/pytest_prefill.log)"
timeout 900 python -m pytest tests/test_serving.py tests/test_serving_8b.py -q -p no:cacheprovider > $O/pytest_serving.log 2>&1; echo "serving tests: $(tail -1 $O/pytest_serving.log)"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_attn_tc -s 74 -c 1 -o $O/ncu_prefill_tc_32k_poly2 python tools/probe_prefill.py > $O/ncu.log 2>&1; tail -1 $O/ncu.log
