# compute-sanitizer evidence: memcheck / racecheck / synccheck on the attention
# kernels (incl. the tcgen05 prefill) and memcheck on the device-polled merge
# path (controller kernel, padding rows, work ring) end to end (tiny model)
O=gpurun_out/sanitize; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  echo "== $tool: attention ops"
  timeout 900 $CS --tool $tool --print-limit 20 python -m pytest tests/test_ops_gpu.py -m gpu -q -p no:cacheprovider -k "prefill_attention_causal and 32-8 or decode_attention_fused" > $O/$tool.ops.log 2>&1
  grep -E "ERROR SUMMARY|passed|failed" $O/$tool.ops.log | tail -3
done
echo "== memcheck: device-polled merges (equivalence test)"
timeout 1500 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_device_merges.py -m gpu -q -p no:cacheprovider > $O/memcheck.pg.log 2>&1
grep -E "ERROR SUMMARY|passed|failed" $O/memcheck.pg.log | tail -3
