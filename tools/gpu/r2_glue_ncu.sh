# ncu captures of the glue kernels at the bench's mean batch (29 rows)
O=gpurun_out/glue; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
for k in qkv_rope_scatter residual_add_norm silu_mul; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 40 -c 1 -o $O/ncu_$k python tools/probe_layer.py 29 > $O/ncu_$k.log 2>&1; tail -1 $O/ncu_$k.log
done
