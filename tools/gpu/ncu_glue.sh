python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for k in residual_add_norm_kernel qkv_rope_scatter_kernel decode_attn_kernel; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 200 -c 2 -o gpurun_out/prof_$k python tools/probe_step.py 8 700 2 3 > /dev/null 2>&1
done
ls gpurun_out
