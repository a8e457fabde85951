python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:gemm_bf16 -s 4 -c 4 -o gpurun_out/prof_gemm512 python tools/probe_layer.py 512 > gpurun_out/ncu_big.log 2>&1
tail -2 gpurun_out/ncu_big.log
