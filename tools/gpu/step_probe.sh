python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/probe_gemm_fused.py 8 32 2>&1
for a in "8 700 0" "32 700 0"; do for f in 0 1 4 5; do printf "fused %d " $f; HS_FUSED=$f timeout 120 python tools/probe_step.py $a 30 2>&1 | grep "device-only\|rror"; done; done
