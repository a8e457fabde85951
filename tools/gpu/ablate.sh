# per-kernel in-stream cost by ablation (HS_SKIP) on whole iterations (tools/probe_step.py)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for a in "8 700 0" "32 700 0"; do
  for m in 0 1 2 4 8 16 29 31 32 64 128 256 480 511; do
    printf "skip %3d  " $m; HS_SKIP=$m timeout 300 python tools/probe_step.py $a 30 2>&1 | grep "device-only"
  done
done
