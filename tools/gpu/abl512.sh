python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for m in 0 1 2 4 8 16 480 511; do printf "skip %3d  " $m; HS_SKIP=$m timeout 200 python tools/probe_step.py 512 64 0 6 2>&1 | grep -o "device-only.*"; done
