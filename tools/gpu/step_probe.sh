python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for mb in 0 16 32 64; do echo "HS_L2PF_MB=$mb"; for a in "8 700 0" "32 700 0" "8 700 4"; do HS_L2PF_MB=$mb timeout 300 python tools/probe_step.py $a 40 2>&1 | grep device; done; done
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
