# C1 host attention pool: software prefetch distance x AMX on/off
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for pf in 0 2 4 8; do for a in 1 0; do echo "pf=$pf amx=$a"; HS_CPU_PF=$pf HS_CPU_AMX=$a timeout 300 python tools/probe_cpu_attn.py 9000 32 14 2>&1 | tail -1; done; done
HS_CPU_PF=4 timeout 300 python tools/probe_cpu_attn.py 9000 32 1 2>&1 | tail -1
