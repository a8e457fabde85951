python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for e in X=1 HS_EXP_NOZERO=1; do echo $e; env $e timeout 300 python tools/probe_layer.py 512 128 32 2>&1 | grep -o "n=.*gemms *[0-9.]*"; done
