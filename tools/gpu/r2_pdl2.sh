# PDL early release + fewer GEMM stages (so the next GEMM's CTAs co-reside and prefetch)
O=gpurun_out/pdl2; mkdir -p $O
for defs in "-DHS_PDL_EARLY=1 -DHS_GEMM_ST16=3 -DHS_GEMM_ST32=3" "-DHS_PDL_EARLY=0 -DHS_GEMM_ST16=3 -DHS_GEMM_ST32=3" "-DHS_PDL_EARLY=1 -DHS_GEMM_ST16=2 -DHS_GEMM_ST32=2" "-DHS_PDL_EARLY=1 -DHS_GEMM_ST16=4 -DHS_GEMM_ST32=4"; do
  rm -f build/libhs/*.o
  HS_NVCC_DEFS="$defs" python -c "from paper_2603_12831_b200 import _build; _build.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
  echo "== $defs"
  timeout 300 python tools/probe_layer.py 8 16 29 > $O/probe.txt 2>&1; cat $O/probe.txt
done
