for st in 4 5 6; do
  export HS_NVCC_DEFS="-DHS_GEMM_ST16=$st -DHS_GEMM_ST32=4"
  python -m paper_2603_12831_b200._build --force > /dev/null 2>&1 || { echo "build failed"; continue; }
  for wg in 0 1; do
    for a in "8 700 0" "16 700 2"; do printf "st16=$st wg=$wg $a "; HS_DEC_WG=$wg timeout 120 python tools/probe_step.py $a 30 2>&1 | grep -o "device-only.*"; done
  done
done
