# shared-memory stage counts (decode attention / GEMM) under PDL co-residency
# stage-count sweep: decode-attention smem vs GEMM co-residency under PDL
for v in "3 6 5" "2 6 5" "2 4 4" "3 4 4" "2 5 4" "2 4 3"; do
  set -- $v
  export HS_NVCC_DEFS="-DHS_DEC_STAGES=$1 -DHS_GEMM_ST16=$2 -DHS_GEMM_ST32=$3"
  python -m paper_2603_12831_b200._build --force > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  echo "== dec $1 g16 $2 g32 $3"
  for a in "8 700 0" "32 700 0" "16 2000 0" "4 9000 0"; do timeout 300 python tools/probe_step.py $a 30 2>&1 | grep "device-only"; done
done
