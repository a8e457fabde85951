#!/bin/bash
# One GPU session: tests, smoke, calibration, bench, ncu launch list + captures.
# Outputs land in gpurun_out/ (merged back by gpurun).
set -u
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
echo "== pytest -m gpu"; timeout 900 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
if [ "${CALIBRATE:-0}" = "1" ]; then
  echo "== calibrate"; timeout 600 python bench.py --calibrate --calibrate-out $O/b200_llama3-8b_models.json --steps 8 --warmup 4 --no-cpu-baseline > $O/calibrate.log 2>&1; tail -c 400 $O/calibrate.log
  cp $O/b200_llama3-8b_models.json profiles/ 2>/dev/null
fi
echo "== bench"; timeout 900 python bench.py ${BENCH_ARGS:-} > $O/bench.log 2>&1; tail -c 2500 $O/bench.log
if [ "${NCU:-1}" = "1" ]; then
  echo "== ncu launch list"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches.csv python bench.py --steps 4 --warmup 2 --be-chains 32 --ls-rate 0 --ls-decodes 8 --no-cpu-baseline > $O/ncu_launch.log 2>&1; tail -2 $O/ncu_launch.log
  echo "== ncu full gemm"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 140 -c 4 -o $O/prof_gemm python bench.py --steps 2 --warmup 1 --be-chains 32 --ls-rate 0 --ls-decodes 8 --no-cpu-baseline > $O/ncu_gemm.log 2>&1; tail -2 $O/ncu_gemm.log
  echo "== ncu full decode attn"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 40 -c 2 -o $O/prof_dec python bench.py --steps 2 --warmup 1 --be-chains 32 --ls-rate 0 --ls-decodes 8 --no-cpu-baseline > $O/ncu_dec.log 2>&1; tail -2 $O/ncu_dec.log
fi
ls -la $O
