# round-2 evidence: profiler accuracy, steady-state launch list, PCIe counters
# of the piggyback kernels, decode-attention and large-batch GEMM captures
O=gpurun_out/prof_r2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
echo "== profiler"; timeout 600 python -m pytest tests/test_profiler.py -q -m gpu -s -p no:cacheprovider 2>&1 | grep -E "accuracy|passed|failed|^E" | head
echo "== launch list (bench steady state)"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 30000 -c 3000 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --profile-steps 0 --no-cpu-baseline --sweep "" > $O/ncu_launch.log 2>&1
python tools/ncu_summary.py $O/launches_bench.csv > $O/launches_bench.txt; head -20 $O/launches_bench.txt
echo "== PCIe counters (RoPE/ship + result gather launches, 16 decodes + 16 merges + 16 carries)"
timeout 600 ncu --metrics gpu__time_duration.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:qkv_rope -s 64 -c 16 --csv --log-file $O/pcie_rope.csv python tools/probe_step.py 16 700 16 4 > $O/ncu_pcie.log 2>&1; tail -3 $O/pcie_rope.csv
echo "== decode attention (16 x 700)"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 40 -c 1 -o $O/ncu_decode_16x700 python tools/probe_step.py 16 700 2 2 > $O/ncu_dec.log 2>&1; tail -1 $O/ncu_dec.log
echo "== GEMM at 512 rows"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 40 -c 4 -o $O/ncu_gemm_512 python tools/probe_step.py 512 64 0 2 > $O/ncu_gemm.log 2>&1; tail -1 $O/ncu_gemm.log
ls -la $O
