O=gpurun_out/rbench5; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
HS_CPU_HOST_TRACE=1 timeout 600 python bench.py --steps 3 --warmup 3 --remote-hosts 1 --no-cpu-baseline --sweep "" --profile-steps 0 > $O/bench_r1.log 2>&1
grep -c "hs cpu host: op" $O/bench_r1.log; grep -c "hs remote host: send" $O/bench_r1.log
grep "hs " $O/bench_r1.log | head -60 > $O/head.txt; grep "hs " $O/bench_r1.log | tail -40 > $O/tail.txt
