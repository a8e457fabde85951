O=gpurun_out/rbench3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python bench.py --steps 10 --warmup 3 --remote-hosts 1 --no-cpu-baseline --sweep "" --profile-steps 0 > $O/bench_r1.log 2>&1
grep '^{' $O/bench_r1.log | tail -1 > $O/bench_r1.json
python -c "import json;d=json.load(open('$O/bench_r1.json'));print(d['value'], json.dumps(d['remote_hosts'],indent=0))" || tail -30 $O/bench_r1.log
