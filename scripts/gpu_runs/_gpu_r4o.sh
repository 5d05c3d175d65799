# Final bench line of the session (default arguments).
set -x
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1
echo "bench rc=$?"
tail -1 gpurun_out/bench_final.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'], d['cpu_baseline'])"
