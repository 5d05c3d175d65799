# CPU arms through all 40 layers: reference arm (defaults) and the product arm's cpu_baseline.
set -x
t0=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err
echo "ref rc=$? wall $(( $(date +%s) - t0 )) s"; tail -1 gpurun_out/bench_ref.log | cut -c1-900
t0=$(date +%s); timeout 900 python bench.py --no-serving --no-decode > gpurun_out/bench_cpu.log 2> gpurun_out/bench_cpu.err
echo "bench rc=$? wall $(( $(date +%s) - t0 )) s"; tail -1 gpurun_out/bench_cpu.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['cpu_baseline'])"
