timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "layernorm or gemm_residual" > gpurun_out/pytest_norm.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_norm.log
for r in 1 2; do
  TK_BENCH_WATCHDOG=150 timeout 180 python bench.py --steps 3 --warmup 3 --no-serving --no-decode --no-cpu-baseline > gpurun_out/bench_n$r.log 2>&1
  python -c "
import json;l=json.loads(open('gpurun_out/bench_n$r.log').read().strip().splitlines()[-1])
print('run $r', l['value'], l['roofline']['frac'], {k: round(v['ms']/3,1) for k,v in l['kernels'].items()}, l['kernels']['other'], l['clocks']['sm_mhz'])" 2>&1 | tail -1
done
