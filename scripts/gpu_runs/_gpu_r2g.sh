timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity_scale.py -q -x -p no:cacheprovider > gpurun_out/pytest_cs8.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/pytest_cs8.log
for c in 1 0; do echo "CS8=$c"; TK_GEMM_CS8=$c TK_GEMM_DEBUG=1 timeout 200 python scripts/gemm_bench.py --shapes qkv fc1 2>&1 | tail -4; done
for c in 1 0 1 0; do
  TK_GEMM_CS8=$c TK_BENCH_WATCHDOG=150 timeout 180 python bench.py --steps 3 --warmup 3 --no-serving --no-decode --no-cpu-baseline > gpurun_out/bench_cs$c.log 2>&1
  python -c "
import json;l=json.loads(open('gpurun_out/bench_cs$c.log').read().strip().splitlines()[-1])
print('cs8=$c', l['value'], l['roofline']['frac'], {k: v['ms'] for k,v in l['kernels'].items()}, l['clocks']['sm_mhz'])" 2>&1 | tail -1
done
