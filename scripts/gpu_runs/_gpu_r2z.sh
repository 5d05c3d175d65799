timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py -q -x -p no:cacheprovider > gpurun_out/p.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/p.log
b() { env $1 TK_BENCH_WATCHDOG=150 timeout 180 python bench.py --steps 3 --warmup 3 --no-serving --no-decode --no-cpu-baseline > gpurun_out/b.log 2>&1
  python -c "
import json;l=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1])
print('$1', l['value'], l['kernels']['other'], l['clocks']['sm_mhz'])" 2>&1 | tail -1; }
for r in 1 2; do b TK_X=1; done
