b() { env $1 TK_BENCH_WATCHDOG=150 timeout 180 python bench.py --steps 3 --warmup 3 --no-serving --no-decode --no-cpu-baseline > gpurun_out/b.log 2>&1
  python -c "
import json;l=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1])
print('$1', l['value'], l['kernels']['attention']['ms'], l['clocks']['sm_mhz'])" 2>&1 | tail -1; }
for r in 1 2; do for v in 0 2 9 10 11 1; do b TK_FA_VARIANT=$v; done; done
