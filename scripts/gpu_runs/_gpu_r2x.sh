b() { env $1 TK_BENCH_WATCHDOG=150 timeout 180 python bench.py --steps 3 --warmup 3 --no-serving --no-decode --no-cpu-baseline > gpurun_out/b.log 2>&1
  python -c "
import json;l=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1])
print('$1', l['value'], {k: round(v['ms']/3,1) for k,v in l['kernels'].items()}, l['kernels']['other']['launches'], l['clocks']['sm_mhz'])" 2>&1 | tail -1; }
for r in 1 2; do b TK_X=1; b TK_NO_FUSED_KV=1; done
