timeout 180 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "gemm" > gpurun_out/p1.log 2>&1
echo "gemm tests rc=$?"; tail -3 gpurun_out/p1.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest gpu rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for cfg in "32 2048" "128 512" "8 512"; do set -- $cfg; timeout 300 python scripts/decode_bench.py --batch $1 --ctx $2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['batch'], d['ctx'], d['step_ms'], d['tok_s'])"; done
TK_BENCH_WATCHDOG=150 timeout 180 python bench.py --steps 3 --warmup 3 --no-serving --no-decode --no-cpu-baseline > gpurun_out/b.log 2>&1
python -c "
import json;l=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1])
print(l['value'], {k: round(v['ms']/3,1) for k,v in l['kernels'].items()}, l['clocks']['sm_mhz'])"
