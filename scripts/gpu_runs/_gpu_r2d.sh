timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity_scale.py -q -x -p no:cacheprovider > gpurun_out/pytest_w144.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/pytest_w144.log
for w in 1 0; do echo "W144=$w"; TK_GEMM_W144=$w TK_GEMM_DEBUG=1 timeout 300 python scripts/gemm_bench.py --shapes qkv o fc1 fc2 2>&1 | grep -v "^gemm M=" | tail -4; done
for w in 1 0 1 0; do
  TK_GEMM_W144=$w timeout 600 python bench.py --steps 4 --warmup 3 --no-serving --no-decode --no-cpu-baseline > gpurun_out/bench_w$w.log 2>&1
  python -c "
import json;l=json.loads(open('gpurun_out/bench_w$w.log').read().strip().splitlines()[-1])
print('w144=$w', l['value'], l['roofline']['frac'], {k: v['ms'] for k,v in l['kernels'].items()}, l['clocks']['sm_mhz'])"
done
