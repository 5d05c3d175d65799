timeout 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "gemm" > gpurun_out/pytest_gemm.log 2>&1
echo "pytest gemm rc=$?"; tail -3 gpurun_out/pytest_gemm.log
timeout 300 python scripts/gemm_bench.py --shapes qkv o fc1 fc2 --iters 30 2>&1 | tail -4
for s in fc2 o qkv; do echo "trace $s"; timeout 300 python scripts/gemm_trace.py --shape $s 2>&1 | head -1 | cut -c1-300; done
for v in 1 0; do echo "combine=$v"; TK_FA_COMBINE=$v timeout 300 python scripts/attn_bench.py --prefix 0 2048 7680 2>&1 | tail -3; done
timeout 600 python bench.py --steps 4 --warmup 3 --no-serving --no-decode --no-cpu-baseline > gpurun_out/bench_g.log 2>&1
python -c "
import json,sys;l=json.loads(open('gpurun_out/bench_g.log').read().strip().splitlines()[-1])
print('bench', l['value'], l['roofline']['frac'], {k: v['ms'] for k,v in l['kernels'].items()}, l['clocks']['sm_mhz'])"
