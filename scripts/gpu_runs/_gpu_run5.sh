timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py tests/test_gpu_parity_scale.py -q -p no:cacheprovider > gpurun_out/pytest_attn.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_attn.log
for ks in 2 1; do echo "KS=$ks"; TK_GEMM_KS=$ks timeout 300 python scripts/gemm_bench.py --shapes o fc2 --iters 30 2>&1 | tail -3; done
for v in 1 0; do
  TK_FA_COMBINE=$v timeout 600 python bench.py --steps 4 --warmup 3 --no-serving --no-decode --no-cpu-baseline > gpurun_out/bench_fa_$v.log 2>&1
  python -c "
import json,sys;l=json.loads(open('gpurun_out/bench_fa_$v.log').read().strip().splitlines()[-1])
print('combine=$v', l['value'], l['kernels']['attention'], l['share_of_step']['attention'], l['clocks']['sm_mhz'])"
done
TK_GEMM_KS=1 timeout 600 python bench.py --steps 4 --warmup 3 --no-serving --no-decode --no-cpu-baseline > gpurun_out/bench_ks1.log 2>&1
python -c "
import json,sys;l=json.loads(open('gpurun_out/bench_ks1.log').read().strip().splitlines()[-1])
print('ks1', l['value'], l['kernels']['o_gemm'], l['kernels']['fc2_gemm'], l['clocks']['sm_mhz'])"
