timeout 90 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "chunk_attention_mixed" > gpurun_out/pytest_fa64a.log 2>&1
echo "pytest mixed rc=$?"; tail -3 gpurun_out/pytest_fa64a.log
timeout 120 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "chunk_attention" > gpurun_out/pytest_fa64.log 2>&1
echo "pytest kernels rc=$?"; tail -3 gpurun_out/pytest_fa64.log
timeout 300 python -m pytest tests/test_gpu_model.py tests/test_gpu_parity_scale.py -q -x -p no:cacheprovider > gpurun_out/pytest_fa64m.log 2>&1
echo "pytest model rc=$?"; tail -3 gpurun_out/pytest_fa64m.log
for v in 0 12; do echo "variant=$v"; TK_FA_VARIANT=$v timeout 120 python scripts/attn_bench.py --prefix 0 512 2048 4096 7680 2>&1 | tail -5; done
for v in 0 12 0 12; do
  TK_FA_VARIANT=$v TK_BENCH_WATCHDOG=150 timeout 180 python bench.py --steps 3 --warmup 3 --no-serving --no-decode --no-cpu-baseline > gpurun_out/bench_fa$v.log 2>&1
  python -c "
import json;l=json.loads(open('gpurun_out/bench_fa$v.log').read().strip().splitlines()[-1])
print('fa=$v', l['value'], l['kernels']['attention'], l['share_of_step']['attention'], l['clocks']['sm_mhz'])" 2>&1 | tail -1
done
