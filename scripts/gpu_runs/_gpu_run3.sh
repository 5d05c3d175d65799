timeout 600 python -m pytest tests/test_gpu_multi.py tests/test_gpu_executor.py -q -p no:cacheprovider > gpurun_out/pytest_multi.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/pytest_multi.log
for impl in cta warp cta warp; do
  TK_NORM_IMPL=$impl timeout 600 python bench.py --steps 4 --warmup 3 --no-serving --no-decode --no-cpu-baseline > gpurun_out/bench_norm_$impl.log 2>&1
  python -c "
import json,sys;l=json.loads(open('gpurun_out/bench_norm_$impl.log').read().strip().splitlines()[-1])
print('$impl', l['value'], l['kernels']['other'], l['share_of_step']['other'], l['clocks']['sm_mhz'])"
done
