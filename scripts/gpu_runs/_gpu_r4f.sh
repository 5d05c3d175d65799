# Chunk attention: second-half exponentials ordered behind the first P half's release
# (TK_FA_VARIANT=12) -- parity, isolated and in-situ A/B.
set -x
TK_FA_VARIANT=12 timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -p no:cacheprovider -k "attention" > gpurun_out/pytest_attn12.log 2>&1
echo "pytest v12 rc=$?"; tail -3 gpurun_out/pytest_attn12.log
for v in 0 12 0 12; do
TK_FA_VARIANT=$v timeout 300 python scripts/attn_bench.py --prefix 0 2048 4096 7680 > gpurun_out/attn_v$v.log 2>&1
echo "attn v$v rc=$?"; tail -4 gpurun_out/attn_v$v.log | cut -c1-100
done
for v in 0 12 0 12; do
TK_FA_VARIANT=$v timeout 600 python bench.py --no-serving --no-decode --no-cpu-baseline > gpurun_out/bench_v$v.log 2>&1
echo "bench v$v rc=$?"
tail -1 gpurun_out/bench_v$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['kernels']['attention'], d['clocks']['sm_mhz'])"
done
