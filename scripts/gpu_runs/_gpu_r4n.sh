# Double-buffered-S chunk attention (TK_FA_DB=1): parity + isolated A/B.
set -x
TK_FA_DB=1 timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -p no:cacheprovider -k "attention and not cta_pair" > gpurun_out/pytest_db.log 2>&1
echo "pytest db rc=$?"; tail -3 gpurun_out/pytest_db.log | cut -c1-300
for v in 0 1; do
TK_FA_DB=$v timeout 300 python scripts/attn_bench.py --prefix 0 2048 4096 7680 > gpurun_out/attn_db$v.log 2>&1
echo "attn db=$v rc=$?"; tail -4 gpurun_out/attn_db$v.log | cut -c1-140
done
