# Split-softmax chunk attention (TK_FA_SPLIT=1, 16 softmax warps): parity + isolated A/B.
set -x
TK_FA_SPLIT=1 timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -p no:cacheprovider -k "attention and not cta_pair" > gpurun_out/pytest_split.log 2>&1
echo "pytest split rc=$?"; tail -15 gpurun_out/pytest_split.log | cut -c1-300
for v in 0 1; do
TK_FA_SPLIT=$v timeout 300 python scripts/attn_bench.py --prefix 0 2048 4096 7680 > gpurun_out/attn_split$v.log 2>&1
echo "attn split=$v rc=$?"; tail -4 gpurun_out/attn_split$v.log | cut -c1-140
done
