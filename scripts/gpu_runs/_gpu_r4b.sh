# CTA-pair chunk attention: first light (microbench both kernels, kernel parity tests).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
TK_FA_PAIR=0 timeout 300 python scripts/attn_bench.py --prefix 0 512 2048 4096 7680 > gpurun_out/attn_single.log 2>&1
echo "single rc=$?"; tail -8 gpurun_out/attn_single.log
TK_FA_PAIR=1 timeout 300 python scripts/attn_bench.py --prefix 0 512 2048 4096 7680 > gpurun_out/attn_pair.log 2>&1
echo "pair rc=$?"; tail -8 gpurun_out/attn_pair.log
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -p no:cacheprovider -k attention > gpurun_out/pytest_attn.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/pytest_attn.log
