# OPT-13B-width C2-round parity through both chunk-attention kernels.
set -x
export TK_PARITY_LOG=gpurun_out/parity_c2.jsonl
rm -f $TK_PARITY_LOG
timeout 900 python -m pytest tests/test_gpu_parity_scale.py -m gpu -q -x -p no:cacheprovider -k c2_round > gpurun_out/pytest_c2.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_c2.log; cat $TK_PARITY_LOG
