export TK_PARITY_LOG=gpurun_out/parity.jsonl
rm -f $TK_PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
