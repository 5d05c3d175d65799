export TK_PARITY_LOG=gpurun_out/parity.jsonl
rm -f $TK_PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 1500 python bench.py > gpurun_out/bench.log 2>gpurun_out/bench.err
echo "bench rc=$?"
tail -5 gpurun_out/bench.err
