# Session-6 baseline: -m gpu tests + default bench on the restored tree.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
export TK_PARITY_LOG=gpurun_out/parity.jsonl
rm -f $TK_PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
echo "bench rc=$?"
tail -c 1500 gpurun_out/bench.log
