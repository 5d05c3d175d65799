set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
export TK_PARITY_LOG=gpurun_out/parity.jsonl
rm -f $TK_PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1500 python bench.py > gpurun_out/bench.log 2>gpurun_out/bench.err
echo "bench rc=$?"
tail -5 gpurun_out/bench.err
tail -c 4000 gpurun_out/bench.log
