export TK_PARITY_LOG=gpurun_out/parity_replay.jsonl
rm -f $TK_PARITY_LOG
timeout 900 python -m pytest tests/test_gpu_replay.py -q -x -p no:cacheprovider -s > gpurun_out/pytest_replay.log 2>&1
echo "replay rc=$?"; tail -6 gpurun_out/pytest_replay.log; cat $TK_PARITY_LOG
