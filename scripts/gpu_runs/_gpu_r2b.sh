export TK_PARITY_LOG=gpurun_out/parity.jsonl
rm -f $TK_PARITY_LOG
timeout 900 python -m pytest tests/test_gpu_replay.py -q -x -s -p no:cacheprovider > gpurun_out/pytest_replay.log 2>&1
echo "replay rc=$?"; tail -5 gpurun_out/pytest_replay.log; cat $TK_PARITY_LOG
timeout 300 python scripts/attn_bench.py --prefix 0 128 256 512 1024 2048 3072 4096 6144 7680 2>&1 | tail -10
timeout 900 python bench.py --steps 2 --warmup 3 --no-serving --no-cpu-baseline > gpurun_out/bench_pred.log 2>gpurun_out/bench_pred.err
echo "bench rc=$?"; tail -3 gpurun_out/bench_pred.err
python -c "
import json;l=json.loads(open('gpurun_out/bench_pred.log').read().strip().splitlines()[-1])
print(json.dumps(l['predictor'])); print(l['value'], l['clocks'])"
