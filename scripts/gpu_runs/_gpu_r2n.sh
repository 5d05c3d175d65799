export TK_PARITY_LOG=gpurun_out/parity.jsonl
rm -f $TK_PARITY_LOG
timeout 120 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "long_prefix" > gpurun_out/pytest_d64k.log 2>&1
echo "pytest d64 kernels rc=$?"; tail -3 gpurun_out/pytest_d64k.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest gpu rc=$?"; tail -4 gpurun_out/pytest_gpu.log
for mb in 2 4 8; do echo "min_blocks=$mb"; TK_FA_MIN_BLOCKS=$mb timeout 120 python scripts/attn_bench.py --prefix 0 512 1024 2048 2>&1 | tail -4 | cut -c1-90; done
for a in 0 1; do
  if [ $a = 1 ]; then export TK_ATTN_MMA_SYNC=1; fi
  TK_BENCH_WATCHDOG=600 timeout 700 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_d64_$a.log 2>gpurun_out/bench_d64_$a.err
  echo "bench mma_sync=$a rc=$?"; tail -2 gpurun_out/bench_d64_$a.err
  python - <<PY
import json;l=json.loads(open('gpurun_out/bench_d64_$a.log').read().strip().splitlines()[-1])
print(json.dumps(l['predictor'])[:700])
c1=l['serving']['c1_tiny_decoder_1p1d']['device']
print('c1', c1.get('ttft_avg_ms'), c1.get('jct_avg_ms'), c1.get('prefill_tok_s_device'), c1.get('decode_tok_s_device'), c1.get('error'))
PY
done
