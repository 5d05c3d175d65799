export TK_PARITY_LOG=gpurun_out/parity.jsonl
rm -f $TK_PARITY_LOG
timeout 120 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "long_prefix" > gpurun_out/pytest_d64k.log 2>&1
echo "pytest d64 kernels rc=$?"; tail -2 gpurun_out/pytest_d64k.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest gpu rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for f in 0 1; do
  if [ $f = 1 ]; then export TK_NO_FUSED_DECODE_KV=1; fi
  timeout 300 python scripts/decode_bench.py --batch 32 --ctx 2048 2>&1 | tail -2
  timeout 300 python scripts/decode_bench.py --batch 128 --ctx 512 2>&1 | tail -2
done
unset TK_NO_FUSED_DECODE_KV
TK_BENCH_WATCHDOG=1200 timeout 1300 python bench.py > gpurun_out/bench.log 2>gpurun_out/bench.err
echo "bench rc=$?"; tail -2 gpurun_out/bench.err
python - <<PY
import json;l=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1])
print(l['value'], l['e2e']['value'], l['roofline']['frac'], l['gpu_launches'], l['clocks'])
print({k:(v['decode_tok_s'],v['step_ms'],v.get('host_enqueue_us_per_step')) for k,v in l['decode'].items()})
sv=l['serving']
for k,v in sv.items():
    if isinstance(v,dict) and 'ttft_avg_ms' in v: print(k, v['ttft_avg_ms'], v['jct_avg_ms'], v['tok_s_per_gpu'], v.get('decode_tok_s_device'))
print('c1', json.dumps(sv.get('c1_tiny_decoder_1p1d'))[:900])
print('pred', json.dumps(l['predictor'])[:900])
PY
