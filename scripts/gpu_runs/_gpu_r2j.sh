export TK_PARITY_LOG=gpurun_out/parity.jsonl
rm -f $TK_PARITY_LOG
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -8 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
TK_BENCH_WATCHDOG=1200 timeout 1300 python bench.py > gpurun_out/bench.log 2>gpurun_out/bench.err
echo "bench rc=$?"; tail -3 gpurun_out/bench.err
python - <<PY
import json;l=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1])
print(l['value'], l['e2e']['value'], l['roofline']['frac'], l['gpu_launches'], l['clocks'])
print({k:(v['decode_tok_s'],v['step_ms']) for k,v in l['decode'].items()})
sv=l['serving']
for k,v in sv.items():
    if isinstance(v,dict) and 'ttft_avg_ms' in v: print(k, v['ttft_avg_ms'], v['jct_avg_ms'], v['tok_s_per_gpu'], v.get('decode_tok_s_device'))
print('c1', json.dumps(sv.get('c1_tiny_decoder_1p1d'))[:1500])
print('pred', json.dumps(l['predictor'])[:800])
PY
