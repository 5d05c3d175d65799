timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest gpu rc=$?"; tail -2 gpurun_out/pytest_gpu.log
TK_BENCH_WATCHDOG=1200 timeout 1300 python bench.py > gpurun_out/bench.log 2>gpurun_out/bench.err
echo "bench rc=$?"; tail -2 gpurun_out/bench.err
python - <<PY
import json;l=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1])
print(l['value'], l['e2e']['value'], l['roofline']['frac'], l['gpu_launches'], l['clocks'])
print({k:(v['decode_tok_s'],v['step_ms'],v.get('host_enqueue_us_per_step'), v['attention_roofline']['frac']) for k,v in l['decode'].items()})
sv=l['serving']
for k,v in sv.items():
    if isinstance(v,dict) and 'ttft_avg_ms' in v: print(k, v['ttft_avg_ms'], v['jct_avg_ms'], v['tok_s_per_gpu'], v.get('decode_tok_s_device'))
c1=sv['c1_tiny_decoder_1p1d']['device']; print('c1', c1.get('ttft_avg_ms'), c1.get('jct_avg_ms'), c1.get('tok_s_per_gpu'))
print('pred', l['predictor']['device_us'], l['predictor']['corun'].get('measured_tax'))
PY
