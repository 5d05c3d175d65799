export TK_PARITY_LOG=gpurun_out/parity.jsonl
rm -f $TK_PARITY_LOG
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
for g in 1 0; do
  if [ $g = 0 ]; then export TK_NO_DECODE_GRAPH=1; fi
  TK_BENCH_WATCHDOG=900 timeout 1000 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_g$g.log 2>gpurun_out/bench_g$g.err
  echo "bench g=$g rc=$?"; tail -3 gpurun_out/bench_g$g.err
  python - <<PY
import json;l=json.loads(open('gpurun_out/bench_g$g.log').read().strip().splitlines()[-1])
print('g=$g', l['value'], {k:(v['decode_tok_s'],v['step_ms']) for k,v in l['decode'].items()})
sv=l['serving']
for k,v in sv.items():
    if isinstance(v,dict) and 'ttft_avg_ms' in v: print(k, v['ttft_avg_ms'], v['jct_avg_ms'], v['tok_s_per_gpu'], v.get('decode_tok_s_device'))
c1=sv.get('c1_tiny_decoder_1p1d',{})
print('c1', json.dumps(c1)[:600])
PY
done
