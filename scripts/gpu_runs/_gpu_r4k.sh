# Final check of the session's HEAD: -m gpu suite, smoke(), reference arm, default bench.
set -x
export TK_PARITY_LOG=gpurun_out/parity.jsonl
rm -f $TK_PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1
echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log | cut -c1-600
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
echo "bench rc=$?"
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'], {k: v.get('decode_tok_s') for k, v in d['decode'].items()})"
