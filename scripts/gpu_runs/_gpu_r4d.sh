# Persisting L2 window for the residual stream (A/B in situ) + CTA-pair kernel parity.
set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -p no:cacheprovider -k "attention" > gpurun_out/pytest_attn.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/pytest_attn.log
for pv in 1 0 1 0; do
TK_L2_PERSIST=$pv timeout 600 python bench.py --no-serving --no-decode --no-cpu-baseline > gpurun_out/bench_l2p$pv.log 2>&1
echo "bench l2persist=$pv rc=$?"
tail -1 gpurun_out/bench_l2p$pv.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print(d['value'], {n: (v['ms'], v['tflops'] or v['gbs']) for n, v in k.items()}, d['clocks']['sm_mhz'])"
done
