# CTA-pair chunk attention: exponential split sweep (isolated) and in-situ prefill A/B.
set -x
for v in 4 2 3; do
TK_FA_PAIR_POLY=$v timeout 300 python scripts/attn_bench.py --prefix 0 2048 4096 7680 > gpurun_out/attn_pair_p$v.log 2>&1
echo "pair poly $v rc=$?"; tail -4 gpurun_out/attn_pair_p$v.log | cut -c1-110
done
for pr in 0 1 0 1; do
TK_FA_PAIR=$pr timeout 600 python bench.py --no-serving --no-decode --no-cpu-baseline > gpurun_out/bench_pair$pr.log 2>&1
echo "bench pair=$pr rc=$?"
tail -1 gpurun_out/bench_pair$pr.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['kernels']['attention'], d['clocks']['sm_mhz'])"
done
