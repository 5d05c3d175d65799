# Decode skinny GEMM: L2 prefetch distance sweep (TK_SKINNY_PF) at B=32/ctx 2048 and B=128/ctx 512.
set -x
for b in "32 2048" "128 512"; do
set -- $b
for pf in 0 8 16 32 0; do
TK_SKINNY_PF=$pf timeout 300 python scripts/decode_bench.py --batch $1 --ctx $2 --steps 20 > gpurun_out/dec_pf.log 2>&1
echo "B=$1 ctx=$2 pf=$pf rc=$?"; tail -1 gpurun_out/dec_pf.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['step_ms'], d['tok_s'], d['kernels_ms_per_step'])"
done
done
