# ncu --set full of the single-CTA and CTA-pair chunk attention at prefix 4096 (512 queries, 40 heads).
set -x
for pr in 0 1; do
TK_FA_PAIR=$pr timeout 600 ncu --set full --clock-control none --import-source on -k regex:"chunk_attn_fa" -s 2 -c 1 -o gpurun_out/r02_attn_pair$pr python scripts/attn_bench.py --prefix 4096 --iters 3 > gpurun_out/ncu_attn$pr.log 2>&1
echo "ncu pair=$pr rc=$?"; tail -2 gpurun_out/ncu_attn$pr.log
done
ls -la gpurun_out/*.ncu-rep
