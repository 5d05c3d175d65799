# round-2 evidence: launch list inside a bench round + --set full of one in-situ layer
# (QKV/O/FC1/FC2 GEMMs, chunk attention + combine, add+norm) and of decode kernels
CMD="python bench.py --steps 1 --warmup 1 --no-serving --no-decode --no-cpu-baseline"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 60000 -c 3000 --csv --log-file gpurun_out/r02_launches.csv $CMD > gpurun_out/ncu_l.log 2>&1
echo "ncu launches rc=$?"; tail -2 gpurun_out/ncu_l.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"norm_kernel|fa_combine|chunk_attn_fa|gemm_pair" -s 6000 -c 8 -o gpurun_out/r02_layer_final $CMD > gpurun_out/ncu_f.log 2>&1
echo "ncu full rc=$?"; tail -2 gpurun_out/ncu_f.log
timeout 900 ncu --set full --clock-control none -k regex:"decode_attn|gemm_skinny|kv_write" -s 2000 -c 6 -o gpurun_out/r02_decode python scripts/decode_bench.py > gpurun_out/ncu_d.log 2>&1
echo "ncu decode rc=$?"; tail -2 gpurun_out/ncu_d.log
ls -la gpurun_out/*.ncu-rep
