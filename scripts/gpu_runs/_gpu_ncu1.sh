ncu --set full --clock-control none --import-source on -k regex:"norm_kernel|fa_combine|chunk_attn_fa|gemm_pair" -s 3000 -c 8 -o gpurun_out/r02_layer python bench.py --steps 1 --warmup 3 --no-serving --no-decode --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu1.log
