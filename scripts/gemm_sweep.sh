# Time the pair-GEMM schedules (TK_GEMM_CFG="BN,CS,DP") at the OPT-13B chunk shapes,
# next to cuBLAS (torch.matmul) on the same shapes.
for cfg in "" "256,4,0" "256,2,0" "160,2,0"; do
  echo "cfg=$cfg"
  TK_GEMM_CFG="$cfg" python scripts/gemm_bench.py --shapes qkv o fc1 fc2 --iters 20
done
