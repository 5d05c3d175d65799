# Stream-K cluster-count sweep (TK_GEMM_MAX_CTAS caps the CTAs and skips the split-minimising pick).
for n in 0 120 128 136 140 144 148; do
  echo "ctas=$n"
  TK_GEMM_MAX_CTAS=$n python scripts/gemm_bench.py --shapes qkv fc1 fc2 --iters 20
done
