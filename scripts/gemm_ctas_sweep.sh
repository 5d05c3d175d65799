# Stream-K cluster-count sweep (TK_GEMM_MAX_CTAS caps the CTAs and skips the split-minimising pick).
for n in 0 120 128 132 136 148; do
  echo "ctas=$n"
  TK_GEMM_MAX_CTAS=$n python scripts/gemm_bench.py --shapes qkv o fc1 fc2 --iters 20
done
