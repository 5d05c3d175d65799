for v in 1 0; do echo "combine=$v"; TK_FA_COMBINE=$v timeout 300 python scripts/attn_bench.py --prefix 0 1024 2048 4096 7680 2>&1 | tail -5; done
for ks in 2 1; do echo "trace KS=$ks"; TK_GEMM_KS=$ks timeout 300 python scripts/gemm_trace.py --shape fc2 2>&1 | tail -3; done
echo "trace o"; timeout 300 python scripts/gemm_trace.py --shape o 2>&1 | tail -3
echo "trace qkv"; timeout 300 python scripts/gemm_trace.py --shape qkv 2>&1 | tail -3
