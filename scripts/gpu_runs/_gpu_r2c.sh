export TK_LIB=paper_2401_11181_b200/lib/libtetri_exp.so
echo "cublas"; timeout 300 python scripts/gemm_bench.py --cublas --shapes qkv o fc1 fc2 2>&1 | tail -4
for e in 0 1 2 3; do echo "exp=$e"; TK_GEMM_EXP=$e timeout 300 python scripts/gemm_bench.py --shapes qkv o fc1 fc2 2>&1 | tail -4; done
echo "exp=0 no-flush"; timeout 300 python scripts/gemm_bench.py --no-flush --shapes qkv o fc1 fc2 2>&1 | tail -4
echo "cublas no-flush"; timeout 300 python scripts/gemm_bench.py --cublas --no-flush --shapes qkv o fc1 fc2 2>&1 | tail -4
