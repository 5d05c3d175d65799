run() { tag=$1; shift; env "$@" TK_BENCH_WATCHDOG=100 timeout 130 python bench.py --steps 1 --warmup 1 --no-serving --no-decode --no-cpu-baseline > gpurun_out/bench_$tag.log 2>&1; echo "$tag rc=$? $(grep -c . gpurun_out/bench_$tag.log) lines"; tail -c 300 gpurun_out/bench_$tag.log | head -c 300; echo; }
run old TK_LIB=paper_2401_11181_b200/lib/libtetri_old.so
run no144 TK_NO_144=1
run w0 TK_GEMM_W144=0
run w1 TK_GEMM_W144=1
