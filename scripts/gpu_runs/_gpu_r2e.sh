TK_BENCH_WATCHDOG=150 TK_BENCH_VERBOSE=1 timeout 200 python bench.py --steps 1 --warmup 1 --no-serving --no-decode --no-cpu-baseline > gpurun_out/bench_dbg.log 2>&1
echo "rc=$?"; head -c 3000 gpurun_out/bench_dbg.log; echo; tail -c 3000 gpurun_out/bench_dbg.log
