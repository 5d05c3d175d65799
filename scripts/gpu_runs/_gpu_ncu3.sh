# round-2 evidence: launch list inside a bench round + --set full of one in-situ layer
# (QKV/O/FC1/FC2 GEMMs, chunk attention + combine, add+norm) and of decode kernels.
# Reports are summarised on the box (scripts/ncu_summary.py) and not copied back.
mkdir -p /tmp/ncu
CMD="python bench.py --steps 1 --warmup 0 --no-serving --no-decode --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 2800 --csv --log-file gpurun_out/r02_launches.csv $CMD > /tmp/ncu/l.log 2>&1
echo "ncu launches rc=$?"; tail -2 /tmp/ncu/l.log; ls -la gpurun_out/r02_launches.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"norm_kernel|fa_combine|chunk_attn_fa|gemm_pair" -s 6000 -c 8 -o /tmp/ncu/r02_layer_final $CMD > /tmp/ncu/f.log 2>&1
echo "ncu full rc=$?"; tail -1 /tmp/ncu/f.log
python scripts/ncu_summary.py /tmp/ncu/r02_layer_final.ncu-rep --label "r02 final: one OPT-13B layer in situ (bench C2)" > gpurun_out/r02_ncu_layer_final.jsonl
timeout 900 ncu --set full --clock-control none -k regex:"decode_attn|gemm_skinny|kv_write" -s 2000 -c 6 -o /tmp/ncu/r02_decode python scripts/decode_bench.py > /tmp/ncu/d.log 2>&1
echo "ncu decode rc=$?"; tail -1 /tmp/ncu/d.log
python scripts/ncu_summary.py /tmp/ncu/r02_decode.ncu-rep --label "r02 final: decode B=32 ctx 1024 OPT-13B (graph replay)" > gpurun_out/r02_ncu_decode.jsonl
wc -l gpurun_out/*.jsonl
export TK_PARITY_LOG=gpurun_out/parity.jsonl
rm -f $TK_PARITY_LOG
timeout 120 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "long_prefix" > gpurun_out/pytest_d64k.log 2>&1
echo "pytest d64 kernels rc=$?"; tail -3 gpurun_out/pytest_d64k.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest gpu rc=$?"; tail -4 gpurun_out/pytest_gpu.log
for mb in 2 4 8; do echo "min_blocks=$mb"; TK_FA_MIN_BLOCKS=$mb timeout 120 python scripts/attn_bench.py --prefix 0 512 1024 2048 2>&1 | tail -4 | cut -c1-90; done
for a in 0 1; do
  if [ $a = 1 ]; then export TK_ATTN_MMA_SYNC=1; fi
  TK_BENCH_WATCHDOG=600 timeout 700 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_d64_$a.log 2>gpurun_out/bench_d64_$a.err
  echo "bench mma_sync=$a rc=$?"; tail -2 gpurun_out/bench_d64_$a.err
  python - <<PY
import json;l=json.loads(open('gpurun_out/bench_d64_$a.log').read().strip().splitlines()[-1])
print(json.dumps(l['predictor'])[:700])
c1=l['serving']['c1_tiny_decoder_1p1d']['device']
print('c1', c1.get('ttft_avg_ms'), c1.get('jct_avg_ms'), c1.get('prefill_tok_s_device'), c1.get('decode_tok_s_device'), c1.get('error'))
PY
done
