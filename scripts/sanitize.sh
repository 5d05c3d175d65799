# compute-sanitizer over the device tests (VERDICT r1 #8 / SURVEY 5): memcheck,
# racecheck (shared-memory hazards), synccheck (barrier misuse) on the smoke run and
# a small-shape subset of the kernel and model tests (decode graphs, head_dim-64
# attention, whole-unit attention plans).  Logs: gpurun_out/sanitize_*.log
CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out
SEL="test_gemm_matches_fp32 and (512-5120-20480 or 907-2304-768 or 16-5120-20480) or test_paged_decode_attention or test_chunk_attention_mixed_slices or test_layernorm or long_prefix_pieces and (130-77 or 256-300 or 1000-300)"
MSEL="test_decode_graph_steps_match_eager and model0"
for tool in memcheck synccheck racecheck; do
  echo "== $tool smoke"
  timeout 900 $CS --tool $tool --print-limit 20 --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_${tool}_smoke.log 2>&1
  echo "rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|smoke ok|Error" gpurun_out/sanitize_${tool}_smoke.log | head -5
  echo "== $tool kernels"
  timeout 1200 $CS --tool $tool --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "$SEL" > gpurun_out/sanitize_${tool}_kernels.log 2>&1
  echo "rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/sanitize_${tool}_kernels.log | head -5
  echo "== $tool decode graphs"
  timeout 900 $CS --tool $tool --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_model.py -q -p no:cacheprovider -x -k "$MSEL" > gpurun_out/sanitize_${tool}_graphs.log 2>&1
  echo "rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/sanitize_${tool}_graphs.log | head -5
done
