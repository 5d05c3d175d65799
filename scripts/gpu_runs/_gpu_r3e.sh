run() { echo "== $1"; for cfg in "32 2048" "8 512" "128 512"; do set -- $cfg; env TK_GEMM_SKINNY_MAP="$MAP" timeout 300 python scripts/decode_bench.py --batch $1 --ctx $2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['batch'], d['ctx'], d['step_ms'], {k:v for k,v in d['kernels_ms_per_step'].items() if 'gemm' in k and 'head' not in k})"; done; }
MAP="" run base
MAP="5120,5120,80" run o80
MAP="5120,5120,140" run o140
MAP="5120,20480,80" run fc2_80
MAP="5120,20480,128" run fc2_128
MAP="20480,5120,80" run fc1_80
MAP="20480,5120,140" run fc1_140
