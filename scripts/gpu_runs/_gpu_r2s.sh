run() { echo "== $ENVV"; for cfg in "256 1024 llama-2-7b" "32 2048 opt-13b" "128 512 opt-13b" "8 512 opt-13b"; do set -- $cfg; env $ENVV timeout 300 python scripts/decode_bench.py --batch $1 --ctx $2 --model $3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['batch'], d['ctx'], d['step_ms'], d['tok_s'])"; done; }
ENVV="TK_X=1" run
ENVV="TK_NORM_PDL=0" run
ENVV="TK_KVW_PDL=0" run
ENVV="TK_DCOMB_PDL=0" run
ENVV="TK_NORM_PDL=0 TK_KVW_PDL=0 TK_DCOMB_PDL=0" run
