run() { echo "== $1"; shift; for cfg in "256 1024 llama-2-7b" "32 2048 opt-13b" "128 512 opt-13b" "8 512 opt-13b"; do set -- $cfg; env $ENVV timeout 300 python scripts/decode_bench.py --batch $1 --ctx $2 --model $3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['batch'], d['ctx'], d['step_ms'], d['tok_s'], d['host_first_steps_ms'][-1])"; done; }
ENVV="TK_X=1" run default
ENVV="TK_NO_PDL=1" run no_pdl
ENVV="TK_DEC_ATTN_PDL=0" run no_attn_pdl
ENVV="TK_DEC_ATTN_PDL=0 TK_NO_DECODE_GRAPH=1" run no_attn_pdl_nograph
