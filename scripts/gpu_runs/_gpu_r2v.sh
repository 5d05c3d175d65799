for w in -1 0 1 2 3; do echo "whole=$w"; TK_FA_WHOLE=$w timeout 120 python scripts/attn_bench.py --prefix 0 128 256 512 1024 2>&1 | tail -5 | cut -c1-100; done
