for pdl in 0 1; do
  if [ $pdl = 1 ]; then export TK_NO_PDL=1; fi
  echo "TK_NO_PDL=$pdl"
  timeout 300 python scripts/decode_bench.py --batch 256 --ctx 1024 --model llama-2-7b 2>&1 | tail -1 | cut -c1-400
  timeout 300 python scripts/decode_bench.py --batch 32 --ctx 2048 2>&1 | tail -1 | cut -c1-400
  timeout 300 python scripts/decode_bench.py --batch 128 --ctx 512 2>&1 | tail -1 | cut -c1-400
done
unset TK_NO_PDL
echo "graphs off"
TK_NO_DECODE_GRAPH=1 timeout 300 python scripts/decode_bench.py --batch 256 --ctx 1024 --model llama-2-7b 2>&1 | tail -1 | cut -c1-400
