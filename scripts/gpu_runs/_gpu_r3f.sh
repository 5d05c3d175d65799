timeout 600 python scripts/colocated_split.py --split 2 6 --n 64 2>&1 | tail -3 | cut -c1-1500
timeout 600 python scripts/colocated_split.py --split 4 4 --n 64 2>&1 | tail -3 | cut -c1-1500
timeout 600 python scripts/colocated_split.py --split 1 3 --n 64 2>&1 | tail -3 | cut -c1-1500
