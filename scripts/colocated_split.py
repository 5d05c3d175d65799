"""Run a P:D-split serving leg with every instance co-located on GPU 0: exercises
the multi-instance host paths of the multi-GPU legs (dispatch over several decode
instances, handoffs between pools, capacity sizing shared by several decode
instances, one host thread driving them all) on a one-GPU box.

    python scripts/colocated_split.py --split 2 6 --n 64
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--split", type=int, nargs=2, default=[2, 6])
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--model", default="opt-13b")
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    args = argparse.Namespace(seed=a.seed, model=a.model)
    t0 = time.perf_counter()
    out = bench.serving_leg(args, a.split[0], a.split[1], a.n, colocate=True)
    out["wall_s"] = round(time.perf_counter() - t0, 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
