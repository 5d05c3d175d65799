"""KV handoff microbenchmark: tk_kv_send between two co-located instances.

    python scripts/handoff_bench.py [--model opt-13b] [--tokens 512 900 8192]

One copy-kernel launch per request, pages scattered on both sides (as the
executor's page pools leave them).  Prints device time, KV bytes moved and the
HBM roofline fraction (read + write = 2x the bytes) against MEASURED_PEAKS.json.
"""
import argparse
import json
import random
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2401_11181_b200 import native  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="opt-13b")
    ap.add_argument("--tokens", type=int, nargs="*", default=[512, 900, 8192])
    ap.add_argument("--reps", type=int, default=8)
    args = ap.parse_args()
    native.load()
    shape = native.MODELS[args.model]
    peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())
    n_max = (max(args.tokens) + 15) // 16
    src = native.Instance(shape, device=0, seed=0, kv_pages=n_max + 64, max_chunk=64)
    dst = native.Instance(shape, device=0, seed=0, kv_pages=n_max + 64, max_chunk=64)
    rng = random.Random(0)
    for n_tok in args.tokens:
        n = (n_tok + 15) // 16
        sp, dp = rng.sample(range(n_max + 64), n), rng.sample(range(n_max + 64), n)
        for _ in range(3):
            src.kv_send(sp, dst, dp).wait()
        evs = [src.kv_send(sp, dst, dp) for _ in range(args.reps)]
        for e in evs:
            e.wait()
        ns = sorted(e.elapsed_ns for e in evs)[len(evs) // 2]
        nbytes = n * src.page_bytes
        hbm = 2 * nbytes / (ns / 1e9) / 1e9
        print(json.dumps({"tokens": n_tok, "pages": n, "bytes": nbytes, "device_us": round(ns / 1e3, 1),
                          "kv_gb_s": round(nbytes / (ns / 1e9) / 1e9, 1),
                          "hbm_frac": round(hbm / peak["hbm_gbs"], 4)}), flush=True)
    src.close(), dst.close()


if __name__ == "__main__":
    main()
