"""Pipeline timeline of the chunk-attention kernel (CTA 0), from clock64 stamps.

    TK_FA_VARIANT=7 python scripts/attn_trace.py [--prefix 7680] [--variant-exp 1]

Prints, per key block, when the producer issued K_j / V_j, when each tile's
softmax warp saw S_t(j) and released P_t(j), and when the UMMA thread saw P,
issued PV_t(j) and S_t(j+1) -- cycles relative to the first stamp.
"""
import argparse
import ctypes
import os
import sys
from pathlib import Path

os.environ.setdefault("TK_FA_VARIANT", "7")
import torch  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2401_11181_b200 import native  # noqa: E402

KINDS = ["sm_seeS", "sm_relP", "mma_seeP", "mma_PV", "mma_Snext", "prod_K", "prod_V",
         "sm_ldS", "sm_max", "sm_exp"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prefix", type=int, default=7680)
    ap.add_argument("--first", type=int, default=8)
    ap.add_argument("--count", type=int, default=10)
    args = ap.parse_args()
    native.load()
    H, D, pt, L = 40, 128, 16, 2
    ctx = args.prefix + 512
    n_pages = (ctx + pt - 1) // pt
    pool = (torch.randn(n_pages, L, H, 2, pt, D, device="cuda") * 0.5).bfloat16()
    qkv = torch.randn(512, 3 * H * D, device="cuda").bfloat16()
    native.chunk_attention_timed(qkv, 3 * H * D, pool, 1, L, H, D, [(args.prefix, 512, 0, n_pages, 1)],
                                 list(range(n_pages)), iters=3)
    buf = (ctypes.c_uint64 * (10 * 2 * 512))()
    native.check(native.load().tk_debug_fa_trace(buf, 10 * 2 * 512), "trace")
    get = lambda k, t, j: buf[(k * 2 + t) * 512 + j]  # noqa: E731
    base = min(v for v in buf if v) if any(buf) else 0
    print("block " + " ".join(f"{k}{t}".rjust(11) for k in KINDS[:5] for t in (0, 1)) + " "
          + " ".join(k.rjust(9) for k in KINDS[5:]))
    prev = None
    for j in range(args.first, args.first + args.count):
        row = [get(k, t, j) for k in range(5) for t in (0, 1)] + [get(5, 0, j), get(6, 0, j)]
        rel = [(v - base) if v else -1 for v in row]
        print(f"{j:5d} " + " ".join(f"{v:11d}" for v in rel[:10]) + " " + " ".join(f"{v:9d}" for v in rel[10:]))
        if prev is not None and row[0] and prev[0]:
            pass
        prev = row
    # per-block period of tile 0 (S seen -> next S seen) and the split of it
    per = [get(0, 0, j + 1) - get(0, 0, j) for j in range(args.first, args.first + args.count)]
    sm = [get(1, 0, j) - get(0, 0, j) for j in range(args.first, args.first + args.count)]
    wait = [get(0, 0, j + 1) - get(1, 0, j) for j in range(args.first, args.first + args.count)]
    print("tile0 period", sum(per) // len(per), "softmax", sum(sm) // len(sm),
          "P->next S", sum(wait) // len(wait), "cycles (mean)")
    rng = range(args.first, args.first + args.count)
    if get(7, 0, args.first):
        def mean(a, b):
            return sum(get(b, 0, j) - get(a, 0, j) for j in rng) // len(rng)
        print("softmax split (tile 0): S seen -> S loaded", mean(0, 7), "| -> max exchanged",
              mean(7, 8), "| -> exps+P stores issued", mean(8, 9), "| -> P released", mean(9, 1))


if __name__ == "__main__":
    main()
