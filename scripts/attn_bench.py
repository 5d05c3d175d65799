"""Chunk-attention microbenchmark at the OPT-13B shape (40 heads x 128).

    python scripts/attn_bench.py [--prefix 4096] [--len 512] [--iters 10]

Times tk_chunk_attention for one 512-token slice over a paged prefix and
checks it against a torch fp32 reference on a few heads.
"""
import argparse
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2401_11181_b200 import native  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prefix", type=int, default=4096)
    ap.add_argument("--len", type=int, default=512)
    ap.add_argument("--heads", type=int, default=40)
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--pool-pages", type=int, default=0, help="pool size (pages); 0 = just enough")
    args = ap.parse_args()
    native.load()
    H, D, pt, L = args.heads, 128, 16, args.layers
    ctx = args.prefix + args.len
    n_pages = (ctx + pt - 1) // pt
    g = torch.Generator(device="cuda").manual_seed(0)
    total = max(n_pages, args.pool_pages)
    pool = torch.zeros(total, L, H, 2, pt, D, device="cuda", dtype=torch.bfloat16)
    perm = torch.randperm(total, generator=torch.Generator().manual_seed(1)).tolist()[:n_pages]
    for p_ in perm:
        pool[p_] = (torch.randn(L, H, 2, pt, D, device="cuda", generator=g) * 0.5).bfloat16()
    slices = [(args.prefix, args.len, 0, n_pages, 1)]
    qkv = torch.randn(args.len, 3 * H * D, device="cuda", generator=g).bfloat16()
    layer = L - 1
    o = native.chunk_attention(qkv, 3 * H * D, pool, layer, L, H, D, slices, perm, pt)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(args.iters):
        o = native.chunk_attention(qkv, 3 * H * D, pool, layer, L, H, D, slices, perm, pt)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) / args.iters * 1e3
    flops = 4 * D * H * sum(args.prefix + i + 1 for i in range(args.len))
    # reference on 2 heads
    err = 0.0
    for h in (0, H - 1):
        K = torch.cat([pool[p, layer, h, 0] for p in perm], 0)[:ctx].float()
        V = torch.cat([pool[p, layer, h, 1] for p in perm], 0)[:ctx].float()
        q = qkv[:, h * D:(h + 1) * D].float()
        s = (q @ K.t()) * D ** -0.5
        qpos = torch.arange(args.prefix, ctx, device="cuda")[:, None]
        s = s.masked_fill(torch.arange(ctx, device="cuda")[None] > qpos, float("-inf"))
        ref = torch.softmax(s, -1) @ V
        err = max(err, (o[:, h * D:(h + 1) * D].float() - ref).abs().max().item())
    print(json.dumps({"prefix": args.prefix, "len": args.len, "heads": H, "ms_incl_staging": ms,
                      "tflops_incl_staging": flops / (ms / 1e3) / 1e12, "max_abs_err": err}))


if __name__ == "__main__":
    main()
