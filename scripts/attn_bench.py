"""Chunk-attention microbenchmark at the OPT-13B shape (40 heads x 128).

    python scripts/attn_bench.py [--prefix 0 2048 4096 7680] [--len 512] [--iters 20]

Times tk_chunk_attention_timed (device time of back-to-back launches, CUDA
events on the launching stream, work list staged once) for one 512-token
slice over a paged prefix, and checks it against a torch fp32 reference on
two heads.  The KV pool (pages scattered at random) is larger than L2 for
prefixes >= 2048, like the serving pool.
"""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2401_11181_b200 import native  # noqa: E402


def run(prefix, length, H, L, iters, peak):
    D, pt = 128, 16
    ctx = prefix + length
    n_pages = (ctx + pt - 1) // pt
    g = torch.Generator(device="cuda").manual_seed(0)
    pool = (torch.randn(n_pages, L, H, 2, pt, D, device="cuda", generator=g) * 0.5).bfloat16()
    perm = torch.randperm(n_pages, generator=torch.Generator().manual_seed(1)).tolist()
    slices = [(prefix, length, 0, n_pages, 1)]
    qkv = torch.randn(length, 3 * H * D, device="cuda", generator=g).bfloat16()
    layer = L - 1
    o, us = native.chunk_attention_timed(qkv, 3 * H * D, pool, layer, L, H, D, slices, perm,
                                         iters=iters)
    flops = 4 * D * H * sum(prefix + i + 1 for i in range(length))
    err = 0.0
    for h in (0, H - 1):
        K = torch.cat([pool[p, layer, h, 0] for p in perm], 0)[:ctx].float()
        V = torch.cat([pool[p, layer, h, 1] for p in perm], 0)[:ctx].float()
        q = qkv[:, h * D:(h + 1) * D].float()
        s = (q @ K.t()) * D ** -0.5
        qpos = torch.arange(prefix, ctx, device="cuda")[:, None]
        s = s.masked_fill(torch.arange(ctx, device="cuda")[None] > qpos, float("-inf"))
        ref = torch.softmax(s, -1) @ V
        err = max(err, (o[:, h * D:(h + 1) * D].float() - ref).abs().max().item())
    tf = flops / (us * 1e-6) / 1e12
    return {"prefix": prefix, "len": length, "heads": H, "device_us": round(us, 2),
            "tflops": round(tf, 1), "frac_burst": round(tf / peak, 3), "max_abs_err": err}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prefix", type=int, nargs="*", default=[0, 2048, 4096, 7680])
    ap.add_argument("--len", type=int, default=512)
    ap.add_argument("--heads", type=int, default=40)
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    native.load()
    peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())
    for p in args.prefix:
        print(json.dumps(run(p, args.len, args.heads, args.layers, args.iters,
                             peak["bf16_tflops"])), flush=True)


if __name__ == "__main__":
    main()
