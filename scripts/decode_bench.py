"""Decode-step microbenchmark (OPT-13B shape): B rows at context ~ctx.

    python scripts/decode_bench.py [--batch 32] [--ctx 1024] [--steps 20]

Runs tk_decode_step repeatedly (the KV of the contexts is whatever the pool
holds: timing only), with per-kernel-class CUDA-event profiling.
"""
import argparse
import json
import time
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2401_11181_b200 import native  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--ctx", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--model", default="opt-13b")
    args = ap.parse_args()
    native.load()
    m = native.MODELS[args.model]
    pages_per = (args.ctx + args.steps + 16) // 16
    inst = native.Instance(m, device=0, seed=0, kv_pages=args.batch * pages_per,
                           max_chunk=max(64, args.batch))
    bt = list(range(args.batch * pages_per))
    last = [7] * args.batch
    for i in range(3):
        ev, _ = inst.decode_step(last, [args.ctx + i] * args.batch, bt, pages_per)
        ev.wait()
    host = [0.0]
    per_step = []

    def run(off):
        evs = []
        for i in range(args.steps):
            t0 = time.perf_counter()
            ev, out = inst.decode_step(last, [args.ctx + off + i] * args.batch, bt, pages_per)
            host[0] += time.perf_counter() - t0
            per_step.append(round((time.perf_counter() - t0) * 1e3, 3))
            evs.append(ev)
        for e in evs:
            e.wait()
        return native.event_elapsed_ns(evs[0], evs[-1])
    # timed without per-kernel events (they would serialise the launches), then
    # once more with them for the per-class breakdown
    total_ns = run(3)
    host_ms = host[0] * 1e3 / args.steps
    inst.profile(True)
    run(3)
    prof = inst.profile_read()
    step_ms = total_ns / 1e6 / args.steps
    weights = m.params * 2
    kv = args.batch * (args.ctx + 3 + args.steps / 2) * m.kv_bytes_per_token
    print(json.dumps({
        "batch": args.batch, "ctx": args.ctx, "step_ms": round(step_ms, 3),
        "host_enqueue_ms": round(host_ms, 3),
        "host_first_steps_ms": per_step[:4],
        "tok_s": round(args.batch / step_ms * 1e3, 1),
        "hbm_floor_ms": round((weights + kv) / 6554.2e9 * 1e3, 3),
        "kernels_ms_per_step": {k: round(v["ms"] / args.steps, 3) for k, v in prof.items()},
        "attention_gbs": round(prof["attention"]["bytes"] / (prof["attention"]["ms"] / 1e3) / 1e9, 1)
        if prof["attention"]["ms"] else None,
    }))


if __name__ == "__main__":
    main()
