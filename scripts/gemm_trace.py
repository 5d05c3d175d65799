"""Pipeline timeline of the pair GEMM (CTA 0), from clock64 stamps.

    python scripts/gemm_trace.py [--shape fc2] [--cfg 256,4,0]

Per k-block: when the UMMA warp started waiting for the stage (0), got it (1)
and had issued its MMAs + commit (2); when the producer started waiting for a
free stage (3) and got it (4).  Steady-state means tell whether the tensor
pipe is fed (issuer waits ~0, producer waits ~one MMA period) or starved
(issuer waits on data).
"""
import argparse
import ctypes
import json
import os
import sys
from pathlib import Path

os.environ["TK_GEMM_TRACE"] = "1"
# the hooks exist only in the experiments build (lib/libtetri_exp.so)
os.environ.setdefault("TK_LIB", str(Path(__file__).resolve().parents[1] /
                                    "paper_2401_11181_b200" / "lib" / "libtetri_exp.so"))
import torch  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2401_11181_b200 import native  # noqa: E402

SHAPES = {"qkv": (15360, 5120), "o": (5120, 5120), "fc1": (20480, 5120), "fc2": (5120, 20480)}
N_TRACE = 1024


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="fc2")
    ap.add_argument("--m", type=int, default=512)
    ap.add_argument("--stages", type=int, default=8, help="ring depth of the traced config")
    args = ap.parse_args()
    native.load()
    N, K = SHAPES[args.shape]
    M = args.m
    a = torch.randn(M, K, device="cuda").bfloat16()
    b = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
    out = torch.zeros(M, N, device="cuda").bfloat16()
    nb = ctypes.c_int64()
    native.check(native.load().tk_gemm_workspace_bytes(M, N, K, ctypes.byref(nb)))
    ws = torch.zeros(nb.value, dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        native.gemm(a, b, epilogue=native.EPI_BF16, out=out, workspace=ws)
    flush.zero_()
    native.gemm(a, b, epilogue=native.EPI_BF16, out=out, workspace=ws)
    torch.cuda.synchronize()
    buf = (ctypes.c_uint64 * (6 * N_TRACE))()
    native.check(native.load().tk_debug_gemm_trace(buf, 6 * N_TRACE), "trace")
    get = lambda k, j: buf[k * N_TRACE + j]  # noqa: E731
    n = 0
    while n < N_TRACE and get(1, n):
        n += 1
    if n < 8:
        print("no trace (the shape took another kernel?)")
        return
    base = get(0, 0)
    lo, hi = min(8, n // 4), max(n - 8, 3 * n // 4)
    rng = range(lo, hi)
    mean = lambda f: sum(f(j) for j in rng) / len(rng)  # noqa: E731
    period = mean(lambda j: get(0, j + 1) - get(0, j))
    wait_full = mean(lambda j: get(1, j) - get(0, j))
    issue = mean(lambda j: get(2, j) - get(1, j))
    prod = [j for j in rng if get(4, j) and get(3, j)]
    wait_empty = sum(get(4, j) - get(3, j) for j in prod) / max(1, len(prod))
    tiles = [get(5, t) - base for t in range(8) if get(5, t)]
    res = {"shape": args.shape, "M": M, "N": N, "K": K, "kblocks_cta0": n,
           "period_cycles": round(period, 1), "issuer_wait_full": round(wait_full, 1),
           "issue_cycles": round(issue, 1), "producer_wait_empty": round(wait_empty, 1),
           "first_full_after_start": get(1, 0) - base,
           "total_cycles": get(2, n - 1) - base, "epilogue_seen_at": tiles}
    print(json.dumps(res))
    cta = (ctypes.c_uint64 * (7 * 256))()
    native.check(native.load().tk_debug_gemm_cta_trace(cta, 7 * 256), "cta trace")
    n_cta = sum(1 for c in range(256) if cta[c])
    t0 = min(cta[c] for c in range(n_cta))
    rel = lambda k: [(cta[k * 256 + c] - t0) / 1e3 if cta[k * 256 + c] else None for c in range(n_cta)]  # noqa: E731
    ent, first, last, epi, ext, saw, ready = (rel(k) for k in range(7))
    lead = [c for c in range(n_cta) if first[c] is not None]
    summ = lambda v: (round(min(v), 2), round(sorted(v)[len(v) // 2], 2), round(max(v), 2))  # noqa: E731
    print(json.dumps({"ctas": n_cta, "entry_us(min,med,max)": summ([x for x in ent if x is not None]),
                      "first_stage_us": summ([first[c] for c in lead]),
                      "last_commit_us": summ([last[c] for c in lead]),
                      "epilogue_done_us": summ([x for x in epi if x is not None]),
                      "exit_us": summ([x for x in ext if x is not None]),
                      "mainloop_us": summ([last[c] - first[c] for c in lead])}))
    fx = [c for c in range(n_cta) if ready[c] is not None and saw[c] is not None]
    if fx:
        print(json.dumps({"fixup_ctas": len(fx),
                          "saw_last_acc_after_commit_us": summ([saw[c] - last[c - c % 2] for c in fx if last[c - c % 2] is not None]),
                          "partials_ready_wait_us": summ([ready[c] - saw[c] for c in fx]),
                          "fixup_work_us": summ([epi[c] - ready[c] for c in fx if epi[c] is not None])}))
    S = args.stages
    lat = [(get(4, j + S) - get(2, j), get(1, j + S) - get(4, j + S), get(0, j + S) - get(4, j + S))
           for j in range(lo, min(hi, n - S)) if get(4, j + S)]
    if lat:
        print(json.dumps({"stages": S, "commit_to_refill": round(sum(a for a, _, _ in lat) / len(lat), 1),
                          "refill_to_full_seen": round(sum(b for _, b, _ in lat) / len(lat), 1),
                          "refill_to_issuer_ready": round(sum(c for _, _, c in lat) / len(lat), 1)}))
    for j in list(range(0, 6)) + list(range(n // 2, n // 2 + 6)):
        print(j, [(get(k, j) - base) if get(k, j) else -1 for k in range(5)])


if __name__ == "__main__":
    main()
