"""Microbenchmark of the tcgen05 GEMM at the OPT-13B chunk shapes (M=512).

    python scripts/gemm_bench.py [--iters 50] [--m 512]

Times each shape with CUDA events on the launching stream (after warm-up) and
prints TFLOP/s against MEASURED_PEAKS.json.  Weights (B) are larger than L2
for every shape except O-proj; a 256 MB buffer is rewritten between
iterations to flush L2.
"""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2401_11181_b200 import native  # noqa: E402

# epilogues as the runtime uses them (O-proj / FC2 store bf16; the next norm adds the residual)
SHAPES = {"qkv": (15360, 5120, native.EPI_BF16_BIAS), "o": (5120, 5120, native.EPI_BF16_BIAS),
          "fc1": (20480, 5120, native.EPI_BF16_BIAS_RELU), "fc2": (5120, 20480, native.EPI_BF16_BIAS)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--m", type=int, nargs="*", default=[512])
    ap.add_argument("--shapes", nargs="*", default=list(SHAPES))
    ap.add_argument("--nk", nargs="*", default=[],
                    help="extra N,K shapes (bf16+bias epilogue), e.g. 5120,2560")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--cublas", action="store_true",
                    help="time torch.matmul (cuBLAS) on the same shapes instead, for reference")
    ap.add_argument("--epi", default=None, choices=["bf16", "f32", "resid"],
                    help="override the shape's epilogue (isolates epilogue cost)")
    ap.add_argument("--chain", type=int, default=0,
                    help="time N back-to-back layers of all --shapes (decode-style weight streaming)")
    args = ap.parse_args()
    for nk in args.nk:
        n_, k_ = (int(x) for x in nk.split(","))
        SHAPES[nk] = (n_, k_, native.EPI_BF16_BIAS)
        args.shapes.append(nk)
    native.load()
    if args.chain:
        return chain(args)
    peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for M in args.m:
        for name in args.shapes:
            N, K, epi = SHAPES[name]
            if args.epi:
                epi = {"bf16": native.EPI_BF16, "f32": native.EPI_F32,
                       "resid": native.EPI_F32_BIAS_RESID}[args.epi]
            a = torch.randn(M, K, device="cuda").bfloat16()
            b = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
            bias = torch.zeros(N, device="cuda").bfloat16()
            out = torch.zeros(M, N, device="cuda",
                              dtype=torch.float32 if epi >= 3 else torch.bfloat16)
            import ctypes
            nb = ctypes.c_int64()
            native.check(native.load().tk_gemm_workspace_bytes(M, N, K, ctypes.byref(nb)))
            ws = torch.zeros(nb.value, dtype=torch.uint8, device="cuda")
            if args.cublas:
                bt = b.t()
                run = lambda: torch.matmul(a, bt)  # noqa: E731
            else:
                run = lambda: native.gemm(a, b, bias=bias, epilogue=epi, out=out, workspace=ws)  # noqa: E731
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            times = []
            for _ in range(args.iters):
                if not args.no_flush:
                    flush.zero_()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                run()
                e.record()
                e.synchronize()
                times.append(s.elapsed_time(e))
            ms = sorted(times)[len(times) // 2]
            tf = 2 * M * N * K / (ms / 1e3) / 1e12
            print(json.dumps({"shape": name, "epi": "cublas" if args.cublas else epi, "M": M, "N": N, "K": K, "median_us": round(ms * 1e3, 2),
                              "tflops": round(tf, 1),
                              "frac_burst": round(tf / peak["bf16_tflops"], 3)}))


def chain(args):
    """--chain N: N layers x (the shapes in order) back to back, no L2 flush; weights are
    distinct per layer (larger than L2), like a decode step's GEMM sequence."""
    import ctypes
    for M in args.m:
        layers = []
        for li in range(args.chain):
            ops = []
            for name in args.shapes:
                N, K, epi = SHAPES[name]
                b = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
                ops.append((N, K, epi, b))
            layers.append(ops)
        acts = {K: torch.randn(M, K, device="cuda").bfloat16() for K in {5120, 20480}}
        outs = {}
        nb = ctypes.c_int64()
        ws_bytes = 0
        for N, K, epi, _ in layers[0]:
            native.check(native.load().tk_gemm_workspace_bytes(M, N, K, ctypes.byref(nb)))
            ws_bytes = max(ws_bytes, nb.value)
            outs[(N, K)] = torch.zeros(M, N, device="cuda",
                                       dtype=torch.float32 if epi >= 3 else torch.bfloat16)
        ws = torch.zeros(ws_bytes, dtype=torch.uint8, device="cuda")

        def run():
            for ops in layers:
                for N, K, epi, b in ops:
                    native.gemm(acts[K], b, epilogue=epi, out=outs[(N, K)], workspace=ws)
        for _ in range(2):
            run()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        run()
        e.record()
        e.synchronize()
        ms = s.elapsed_time(e)
        wbytes = sum(N * K * 2 for ops in layers for N, K, _, _ in ops)
        print(json.dumps({"chain_layers": args.chain, "M": M, "shapes": args.shapes,
                          "ms": round(ms, 3), "weight_gbs": round(wbytes / ms / 1e6, 1)}))


if __name__ == "__main__":
    main()
