"""End-to-end serving run on B200: the reference scheduler + CUDA executor.

    python scripts/e2e_mixed.py [--n 32] [--model opt-13b] [--split 1:1] [--sim]

Prints one JSON line: mean/p50/p99 TTFT and JCT (measured clock), prefill and
decode tokens/s (device time), KV handoff GB/s, and the same workload's
pdsim-modeled numbers from the simulated executor for context.
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2401_11181_b200 as tk  # noqa: E402
from paper_2401_11181_b200.experiment import run_experiment  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--model", default="opt-13b")
    ap.add_argument("--split", default="1:1")
    ap.add_argument("--capacity", type=int, default=40000)
    ap.add_argument("--prefill-pages", type=int, default=2048)
    ap.add_argument("--mixture", default="")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--system", default="disaggregated", choices=["disaggregated", "coupled"])
    args = ap.parse_args()
    npf, ndc = (int(x) for x in args.split.split(":"))
    cfg = {
        "system": args.system,
        "cluster": {"prefill": npf, "decode": ndc} if args.system == "disaggregated"
        else {"coupled": 1},
        "workload": {"n_requests": args.n},
        "cost_model": {"preset": "nvlink300", "mem_capacity_tokens": args.capacity},
        "model": {"name": args.model, "prefill_pages": args.prefill_pages, "staging_pages": 512,
                  "max_decode_batch": 256},
    }
    if args.mixture:
        cfg["workload"]["mixture"] = {k: 1.0 for k in args.mixture.split(",")}
    sim = run_experiment(tk.config_from_dict(cfg), seed=args.seed).summary
    t0 = time.perf_counter()
    res = run_experiment(tk.config_from_dict(dict(cfg, executor="cuda")), seed=args.seed)
    wall = time.perf_counter() - t0
    s, d = res.summary, res.summary["device"]
    out = {
        "workload": f"{args.mixture or 'Mixed'}-{args.n}, "
                    f"{f'{npf}P:{ndc}D' if args.system == 'disaggregated' else 'coupled x1'}, "
                    f"{args.model}, burst",
        "ttft_avg_ms": s["ttft"]["avg_us"] / 1e3, "ttft_p50_ms": s["ttft"]["p50_us"] / 1e3,
        "ttft_p99_ms": s["ttft"]["p99_us"] / 1e3,
        "jct_avg_ms": s["jct"]["avg_us"] / 1e3, "jct_p50_ms": s["jct"]["p50_us"] / 1e3,
        "jct_p99_ms": s["jct"]["p99_us"] / 1e3,
        "makespan_s": s["makespan_us"] / 1e6, "wall_s": wall,
        "prefill_tok_s_device": d.get("prefill_tok_s_device"),
        "decode_tok_s_device": d.get("decode_tok_s_device"),
        "decode_tok_s_wall": d["decode_tokens"] / (s["makespan_us"] / 1e6),
        "handoff_gb_s": d.get("handoff_gb_s"), "kv_bytes_sent": d["kv_bytes_sent"],
        "resource_usage_s": s["resource_usage_us"] / 1e6, "perf_per_dollar": s["perf_per_dollar"],
        "decode_steps": d["decode_steps"], "completed": s["completed"],
        "modeled_reference": {"ttft_avg_ms": sim["ttft"]["avg_us"] / 1e3,
                              "jct_avg_ms": sim["jct"]["avg_us"] / 1e3,
                              "makespan_s": sim["makespan_us"] / 1e6},
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
