"""Generate scheduler-decision golden fixtures from the unmodified reference.

Key order is preserved (mixture order drives rng.choices).  Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_sched_golden.py

For each config/seed it records, from pdsim itself: requests.csv rows, the
summary, every prefill dispatch (t, req, dst, fell_back), every chunk's
(start time, slices, padded) and every decode iteration's batch membership
(row order) plus IterationRecord fields.  The reference is wrapped, never
edited: ``PrefillInstance._schedule_next_chunk`` and
``DecodeInstance._boundary`` are intercepted to read state they already hold.
"""

from __future__ import annotations

import gzip
import json
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")

import pdsim  # noqa: E402
from pdsim import decode as pd_decode  # noqa: E402
from pdsim import prefill as pd_prefill  # noqa: E402

OUT = Path(__file__).with_name("sched_decisions.json.gz")

CASES = [
    ("c1_mixed128_1p1d_roce", {}, 0),
    ("c1_mixed128_1p1d_seed1", {}, 1),
    ("c3_lpld_hpld_1p1d_nvlink", {"workload": {"mixture": {"LPLD": 0.5, "HPLD": 0.5}},
                                  "cost_model": {"preset": "nvlink300"}}, 0),
    ("c4_mixed128_1p3d", {"cluster": {"prefill": 1, "decode": 3},
                          "cost_model": {"preset": "nvlink300"}}, 0),
    ("c4_mixed128_2p2d", {"cluster": {"prefill": 2, "decode": 2},
                          "cost_model": {"preset": "nvlink300"}}, 0),
    ("c4_mixed128_2p6d", {"cluster": {"prefill": 2, "decode": 6},
                          "cost_model": {"preset": "nvlink300"}}, 0),
    ("c4_mixed128_4p4d", {"cluster": {"prefill": 4, "decode": 4},
                          "cost_model": {"preset": "nvlink300"}}, 2),
    ("c4_mixed512_2p2d", {"cluster": {"prefill": 2, "decode": 2},
                          "workload": {"n_requests": 512},
                          "cost_model": {"preset": "nvlink300"}}, 0),
    ("c5_lphd_hphd_2p6d_llama", {"cluster": {"prefill": 2, "decode": 6},
                                 "workload": {"n_requests": 256,
                                              "mixture": {"LPHD": 0.5, "HPHD": 0.5}},
                                 "cost_model": {"preset": "nvlink300",
                                                "kv_bytes_per_token": 524288}}, 0),
    ("greedy_swaps", {"cluster": {"prefill": 1, "decode": 2},
                      "policies": {"decode": "greedy"},
                      "cost_model": {"mem_capacity_tokens": 16000}}, 2),
    ("reserve_static_fcfs_seq", {"policies": {"decode": "reserve_static", "prefill": "fcfs"},
                                 "predictor": {"mode": "sequential", "granularity": 100}}, 4),
    ("ljf_random_poisson", {"cluster": {"prefill": 2, "decode": 2},
                            "policies": {"prefill": "ljf", "dispatcher": "random"},
                            "workload": {"arrival": "poisson", "rate_per_s": 20,
                                         "n_requests": 96}}, 5),
    ("imbalance_upper_nopred", {"cluster": {"prefill": 1, "decode": 3},
                                "policies": {"dispatcher": "imbalance",
                                             "admission_bound": "upper"},
                                "predictor": {"enabled": False}}, 6),
    ("coupled_64", {"system": "coupled", "workload": {"n_requests": 64}}, 1),
    ("chunk512_small_pages", {"cost_model": {"chunk_size": 256, "page_size": 8,
                                             "mem_capacity_tokens": 40000}}, 7),
]


def capture(cfg: dict, seed: int) -> dict:
    chunks: dict[str, list] = {}
    batches: dict[str, list] = {}
    orig_chunk = pd_prefill.PrefillInstance._schedule_next_chunk
    orig_boundary = pd_decode.DecodeInstance._boundary

    def chunk_hook(self, extra_cost=0):
        rnd = self._round
        c = rnd.chunks[rnd.next_chunk]
        chunks.setdefault(self.id, []).append(
            [self.engine.now, [list(s) for s in c.slices], c.padded])
        return orig_chunk(self, extra_cost)

    def boundary_hook(self):
        n_before = len(self.iteration_log)
        orig_boundary(self)
        if len(self.iteration_log) > n_before:
            batches.setdefault(self.id, []).append([r.req.id for r in self.running])

    pd_prefill.PrefillInstance._schedule_next_chunk = chunk_hook
    pd_decode.DecodeInstance._boundary = boundary_hook
    try:
        res = pdsim.run_experiment(pdsim.config_from_dict(cfg), seed=seed)
    finally:
        pd_prefill.PrefillInstance._schedule_next_chunk = orig_chunk
        pd_decode.DecodeInstance._boundary = orig_boundary
    insts = res.control.instances
    return {
        "rows": res.rows,
        "summary": res.summary,
        "dispatches": {k: [list(d) for d in v.dispatches]
                       for k, v in insts.items() if hasattr(v, "dispatches")},
        "chunks": chunks,
        "batches": batches,
        "iterations": {k: [list(vars(r).values()) for r in v.iteration_log]
                       for k, v in insts.items() if hasattr(v, "iteration_log")},
    }


def main() -> None:
    golden = {}
    for name, cfg, seed in CASES:
        golden[name] = {"config": cfg, "seed": seed, **capture(cfg, seed)}
        print(name, golden[name]["summary"]["jct"]["avg_us"])
    with gzip.GzipFile(OUT, "wb", mtime=0) as fh:
        fh.write(json.dumps(golden, separators=(",", ":")).encode())
    print("wrote", OUT, OUT.stat().st_size, "bytes")


if __name__ == "__main__":
    main()
