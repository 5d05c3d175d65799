"""Shared parity checks for the device-vs-oracle model tests.

Logit tolerance (bf16 device path vs the fp32 oracle): per row,
max |device - oracle| <= LOGIT_TOL x (max - min of the oracle row), and
cosine similarity >= LOGIT_COS.  Greedy tokens must be identical on every
row whose oracle top-1/top-2 margin exceeds that bound ("decided" rows),
and on every row the device's token must lie within the bound of the
oracle's maximum (no row may pick a token the oracle scores clearly lower).
Measured errors are appended to $TK_PARITY_LOG (JSON lines) when set, so the
achieved precision is on record next to the bound.
"""

from __future__ import annotations

import json
import os

import torch

LOGIT_TOL = 0.01
LOGIT_COS = 0.9999


def record(name: str, **kv) -> None:
    path = os.environ.get("TK_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps({"test": name, **kv}) + "\n")
    print(name, kv)


def logits_close(got: torch.Tensor, ref: torch.Tensor, tol: float = LOGIT_TOL,
                 cos_min: float = LOGIT_COS) -> tuple[float, float]:
    got, ref = got.float().cpu(), ref.float().cpu()
    span = (ref.max(-1).values - ref.min(-1).values).clamp_min(1e-6)
    err = ((got - ref).abs().max(-1).values / span).max().item()
    cos = torch.nn.functional.cosine_similarity(got, ref, dim=-1).min().item()
    assert err <= tol and cos >= cos_min, (err, cos)
    return err, cos


def greedy_agrees(got: torch.Tensor, ref: torch.Tensor, tol: float = LOGIT_TOL) -> int:
    """Returns the number of decided rows (all of which must agree)."""
    got, ref = got.float().cpu(), ref.float().cpu()
    top2 = ref.topk(2, dim=-1)
    span = ref.max(-1).values - ref.min(-1).values
    decided = (top2.values[:, 0] - top2.values[:, 1]) > tol * span
    g = got.argmax(-1)
    assert (g[decided] == ref.argmax(-1)[decided]).all(), "greedy token differs on a decided row"
    # undecided rows: the device's pick is a near-tie of the oracle's maximum
    picked = ref.gather(1, g[:, None])[:, 0]
    assert ((top2.values[:, 0] - picked) <= tol * span).all(), "greedy pick outside the tie band"
    return int(decided.sum())
