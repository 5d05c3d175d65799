"""Replay mode (SURVEY.md section 7 mode 2): the reference's decisions executed on
the device.

``executor: "replay"`` runs the scheduler on pdsim's modeled clock -- so every
dispatch, chunk layout, decode batch and swap is the reference's own decision --
and executes each decision on the GPU through the C ABI before its modeled
completion is scheduled.  These tests take golden configs recorded from the
unmodified pdsim (tests/golden/sched_decisions.json.gz) and require, in ONE run:

* the decision trace is bit-identical to pdsim's (rows, summary, dispatches,
  chunk slices, batch membership per iteration, iteration records);
* the tokens the device generated under those decisions are the fp32 oracle's
  greedy tokens: each sampled request's prompt + generated tokens is run through
  the oracle (teacher-forced, whole sequence, no paging) and at every generated
  position the device's token must be the oracle's argmax where the oracle's
  top-1/top-2 margin exceeds 1% of the logit range, and within that band of the
  maximum everywhere (tests/parity_util.py tolerance).

The device model is the 2-layer tiny OPT with a 10,240-row position table (pdsim's
longest request: 8192-token prompt + 2048 decodes); the cost model keeps the
reference's constants, so decisions are independent of the executing shape.
Wrap points of the reference: pdsim/prefill.py:348 (chunks), pdsim/decode.py:248
(batches).
"""

import gzip
import json
from pathlib import Path

import pytest
import torch

import paper_2401_11181_b200 as tk
from oracle.model_ref import OracleModel, Shape
from paper_2401_11181_b200 import native
from paper_2401_11181_b200.workload import token_ids_for
from parity_util import LOGIT_TOL, record
from test_sched_parity import _trace

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).parent / "golden" / "sched_decisions.json.gz"
MODEL = native.TINY_LONG
# OPT-13B width (2 layers) with the 10,240-row position table: the replay then runs the
# benchmarked kernels -- M=512 pair / 144-wide GEMM schedules, the QKV->page epilogue at
# 40 heads, attention pieces over real prefixes, graph decode steps at many buckets
OPT13B_2L = native.ModelShape("opt13b-2l", native.TK_ARCH_OPT, 2, 5120, 40, 20480, 50272,
                              max_positions=10240)
SEED = 0


def _golden(name):
    with gzip.open(GOLDEN) as fh:
        return json.loads(fh.read())[name]


def _oracle(m=MODEL):
    inst = native.Instance(m, device=0, seed=SEED, kv_pages=8, page_tokens=16, max_chunk=16)
    ora = OracleModel.from_instance(Shape(m.arch, m.n_layers, m.hidden, m.n_heads, m.ffn,
                                          m.vocab, m.max_positions), inst, device="cuda")
    inst.close()
    return ora


def _check_tokens(ora, requests, token_log, picks, model=MODEL):
    """Teacher-forced oracle over prompt + generated tokens of the picked requests."""
    decided = total = 0
    for rid in picks:
        req = requests[rid]
        gen = token_log[rid]
        # first token + one per decode step (pdsim/decode.py:336-351)
        assert len(gen) == req.true_decode_len + 1, (rid, len(gen), req.true_decode_len)
        prompt = token_ids_for(req, model.vocab, SEED)
        seq = prompt + gen[:-1]
        ref = ora.full_forward(seq)[len(prompt) - 1:].float().cpu()
        g = torch.tensor(gen, dtype=torch.long)
        top2 = ref.topk(2, dim=-1)
        span = ref.max(-1).values - ref.min(-1).values
        dec = (top2.values[:, 0] - top2.values[:, 1]) > LOGIT_TOL * span
        assert (g[dec] == ref.argmax(-1)[dec]).all(), f"request {rid}: token differs on a decided step"
        picked = ref.gather(1, g[:, None])[:, 0]
        assert ((top2.values[:, 0] - picked) <= LOGIT_TOL * span).all(), \
            f"request {rid}: token outside the oracle's tie band"
        decided += int(dec.sum())
        total += len(gen)
    return decided, total


@pytest.mark.parametrize("name,n_check,model", [("c1_mixed128_1p1d_roce", 16, MODEL),
                                                ("greedy_swaps", 10, MODEL),
                                                ("coupled_64", 10, MODEL),
                                                ("c1_mixed128_1p1d_roce", 8, OPT13B_2L)],
                         ids=["mixed128-tiny", "greedy_swaps-tiny", "coupled64-tiny",
                              "mixed128-opt13b-width"])
def test_replay_reproduces_reference_decisions_and_oracle_tokens(name, n_check, model):
    case = _golden(name)
    native.MODELS.setdefault(model.name, model)
    cfg = dict(case["config"], executor="replay", model={"name": model.name, "seed": SEED,
                                                               "prefill_pages": 8192})
    res = tk.run_experiment(tk.config_from_dict(cfg), seed=case["seed"])
    got = json.loads(json.dumps(_trace(res)))
    dev = got["summary"].pop("device")
    for key in ("rows", "summary", "dispatches", "chunks", "batches", "iterations"):
        assert got[key] == case[key], f"{name}: replay {key} diverged from pdsim"
    # every decision was executed on the device
    n_chunks = sum(len(v) for v in case["chunks"].values())
    n_iters = sum(len(v) for v in case["batches"].values())
    if name != "coupled_64":
        assert dev["prefill_chunks"] == n_chunks
        assert dev["decode_steps"] == n_iters
    ex_log = res.control.executor.token_log
    requests = {rid: rec.req for rid, rec in res.control.table.items()}
    assert set(ex_log) == set(requests), "every request generated tokens on the device"
    # sample: the longest prompts, the longest decodes, and an even spread of ids (at
    # OPT-13B width, sequences up to 4k tokens: the oracle's dense [H, n, n] scores)
    cap = 4096 if model.hidden > 1024 else 1 << 30
    cand = {r: q for r, q in requests.items() if q.prompt_len + q.true_decode_len <= cap}
    by_prompt = sorted(cand, key=lambda r: -cand[r].prompt_len)[:3]
    by_decode = sorted(cand, key=lambda r: -cand[r].true_decode_len)[:3]
    ids = sorted(cand)
    spread = [ids[int(i * len(ids) / (n_check - 6))] for i in range(n_check - 6)]
    picks = list(dict.fromkeys(by_prompt + by_decode + spread))
    ora = _oracle(model)
    decided, total = _check_tokens(ora, requests, ex_log, picks, model)
    record(f"replay_{name}_{model.name}", requests_checked=len(picks), tokens=total,
           decided=decided, chunks=n_chunks, iterations=n_iters)
    assert decided >= total // 3, (decided, total)
