"""Scheduler decision parity with the reference.

Golden fixtures (tests/golden/sched_decisions.json.gz, made by
tests/golden/make_sched_golden.py from the unmodified pdsim) pin, per config
and seed: requests.csv rows, the summary, every dispatch, every chunk's slice
layout and start time, and every decode iteration's batch membership and
record.  The live-reference variant re-runs pdsim where it is available.
"""

import gzip
import json
from pathlib import Path

import pytest

import paper_2401_11181_b200 as tk

GOLDEN = Path(__file__).parent / "golden" / "sched_decisions.json.gz"


def _golden():
    with gzip.open(GOLDEN) as fh:
        return json.loads(fh.read())


CASES = _golden()


def _trace(result):
    insts = result.control.instances
    return {
        "rows": result.rows,
        "summary": result.summary,
        "dispatches": {k: [list(d) for d in v.dispatches]
                       for k, v in insts.items() if hasattr(v, "dispatches")},
        "chunks": {k: [[t, [list(s) for s in sl], pad] for t, sl, pad in v.chunk_log]
                   for k, v in insts.items() if getattr(v, "chunk_log", None)},
        "batches": {k: [list(b) for b in v.batch_log]
                    for k, v in insts.items() if getattr(v, "batch_log", None)},
        "iterations": {k: [list(vars(r).values()) for r in v.iteration_log]
                       for k, v in insts.items() if hasattr(v, "iteration_log")},
    }


@pytest.mark.parametrize("name", sorted(CASES))
def test_decisions_match_reference_golden(name):
    case = CASES[name]
    res = tk.run_experiment(tk.config_from_dict(case["config"]), seed=case["seed"])
    got = json.loads(json.dumps(_trace(res)))
    for key in ("rows", "summary", "dispatches", "chunks", "batches", "iterations"):
        assert got[key] == case[key], f"{name}: {key} diverged from pdsim"


@pytest.mark.parametrize("seed", [0, 11])
@pytest.mark.parametrize("cfg", [
    {"cluster": {"prefill": 3, "decode": 5}, "cost_model": {"preset": "indirect"},
     "workload": {"n_requests": 200}},
    {"policies": {"decode": "greedy", "sched_batch": 4},
     "cost_model": {"mem_capacity_tokens": 9600}},
])
def test_decisions_match_live_reference(pdsim_ref, cfg, seed):
    ref = pdsim_ref.run_experiment(pdsim_ref.config_from_dict(cfg), seed=seed)
    mine = tk.run_experiment(tk.config_from_dict(cfg), seed=seed)
    assert mine.rows == ref.rows
    assert mine.summary == ref.summary
    for iid, inst in ref.control.instances.items():
        other = mine.control.instances[iid]
        if hasattr(inst, "dispatches"):
            assert other.dispatches == inst.dispatches
        if hasattr(inst, "iteration_log"):
            assert [vars(r) for r in other.iteration_log] == [vars(r) for r in inst.iteration_log]


def test_event_trace_identical_to_reference(pdsim_ref):
    cfg = {"cluster": {"prefill": 2, "decode": 2}, "workload": {"n_requests": 48},
           "events": True}
    ref = pdsim_ref.run_experiment(pdsim_ref.config_from_dict(cfg), seed=3)
    mine = tk.run_experiment(tk.config_from_dict(cfg), seed=3)
    assert mine.events == ref.events


def test_spec_engine_oracle():
    """SPEC.md:543 engine oracle: 1x512 prompt, 1 decode step, nvlink300."""
    cfg = tk.config_from_dict({
        "workload": {"class": "LPLD", "n_requests": 1, "lengths": {
            "light_prompt": {"median": 512, "sigma": 0.0, "lo": 512, "hi": 512},
            "light_decode": {"median": 1, "sigma": 0.0, "lo": 1, "hi": 1}}},
        "predictor": {"enabled": False},
        "cost_model": {"preset": "nvlink300", "t_chunk_us": 50_000,
                       "t_prefill_overhead_us": 5_000, "decode_a_us": 2_000,
                       "decode_b_us": 150, "decode_c_us_per_token": 0.0},
        "events": True})
    res = tk.run_experiment(cfg, seed=0)
    row = res.rows[0]
    assert row["ttft_us"] == 55_000
    assert row["jct_us"] == 58_549
    arrivals = [e for e in res.events if e["kind"] == "kv_arrival"]
    assert arrivals[0]["t"] == 56_399
