"""The unchanged scheduler driving real device work (executor="cuda").

Checks conservation and causality of a measured-clock run (every request
prefilled, handed off and decoded exactly as many steps as pdsim would run
it), that the physical KV pages come back to the pools, and that the first
scheduling round's chunk layout equals the simulated run's (it depends only
on the burst, not on timing).
"""

import pytest

import paper_2401_11181_b200 as tk
from paper_2401_11181_b200.experiment import make_executor, run_experiment

pytestmark = pytest.mark.gpu

CFG = {
    "cluster": {"prefill": 1, "decode": 1},
    "workload": {"n_requests": 24, "mixture": {"LPLD": 0.5, "LPHD": 0.5},
                 "lengths": {"heavy_decode": {"hi": 300}}},
    "cost_model": {"preset": "nvlink300", "mem_capacity_tokens": 16000},
    "model": {"name": "tiny", "prefill_pages": 1024, "staging_pages": 256,
              "max_decode_batch": 64},
}


def test_cuda_executor_end_to_end():
    cfg = tk.config_from_dict(dict(CFG, executor="cuda"))
    res = run_experiment(cfg, seed=0)
    s = res.summary
    assert s["completed"] == s["n_requests"] == 24
    for row in res.rows:
        assert 0 <= row["wait_us"] <= row["ttft_us"] <= row["jct_us"]
    dev = s["device"]
    reqs = tk.generate(cfg.workload_spec, tk.RngStreams(0).stream("workload"))
    assert dev["prefill_tokens"] == sum(r.prompt_len for r in reqs)
    assert dev["decode_tokens"] == sum(r.true_decode_len for r in reqs)
    assert dev["kv_bytes_sent"] == sum(
        -(-r.prompt_len // 16) for r in reqs) * 16 * 2 * 2 * 256 * 2  # pages x page bytes
    assert dev["predict_calls"] >= 1
    # the first round's chunk layout does not depend on timing
    sim = run_experiment(tk.config_from_dict(CFG), seed=0)
    n = len(sim.control.instances["p0"].chunk_log)
    first_sim = [c[1:] for c in sim.control.instances["p0"].chunk_log][: min(n, 3)]
    first_dev = [c[1:] for c in res.control.instances["p0"].chunk_log][: len(first_sim)]
    assert first_dev == first_sim


def test_cuda_executor_greedy_swaps_restore_pages():
    cfg = tk.config_from_dict({
        "executor": "cuda",
        "workload": {"class": "LPLD", "n_requests": 6, "lengths": {
            "light_prompt": {"median": 16, "sigma": 0.0, "lo": 16, "hi": 16},
            "light_decode": {"median": 64, "sigma": 0.0, "lo": 64, "hi": 64}}},
        "policies": {"prefill": "fcfs", "decode": "greedy"},
        "predictor": {"granularity": 16, "accuracy": 1.0},
        "cost_model": {"mem_capacity_tokens": 320, "preset": "nvlink300"},
        "model": {"name": "tiny", "prefill_pages": 64, "staging_pages": 64,
                  "max_decode_batch": 16},
    })
    executor = make_executor(cfg)
    res = run_experiment(cfg, seed=5, executor=executor)
    assert res.summary["completed"] == 6
    assert res.summary["swap_events_total"] > 0
    # every physical page is back in its pool
    for iid, pool in executor.pools.items():
        assert len(pool.free) == pool.n_pages, iid


def test_cuda_executor_coupled_baseline():
    """The vLLM-like coupled instance (pdsim/coupled.py) on the device."""
    cfg = dict(CFG, system="coupled", cluster={"coupled": 1}, executor="cuda")
    executor = make_executor(tk.config_from_dict(cfg))
    res = run_experiment(tk.config_from_dict(cfg), seed=0, executor=executor)
    s = res.summary
    assert s["completed"] == s["n_requests"] == 24
    for row in res.rows:
        assert row["ttft_us"] <= row["jct_us"]
    reqs = tk.generate(tk.config_from_dict(cfg).workload_spec, tk.RngStreams(0).stream("workload"))
    assert s["device"]["prefill_tokens"] == sum(r.prompt_len for r in reqs)
    assert s["device"]["decode_tokens"] == sum(r.true_decode_len for r in reqs)
    for pool in executor.pools.values():
        assert len(pool.free) == pool.n_pages


def test_cuda_executor_chunk_kv_streaming_matches_whole_handoff():
    """kv_streaming=chunk: pages leave after each chunk (complete pages only, the
    straddling page with the next part); the decode side sees the same KV, so
    the generated tokens equal the whole-request handoff's."""
    def run(streaming, n, seed):
        cfg = tk.config_from_dict({
            "executor": "cuda", "kv_streaming": streaming,
            "workload": {"class": "HPLD", "n_requests": n, "lengths": {
                "heavy_prompt": {"median": 700, "sigma": 0.3, "lo": 520, "hi": 1000},
                "light_decode": {"median": 8, "sigma": 0.0, "lo": 8, "hi": 8}}},
            "cost_model": {"preset": "nvlink300", "mem_capacity_tokens": 16000},
            "model": {"name": "tiny", "prefill_pages": 256, "staging_pages": 256,
                      "max_decode_batch": 16}})
        ex = make_executor(cfg)
        res = run_experiment(cfg, seed=seed, executor=ex)
        assert res.summary["completed"] == n
        for iid, pool in ex.pools.items():
            assert len(pool.free) == pool.n_pages, iid
        return res, ex

    # one request: batch of one at every step, so the decode arithmetic is identical
    (r0, e0), (r1, e1) = run("off", 1, 0), run("chunk", 1, 0)
    assert e1.first_token == e0.first_token and e1.last_token == e0.last_token
    assert e1.stats["kv_bytes_sent"] == e0.stats["kv_bytes_sent"]
    # several requests: same pages moved in total, same first tokens
    (r0, e0), (r1, e1) = run("off", 6, 2), run("chunk", 6, 2)
    assert e1.first_token == e0.first_token
    assert e1.stats["kv_bytes_sent"] == e0.stats["kv_bytes_sent"]


def test_cuda_executor_flip_keeps_device_state(tmp_path):
    """Instance flips on the device (pdsim/control.py:408-482; reference test
    tests/test_control.py:145-157 on its two-wave trace): the role changes
    without a new device instance -- same weights, pool and streams -- and every
    request completes and every page returns to its pool."""
    lines = ["arrival_us,prompt_len,decode_len"]
    for wave in (0, 1_500_000):
        lines += [f"{wave},{20 + i},{10 + i}" for i in range(8)]
    trace = tmp_path / "waves.csv"
    trace.write_text("\n".join(lines) + "\n")
    cfg = tk.config_from_dict({
        "executor": "cuda", "cluster": {"prefill": 2, "decode": 2},
        "workload": {"class": "Trace", "trace_path": str(trace)},
        "flip": {"enabled": True, "threshold": 0.5, "window_us": 400_000},
        "cost_model": {"preset": "nvlink300", "mem_capacity_tokens": 4096},
        "model": {"name": "tiny", "prefill_pages": 128, "staging_pages": 64,
                  "max_decode_batch": 16}})
    ex = make_executor(cfg)
    res = run_experiment(cfg, seed=4, executor=ex)
    handles = {k: id(v) for k, v in ex.insts.items()}
    assert res.summary["completed"] == 16
    assert res.summary["flips_completed"] >= 1
    assert ex.stats["flips"] == res.summary["flips_completed"]
    assert set(handles) == {"p0", "p1", "d0", "d1"}  # no instance created by a flip
    for rec in res.control.flip_records:
        assert 5_000 <= rec.latency_us <= 7_000
    for iid, pool in ex.pools.items():
        assert len(pool.free) == pool.n_pages, iid


def test_cuda_executor_streaming_two_by_two_colocated():
    """kv_streaming=chunk with 2 prefill + 2 decode instances sharing one device:
    every request completes and every physical page returns to its pool."""
    cfg = tk.config_from_dict({
        "executor": "cuda", "kv_streaming": "chunk", "cluster": {"prefill": 2, "decode": 2},
        "workload": {"n_requests": 24, "mixture": {"HPLD": 0.5, "LPLD": 0.5},
                     "lengths": {"heavy_prompt": {"hi": 800}}},
        "cost_model": {"preset": "nvlink300", "mem_capacity_tokens": 16000},
        "model": {"name": "tiny", "prefill_pages": 512, "staging_pages": 256,
                  "max_decode_batch": 32}})
    ex = make_executor(cfg)
    res = run_experiment(cfg, seed=3, executor=ex)
    assert res.summary["completed"] == 24
    assert not ex._streams
    for iid, pool in ex.pools.items():
        assert len(pool.free) == pool.n_pages, iid
