"""Chunk-level KV streaming (PAPER.md:441-444 future work).

Off by default, so every reference-parity test runs the reference's semantics.
With ``kv_streaming: chunk`` each prefilled chunk's KV leaves for the decode
instance as soon as the chunk is done; only the last part is on the TTFT->decode
critical path.  Sim mode models each part as transfer_latency(part tokens)
(pdsim/costs.py:130-139).
"""
import pytest

import paper_2401_11181_b200 as tk
from paper_2401_11181_b200 import costs
from paper_2401_11181_b200.experiment import ConfigError


def _one(prompt: int, streaming: str, preset: str = "default") -> dict:
    cm = {"t_chunk_us": 50_000, "t_prefill_overhead_us": 5_000, "decode_a_us": 2_000,
          "decode_b_us": 150, "decode_c_us_per_token": 0.0}
    if preset != "default":
        cm["preset"] = preset
    cfg = tk.config_from_dict({
        "workload": {"class": "HPLD", "n_requests": 1, "lengths": {
            "heavy_prompt": {"median": prompt, "sigma": 0.0, "lo": prompt, "hi": prompt},
            "light_decode": {"median": 1, "sigma": 0.0, "lo": 1, "hi": 1}}},
        "predictor": {"enabled": False}, "cost_model": cm, "events": True,
        "kv_streaming": streaming})
    return tk.run_experiment(cfg, seed=0)


def test_config_validation():
    with pytest.raises(ConfigError):
        tk.config_from_dict({"kv_streaming": "layer"})
    assert tk.config_from_dict({}).kv_streaming == "off"


@pytest.mark.parametrize("prompt", [2048, 4000, 8192])
def test_streamed_arrival_is_first_token_plus_last_part(prompt):
    off, on = _one(prompt, "off"), _one(prompt, "chunk")
    p = costs.load_calibration({})
    a_off = [e for e in off.events if e["kind"] == "kv_arrival"][0]["t"]
    a_on = [e for e in on.events if e["kind"] == "kv_arrival"][0]["t"]
    ttft = off.rows[0]["ttft_us"]
    assert on.rows[0]["ttft_us"] == ttft  # prefill itself is unchanged
    assert a_off == ttft + costs.transfer_latency(p, prompt)
    # every earlier 512-token part (16.8 ms at 25 GB/s) finishes inside the next
    # 50 ms chunk, so only the tail part remains after the first token
    tail = prompt - 512 * ((prompt - 1) // 512)
    assert a_on == ttft + costs.transfer_latency(p, tail)
    assert off.rows[0]["jct_us"] - on.rows[0]["jct_us"] == a_off - a_on


def test_slow_link_arrival_is_latest_part_end():
    # a link much slower than the chunks: the big first part (512 tokens) ends after
    # the short tail (488 tokens) sent one chunk later, and bounds the arrival
    cfg = {"t_chunk_us": 5_000, "t_prefill_overhead_us": 1, "bandwidth_bytes_per_s": 10**9}
    res = tk.run_experiment(tk.config_from_dict({
        "workload": {"class": "HPLD", "n_requests": 1, "lengths": {
            "heavy_prompt": {"median": 1000, "sigma": 0.0, "lo": 1000, "hi": 1000},
            "light_decode": {"median": 1, "sigma": 0.0, "lo": 1, "hi": 1}}},
        "predictor": {"enabled": False}, "cost_model": cfg, "events": True,
        "kv_streaming": "chunk"}), seed=0)
    p = costs.load_calibration(cfg)
    first_done = [e for e in res.events if e["kind"] == "chunk_done"][0]["t"]
    arrival = [e for e in res.events if e["kind"] == "kv_arrival"][0]["t"]
    assert arrival == first_done + costs.transfer_latency(p, 512)
    assert arrival > res.rows[0]["ttft_us"] + costs.transfer_latency(p, 488)


@pytest.mark.parametrize("n_prefill,n_decode", [(1, 1), (2, 2)])
def test_mixed_workload_completes_and_is_deterministic(n_prefill, n_decode):
    cfg = tk.config_from_dict({"cluster": {"prefill": n_prefill, "decode": n_decode},
                               "workload": {"n_requests": 64}, "kv_streaming": "chunk"})
    a = tk.run_experiment(cfg, seed=4)
    b = tk.run_experiment(cfg, seed=4)
    assert a.summary["completed"] == 64
    assert [r["jct_us"] for r in a.rows] == [r["jct_us"] for r in b.rows]
    off = tk.run_experiment(tk.config_from_dict({"cluster": {"prefill": n_prefill,
                                                             "decode": n_decode},
                                                 "workload": {"n_requests": 64}}), seed=4)
    # the handoff tail shrinks; prefill-side timing is the same work
    assert a.summary["jct"]["avg_us"] <= off.summary["jct"]["avg_us"] * 1.02


def _two_waves(tmp_path, prompt=1500):
    lines = ["arrival_us,prompt_len,decode_len"]
    for wave in (0, 1_500_000):
        lines += [f"{wave},{prompt + 37 * i},{10 + i}" for i in range(8)]
    path = tmp_path / "waves.csv"
    path.write_text("\n".join(lines) + "\n")
    return path


def test_streaming_with_flips_completes(tmp_path):
    """Flips (pdsim/control.py:408-482) with streamed handoffs in flight: a decode
    instance being drained is excluded from dispatch, so streams only target live
    decode instances; every request completes."""
    cfg = tk.config_from_dict({
        "cluster": {"prefill": 2, "decode": 2},
        "workload": {"class": "Trace", "trace_path": str(_two_waves(tmp_path))},
        "flip": {"enabled": True, "threshold": 0.5, "window_us": 400_000},
        "cost_model": {"t_chunk_us": 2_000, "t_prefill_overhead_us": 50, "decode_a_us": 200,
                       "decode_b_us": 5, "decode_c_us_per_token": 0.001},
        "kv_streaming": "chunk", "max_events": 2_000_000})
    res = tk.run_experiment(cfg, seed=4)
    assert res.summary["completed"] == 16
    assert res.summary["flips_completed"] >= 1
    for row in res.rows:
        assert row["ttft_us"] <= row["jct_us"]
