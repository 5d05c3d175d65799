"""Host logic of B200 mode that needs no device.

* the handoff's byte count is the device model's KV per token
  (pdsim/costs.py:137);
* real-clock metric timestamps come from the device completion stamp, clamped
  to [enqueue, poll], while the sim clock is untouched (pdsim/engine.py:102-132);
* resource usage billed per physical GPU beside pdsim's per-instance episode
  sum (pdsim/experiment.py:270-305);
* instance placement over ordinals for the P:D splits the bench runs.
"""

import pytest

import paper_2401_11181_b200 as tk
from paper_2401_11181_b200.control import BusyEpisode
from paper_2401_11181_b200.cuda_executor import place_instance
from paper_2401_11181_b200.engine import Engine
from paper_2401_11181_b200.experiment import ConfigError, _physical_resource
from paper_2401_11181_b200.native import MODELS


def test_cuda_mode_derives_kv_bytes_from_the_model():
    for name in ("opt-13b", "llama-2-7b", "tiny"):
        cfg = tk.config_from_dict({"executor": "cuda", "model": {"name": name}})
        assert cfg.params.kv_bytes_per_token == MODELS[name].kv_bytes_per_token
    assert MODELS["opt-13b"].kv_bytes_per_token == 819_200       # pdsim/costs.py:51
    assert MODELS["llama-2-7b"].kv_bytes_per_token == 524_288
    # sim mode keeps the reference default untouched
    assert tk.config_from_dict({}).params.kv_bytes_per_token == 819_200


def test_cuda_mode_rejects_a_kv_bytes_mismatch():
    with pytest.raises(ConfigError, match="kv_bytes_per_token"):
        tk.config_from_dict({"executor": "cuda", "model": {"name": "llama-2-7b"},
                             "cost_model": {"kv_bytes_per_token": 819_200}})
    with pytest.raises(ConfigError, match="model.name"):
        tk.config_from_dict({"executor": "cuda", "model": {"name": "gpt-5"}})


def test_replay_mode_keeps_the_reference_cost_model():
    """executor "replay" (decisions on pdsim's modeled clock, executed on the
    device): the cost model keeps the reference constants whatever model runs."""
    cfg = tk.config_from_dict({"executor": "replay", "model": {"name": "tiny-long"}})
    assert cfg.params.kv_bytes_per_token == 819_200
    assert cfg.params == tk.config_from_dict({}).params
    with pytest.raises(ConfigError, match="executor"):
        tk.config_from_dict({"executor": "emulate"})


class _Work:
    """A device handle: completes at host time ``t`` (perf_counter seconds)."""

    def __init__(self, t):
        self.t, self.ready = t, False

    def done(self):
        return self.ready

    def done_time(self):
        if not self.ready:
            return None
        return self.t() if callable(self.t) else self.t


def test_real_clock_stamps_device_completion_time():
    import time
    eng = Engine(clock="real")
    seen = []
    eng.register("x", lambda ev: seen.append((eng.now, eng.event_time)))
    eng._t0 = time.perf_counter() - 0.05          # the host clock reads ~50,000 us
    eng.now = 10_000
    early, mid = _Work(eng._t0 + 2_000e-6), _Work(eng._t0 + 20_000e-6)
    eng.after(early, "x", "a")                    # enqueued at 10,000 us
    eng.after(mid, "x", "b")
    early.ready = mid.ready = True
    eng._harvest()                                # polled at >= 50,000 us
    eng.run()
    (now_a, stamp_a), (now_b, stamp_b) = seen
    assert now_a >= 50_000 and now_b >= 50_000    # the loop's clock is the poll time
    assert stamp_a == 10_000                      # clamped up to the enqueue time
    assert stamp_b == 20_000                      # the device's own completion time


def test_sim_clock_event_time_is_fire_time():
    eng = Engine(clock="sim")
    seen = []
    eng.register("x", lambda ev: seen.append((eng.now, eng.event_time)))
    eng.after(500, "x", "a")
    eng.after(900, "x", "b")
    eng.run()
    assert seen == [(500, 500), (900, 900)]


class _Ctl:
    def __init__(self, eps, insts):
        self._eps, self.instances = eps, insts

    def episodes(self):
        return self._eps


def _ep(iid, lo, hi):
    e = BusyEpisode(iid, "prefill" if iid[0] == "p" else "decode")
    e.first_work_start, e.last_work_end = lo, hi
    return e


def test_physical_resource_bills_a_shared_gpu_once():
    eps = [_ep("p0", 0, 600_000), _ep("d0", 100_000, 1_000_000)]
    ctl = _Ctl(eps, {"p0": None, "d0": None})
    co = _physical_resource(ctl, lambda iid: 0, completed=10)
    assert co["gpus_used"] == 1 and co["gpu_resource_us"] == 1_000_000
    assert co["perf_per_dollar_physical"] == pytest.approx(10.0)
    split = _physical_resource(ctl, lambda iid: 0 if iid == "p0" else 1, completed=10)
    assert split["gpus_used"] == 2 and split["gpu_resource_us"] == 1_500_000
    # pdsim's own figure sums episode spans: equal to the split, double-bills co-location
    assert sum(e.span_us for e in eps) == 1_500_000


@pytest.mark.parametrize("n_p,n_d,n_dev,expect", [
    (1, 1, 2, {"p0": 0, "d0": 1}),
    (1, 3, 4, {"p0": 0, "d0": 1, "d1": 2, "d2": 3}),
    (2, 2, 4, {"p0": 0, "p1": 1, "d0": 2, "d1": 3}),
    (2, 6, 8, {"p0": 0, "p1": 1, **{f"d{j}": 2 + j for j in range(6)}}),
    (4, 4, 8, {**{f"p{i}": i for i in range(4)}, **{f"d{j}": 4 + j for j in range(4)}}),
    (1, 1, 1, {"p0": 0, "d0": 0}),
])
def test_placement_of_splits(n_p, n_d, n_dev, expect):
    got = {iid: place_instance(iid, n_p, n_dev) for iid in expect}
    assert got == expect
