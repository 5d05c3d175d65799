"""Known-answer and property tests for the host scheduler.

Each block restates the reference's own unit tests for that function
(pdsim tests/test_costs.py, test_prefill.py, test_decode.py, test_engine.py,
test_workload.py, test_control.py) against this package.
"""

import random
import statistics

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2401_11181_b200 as tk
from paper_2401_11181_b200 import costs
from paper_2401_11181_b200.costs import (CostModelParams, chunk_cost, decode_iter_latency,
                                         load_calibration, mixed_iter_latency, pages_needed,
                                         prefill_latency, transfer_latency)
from paper_2401_11181_b200.decode import (DecodeInstance, DecodePolicy, DecodingRequest,
                                          PagedKvStore, admits, reserve_pages)
from paper_2401_11181_b200.engine import Engine, RngStreams, SimulationError, collecting_trace_sink
from paper_2401_11181_b200.prefill import (DecodeLoadView, LengthBucket, PredictorModel,
                                           PrefillPolicy, choose_decode_instance, chunkify,
                                           schedule_round)
from paper_2401_11181_b200.workload import Request, WorkloadSpec, export_trace, generate, load_trace

P = CostModelParams(t_chunk_us=50_000, t_prefill_overhead_us=5_000, decode_a_us=2_000.0,
                    decode_b_us=150.0, decode_c_us_per_token=0.25)


def R(rid, prompt, decode=10, arrival=0):
    return Request(id=rid, arrival_us=arrival, prompt_len=prompt, true_decode_len=decode)


# -- cost model (tests/test_costs.py) ------------------------------------------

def test_cost_kats():
    assert prefill_latency(P, 512, 1) == 55_000
    assert prefill_latency(P, 1024, 1) == 105_000
    assert prefill_latency(P, 1, 1) == prefill_latency(P, 512, 1)
    assert prefill_latency(P, 300, 2) == 60_000
    assert prefill_latency(P, 512, 1, True) * 10 == prefill_latency(P, 512, 1) * 11
    assert decode_iter_latency(P, 1, 0) == 2_150
    assert decode_iter_latency(P, 2, 300) == 2_375
    assert decode_iter_latency(P, 1, 800) - decode_iter_latency(P, 1, 400) == 100
    # banker's rounding exactly as Python round(): 6030.5 -> 6030
    assert decode_iter_latency(CostModelParams(), 1, 150) == 6030


def test_transfer_kats():
    p = CostModelParams(bandwidth_bytes_per_s=25_000_000_000)
    assert costs.kv_transfer_bytes(p, 512) == 419_430_400
    assert transfer_latency(p, 512) == 16_778  # ceil(16777.216)
    nv = CostModelParams(bandwidth_bytes_per_s=300_000_000_000)
    assert transfer_latency(nv, 512) == 1_399
    assert pages_needed(p, 0) == 0 and pages_needed(p, 16) == 1 and pages_needed(p, 17) == 2


def test_mixed_degenerates():
    assert mixed_iter_latency(P, 0, 4, 1000) == decode_iter_latency(P, 4, 1000)
    assert mixed_iter_latency(P, 700, 0, 0, n_prefill=2) == prefill_latency(P, 700, 2)
    with pytest.raises(ValueError):
        mixed_iter_latency(P, 0, 0, 0)


def test_chunk_costs_sum_to_batch_formula():
    parts = [chunk_cost(P, 1, False)] * 5 + [chunk_cost(P, 0, False)] * 2
    assert sum(parts) == prefill_latency(P, 7 * 512, 5)


@given(x=st.integers(1, 10_000), y=st.integers(1, 10_000))
def test_transfer_subadditive(x, y):
    p = CostModelParams(transfer_fixed_us=37)
    lhs = transfer_latency(p, x) + transfer_latency(p, y) - 37
    assert 0 <= lhs - transfer_latency(p, x + y) <= 38


@settings(max_examples=100)
@given(t=st.integers(1, 50_000), more=st.integers(0, 50_000), b=st.integers(1, 512),
       kv=st.integers(0, 500_000))
def test_monotone(t, more, b, kv):
    p = CostModelParams()
    assert prefill_latency(p, t + more, 1) >= prefill_latency(p, t, 1)
    assert decode_iter_latency(p, b, kv + more) >= decode_iter_latency(p, b, kv)
    assert transfer_latency(p, t + more) >= transfer_latency(p, t)


def test_calibration(tmp_path):
    f = tmp_path / "c.json"
    f.write_text('{"preset": "nvlink300", "t_chunk_us": 40000}')
    p = load_calibration(f)
    assert (p.t_chunk_us, p.bandwidth_bytes_per_s) == (40_000, 300_000_000_000)
    assert load_calibration({"preset": "indirect"}).transfer_fixed_us == 200
    for bad, msg in [({"nonsense": 1}, "unknown calibration key"),
                     ({"preset": "modem56k"}, "preset"),
                     ({"mem_capacity_tokens": 1001}, "page_size must divide"),
                     ({"bandwidth_bytes_per_s": 0}, "bandwidth")]:
        with pytest.raises(ValueError, match=msg):
            load_calibration(bad)


# -- prefill (tests/test_prefill.py) ----------------------------------------------

def test_round_orders():
    raw = [R(1, 300), R(2, 18), R(3, 512)]
    assert [r.id for r in schedule_round(PrefillPolicy("fcfs"), raw)[0]] == [1, 2, 3]
    assert [r.id for r in schedule_round(PrefillPolicy("sjf"), raw)[0]] == [2, 1, 3]
    assert [r.id for r in schedule_round(PrefillPolicy("ljf"), raw)[0]] == [3, 1, 2]
    head, tail = schedule_round(PrefillPolicy("sjf", 2), [R(1, 300), R(2, 500), R(3, 1)])
    assert [r.id for r in head] == [1, 2] and [r.id for r in tail] == [3]
    ties = [R(5, 100, arrival=10), R(2, 100), R(1, 100, arrival=10)]
    assert [r.id for r in schedule_round(PrefillPolicy("sjf"), ties)[0]] == [2, 1, 5]


def test_chunk_layout_kat():
    chunks = chunkify([R(0, 18), R(1, 100), R(2, 512), R(3, 900)], 512)
    assert [c.slices for c in chunks] == [
        [(0, 0, 18), (1, 0, 100), (2, 0, 394)], [(2, 394, 118), (3, 0, 394)], [(3, 394, 506)]]
    assert [c.padded for c in chunks] == [0, 0, 6]
    assert chunkify([R(0, 1)], 512)[0].padded == 511


@settings(max_examples=150)
@given(prompts=st.lists(st.integers(1, 1500), min_size=1, max_size=20),
       size=st.integers(1, 700))
def test_chunkify_reassembles(prompts, size):
    chunks = chunkify([R(i, p) for i, p in enumerate(prompts)], size)
    cursor = {}
    for c in chunks:
        assert c.real_tokens + c.padded == size
        for rid, start, n in c.slices:
            assert cursor.get(rid, 0) == start
            cursor[rid] = start + n
    assert cursor == dict(enumerate(prompts))
    assert all(c.padded == 0 for c in chunks[:-1])


def test_predictor_semantics():
    exact = PredictorModel(granularity=200, accuracy=1.0)
    assert exact.predict(R(0, 10, 130), random.Random(0)) == LengthBucket(0, 200)
    b = exact.predict(R(1, 10, 200), random.Random(0))
    assert (b.index, b.lower, b.upper) == (1, 200, 400)
    noisy = PredictorModel(granularity=200, accuracy=0.5)
    rng = random.Random(1)
    assert noisy.predict(R(7, 10, 450), rng) is noisy.predict(R(7, 10, 450), rng)
    assert PredictorModel(granularity=100).effective_accuracy == 0.589
    assert PredictorModel(granularity=400).effective_accuracy == 0.85
    assert PredictorModel().n_buckets == 41


def test_predictor_accuracy_and_confusion():
    m = PredictorModel(granularity=200, accuracy=0.749)
    rng = random.Random(42)
    n = 50_000
    hits = sum(m.predict(R(i, 10, i % 1000 + 1), rng).index == (i % 1000 + 1) // 200
               for i in range(n))
    assert abs(hits / n - 0.749) <= 0.008
    wrong = PredictorModel(granularity=200, accuracy=1e-9, max_decode_len=2000)
    rng = random.Random(4)
    counts = {}
    for i in range(3000):
        idx = wrong.predict(R(i, 10, 1000), rng).index
        assert idx != 5 and 0 <= idx <= 9
        counts[idx] = counts.get(idx, 0) + 1
    assert counts[4] + counts[6] > counts.get(3, 0) + counts.get(7, 0)


def V(i, free, h, l):
    return DecodeLoadView(i, free, h, l, 16)


def test_dispatcher_kats():
    b3 = LengthBucket(3, 200)
    assert choose_decode_instance(R(0, 100), b3, {"d0": V("d0", 10, 5, 0)},
                                  random.Random(0))[0] == "d0"
    loads = {"A": V("A", 10_000, 3, 1), "B": V("B", 10_000, 1, 3)}
    for s in range(10):
        assert choose_decode_instance(R(0, 100), b3, loads, random.Random(s)) == ("B", False)
    loads = {"A": V("A", 1_000, 9, 0), "B": V("B", 10, 0, 9)}
    assert choose_decode_instance(R(0, 100), b3, loads, random.Random(0)) == ("A", False)
    loads = {"A": V("A", 5, 1, 1), "B": V("B", 9, 1, 1)}
    assert choose_decode_instance(R(0, 4_000), b3, loads, random.Random(0)) == ("B", True)
    # equal free tokens in the fallback: the larger id wins (max over (free, id))
    loads = {"d1": V("d1", 5, 0, 0), "d2": V("d2", 5, 0, 0)}
    assert choose_decode_instance(R(0, 4_000), b3, loads, random.Random(0))[0] == "d2"


def test_commit_echo():
    v = V("d0", 100, 0, 0)
    v.commit(R(0, 100), LengthBucket(1, 200))
    assert (v.free_pages, v.heavy, v.light) == (100 - 32, 1, 0)


# -- decode (tests/test_decode.py) -----------------------------------------------------

def D(rid, prompt, decode=64, idx=0, g=16, gen=0):
    d = DecodingRequest(req=R(rid, prompt, decode), bucket=LengthBucket(idx, g))
    d.generated = gen
    return d


def test_admission_kats():
    p10 = CostModelParams(mem_capacity_tokens=160)
    for pol in ("greedy", "reserve_static", "reserve_dynamic"):
        assert admits(DecodePolicy(pol), p10, PagedKvStore(10, 16), [], D(0, 16, idx=2))
    p12 = CostModelParams(mem_capacity_tokens=192)
    s12 = PagedKvStore(12, 16)
    s12.allocate(0, 1)
    inc = D(1, 16, idx=10)
    assert reserve_pages(p12, inc, "lower") == 11
    assert not admits(DecodePolicy("reserve_static"), p12, s12, [D(0, 16, idx=1)], inc)
    s13 = PagedKvStore(13, 16)
    s13.allocate(0, 1)
    assert admits(DecodePolicy("reserve_static"), CostModelParams(mem_capacity_tokens=208),
                  s13, [D(0, 16, idx=1)], inc)
    p20 = CostModelParams(mem_capacity_tokens=320)
    s20 = PagedKvStore(20, 16)
    a, b = D(0, 16, 32, idx=1, gen=15), D(1, 16, 256, idx=10)
    s20.allocate(0, 2)
    s20.allocate(1, 1)
    inc = D(2, 64, idx=4)
    assert not admits(DecodePolicy("reserve_static"), p20, s20, [a, b], inc)
    assert admits(DecodePolicy("reserve_dynamic"), p20, s20, [a, b], inc)
    full = PagedKvStore(10, 16)
    full.allocate(0, 10)
    assert not admits(DecodePolicy("reserve_dynamic"), p10, full, [D(0, 144, 4, gen=3)], D(1, 64))
    capped = PagedKvStore(10, 16)
    capped.allocate(0, 2)
    assert not admits(DecodePolicy("greedy", max_batch=1), p10, capped, [D(0, 16)], D(1, 16))


def test_store_invariants():
    s = PagedKvStore(4, 16)
    s.allocate(0, 3)
    with pytest.raises(SimulationError, match="exceed capacity"):
        s.allocate(1, 2)
    s = PagedKvStore(10, 16)
    s.allocate(0, 4)
    assert s.evict(0) == 4 and s.resident_pages == 0 and s.swapped == {0: 4}
    assert s.swap_in(0) == 4 and s.resident == {0: 4} and s.free_pages == 6


class Stub:
    def __init__(self):
        self.completed, self.swaps, self.busy = [], [], []

    def note_kv_arrival(self, i): pass
    def note_busy(self, i, a, b): self.busy.append((a, b))
    def note_swap(self, req, pages): self.swaps.append((req.id, pages))
    def record_completion(self, req): self.completed.append(req.id)
    def inflight_to(self, i): return 0


def test_iteration_formula_and_release():
    params = CostModelParams(decode_a_us=2000, decode_b_us=150, decode_c_us_per_token=0.25,
                             mem_capacity_tokens=160_000)
    eng, ctl = Engine(), Stub()
    inst = DecodeInstance("d0", eng, params, DecodePolicy("greedy"), ctl)
    for rid, prompt in ((0, 100), (1, 200)):
        r = R(rid, prompt, 1)
        r.set_phase("transferring")
        eng.schedule(0, "d0", "kv_arrival", {"req": r, "bucket": LengthBucket(0, 16)})
    eng.run()
    rec = inst.iteration_log[0]
    assert (rec.batch_size, rec.kv_tokens, rec.latency_us) == (2, 300, 2375)
    assert ctl.completed == [0, 1] and inst.store.resident_pages == 0


def test_victims_largest_first():
    eng = Engine()
    inst = DecodeInstance("d0", eng, CostModelParams(mem_capacity_tokens=192),
                          DecodePolicy("greedy"), Stub())
    small, big = D(0, 64), D(1, 128)
    inst.store.allocate(0, 4)
    inst.store.allocate(1, 8)
    inst.running = [small, big]
    assert inst.swap_out(6, exclude=D(2, 16)) == 8
    assert 1 in inst.store.swapped and big in inst.queue and big.was_swapped
    inst2 = DecodeInstance("d1", eng, CostModelParams(mem_capacity_tokens=64),
                           DecodePolicy("greedy"), Stub())
    inst2.store.allocate(0, 4)
    inst2.running = [D(0, 64)]
    with pytest.raises(SimulationError, match="cannot fit"):
        inst2.swap_out(10, exclude=D(1, 160))


def _overcommit(policy):
    return tk.config_from_dict({
        "workload": {"class": "LPLD", "n_requests": 6, "lengths": {
            "light_prompt": {"median": 16, "sigma": 0.0, "lo": 16, "hi": 16},
            "light_decode": {"median": 64, "sigma": 0.0, "lo": 64, "hi": 64}}},
        "policies": {"prefill": "fcfs", "decode": policy},
        "predictor": {"granularity": 16, "accuracy": 1.0},
        "cost_model": {"mem_capacity_tokens": 320, "t_chunk_us": 500,
                       "t_prefill_overhead_us": 10, "decode_a_us": 100, "decode_b_us": 5,
                       "decode_c_us_per_token": 0.01, "preset": "nvlink300"}})


def test_greedy_thrashes_reserve_does_not():
    g = tk.run_experiment(_overcommit("greedy"), seed=5)
    assert g.summary["swap_events_total"] > 0 and g.summary["completed"] == 6
    for pol in ("reserve_dynamic", "reserve_static"):
        assert tk.run_experiment(_overcommit(pol), seed=5).summary["swap_events_total"] == 0
    assert all(r["wait_us"] <= r["ttft_us"] <= r["jct_us"] for r in g.rows)


# -- engine (tests/test_engine.py) ----------------------------------------------------------

def test_engine_contract():
    eng = Engine()
    fired = []
    eng.register("a", lambda e: fired.append((e.fire_time, e.data.get("tag"))))
    for tag in ("x", "y", "z"):
        eng.schedule(5, "a", "t", {"tag": tag})
    h = eng.schedule(1, "a", "doomed")
    eng.cancel(h)
    eng.schedule(2, "a", "t", {"tag": "early"})
    eng.run(until=3)
    assert fired == [(2, "early")] and eng.now == 3
    eng.run()
    assert [t for _, t in fired] == ["early", "x", "y", "z"]
    with pytest.raises(SimulationError):
        eng.schedule(4, "a", "t")
    capped = Engine(max_events=10)
    capped.register("a", lambda e: capped.schedule(capped.now, "a", "t"))
    capped.schedule(0, "a", "t")
    with pytest.raises(SimulationError, match="event cap"):
        capped.run()
    e2 = Engine()
    n = []
    e2.register("a", lambda e: n.append(1))
    for t in range(5):
        e2.schedule(t, "a", "t")
    e2.run(stop=lambda: len(n) >= 2)
    assert len(n) == 2


def test_rng_streams():
    a = [RngStreams(99).stream("a").random() for _ in range(1)]
    s = RngStreams(99)
    s.stream("b").random()
    assert s.stream("a").random() == a[0]
    # derivation pinned: first draw of stream "workload" for seed 0
    import hashlib
    seed = int.from_bytes(hashlib.sha256(b"0:workload").digest()[:8], "big")
    assert RngStreams(0).stream("workload").random() == random.Random(seed).random()


def test_device_handles_through_engine():
    class Done:
        def __init__(self):
            self.n = 0

        def done(self):
            self.n += 1
            return self.n > 2

    eng = Engine()
    got = []
    eng.register("a", lambda e: got.append((eng.now, e.kind)))
    eng.after(7, "a", "modeled")
    eng.after(Done(), "a", "device")
    eng.run()
    assert ("device" in [k for _, k in got]) and (7, "modeled") in got


# -- workload (tests/test_workload.py) ---------------------------------------------------------

def _rng(seed=0):
    return RngStreams(seed).stream("workload")


@pytest.mark.parametrize("klass", ["LPLD", "LPHD", "HPLD", "HPHD"])
def test_class_bounds(klass):
    for r in generate(WorkloadSpec(klass=klass, n_requests=300), _rng(3)):
        assert r.klass == klass


def test_workload_statistics():
    lp = generate(WorkloadSpec(klass="LPLD", n_requests=5000), _rng(1))
    assert 14.4 <= statistics.median(r.prompt_len for r in lp) <= 21.6
    mix = generate(WorkloadSpec(n_requests=5000), _rng(2))
    assert abs(sum(r.heavy_decode for r in mix) / 5000 - 0.5) <= 0.03
    lens = [r.prompt_len for r in mix]
    assert max(lens) / min(lens) >= 100


def test_poisson_and_validation():
    reqs = generate(WorkloadSpec(klass="LPLD", n_requests=50, arrival="poisson",
                                 rate_per_s=100), _rng(5))
    assert [r.arrival_us for r in reqs] == sorted(r.arrival_us for r in reqs)
    with pytest.raises(ValueError, match="rate_per_s"):
        WorkloadSpec(klass="LPLD", arrival="poisson", rate_per_s=0).validate()
    r = R(0, 10)
    r.set_phase("decoding")
    with pytest.raises(SimulationError):
        r.set_phase("queued")


def test_trace_io(tmp_path):
    src = tmp_path / "in.csv"
    src.write_text("arrival_us,prompt_len,decode_len,sla_us\n0,18,100,250000\n5,9,3,\n")
    out = tmp_path / "out.csv"
    export_trace(load_trace(src), out)
    assert out.read_text() == src.read_text()
    src.write_text("arrival_us,prompt_len,decode_len\n500,10,10\n0,20,20\n")
    assert [r.arrival_us for r in load_trace(src)] == [0, 500]
    src.write_text("arrival_us,prompt_len,decode_len\n0,18,100\nnope,1,1\n")
    with pytest.raises(ValueError, match="line 3"):
        load_trace(src)
    src.write_text("bad,header\n")
    with pytest.raises(ValueError, match="line 1"):
        load_trace(src)


# -- control plane (tests/test_control.py) ------------------------------------------------------

def _control():
    from paper_2401_11181_b200.control import ControlPlane, FlipPolicy
    from paper_2401_11181_b200.coupled import CoupledConfig
    eng = Engine()
    return eng, ControlPlane(eng, RngStreams(0), CostModelParams(),
                             prefill_policy=PrefillPolicy(), decode_policy=DecodePolicy(),
                             dispatch_policy="power_of_two", predictor=PredictorModel(),
                             flip_policy=FlipPolicy(), coupled_config=CoupledConfig())


def test_routing_alternates_and_stale_snapshot():
    res = tk.run_experiment(tk.config_from_dict({
        "cluster": {"prefill": 2, "decode": 1}, "workload": {"class": "LPLD", "n_requests": 8}}),
        seed=3)
    assert {r["prefill_instance"] for r in res.rows} == {"p0", "p1"}
    _, ctl = _control()
    p0 = ctl.add_prefill_instance("p0")
    d0 = ctl.add_decode_instance("d0")
    ctl.broadcast_loads()
    before = p0.loads["d0"].free_pages
    d0.store.allocate(999, 100)
    assert p0.loads["d0"].free_pages == before
    ctl.broadcast_loads()
    assert p0.loads["d0"].free_pages == before - 100


def test_monitor_cadence_and_accounting():
    res = tk.run_experiment(tk.config_from_dict({
        "workload": {"class": "LPLD", "n_requests": 4}, "events": True}), seed=1)
    ticks = [e["t"] for e in res.events if e["kind"] == "monitor_tick"]
    assert ticks[0] == 0 and all(b - a == 100_000 for a, b in zip(ticks, ticks[1:]))
    _, ctl = _control()
    ctl.add_prefill_instance("p0")
    ctl.add_decode_instance("d0")
    ctl.note_busy("p0", 0, 1_000_000)
    ctl.note_busy("d0", 1_000_000, 3_000_000)
    assert sum(ep.span_us for ep in ctl.episodes()) == 3_000_000
    req = R(0, 10, 5)
    ctl.route_request(req)
    ctl.note_first_token(req, 0)
    ctl.record_completion(req)
    with pytest.raises(SimulationError, match="twice"):
        ctl.record_completion(req)


def test_config_errors_and_cli(tmp_path):
    with pytest.raises(tk.ConfigError, match="bogus"):
        tk.config_from_dict({"bogus": 1})
    with pytest.raises(tk.ConfigError, match="executor"):
        tk.config_from_dict({"executor": "tpu"})
    from paper_2401_11181_b200.cli import main
    cfg = tmp_path / "c.json"
    cfg.write_text('{"workload": {"n_requests": 16}}')
    assert main(["run", "--config", str(cfg), "--out", str(tmp_path / "a")]) == 0
    assert main(["run", "--config", str(cfg), "--seed", "1", "--out", str(tmp_path / "b")]) == 0
    cfg.write_text('{"cluster": {"prefill": 0}}')
    assert main(["run", "--config", str(cfg), "--out", str(tmp_path / "c")]) == 2
