"""KV handoff engines and the disaggregated system across GPUs.

* Both handoff engines (tk_kv_send_ex: the SM page-copy kernel and the copy
  engines) move scattered pages bit-exactly, on one device (co-located P and D)
  and -- with two or more devices -- from one GPU's pool into a peer's over
  NVLink, after which decode on the receiver equals decode on the sender
  (pdsim/prefill.py:420-424, the handoff the reference models with
  costs.py:130-139).
* A 1P:1D run with the instances on two GPUs (BASELINE.json configs[2]) through
  the unchanged scheduler: every request completes, the handoff bytes are the
  prompts' pages, every page returns to its pool.
* Completion stamps (CUDA events mapped to the host clock) order correctly and
  physical-GPU accounting bills a shared GPU once.
Tests needing two devices skip on a one-GPU box.
"""

import ctypes

import numpy as np
import pytest

import paper_2401_11181_b200 as tk
from paper_2401_11181_b200 import native
from paper_2401_11181_b200.experiment import run_experiment

pytestmark = pytest.mark.gpu

PT = 16


def _n_dev() -> int:
    try:
        return native.device_count()
    except Exception:  # CPU container: collected, deselected by -m "not gpu"
        return 0


def _pairs():
    n = _n_dev()
    out = [(0, 0)]
    if n >= 2:
        out += [(0, 1), (1, 0), (0, n - 1)]
    return out


def _seed_pages(inst, pages, rng):
    pb = inst.page_bytes
    data = rng.integers(0, 256, size=len(pages) * pb, dtype=np.uint8)
    h = native.host_alloc(len(pages) * pb)
    try:
        ctypes.memmove(h, data.ctypes.data, len(pages) * pb)
        inst.swap_in(pages, h).wait()
    finally:
        native.host_free(h)
    return data


def _read_pages(inst, pages):
    pb = inst.page_bytes
    h = native.host_alloc(len(pages) * pb)
    try:
        inst.swap_out(pages, h).wait()
        return np.frombuffer((ctypes.c_uint8 * (len(pages) * pb)).from_address(h),
                             dtype=np.uint8).copy()
    finally:
        native.host_free(h)


@pytest.mark.parametrize("engine", ["sm", "ce", "auto"])
@pytest.mark.parametrize("pair", _pairs())
def test_kv_send_engines_bit_exact(engine, pair):
    src_dev, dst_dev = pair
    model = native.TINY_OPT
    n = 300
    p = native.Instance(model, device=src_dev, seed=5, kv_pages=n + 40, max_chunk=64)
    d = native.Instance(model, device=dst_dev, seed=5, kv_pages=n + 70, max_chunk=64)
    rng = np.random.default_rng(7)
    # distinct pages, scattered, with one run of consecutive pages on both sides
    # (the copy engine coalesces runs)
    src_run, dst_run = list(range(n + 20, n + 30)), list(range(n + 50, n + 60))
    src = [x for x in rng.permutation(n + 40).tolist() if x not in src_run][: n - 10]
    dst = [x for x in rng.permutation(n + 70).tolist() if x not in dst_run][: n - 10]
    src[10:10] = src_run
    dst[10:10] = dst_run
    data = _seed_pages(p, src, rng)
    ev = p.kv_send(src, d, dst, engine)
    ev.wait()
    assert ev.elapsed_ns > 0
    assert np.array_equal(_read_pages(d, dst), data)
    p.close(), d.close()


def test_kv_send_engine_is_validated():
    p = native.Instance(native.TINY_OPT, device=0, seed=5, kv_pages=8, max_chunk=64)
    with pytest.raises(ValueError):
        p.kv_send([0], p, [1], "dma")
    p.close()


@pytest.mark.skipif(_n_dev() < 2, reason="needs two GPUs")
def test_cross_gpu_handoff_then_decode_on_receiver():
    """Prefill on GPU 0, pages sent to GPU 1 over NVLink, decode on GPU 1 gives
    the logits decode on GPU 0 gives (same weights: same seed)."""
    from paper_2401_11181_b200.workload import Request, token_ids_for
    model = native.TINY_OPT
    n_tok = 300
    req = Request(id=0, arrival_us=0, prompt_len=n_tok, true_decode_len=4)
    ids = token_ids_for(req, model.vocab, seed=1)
    n_pages = (n_tok + 4 + PT - 1) // PT
    for engine in ("sm", "ce"):
        p = native.Instance(model, device=0, seed=5, kv_pages=n_pages, max_chunk=512)
        d = native.Instance(model, device=1, seed=5, kv_pages=n_pages + 9, max_chunk=64)
        bt = list(range(n_pages))
        ev, toks = p.prefill_chunk(ids, [(0, n_tok, 0, n_pages, 1)], bt)
        ev.wait()
        first = int(toks[0])
        src = bt[: (n_tok + PT - 1) // PT]
        dst = [n_pages + 8 - i for i in range(len(src))]
        p.kv_send(src, d, dst, engine).wait()
        for s_, d_ in zip(src, dst):
            assert np.array_equal(p.read_page(s_), d.read_page(d_))
        stride = n_pages
        bt_dst = dst + list(range(len(dst), stride))
        e1, _, l1 = p.decode_step([first], [n_tok], bt, stride, want_logits=True)
        e2, _, l2 = d.decode_step([first], [n_tok], bt_dst, stride, want_logits=True)
        e1.wait(), e2.wait()
        assert np.array_equal(l1, l2), engine
        p.close(), d.close()


CFG = {
    "cluster": {"prefill": 1, "decode": 1},
    "workload": {"n_requests": 24, "mixture": {"LPLD": 0.5, "HPLD": 0.5},
                 "lengths": {"heavy_prompt": {"hi": 900}}},
    "cost_model": {"preset": "nvlink300", "mem_capacity_tokens": 16000},
    "model": {"name": "tiny", "prefill_pages": 1024, "staging_pages": 256,
              "max_decode_batch": 64},
}


def _check_run(res, cfg):
    s = res.summary
    assert s["completed"] == s["n_requests"]
    for row in res.rows:
        assert 0 <= row["wait_us"] <= row["ttft_us"] <= row["jct_us"]
    reqs = tk.generate(cfg.workload_spec, tk.RngStreams(0).stream("workload"))
    dev = s["device"]
    assert dev["kv_bytes_sent"] == sum(-(-r.prompt_len // PT) for r in reqs) * PT * 2 * 2 * 256 * 2
    assert dev["decode_tokens"] == sum(r.true_decode_len for r in reqs)
    return dev


@pytest.mark.parametrize("engine", ["auto", "ce"])
def test_colocated_run_stamps_and_physical_accounting(engine):
    raw = dict(CFG, executor="cuda", devices={"p0": 0, "d0": 0},
               model=dict(CFG["model"], kv_send_engine=engine))
    cfg = tk.config_from_dict(raw)
    res = run_experiment(cfg, seed=0)
    dev = _check_run(res, cfg)
    assert dev["gpus_used"] == 1
    # one GPU billed once: at most pdsim's sum of the two instances' episode spans
    assert 0 < dev["gpu_resource_us"] <= res.summary["resource_usage_us"]
    assert dev["perf_per_dollar_physical"] >= res.summary["perf_per_dollar"]
    # completion stamps are device times: never after the run's end
    assert max(r["jct_us"] for r in res.rows) <= res.summary["makespan_us"]


def test_capacity_from_hbm_sizes_the_decode_pool():
    free, total = native.device_memory(0)
    reserve = free / 1e9 - 8.0  # leave ~8 GB to size from (a tiny model's pages are 32 KB)
    raw = dict(CFG, executor="cuda", devices={"p0": 0, "d0": 0},
               model=dict(CFG["model"], capacity_from_hbm=True, hbm_reserve_gb=reserve))
    cfg = tk.config_from_dict(raw)
    res = run_experiment(cfg, seed=0)
    _check_run(res, cfg)
    cap = res.summary["device"]["mem_capacity_tokens"]
    pb = native.TINY_OPT.kv_bytes_per_token * PT
    assert cap % PT == 0 and cap > 16000
    assert 3e9 < cap // PT * pb < 8e9


@pytest.mark.skipif(_n_dev() < 2, reason="needs two GPUs")
@pytest.mark.parametrize("engine", ["auto", "ce"])
def test_two_gpu_disaggregated_run(engine):
    raw = dict(CFG, executor="cuda", devices={"p0": 0, "d0": 1},
               model=dict(CFG["model"], kv_send_engine=engine))
    cfg = tk.config_from_dict(raw)
    res = run_experiment(cfg, seed=0)
    dev = _check_run(res, cfg)
    assert dev["gpus_used"] == 2 and dev["devices"] == {"p0": 0, "d0": 1}
    assert dev["handoff_gb_s"] > 0
