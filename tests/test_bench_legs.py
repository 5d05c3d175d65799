"""The serving legs bench.py runs (1 GPU co-located, and the P:D splits of the
multi-GPU run: C3 1P:1D, C4 1:3 / 2:2 / 2:6 / 4:4, C5 Llama-2-7B 2:6) -- device-free
checks, so a configuration error cannot first surface on an 8-GPU box:

* every leg's config parses in sim and in CUDA mode (kv_bytes_per_token matches the
  device model, pdsim/costs.py:51), places p{i} on GPU i and d{j} on GPU n_prefill+j
  (one instance per GPU, pdsim/experiment.py:226-231);
* the same leg runs to completion on pdsim's modeled clock (the scheduler half of the
  leg, whose wall time the bench reports as the scheduler's CPU baseline).
"""

import sys
from pathlib import Path

import pytest

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import bench  # noqa: E402
import paper_2401_11181_b200 as tk  # noqa: E402
from paper_2401_11181_b200.cuda_executor import place_instance  # noqa: E402
from paper_2401_11181_b200.native import MODELS  # noqa: E402

LEGS = [(n, *leg) for n, legs in sorted(bench.MULTI_GPU_LEGS.items()) for leg in legs]


@pytest.mark.parametrize("n_gpus,name,n_p,n_d,mix,model", LEGS,
                         ids=[leg[1] for leg in LEGS])
def test_multi_gpu_leg_config_and_schedule(n_gpus, name, n_p, n_d, mix, model):
    model = model or "opt-13b"
    n_req = 96 if name.startswith("c5") else 64  # smaller than the bench's, same shape
    cfg = bench.serving_config(0, n_p, n_d, n_req, mix, model)
    assert n_p + n_d == n_gpus
    dev = tk.config_from_dict(dict(cfg, executor="cuda"))
    assert dev.params.kv_bytes_per_token == MODELS[model].kv_bytes_per_token
    ids = [f"p{i}" for i in range(n_p)] + [f"d{j}" for j in range(n_d)]
    placed = [place_instance(i, n_p, n_gpus, dev.devices) for i in ids]
    assert sorted(placed) == list(range(n_gpus)), placed
    sim = tk.config_from_dict(bench.sim_config(cfg))
    res = tk.run_experiment(sim, seed=0)
    assert len(res.rows) == n_req
    assert res.summary["ttft"]["avg_us"] > 0 and res.summary["jct"]["avg_us"] > 0


@pytest.mark.parametrize("kw", [dict(n_prefill=1, n_decode=1, colocate=True),
                                dict(n_prefill=1, n_decode=0, colocate=True, coupled=True),
                                dict(n_prefill=1, n_decode=1, colocate=True,
                                     mixture=bench.C5_MIX, model="llama-2-7b"),
                                dict(n_prefill=1, n_decode=1, colocate=True, model="opt-125m")])
def test_one_gpu_legs_colocate_everything_on_gpu0(kw):
    cfg = bench.serving_config(0, n_requests=32, **kw)
    assert set(cfg["devices"].values()) == {0}
    dev = tk.config_from_dict(dict(cfg, executor="cuda"))
    assert dev.devices == cfg["devices"]
    res = tk.run_experiment(tk.config_from_dict(bench.sim_config(cfg)), seed=0)
    assert len(res.rows) == 32
