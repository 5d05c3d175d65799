"""Multi-GPU host logic on CPU: instance placement over ordinals, and the
bench's max-over-ranks timing with world_size 2 over gloo (127.0.0.1)."""

import os
import socket
import sys
from pathlib import Path

import pytest
import torch.multiprocessing as mp

from paper_2401_11181_b200.cuda_executor import place_instance

ROOT = Path(__file__).resolve().parents[1]


def test_placement_splits():
    # 2:6 on 8 GPUs: prefill on 0-1, decode on 2-7
    assert [place_instance(f"p{i}", 2, 8) for i in range(2)] == [0, 1]
    assert [place_instance(f"d{i}", 2, 8) for i in range(6)] == [2, 3, 4, 5, 6, 7]
    # 4:4 on 8, 1:3 and 2:2 on 4
    assert [place_instance(f"d{i}", 4, 8) for i in range(4)] == [4, 5, 6, 7]
    assert [place_instance(f"d{i}", 1, 4) for i in range(3)] == [1, 2, 3]
    # 1P:1D co-located on one GPU
    assert place_instance("p0", 1, 1) == place_instance("d0", 1, 1) == 0
    # explicit map wins
    assert place_instance("d0", 1, 8, {"d0": 5}) == 5


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    sys.path.insert(0, str(ROOT))
    import bench
    import torch.distributed as dist
    w, r, local = bench.dist_setup("gloo")
    bench.barrier(w)
    got = bench.dist_max(float(r + 1) * 1.5, w)   # per-rank "device seconds"
    bench.barrier(w)
    # the bench's hand-off: every rank leaves the group after the last collective,
    # then rank 0 alone runs the single-process multi-GPU legs; leaving twice is safe
    bench.leave_group(w)
    bench.leave_group(w)
    q.put((r, w, local, got, dist.is_initialized()))


def test_bench_max_over_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == [(0, 2, 0, 3.0, False), (1, 2, 1, 3.0, False)]


def test_reference_arm_other_ranks_exit_quietly(capsys):
    sys.path.insert(0, str(ROOT))
    import argparse
    import bench
    bench.run_reference(argparse.Namespace(steps=1, warmup=0, gpus=2, seed=0), world=2, rank=1)
    assert capsys.readouterr().out == ""
