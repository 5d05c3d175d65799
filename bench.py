#!/usr/bin/env python
"""Benchmark of the TetriInfer chunked-prefill data path on B200 (BASELINE.json configs[1]).

Workload (C2): OPT-13B-shaped random-init weights (bf16), 64 prompts drawn
uniformly from {2048, 4096, 6144, 8192} tokens (synthetic token ids), the
reference prefill scheduler (SJF, PrefillSchedBatch 16, ChunkSize 512; pdsim
schedule_round/chunkify) on one prefill instance per GPU.

A *step* is one scheduling round: the 16 prompts of the round chunked at 512
and run chunk by chunk through the C ABI (tk_prefill_chunk), each chunk
attending over its requests' accumulated paged KV, first tokens read back for
the finishing prompts.  Rounds cycle through the workload's 4 rounds.

* ``value``  prefill tokens/s from device time (CUDA events on the compute
  stream from the first chunk's start to the last chunk's end of each round),
  whole job over all ranks (max time over ranks).
* ``e2e``    same tokens over host wall time of the same rounds through the
  public API with host buffers: ids/slices/page tables staged from pinned host
  memory each chunk, first tokens read back each chunk.
* ``roofline`` dominant kernel = the tcgen05 GEMM (QKV/O/FC1/FC2): algorithmic
  FLOPs / summed CUDA-event durations of its launches in the timed region,
  against MEASURED_PEAKS.json bf16 sustained (a kernel timed inside a long step).
* ``cpu_baseline`` the fp32 oracle port (oracle/model_ref.py) on the host cores
  on a bounded sample (sampled chunks, each through all 40 OPT-13B layers).

Multi-GPU (torchrun): every rank runs an independent prefill replica of the
same workload (weak scaling; the prefill path has no data-path collective).
``--impl reference`` times the CPU port alone (rank 0; other ranks exit 0).
"""

from __future__ import annotations

import argparse
import json
import os
import random
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PROMPT_CHOICES = (2048, 4096, 6144, 8192)
N_PROMPTS = 64
CHUNK = 512
SCHED_BATCH = 16
PAGE = 16
METRIC = "prefill tok/s & decode tok/s per GPU; mean TTFT and JCT on mixed workload"


def build_workload(seed: int = 0):
    from paper_2401_11181_b200.engine import RngStreams
    from paper_2401_11181_b200.prefill import PrefillPolicy, chunkify, schedule_round
    from paper_2401_11181_b200.workload import Request
    rng = RngStreams(seed).stream("workload")
    reqs = [Request(id=i, arrival_us=0, prompt_len=rng.choice(PROMPT_CHOICES), true_decode_len=1)
            for i in range(N_PROMPTS)]
    rounds, raw = [], list(reqs)
    while raw:
        batch, raw = schedule_round(PrefillPolicy("sjf", SCHED_BATCH), raw)
        rounds.append((batch, chunkify(batch, CHUNK)))
    return reqs, rounds


def round_plan(batch, chunks, vocab: int, seed: int):
    """Per chunk: (ids, slices, block_tables, real_tokens); pages laid out per request."""
    from paper_2401_11181_b200.workload import token_ids_for
    tables, nxt = {}, 0
    for r in batch:
        n = (r.prompt_len + PAGE - 1) // PAGE
        tables[r.id] = list(range(nxt, nxt + n))
        nxt += n
    lens = {r.id: r.prompt_len for r in batch}
    ids_of = {r.id: token_ids_for(r, vocab, seed) for r in batch}
    plan = []
    for c in chunks:
        ids, slices, bt = [], [], []
        for rid, start, n in c.slices:
            ids += ids_of[rid][start:start + n]
            slices.append((start, n, len(bt), len(tables[rid]), int(start + n == lens[rid])))
            bt += tables[rid]
        plan.append((ids, slices, bt, c.real_tokens))
    return plan, nxt


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows: list[list[str]] = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if len(r) >= 8 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for r in self.rows if len(r) >= 8
                          for n, v in zip(names, r[4:8]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                "source": "MEASURED_PEAKS.json"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "source": "fallback (B200_PROFILING.md)"}


def gemm_traffic(prof: dict):
    """DRAM bytes per GEMM launch (dram__bytes_read.sum + dram__bytes_write.sum from the
    committed ncu --set full capture of an in-situ layer, profiles/r02_gemm_traffic.json),
    weighted by this run's launches of each shape, next to the algorithmic bytes."""
    p = ROOT / "profiles" / "r02_gemm_traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    kinds = {"qkv_gemm": "qkv", "o_gemm": "o", "fc1_gemm": "fc1", "fc2_gemm": "fc2"}
    n = sum(prof[k]["launches"] for k in kinds)
    if not n:
        return None
    dram = sum(prof[k]["launches"] * d["dram_bytes_per_launch"][v] for k, v in kinds.items()) / n
    alg = sum(prof[k]["launches"] * d["algorithmic_bytes_per_launch"][v] for k, v in kinds.items()) / n
    return {"dram_bytes_per_launch": int(dram), "algorithmic_bytes_per_launch": int(alg),
            "ratio": round(dram / alg, 3), "source": "profiles/r02_gemm_traffic.json (M=512 shapes, in situ)"}


# ---------------------------------------------------------------- CPU port (oracle)

def cpu_port_sample(plan_chunks, max_seconds: float = 25.0, threads: int | None = None,
                    layers: int = 40):
    """fp32 oracle timing of sampled chunks through `layers` OPT-13B layers each.

    layers=40 runs the whole 40-layer stack per chunk (one layer's random weights
    reused by every layer: the same FLOPs and weight traffic per layer, 2.5 GB of
    fp32 weights instead of 100 GB of host memory); the LM head (0.06% of the GPU
    step) is left out.  layers=1 is a cheap warm-up.
    plan_chunks: list of (slices, real_tokens).  Returns (tok_s, cores, sample_desc).
    """
    import torch
    from oracle.model_ref import ARCH_OPT, OracleModel, PagedCache, Shape
    cores = threads or os.cpu_count() or 1
    torch.set_num_threads(cores)
    full_layers = 40
    shape = Shape(ARCH_OPT, n_layers=1, hidden=5120, n_heads=40, ffn=20480, vocab=8,
                  max_positions=10240)
    g = torch.Generator().manual_seed(0)
    h, f = 5120, 20480
    w = {"embed_tokens.weight": torch.zeros(8, h),
         "embed_positions.weight": torch.zeros(10242, h),
         "layers.0.self_attn_layer_norm.weight": torch.ones(h),
         "layers.0.self_attn_layer_norm.bias": torch.zeros(h),
         "layers.0.self_attn.qkv_proj.weight": torch.randn(3 * h, h, generator=g) * 0.02,
         "layers.0.self_attn.qkv_proj.bias": torch.zeros(3 * h),
         "layers.0.self_attn.out_proj.weight": torch.randn(h, h, generator=g) * 0.02,
         "layers.0.self_attn.out_proj.bias": torch.zeros(h),
         "layers.0.final_layer_norm.weight": torch.ones(h),
         "layers.0.final_layer_norm.bias": torch.zeros(h),
         "layers.0.fc1.weight": torch.randn(f, h, generator=g) * 0.02,
         "layers.0.fc1.bias": torch.zeros(f),
         "layers.0.fc2.weight": torch.randn(h, f, generator=g) * 0.02,
         "layers.0.fc2.bias": torch.zeros(h)}
    ora = OracleModel(shape, w)
    spent, tokens, done = 0.0, 0, 0
    for slices, real in plan_chunks:
        top = max(s + n for s, n, *_ in slices)
        cache = PagedCache(shape, (top + PAGE - 1) // PAGE * len(slices) + 1, PAGE)
        rows, row, tbl_off = [], 0, 0
        for s, n, *_ in slices:
            np_ = (s + n + PAGE - 1) // PAGE
            table = list(range(tbl_off, tbl_off + np_))
            tbl_off += np_
            rows.append((table, torch.arange(s, s + n), slice(row, row + n)))
            row += n
        x = torch.randn(real, h, generator=g)
        t = time.perf_counter()
        with torch.no_grad():
            for _ in range(layers):
                x = ora.layer(0, x, rows, cache)
        spent += time.perf_counter() - t
        tokens += real
        done += 1
        if spent > max_seconds:
            break
    tok_s = tokens / (spent * full_layers / layers)
    if layers == full_layers:
        desc = (f"fp32 torch oracle, {done} sampled C2 chunks ({tokens} tokens), each through "
                f"all {full_layers} OPT-13B layers (one layer's weights reused) incl. paged causal "
                f"attention over the real prefix; LM head omitted")
    else:
        desc = (f"fp32 torch oracle, {done} sampled C2 chunks ({tokens} tokens), {layers} "
                f"OPT-13B layer(s) each, x{full_layers / layers:g} extrapolated")
    return tok_s, cores, desc


# ---------------------------------------------------------------- arms

def dist_setup(backend: str = "nccl"):
    """One process per GPU (torchrun env); nccl on the box, gloo in CPU tests."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        import torch
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return world, rank, local


def dist_max(value: float, world: int) -> float:
    """Max over ranks (the timing rule: whole-job time = slowest rank)."""
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def leave_group(world: int):
    """Tear the process group down once the last collective is done (torchrun ranks
    exit while rank 0 alone runs the multi-GPU legs)."""
    if world > 1:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()


def run_reference(args, world, rank):
    if rank != 0:
        return
    reqs, rounds = build_workload(args.seed)
    all_chunks = [(c.slices, c) for _, chs in rounds for c in chs]
    n = len(all_chunks)
    total = args.warmup + args.steps
    idx = [int(i * n / total) for i in range(total)]
    samples = []
    for i in idx:
        batch = [r for r, chs in rounds if all_chunks[i][1] in chs][0]
        lens = {r.id: r.prompt_len for r in batch}
        sl = [(s, ln, 0, 0, int(s + ln == lens[rid])) for rid, s, ln in all_chunks[i][1].slices]
        samples.append((sl, all_chunks[i][1].real_tokens))
    # warmup steps untimed (one layer each: threads, allocator, page cache)
    for s in samples[:args.warmup]:
        cpu_port_sample([s], max_seconds=1e9, layers=1)
    t0 = time.perf_counter()
    tok_s, cores, desc = cpu_port_sample(samples[args.warmup:], max_seconds=1e9)
    wall = time.perf_counter() - t0
    line = {
        "impl": "reference", "metric": METRIC, "value": round(tok_s, 3), "unit": "tok/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(wall / max(1, args.steps) * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": "C2: OPT-13B-shaped chunked prefill, ChunkSize 512, 64 prompts "
                               "uniform over 2k/4k/6k/8k, SJF PrefillSchedBatch 16",
                   "step": "one sampled chunk through all 40 layers (CPU port)"},
        "cpu_baseline": {"value": round(tok_s, 3), "unit": "tok/s", "cores": cores,
                         "kind": "port", "sample": desc},
        "e2e": {"value": round(tok_s, 3), "unit": "tok/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def run_ours(args, world, rank, local):
    from paper_2401_11181_b200 import native
    native.load()
    shape = native.MODELS[args.model]
    reqs, rounds = build_workload(args.seed)
    plans, max_pages = [], 0
    for batch, chunks in rounds:
        plan, pages = round_plan(batch, chunks, shape.vocab, args.seed)
        plans.append(plan)
        max_pages = max(max_pages, pages)
    # torchrun: one replica per rank on its LOCAL_RANK device.  A plain
    # ``python bench.py --gpus N``: one process drives N replicas (devices 0..N-1),
    # issuing every round's chunks to all of them before waiting on any.
    if world == 1 and args.gpus > 1:
        n_dev = native.device_count()
        if n_dev < args.gpus:
            raise SystemExit(f"bench.py --gpus {args.gpus}: only {n_dev} CUDA device(s) visible")
        devs = list(range(args.gpus))
    else:
        devs = [local]
    insts = [native.Instance(shape, device=d, seed=args.seed, kv_pages=max_pages,
                             page_tokens=PAGE, max_chunk=CHUNK) for d in devs]
    inst = insts[0]

    def run_round(plan, which=None):
        which = insts if which is None else which
        evs = [[] for _ in which]
        toks = h2d = d2h = 0
        verbose = os.environ.get("TK_BENCH_VERBOSE")
        for ci, (ids, slices, bt, real) in enumerate(plan):
            for k, ins in enumerate(which):
                ev, out = ins.prefill_chunk(ids, slices, bt)
                if verbose:
                    ev.wait()
                    print(f"dev {ins.device} chunk {ci} slices={[(s[0], s[1]) for s in slices]} "
                          f"{ev.elapsed_ns / 1e6:.2f} ms", file=sys.stderr, flush=True)
                a, b = ins.staged_bytes()
                h2d, d2h = h2d + a, d2h + b
                evs[k].append((ev, out))
                toks += real
        for per in evs:
            for ev, _ in per:
                ev.wait()  # publishes each chunk's first tokens to host memory
        # device time of the slowest replica (max over devices)
        dev_ns = max(native.event_elapsed_ns(per[0][0], per[-1][0]) for per in evs)
        return toks, dev_ns, h2d, d2h

    for i in range(args.warmup):
        run_round(plans[i % len(plans)])
    for ins in insts:
        ins.sync()
    clocks = ClockSampler(local if len(devs) == 1 else ",".join(map(str, devs)))
    barrier(world)
    for ins in insts:
        ins.sync()
    clocks.start()
    launches0 = native.launch_count()
    t0 = time.perf_counter()
    tokens = dev_ns = h2d = d2h = 0
    for i in range(args.steps):
        t, ns, a, b = run_round(plans[(args.warmup + i) % len(plans)])
        tokens, dev_ns, h2d, d2h = tokens + t, dev_ns + ns, h2d + a, d2h + b
    for ins in insts:
        ins.sync()
    wall = time.perf_counter() - t0
    launches = native.launch_count() - launches0
    barrier(world)
    clk = clocks.stop()
    # Per-kernel breakdown (roofline, shares): the same rounds again on the first
    # replica, every launch bracketed by CUDA events on the compute stream.  Kept
    # out of the timed region above so the event records do not perturb `value`.
    inst.profile(True)
    prof_ns = 0
    for i in range(args.steps):
        prof_ns += run_round(plans[(args.warmup + i) % len(plans)], [inst])[1]
    inst.sync()
    prof = inst.profile_read()
    inst.profile(False)

    dev_s = dist_max(dev_ns / 1e9, world)
    wall_s = dist_max(wall, world)
    total_tokens = tokens * world  # tokens already counts every replica of this process
    n_gpus = world * len(devs)
    peaks = measured_peaks()
    gemm_kinds = ("qkv_gemm", "o_gemm", "fc1_gemm", "fc2_gemm")
    g_ms = sum(prof[k]["ms"] for k in gemm_kinds)
    g_fl = sum(prof[k]["flops"] for k in gemm_kinds)
    g_n = sum(prof[k]["launches"] for k in gemm_kinds)
    achieved = g_fl / (g_ms / 1e3) / 1e12 if g_ms else 0.0
    traffic = gemm_traffic(prof)
    peak = peaks["bf16_tflops_sustained"]
    attn = prof["attention"]
    for ins in insts[1:]:
        ins.close()
    if rank != 0:
        inst.close()
        barrier(world)  # rank 0 runs the cross-GPU legs once every replica is closed
        leave_group(world)
        return
    line = {
        "metric": METRIC,
        "value": round(total_tokens / dev_s, 2),
        "unit": "tok/s",
        "n_gpus": n_gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(dev_s / args.steps * 1e3, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (random-init OPT-13B-shaped weights, synthetic token ids)",
        "config": {
            "workload": "C2: OPT-13B-shaped chunked prefill only, ChunkSize 512, 64 prompts "
                        "uniform over 2k/4k/6k/8k tokens, SJF PrefillSchedBatch 16, 1 prefill "
                        "instance per GPU",
            "model": shape.name, "chunk_size": CHUNK, "page_tokens": PAGE,
            "step": "one scheduling round (16 prompts, all chunks, first tokens read back)",
            "tokens_per_step": tokens // max(1, args.steps),
            "parallelism": (f"prefill replicas x{n_gpus} (weak; "
                            + ("torchrun, one rank per GPU" if world > 1 else
                               "one process driving every GPU") + ")"),
            "l2": "inputs larger than L2 (25.8 GB of weights streamed per chunk)",
        },
        "e2e": {"value": round(total_tokens / wall_s, 2), "unit": "tok/s",
                "h2d_bytes_per_step": h2d // max(1, args.steps),
                "d2h_bytes_per_step": d2h // max(1, args.steps)},
        "gpu_launches": launches,
        "roofline": {
            "kernel": "gemm_pair_kernel (tcgen05 cta_group::2; QKV/O/FC1/FC2)",
            "bound": "tensor", "achieved": round(achieved, 2), "peak": peak,
            "unit": "TFLOP/s", "frac": round(achieved / peak, 4),
            "peak_source": peaks["source"] + " bf16_tflops_sustained",
            "launches": g_n, "avg_launch_us": round(g_ms * 1e3 / max(1, g_n), 2),
            "traffic": traffic["dram_bytes_per_launch"] if traffic else None,
            "traffic_detail": traffic,
        },
        "kernels": {k: {"launches": v["launches"], "ms": round(v["ms"], 3),
                        "tflops": round(v["flops"] / (v["ms"] / 1e3) / 1e12, 2) if v["ms"] and v["flops"] else None,
                        "gbs": round(v["bytes"] / (v["ms"] / 1e3) / 1e9, 1) if v["ms"] else None}
                    for k, v in prof.items()},
        "clocks": clk,
    }
    line["share_of_step"] = {k: round(v["ms"] / (prof_ns / 1e6), 4) for k, v in prof.items()}
    inst.close()
    if n_gpus > 1:
        barrier(world)  # every other rank has closed its replica
        leave_group(world)  # no collective is pending while the single-process legs run
        line["multi_gpu"] = guarded(lambda: multi_gpu_run(args, n_gpus, peaks))
    if n_gpus == 1 and not args.no_decode:
        line["decode"] = decode_run(args, shape, local, peaks)
        if args.model == "opt-13b":
            # BASELINE.json configs[4] at one GPU: Llama-2-7B-shaped large decode batches
            line["decode"].update(decode_run(args, native.MODELS["llama-2-7b"], local, peaks,
                                             configs=((256, 1024),), tag="llama-2-7b_"))
    if n_gpus == 1 and not args.no_decode:
        line["kv_handoff"] = guarded(lambda: handoff_run(args, shape, local, local, peaks))
        line["kv_handoff"]["overlap"] = guarded(lambda: overlap_run(args, shape, local, local))
        line["predictor"] = predictor_run(args, local, peaks)
        line["predictor"]["corun"] = guarded(lambda: predictor_corun(args, shape, local))
    if n_gpus == 1 and not args.no_serving:
        line["serving"] = serving_run(args)
    if n_gpus == 1 and not args.no_cpu_baseline:
        all_chunks = [(p[1], p[3]) for plan in plans for p in plan]
        pick = [all_chunks[int(i * len(all_chunks) / 6)] for i in range(6)]
        tok_s, cores, desc = cpu_port_sample(pick, max_seconds=args.cpu_seconds)
        line["cpu_baseline"] = {"value": round(tok_s, 3), "unit": "tok/s", "cores": cores,
                                "kind": "port", "sample": desc}
    print(json.dumps(line))


def decode_run(args, shape, device: int, peaks: dict, configs=((32, 2048), (128, 512)),
               tag: str = "") -> dict:
    """Decode steps (tk_decode_step) at a fixed batch/context: tok/s and the
    paged decode-attention kernel against the HBM roofline (CUDA events)."""
    from paper_2401_11181_b200 import native
    out = {}
    for batch, ctx in configs:  # OPT-13B pools of ~55 GB each
        steps = 16
        pages_per = (ctx + steps + 3 + 16) // 16
        inst = native.Instance(shape, device=device, seed=args.seed,
                               kv_pages=batch * pages_per, max_chunk=max(64, batch))
        bt = list(range(batch * pages_per))
        last = [7] * batch
        for i in range(3):
            ev, _ = inst.decode_step(last, [ctx + i] * batch, bt, pages_per)
            ev.wait()
        # timed without per-kernel events, then a profiled pass for the breakdown
        evs, t_call = [], []
        for i in range(steps):
            t_host = time.perf_counter()
            evs.append(inst.decode_step(last, [ctx + 3 + i] * batch, bt, pages_per)[0])
            t_call.append(time.perf_counter() - t_host)
        # host cost of one call: the first calls only (later ones wait for a staging slot)
        host_us = sorted(t_call[:6])[3] * 1e6
        ns = native.event_elapsed_ns(evs[0], evs[-1])
        inst.profile(True)
        pevs = [inst.decode_step(last, [ctx + 3 + i] * batch, bt, pages_per)[0]
                for i in range(steps)]
        pns = native.event_elapsed_ns(pevs[0], pevs[-1])
        prof = inst.profile_read()
        inst.close()
        att = prof["attention"]
        gbs = att["bytes"] / (att["ms"] / 1e3) / 1e9
        gemm_ms = sum(prof[k]["ms"] for k in ("qkv_gemm", "o_gemm", "fc1_gemm", "fc2_gemm"))
        gemm_bytes = sum(prof[k]["bytes"] for k in ("qkv_gemm", "o_gemm", "fc1_gemm", "fc2_gemm"))
        out[f"{tag}b{batch}_ctx{ctx}"] = {
            "decode_tok_s": round(batch * steps / (ns / 1e9), 1),
            "step_ms": round(ns / 1e6 / steps, 3),
            "attention_roofline": {"bound": "hbm", "achieved": round(gbs, 1),
                                   "peak": peaks["hbm_gbs"], "unit": "GB/s",
                                   "frac": round(gbs / peaks["hbm_gbs"], 4),
                                   "launches": att["launches"]},
            "gemm_weight_stream_gbs": round(gemm_bytes / (gemm_ms / 1e3) / 1e9, 1),
            "host_enqueue_us_per_step": round(host_us, 1),
            "cuda_graph": not os.environ.get("TK_NO_DECODE_GRAPH"),
            "share_of_step": {k: round(v["ms"] / (pns / 1e6), 4) for k, v in prof.items()},
        }
    return out


NVLINK_GBS = 900.0  # NVLink 5 per direction per GPU (spec)


def p2p_copy_gbs(src: int, dst: int, nbytes: int = 1 << 30) -> float:
    """Measured device->peer copy bandwidth (torch copy over NVLink, best of 5,
    CUDA events on the source): the achievable figure beside the 900 GB/s spec."""
    import torch
    a = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{src}")
    b = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{dst}")
    best = 0.0
    with torch.cuda.device(src):
        for _ in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            b.copy_(a, non_blocking=True)
            e1.record()
            e1.synchronize()
            best = max(best, nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
    del a, b
    torch.cuda.empty_cache()
    return best


def handoff_run(args, shape, src_dev: int, dst_dev: int, peaks: dict,
                prompts=(512, 900, 8192), engines=("sm", "ce"), p2p_gbs: float | None = None) -> dict:
    """P->D KV handoff (tk_kv_send_ex, pdsim/prefill.py:420-424): one request's
    prompt pages, scattered on both sides, from an instance on ``src_dev`` to one
    on ``dst_dev``.  bytes = prompt pages x page bytes (costs.py:137 rounds to
    whole pages here).  Co-located (same device): HBM-bound, traffic 2 x bytes.
    Across devices: NVLink-bound, against 900 GB/s per direction (spec) and the
    measured peer copy bandwidth.  Engines: "sm" = the page-copy kernel (peer
    stores), "ce" = copy engines."""
    import random

    from paper_2401_11181_b200 import costs, native
    n_max = (max(prompts) + PAGE - 1) // PAGE
    src = native.Instance(shape, device=src_dev, seed=args.seed, kv_pages=n_max + 64, max_chunk=64)
    dst = native.Instance(shape, device=dst_dev, seed=args.seed, kv_pages=n_max + 64, max_chunk=64)
    rng = random.Random(args.seed)
    local = src_dev == dst_dev
    out = {"src_device": src_dev, "dst_device": dst_dev,
           "link": "device-local copy (co-located P and D), HBM-bound" if local else
                   "NVLink 5 / NVSwitch peer path"}
    if not local and p2p_gbs:
        out["p2p_copy_gbs_measured"] = round(p2p_gbs, 1)
    for engine in engines:
        res = {}
        for n_tok in prompts:
            n = (n_tok + PAGE - 1) // PAGE
            sp, dp = rng.sample(range(n_max + 64), n), rng.sample(range(n_max + 64), n)
            for _ in range(3):
                src.kv_send(sp, dst, dp, engine).wait()
            evs = [src.kv_send(sp, dst, dp, engine) for _ in range(8)]
            for e in evs:
                e.wait()
            ns = sorted(e.elapsed_ns for e in evs)[len(evs) // 2]
            nbytes = n * src.page_bytes
            gbs = nbytes / (ns / 1e9) / 1e9
            r = {"pages": n, "bytes": nbytes, "device_us": round(ns / 1e3, 1),
                 "handoff_gb_s": round(gbs, 1),
                 "reference_modeled_us_nvlink300": costs.transfer_latency(
                     costs.load_calibration({"preset": "nvlink300"}), n_tok)}
            if local:
                hbm = 2 * gbs
                r["roofline"] = {"bound": "hbm", "achieved": round(hbm, 1),
                                 "peak": peaks["hbm_gbs"], "unit": "GB/s",
                                 "frac": round(hbm / peaks["hbm_gbs"], 4)}
            else:
                r["roofline"] = {"bound": "nvlink", "achieved": round(gbs, 1),
                                 "peak": NVLINK_GBS, "unit": "GB/s",
                                 "frac": round(gbs / NVLINK_GBS, 4)}
                if p2p_gbs:
                    r["roofline"]["frac_of_measured_p2p"] = round(gbs / p2p_gbs, 4)
            res[f"prompt{n_tok}"] = r
        out[engine] = res
    src.close(), dst.close()
    return out


def overlap_run(args, shape, src_dev: int, dst_dev: int, prefix: int = 4096,
                send_tokens: int = 8192, engines=("sm", "ce"), reps: int = 5) -> dict:
    """Handoff/compute overlap (pdsim/prefill.py:420-424: sends run free beside
    the next chunk).  One 512-token chunk at a ``prefix``-token prefix on the
    prefill instance, alone and with a ``send_tokens``-token request's handoff
    issued right before it (the send waits for the previous chunk, then runs
    on the copy stream while this chunk computes).  Reported per engine: chunk
    time alone / under the send, send time alone / under the chunk, and the
    overlap efficiency (alone chunk + alone send) / concurrent makespan."""
    import random
    import statistics as st

    from paper_2401_11181_b200 import native
    from paper_2401_11181_b200.workload import Request, token_ids_for
    n_req = (prefix + CHUNK + PAGE - 1) // PAGE
    n_send = (send_tokens + PAGE - 1) // PAGE
    src = native.Instance(shape, device=src_dev, seed=args.seed, kv_pages=n_req + n_send,
                          page_tokens=PAGE, max_chunk=CHUNK)
    dst = native.Instance(shape, device=dst_dev, seed=args.seed, kv_pages=n_send,
                          page_tokens=PAGE, max_chunk=64)
    req = Request(id=0, arrival_us=0, prompt_len=prefix + CHUNK, true_decode_len=1)
    ids = token_ids_for(req, shape.vocab, args.seed)
    bt = list(range(n_req))
    for c0 in range(0, prefix, CHUNK):  # fill the prefix KV once
        src.prefill_chunk(ids[c0:c0 + CHUNK], [(c0, CHUNK, 0, n_req, 0)], bt)[0].wait()
    chunk = (ids[prefix:], [(prefix, CHUNK, 0, n_req, 1)], bt)
    rng = random.Random(args.seed)
    sp = [n_req + i for i in rng.sample(range(n_send), n_send)]
    dp = rng.sample(range(n_send), n_send)
    for _ in range(2):
        src.prefill_chunk(*chunk)[0].wait()
    alone = []
    for _ in range(reps):
        alone.append(src.prefill_chunk(*chunk)[0].wait())
    out = {"chunk": f"512 tokens at prefix {prefix} ({shape.name})",
           "send": f"{send_tokens}-token request ({n_send} pages, {n_send * src.page_bytes} B)",
           "devices": [src_dev, dst_dev], "chunk_alone_us": round(st.median(alone) / 1e3, 1)}
    for engine in engines:
        s_alone, c_under, s_under, span = [], [], [], []
        for _ in range(reps):
            s_alone.append(src.kv_send(sp, dst, dp, engine).wait())
        for _ in range(reps):
            src.prefill_chunk(*chunk)[0].wait()
            pre = src.prefill_chunk(*chunk)[0]          # chunk k
            sev = src.kv_send(sp, dst, dp, engine)      # its handoff, after chunk k
            cev = src.prefill_chunk(*chunk)[0]          # chunk k+1, concurrent with the send
            c_under.append(cev.wait())
            s_under.append(sev.wait())
            pre.wait()
            span.append(max(native.event_elapsed_ns(sev, cev), native.event_elapsed_ns(sev, sev)))
        ca, sa = st.median(alone), st.median(s_alone)
        mk = st.median(span)
        out[engine] = {"send_alone_us": round(sa / 1e3, 1),
                       "chunk_under_send_us": round(st.median(c_under) / 1e3, 1),
                       "send_under_chunk_us": round(st.median(s_under) / 1e3, 1),
                       "makespan_us": round(mk / 1e3, 1),
                       "chunk_slowdown": round(st.median(c_under) / ca, 4),
                       "overlap_efficiency": round((ca + sa) / mk, 4)}
    src.close(), dst.close()
    return out


def guarded(fn):
    """Run an auxiliary leg; a failure is recorded in the line instead of losing it."""
    try:
        return fn()
    except Exception as e:  # noqa: BLE001 -- reported, never hidden
        import traceback
        traceback.print_exc()
        return {"error": f"{type(e).__name__}: {e}"[:400]}


def predictor_run(args, device: int, peaks: dict, n: int = 16, length: int = 512) -> dict:
    """Length predictor (tk_predict, pdsim/prefill.py:99): OPT-125M-class classifier
    over one round's prompts (16 x 512 tokens), device time."""
    import random

    from paper_2401_11181_b200 import native
    m = native.PREDICTOR_125M
    inst = native.Instance(m, device=device, seed=args.seed + 1, kv_pages=n * (length // PAGE) + 8,
                           max_chunk=n * length)
    rng = random.Random(args.seed)
    ids = [rng.randrange(2, m.vocab) for _ in range(n * length)]
    for _ in range(3):
        inst.predict(ids, [length] * n, length)[0].wait()
    evs = [inst.predict(ids, [length] * n, length)[0] for _ in range(10)]
    ns = native.event_elapsed_ns(evs[0], evs[-1]) / len(evs)  # start of first .. end of last
    inst.close()
    params = 12 * (4 * 768 * 768 + 2 * 768 * 3072)
    flops = 2 * params * n * length + 4 * 768 * 12 * n * length * (length + 1) / 2
    tf = flops / (ns / 1e9) / 1e12
    return {"batch": n, "len": length, "device_us": round(ns / 1e3, 1),
            "tflops": round(tf, 1), "frac_of_peak": round(tf / peaks["bf16_tflops_sustained"], 4),
            "note": "tiny model: launch/latency bound, not tensor bound"}


def predictor_corun(args, shape, device: int, prompt: int = 2048, reps: int = 5) -> dict:
    """Parallel-mode predictor cost (pdsim/prefill.py:338-346; modeled as the 1.10
    chunk tax, pdsim/costs.py:49; the paper measured +10% prefill latency,
    PAPER.md:773-774): one round's prefill -- a ``prompt``-token request's 512-token
    chunks on the OPT-13B prefill instance -- alone, and with the round's
    predictor pass (16 x 512 tokens, OPT-125M-class) issued on its own instance's
    stream just before the first chunk, as CudaExecutor.predict_round does."""
    import random
    import statistics as st

    from paper_2401_11181_b200 import native
    from paper_2401_11181_b200.workload import Request, token_ids_for
    m = native.PREDICTOR_125M
    pred = native.Instance(m, device=device, seed=args.seed + 1, kv_pages=16 * 32 + 8,
                           max_chunk=16 * 512)
    n_pages = (prompt + PAGE - 1) // PAGE
    big = native.Instance(shape, device=device, seed=args.seed, kv_pages=n_pages,
                          page_tokens=PAGE, max_chunk=CHUNK)
    ids = token_ids_for(Request(id=0, arrival_us=0, prompt_len=prompt, true_decode_len=1),
                        shape.vocab, args.seed)
    bt = list(range(n_pages))
    chunks = [(ids[c:c + CHUNK], [(c, CHUNK, 0, n_pages, int(c + CHUNK >= prompt))], bt)
              for c in range(0, prompt, CHUNK)]
    rng = random.Random(args.seed)
    pids = [rng.randrange(2, m.vocab) for _ in range(16 * 512)]

    def one(with_pred: bool, with_chunks: bool = True):
        pev = pred.predict(pids, [512] * 16, 512)[0] if with_pred else None
        evs = [big.prefill_chunk(*c)[0] for c in chunks] if with_chunks else []
        if not evs:
            return pev.wait(), 0, 0
        chunk_ns = native.event_elapsed_ns(evs[0], evs[-1])
        if pev is None:
            return 0, chunk_ns, chunk_ns
        span = max(native.event_elapsed_ns(pev, evs[-1]), native.event_elapsed_ns(pev, pev))
        return native.event_elapsed_ns(pev, pev), chunk_ns, span

    for _ in range(2):
        one(True)
    alone = st.median(one(False)[1] for _ in range(reps))
    p_alone = st.median(one(True, False)[0] for _ in range(reps))
    runs = [one(True) for _ in range(reps)]
    p_under = st.median(r[0] for r in runs)
    c_under = st.median(r[1] for r in runs)
    span = st.median(r[2] for r in runs)
    pred.close(), big.close()
    return {"round": f"{prompt}-token prompt, {len(chunks)} chunks of 512 ({shape.name})",
            "predictor": "16 x 512 tokens, OPT-125M-class classifier, own stream",
            "round_alone_us": round(alone / 1e3, 1),
            "predictor_alone_us": round(p_alone / 1e3, 1),
            "round_with_predictor_us": round(c_under / 1e3, 1),
            "predictor_under_round_us": round(p_under / 1e3, 1),
            "makespan_us": round(span / 1e3, 1),
            "measured_tax": round(span / alone, 4),
            "reference_modeled_tax": 1.10,
            "paper": "+10% prefill latency in parallel mode (PAPER.md:773-774)"}


def c1_cpu_sample(args, seconds: float = 12.0) -> dict:
    """BASELINE.json configs[0] / BASELINE.md section 4 item 2: the fp32 oracle runs
    the tiny decoder (OPT-125M shape, all 12 layers, LM head) on the host cores over
    a bounded sample of the same Mixed-128 workload: the first SJF round's chunks
    (ChunkSize 512, pdsim/prefill.py:140-165) for ~``seconds``/2, then decode steps
    of the prefilled requests as one batch for the rest."""
    import torch

    import paper_2401_11181_b200 as tk
    from oracle.model_ref import ARCH_OPT, OracleModel, PagedCache, Shape, random_weights
    from paper_2401_11181_b200 import native, workload
    from paper_2401_11181_b200.engine import RngStreams
    from paper_2401_11181_b200.prefill import chunkify
    cores = os.cpu_count() or 1
    torch.set_num_threads(cores)
    m = native.OPT_125M
    shape = Shape(ARCH_OPT, m.n_layers, m.hidden, m.n_heads, m.ffn, m.vocab, m.max_positions)
    ora = OracleModel(shape, random_weights(shape, args.seed))
    cfg = tk.config_from_dict({"workload": {"n_requests": 128}})
    reqs = workload.generate(cfg.workload_spec, RngStreams(args.seed).stream("workload"))
    batch = sorted(reqs[:16], key=lambda r: (r.prompt_len, r.arrival_us, r.id))
    tables, nxt = {}, 0
    for r in batch:
        k = (r.prompt_len + 64 + PAGE - 1) // PAGE
        tables[r.id] = list(range(nxt, nxt + k))
        nxt += k
    cache = PagedCache(shape, nxt, PAGE)
    prompts = {r.id: workload.token_ids_for(r, m.vocab, args.seed) for r in batch}
    lens = {r.id: r.prompt_len for r in batch}
    p_tok, p_s, done = 0, 0.0, set()
    for c in chunkify(batch, 512):
        ids, slices, bt = [], [], []
        for rid, st, n in c.slices:
            ids += prompts[rid][st:st + n]
            slices.append((st, n, len(bt), len(tables[rid]), int(st + n == lens[rid])))
            bt += tables[rid]
            if st + n == lens[rid]:
                done.add(rid)
        t = time.perf_counter()
        ora.prefill_chunk(cache, ids, slices, bt)
        p_s += time.perf_counter() - t
        p_tok += len(ids)
        if p_s > seconds / 2:
            break
    rids = [r.id for r in batch if r.id in done]
    d_tok, d_s, step = 0, 0.0, 0
    while rids and d_s < seconds / 2 and step < 64:
        t = time.perf_counter()
        ora.decode_step(cache, [7] * len(rids), [lens[r] + step for r in rids],
                        [tables[r] for r in rids])
        d_s += time.perf_counter() - t
        d_tok += len(rids)
        step += 1
    return {"prefill_tok_s": round(p_tok / p_s, 1) if p_s else None,
            "decode_tok_s": round(d_tok / d_s, 1) if d_s else None, "cores": cores,
            "kind": "port",
            "sample": f"fp32 oracle, OPT-125M shape (12 layers + LM head): {p_tok} prompt tokens "
                      f"of the first SJF round's chunks, then {step} decode steps of a batch of "
                      f"{len(rids)} prefilled requests (Mixed-128 seed {args.seed})"}


def c1_run(args) -> dict:
    """BASELINE.json configs[0] on the device: the tiny decoder (OPT-125M shape),
    ChunkSize 512, 1 prefill + 1 decode instance (co-located on one GPU), the
    four-class Mixed-128 workload; beside it the fp32 oracle on the host cores."""
    return {"device": guarded(lambda: serving_leg(args, 1, 1, 128, model="opt-125m",
                                                  colocate=True)),
            "cpu_oracle": guarded(lambda: c1_cpu_sample(args))}


C3_MIX = {"LPLD": 0.5, "HPLD": 0.5}     # summarization-like (BASELINE configs[2])
C5_MIX = {"LPHD": 0.5, "HPHD": 0.5}     # content creation (BASELINE configs[4])


def serving_config(seed: int, n_prefill: int, n_decode: int, n_requests: int,
                   mixture: dict | None = None, model: str = "opt-13b", colocate: bool = False,
                   coupled: bool = False, capacity_tokens: int | None = None) -> dict:
    """The experiment config of one serving leg (pdsim keys + devices / model):
    p{i} on GPU i, d{j} on GPU n_prefill + j, or all on GPU 0 when ``colocate``.
    Device-free, so the CPU tests check every leg's config and scheduling."""
    from paper_2401_11181_b200 import native
    shape = native.MODELS[model]
    wl = {"n_requests": n_requests}
    if mixture:
        wl["mixture"] = dict(mixture)
    cm = {"preset": "nvlink300", "kv_bytes_per_token": shape.kv_bytes_per_token}
    if capacity_tokens:
        cm["mem_capacity_tokens"] = capacity_tokens
    mcfg = {"name": model, "prefill_pages": 2048, "staging_pages": 512,
            "max_decode_batch": 256, "seed": seed}
    if capacity_tokens is None:
        mcfg["capacity_from_hbm"] = True
    devices = {}
    if not coupled:
        devices.update({f"p{i}": i for i in range(n_prefill)})
        devices.update({f"d{j}": n_prefill + j for j in range(n_decode)})
        cluster = {"prefill": n_prefill, "decode": n_decode}
    else:
        cluster = {"coupled": n_prefill}
        devices.update({f"c{i}": i for i in range(n_prefill)})
    if colocate:
        devices = {k: 0 for k in devices}
    cfg = {"cluster": cluster, "workload": wl, "cost_model": cm, "model": mcfg,
           "devices": devices}
    if coupled:
        cfg["system"] = "coupled"
    return cfg


def sim_config(cfg: dict) -> dict:
    """The same leg on pdsim's modeled clock (no device keys the sim rejects)."""
    return dict(cfg, model={k: v for k, v in cfg["model"].items() if k != "capacity_from_hbm"})


def serving_leg(args, n_prefill: int, n_decode: int, n_requests: int, mixture: dict | None = None,
                model: str | None = None, colocate: bool = False, coupled: bool = False,
                streaming: bool = False, capacity_tokens: int | None = None) -> dict:
    """One serving run through the reference scheduler + CUDA executor (real
    clock, completion stamps = CUDA-event times) on GPUs 0.. (p{i} then d{j}),
    or every instance on GPU 0 when ``colocate``, beside the same workload on the modeled clock (pdsim's V100 cost
    model through this package's bit-identical port; its single-thread wall time
    is the CPU baseline of the scheduler)."""
    import paper_2401_11181_b200 as tk
    from paper_2401_11181_b200 import native
    from paper_2401_11181_b200.experiment import run_experiment
    model = model or args.model
    n_gpus = 1 if colocate else n_prefill + n_decode
    if n_gpus > native.device_count():
        raise RuntimeError(f"{n_prefill}P:{n_decode}D needs {n_gpus} GPUs, "
                           f"{native.device_count()} visible")
    cfg = serving_config(args.seed, n_prefill, n_decode, n_requests, mixture, model, colocate,
                         coupled, capacity_tokens)
    t0 = time.perf_counter()
    sim = run_experiment(tk.config_from_dict(sim_config(cfg)), seed=args.seed).summary
    sim_wall = time.perf_counter() - t0
    dev_cfg = dict(cfg, executor="cuda")
    if streaming:
        dev_cfg["kv_streaming"] = "chunk"
    res = run_experiment(tk.config_from_dict(dev_cfg), seed=args.seed)
    s, d = res.summary, res.summary["device"]
    gen_tokens = sum(r["decode_len"] for r in res.rows)
    prompt_tokens = sum(r["prompt_len"] for r in res.rows)
    phys = d.get("gpus_used", n_gpus)
    out = {
        "system": "coupled" if coupled else "tetriinfer",
        "split": f"{n_prefill}C" if coupled else f"{n_prefill}P:{n_decode}D",
        "gpus": phys, "model": model, "n_requests": n_requests,
        "mixture": mixture or "DEFAULT_MIXTURE (uniform four-class)",
        "ttft_avg_ms": round(s["ttft"]["avg_us"] / 1e3, 2),
        "jct_avg_ms": round(s["jct"]["avg_us"] / 1e3, 2),
        "ttft_p99_ms": round(s["ttft"]["p99_us"] / 1e3, 2),
        "jct_p99_ms": round(s["jct"]["p99_us"] / 1e3, 2),
        "makespan_s": round(s["makespan_us"] / 1e6, 3),
        "tok_s_per_gpu": round((gen_tokens + prompt_tokens) / (s["makespan_us"] / 1e6) / phys, 1),
        "decode_tok_s_per_gpu": round(gen_tokens / (s["makespan_us"] / 1e6) / phys, 1),
        "prefill_tok_s_device": round(d.get("prefill_tok_s_device", 0.0), 1),
        "decode_tok_s_device": round(d.get("decode_tok_s_device", 0.0), 1),
        "kv_handoff_gb_s": round(d.get("handoff_gb_s", 0.0), 1),
        "decode_capacity_tokens": d.get("mem_capacity_tokens"),
        "perf_per_dollar": round(s["perf_per_dollar"], 4),
        "perf_per_dollar_physical": round(d.get("perf_per_dollar_physical", 0.0), 4),
        "gpu_resource_s": round(d.get("gpu_resource_us", 0) / 1e6, 3),
        "reference_modeled": {"ttft_avg_ms": round(sim["ttft"]["avg_us"] / 1e3, 2),
                              "jct_avg_ms": round(sim["jct"]["avg_us"] / 1e3, 2),
                              "scheduler_wall_s": round(sim_wall, 3),
                              "note": "pdsim cost model (V100-calibrated) on the same workload; "
                                      "wall time of the single-thread scheduler port"},
    }
    if streaming:
        out["kv_streaming"] = "chunk"
    return out


def serving_run(args) -> dict:
    """One GPU, co-located instances: Mixed-N (C1/C4 proxy) TetriInfer vs the
    coupled baseline, and the Llama-2-7B LPHD/HPHD decode-heavy mix (C5 proxy)."""
    n = args.serving_n
    out = {"note": "1 GPU: prefill and decode instances co-located (separate streams and "
                   "pools, device-local KV handoff); perf_per_dollar_physical bills the GPU "
                   "once, perf_per_dollar is pdsim's sum of instance episode spans"}
    out[f"mixed{n}_1p1d"] = guarded(lambda: serving_leg(args, 1, 1, n, colocate=True))
    out[f"mixed{n}_1p1d_streaming"] = guarded(
        lambda: serving_leg(args, 1, 1, n, colocate=True, streaming=True))
    out[f"mixed{n}_coupled"] = guarded(lambda: serving_leg(args, 1, 0, n, colocate=True,
                                                           coupled=True))
    out["c5proxy_llama_lphd_hphd_1p1d"] = guarded(
        lambda: serving_leg(args, 1, 1, n, mixture=C5_MIX, model="llama-2-7b", colocate=True))
    out["c1_tiny_decoder_1p1d"] = c1_run(args)
    return out


# P:D-split serving legs per GPU count (BASELINE.json configs[2..4]):
# (name, prefill instances, decode instances, mixture, model)
MULTI_GPU_LEGS = {
    2: [("c3_1p1d", 1, 1, C3_MIX, None)],
    4: [("c4_1p3d", 1, 3, None, None), ("c4_2p2d", 2, 2, None, None)],
    8: [("c4_2p6d", 2, 6, None, None), ("c4_4p4d", 4, 4, None, None),
        ("c5_llama_2p6d", 2, 6, C5_MIX, "llama-2-7b")],
}


def multi_gpu_run(args, n: int, peaks: dict) -> dict:
    """The disaggregated system on n GPUs of this box (one host process drives
    every instance; pdsim/control.py's scheduler is centralised):
    cross-GPU KV handoff over NVLink (SM peer-store kernel vs copy engines),
    handoff/compute overlap, and P:D-split serving -- C3 (1P:1D, LPLD/HPLD) on 2
    GPUs, C4 splits 1:3 and 2:2 on 4, 2:6 and 4:4 on 8, C5 (Llama-2-7B,
    LPHD/HPHD, 2:6) on 8 (BASELINE.json configs[2..4])."""
    from paper_2401_11181_b200 import native
    shape = native.MODELS[args.model]
    out = {"n_gpus": n}
    p2p = guarded(lambda: p2p_copy_gbs(0, 1))
    gbs = p2p if isinstance(p2p, float) else None
    out["kv_handoff_nvlink"] = guarded(lambda: handoff_run(args, shape, 0, 1, peaks, p2p_gbs=gbs))
    out["overlap_nvlink"] = guarded(lambda: overlap_run(args, shape, 0, 1))
    n_req = {"c5_llama_2p6d": args.c5_n}
    for name, p, d, mix, model in MULTI_GPU_LEGS.get(n, []):
        out[name] = guarded(lambda: serving_leg(args, p, d, n_req.get(name, args.serving_multi_n),
                                                mixture=mix, model=model))
    return out


def main():
    if os.environ.get("TK_BENCH_WATCHDOG"):
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["TK_BENCH_WATCHDOG"]), exit=True)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="tetri", choices=["tetri", "reference"])
    ap.add_argument("--model", default="opt-13b")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-serving", action="store_true")
    ap.add_argument("--no-decode", action="store_true")
    ap.add_argument("--serving-n", type=int, default=128)
    ap.add_argument("--serving-multi-n", type=int, default=128)
    ap.add_argument("--c5-n", type=int, default=1024)
    args = ap.parse_args()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    leave_group(world)


if __name__ == "__main__":
    main()
