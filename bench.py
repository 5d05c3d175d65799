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
  on a bounded sample (one OPT-13B layer on sampled chunks, x40 layers).

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
    committed ncu --set full captures, profiles/r01_gemm_traffic.json), weighted by this
    run's launches of each shape, next to the algorithmic bytes of the same launches."""
    p = ROOT / "profiles" / "r01_gemm_traffic.json"
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
            "ratio": round(dram / alg, 3), "source": "profiles/r01_gemm_traffic.json (M=512 shapes)"}


# ---------------------------------------------------------------- CPU port (oracle)

def cpu_port_sample(plan_chunks, max_seconds: float = 25.0, threads: int | None = None):
    """fp32 oracle timing of sampled chunks, one OPT-13B layer each (x40 extrapolated).

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
            ora.layer(0, x, rows, cache)
        spent += time.perf_counter() - t
        tokens += real
        done += 1
        if spent * full_layers > 0 and spent > max_seconds:
            break
    tok_s = tokens / (spent * full_layers)
    desc = (f"fp32 torch oracle, {done} sampled C2 chunks ({tokens} tokens), one OPT-13B layer "
            f"each incl. paged causal attention over the real prefix, x{full_layers} layers")
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
    # warmup steps untimed
    for s in samples[:args.warmup]:
        cpu_port_sample([s], max_seconds=1e9)
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
                   "step": "one sampled chunk, one layer x40 (CPU port)"},
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
    inst = native.Instance(shape, device=local, seed=args.seed, kv_pages=max_pages,
                           page_tokens=PAGE, max_chunk=CHUNK)

    def run_round(plan):
        evs, toks = [], 0
        h2d = d2h = 0
        verbose = os.environ.get("TK_BENCH_VERBOSE")
        for ci, (ids, slices, bt, real) in enumerate(plan):
            ev, out = inst.prefill_chunk(ids, slices, bt)
            if verbose:
                ev.wait()
                print(f"chunk {ci} slices={[(s[0], s[1]) for s in slices]} "
                      f"{ev.elapsed_ns / 1e6:.2f} ms", file=sys.stderr, flush=True)
            a, b = inst.staged_bytes()
            h2d, d2h = h2d + a, d2h + b
            evs.append((ev, out))
            toks += real
        for ev, _ in evs:
            ev.wait()  # publishes each chunk's first tokens to host memory
        dev_ns = native.event_elapsed_ns(evs[0][0], evs[-1][0])
        return toks, dev_ns, h2d, d2h

    for i in range(args.warmup):
        run_round(plans[i % len(plans)])
    inst.sync()
    clocks = ClockSampler(local)
    barrier(world)
    inst.sync()
    clocks.start()
    launches0 = native.launch_count()
    t0 = time.perf_counter()
    tokens = dev_ns = h2d = d2h = 0
    for i in range(args.steps):
        t, ns, a, b = run_round(plans[(args.warmup + i) % len(plans)])
        tokens, dev_ns, h2d, d2h = tokens + t, dev_ns + ns, h2d + a, d2h + b
    inst.sync()
    wall = time.perf_counter() - t0
    launches = native.launch_count() - launches0
    barrier(world)
    clk = clocks.stop()
    # Per-kernel breakdown (roofline, shares): the same rounds again, every
    # launch bracketed by CUDA events on the compute stream.  Kept out of the
    # timed region above so the event records do not perturb `value`.
    inst.profile(True)
    prof_ns = 0
    for i in range(args.steps):
        prof_ns += run_round(plans[(args.warmup + i) % len(plans)])[1]
    inst.sync()
    prof = inst.profile_read()
    inst.profile(False)

    dev_s = dist_max(dev_ns / 1e9, world)
    wall_s = dist_max(wall, world)
    total_tokens = tokens * world
    peaks = measured_peaks()
    gemm_kinds = ("qkv_gemm", "o_gemm", "fc1_gemm", "fc2_gemm")
    g_ms = sum(prof[k]["ms"] for k in gemm_kinds)
    g_fl = sum(prof[k]["flops"] for k in gemm_kinds)
    g_n = sum(prof[k]["launches"] for k in gemm_kinds)
    achieved = g_fl / (g_ms / 1e3) / 1e12 if g_ms else 0.0
    traffic = gemm_traffic(prof)
    peak = peaks["bf16_tflops_sustained"]
    attn = prof["attention"]
    if rank != 0:
        return
    line = {
        "metric": METRIC,
        "value": round(total_tokens / dev_s, 2),
        "unit": "tok/s",
        "n_gpus": world,
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
            "parallelism": f"replicas x{world} (weak)",
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
    if world == 1 and not args.no_decode:
        line["decode"] = decode_run(args, shape, local, peaks)
        if args.model == "opt-13b":
            # BASELINE.json configs[4] at one GPU: Llama-2-7B-shaped large decode batches
            line["decode"].update(decode_run(args, native.MODELS["llama-2-7b"], local, peaks,
                                             configs=((256, 1024),), tag="llama-2-7b_"))
    if world == 1 and not args.no_decode:
        line["kv_handoff"] = handoff_run(args, shape, local, peaks)
        line["predictor"] = predictor_run(args, local, peaks)
    if world == 1 and not args.no_serving:
        line["serving"] = serving_run(args)
    if world == 1 and not args.no_cpu_baseline:
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
        evs = [inst.decode_step(last, [ctx + 3 + i] * batch, bt, pages_per)[0]
               for i in range(steps)]
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
            "share_of_step": {k: round(v["ms"] / (pns / 1e6), 4) for k, v in prof.items()},
        }
    return out


def handoff_run(args, shape, device: int, peaks: dict, prompts=(512, 900, 8192)) -> dict:
    """P->D KV handoff (tk_kv_send, pdsim/prefill.py:420-424) between two
    instances co-located on one GPU: one copy-kernel launch per request, pages
    scattered on both sides.  bytes = prompt pages x page bytes (costs.py:137
    rounds to whole pages here); HBM traffic = 2 x bytes (read + write)."""
    import random

    from paper_2401_11181_b200 import costs, native
    n_max = (max(prompts) + PAGE - 1) // PAGE
    src = native.Instance(shape, device=device, seed=args.seed, kv_pages=n_max + 64, max_chunk=64)
    dst = native.Instance(shape, device=device, seed=args.seed, kv_pages=n_max + 64, max_chunk=64)
    rng = random.Random(args.seed)
    out = {"note": "single GPU: device-local copy bounded by HBM; NVLink peer stores use the "
                   "same kernel with a peer destination pool (not measurable on a 1-GPU box)"}
    for n_tok in prompts:
        n = (n_tok + PAGE - 1) // PAGE
        sp, dp = rng.sample(range(n_max + 64), n), rng.sample(range(n_max + 64), n)
        for _ in range(3):
            src.kv_send(sp, dst, dp).wait()
        evs = [src.kv_send(sp, dst, dp) for _ in range(8)]
        for e in evs:
            e.wait()
        ns = sorted(e.elapsed_ns for e in evs)[len(evs) // 2]
        nbytes = n * src.page_bytes
        hbm = 2 * nbytes / (ns / 1e9) / 1e9
        out[f"prompt{n_tok}"] = {
            "pages": n, "bytes": nbytes, "device_us": round(ns / 1e3, 1),
            "handoff_gb_s": round(nbytes / (ns / 1e9) / 1e9, 1),
            "roofline": {"bound": "hbm", "achieved": round(hbm, 1), "peak": peaks["hbm_gbs"],
                         "unit": "GB/s", "frac": round(hbm / peaks["hbm_gbs"], 4)},
            "reference_modeled_us_nvlink300": costs.transfer_latency(
                costs.load_calibration({"preset": "nvlink300"}), n_tok),
        }
    src.close(), dst.close()
    return out


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
    ns = native.event_elapsed_ns(evs[0], evs[-1]) / (len(evs) - 1)
    inst.close()
    params = 12 * (4 * 768 * 768 + 2 * 768 * 3072)
    flops = 2 * params * n * length + 4 * 768 * 12 * n * length * (length + 1) / 2
    tf = flops / (ns / 1e9) / 1e12
    return {"batch": n, "len": length, "device_us": round(ns / 1e3, 1),
            "tflops": round(tf, 1), "frac_of_peak": round(tf / peaks["bf16_tflops_sustained"], 4),
            "note": "tiny model: launch/latency bound, not tensor bound"}


def serving_run(args) -> dict:
    """Mixed workload through the reference scheduler + CUDA executor (measured clock)."""
    import paper_2401_11181_b200 as tk
    from paper_2401_11181_b200.experiment import run_experiment
    cfg = {"cluster": {"prefill": 1, "decode": 1},
           "workload": {"n_requests": args.serving_n},
           "cost_model": {"preset": "nvlink300", "mem_capacity_tokens": 40000},
           "model": {"name": args.model, "prefill_pages": 2048, "staging_pages": 512,
                     "max_decode_batch": 256, "seed": args.seed}}
    sim = run_experiment(tk.config_from_dict(cfg), seed=args.seed).summary
    res = run_experiment(tk.config_from_dict(dict(cfg, executor="cuda")), seed=args.seed)
    s, d = res.summary, res.summary["device"]
    st = run_experiment(tk.config_from_dict(dict(cfg, executor="cuda", kv_streaming="chunk")),
                        seed=args.seed).summary
    coupled_cfg = dict(cfg, system="coupled", cluster={"coupled": 1}, executor="cuda")
    c = run_experiment(tk.config_from_dict(coupled_cfg), seed=args.seed).summary
    return {
        "workload": f"Mixed-{args.serving_n} (four-class, burst), 1 prefill + 1 decode instance "
                    f"co-located on one GPU, {args.model}, reserve_dynamic, power-of-two, "
                    "predictor g=200 p=0.749 (device classifier for cost)",
        "ttft_avg_ms": round(s["ttft"]["avg_us"] / 1e3, 2),
        "jct_avg_ms": round(s["jct"]["avg_us"] / 1e3, 2),
        "ttft_p99_ms": round(s["ttft"]["p99_us"] / 1e3, 2),
        "jct_p99_ms": round(s["jct"]["p99_us"] / 1e3, 2),
        "prefill_tok_s": round(d.get("prefill_tok_s_device", 0.0), 1),
        "decode_tok_s": round(d.get("decode_tok_s_device", 0.0), 1),
        "kv_handoff_gb_s": round(d.get("handoff_gb_s", 0.0), 1),
        "makespan_s": round(s["makespan_us"] / 1e6, 3),
        "reference_modeled": {"ttft_avg_ms": round(sim["ttft"]["avg_us"] / 1e3, 2),
                              "jct_avg_ms": round(sim["jct"]["avg_us"] / 1e3, 2),
                              "note": "pdsim cost model (V100-calibrated), same workload"},
        "coupled_baseline": {"system": "coupled (vLLM-like, pdsim/coupled.py) on the same GPU",
                             "ttft_avg_ms": round(c["ttft"]["avg_us"] / 1e3, 2),
                             "jct_avg_ms": round(c["jct"]["avg_us"] / 1e3, 2),
                             "perf_per_dollar": round(c["perf_per_dollar"], 4)},
        "perf_per_dollar": round(s["perf_per_dollar"], 4),
        "kv_streaming_chunk": {"note": "same run with each chunk's KV shipped as it completes",
                               "ttft_avg_ms": round(st["ttft"]["avg_us"] / 1e3, 2),
                               "jct_avg_ms": round(st["jct"]["avg_us"] / 1e3, 2)},
    }


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
    ap.add_argument("--serving-n", type=int, default=32)
    args = ap.parse_args()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
