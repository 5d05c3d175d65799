"""End-to-end device parity at the widths the benchmarks are quoted on.

The toy-width tests (test_gpu_model.py) cannot reach the schedules the
benchmark runs: the 40-head attention plan with stream-K pieces and the
combine kernel, the QKV GEMM epilogue that scatters K/V straight into pages
at 40 heads, the 144/160-wide 2-CTA GEMM schedules at N=5120, the
10,242-row learned positions and the 50,272-row LM head.  These tests run
the real widths with two layers (the per-layer work is identical for all
40), through the C ABI, against the fp32 oracle executed on the same GPU
(oracle/model_ref.py with TF32 off -- the checker, never the product):

* OPT-13B width on the reference's own prompt lengths [18, 100, 512, 900]
  (pkg/tests/test_prefill.py:58-67 chunk layout), then decode steps;
* OPT-13B width on one full C2 scheduling round (bench.py workload: SJF 16 of
  {2048, 4096, 6144, 8192}, 144 chunks, prefixes up to 7680), first-token
  logits of all 16 prompts, KV pages, then decode steps at ctx up to 8193;
* Llama-2-7B width at decode batch 128 with contexts up to 4096 (configs[4]
  shape), KV pages seeded through the swap path;
* the OPT-125M-shaped length predictor's 41 class scores (not just argmax).

Tolerances: tests/parity_util.py (logits within 1% of the row's range,
cosine >= 0.9999, greedy identity on decided rows, minimum decided counts).
"""

import ctypes
import random

import numpy as np
import pytest
import torch

import bench
from oracle.model_ref import OracleModel, PagedCache, Shape, bf16_bits_to_f32
from paper_2401_11181_b200 import native
from paper_2401_11181_b200.prefill import chunkify
from paper_2401_11181_b200.workload import Request, token_ids_for
from parity_util import greedy_agrees, logits_close, record

pytestmark = pytest.mark.gpu

PT = 16
OPT13B_2L = native.ModelShape("opt-13b-2l", native.TK_ARCH_OPT, 2, 5120, 40, 20480, 50272,
                              max_positions=10240)
LLAMA7B_2L = native.ModelShape("llama-2-7b-2l", native.TK_ARCH_LLAMA, 2, 4096, 32, 11008, 32000,
                               max_positions=4096)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    native.load()


def _oshape(m: native.ModelShape) -> Shape:
    return Shape(m.arch, m.n_layers, m.hidden, m.n_heads, m.ffn, m.vocab, m.max_positions,
                 m.n_labels, m.norm_eps, m.rope_theta)


def _tables(reqs, extra_tokens=8):
    tables, nxt = {}, 0
    for r in reqs:
        np_ = (r.prompt_len + extra_tokens + PT - 1) // PT
        tables[r.id] = list(range(nxt, nxt + np_))
        nxt += np_
    return tables, nxt


def _prefill_both(inst, ora, cache, chunks, prompts, lens, tables):
    """Every chunk on the device and the oracle; returns per emitting request
    (device logits row, oracle row, device first token)."""
    out = {}
    for chunk in chunks:
        ids, slices, bt = [], [], []
        for rid, start, n in chunk.slices:
            ids += prompts[rid][start:start + n]
            slices.append((start, n, len(bt), len(tables[rid]), int(start + n == lens[rid])))
            bt += tables[rid]
        ev, toks, logits = inst.prefill_chunk(ids, slices, bt, want_logits=True)
        ev.wait()
        ref = ora.prefill_chunk(cache, ids, slices, bt)
        e = 0
        for i, (rid, s, n) in enumerate(chunk.slices):
            if s + n == lens[rid]:
                out[rid] = (torch.from_numpy(logits[e].copy()), ref[e].cpu(), int(toks[i]))
                e += 1
            else:
                assert toks[i] == -1
    return out


def _decode_both(inst, ora, cache, rids, last, ctx, tables, steps):
    errs, decided, rows = [], 0, 0
    stride = max(len(tables[r]) for r in rids)
    for _ in range(steps):
        bt = []
        for r in rids:
            bt += tables[r] + [tables[r][0]] * (stride - len(tables[r]))
        ev, toks, logits = inst.decode_step(last, ctx, bt, stride, want_logits=True)
        ev.wait()
        ref = ora.decode_step(cache, last, ctx, [tables[r] for r in rids]).cpu()
        got = torch.from_numpy(logits)
        errs.append(logits_close(got, ref)[0])
        decided += greedy_agrees(got, ref)
        rows += len(rids)
        assert list(toks) == [int(v) for v in np.argmax(logits, axis=1)]
        last = [int(v) for v in ref.argmax(-1)]  # both sides continue on the oracle's tokens
        ctx = [c + 1 for c in ctx]
    return max(errs), decided, rows


def _page_rel_err(inst, cache, page, s: Shape) -> float:
    """Normwise relative error of one device KV page vs the oracle's, per
    (layer, K|V, head) block of [16 tokens x head_dim]."""
    got = bf16_bits_to_f32(inst.read_page(page)).view(
        s.n_layers, s.n_heads, 2, PT, s.head_dim).transpose(1, 2)  # -> [L][K|V][H][16][D]
    ref = cache.pages[page].cpu()
    num = (got - ref).flatten(3).norm(dim=-1)
    den = ref.flatten(3).norm(dim=-1).clamp_min(1e-12)
    return (num / den).max().item()


def test_opt13b_width_reference_prompts():
    """pdsim's own prompt lengths at OPT-13B width: chunk layout (0,0,18),(1,0,100),
    (2,0,394) | (2,394,118),(3,0,394) | (3,394,506) (pkg/tests/test_prefill.py:58-67),
    first tokens, then three decode steps."""
    m = OPT13B_2L
    lens = [18, 100, 512, 900]
    reqs = [Request(id=i, arrival_us=0, prompt_len=n, true_decode_len=4) for i, n in enumerate(lens)]
    chunks = chunkify(reqs, 512)
    assert [c.slices for c in chunks] == [[(0, 0, 18), (1, 0, 100), (2, 0, 394)],
                                          [(2, 394, 118), (3, 0, 394)], [(3, 394, 506)]]
    assert chunks[-1].padded == 6
    tables, n_pages = _tables(reqs)
    inst = native.Instance(m, device=0, seed=21, kv_pages=n_pages, max_chunk=512)
    ora = OracleModel.from_instance(_oshape(m), inst, device="cuda")
    cache = PagedCache(ora.s, n_pages, PT, device="cuda")
    prompts = {r.id: token_ids_for(r, m.vocab, seed=21) for r in reqs}
    out = _prefill_both(inst, ora, cache, chunks, prompts, dict(enumerate(lens)), tables)
    got = torch.stack([out[i][0] for i in range(4)])
    ref = torch.stack([out[i][1] for i in range(4)])
    err, cos = logits_close(got, ref)
    decided = greedy_agrees(got, ref)
    assert [out[i][2] for i in range(4)] == got.argmax(-1).tolist()
    page_err = max(_page_rel_err(inst, cache, tables[3][p], ora.s) for p in (0, 24, 56))
    assert page_err < 2e-2, page_err
    d_err, d_dec, d_rows = _decode_both(inst, ora, cache, list(range(4)),
                                        [int(v) for v in ref.argmax(-1)], list(lens), tables, 3)
    record("opt13b_width_reference_prompts", prefill_max_err=err, prefill_min_cos=cos,
           prefill_decided=decided, kv_page_rel_err=page_err, decode_max_err=d_err,
           decode_decided=d_dec, decode_rows=d_rows)
    assert decided + d_dec >= (4 + d_rows) // 2, "too few decided rows to test greedy identity"
    inst.close()


@pytest.mark.parametrize("pair_attention", [False, True], ids=["attn1cta", "attn2cta"])
def test_opt13b_width_c2_round(monkeypatch, pair_attention):
    """One full C2 scheduling round at OPT-13B width (144 chunks of 512, prefixes
    to 7680): the benchmark's own chunk layout, first-token logits of all 16
    prompts, KV pages deep in the 8192-token prompt, then decode at ctx <= 8193.
    attn2cta: the same round through the CTA-pair chunk attention (TK_FA_PAIR=1)."""
    if pair_attention:
        monkeypatch.setenv("TK_FA_PAIR", "1")
    m = OPT13B_2L
    _, rounds = bench.build_workload(0)
    batch, chunks = rounds[0]
    assert len(chunks) == 144 and max(r.prompt_len for r in batch) == 8192
    lens = {r.id: r.prompt_len for r in batch}
    tables, n_pages = _tables(batch)
    inst = native.Instance(m, device=0, seed=0, kv_pages=n_pages, max_chunk=512)
    ora = OracleModel.from_instance(_oshape(m), inst, device="cuda")
    cache = PagedCache(ora.s, n_pages, PT, device="cuda")
    prompts = {r.id: token_ids_for(r, m.vocab, seed=0) for r in batch}
    out = _prefill_both(inst, ora, cache, chunks, prompts, lens, tables)
    rids = [r.id for r in batch]
    assert sorted(out) == sorted(rids)
    got = torch.stack([out[r][0] for r in rids])
    ref = torch.stack([out[r][1] for r in rids])
    err, cos = logits_close(got, ref)
    decided = greedy_agrees(got, ref)
    longest = max(rids, key=lambda r: lens[r])
    page_err = max(_page_rel_err(inst, cache, tables[longest][p], ora.s) for p in (0, 255, 511))
    assert page_err < 2e-2, page_err
    d_err, d_dec, d_rows = _decode_both(inst, ora, cache, rids, [int(v) for v in ref.argmax(-1)],
                                        [lens[r] for r in rids], tables, 2)
    record("opt13b_width_c2_round" + ("_cta_pair" if pair_attention else ""), chunks=len(chunks), prefill_max_err=err, prefill_min_cos=cos,
           prefill_decided=decided, kv_page_rel_err=page_err, decode_max_err=d_err,
           decode_decided=d_dec, decode_rows=d_rows)
    assert decided >= 8 and d_dec >= d_rows // 2, (decided, d_dec, d_rows)
    inst.close()


def test_llama7b_width_decode_batch128():
    """Llama-2-7B width (RMSNorm, RoPE, SwiGLU), decode batch 128 with contexts up
    to 4096 over scattered pages (configs[4] shape at two layers).  The prefix KV
    is seeded with random pages through tk_swap_in; the oracle holds the same
    pages; two decode steps append RoPE'd K/V and must match."""
    m = LLAMA7B_2L
    s = _oshape(m)
    rng = random.Random(7)
    ctxs = [rng.randint(1, 2048) for _ in range(120)] + [4096, 4095, 3999, 3500, 2500, 4090, 17, 1]
    rng.shuffle(ctxs)
    B = len(ctxs)
    steps = 2
    need = [(c + steps + PT - 1) // PT for c in ctxs]
    n_pages = sum(need) + 8
    perm = list(range(n_pages))
    rng.shuffle(perm)
    tables, cur = {}, 0
    for b in range(B):
        tables[b] = perm[cur:cur + need[b]]
        cur += need[b]
    inst = native.Instance(m, device=0, seed=5, kv_pages=n_pages, max_chunk=B)
    ora = OracleModel.from_instance(s, inst, device="cuda")
    cache = PagedCache(s, n_pages, PT, device="cuda")
    pb = inst.page_bytes
    per = 512
    host = torch.empty(per * pb // 2, dtype=torch.bfloat16, pin_memory=True)
    g = torch.Generator(device="cuda").manual_seed(11)
    for lo in range(0, n_pages, per):
        ids = list(range(lo, min(n_pages, lo + per)))
        data = torch.randn(len(ids), s.n_layers, s.n_heads, 2, PT, s.head_dim, device="cuda",
                           generator=g).bfloat16()
        host[:data.numel()].copy_(data.flatten())
        inst.swap_in(ids, host.data_ptr()).wait()
        cache.pages[ids] = data.permute(0, 1, 3, 2, 4, 5).float()
    last = [rng.randrange(2, m.vocab) for _ in range(B)]
    d_err, d_dec, d_rows = _decode_both(inst, ora, cache, list(range(B)), last, ctxs, tables, steps)
    record("llama7b_width_decode_b128", batch=B, max_ctx=max(ctxs), decode_max_err=d_err,
           decode_decided=d_dec, decode_rows=d_rows)
    assert d_dec >= d_rows // 2, (d_dec, d_rows)
    inst.close()


def test_predictor_scores_match_oracle():
    """OPT-125M-shaped length predictor (12 layers, 41 buckets): class scores of
    a round's prompts (ids padded to the longest) vs the oracle's
    last-token scores."""
    m = native.PREDICTOR_125M
    inst = native.Instance(m, device=0, seed=9, kv_pages=16 * 32 + 8, max_chunk=16 * 512)
    ora = OracleModel.from_instance(_oshape(m), inst, device="cuda")
    lens = [18, 512, 77, 300, 900, 1, 255, 256, 64, 128, 400, 33, 512, 7, 100, 480]
    g = torch.Generator().manual_seed(0)
    prompts = [torch.randint(2, m.vocab, (n,), generator=g).tolist() for n in lens]
    buckets, scores = inst.predict_scores(sum(prompts, []), lens, max_len=512)
    ref = torch.stack([ora.full_forward(p[:512])[-1] for p in prompts]).cpu()
    got = torch.from_numpy(scores)
    err, cos = logits_close(got, ref)
    decided = greedy_agrees(got, ref)
    assert buckets == got.argmax(-1).tolist()
    record("predictor_scores", max_err=err, min_cos=cos, decided=decided, rows=len(lens))
    inst.close()
