"""Kernel-level parity on the B200: each sm_100a kernel against a plain torch
fp32 reference of the same op (the floating-point tier of the oracle).

Tolerances are bf16 ones: outputs are rounded to bf16 (8 bits of mantissa,
relative step 2^-8 = 0.0039), accumulations are fp32.
"""

import pytest
import torch

from paper_2401_11181_b200 import native

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    native.load()


def _rel_err(x, ref):
    return ((x.float() - ref).abs().max() / ref.abs().max().clamp_min(1e-6)).item()


@pytest.mark.parametrize("M,N,K", [
    (128, 256, 64),      # one tile, one k-block
    (512, 5120, 5120),   # OPT-13B O-proj at ChunkSize 512
    (512, 15360, 5120),  # fused QKV
    (300, 1024, 768),    # ragged M (TMA zero-fill, masked rows)
    (7, 50272, 256),     # LM-head-like: N not a multiple of the tile
    (33, 3072, 768),     # decode-sized M, BN=256, stream-K split
    (64, 768, 3072),     # BN=128 path
    (512, 48, 768),      # classifier head (N=48)
    (256, 5120, 5120),   # 2-CTA cluster multicast
    (1024, 3072, 768),   # two m-groups of a 4-CTA cluster
    (384, 2048, 1024),   # tiles_m=3 -> no cluster
    (1, 5120, 5120),     # skinny (swap-AB) path: single decode row
    (16, 5120, 20480),   # skinny NB=16, long K (many stream-K contributors)
    (100, 20480, 5120),  # skinny NB=128
    (128, 15360, 5120),  # skinny at the M boundary
    (907, 2304, 768),    # narrow (160-wide) pair tiles, ragged last n-tile, two m-groups
    (512, 5000, 4096),   # narrow, N not a multiple of 160
    (907, 768, 768),     # BN=128 with a 4-CTA cluster (predictor O-proj)
    (907, 768, 3072),    # same, FC2
    (512, 5120, 20480),  # FC2: stream-K, final fixups through the bulk-copied partials
    (512, 20480, 5120),  # FC1: split tiles mid-range and at the end (8-CTA clusters)
    (512, 15360, 5120),  # QKV shape: 2 x 2 pairs per cluster, A and B multicast
    (1024, 5120, 5120),  # two cluster m-groups of the 8-CTA schedule
    (512, 2560, 20480),  # 3-4 contributors per tile (partials beyond the ring: register path)
])
def test_gemm_matches_fp32(M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    a = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    b = (torch.randn(N, K, device="cuda", generator=g) * 0.05).bfloat16()
    ref = a.float() @ b.float().t()
    out = native.gemm(a, b, epilogue=native.EPI_F32)
    torch.cuda.synchronize()
    assert _rel_err(out, ref) < 2e-3
    bias = (torch.randn(N, device="cuda", generator=g)).bfloat16()
    out2 = native.gemm(a, b, bias=bias, epilogue=native.EPI_BF16_BIAS_RELU)
    ref2 = torch.relu(ref + bias.float())
    assert _rel_err(out2, ref2) < 1e-2


@pytest.mark.parametrize("M", [512, 32])
def test_gemm_residual_epilogue_and_workspace_reuse(M):
    N, K = 5120, 20480  # FC2 shape; several CTAs share each tile
    g = torch.Generator(device="cuda").manual_seed(1)
    a = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    b = (torch.randn(N, K, device="cuda", generator=g) * 0.02).bfloat16()
    bias = torch.randn(N, device="cuda", generator=g).bfloat16()
    resid = torch.randn(M, N, device="cuda", generator=g)
    ws = None
    for _ in range(3):  # the stream-K workspace must come back zeroed each time
        out = resid.clone()
        import ctypes
        nbytes = ctypes.c_int64()
        native.check(native.load().tk_gemm_workspace_bytes(M, N, K, ctypes.byref(nbytes)))
        if ws is None:
            ws = torch.zeros(nbytes.value, dtype=torch.uint8, device="cuda")
        native.gemm(a, b, bias=bias, epilogue=native.EPI_F32_BIAS_RESID, out=out, workspace=ws)
        torch.cuda.synchronize()
        ref = resid + a.float() @ b.float().t() + bias.float()
        assert _rel_err(out, ref) < 2e-3


def test_layernorm_and_argmax():
    x = torch.randn(37, 5120, device="cuda") * 3 + 1
    w = torch.randn(5120, device="cuda").bfloat16()
    b = torch.randn(5120, device="cuda").bfloat16()
    y = native.layernorm(x, w, b)
    ref = torch.nn.functional.layer_norm(x, (5120,), w.float(), b.float(), 1e-5)
    assert (y.float() - ref).abs().max().item() < 0.05
    logits = torch.randn(9, 50272, device="cuda")
    logits[3, 17] = logits[3, 40000] = 100.0  # tie -> first index
    idx = native.argmax(logits)
    assert idx.tolist() == logits.argmax(dim=1).tolist()
    assert idx[3].item() == 17


def _pool(n_pages, L, H, D, pt, gen):
    return (torch.randn(n_pages, L, H, 2, pt, D, device="cuda", generator=gen) * 0.5).bfloat16()


def _gather_kv(pool, layer, pages, n_tok, pt):
    # -> K, V [H, n_tok, D] fp32 for one request
    ks, vs = [], []
    for p in pages:  # pool: [page][layer][head][K|V][slot][d]
        ks.append(pool[p, layer, :, 0])
        vs.append(pool[p, layer, :, 1])
    K = torch.cat(ks, dim=1)[:, :n_tok].float()
    V = torch.cat(vs, dim=1)[:, :n_tok].float()
    return K, V


# Attention parity metric.  Per (query row, head): normwise relative error
# ||o - ref|| / ||ref|| and cosine similarity.  Long contexts make the outputs
# themselves small (a near-uniform softmax averages thousands of V rows), so
# an absolute tolerance cannot see a dropped page; a normwise relative one
# can.  bf16 output rounding alone gives ~3e-3; a dropped 16-key page, a
# dropped 128-key block or a causal mask shifted by one give >= 4e-2 at the
# sizes below (measured on the reference itself, and asserted as negative
# controls in every test).  Scores are sharpened (q x4, score std ~2) so that
# individual keys matter.
ATTN_REL = 1e-2
ATTN_COS = 0.9999
Q_SHARPEN = 4.0


def _attn_metric(got, ref):
    """got/ref [..., D] -> (max normwise relative error, min cosine)."""
    got, ref = got.float(), ref.float()
    rel = (got - ref).norm(dim=-1) / ref.norm(dim=-1).clamp_min(1e-12)
    cos = torch.nn.functional.cosine_similarity(got, ref, dim=-1)
    return rel.max().item(), cos.min().item()


def _attn_ok(m) -> bool:
    return m[0] <= ATTN_REL and m[1] >= ATTN_COS


def _ref_attention(q, K, V, qpos, scale, mask_shift=0):
    """q [H, n, D], K/V [H, ctx, D] fp32, causal by absolute position (+ shift)."""
    sc = torch.einsum("hqd,hkd->hqk", q, K) * scale
    kpos = torch.arange(K.shape[1], device=q.device)[None, :]
    sc = sc.masked_fill(kpos > qpos[:, None] + mask_shift, float("-inf"))
    p = torch.nan_to_num(torch.softmax(sc, -1))
    return torch.einsum("hqk,hkd->hqd", p, V)


def _decode_case(ctxs, seed, H=8, L=3, D=128, pt=16):
    g = torch.Generator(device="cuda").manual_seed(seed)
    n_pages = sum((c + pt - 1) // pt for c in ctxs) + 4
    pool = _pool(n_pages, L, H, D, pt, g)
    perm = torch.randperm(n_pages, generator=torch.Generator().manual_seed(0)).tolist()
    stride = max((c + pt - 1) // pt for c in ctxs)
    bt = torch.zeros(len(ctxs), stride, dtype=torch.int32)
    cur, tables = 0, []
    for b, c in enumerate(ctxs):
        np_ = (c + pt - 1) // pt
        pages = perm[cur:cur + np_]
        cur += np_
        bt[b, :np_] = torch.tensor(pages, dtype=torch.int32)
        tables.append(pages)
    q = (torch.randn(len(ctxs), H, D, device="cuda", generator=g) * Q_SHARPEN).bfloat16()
    return pool, bt, tables, q, perm[cur:]


@pytest.mark.parametrize("ctxs,D", [([1], 128), ([16, 17, 300], 128),
                                    ([1000, 4097, 40, 2048, 9000], 128),
                                    ([8192, 3000, 10240, 511], 128),
                                    ([1, 33, 300], 64), ([1000, 4097, 40, 2048], 64)])
def test_paged_decode_attention(ctxs, D):
    """head_dim 64 is the OPT-125M tiny decoder (BASELINE.json configs[0])."""
    L, H, pt, layer = 3, 8, 16, 1
    pool, bt, tables, q, spare = _decode_case(ctxs, len(ctxs) * 7 + ctxs[0], H, L, D, pt)
    lens = torch.tensor(ctxs, dtype=torch.int32, device="cuda")
    o = native.paged_decode_attention(q, pool, layer, L, bt.cuda(), lens, pt)
    torch.cuda.synchronize()
    worst = (0.0, 1.0)
    for b, c in enumerate(ctxs):
        K, V = _gather_kv(pool, layer, tables[b], c, pt)
        qpos = torch.tensor([c - 1], device="cuda")
        ref = _ref_attention(q[b].float()[:, None], K, V, qpos, D ** -0.5)[:, 0]
        m = _attn_metric(o[b], ref)
        worst = (max(worst[0], m[0]), min(worst[1], m[1]))
        assert _attn_ok(m), (c, m)
        if c >= 2:  # negative control: missing the newest key must be detected
            if c <= 64:
                short = _ref_attention(q[b].float()[:, None], K, V, qpos, D ** -0.5, -1)[:, 0]
                assert not _attn_ok(_attn_metric(o[b], short)), c
    # negative control on the device: one page of the longest context replaced
    b = max(range(len(ctxs)), key=lambda i: ctxs[i])
    if ctxs[b] >= 64:
        bad = bt.clone()
        bad[b, len(tables[b]) // 2] = spare[0] if spare else tables[b][0]
        o_bad = native.paged_decode_attention(q, pool, layer, L, bad.cuda(), lens, pt)
        K, V = _gather_kv(pool, layer, tables[b], ctxs[b], pt)
        ref = _ref_attention(q[b].float()[:, None], K, V, torch.tensor([ctxs[b] - 1],
                                                                       device="cuda"),
                             D ** -0.5)[:, 0]
        assert not _attn_ok(_attn_metric(o_bad[b], ref)), "dropped page not detected"
    print(f"decode attention {ctxs}: max rel {worst[0]:.2e}, min cos {worst[1]:.6f}")


def _chunk_case(reqs, H, seed, L=2, D=128, pt=16, scatter=True):
    g = torch.Generator(device="cuda").manual_seed(seed)
    pages_per = [(s + n + pt - 1) // pt for s, n in reqs]
    n_pages = sum(pages_per) + 2
    pool = _pool(n_pages, L, H, D, pt, g)
    order = (torch.randperm(n_pages, generator=torch.Generator().manual_seed(3)).tolist()
             if scatter else list(range(n_pages)))
    bt, slices, off = [], [], 0
    for (s, n), np_ in zip(reqs, pages_per):
        slices.append((s, n, off, np_, 1))
        bt.extend(order[off:off + np_])
        off += np_
    n_tok = sum(n for _, n in reqs)
    qkv = torch.randn(n_tok, 3 * H * D, device="cuda", generator=g)
    qkv[:, :H * D] *= Q_SHARPEN
    return pool, bt, slices, qkv.bfloat16(), order[off:]


def _check_chunk(o, qkv, pool, bt, slices, layer, H, D, pt, negative=True):
    row, worst = 0, (0.0, 1.0)
    for (s, n, bto, np_, _) in slices:
        K, V = _gather_kv(pool, layer, bt[bto:bto + np_], s + n, pt)
        q = qkv[row:row + n, :H * D].float().view(n, H, D).transpose(0, 1)  # H, n, D
        qpos = torch.arange(s, s + n, device="cuda")
        ref = _ref_attention(q, K, V, qpos, D ** -0.5).transpose(0, 1)  # n, H, D
        got = o[row:row + n].view(n, H, D)
        m = _attn_metric(got, ref)
        worst = (max(worst[0], m[0]), min(worst[1], m[1]))
        assert _attn_ok(m), (s, n, m)
        if negative:  # a causal mask off by one either way must be detected
            for shift in (-1, 1):
                bad = _ref_attention(q, K, V, qpos, D ** -0.5, shift).transpose(0, 1)
                assert not _attn_ok(_attn_metric(got, bad)), (s, n, shift)
        row += n
    return worst


def test_chunk_attention_mixed_slices():
    """A chunk holding a prompt tail with a long prefix, two whole prompts and the
    head of a fourth prompt (several slices per chunk, as pdsim chunkify packs)."""
    L, H, D, pt, layer = 2, 4, 128, 16, 1
    reqs = [(394, 118), (0, 18), (0, 100), (0, 276)]
    pool, bt, slices, qkv, spare = _chunk_case(reqs, H, 5, L, D, pt)
    o = native.chunk_attention(qkv, 3 * H * D, pool, layer, L, H, D, slices, bt, pt)
    torch.cuda.synchronize()
    worst = _check_chunk(o, qkv, pool, bt, slices, layer, H, D, pt)
    # negative control on the device: one prefix page of the first slice swapped
    bad_bt = list(bt)
    bad_bt[3] = spare[0]
    o_bad = native.chunk_attention(qkv, 3 * H * D, pool, layer, L, H, D, slices, bad_bt, pt)
    with pytest.raises(AssertionError):
        _check_chunk(o_bad, qkv, pool, bt, slices[:1], layer, H, D, pt, negative=False)
    print(f"chunk attention mixed: max rel {worst[0]:.2e}, min cos {worst[1]:.6f}")


@pytest.mark.parametrize("prefix,n,H,D", [(0, 512, 40, 128), (2048, 512, 40, 128),
                                          (3000, 512, 40, 128), (4096, 512, 40, 128),
                                          (7680, 512, 8, 128), (130, 77, 40, 128),
                                          (256, 300, 3, 128),
                                          # head_dim 64: the OPT-125M-class predictor /
                                          # tiny decoder on the same tcgen05 kernel
                                          (0, 512, 12, 64), (2048, 512, 12, 64),
                                          (130, 77, 12, 64), (1000, 300, 5, 64)])
def test_chunk_attention_long_prefix_pieces(prefix, n, H, D):
    """One slice over a long paged prefix (the C2 regime: 2k-8k prompts in 512
    chunks): the stream-K plan cuts (head, tile pair) work into pieces merged by
    the combine kernel; unaligned starts and lone tiles.  Every head is checked,
    with negative controls (shifted mask, and a dropped 128-key block on the
    device)."""
    L, pt, layer = 2, 16, 0
    pool, bt, slices, qkv, spare = _chunk_case([(prefix, n)], H, prefix + n, L, D, pt)
    o = native.chunk_attention(qkv, 3 * H * D, pool, layer, L, H, D, slices, bt, pt)
    torch.cuda.synchronize()
    worst = _check_chunk(o, qkv, pool, bt, slices, layer, H, D, pt)
    if prefix >= 256:
        # a whole 128-key block (8 pages) of the prefix replaced by other pages
        bad_bt = list(bt)
        for i in range(8):
            bad_bt[(prefix // 2) // pt + i] = spare[i % len(spare)] if spare else bt[0]
        o_bad = native.chunk_attention(qkv, 3 * H * D, pool, layer, L, H, D, slices, bad_bt, pt)
        with pytest.raises(AssertionError):
            _check_chunk(o_bad, qkv, pool, bt, slices, layer, H, D, pt, negative=False)
    print(f"chunk attention prefix {prefix} n {n} H {H}: max rel {worst[0]:.2e}, "
          f"min cos {worst[1]:.6f}")


@pytest.mark.parametrize("reqs,H", [([(394, 118), (0, 18), (0, 100), (0, 276)], 4),
                                     ([(0, 512)], 40), ([(2048, 512)], 40), ([(7680, 512)], 8),
                                     ([(130, 77)], 40), ([(256, 300)], 3), ([(3000, 700)], 5)])
def test_chunk_attention_cta_pair_kernel(monkeypatch, reqs, H):
    """The cta_group::2 form of the chunk attention (TK_FA_PAIR=1: 512-row quads,
    M=256 pair MMAs, each CTA holding half of every K/V block): mixed slices,
    short and long prefixes (stream-K pieces over four sub-tiles), ragged quads,
    with the same negative controls as the single-CTA kernel."""
    monkeypatch.setenv("TK_FA_PAIR", "1")
    L, D, pt, layer = 2, 128, 16, 1
    pool, bt, slices, qkv, spare = _chunk_case(reqs, H, 7, L, D, pt)
    o = native.chunk_attention(qkv, 3 * H * D, pool, layer, L, H, D, slices, bt, pt)
    torch.cuda.synchronize()
    worst = _check_chunk(o, qkv, pool, bt, slices, layer, H, D, pt)
    prefix = reqs[0][0]
    if prefix >= 256:
        bad_bt = list(bt)
        for i in range(8):
            bad_bt[(prefix // 2) // pt + i] = spare[i % len(spare)] if spare else bt[0]
        o_bad = native.chunk_attention(qkv, 3 * H * D, pool, layer, L, H, D, slices, bad_bt, pt)
        with pytest.raises(AssertionError):
            _check_chunk(o_bad, qkv, pool, bt, slices[:1], layer, H, D, pt, negative=False)
    print(f"cta-pair chunk attention {reqs} H {H}: max rel {worst[0]:.2e}, min cos {worst[1]:.6f}")


def test_gemm_shared_workspace_across_shapes():
    """One workspace serves every GEMM shape of a layer (as in the runtime)."""
    import ctypes
    shapes = [(512, 15360, 5120), (512, 5120, 5120), (33, 20480, 5120), (512, 5120, 20480),
              (7, 50272, 5120)]
    need = 0
    for M, N, K in shapes:
        nb = ctypes.c_int64()
        native.check(native.load().tk_gemm_workspace_bytes(M, N, K, ctypes.byref(nb)))
        need = max(need, nb.value)
    ws = torch.zeros(need, dtype=torch.uint8, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(3)
    for _ in range(2):
        for M, N, K in shapes:
            a = torch.randn(M, K, device="cuda", generator=g).bfloat16()
            b = (torch.randn(N, K, device="cuda", generator=g) * 0.02).bfloat16()
            out = native.gemm(a, b, epilogue=native.EPI_F32, workspace=ws)
            torch.cuda.synchronize()
            assert _rel_err(out, a.float() @ b.float().t()) < 2e-3, (M, N, K)


@pytest.mark.parametrize("M,N,K", [
    (512, 2560, 20480),  # pair kernel, 3-4 contributors per split tile
    (16, 5120, 20480),   # skinny (decode) GEMM, up to 16 contributors per tile
    (100, 20480, 5120),  # skinny NB=128
    (384, 5120, 20480),  # odd m-tile count: the 1-CTA kernel's fixup
])
def test_gemm_is_deterministic(M, N, K):
    """Split (stream-K) tiles are summed in contributor order with the finishing
    CTA's own accumulator at its rank, so repeated runs are bit-identical whatever
    the arrival order of the contributors."""
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    a = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    b = (torch.randn(N, K, device="cuda", generator=g) * 0.05).bfloat16()
    outs = []
    for _ in range(6):
        outs.append(native.gemm(a, b, epilogue=native.EPI_F32).clone())
        torch.cuda.synchronize()
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
    ref = a.float() @ b.float().t()
    assert _rel_err(outs[0], ref) < 2e-3
