"""Chunk-attention work plan (host side of attention_tc.cu, via tk_fa_plan; no GPU).

The plan pairs 128-row query tiles of each slice, splits the (head, pair,
128-key block) space stream-K style into one contiguous range per CTA, and
numbers the pieces of (pair, head)s cut by a range boundary.  These properties
are what the kernel and its combine pass rely on.  The CTA-pair kernel's plan
(span 512) has the same structure over 512-row quads and 2-CTA clusters.
"""
from collections import defaultdict

from hypothesis import given, settings, strategies as st

from paper_2401_11181_b200 import native

KEYS = 128


def _slices(draw_lens, draw_starts):
    out, off = [], 0
    for n, s in zip(draw_lens, draw_starts):
        pages = (s + n + 15) // 16
        out.append((s, n, off, pages, 1))
        off += pages
    return out


def check_plan(slices, heads, max_ctas, span=256):
    pairs, units, off, n_pieces = native.fa_plan(slices, heads, max_ctas, span)
    # records tile every slice's rows in order, `span` rows at a time
    row = 0
    by_slice = defaultdict(list)
    for i, (sl, row0, pos0, n0, n1, nblk) in enumerate(pairs):
        by_slice[sl].append((row0, pos0, n0, n1, nblk))
    for i, (start, n, *_rest) in enumerate(slices):
        got = by_slice[i]
        assert sum(a[2] + a[3] for a in got) == n
        for k, (row0, pos0, n0, n1, nblk) in enumerate(got):
            assert row0 == row + span * k and pos0 == start + span * k
            if span == 256:
                assert 1 <= n0 <= 128 and 0 <= n1 <= 128 and (n1 == 0 or n0 == 128)
            else:  # a quad: all its rows in nrows0, full unless the slice's last
                assert n1 == 0 and 1 <= n0 <= 512 and (n0 == 512 or k == len(got) - 1)
            kv_end = pos0 + (128 + n1 if n1 else n0)
            assert nblk == (kv_end + KEYS - 1) // KEYS
        row += n
    # units: every (pair, head) covered by contiguous, disjoint key ranges
    assert off[0] == 0 and off[-1] == len(units) and off == sorted(off)
    assert len(off) - 1 <= max_ctas
    cover = defaultdict(list)
    for pair, head, kb0, kb1, piece in units:
        assert 0 <= head < heads and kb0 < kb1
        cover[(pair, head)].append((kb0, kb1, piece))
    assert len(cover) == len(pairs) * heads
    pieces = []
    for (pair, head), rs in cover.items():
        rs.sort()
        assert rs[0][0] == 0 and rs[-1][1] == pairs[pair][5]
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        if len(rs) == 1:
            assert rs[0][2] == -1
        else:
            ids = [r[2] for r in rs]
            assert all(p >= 0 for p in ids) and ids == list(range(ids[0], ids[0] + len(ids)))
            pieces += ids
    assert sorted(pieces) == list(range(n_pieces))
    # the partial buffer holds 2 * 148 pieces of two 128-row tiles (quads: four)
    assert n_pieces <= (2 * 148 if span == 256 else 148)
    per_cta = [sum(u[3] - u[2] for u in units[off[c]:off[c + 1]]) for c in range(len(off) - 1)]
    whole = n_pieces == 0 and len(off) - 1 == len(units) == len(pairs) * heads
    total = sum(per_cta)
    if whole and len(per_cta) > 1:
        # whole-unit plan (short prefixes): one (head, pair) per CTA, chosen only when the
        # longest unit is within 3 key blocks of the stream-K share (attention_tc.cu)
        g = min(max_ctas, max(1, total // 2))
        assert max(per_cta) <= -(-total // g) + 3
    else:
        # stream-K balance: CTA block totals differ by at most one
        assert max(per_cta) - min(per_cta) <= 1


def test_plan_c2_chunks():
    for prefix in (0, 512, 2048, 7680):
        check_plan([(prefix, 512, 0, (prefix + 512 + 15) // 16, 1)], 40, 148)


def test_plan_mixed_slices_and_tiny_chunks():
    check_plan(_slices([118, 18, 100, 276], [394, 0, 0, 0]), 40, 148)
    check_plan(_slices([1], [0]), 1, 148)
    check_plan(_slices([300], [256]), 3, 7)


@settings(max_examples=60, deadline=None)
@given(st.lists(st.tuples(st.integers(1, 600), st.integers(0, 8000)), min_size=1, max_size=6),
       st.integers(1, 40), st.sampled_from([1, 7, 74, 148]))
def test_plan_properties(sl, heads, max_ctas):
    check_plan(_slices([a for a, _ in sl], [b for _, b in sl]), heads, max_ctas)


def test_quad_plan_c2_chunks_and_mixed():
    """CTA-pair kernel plans (TK_FA_PAIR=1): 512-row quads over 74 clusters."""
    for prefix in (0, 512, 2048, 7680):
        check_plan([(prefix, 512, 0, (prefix + 512 + 15) // 16, 1)], 40, 74, 512)
    check_plan(_slices([118, 18, 100, 276], [394, 0, 0, 0]), 4, 74, 512)
    check_plan(_slices([700], [3000]), 5, 74, 512)
    check_plan(_slices([1], [0]), 1, 74, 512)


@settings(max_examples=40, deadline=None)
@given(st.lists(st.tuples(st.integers(1, 1200), st.integers(0, 8000)), min_size=1, max_size=5),
       st.integers(1, 40), st.sampled_from([1, 7, 37, 74]))
def test_quad_plan_properties(sl, heads, max_ctas):
    check_plan(_slices([a for a, _ in sl], [b for _, b in sl]), heads, max_ctas, 512)
