"""Pins for oracle/csla.py (O3) — the paper's own sparsity tables, SPEC.md worked examples,
structural properties and a brute-force block aggregation."""
import os

import numpy as np
import pytest

from oracle.csla import (aligned_coord, block_mask_from_token_mask, flex_sparsity, local_block_mask,
                         retile, token_mask)
from oracle.geometry import INFINITY_1K_SIDES, Schedule

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "csla_sparsity.txt")
SCHED = Schedule(INFINITY_1K_SIDES)
NQ, NKV = 4096, 10521


def _golden_rows():
    rows = []
    for line in open(GOLDEN):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        sink, w, block, pct, *src = line.split()
        w11, w12, w13 = (int(x) for x in w.split(","))
        rows.append((int(sink), (w13, w12, w11, 1, 1), block, float(pct), " ".join(src)))
    return rows


@pytest.fixture(scope="module")
def masks():
    cache = {}

    def get(sink, windows):
        key = (sink, tuple(windows))
        if key not in cache:
            cache[key] = local_block_mask(SCHED, 13, 128, sink, windows)
        return cache[key]
    return get


@pytest.mark.parametrize("row", _golden_rows(), ids=lambda r: r[4])
def test_paper_sparsity(row, masks):
    """Every printed sparsity is an integer active-block count under the FlexAttention
    convention (READING 6); the oracle must hit that count exactly."""
    sink, windows, block, pct, _ = row
    bm = masks(sink, windows)
    if block == "64r":
        bm, B = retile(bm, 128, 64, NQ, NKV), 64
    else:
        B = int(block)
    implied = (1 - pct / 100) * NQ * NKV / (B * B)
    A = int(round(implied))
    assert abs(implied - A) < 0.5 * NQ * NKV / (B * B) * 1e-4 + 1e-9   # the 2-decimal rounding
    assert int(bm.sum()) == A
    assert round(flex_sparsity(int(bm.sum()), NQ, NKV, B), 2) == pct


def test_table_orderings(masks):
    """Table csla_ablation orderings."""
    sp = lambda s, w: flex_sparsity(int(masks(s, w).sum()), NQ, NKV, 128)
    W = lambda a, b, c: (c, b, a, 1, 1)
    assert sp(5, W(1, 3, 5)) > sp(5, W(3, 5, 7)) > sp(5, W(5, 7, 9)) > sp(5, W(7, 9, 11))
    assert sp(5, W(3, 5, 7)) > sp(6, W(3, 5, 7)) > sp(7, W(3, 5, 7)) > sp(8, W(3, 5, 7))


def test_default_rows_shape(masks):
    bm = masks(5, (7, 5, 3, 1, 1))
    per_row = bm.sum(1)
    assert per_row.min() == 10 and per_row.max() == 15
    assert bm.any(0).sum() == 77
    assert bm[:, 0].all()                                    # sink block in every row


def test_true_b64_is_sparser(masks):
    """Block-size monotonicity: coarser blocks only merge active regions."""
    b64 = local_block_mask(SCHED, 13, 64)
    s64 = flex_sparsity(int(b64.sum()), NQ, NKV, 64)
    s128 = flex_sparsity(int(masks(5, (7, 5, 3, 1, 1)).sum()), NQ, NKV, 128)
    assert s64 >= s128
    assert (retile(b64, 64, 128, NQ, NKV) == masks(5, (7, 5, 3, 1, 1))).all()


def test_corner_window_clip():
    """Query (0,0) at K=13 with window 7 on scale 13: the 4x4 corner clip = 16 keys."""
    M = token_mask(SCHED, 13, 0, (7,))
    assert M[0].sum() == 16
    assert set(np.nonzero(M[0])[0] - SCHED.C(12)) == {x * 64 + y for x in range(4) for y in range(4)}


def test_window_one_single_key():
    """Window 1 on a scale -> exactly the single aligned key."""
    M = token_mask(SCHED, 13, 0, (0, 0, 0, 1))        # only scale 10 (side 32), window 1
    assert (M.sum(1) == 1).all()
    # query (63, 63) of 64x64 aligns to round(63*32/64)=round(31.5)=32 -> clamped to 31
    j = np.nonzero(M[4095])[0][0] - SCHED.C(9)
    assert j == 31 * 32 + 31


def test_alignment_rounding_examples():
    assert aligned_coord(63, 64, 48) == 47        # round(47.25)
    assert aligned_coord(1, 64, 32) == 0          # round(0.5) = 0, half-to-even (READING 3)
    assert aligned_coord(3, 64, 32) == 2          # round(1.5) = 2
    assert aligned_coord(63, 64, 1) == 0          # round(63/64) = 1 -> clamp (READING 4)
    for s in (1, 2, 4, 6, 8, 12, 16, 20, 24, 32, 40, 48, 64):
        assert [aligned_coord(x, s, s) for x in range(s)] == list(range(s))   # same grid: id


def test_block_one_is_token_mask():
    sched = Schedule([1, 2, 4, 8])
    M = token_mask(sched, 4, 2, (3, 3))
    assert (block_mask_from_token_mask(M, 1) == M).all()


def test_all_active():
    M = np.ones((64, 85), dtype=bool)
    assert block_mask_from_token_mask(M, 16).all()


def test_block_aggregation_bruteforce():
    rng = np.random.default_rng(0)
    M = rng.random((37, 53)) < 0.02
    for B in (1, 3, 8, 16):
        bm = block_mask_from_token_mask(M, B)
        for u in range(bm.shape[0]):
            for v in range(bm.shape[1]):
                want = any(M[q, k] for q in range(u * B, min((u + 1) * B, 37))
                           for k in range(v * B, min((v + 1) * B, 53)))
                assert bm[u, v] == want


def test_sink_prefix():
    M = token_mask(SCHED, 13, 5, (7, 5, 3, 1, 1))
    assert M[:, :121].all()                           # PAPER.md:971 "just 121 KV tokens"
    assert not M[:, 121:SCHED.C(8)].any()             # scales 6..8 masked (READING 5)
