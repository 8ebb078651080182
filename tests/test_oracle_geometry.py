"""Pins for oracle/geometry.py (O1/O2) — against numbers the paper prints and exhaustive checks."""
from fractions import Fraction

import pytest

from oracle.geometry import INFINITY_1K_SIDES, Schedule, kv_blocks, query_blocks, rne


def test_paper_sums():
    s = Schedule(INFINITY_1K_SIDES)
    assert s.C(3) == 21            # PAPER.md:860  "C_3 = 1x1 + 2x2 + 4x4 = 21"
    assert s.C(5) == 121           # PAPER.md:971  "the first 5 scales contain just 121 KV tokens"
    assert s.N(13) == 4096         # PAPER.md:413  q_len = 4096
    assert s.C(13) == 10521        # PAPER.md:413  kv_len = 10521
    assert s.C(12) == 6425 and s.C(11) == 4121


def test_decompose_examples():
    s = Schedule(INFINITY_1K_SIDES)
    assert s.decompose(0) == (1, 0)
    assert s.decompose(21) == (4, 0)          # first token of scale 4
    assert s.decompose(10520) == (13, 4095)
    assert s.decompose(120) == (5, 63)


def test_decompose_roundtrip_exhaustive():
    s = Schedule(INFINITY_1K_SIDES)
    j = 0
    for l in range(1, s.K + 1):
        for d in range(s.N(l)):
            assert s.decompose(j) == (l, d)
            assert s.recompose(l, d) == j
            j += 1
    assert j == s.C(13)


def test_rne_is_bankers_rounding():
    for den in range(1, 70):
        for num in range(-200, 200):
            f = Fraction(num, den)
            r = rne(num, den)
            assert abs(f - r) <= Fraction(1, 2)
            if abs(f - r) == Fraction(1, 2):
                assert r % 2 == 0
    assert rne(1, 2) == 0 and rne(3, 2) == 2 and rne(5, 2) == 2 and rne(-1, 2) == 0


def test_schedule_validation():
    with pytest.raises(ValueError):
        Schedule([])
    with pytest.raises(ValueError):
        Schedule([2, 1])
    with pytest.raises(ValueError):
        Schedule([0, 1])


def test_blocks_ragged():
    qb = query_blocks(1600, 128)
    assert len(qb) == 13 and len(qb[-1]) == 64
    kb = kv_blocks(10521, 128)
    assert len(kb) == 83 and len(kb[-1]) == 25
    assert kb[50].start == 6400 and 6425 in kb[50]   # blocks straddle scale boundaries
