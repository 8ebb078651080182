"""Pins for oracle/mapping.py (O5)."""
import os

import numpy as np
import pytest

from oracle.geometry import INFINITY_1K_SIDES, Schedule, ceil_div
from oracle.mapping import map_pattern, map_token, phi

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "phi_tables.txt")
INF = Schedule(INFINITY_1K_SIDES)


def _phi_rows():
    for line in open(GOLDEN):
        line = line.strip()
        if line and not line.startswith("#"):
            head, tail = line.split(":")
            gs, gk = (int(x) for x in head.split())
            yield gs, gk, [int(x) for x in tail.split()]


@pytest.mark.parametrize("gs,gk,table", list(_phi_rows()))
def test_phi_tables(gs, gk, table):
    assert [phi(g, gs, gk) for g in range(gk)] == table


def test_phi_spec_example():
    assert phi(0, 9, 22) == 0          # round(0.5/22*9 - 0.5) = round(-0.295) = 0


def test_dap_spec_examples():
    lp, rows, cols = map_token(INF, 21, 11, 13, "point")
    assert lp == 6 and INF.C(lp - 1) + rows[0] * INF.s(lp) + cols[0] == 121
    s = Schedule([1, 2, 6])                                  # (1,1) of 2x2 -> 6x6
    lp, rows, cols = map_token(s, 1 + 3, 2, 3, "point")
    assert lp == 3 and rows[0] * 6 + cols[0] == 21
    lp, _, _ = map_token(INF, INF.C(9), 11, 13, "footprint")  # scale 10 -> 12
    assert lp == 12


def _random_src(sched, S, B, density, seed):
    rng = np.random.default_rng(seed)
    return rng.random((ceil_div(sched.N(S), B), ceil_div(sched.C(S), B))) < density


@pytest.mark.parametrize("mode", ["footprint", "point"])
def test_identity_when_S_equals_K(mode):
    sched = Schedule([1, 2, 4, 6, 8, 12, 16])
    for B in (1, 4, 16, 32):
        src = _random_src(sched, 7, B, 0.3, B)
        dst = map_pattern(src, sched, 7, 7, B, 0, mode)
        assert (dst == src).all()


def test_point_within_footprint():
    sched = Schedule([1, 2, 4, 6, 8, 12, 16, 20])
    for B in (4, 16):
        src = _random_src(sched, 6, B, 0.3, 7)
        p = map_pattern(src, sched, 6, 8, B, 0, "point")
        f = map_pattern(src, sched, 6, 8, B, 0, "footprint")
        assert (f | ~p).all()


def test_footprint_is_preimage_of_downsampling():
    """Mapped patterns nest under the up-sampling (north_star): at token level (B = 1) the
    footprint of a source token set T equals { t' : down(t') in T }, where down() is the
    closed-form nearest-lower down-sampling x = ceil((x'+1) s_l / s_l') - 1 per coordinate,
    applied scale by scale with l = l' - (K - S)."""
    sched = Schedule([1, 2, 4, 6, 8, 12, 16, 20])
    S, K = 5, 8
    src = _random_src(sched, S, 1, 0.2, 3)
    dst = map_pattern(src, sched, S, K, 1, 0, "footprint")
    for g in range(dst.shape[0]):
        T = set(np.nonzero(src[phi(g, sched.N(S), sched.N(K))])[0])
        want = set()
        for lp in range(1 + K - S, K + 1):
            l = lp - (K - S)
            s, sp = sched.s(l), sched.s(lp)
            down = lambda xp: -(-(xp + 1) * s // sp) - 1
            for xp in range(sp):
                for yp in range(sp):
                    if sched.C(l - 1) + down(xp) * s + down(yp) in T:
                        want.add(sched.C(lp - 1) + xp * sp + yp)
        assert set(np.nonzero(dst[g])[0]) == want


def test_footprint_tiles_target_scales():
    """Each target token of scales K-S+1..K has exactly one source token (partition)."""
    sched = Schedule(INFINITY_1K_SIDES)
    S, K = 11, 13
    hits = np.zeros(sched.C(K), dtype=int)
    for j in range(sched.C(S)):
        lp, rows, cols = map_token(sched, j, S, K, "footprint")
        for x in rows:
            for y in cols:
                hits[sched.C(lp - 1) + x * sched.s(lp) + y] += 1
    assert (hits[sched.C(K - S):] == 1).all() and (hits[:sched.C(K - S)] == 0).all()


def test_sink_in_every_row():
    sched = Schedule(INFINITY_1K_SIDES)
    B = 128
    src = np.zeros((ceil_div(1600, B), ceil_div(4121, B)), dtype=bool)
    src[:, 20] = True
    dst = map_pattern(src, sched, 11, 13, B, 5, "footprint")
    assert dst[:, 0].all()
    assert dst.shape == (32, 83)
