"""O5 — cross-scale sparse index mapping M_{S->K}.  TEST INFRASTRUCTURE ONLY.

Definitions followed (PAPER.md App. "Cross-Scale Sparse Index Mapping")
  Query Block Homography  phi(g_K) = round((g_K + 0.5) / G_K * G_S - 0.5) clipped to [0, G_S-1]
        PAPER.md:841-851.  READING 15: round-half-to-even of the exact rational, then clamp;
        G = ceil(N / B) query blocks, G_{K-1} read as G_K - 1.
  Decompose  (l, delta_S) of global index j
        (READING 2: half-open C_{l-1} <= j < C_l)
  Relative Alignment  l' = K - (S - l)
  Spatial Projection  u' = floor(u * h_l' / h_l), v' = floor(v * w_l' / w_l),
        delta_K = u' * w_l' + v', j' = C_{l'} + delta_K
        (C_{l'} there is the offset of scale l', i.e. C_{l'-1} in the half-open convention.)
        READING 14: the literal point map (mode "point") lands a source token on one target
        token, which does not cover the up-sampled region (it can leave gaps between the points
        when h_l' > h_l).  The default mode "footprint" maps source row u to the forward interval
        [floor(u h_l'/h_l), floor((u+1) h_l'/h_l) - 1] (and likewise columns): it contains the
        point, tiles scale l' exactly, and is the identity when S = K.
  Sink union  inds^(K) = A_sink U M_{S->K}(inds^(S))
  READING 10: patterns are block patterns: every real token j < C_S of an active source KV block
        is mapped, and a target KV block is active iff it holds a mapped target token.

Pins (tests/test_oracle_mapping.py): S = K is the identity in both modes; point <= footprint;
footprint equals the pre-image of the active source tokens under the closed-form down-sampling
x = ceil((x'+1) s_l / s_l') - 1 (independent characterisation of "nests under the up-sampling");
the phi tables for G 13 -> 32 and 8 -> 13 worked by hand from PAPER.md:848 (SURVEY.md §8c,
tests/golden/phi_tables.txt); SPEC.md:268-270 (j = 21 -> 121 for S = 11, K = 13) and
SPEC.md:86 ((1,1) of 2x2 -> offset 21 of 6x6); the sink is a subset of every row.
"""
from __future__ import annotations

from fractions import Fraction
from typing import Tuple

import numpy as np

from .geometry import Schedule, ceil_div


def phi(g_K: int, G_S: int, G_K: int) -> int:
    """Query Block Homography (READING 15)."""
    x = Fraction(2 * g_K + 1, 2 * G_K) * G_S - Fraction(1, 2)
    return min(max(round(x), 0), G_S - 1)


def map_token(sched: Schedule, j: int, S: int, K: int, mode: str) -> Tuple[int, range, range]:
    """Decompose-Align-Project of global index j < C_S.  Returns (l', rows, cols) of scale l'."""
    l, delta = sched.decompose(j)                       # Decomposition
    lp = K - (S - l)                                    # Relative Alignment
    s_l, s_lp = sched.s(l), sched.s(lp)
    u, v = divmod(delta, s_l)                           # de-linearise
    if mode == "point":                                 # PAPER.md:878 literally
        up, vp = (u * s_lp) // s_l, (v * s_lp) // s_l
        return lp, range(up, up + 1), range(vp, vp + 1)
    if mode == "footprint":                             # READING 14
        return (lp, range((u * s_lp) // s_l, ((u + 1) * s_lp) // s_l),
                range((v * s_lp) // s_l, ((v + 1) * s_lp) // s_l))
    raise ValueError(mode)


def map_pattern(src: np.ndarray, sched: Schedule, S: int, K: int, B: int, sink_scales: int,
                mode: str = "footprint") -> np.ndarray:
    """Map a source block pattern (G_S x G_kvS bool) at decision scale S to target K."""
    n_qS, n_kvS = sched.N(S), sched.C(S)
    G_S, G_K = ceil_div(n_qS, B), ceil_div(sched.N(K), B)
    G_kvK = ceil_div(sched.C(K), B)
    assert src.shape == (G_S, ceil_div(n_kvS, B))
    dst = np.zeros((G_K, G_kvK), dtype=bool)
    nsb = ceil_div(sched.C(sink_scales), B) if sink_scales > 0 else 0
    for g in range(G_K):
        gs = phi(g, G_S, G_K)
        for v in np.nonzero(src[gs])[0]:
            for j in range(v * B, min((v + 1) * B, n_kvS)):
                lp, rows, cols = map_token(sched, j, S, K, mode)
                base = sched.C(lp - 1)
                for xp in rows:
                    for yp in cols:
                        dst[g, (base + xp * sched.s(lp) + yp) // B] = True
        dst[g, :min(nsb, G_kvK)] = True                 # sink union
    return dst
