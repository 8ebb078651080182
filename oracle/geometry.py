"""O1/O2 — scale-schedule geometry.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Definitions followed
  N_k = h_k w_k (square grids, h_k = w_k = s_k), N_{<=k} = sum_{i<=k} N_i
        PAPER.md:200-201 (§3.1 Background).
  C_i cumulative token counts, e.g. C_3 = 1x1 + 2x2 + 4x4 = 21
        PAPER.md:860 (App. "Relative Scale Alignment", Decomposition bullet).
  Decomposition of a global KV index j into (scale l, offset delta)
        PAPER.md:861-863.  READING 2: the printed `l = max{i | C_i <= j},
        delta = j - C_l` is off by one; we use the half-open C_{l-1} <= j < C_l.
  De-linearisation of delta into 2-D (u, v), row-major     PAPER.md:876.
  Blocks of size B along query and key axes, u in 0..ceil(N_k/B)-1, v in 0..ceil(N_{<=k}/B)-1
        PAPER.md:398 (§3.3 "Block-wise Sparse Mask").  KV blocks start at 0 and straddle scale
        boundaries (FlexAttention convention).
  Infinity-1K side list 1,2,4,6,8,12,16,20,24,32,40,48,64: never printed by the paper; it is the
        list that satisfies q_len = 4096, kv_len = 10521 and "the first 5 scales
        contain just 121 KV tokens".  Pinned by those three sums in the tests.

Pins: C_3 = 21, C_5 = 121, C_13 = 10521 and N_13 = 4096
(PAPER.md:413); decompose/recompose round trip (exhaustive); rne() against Python's
round(Fraction) (banker's rounding of the exact rational).
"""
from __future__ import annotations

from fractions import Fraction
from typing import List, Sequence, Tuple

INFINITY_1K_SIDES: Tuple[int, ...] = (1, 2, 4, 6, 8, 12, 16, 20, 24, 32, 40, 48, 64)


class Schedule:
    """Scale schedule.  Scales are 1-based as in the paper (READING 1)."""

    def __init__(self, sides: Sequence[int]):
        sides = [int(s) for s in sides]
        if not sides:
            raise ValueError("empty schedule")
        if any(s < 1 for s in sides):
            raise ValueError("sides must be >= 1")
        if any(b < a for a, b in zip(sides, sides[1:])):
            raise ValueError("sides must be non-decreasing")
        self.sides: List[int] = sides
        self.K = len(sides)

    def s(self, k: int) -> int:
        """Side s_k of scale k (1-based)."""
        return self.sides[k - 1]

    def N(self, k: int) -> int:
        """N_k = s_k^2 tokens of scale k."""
        return self.sides[k - 1] ** 2

    def C(self, k: int) -> int:
        """C_k = sum_{i<=k} N_i, with C_0 = 0."""
        return sum(self.N(i) for i in range(1, k + 1))

    def decompose(self, j: int) -> Tuple[int, int]:
        """Global KV index j -> (l, delta) with C_{l-1} <= j < C_l, delta = j - C_{l-1}."""
        if j < 0 or j >= self.C(self.K):
            raise ValueError("index out of range")
        for l in range(1, self.K + 1):
            if self.C(l - 1) <= j < self.C(l):
                return l, j - self.C(l - 1)
        raise AssertionError("unreachable")

    def recompose(self, l: int, delta: int) -> int:
        return self.C(l - 1) + delta


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


def rne(num: int, den: int) -> int:
    """Round-half-to-even of the exact rational num/den (READING 3: torch.round semantics)."""
    return round(Fraction(num, den))


def query_blocks(n_q: int, B: int) -> List[range]:
    """Query block u covers tokens [uB, min((u+1)B, N_k))."""
    return [range(u * B, min((u + 1) * B, n_q)) for u in range(ceil_div(n_q, B))]


def kv_blocks(n_kv: int, B: int) -> List[range]:
    """KV block v covers flat cache indices [vB, min((v+1)B, C_k))."""
    return [range(v * B, min((v + 1) * B, n_kv)) for v in range(ceil_div(n_kv, B))]
