"""NEXT(4) — KV-cache compression for CSLA layers: keep only the sink scales and the scales the
local windows read.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Definitions followed
  "+ KV Comp.": "retaining only sinks and local scales KV Cache"           PAPER.md:1170 (Tab.
        efficiency_memory)
  A CSLA layer at target K attends only M^(K) (oracle/csla.token_mask): keys
  of the sink scales h <= sink_scales and of the scales h with window w_h > 0.  Every other
  scale's keys are masked for every query, so the cache of such a layer need not hold them.
  READING 23: the compressed cache is the kept scales' rows in scale order (their row-major
  layouts unchanged); the CSLA block mask of the compressed layer is Eq. block_mask
   applied to the token mask restricted to the kept columns, re-blocked at B
  over the compressed index (blocks straddle the kept scales just as they straddle scales in
  the full cache, READING 9).

Pins (tests/test_oracle_kv_compress.py): nothing dropped => the full cache and the full CSLA
mask; at B = 1 attention over the compressed cache with the compressed mask equals the full
token-masked attention (dropped columns are never attended); the kept row count of Infinity-1K
K = 13 with the default windows is C_5 + (C_13 - C_8) = 9721.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np

from .csla import block_mask_from_token_mask, token_mask, window_of_scale
from .geometry import Schedule


def kept_scales(K: int, sink_scales: int, windows: Sequence[int]) -> List[int]:
    """Scales 1..K a CSLA layer at K reads: the sink scales and those with a window."""
    return [h for h in range(1, K + 1) if h <= sink_scales or window_of_scale(K, h, windows) > 0]


def kept_ranges(sched: Schedule, K: int, sink_scales: int,
                windows: Sequence[int]) -> List[Tuple[int, int]]:
    """[C_{h-1}, C_h) row ranges of the full cache that the compressed cache keeps, merged."""
    out: List[Tuple[int, int]] = []
    for h in kept_scales(K, sink_scales, windows):
        lo, hi = sched.C(h - 1), sched.C(h)
        if out and out[-1][1] == lo:
            out[-1] = (out[-1][0], hi)
        else:
            out.append((lo, hi))
    return out


def kept_index(sched: Schedule, K: int, sink_scales: int, windows: Sequence[int]) -> np.ndarray:
    """Full-cache row of every compressed-cache row, in order."""
    return np.concatenate([np.arange(lo, hi) for lo, hi in kept_ranges(sched, K, sink_scales, windows)])


def compress(cache: np.ndarray, sched: Schedule, K: int, sink_scales: int,
             windows: Sequence[int]) -> np.ndarray:
    """The compressed cache of one (b, h): rows of the kept scales, in order."""
    return np.asarray(cache)[kept_index(sched, K, sink_scales, windows)]


def compressed_local_block_mask(sched: Schedule, K: int, B: int, sink_scales: int,
                                windows: Sequence[int]) -> np.ndarray:
    """CSLA block mask over the compressed index (READING 23)."""
    M = token_mask(sched, K, sink_scales, windows)
    return block_mask_from_token_mask(M[:, kept_index(sched, K, sink_scales, windows)], B)
