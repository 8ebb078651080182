"""O3 — Cross-Scale Local Sparse Attention (CSLA) masks.  TEST INFRASTRUCTURE ONLY.

Definitions followed (§3.3 "Cross-Scale Local Sparse Attention")
  aligned coordinates  (x~, y~) = (round(x/H_k * H_h), round(y/W_k * W_h))
      READING 3: round = round-half-to-even of the exact rational x*s_h/s_k, corner aligned.
      READING 4: clamp to s_h - 1 (round can reach s_h, e.g. s_h = 1, x = 63 of 64).
  local mask  M_local^(k,h)(q,k) = 1(|x~ - x_k| <= r_h and |y~ - y_k| <= r_h)
      r_h = floor(w_h / 2)
      windows clip at the grid edge (no wrap): the indicator is a pure coordinate bound.
  sink mask   M_sink(q,k) = 1[k in S], S = tokens of scales <= sink_scales
  union       M^(k) = M_sink OR (OR over historical scales h of M_local^(k,h))
      READING 1: 1-based scales, union over h = 1..k.
      READING 5: window vector is relative to the target scale: windows[i] applies to scale
      k - i; scales not covered by the vector (and not sink) are masked.  The paper default
      "[3, 5, 7] for the last 3 scales" with scales 10 and 9 at window 1 and
      scales 6..8 masked is the (7,5,3,1,1) vector -- the unique reading that reproduces all
      11 sparsities of Table csla_ablation.
  block mask  B^(k)(u,v) = OR_{q in B_u} OR_{k in B_v} M^(k)(q,k)
      (Eq. block_mask), over the real tokens of the ragged last blocks.
  sparsity    FlexAttention BlockMask.sparsity(): 100 * (1 - A * B * B / (N_q * N_kv))
      READING 6: ragged blocks count as full.

Pins (tests/test_oracle_csla.py): the 11 sparsities of Table csla_ablation and the 83.46% /
83.50% rows of Table kernel_speed (tests/golden/csla_sparsity.txt),
the 16-key clipped corner window, window 1 -> a single key, B = 1
returns the token mask, all-active token mask -> all-active block mask, orderings of Table
csla_ablation, and block_mask_from_token_mask against a brute-force per-pair OR.
"""
from __future__ import annotations

from typing import Sequence

import numpy as np

from .geometry import Schedule, ceil_div, rne

DEFAULT_WINDOWS = (7, 5, 3, 1, 1)   # relative to the target scale: K, K-1, K-2, K-3, K-4
DEFAULT_SINK_SCALES = 5


def aligned_coord(x: int, s_k: int, s_h: int) -> int:
    """x~ = min(round(x * s_h / s_k), s_h - 1)   (READINGS 3-4)."""
    return min(rne(x * s_h, s_k), s_h - 1)


def window_of_scale(K: int, h: int, windows: Sequence[int]) -> int:
    """w_h for historical scale h of target K (READING 5).  0 = masked."""
    i = K - h
    return int(windows[i]) if 0 <= i < len(windows) else 0


def token_mask(sched: Schedule, K: int, sink_scales: int, windows: Sequence[int]) -> np.ndarray:
    """M^(K)(q, j) as a bool array of shape (N_K, C_K)."""
    s_K = sched.s(K)
    n_q, n_kv = sched.N(K), sched.C(K)
    M = np.zeros((n_q, n_kv), dtype=bool)
    qx = np.arange(n_q) // s_K          # query (x, y) = divmod(t, s_K), row-major
    qy = np.arange(n_q) % s_K
    # sink mask: every key of the scales <= sink_scales
    M[:, : sched.C(min(sink_scales, K))] = True
    for h in range(1, K + 1):
        w = window_of_scale(K, h, windows)
        if w <= 0:
            continue
        r = w // 2
        s_h = sched.s(h)
        table = np.array([aligned_coord(x, s_K, s_h) for x in range(s_K)])
        xt, yt = table[qx], table[qy]                              # (x~, y~) per query
        kx = np.arange(s_h * s_h) // s_h
        ky = np.arange(s_h * s_h) % s_h
        local = (np.abs(xt[:, None] - kx[None, :]) <= r) & (np.abs(yt[:, None] - ky[None, :]) <= r)
        M[:, sched.C(h - 1): sched.C(h)] |= local                  # OR over scales
    return M


def block_mask_from_token_mask(M: np.ndarray, B: int) -> np.ndarray:
    """Eq. block_mask: B(u, v) = OR of M over the real tokens of tile (u, v)."""
    n_q, n_kv = M.shape
    gq, gkv = ceil_div(n_q, B), ceil_div(n_kv, B)
    P = np.zeros((gq * B, gkv * B), dtype=bool)     # padding tokens are not real -> False
    P[:n_q, :n_kv] = M
    return P.reshape(gq, B, gkv, B).any(axis=(1, 3))


def local_block_mask(sched: Schedule, K: int, B: int, sink_scales: int = DEFAULT_SINK_SCALES,
                     windows: Sequence[int] = DEFAULT_WINDOWS) -> np.ndarray:
    """The CSLA block mask B^(K) (G_q x G_kv bool), identical for every (batch, head)."""
    return block_mask_from_token_mask(token_mask(sched, K, sink_scales, windows), B)


def flex_sparsity(active_blocks: int, n_q: int, n_kv: int, B: int) -> float:
    """FlexAttention BlockMask.sparsity() in percent (READING 6)."""
    return 100.0 * (1.0 - active_blocks * B * B / (n_q * n_kv))


def retile(block_mask: np.ndarray, B: int, B2: int, n_q: int, n_kv: int) -> np.ndarray:
    """Expand a B-granular block mask to tokens and re-aggregate at B2 (READING 7: the paper's
    'block size 64' row is the B=128 mask re-tiled at 64)."""
    tok = np.repeat(np.repeat(block_mask, B, axis=0), B, axis=1)[:n_q, :n_kv]
    return block_mask_from_token_mask(tok, B2)
