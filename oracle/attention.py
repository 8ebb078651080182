"""O6-O8 — merge to block lists, block-sparse and dense cross-scale attention.
TEST INFRASTRUCTURE ONLY.

Definitions followed
  O_k = Softmax(Q_k K_{<=k}^T / sqrt(d)) V_{<=k}         PAPER.md:204-212 (Eq. attn_cross_scale)
  Delta O^(k) = Softmax(Q^(k) K_inds^T) V_inds  -- a fresh softmax renormalised over the listed
        keys only                                         PAPER.md:318-328 (Eq. sparse_update)
        READING 17: the 1/sqrt(d) printed in Eq. 1 is applied here too.
  Block-sparse form (CSLA): query block u attends every real token of every
        listed KV block ("every active block represents a dense local window", READING 9);
        tokens >= C_K are never attended (READING 20).
  Merge (O6, READING 19): the list of row u is the ascending set bits of the OR of the block
        masks in use.

Pins (tests/test_oracle_attention.py): dense() against an independent per-element triple loop
(<= 1e-12); block_sparse() with every block listed equals dense() (<= 1e-12,
SPEC.md:158); a sink-only list equals attention truncated to the sink prefix;
a single key returns its value row; equal logits return the mean value row; outputs are convex
combinations of value rows; invariance to a per-row logit shift.
"""
from __future__ import annotations

import math
from typing import List, Optional, Sequence

import numpy as np

from .geometry import ceil_div


def softmax_rows(z: np.ndarray) -> np.ndarray:
    z = z - z.max(axis=1, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=1, keepdims=True)


def dense(q: np.ndarray, k: np.ndarray, v: np.ndarray, n_kv: int,
          scale: Optional[float] = None) -> np.ndarray:
    """O8: Eq. attn_cross_scale for one (b, h).  q (N_k, D); k, v (>= n_kv, D).  fp64."""
    q, k, v = (np.asarray(a, dtype=np.float64) for a in (q, k, v))
    if scale is None:
        scale = 1.0 / math.sqrt(q.shape[1])
    return softmax_rows((q @ k[:n_kv].T) * scale) @ v[:n_kv]


def merge_lists(masks: Sequence[np.ndarray]) -> List[np.ndarray]:
    """O6: per row, ascending active block indices of the OR of the masks."""
    m = np.zeros_like(masks[0], dtype=bool)
    for x in masks:
        m |= x
    return [np.nonzero(row)[0] for row in m]


def to_csr(lists: Sequence[np.ndarray]):
    row_ptr = np.zeros(len(lists) + 1, dtype=np.int64)
    for i, l in enumerate(lists):
        row_ptr[i + 1] = row_ptr[i] + len(l)
    col = np.concatenate([np.asarray(l, dtype=np.int64) for l in lists]) if lists else np.zeros(0)
    return row_ptr, col


def block_sparse(q: np.ndarray, k: np.ndarray, v: np.ndarray, n_kv: int, B: int,
                 lists: Sequence[Sequence[int]], scale: Optional[float] = None,
                 rows: Optional[Sequence[int]] = None) -> np.ndarray:
    """O7 for one (b, h): query block u attends the real tokens of its listed KV blocks.
    `rows` optionally restricts the computation to a subset of query blocks (others are NaN)."""
    q, k, v = (np.asarray(a, dtype=np.float64) for a in (q, k, v))
    n_q, D = q.shape
    if scale is None:
        scale = 1.0 / math.sqrt(D)
    out = np.full((n_q, v.shape[1]), np.nan)
    for u in (range(ceil_div(n_q, B)) if rows is None else rows):
        if len(lists[u]) == 0:
            raise ValueError(f"query block {u} has no active KV block")
        J = np.concatenate([np.arange(b * B, min((b + 1) * B, n_kv)) for b in sorted(lists[u])])
        qu = q[u * B: min((u + 1) * B, n_q)]
        out[u * B: u * B + len(qu)] = softmax_rows((qu @ k[J].T) * scale) @ v[J]
    return out


def brute_force(q, k, v, n_kv, allowed=None, scale=None) -> np.ndarray:
    """Per-element triple loop over (t, j, d); `allowed(t, j)` restricts the keys.  Tiny only."""
    q, k, v = (np.asarray(a, dtype=np.float64) for a in (q, k, v))
    n_q, D = q.shape
    if scale is None:
        scale = 1.0 / math.sqrt(D)
    out = np.zeros((n_q, v.shape[1]))
    for t in range(n_q):
        js = [j for j in range(n_kv) if allowed is None or allowed(t, j)]
        z = [sum(q[t, d] * k[j, d] for d in range(D)) * scale for j in js]
        m = max(z)
        w = [math.exp(x - m) for x in z]
        s = sum(w)
        for d in range(v.shape[1]):
            out[t, d] = sum(w[i] * v[j, d] for i, j in enumerate(js)) / s
    return out
