"""NEXT(1) — the CS4A dense-attention cache residual and its cross-scale reuse.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Definitions followed
  O^(S)_cache = O^(S)_dense - Softmax(Q^(S) K_inds^T) V_inds
        "we define the dense attention cache by subtracting the sparse component"; the sparse
        term is the block-sparse attention over the decision-scale pattern (READINGS 10, 17).
  O^(k) ~= O^(k)_cache + Delta O^(k),  Delta O^(k) = Softmax(Q^(k) K_inds(k)^T) V_inds(k)
        PAPER.md:318-334; "O^(k)_cache denotes the upsampled cache prediction from scale S".
  Upsampling (READING 22): nearest neighbour over the 2-D query grid, target query (x, y) of
        side s_k copies the cache row of source query (floor(x s_S / s_k), floor(y s_S / s_k))
        (the paper names no interpolation).

Pins (tests/test_oracle_cache.py): the reconstruction identity o_cache + sparse = dense
(<= 1e-12, by the definition's linearity); every block listed => o_cache = 0
(SPEC.md:238, 297); upsample of a constant is that constant, upsample with s_S = s_k is the
identity, and a brute-force pixel-replication of a small grid (np.repeat for integer ratios);
the cached output minus the sparse output equals the upsampled cache exactly.
"""
from __future__ import annotations

import numpy as np

from .attention import block_sparse, dense


def cache_residual(q_S, k, v, n_kv_S: int, B: int, lists_S) -> np.ndarray:
    """O^(S)_cache for one (b, h): q_S (N_S, D); k, v (>= n_kv_S, D); lists_S per query block."""
    return dense(q_S, k, v, n_kv_S) - block_sparse(q_S, k, v, n_kv_S, B, lists_S)


def upsample_nn(o_cache: np.ndarray, s_S: int, s_k: int) -> np.ndarray:
    """(s_S*s_S, D) -> (s_k*s_k, D), nearest neighbour over the query grid (READING 22)."""
    o_cache = np.asarray(o_cache)
    out = np.empty((s_k * s_k, o_cache.shape[1]), dtype=o_cache.dtype)
    for x in range(s_k):
        for y in range(s_k):
            xs = (x * s_S) // s_k
            ys = (y * s_S) // s_k
            out[x * s_k + y] = o_cache[xs * s_S + ys]
    return out


def cached_sparse(q_k, k, v, n_kv_k: int, B: int, lists_k, o_cache_S: np.ndarray, s_S: int,
                  s_k: int) -> np.ndarray:
    """O^(k) ~= upsample(O^(S)_cache) + Delta O^(k) for one (b, h)."""
    return block_sparse(q_k, k, v, n_kv_k, B, lists_k) + upsample_nn(o_cache_S, s_S, s_k)
