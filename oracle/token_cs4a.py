"""NEXT(2) — token-granular CS4A, the paper's own CS4A granularity.  TEST INFRASTRUCTURE ONLY
(see oracle/__init__.py): plain fp64 numpy, written from the paper's definitions in their order.

Definitions followed
  P^(S) = Softmax(Q^(S) K^T / sqrt(d)) over the keys j < C_S
  query blocks of C contiguous rows, G_S = ceil(N_S / C) (C = 192)
        (READING 15: the ceiling of PAPER.md:843; the last block is ragged)
  Column-Sum  A^(S)[g, j] = sum_{q in block g} P^(S)[q, j]
  inds^(S)[g] = TopK_j A^(S)[g, :] with k = ceil(alpha C_S) keys
        (READING 11: "Top-K around 0.2" is the fraction alpha of the keys; ties go
        to the smaller j).  The paper adds no sink at S; select_tokens'
        n_sink_tokens > 0 is READING 25's "sink_in_source" option, 0 on the paper-literal path
  M_{S->K}: target query block g_K reads source block phi(g_K)
        (oracle/mapping.phi with C-row blocks); each selected source token is projected by
        Decompose-Align-Project with the forward-interval footprint
        (oracle/mapping.map_token, READING 14); the sink tokens are added
  Delta O^(K) for the rows of block g_K: Softmax(q K_J^T / sqrt(d)) V_J over the tokens J(g_K)
        it selects

  O_cache on the token path: O_cache^(S) = O_dense^(S) - Delta O^(S) over inds^(S), reused at K
        through the nearest-neighbour upsampling of oracle/cache.py

Pins (tests/test_oracle_token_cs4a.py): column sums of every block add up to its row count
(softmax rows sum to 1) and equal a per-element exp-loop brute force on a tiny schedule; top-k
with k >= C_S selects every key and picks a planted dominant key at k = 1; the token map at S = K
is the identity plus the sink, and its block-OR equals the (separately pinned) block mapping of
the block-OR of the source selection when C = B; token-sparse attention with every token equals
dense attention and with the tokens of whole blocks equals the block-sparse oracle; the token
O_cache vanishes when every token is selected and equals the (pinned) block O_cache when whole
blocks are selected.
"""
from __future__ import annotations

import math

import numpy as np

from .attention import dense, softmax_rows
from .cache import upsample_nn
from .geometry import Schedule, ceil_div
from .mapping import map_token, phi


def colsum(q: np.ndarray, k: np.ndarray, n_kv: int, C: int) -> np.ndarray:
    """A^(S) for one (b, h): (G_S, n_kv) fp64 column sums of P over query blocks of C rows."""
    q, k = np.asarray(q, np.float64), np.asarray(k, np.float64)
    P = softmax_rows((q @ k[:n_kv].T) / math.sqrt(q.shape[1]))
    G = ceil_div(q.shape[0], C)
    return np.stack([P[g * C:(g + 1) * C].sum(axis=0) for g in range(G)])


def select_tokens(a_row: np.ndarray, k_tok: int, n_sink_tokens: int) -> np.ndarray:
    """TopK of one column-sum row (ties to the smaller j), then the first n_sink_tokens tokens
    (0 in the paper-literal order, READING 25)."""
    order = sorted(range(len(a_row)), key=lambda j: (-a_row[j], j))
    sel = np.zeros(len(a_row), dtype=bool)
    sel[order[:k_tok]] = True
    sel[:n_sink_tokens] = True
    return sel


def topk_count(n_kv: int, alpha: float) -> int:
    """k = ceil(alpha * C_S), at least 1 (READING 11)."""
    return max(1, math.ceil(alpha * n_kv))


def map_tokens(src: np.ndarray, sched: Schedule, S: int, K: int, C: int, sink_scales: int,
               mode: str = "footprint") -> np.ndarray:
    """(G_S, C_S) source token selection -> (G_K, C_K) target token selection."""
    G_S, G_K = ceil_div(sched.N(S), C), ceil_div(sched.N(K), C)
    assert src.shape == (G_S, sched.C(S))
    dst = np.zeros((G_K, sched.C(K)), dtype=bool)
    n_sink = sched.C(sink_scales) if sink_scales > 0 else 0
    for g in range(G_K):
        for j in np.nonzero(src[phi(g, G_S, G_K)])[0]:
            lp, rows, cols = map_token(sched, int(j), S, K, mode)
            base = sched.C(lp - 1)
            for xp in rows:
                for yp in cols:
                    dst[g, base + xp * sched.s(lp) + yp] = True
        dst[g, :n_sink] = True
    return dst


def token_sparse(q: np.ndarray, k: np.ndarray, v: np.ndarray, C: int, sel: np.ndarray,
                 rows=None) -> np.ndarray:
    """Delta O for one (b, h): rows of query block g attend the tokens sel[g] (bool, n_kv)."""
    q, k, v = (np.asarray(a, np.float64) for a in (q, k, v))
    n_q, D = q.shape
    out = np.full((n_q, v.shape[1]), np.nan)
    for g in (range(ceil_div(n_q, C)) if rows is None else rows):
        J = np.nonzero(sel[g])[0]
        if len(J) == 0:
            raise ValueError(f"query block {g} selects no key")
        qg = q[g * C:min((g + 1) * C, n_q)]
        out[g * C:g * C + len(qg)] = softmax_rows((qg @ k[J].T) / math.sqrt(D)) @ v[J]
    return out


def token_cache_residual(q_S, k, v, n_kv_S: int, C: int, sel_S: np.ndarray) -> np.ndarray:
    """O_cache^(S) for one (b, h): dense minus token-sparse attention at S."""
    return dense(q_S, k, v, n_kv_S) - token_sparse(q_S, k, v, C, sel_S)


def token_cached_sparse(q_k, k, v, C: int, sel_k: np.ndarray, o_cache_S: np.ndarray, s_S: int,
                        s_k: int) -> np.ndarray:
    """O^(k) ~= upsample(O_cache^(S)) + Delta O^(k) on the token path."""
    return token_sparse(q_k, k, v, C, sel_k) + upsample_nn(o_cache_S, s_S, s_k)
