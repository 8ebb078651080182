"""O4 — block-level sparse-pattern predictor at the decision scale S.  TEST INFRASTRUCTURE ONLY.

Definitions followed (§3.2 "Sparse Decision Scale", App. "Hardware-Efficient Sparse
Computation")
  P^(S) = Softmax(Q^(S) K^(S)T / sqrt(d))  over the keys j < C_S
  column sums D^(S)_{b,h,i,j} = sum_{q in query block i} P^(S)_{b,h,q,j}
  Top-k over the column sums -> inds^(S)  (the Top-K alone)
  The paper adds the sink only at the target, after the mapping:
        inds^(k) <- Concat(S, inds^(k))
        inds^(K) = A_sink U M_{S->K}(inds^(S))
  READING 25: `sink_scales` of predict_pattern is therefore 0 on the paper-literal path (the
      default composition, oracle/cs4a.py).  A positive value gives the alternative
      "sink_in_source" composition — the sink OR-ed into the S-level pattern after the selection,
      which the mapping then carries to K — kept as an option (north_star: "always including the
      attention-sink blocks ... (2) carries that block pattern").
  READING 10: the predictor works at block granularity with the attention block size B, so the
      scored quantity is the block mass  mass[u, v] = sum_{j in KV block v, j < C_S} D[u, j]
      (= sum_{q in u} sum_{j in v} P[q, j]), and inds are KV *blocks*.
  READING 11: Top-K takes an integer k (the harness converts a fraction alpha).  Ties are broken
      toward the smaller block index: order by (mass desc, v asc), keep the first k.
  READING 12: THRESHOLD(tau) keeps mass[u, v] >= tau * |u| (inclusive; |u| = rows of block u),
      i.e. the mean per-query probability mass in the block is at least tau.
  READING 13: sink blocks are v < ceil(C_{sink_scales} / B), in full.

Pins (tests/test_oracle_predictor.py): sum_v mass[u, v] = |u| (softmax rows sum to one), a
brute-force double loop over (q, j) on tiny inputs, k = G_kv selects every block, the planted
dominant key is selected at k = 1, the tie rule on [0.1, 0.5, 0.5, 0.2]
(SPEC.md:206), and top-k against an exhaustive subset search on small rows.
"""
from __future__ import annotations

import math
from typing import Optional

import numpy as np

from .geometry import Schedule, ceil_div


def block_mass(q: np.ndarray, k: np.ndarray, sched: Schedule, S: int, B: int,
               scale: Optional[float] = None) -> np.ndarray:
    """mass[u, v] for one (b, h).  q: (N_S, D), k: (>= C_S, D).  fp64."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    n_q, n_kv = sched.N(S), sched.C(S)
    D = q.shape[1]
    if scale is None:
        scale = 1.0 / math.sqrt(D)
    z = (q[:n_q] @ k[:n_kv].T) * scale
    z = z - z.max(axis=1, keepdims=True)
    P = np.exp(z)
    P = P / P.sum(axis=1, keepdims=True)                                # row softmax
    gq, gkv = ceil_div(n_q, B), ceil_div(n_kv, B)
    Dcol = np.zeros((gq, n_kv))
    for i in range(gq):
        Dcol[i] = P[i * B: min((i + 1) * B, n_q)].sum(axis=0)
    mass = np.zeros((gq, gkv))
    for v in range(gkv):                                                 # READING 10
        mass[:, v] = Dcol[:, v * B: min((v + 1) * B, n_kv)].sum(axis=1)
    return mass


def select_topk(mass_row: np.ndarray, k: int) -> np.ndarray:
    """Indices of the k largest masses, ties to the smaller v (READING 11); ascending order."""
    order = sorted(range(len(mass_row)), key=lambda v: (-mass_row[v], v))
    return np.array(sorted(order[:k]), dtype=np.int64)


def select_threshold(mass_row: np.ndarray, tau: float, rows_in_block: int) -> np.ndarray:
    """Blocks with mass >= tau * |u| (READING 12)."""
    return np.array([v for v in range(len(mass_row)) if mass_row[v] >= tau * rows_in_block],
                    dtype=np.int64)


def sink_blocks(sched: Schedule, sink_scales: int, B: int) -> int:
    """Number of leading KV blocks that hold the sink tokens (READING 13)."""
    return ceil_div(sched.C(sink_scales), B) if sink_scales > 0 else 0


def predict_pattern(q: np.ndarray, k: np.ndarray, sched: Schedule, S: int, B: int,
                    sink_scales: int, mode: str = "topk", topk: int = 1, tau: float = 0.0,
                    scale: Optional[float] = None):
    """Boolean source pattern (G_S x G_kvS) for one (b, h), plus the masses.
    Selection first; sink_scales > 0 then ORs the sink blocks into the S-level
    pattern (READING 25's "sink_in_source" option; the paper adds them at the target only)."""
    mass = block_mass(q, k, sched, S, B, scale)
    gq, gkv = mass.shape
    n_q = sched.N(S)
    pat = np.zeros((gq, gkv), dtype=bool)
    nsb = min(sink_blocks(sched, sink_scales, B), gkv)
    for u in range(gq):
        if mode == "topk":
            sel = select_topk(mass[u], topk)
        elif mode == "threshold":
            sel = select_threshold(mass[u], tau, min((u + 1) * B, n_q) - u * B)
        else:
            raise ValueError(mode)
        pat[u, sel] = True
        pat[u, :nsb] = True
    return pat, mass
