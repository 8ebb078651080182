"""CS4A pattern composition: decision-scale selection, mapping to the target scale, sink.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper's order (§3.2, App. "Cross-Scale Sparse Index Mapping"):
  inds^(S)  = TopK(D^(S))                         the Top-K alone
  O_cache^(S) subtracts the sparse term over inds^(S)
  inds^(k)  = M_{S->k}(inds^(S)), then Concat(S, inds^(k))
  inds^(K)  = A_sink U M_{S->K}(inds^(S))
READING 25: this paper-literal order is the default.  `sink_in_source=True` gives
the alternative composition the first round used — the sink blocks OR-ed into the S-level
pattern (after the selection) and mapped along with it — under which the sink block(s) of S also
pull in their footprint at K (at Infinity-1K 11 -> 13, B = 128: block 0 -> blocks 0..4).

Pins (tests/test_oracle_cs4a.py): the S-level pattern of the paper-literal order holds exactly k
blocks per row (Top-K only); an empty source maps to exactly the sink blocks; the sink block of
S = 11 maps to blocks {0, 1, 2, 3, 4} at K = 13, B = 128 (worked by hand from the schedule); the
two compositions differ by exactly the image of the sink blocks.
"""
from __future__ import annotations

from .mapping import map_pattern
from .predictor import predict_pattern


def cs4a_patterns(q_S, k, sched, S: int, K: int, B: int, sink_scales: int, mode: str = "topk",
                  topk: int = 1, tau: float = 0.0, map_mode: str = "footprint",
                  sink_in_source: bool = False, scale=None):
    """(pattern at S, pattern at K, masses) for one (b, h).

    pattern_S is the S-level index set the O_cache residual subtracts over; pattern_K is the
    target pattern the CS4A attention at K attends."""
    src, mass = predict_pattern(q_S, k, sched, S, B, sink_scales if sink_in_source else 0, mode,
                                topk, tau, scale)
    dst = map_pattern(src, sched, S, K, B, sink_scales, map_mode)     # A_sink U M(inds^(S))
    return src, dst, mass
