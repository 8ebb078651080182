"""Pins for oracle/kv_compress.py (NEXT(4), KV compression for CSLA layers)."""
import numpy as np

from oracle.attention import brute_force, block_sparse
from oracle.csla import local_block_mask, token_mask
from oracle.geometry import INFINITY_1K_SIDES, Schedule, ceil_div
from oracle.kv_compress import (compress, compressed_local_block_mask, kept_index, kept_ranges,
                                kept_scales)

INF = Schedule(INFINITY_1K_SIDES)


def test_kept_rows_infinity():
    assert kept_scales(13, 5, (7, 5, 3, 1, 1)) == [1, 2, 3, 4, 5, 9, 10, 11, 12, 13]
    assert kept_ranges(INF, 13, 5, (7, 5, 3, 1, 1)) == [(0, INF.C(5)), (INF.C(8), INF.C(13))]
    assert len(kept_index(INF, 13, 5, (7, 5, 3, 1, 1))) == INF.C(5) + INF.C(13) - INF.C(8) == 9721


def test_nothing_dropped_is_identity():
    s = Schedule([1, 2, 4, 6, 8])
    w = (3, 3, 3, 3, 3)
    assert np.array_equal(kept_index(s, 5, 0, w), np.arange(s.C(5)))
    for B in (1, 4, 16):
        assert np.array_equal(compressed_local_block_mask(s, 5, B, 0, w),
                              local_block_mask(s, 5, B, 0, w))


def test_token_level_attention_is_unchanged():
    """B = 1: the compressed layer attends exactly the same keys (brute force on both sides)."""
    s = Schedule([1, 2, 4, 6, 8])
    K, sink, w, D = 5, 2, (3, 1), 8
    rng = np.random.default_rng(3)
    q, k, v = rng.standard_normal((s.N(K), D)), rng.standard_normal((s.C(K), D)), \
        rng.standard_normal((s.C(K), D))
    M = token_mask(s, K, sink, w)
    full = brute_force(q, k, v, s.C(K), allowed=lambda t, j: M[t, j])
    kc, vc = compress(k, s, K, sink, w), compress(v, s, K, sink, w)
    Mc = compressed_local_block_mask(s, K, 1, sink, w)
    lists = [np.nonzero(r)[0] for r in Mc]
    comp = block_sparse(q, kc, vc, len(kc), 1, lists)
    assert len(kc) < s.C(K)                        # scale 3 is dropped
    assert np.allclose(comp, full, atol=1e-12)
