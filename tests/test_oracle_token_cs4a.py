"""Pins for oracle/token_cs4a.py (NEXT(2), token-granular CS4A)."""
import math

import numpy as np
import pytest

from oracle.attention import block_sparse, dense
from oracle.geometry import Schedule, ceil_div
from oracle.mapping import map_pattern
from oracle.cache import cache_residual
from oracle.token_cs4a import (colsum, map_tokens, select_tokens, token_cache_residual, token_sparse,
                               topk_count)

TINY = Schedule([1, 2, 4, 8])          # C = 1, 5, 21, 85
EQ = Schedule([1, 2, 4, 6, 8, 12, 16])


def _rand(seed, *shape):
    return np.random.default_rng(seed).standard_normal(shape)


def test_colsum_rows_add_up():
    q, k = _rand(0, EQ.N(5), 32), _rand(1, EQ.C(5), 32)
    for C in (16, 24, 64):
        a = colsum(q, k, EQ.C(5), C)
        rows = [min((g + 1) * C, EQ.N(5)) - g * C for g in range(ceil_div(EQ.N(5), C))]
        assert np.allclose(a.sum(1), rows, rtol=0, atol=1e-12)


def test_colsum_bruteforce():
    """Per-element exp loops, independent of the matrix formulation."""
    q, k = _rand(2, TINY.N(3), 4), _rand(3, TINY.C(3), 4)
    C, n = 6, TINY.C(3)
    a = colsum(q, k, n, C)
    for g in range(ceil_div(TINY.N(3), C)):
        for j in range(n):
            tot = 0.0
            for t in range(g * C, min((g + 1) * C, TINY.N(3))):
                z = [sum(q[t, d] * k[i, d] for d in range(4)) / 2.0 for i in range(n)]
                m = max(z)
                tot += math.exp(z[j] - m) / sum(math.exp(x - m) for x in z)
            assert abs(a[g, j] - tot) < 1e-12


def test_select_all_and_planted():
    row = _rand(4, 50) ** 2
    assert select_tokens(row, 50, 0).all() and select_tokens(row, 500, 0).all()
    row[17] = 1e9
    sel = select_tokens(row, 1, 3)
    assert sel[17] and sel[:3].all() and sel.sum() == 4
    ties = np.ones(10)
    assert list(np.nonzero(select_tokens(ties, 4, 0))[0]) == [0, 1, 2, 3]   # ties -> smaller j
    assert topk_count(4121, 0.2) == 825 and topk_count(10, 0.0) == 1


def test_map_identity_at_same_scale():
    rng = np.random.default_rng(5)
    C = 16
    src = rng.random((ceil_div(EQ.N(6), C), EQ.C(6))) < 0.1
    out = map_tokens(src, EQ, 6, 6, C, 3)
    want = src.copy()
    want[:, :EQ.C(3)] = True
    assert np.array_equal(out, want)


@pytest.mark.parametrize("S,K", [(5, 7), (4, 6), (5, 6)])
def test_map_agrees_with_block_mapping(S, K):
    """With C = B the block-OR of the token map equals the pinned block map of the block-OR."""
    B = 16
    rng = np.random.default_rng(S * 10 + K)
    src = rng.random((ceil_div(EQ.N(S), B), EQ.C(S))) < 0.05
    dst = map_tokens(src, EQ, S, K, B, 3)
    gkv_S, gkv_K = ceil_div(EQ.C(S), B), ceil_div(EQ.C(K), B)
    src_blk = np.stack([[src[g, v * B:(v + 1) * B].any() for v in range(gkv_S)]
                        for g in range(src.shape[0])])
    dst_blk = np.stack([[dst[g, v * B:(v + 1) * B].any() for v in range(gkv_K)]
                        for g in range(dst.shape[0])])
    # the token map of a block's *selected* tokens is contained in the block map of the block;
    # selecting whole blocks makes them equal
    full = np.repeat(src_blk, B, axis=1)[:, :EQ.C(S)]
    dst_full = map_tokens(full, EQ, S, K, B, 3)
    dst_full_blk = np.stack([[dst_full[g, v * B:(v + 1) * B].any() for v in range(gkv_K)]
                             for g in range(dst_full.shape[0])])
    want = map_pattern(src_blk, EQ, S, K, B, 3, "footprint")
    assert np.array_equal(dst_full_blk, want)
    assert not (dst_blk & ~want).any()


def test_token_sparse_reduces_to_dense_and_block_sparse():
    n_q, n_kv, D, C = EQ.N(6), EQ.C(6), 16, 24
    q, k, v = _rand(6, n_q, D), _rand(7, n_kv, D), _rand(8, n_kv, D)
    G = ceil_div(n_q, C)
    assert np.allclose(token_sparse(q, k, v, C, np.ones((G, n_kv), bool)), dense(q, k, v, n_kv),
                       atol=1e-12)
    rng = np.random.default_rng(9)
    blk = rng.random((G, ceil_div(n_kv, C))) < 0.3
    blk[:, 0] = True
    sel = np.repeat(blk, C, axis=1)[:, :n_kv]
    want = block_sparse(q, k, v, n_kv, C, [np.nonzero(r)[0] for r in blk])
    assert np.allclose(token_sparse(q, k, v, C, sel), want, atol=1e-12)


def test_token_cache_residual():
    n_q, n_kv, D, C = EQ.N(5), EQ.C(5), 16, 16
    q, k, v = _rand(10, n_q, D), _rand(11, n_kv, D), _rand(12, n_kv, D)
    G = ceil_div(n_q, C)
    assert np.abs(token_cache_residual(q, k, v, n_kv, C, np.ones((G, n_kv), bool))).max() < 1e-12
    rng = np.random.default_rng(13)
    blk = rng.random((G, ceil_div(n_kv, C))) < 0.4
    blk[:, 0] = True
    sel = np.repeat(blk, C, axis=1)[:, :n_kv]
    want = cache_residual(q, k, v, n_kv, C, [np.nonzero(r)[0] for r in blk])
    assert np.allclose(token_cache_residual(q, k, v, n_kv, C, sel), want, atol=1e-12)
