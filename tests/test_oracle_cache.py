"""Pins of oracle/cache.py (NEXT 1: O_cache residual) — CPU only."""
import numpy as np

from oracle.attention import block_sparse, dense, merge_lists
from oracle.cache import cache_residual, cached_sparse, upsample_nn
from oracle.geometry import Schedule, ceil_div
from oracle.predictor import predict_pattern
from synth import kv_cache_iid, q_iid, structured_qkv

SIDES = [1, 2, 4, 6, 8, 12]
S, K, B, D = 5, 6, 16, 32


def _inputs(seed=0):
    sched = Schedule(SIDES)
    qS = q_iid(seed, S, 0, 1, sched.N(S), D)[0].double().numpy()
    qK = q_iid(seed, K, 0, 1, sched.N(K), D)[0].double().numpy()
    k, v = kv_cache_iid(seed, 0, 1, sched.C(K), D)
    return sched, qS, qK, k[0].double().numpy(), v[0].double().numpy()


def test_reconstruction_identity():
    sched, qS, _, k, v = _inputs(1)
    src, _ = predict_pattern(qS, k, sched, S, B, 2, "topk", 2)
    lists = merge_lists([src])
    oc = cache_residual(qS, k, v, sched.C(S), B, lists)
    recon = oc + block_sparse(qS, k, v, sched.C(S), B, lists)
    assert np.abs(recon - dense(qS, k, v, sched.C(S))).max() <= 1e-12


def test_all_blocks_gives_zero_cache():
    sched, qS, _, k, v = _inputs(2)
    gq, gkv = ceil_div(sched.N(S), B), ceil_div(sched.C(S), B)
    lists = [np.arange(gkv)] * gq
    oc = cache_residual(qS, k, v, sched.C(S), B, lists)
    assert np.abs(oc).max() <= 1e-12


def test_partial_lists_give_nonzero_cache():
    sched, qS, _, k, v = _inputs(3)
    gq = ceil_div(sched.N(S), B)
    lists = [np.array([0])] * gq
    assert np.abs(cache_residual(qS, k, v, sched.C(S), B, lists)).max() > 1e-3


def test_upsample_constant_identity_and_replication():
    c = np.full((8 * 8, 3), 0.25)
    assert np.array_equal(upsample_nn(c, 8, 12), np.full((12 * 12, 3), 0.25))
    rng = np.random.default_rng(0)
    x = rng.standard_normal((6 * 6, 4))
    assert np.array_equal(upsample_nn(x, 6, 6), x)
    # integer ratio: nearest neighbour is plain pixel replication of the 2-D grid
    small = rng.standard_normal((4, 4, 2))
    want = np.repeat(np.repeat(small, 3, axis=0), 3, axis=1).reshape(144, 2)
    assert np.array_equal(upsample_nn(small.reshape(16, 2), 4, 12), want)


def test_cached_output_is_sparse_plus_upsampled_cache():
    sched, qS, qK, k, v = _inputs(4)
    gq = ceil_div(sched.N(K), B)
    src, _ = predict_pattern(qS, k, sched, S, B, 2, "topk", 2)
    oc = cache_residual(qS, k, v, sched.C(S), B, merge_lists([src]))
    lists_k = [np.array([0, 1, 2])] * gq
    out = cached_sparse(qK, k, v, sched.C(K), B, lists_k, oc, SIDES[S - 1], SIDES[K - 1])
    delta = block_sparse(qK, k, v, sched.C(K), B, lists_k)
    assert np.abs(out - delta - upsample_nn(oc, SIDES[S - 1], SIDES[K - 1])).max() <= 1e-14
