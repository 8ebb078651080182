"""GPU parity of the block-sparse / dense attention kernel (a6/a7) through the C ABI against the
fp64 oracle on the same bf16 inputs: max |diff| <= 1e-2 and mean |diff| <= 1e-3 (north_star)."""
import numpy as np
import pytest
import torch

from oracle.attention import block_sparse, dense, merge_lists
from oracle.csla import local_block_mask
from oracle.geometry import INFINITY_1K_SIDES, Schedule, ceil_div
from synth import kv_cache_iid, q_iid
from tests.helpers import (EQ256, INF2B, MAX_ABS, MEAN_ABS, TINY, attn_errors, bool_to_bits,
                           csr_lists, to_np)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sv():
    import paper_2602_04361_b200 as m
    return m


def _inputs(sides, K, D, bh, seed=0, cap_extra=0):
    sched = Schedule(sides)
    q = q_iid(seed, K, 0, bh, sched.N(K), D)
    k, v = kv_cache_iid(seed, 0, bh, sched.C(K), D, capacity=sched.C(K) + cap_extra)
    return sched, q.cuda(), k.cuda(), v.cuda()


def _lists_from_bool(sv, masks_bh):
    bh, gq, gkv = masks_bh.shape
    return sv.build_block_lists(bh, gq, gkv, [(torch.from_numpy(bool_to_bits(masks_bh)).cuda(), False)])


def _check(got, want, rows=None):
    g = to_np(got)
    if rows is not None:
        g, want = g[rows], want[rows]
    mx, mean = attn_errors(g, want)
    assert mx <= MAX_ABS and mean <= MEAN_ABS, (mx, mean)
    return mx, mean


@pytest.mark.parametrize("D", [64, 128])
@pytest.mark.parametrize("B", [16, 32, 64, 128])
def test_random_lists(sv, D, B):
    """Random ascending lists incl. the ragged last KV block, ragged query tiles (N=144)."""
    sides = [1, 2, 4, 6, 8, 12, 16, 20]          # C = ..., 665, 1065; N_8 = 400
    K, bh = 8, 3
    sched, q, k, v = _inputs(sides, K, D, bh, seed=B + D, cap_extra=40)
    gq, gkv = ceil_div(sched.N(K), B), ceil_div(sched.C(K), B)
    rng = np.random.default_rng(B)
    m = rng.random((bh, gq, gkv)) < 0.3
    m[:, :, gkv - 1] |= rng.random((bh, gq)) < 0.5
    m[:, :, 0] |= ~m.any(2)
    rp, ci, st = _lists_from_bool(sv, m)
    o = sv.block_sparse_attn(sides, K, B, q, k, v, rp, ci)
    torch.cuda.synchronize()
    assert st.item() == 0
    for b in range(bh):
        want = block_sparse(to_np(q[b]), to_np(k[b]), to_np(v[b]), sched.C(K), B,
                            merge_lists([m[b]]))
        _check(o[b], want)


@pytest.mark.parametrize("cfg", [TINY, EQ256], ids=["tiny", "256eq"])
def test_csla_pipeline_small(sv, cfg):
    """GPU local mask -> GPU lists -> GPU attention vs oracle mask -> oracle attention."""
    sides, K, B, D, bh = cfg["sides"], cfg["K"], cfg["B"], cfg["D"], cfg["bh"]
    sched, q, k, v = _inputs(sides, K, D, bh, seed=1)
    g = sv.geometry(sides, K, B)
    mask = sv.local_mask(sides, K, B, cfg["sink"], cfg["windows"])
    rp, ci, st = sv.build_block_lists(bh, g["G_q"], g["G_kv"], [(mask, True)])
    o = sv.block_sparse_attn(sides, K, B, q, k, v, rp, ci)
    torch.cuda.synchronize()
    assert st.item() == 0
    lists = merge_lists([local_block_mask(sched, K, B, cfg["sink"], cfg["windows"])])
    for b in range(bh):
        want = block_sparse(to_np(q[b]), to_np(k[b]), to_np(v[b]), sched.C(K), B, lists)
        _check(o[b], want)


@pytest.mark.parametrize("cfg", [TINY, EQ256], ids=["tiny", "256eq"])
def test_dense_small(sv, cfg):
    sides, K, D, bh = cfg["sides"], cfg["K"], cfg["D"], cfg["bh"]
    sched, q, k, v = _inputs(sides, K, D, bh, seed=2)
    lse = torch.empty((bh, sched.N(K)), dtype=torch.float32, device="cuda")
    o = sv.dense_attn(sides, K, q, k, v, lse=lse)
    torch.cuda.synchronize()
    for b in range(bh):
        qb, kb, vb = to_np(q[b]), to_np(k[b]), to_np(v[b])
        _check(o[b], dense(qb, kb, vb, sched.C(K)))
        z = qb @ kb[:sched.C(K)].T / np.sqrt(D)
        ref_lse = np.log(np.exp(z - z.max(1, keepdims=True)).sum(1)) + z.max(1)
        assert np.abs(lse[b].cpu().numpy() - ref_lse).max() < 1e-3


def test_all_blocks_equals_dense_kernel(sv):
    """An all-ones list through the sparse path == the dense path (same kernel, same order:
    bitwise equal)."""
    cfg = EQ256
    sides, K, B, D, bh = cfg["sides"], cfg["K"], 128, cfg["D"], 2
    sched, q, k, v = _inputs(sides, K, D, bh, seed=3)
    gq, gkv = ceil_div(sched.N(K), B), ceil_div(sched.C(K), B)
    rp, ci, _ = _lists_from_bool(sv, np.ones((bh, gq, gkv), dtype=bool))
    o1 = sv.block_sparse_attn(sides, K, B, q, k, v, rp, ci)
    o2 = sv.dense_attn(sides, K, q, k, v)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)


def test_full_size_sampled_rows(sv):
    """2B-shaped config at the bench launch configuration (K=13, B=128, 16 heads, CSLA default):
    sampled query blocks checked against the oracle one by one."""
    cfg = INF2B
    sides, K, B, D, bh = cfg["sides"], cfg["K"], cfg["B"], cfg["D"], cfg["bh"]
    sched, q, k, v = _inputs(sides, K, D, bh, seed=4)
    g = sv.geometry(sides, K, B)
    mask = sv.local_mask(sides, K, B, cfg["sink"], cfg["windows"])
    rp, ci, st = sv.build_block_lists(bh, g["G_q"], g["G_kv"], [(mask, True)])
    o = sv.block_sparse_attn(sides, K, B, q, k, v, rp, ci)
    torch.cuda.synchronize()
    assert st.item() == 0
    lists = merge_lists([local_block_mask(sched, K, B, cfg["sink"], cfg["windows"])])
    rng = np.random.default_rng(0)
    for b in rng.choice(bh, 4, replace=False):
        rows_u = sorted(set(rng.choice(g["G_q"], 5, replace=False)) | {0, g["G_q"] - 1})
        want = block_sparse(to_np(q[b]), to_np(k[b]), to_np(v[b]), sched.C(K), B, lists, rows=rows_u)
        sel = np.concatenate([np.arange(u * B, min((u + 1) * B, sched.N(K))) for u in rows_u])
        _check(o[b], want, rows=sel)


def test_full_size_dense_sampled(sv):
    sides, K, D, bh = list(INFINITY_1K_SIDES), 13, 128, 2
    sched, q, k, v = _inputs(sides, K, D, bh, seed=5)
    o = sv.dense_attn(sides, K, q, k, v)
    torch.cuda.synchronize()
    rows = np.array([0, 1, 777, 2048, 4095])
    for b in range(bh):
        want = dense(to_np(q[b])[rows], to_np(k[b]), to_np(v[b]), sched.C(K))
        mx, mean = attn_errors(to_np(o[b])[rows], want)
        assert mx <= MAX_ABS and mean <= MEAN_ABS


def test_empty_row_gives_zero(sv):
    sides, K, B, D, bh = [1, 2, 4, 8], 4, 16, 64, 1
    sched, q, k, v = _inputs(sides, K, D, bh)
    m = np.zeros((1, 4, 6), dtype=bool)
    m[0, [0, 1, 3], 2] = True                              # row 2 empty
    g = sv.geometry(sides, K, B)
    rp, ci, st = _lists_from_bool(sv, m)
    lse = torch.empty((1, 64), dtype=torch.float32, device="cuda")
    o = sv.block_sparse_attn(sides, K, B, q, k, v, rp, ci, lse=lse)
    torch.cuda.synchronize()
    assert st.item() == 5
    assert (o[0, 32:48] == 0).all() and torch.isinf(lse[0, 32:48]).all()
    assert torch.isfinite(o[0, :32].float()).all()


def test_deterministic(sv):
    cfg = EQ256
    sides, K, B, D, bh = cfg["sides"], cfg["K"], cfg["B"], cfg["D"], cfg["bh"]
    sched, q, k, v = _inputs(sides, K, D, bh, seed=6)
    g = sv.geometry(sides, K, B)
    mask = sv.local_mask(sides, K, B, cfg["sink"], cfg["windows"])
    rp, ci, _ = sv.build_block_lists(bh, g["G_q"], g["G_kv"], [(mask, True)])
    o1 = sv.block_sparse_attn(sides, K, B, q, k, v, rp, ci)
    o2 = sv.block_sparse_attn(sides, K, B, q, k, v, rp, ci)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)


@pytest.mark.parametrize("B", [128, 64])
def test_persistent_schedule_mixed_lengths(sv, B):
    """Many tiles per CTA with very uneven list lengths (1 block up to every block, plus empty
    rows): exercises the persistent two-slot schedule, the Q-buffer rotation and the KV ring
    wrap-around at the full Infinity-1K shape.  Sampled query blocks vs the oracle."""
    sides, K, D, bh = list(INFINITY_1K_SIDES), 13, 128, 40
    sched, q, k, v = _inputs(sides, K, D, bh, seed=7)
    gq, gkv = ceil_div(sched.N(K), B), ceil_div(sched.C(K), B)
    rng = np.random.default_rng(11)
    kind = rng.integers(0, 5, size=(bh, gq))
    m = np.zeros((bh, gq, gkv), dtype=bool)
    for b in range(bh):
        for u in range(gq):
            if kind[b, u] == 0:
                m[b, u, rng.integers(0, gkv)] = True            # a single block
            elif kind[b, u] == 1:
                m[b, u, :] = True                                # every block
            elif kind[b, u] == 2:
                m[b, u, :] = rng.random(gkv) < 0.1
            elif kind[b, u] == 3:
                m[b, u, gkv - 1] = True                          # only the ragged last block
            # kind 4: empty row
    rp, ci, st = _lists_from_bool(sv, m)
    lse = torch.empty((bh, sched.N(K)), dtype=torch.float32, device="cuda")
    o = sv.block_sparse_attn(sides, K, B, q, k, v, rp, ci, lse=lse)
    torch.cuda.synchronize()
    assert st.item() in (0, 5)
    for b in rng.choice(bh, 6, replace=False):
        rows_u = sorted(set(rng.choice(gq, 6, replace=False)) | {0, gq - 1})
        empty = [u for u in rows_u if not m[b, u].any()]
        live = [u for u in rows_u if m[b, u].any()]
        for u in empty:
            assert (o[b, u * B:(u + 1) * B] == 0).all()
            assert torch.isinf(lse[b, u * B:(u + 1) * B]).all()
        if live:
            want = block_sparse(to_np(q[b]), to_np(k[b]), to_np(v[b]), sched.C(K), B,
                                merge_lists([m[b]]), rows=live)
            sel = np.concatenate([np.arange(u * B, min((u + 1) * B, sched.N(K))) for u in live])
            _check(o[b], want, rows=sel)


def test_persistent_schedule_several_batches(sv):
    """More than MAX_TILES (96) tiles per CTA, so every CTA runs a second schedule batch: the
    role state carried from one batch to the next (KV ring position, P and S phases, tiles done,
    Q-buffer use parities) must continue exactly.  Small tiles (N_K = 1024, 8 query tiles per
    head) with 1850 heads = 14800 tiles = 100 per CTA on 148 SMs; heads from the last window
    (second batch) and the first are compared with the oracle."""
    sides, K, B, D, bh = [1, 2, 4, 8, 16, 32], 6, 128, 128, 1850
    sched = Schedule(sides)
    q = q_iid(3, K, 0, bh, sched.N(K), D, device="cuda")
    k, v = kv_cache_iid(3, 0, bh, sched.C(K), D, device="cuda")
    gq, gkv = ceil_div(sched.N(K), B), ceil_div(sched.C(K), B)
    rng = np.random.default_rng(5)
    m = rng.random((bh, gq, gkv)) < 0.35
    m[:, :, 0] = True                                    # sink block in every row
    m[rng.random((bh, gq)) < 0.05] = False               # a few empty rows
    rp, ci, st = _lists_from_bool(sv, m)
    o = sv.block_sparse_attn(sides, K, B, q, k, v, rp, ci)
    torch.cuda.synchronize()
    assert st.item() in (0, 5)
    for b in [0, 1, 900, bh - 60, bh - 2, bh - 1]:
        live = [u for u in range(gq) if m[b, u].any()]
        for u in range(gq):
            if not m[b, u].any():
                assert (o[b, u * B:(u + 1) * B] == 0).all()
        if live:
            want = block_sparse(to_np(q[b]), to_np(k[b]), to_np(v[b]), sched.C(K), B,
                                merge_lists([m[b]]), rows=live)
            sel = np.concatenate([np.arange(u * B, min((u + 1) * B, sched.N(K))) for u in live])
            _check(o[b], want, rows=sel)


def test_bench_shape_repeats_bitwise(sv):
    """Five CSLA launches at the bench shape (96 (b,h), 21 tiles per CTA, two slots, the K/V ring
    wrapping many times) give bit-identical outputs: the persistent schedule is deterministic and
    a barrier race would show as a mismatch."""
    sides, K, B, D, bh = list(INFINITY_1K_SIDES), 13, 128, 128, 96
    sched, q, k, v = _inputs(sides, K, D, bh, seed=9)
    g = sv.geometry(sides, K, B)
    mask = sv.local_mask(sides, K, B, 5, (7, 5, 3, 1, 1))
    rp, ci, st = sv.build_block_lists(bh, g["G_q"], g["G_kv"], [(mask, True)])
    outs = [sv.block_sparse_attn(sides, K, B, q, k, v, rp, ci) for _ in range(5)]
    torch.cuda.synchronize()
    assert st.item() == 0
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
