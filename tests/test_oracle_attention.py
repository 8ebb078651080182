"""Pins for oracle/attention.py (O6-O8)."""
import numpy as np

from oracle.attention import block_sparse, brute_force, dense, merge_lists, to_csr
from oracle.csla import local_block_mask
from oracle.geometry import Schedule, ceil_div
from synth import qkv_iid

TINY = Schedule([1, 2, 4, 8])        # C = 1, 5, 21, 85


def _tiny(D=8, seed=0, scale=4):
    q, k, v = qkv_iid(seed, scale, 0, 1, TINY.N(scale), TINY.C(scale), D)
    return q[0].double().numpy(), k[0].double().numpy(), v[0].double().numpy()


def test_dense_vs_triple_loop():
    """dense == an independent per-element triple loop, <= 1e-12."""
    q, k, v = _tiny(D=4)
    assert np.abs(dense(q, k, v, 85) - brute_force(q, k, v, 85)).max() < 1e-12


def test_all_blocks_equals_dense():
    """every block listed == dense (<= 1e-12 in fp64)."""
    q, k, v = _tiny()
    for B in (1, 16, 32, 64):
        lists = [np.arange(ceil_div(85, B))] * ceil_div(64, B)
        assert np.abs(block_sparse(q, k, v, 85, B, lists) - dense(q, k, v, 85)).max() < 1e-12


def test_block_sparse_vs_masked_bruteforce():
    """Brute force over the token-expanded block mask (CSLA mask of the tiny schedule)."""
    q, k, v = _tiny(D=4)
    B = 16
    bm = local_block_mask(TINY, 4, B, 2, (3, 3))
    lists = merge_lists([bm])
    want = brute_force(q, k, v, 85, allowed=lambda t, j: bm[t // B, j // B])
    assert np.abs(block_sparse(q, k, v, 85, B, lists) - want).max() < 1e-12


def test_sink_only_is_truncated_attention():
    """only the sink column active == attention over KV [0, C_m).  Schedule
    where C_sink is a multiple of B: sides 4,4,8 -> C = 16, 32, 96 with B = 16."""
    s = Schedule([4, 4, 8])
    q, k, v = qkv_iid(3, 3, 0, 1, 64, 96, 8)
    q, k, v = q[0].double().numpy(), k[0].double().numpy(), v[0].double().numpy()
    lists = [np.array([0])] * 4
    assert np.abs(block_sparse(q, k, v, 96, 16, lists) - dense(q, k[:16], v[:16], 16)).max() < 1e-13


def test_single_key_and_uniform():
    q = np.zeros((3, 2)); k = np.random.default_rng(0).random((5, 2)); v = np.arange(10.).reshape(5, 2)
    assert np.allclose(dense(q, k, v, 1), v[0])                 # one key -> its value row
    assert np.allclose(dense(q, k, v, 5), v.mean(0))            # equal logits -> mean row


def test_convex_and_shift_invariant():
    q, k, v = _tiny()
    o = dense(q, k, v, 85)
    assert (o <= v[:85].max(0) + 1e-12).all() and (o >= v[:85].min(0) - 1e-12).all()
    # a per-row shift of the logits: add a multiple of a direction orthogonal to... simpler: a
    # constant key offset c changes every logit of row t by q_t . c
    c = np.random.default_rng(2).standard_normal(q.shape[1])
    assert np.abs(dense(q, k + c, v, 85) - o).max() < 1e-12


def test_merge_and_csr():
    a = np.array([[1, 0, 0, 1], [0, 0, 0, 0]], bool)
    b = np.array([[0, 0, 1, 0], [0, 1, 0, 0]], bool)
    lists = merge_lists([a, b])
    assert [list(x) for x in lists] == [[0, 2, 3], [1]]
    rp, col = to_csr(lists)
    assert list(rp) == [0, 3, 4] and list(col) == [0, 2, 3, 1]
