"""GPU parity of NEXT(2), token-granular CS4A, through the C ABI
against the fp64 oracle (oracle/token_cs4a.py) on the same bf16 inputs:
column sums within 1e-4 relative; the oracle's top-k rule applied to the GPU's fp32 column sums
reproduces the GPU selection bit for bit, and the fp64 selection agrees wherever the k-th/(k+1)-th
gap exceeds 1e-5 relative (the measured column-sum error is ~1e-6); the token map of the GPU
selection is bit-exact; token-list attention within the north-star attention tolerance."""
import numpy as np
import pytest
import torch

from oracle.attention import dense
from oracle.geometry import INFINITY_1K_SIDES, Schedule, ceil_div
from oracle.token_cs4a import colsum, map_tokens, select_tokens, token_sparse, topk_count
from synth import kv_cache_iid, q_iid
from tests.helpers import MAX_ABS, MEAN_ABS, attn_errors, bits_to_bool, to_np

pytestmark = pytest.mark.gpu

CASES = [  # sides, S, K, C, D, bh, sink, alpha
    ([1, 2, 4, 6, 8, 12, 16], 5, 7, 64, 128, 3, 3, 0.2),
    ([1, 2, 4, 8, 16], 4, 5, 64, 64, 2, 2, 0.3),
    (list(INFINITY_1K_SIDES), 11, 13, 192, 128, 2, 5, 0.2),
    (list(INFINITY_1K_SIDES), 10, 11, 128, 128, 2, 5, 0.1),
]
IDS = ["256eq_C64", "d64_C64", "infinity_11to13_C192", "infinity_10to11_C128"]


@pytest.fixture(scope="module")
def sv():
    import paper_2602_04361_b200 as m
    return m


def _run(sv, sides, S, K, C, D, bh, sink, alpha, seed=31):
    sched = Schedule(sides)
    qS = q_iid(seed, S, 0, bh, sched.N(S), D).cuda()
    qK = q_iid(seed, K, 0, bh, sched.N(K), D).cuda()
    k, v = kv_cache_iid(seed, 0, bh, sched.C(K), D)
    k, v = k.cuda(), v.cuda()
    lse = torch.empty((bh, sched.N(S)), dtype=torch.float32, device="cuda")
    sv.dense_attn(sides, S, qS, k, v, lse=lse)
    cs = sv.token_colsum(sides, S, C, qS, k, lse)
    k_tok = topk_count(sched.C(S), alpha)
    sel = sv.token_select(sides, S, C, sink, cs, k_tok)
    dst = sv.token_map(sides, S, K, C, sink, sel)
    G_K = ceil_div(sched.N(K), C)
    rp, ci, st = sv.build_block_lists(bh, G_K, sched.C(K), [(dst, False)])
    o = sv.token_sparse_attn(sides, K, C, qK, k, v, rp, ci)
    torch.cuda.synchronize()
    assert st.item() == 0
    return sched, qS, qK, k, v, cs, sel, dst, o, k_tok


@pytest.mark.parametrize("sides,S,K,C,D,bh,sink,alpha", CASES, ids=IDS)
def test_token_cs4a_parity(sv, sides, S, K, C, D, bh, sink, alpha):
    sched, qS, qK, k, v, cs, sel, dst, o, k_tok = _run(sv, sides, S, K, C, D, bh, sink, alpha)
    n_sink = sched.C(sink)
    got_cs = cs.cpu().numpy().astype(np.float64)
    got_sel = bits_to_bool(sel.cpu().numpy(), sched.C(S))
    got_dst = bits_to_bool(dst.cpu().numpy(), sched.C(K))
    for b in range(bh):
        qb, kb, vb = to_np(qS[b]), to_np(k[b]), to_np(v[b])
        want_cs = colsum(qb, kb, sched.C(S), C)
        err = np.abs(got_cs[b] - want_cs)
        assert (err <= 1e-4 * want_cs + 1e-8).all(), err.max()
        for g in range(want_cs.shape[0]):
            # strict: the oracle rule on the GPU's own fp32 values
            strict = select_tokens(got_cs[b, g].astype(np.float32).astype(np.float64), k_tok, n_sink)
            assert np.array_equal(strict, got_sel[b, g]), (b, g)
            # end to end on fp64 column sums, away from the k-th value
            want = select_tokens(want_cs[g], k_tok, n_sink)
            if k_tok < sched.C(S):
                thr = np.sort(want_cs[g])[::-1][k_tok - 1]
                clear = np.abs(want_cs[g] - thr) > 1e-5 * thr
                clear[:n_sink] = True
                assert np.array_equal(want[clear], got_sel[b, g][clear]), (b, g)
        want_dst = map_tokens(got_sel[b], sched, S, K, C, sink)
        assert np.array_equal(want_dst, got_dst[b]), b
        want_o = token_sparse(to_np(qK[b]), kb, vb, C, got_dst[b])
        mx, mean = attn_errors(to_np(o[b]), want_o)
        assert mx <= MAX_ABS and mean <= MEAN_ABS, (b, mx, mean)


def test_all_tokens_is_dense(sv):
    """k >= C_S at S = K selects every key: token attention equals dense attention."""
    sides, S, C, D, bh = [1, 2, 4, 6, 8, 12], 6, 64, 128, 2
    sched = Schedule(sides)
    q = q_iid(8, S, 0, bh, sched.N(S), D).cuda()
    k, v = kv_cache_iid(8, 0, bh, sched.C(S), D)
    k, v = k.cuda(), v.cuda()
    lse = torch.empty((bh, sched.N(S)), dtype=torch.float32, device="cuda")
    sv.dense_attn(sides, S, q, k, v, lse=lse)
    cs = sv.token_colsum(sides, S, C, q, k, lse)
    sel = sv.token_select(sides, S, C, 0, cs, sched.C(S))
    dst = sv.token_map(sides, S, S, C, 0, sel)
    G = ceil_div(sched.N(S), C)
    rp, ci, st = sv.build_block_lists(bh, G, sched.C(S), [(dst, False)])
    o = sv.token_sparse_attn(sides, S, C, q, k, v, rp, ci)
    torch.cuda.synchronize()
    assert bits_to_bool(sel.cpu().numpy(), sched.C(S)).all()
    for b in range(bh):
        mx, mean = attn_errors(to_np(o[b]), dense(to_np(q[b]), to_np(k[b]), to_np(v[b]), sched.C(S)))
        assert mx <= MAX_ABS and mean <= MEAN_ABS, (mx, mean)


@pytest.mark.parametrize("sides,S,K,C,D,bh,sink,alpha", [CASES[0], CASES[2]], ids=[IDS[0], IDS[2]])
def test_token_cache_path(sv, sides, S, K, C, D, bh, sink, alpha):
    """Token-level O_cache at S and its upsampled reuse at K against the oracle."""
    from oracle.token_cs4a import token_cache_residual, token_cached_sparse
    sched, qS, qK, k, v, cs, sel, dst, o, k_tok = _run(sv, sides, S, K, C, D, bh, sink, alpha)
    G_S, G_K = ceil_div(sched.N(S), C), ceil_div(sched.N(K), C)
    o_dense = sv.dense_attn(sides, S, qS, k, v)
    rpS, ciS, stS = sv.build_block_lists(bh, G_S, sched.C(S), [(sel, False)])
    oc = sv.token_cache_residual(sides, S, C, qS, k, v, rpS, ciS, o_dense)
    rpK, ciK, stK = sv.build_block_lists(bh, G_K, sched.C(K), [(dst, False)])
    o2 = sv.token_sparse_attn_cached(sides, K, C, qK, k, v, rpK, ciK, oc, S)
    torch.cuda.synchronize()
    assert stS.item() == 0 and stK.item() == 0
    got_sel = bits_to_bool(sel.cpu().numpy(), sched.C(S))
    got_dst = bits_to_bool(dst.cpu().numpy(), sched.C(K))
    for b in range(bh):
        qb, kb, vb = to_np(qS[b]), to_np(k[b]), to_np(v[b])
        want_oc = token_cache_residual(qb, kb, vb, sched.C(S), C, got_sel[b])
        mx, mean = attn_errors(to_np(oc[b]), want_oc)
        assert mx <= MAX_ABS and mean <= MEAN_ABS, ("o_cache", b, mx, mean)
        # the cached kernel's inputs include the bf16 O_cache: compared on the GPU's own
        want = token_cached_sparse(to_np(qK[b]), kb, vb, C, got_dst[b], to_np(oc[b]), sides[S - 1],
                                   sides[K - 1])
        mx, mean = attn_errors(to_np(o2[b]), want)
        assert mx <= MAX_ABS and mean <= MEAN_ABS, ("O^(K)", b, mx, mean)


def test_token_attn_empty_and_ragged_lists(sv):
    """Hand-built token lists: an empty list gives zero rows (and the cache row when cached), a
    list of 1 token returns that token's value row, a 130-token list spans a ragged second chunk."""
    sides, K, C, D, bh = [1, 2, 4, 6, 8, 12, 16], 7, 64, 128, 1
    sched = Schedule(sides)
    q = q_iid(61, K, 0, bh, sched.N(K), D).cuda()
    k, v = kv_cache_iid(61, 0, bh, sched.C(K), D)
    k, v = k.cuda(), v.cuda()
    G = ceil_div(sched.N(K), C)                      # 4 query blocks of 64 rows
    rng = np.random.default_rng(3)
    lists = [np.array([], dtype=np.int64), np.array([17]),
             np.sort(rng.choice(sched.C(K), 130, replace=False)),
             np.sort(rng.choice(sched.C(K), 300, replace=False))]
    rp = torch.tensor(np.concatenate([[0], np.cumsum([len(x) for x in lists])]), dtype=torch.int32,
                      device="cuda")
    ci = torch.tensor(np.concatenate(lists), dtype=torch.int32, device="cuda")
    o = sv.token_sparse_attn(sides, K, C, q, k, v, rp, ci)
    oc = torch.randn(bh, sched.N(5), D, device="cuda").bfloat16()
    o2 = sv.token_sparse_attn_cached(sides, K, C, q, k, v, rp, ci, oc, 5)
    torch.cuda.synchronize()
    assert torch.count_nonzero(o[0, :C]) == 0
    from oracle.cache import upsample_nn
    up = upsample_nn(to_np(oc[0]), sides[4], sides[K - 1])
    assert np.abs(to_np(o2[0, :C]) - up[:C]).max() == 0.0          # empty list: the cache row
    assert torch.equal(o[0, C:2 * C], v[0, 17].unsqueeze(0).expand(C, D))
    sel = np.zeros((G, sched.C(K)), dtype=bool)
    for g, l in enumerate(lists):
        sel[g, l] = True
    want = token_sparse(to_np(q[0]), to_np(k[0]), to_np(v[0]), C, sel, rows=[2, 3])
    mx, mean = attn_errors(to_np(o[0])[2 * C:], want[2 * C:])
    assert mx <= MAX_ABS and mean <= MEAN_ABS, (mx, mean)
