"""GPU parity (bit exact) of the integer kernels through the C ABI: CSLA local mask (a1),
index mapping (a4), merge + compaction to CSR (a5)."""
import numpy as np
import pytest
import torch

from oracle.attention import merge_lists, to_csr
from oracle.csla import local_block_mask
from oracle.geometry import INFINITY_1K_SIDES, Schedule, ceil_div
from oracle.mapping import map_pattern
from tests.helpers import EQ256, INF2B, TINY, bits_to_bool, bool_to_bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sv():
    import paper_2602_04361_b200 as m
    return m


ABLATION = [(5, (5, 3, 1, 1, 1)), (5, (3, 3, 3, 1, 1)), (5, (7, 5, 3, 1, 1)), (5, (5, 5, 5, 1, 1)),
            (5, (9, 7, 5, 1, 1)), (5, (7, 7, 7, 1, 1)), (5, (11, 9, 7, 1, 1)), (6, (7, 5, 3, 1, 1)),
            (7, (7, 5, 3, 1, 1)), (8, (7, 5, 3, 1, 1)), (0, (7, 5, 3, 1, 1))]


@pytest.mark.parametrize("sink,windows", ABLATION)
def test_local_mask_ablation_rows(sv, sink, windows):
    sides = list(INFINITY_1K_SIDES)
    got = sv.local_mask(sides, 13, 128, sink, windows)
    torch.cuda.synchronize()
    want = local_block_mask(Schedule(sides), 13, 128, sink, windows)
    assert (bits_to_bool(got.cpu().numpy(), 83) == want).all()
    assert (got.cpu().numpy()[:, -1] >> (83 - 64) == 0).all()     # no bits beyond G_kv


@pytest.mark.parametrize("cfg", [TINY, EQ256, INF2B], ids=["tiny", "256eq", "2b"])
@pytest.mark.parametrize("B", [1, 16, 32, 64, 128])
def test_local_mask_configs(sv, cfg, B):
    sched = Schedule(cfg["sides"])
    for K in range(1, cfg["K"] + 1):
        if K < cfg["K"] - 2 and B > 1:
            continue
        sink = min(cfg["sink"], K)
        got = sv.local_mask(cfg["sides"], K, B, sink, cfg["windows"])
        torch.cuda.synchronize()
        want = local_block_mask(sched, K, B, sink, cfg["windows"])
        assert (bits_to_bool(got.cpu().numpy(), want.shape[1]) == want).all(), (K, B)


def test_local_mask_random_schedules(sv):
    rng = np.random.default_rng(0)
    for trial in range(12):
        n = int(rng.integers(2, 8))
        sides = sorted(int(x) for x in rng.integers(1, 14, size=n))
        K = n
        B = int(rng.choice([1, 3, 8, 16, 32]))
        windows = tuple(int(x) for x in rng.choice([0, 1, 3, 5, 7, 9], size=int(rng.integers(0, n + 1))))
        sink = int(rng.integers(0, K + 1))
        got = sv.local_mask(sides, K, B, sink, windows)
        torch.cuda.synchronize()
        want = local_block_mask(Schedule(sides), K, B, sink, windows)
        assert (bits_to_bool(got.cpu().numpy(), want.shape[1]) == want).all(), (sides, B, windows)


def _rand_src(sched, S, B, bh, density, seed):
    rng = np.random.default_rng(seed)
    return rng.random((bh, ceil_div(sched.N(S), B), ceil_div(sched.C(S), B))) < density


@pytest.mark.parametrize("mode", [0, 1], ids=["footprint", "point"])
@pytest.mark.parametrize("case", [
    dict(sides=[1, 2, 4, 8], S=3, K=4, B=4, sink=2),
    dict(sides=[1, 2, 4, 6, 8, 12, 16], S=5, K=7, B=32, sink=3),
    dict(sides=[1, 2, 4, 6, 8, 12, 16], S=7, K=7, B=16, sink=0),
    dict(sides=list(INFINITY_1K_SIDES), S=11, K=13, B=128, sink=5),
    dict(sides=list(INFINITY_1K_SIDES), S=11, K=12, B=64, sink=5),
    dict(sides=list(INFINITY_1K_SIDES), S=10, K=11, B=128, sink=5),
    dict(sides=list(INFINITY_1K_SIDES), S=9, K=13, B=1, sink=0),
])
def test_map_indices(sv, case, mode):
    sched = Schedule(case["sides"])
    S, K, B, bh = case["S"], case["K"], case["B"], 3
    src = _rand_src(sched, S, B, bh, 0.15 if B > 1 else 0.002, S * 100 + K)
    src_words = torch.from_numpy(bool_to_bits(src)).cuda()
    got = sv.map_indices(case["sides"], S, K, B, case["sink"], src_words, mode)
    torch.cuda.synchronize()
    gkv = ceil_div(sched.C(K), B)
    got = bits_to_bool(got.cpu().numpy(), gkv)
    for b in range(bh):
        want = map_pattern(src[b], sched, S, K, B, case["sink"], ["footprint", "point"][mode])
        assert (got[b] == want).all(), b


def test_build_lists(sv):
    rng = np.random.default_rng(5)
    bh, gq, gkv = 5, 9, 75
    a = rng.random((gq, gkv)) < 0.1                       # broadcast
    b = rng.random((bh, gq, gkv)) < 0.05
    a[:, 0] = True
    rp, ci, st = sv.build_block_lists(bh, gq, gkv, [(torch.from_numpy(bool_to_bits(a)).cuda(), True),
                                                    (torch.from_numpy(bool_to_bits(b)).cuda(), False)])
    torch.cuda.synchronize()
    assert st.item() == 0
    want_rp, want_ci = to_csr([l for x in range(bh) for l in merge_lists([a, b[x]])])
    assert (rp.cpu().numpy() == want_rp).all()
    assert (ci.cpu().numpy()[:want_rp[-1]] == want_ci).all()


def test_build_lists_many_rows(sv):
    rng = np.random.default_rng(6)
    bh, gq, gkv = 96, 32, 83
    m = rng.random((bh, gq, gkv)) < 0.2
    m[..., 3] = True
    rp, ci, st = sv.build_block_lists(bh, gq, gkv, [(torch.from_numpy(bool_to_bits(m)).cuda(), False)])
    torch.cuda.synchronize()
    want_rp, want_ci = to_csr([l for x in range(bh) for l in merge_lists([m[x]])])
    assert st.item() == 0
    assert (rp.cpu().numpy() == want_rp).all() and (ci.cpu().numpy()[:want_rp[-1]] == want_ci).all()


def test_build_lists_errors(sv):
    gq, gkv = 4, 40
    m = np.zeros((gq, gkv), dtype=bool)
    m[:, 1] = True
    m[2, :] = False                                       # empty row
    _, _, st = sv.build_block_lists(1, gq, gkv, [(torch.from_numpy(bool_to_bits(m)).cuda(), True)])
    torch.cuda.synchronize()
    assert st.item() == 5
    m[2, 1] = True
    _, _, st = sv.build_block_lists(1, gq, gkv, [(torch.from_numpy(bool_to_bits(m)).cuda(), True)],
                                    capacity=3)
    torch.cuda.synchronize()
    assert st.item() == 4
