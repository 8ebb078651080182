"""GPU parity of NEXT(4), the compressed KV cache of CSLA layers (READING 23):
kept-row copy exact, compressed CSLA block mask bit-exact against the oracle, and block-sparse
attention over the compressed cache within the north-star tolerance of the oracle."""
import numpy as np
import pytest
import torch

from oracle.attention import block_sparse, merge_lists
from oracle.geometry import INFINITY_1K_SIDES, Schedule, ceil_div
from oracle.kv_compress import compress, compressed_local_block_mask, kept_index
from synth import kv_cache_iid, q_iid
from tests.helpers import MAX_ABS, MEAN_ABS, attn_errors, bits_to_bool, to_np

pytestmark = pytest.mark.gpu

CASES = [  # sides, K, B, sink, windows, bh, D
    ([1, 2, 4, 6, 8, 12, 16], 7, 32, 3, (7, 5, 3, 1, 1), 3, 128),
    (list(INFINITY_1K_SIDES), 13, 128, 5, (7, 5, 3, 1, 1), 2, 128),
    (list(INFINITY_1K_SIDES), 11, 64, 5, (7, 5, 3, 1, 1), 2, 128),
    ([1, 2, 4, 8, 16], 5, 16, 1, (3, 1), 2, 64),
    ([1, 2, 4, 6, 8, 12, 16], 7, 16, 0, (5, 0, 3), 2, 128),      # no sink, a masked gap scale
]
IDS = ["256eq", "infinity_K13", "infinity_K11_B64", "d64", "nosink_gap"]


@pytest.fixture(scope="module")
def sv():
    import paper_2602_04361_b200 as m
    return m


@pytest.mark.parametrize("sides,K,B,sink,windows,bh,D", CASES, ids=IDS)
def test_compressed_csla(sv, sides, K, B, sink, windows, bh, D):
    sched = Schedule(sides)
    q = q_iid(41, K, 0, bh, sched.N(K), D).cuda()
    k, v = kv_cache_iid(41, 0, bh, sched.C(K), D)
    k, v = k.cuda(), v.cuda()
    kept = sv.csla_kept_rows(sides, K, sink, windows)
    idx = kept_index(sched, K, sink, windows)
    assert kept == len(idx)
    kc = sv.compress_kv(sides, K, k, sink, windows)
    vc = sv.compress_kv(sides, K, v, sink, windows)
    mask = sv.local_mask_compressed(sides, K, B, sink, windows)
    g_q, g_kv = ceil_div(sched.N(K), B), ceil_div(kept, B)
    rp, ci, st = sv.build_block_lists(bh, g_q, g_kv, [(mask, True)])
    o = sv.block_sparse_attn_rows(sides, K, B, q, kc, vc, kept, rp, ci)
    torch.cuda.synchronize()
    assert st.item() == 0
    assert torch.equal(kc.cpu(), k.cpu()[:, torch.from_numpy(idx)])
    want_mask = compressed_local_block_mask(sched, K, B, sink, windows)
    assert np.array_equal(bits_to_bool(mask.cpu().numpy(), g_kv), want_mask)
    lists = merge_lists([want_mask])
    for b in range(bh):
        kb, vb = compress(to_np(k[b]), sched, K, sink, windows), compress(to_np(v[b]), sched, K, sink, windows)
        rows = None if sched.N(K) <= 1024 else [0, g_q // 2, g_q - 1]
        want = block_sparse(to_np(q[b]), kb, vb, kept, B, lists, rows=rows)
        sel = np.arange(sched.N(K)) if rows is None else \
            np.concatenate([np.arange(u * B, min((u + 1) * B, sched.N(K))) for u in rows])
        mx, mean = attn_errors(to_np(o[b])[sel], want[sel])
        assert mx <= MAX_ABS and mean <= MEAN_ABS, (b, mx, mean)
