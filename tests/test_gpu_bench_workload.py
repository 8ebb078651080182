"""Parity at the bench workload itself (BASELINE configs[3], the 8B shape bench.py times: 4 x 24 =
96 (b,h), K = 13, S = 11, B = 128, top-5, CSLA + CS4A lists) in bench.py's launch configuration
(one SparseLayer over all 96 units), on the bench's own seeded inputs, checked on sampled units:
predictor masses within 1e-4 of fp64 and the selection rule bit-exact on the GPU's masses,
mapped masks and CSR lists bit-exact, attention rows within the north-star bound."""
import numpy as np
import pytest
import torch

from oracle.attention import block_sparse, merge_lists
from oracle.csla import local_block_mask
from oracle.geometry import INFINITY_1K_SIDES, Schedule, ceil_div
from oracle.mapping import map_pattern
from oracle.predictor import block_mass, select_topk, sink_blocks
from synth import kv_cache_iid, q_iid
from tests.helpers import MAX_ABS, MEAN_ABS, attn_errors, bits_to_bool, csr_lists, to_np

pytestmark = pytest.mark.gpu


def test_bench_workload_sampled_units():
    import paper_2602_04361_b200 as sv
    sides, K, S, B, D, units, sink, topk = list(INFINITY_1K_SIDES), 13, 11, 128, 128, 96, 5, 5
    sched = Schedule(sides)
    dev = torch.device("cuda", 0)
    q = q_iid(0, K, 0, units, sched.N(K), D, device=dev)
    qS = q_iid(0, S, 0, units, sched.N(S), D, device=dev)
    k, v = kv_cache_iid(0, 0, units, sched.C(K), D, device=dev)
    layer = sv.SparseLayer(sides, K, S, B, units, sink_scales=sink, kinds=("csla", "cs4a"), topk=topk)
    layer.build_patterns(qS, k)
    o_csla = layer.attend("csla", q, k, v)
    o_cs4a = layer.attend("cs4a", q, k, v)
    torch.cuda.synchronize()
    assert layer.status.item() == 0
    gS_q, gS_kv = ceil_div(sched.N(S), B), ceil_div(sched.C(S), B)
    gK_q, gK_kv = ceil_div(sched.N(K), B), ceil_div(sched.C(K), B)
    src = bits_to_bool(layer.src.cpu().numpy(), gS_kv)
    mapped = bits_to_bool(layer.mapped.cpu().numpy(), gK_kv)
    mass = layer.mass.cpu().numpy().astype(np.float64)
    local = local_block_mask(sched, K, B, sink, (7, 5, 3, 1, 1))
    csla_lists = csr_lists(*layer.lists["csla"], units * gK_q)
    cs4a_lists = csr_lists(*layer.lists["cs4a"], units * gK_q)
    nsb = sink_blocks(sched, sink, B)
    rows_u = [0, 13, gK_q - 1]
    for b in (0, 47, 95):
        kb, vb = to_np(k[b]), to_np(v[b])
        # predictor: masses (iii) and the selection rule on the GPU's own fp32 masses (i)
        want_mass = block_mass(to_np(qS[b]), kb, sched, S, B)
        rows = np.array([min((u + 1) * B, sched.N(S)) - u * B for u in range(gS_q)], dtype=float)
        assert (np.abs(mass[b] - want_mass) <= 1e-4 * np.abs(want_mass) + 1e-7 * rows[:, None]).all()
        for u in range(gS_q):
            sel = np.zeros(gS_kv, dtype=bool)
            sel[select_topk(mass[b, u].astype(np.float32).astype(np.float64), topk)] = True
            assert np.array_equal(sel, src[b, u]), (b, u)      # Top-K only at S (READING 25)
        # mapping and lists
        assert np.array_equal(mapped[b], map_pattern(src[b], sched, S, K, B, sink, "footprint"))
        assert mapped[b][:, :nsb].all()                        # A_sink U M(inds^(S))
        for u in range(gK_q):
            assert np.array_equal(csla_lists[b * gK_q + u], np.nonzero(local[u])[0])
            assert np.array_equal(cs4a_lists[b * gK_q + u], np.nonzero(mapped[b, u])[0])
        # attention on sampled query blocks
        sel_rows = np.concatenate([np.arange(u * B, min((u + 1) * B, sched.N(K))) for u in rows_u])
        for o, m in ((o_csla, [local[u] for u in range(gK_q)]), (o_cs4a, list(mapped[b]))):
            want = block_sparse(to_np(q[b]), kb, vb, sched.C(K), B, merge_lists([np.array(m)]),
                                rows=rows_u)
            mx, mean = attn_errors(to_np(o[b])[sel_rows], want[sel_rows])
            assert mx <= MAX_ABS and mean <= MEAN_ABS, (b, mx, mean)
