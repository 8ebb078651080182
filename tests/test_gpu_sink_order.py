"""GPU parity of both CS4A sink compositions (DESIGN.md READING 25) on the whole
predictor -> map -> lists -> attention chain (SparseLayer) and on the O_cache step:

  paper-literal (default): inds^(S) = TopK only, inds^(K) = A_sink U M(inds^(S))
                           (PAPER.md:883-890), O_cache over TopK only;
  sink_in_source:          the sink OR-ed into the S-level pattern, then mapped.

The S-level selection is checked with the oracle's rule on the GPU's own fp32 masses (protocol
(i)); the mapped pattern, the CSR lists and the attention against the oracle's cs4a_patterns
composition of that selection."""
import numpy as np
import pytest
import torch

from oracle.attention import block_sparse, merge_lists
from oracle.cache import cache_residual, cached_sparse
from oracle.geometry import Schedule, ceil_div
from oracle.mapping import map_pattern
from oracle.predictor import select_topk, sink_blocks
from synth import kv_cache_iid, q_iid, structured_qkv
from tests.helpers import EQ256, INF2B, MAX_ABS, MEAN_ABS, attn_errors, bits_to_bool, csr_lists, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sv():
    import paper_2602_04361_b200 as m
    return m


@pytest.mark.parametrize("sink_in_source", [False, True], ids=["paper", "sink_in_source"])
@pytest.mark.parametrize("cfg", [EQ256, INF2B], ids=["256eq", "2b"])
def test_layer_chain(sv, cfg, sink_in_source):
    sides, S, K, B, D, sink = cfg["sides"], cfg["S"], cfg["K"], cfg["B"], cfg["D"], cfg["sink"]
    bh, topk = 2, 3
    sched = Schedule(sides)
    qS, kS, _ = structured_qkv(21, sides, S, S, 0, bh, D, sink_scales=sink)
    q = q_iid(21, K, 0, bh, sched.N(K), D).cuda()
    k, v = kv_cache_iid(21, 0, bh, sched.C(K), D)
    k[:, :sched.C(S)] = kS
    k, v, qS = k.cuda(), v.cuda(), qS.cuda()
    layer = sv.SparseLayer(sides, K, S, B, bh, sink_scales=sink, windows=cfg["windows"],
                           kinds=("cs4a",), topk=topk, sink_in_source=sink_in_source)
    layer.build_patterns(qS, k)
    o = layer.attend("cs4a", q, k, v)
    torch.cuda.synchronize()
    assert layer.status.item() == 0
    gS_q, gS_kv = ceil_div(sched.N(S), B), ceil_div(sched.C(S), B)
    gK_q, gK_kv = ceil_div(sched.N(K), B), ceil_div(sched.C(K), B)
    src = bits_to_bool(layer.src.cpu().numpy(), gS_kv)
    mapped = bits_to_bool(layer.mapped.cpu().numpy(), gK_kv)
    mass = layer.mass.cpu().numpy()
    lists = csr_lists(*layer.lists["cs4a"], bh * gK_q)
    nsb = sink_blocks(sched, sink, B)
    for b in range(bh):
        for u in range(gS_q):
            want = np.zeros(gS_kv, dtype=bool)
            want[select_topk(mass[b, u].astype(np.float32).astype(np.float64), topk)] = True
            if sink_in_source:
                want[:nsb] = True
            assert np.array_equal(src[b, u], want), (b, u)
        if not sink_in_source:
            assert (src[b].sum(1) == topk).all()
        want_map = map_pattern(src[b], sched, S, K, B, sink, "footprint")
        assert np.array_equal(mapped[b], want_map)
        assert mapped[b][:, :nsb].all()
        for u in range(gK_q):
            assert np.array_equal(lists[b * gK_q + u], np.nonzero(want_map[u])[0])
        rows_u = [0, gK_q // 2, gK_q - 1]
        sel = np.concatenate([np.arange(u * B, min((u + 1) * B, sched.N(K))) for u in rows_u])
        want_o = block_sparse(to_np(q[b]), to_np(k[b]), to_np(v[b]), sched.C(K), B,
                              merge_lists([want_map]), rows=rows_u)
        mx, mean = attn_errors(to_np(o[b])[sel], want_o[sel])
        assert mx <= MAX_ABS and mean <= MEAN_ABS, (b, mx, mean)


def test_paper_order_is_sparser(sv):
    """At the 2B shape the sink_in_source composition attends a superset of the paper's blocks
    (the sink block's footprint, PAPER.md:883-890 vs READING 25's alternative)."""
    cfg = INF2B
    sides, S, K, B, D, sink = cfg["sides"], cfg["S"], cfg["K"], cfg["B"], cfg["D"], cfg["sink"]
    bh = 2
    sched = Schedule(sides)
    qS = q_iid(0, S, 0, bh, sched.N(S), D).cuda()
    k, _ = kv_cache_iid(0, 0, bh, sched.C(K), D)
    k = k.cuda()
    masks = {}
    for sis in (False, True):
        layer = sv.SparseLayer(sides, K, S, B, bh, sink_scales=sink, kinds=("cs4a",), topk=5,
                               sink_in_source=sis)
        layer.build_patterns(qS, k)
        torch.cuda.synchronize()
        masks[sis] = bits_to_bool(layer.mapped.cpu().numpy(), ceil_div(sched.C(K), B))
    assert (masks[True] | ~masks[False]).all()
    assert masks[True].sum() > masks[False].sum()


@pytest.mark.parametrize("sink_in_source", [False, True], ids=["paper", "sink_in_source"])
def test_step_cache_both_orders(sink_in_source):
    """O_cache at S over the S-level pattern of each composition and the
    cached CS4A outputs at K, through SparsifiedStep (one CS4A layer)."""
    import paper_2602_04361_b200.step as step_mod
    cfg = EQ256
    sides, S, K, B, D, sink = cfg["sides"], cfg["S"], cfg["K"], cfg["B"], cfg["D"], cfg["sink"]
    bh = 2
    sched = Schedule(sides)
    st = step_mod.SparsifiedStep(sides, S, K, B, bh, 1, head_dim=D, sink_scales=sink,
                                 windows=cfg["windows"], topk=2, cs4a_fraction=1.0,
                                 sink_in_source=sink_in_source)
    qs = {k: q_iid(3, k, 0, bh, sched.N(k), D).cuda() for k in range(S, K + 1)}
    kc, vc = kv_cache_iid(3, 0, bh, sched.C(K), D)
    kc, vc = kc.cuda(), vc.cuda()
    out = st.alloc_outputs()[0]
    st.layer(0, qs, kc, vc, out)
    torch.cuda.synchronize()
    assert st.status.item() == 0
    src = bits_to_bool(st.src.cpu().numpy(), st.gS["G_kv"])
    nsb = sink_blocks(sched, sink, B)
    for b in range(bh):
        if sink_in_source:
            assert src[b][:, :nsb].all()
        else:
            assert (src[b].sum(1) == 2).all()
        qb = {k: to_np(qs[k][b]) for k in range(S, K + 1)}
        kb, vb = to_np(kc[b]), to_np(vc[b])
        want_oc = cache_residual(qb[S], kb, vb, sched.C(S), B, merge_lists([src[b]]))
        oc = to_np(st.o_cache[b])          # the cached kernel's own (bf16) input, checked here
        mx, mean = attn_errors(oc, want_oc)
        assert mx <= MAX_ABS and mean <= MEAN_ABS, ("o_cache", mx, mean)
        for k in st.targets:
            want_map = map_pattern(src[b], sched, S, k, B, sink, "footprint")
            got_map = bits_to_bool(st.mapped[k].cpu().numpy(), st.g[k]["G_kv"])[b]
            assert np.array_equal(got_map, want_map), k
            want = cached_sparse(qb[k], kb, vb, sched.C(k), B, merge_lists([want_map]), oc,
                                 sides[S - 1], sides[k - 1])
            mx, mean = attn_errors(to_np(out[k][b]), want)
            assert mx <= MAX_ABS and mean <= MEAN_ABS, (k, mx, mean)
