"""GPU parity of NEXT(3), the sparsified multi-layer tail (paper_2602_04361_b200/step.py,
PAPER.md:983-990, 1227-1241), layer by layer against the fp64 oracle on the same bf16 inputs:
the decision scale is dense, CS4A layers use the predicted pattern mapped to every target scale
plus the upsampled cache residual, CSLA layers the local mask.  Masks bit-exact, outputs within
the north-star attention tolerance."""
import numpy as np
import pytest
import torch

from oracle.attention import block_sparse, dense, merge_lists
from oracle.cache import cache_residual, cached_sparse
from oracle.csla import local_block_mask
from oracle.geometry import Schedule
from oracle.mapping import map_pattern
from synth import kv_cache_iid, q_iid
from tests.helpers import EQ256, MAX_ABS, MEAN_ABS, attn_errors, bits_to_bool, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def step_mod():
    import paper_2602_04361_b200.step as m
    return m


def test_layer_split(step_mod):
    # 6:4 CS4A:CSLA; the CS4A layers are the shallowest
    assert step_mod.layer_split(10) == 6 and step_mod.layer_split(32) == 19
    assert step_mod.layer_split(3) == 2 and step_mod.layer_split(1) == 1


@pytest.mark.parametrize("fused", [True, False], ids=["fused_mass", "predictor"])
def test_sparsified_step_parity(step_mod, fused):
    layers = 3
    cfg = EQ256
    sides, S, K, B, D, sink = cfg["sides"], cfg["S"], cfg["K"], cfg["B"], cfg["D"], cfg["sink"]
    bh = 2
    sched = Schedule(sides)
    st = step_mod.SparsifiedStep(sides, S, K, B, bh, layers, head_dim=D, sink_scales=sink,
                                 windows=cfg["windows"], topk=2, fused=fused)
    assert [st.kind(l) for l in range(layers)] == ["cs4a", "cs4a", "csla"]
    qs = [{k: q_iid(100 + l, k, 0, bh, sched.N(k), D).cuda() for k in range(S, K + 1)}
          for l in range(layers)]
    kvs = [kv_cache_iid(100 + l, 0, bh, sched.C(K), D) for l in range(layers)]
    ks = [k.cuda() for k, _ in kvs]
    vs = [v.cuda() for _, v in kvs]
    outs = st.alloc_outputs()
    st.csla_patterns()
    for l in range(layers):
        st.layer(l, qs[l], ks[l], vs[l], outs[l])
        torch.cuda.synchronize()
        assert st.status.item() == 0
        src = bits_to_bool(st.src.cpu().numpy(), st.gS["G_kv"]) if st.kind(l) == "cs4a" else None
        mapped = {k: bits_to_bool(st.mapped[k].cpu().numpy(), st.g[k]["G_kv"]) for k in st.targets}
        for b in range(bh):
            qb = {k: to_np(qs[l][k][b]) for k in range(S, K + 1)}
            kb, vb = to_np(ks[l][b]), to_np(vs[l][b])
            mx, mean = attn_errors(to_np(outs[l][S][b]), dense(qb[S], kb, vb, sched.C(S)))
            assert mx <= MAX_ABS and mean <= MEAN_ABS, ("dense S", l, mx, mean)
            if st.kind(l) == "cs4a":
                lists_S = merge_lists([src[b]])
                want_oc = cache_residual(qb[S], kb, vb, sched.C(S), B, lists_S)
                got_oc = to_np(st.o_cache[b])
                mx, mean = attn_errors(got_oc, want_oc)
                assert mx <= MAX_ABS and mean <= MEAN_ABS, ("o_cache", l, mx, mean)
                for k in st.targets:
                    want_map = map_pattern(src[b], sched, S, k, B, sink, "footprint")
                    assert np.array_equal(mapped[k][b], want_map), ("mapped", l, k)
                    # the cached kernel's inputs include the bf16 O_cache: compared on the GPU's
                    # own O_cache, itself checked against the oracle above
                    want = cached_sparse(qb[k], kb, vb, sched.C(k), B, merge_lists([want_map]),
                                         got_oc, sides[S - 1], sides[k - 1])
                    mx, mean = attn_errors(to_np(outs[l][k][b]), want)
                    assert mx <= MAX_ABS and mean <= MEAN_ABS, ("cs4a", l, k, mx, mean)
            else:
                for k in st.targets:
                    local = local_block_mask(sched, k, B, sink, cfg["windows"])
                    got_local = bits_to_bool(st.local[k].cpu().numpy(), st.g[k]["G_kv"])
                    assert np.array_equal(got_local, local), ("local", k)
                    want = block_sparse(qb[k], kb, vb, sched.C(k), B, merge_lists([local]))
                    mx, mean = attn_errors(to_np(outs[l][k][b]), want)
                    assert mx <= MAX_ABS and mean <= MEAN_ABS, ("csla", l, k, mx, mean)


def test_run_matches_layerwise(step_mod):
    """run() (the benchmarked call) equals the layer-by-layer calls above bit for bit."""
    cfg = EQ256
    sides, S, K, B, D = cfg["sides"], cfg["S"], cfg["K"], cfg["B"], cfg["D"]
    bh, layers = 2, 2
    sched = Schedule(sides)
    st = step_mod.SparsifiedStep(sides, S, K, B, bh, layers, head_dim=D, sink_scales=cfg["sink"],
                                 topk=2)
    qs = [{k: q_iid(7 + l, k, 0, bh, sched.N(k), D).cuda() for k in range(S, K + 1)}
          for l in range(layers)]
    kvs = [kv_cache_iid(7 + l, 0, bh, sched.C(K), D) for l in range(layers)]
    ks, vs = [k.cuda() for k, _ in kvs], [v.cuda() for _, v in kvs]
    a = st.run(qs, ks, vs)
    b = st.alloc_outputs()
    st.csla_patterns()
    for l in range(layers):
        st.layer(l, qs[l], ks[l], vs[l], b[l])
    torch.cuda.synchronize()
    for l in range(layers):
        for k in a[l]:
            assert torch.equal(a[l][k], b[l][k]), (l, k)


def test_token_granularity_step(step_mod):
    """granularity='token': CS4A layers run the token path (NEXT(2)); every output of a 2-layer
    (CS4A + CSLA) step against the oracle's token path on the GPU's own selections."""
    from oracle.token_cs4a import map_tokens, token_cache_residual, token_cached_sparse
    cfg = EQ256
    sides, S, K, B, D, sink = cfg["sides"], cfg["S"], cfg["K"], cfg["B"], cfg["D"], cfg["sink"]
    bh, layers, C = 2, 2, 64
    sched = Schedule(sides)
    st = step_mod.SparsifiedStep(sides, S, K, B, bh, layers, head_dim=D, sink_scales=sink,
                                 windows=cfg["windows"], cs4a_fraction=0.5, granularity="token",
                                 query_block=C, alpha=0.2)
    qs = [{k: q_iid(50 + l, k, 0, bh, sched.N(k), D).cuda() for k in range(S, K + 1)}
          for l in range(layers)]
    kvs = [kv_cache_iid(50 + l, 0, bh, sched.C(K), D) for l in range(layers)]
    ks, vs = [k.cuda() for k, _ in kvs], [v.cuda() for _, v in kvs]
    outs = st.alloc_outputs()
    st.csla_patterns()
    st.layer(0, qs[0], ks[0], vs[0], outs[0])
    torch.cuda.synchronize()
    assert st.status.item() == 0
    sel = bits_to_bool(st.tsel.cpu().numpy(), sched.C(S))
    for b in range(bh):
        qb = {k: to_np(qs[0][k][b]) for k in range(S, K + 1)}
        kb, vb = to_np(ks[0][b]), to_np(vs[0][b])
        mx, mean = attn_errors(to_np(outs[0][S][b]), dense(qb[S], kb, vb, sched.C(S)))
        assert mx <= MAX_ABS and mean <= MEAN_ABS
        want_oc = token_cache_residual(qb[S], kb, vb, sched.C(S), C, sel[b])
        oc = to_np(st.o_cache[b])
        mx, mean = attn_errors(oc, want_oc)
        assert mx <= MAX_ABS and mean <= MEAN_ABS, ("o_cache", mx, mean)
        for k in st.targets:
            got_map = bits_to_bool(st.tmap[k].cpu().numpy(), sched.C(k))[b]
            want_map = map_tokens(sel[b], sched, S, k, C, sink)
            assert np.array_equal(got_map, want_map), k
            want = token_cached_sparse(qb[k], kb, vb, C, want_map, oc, sides[S - 1], sides[k - 1])
            mx, mean = attn_errors(to_np(outs[0][k][b]), want)
            assert mx <= MAX_ABS and mean <= MEAN_ABS, (k, mx, mean)
