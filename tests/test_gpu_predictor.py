"""GPU parity of the decision-scale predictor (a2/a3) and of the predictor -> mapping chain,
under the protocol of SURVEY.md §8(c): (iii) masses within 1e-4 relative of the fp64 oracle;
(i) strict: the oracle's selection rule applied to the GPU's own fp32 masses reproduces the GPU
selection bit for bit; (ii) end to end: the oracle's selection on fp64 masses agrees on every
decision whose margin exceeds 1e-4 relative, and the standard seeds have no ambiguous decision."""
import numpy as np
import pytest
import torch

from oracle.geometry import INFINITY_1K_SIDES, Schedule, ceil_div
from oracle.mapping import map_pattern
from oracle.predictor import block_mass, select_threshold, select_topk, sink_blocks
from synth import structured_qkv
from tests.helpers import EQ256, INF2B, TINY, bits_to_bool, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sv():
    import paper_2602_04361_b200 as m
    return m


def _struct(cfg, seed, bh, S):
    q, k, _ = structured_qkv(seed, cfg["sides"], S, S, 0, bh, cfg["D"], sink_scales=cfg["sink"])
    return q.cuda(), k.cuda()


def _select(mass_row, mode, k, tau, rows_u, nsb):
    sel = np.zeros(len(mass_row), dtype=bool)
    if mode == 0:
        sel[select_topk(mass_row, k)] = True
    else:
        sel[select_threshold(mass_row, tau, rows_u)] = True
    sel[:nsb] = True
    return sel


def _margins(mass_row, mode, k, tau, rows_u):
    """Relative margin of each decision (protocol ii)."""
    if mode == 0:
        srt = np.sort(mass_row)[::-1]
        if k >= len(srt):
            return np.full(len(mass_row), np.inf)
        kth, nxt = srt[k - 1], srt[k]
        gap = abs(kth - nxt) / max(abs(kth), 1e-30)
        amb = np.isclose(mass_row, kth, rtol=0, atol=0) | np.isclose(mass_row, nxt, rtol=0, atol=0)
        return np.where(amb, gap, np.inf)
    thr = tau * rows_u
    return np.abs(mass_row - thr) / max(thr, 1e-30)


SEED = 11  # standard seed; tests/test_predictor_seeds.py checks it is unambiguous
CASES = [
    (TINY, 16, 0, 1, 0.0), (TINY, 16, 1, 0, 0.02),
    (EQ256, 32, 0, 2, 0.0), (EQ256, 32, 1, 0, 0.05), (EQ256, 16, 0, 3, 0.0),
    (INF2B, 128, 0, 5, 0.0), (INF2B, 128, 1, 0, 0.015), (INF2B, 64, 0, 7, 0.0),
    # a single ragged query tile (64 rows) and a ragged last KV block at B in {64, 128}
    (EQ256, 64, 0, 2, 0.0), (EQ256, 128, 1, 0, 0.05),
]


@pytest.mark.parametrize("cfg,B,mode,k,tau", CASES)
def test_predictor_parity(sv, cfg, B, mode, k, tau):
    S, D = cfg["S"], cfg["D"]
    bh = min(cfg["bh"], 4)
    sched = Schedule(cfg["sides"])
    q, kc = _struct(cfg, SEED, bh, S)
    mask, mass = sv.predict_pattern(cfg["sides"], S, B, cfg["sink"], q, kc, mode, max(k, 1), tau)
    torch.cuda.synchronize()
    gq, gkv = ceil_div(sched.N(S), B), ceil_div(sched.C(S), B)
    got_sel = bits_to_bool(mask.cpu().numpy(), gkv)
    got_mass = mass.cpu().numpy().astype(np.float64)
    nsb = sink_blocks(sched, cfg["sink"], B)
    ambiguous = 0
    for b in range(bh):
        want_mass = block_mass(to_np(q[b]), to_np(kc[b]), sched, S, B)
        # (iii) masses
        rows = np.array([min((u + 1) * B, sched.N(S)) - u * B for u in range(gq)], dtype=float)
        err = np.abs(got_mass[b] - want_mass)
        assert (err <= 1e-4 * np.abs(want_mass) + 1e-7 * rows[:, None]).all(), err.max()
        for u in range(gq):
            # (i) strict: oracle rule on GPU fp32 masses
            strict = _select(got_mass[b, u].astype(np.float32).astype(np.float64), mode, k,
                             np.float32(tau), rows[u], nsb) if mode == 0 else None
            if mode == 1:
                thr = np.float32(tau) * np.float32(rows[u])
                strict = (got_mass[b, u].astype(np.float32) >= thr)
                strict[:nsb] = True
            assert (strict == got_sel[b, u]).all(), (b, u)
            # (ii) end to end against fp64 masses
            want = _select(want_mass[u], mode, k, tau, rows[u], nsb)
            marg = _margins(want_mass[u], mode, k, tau, rows[u])
            clear = marg > 1e-4
            clear[:nsb] = True
            ambiguous += int((~clear).sum())
            assert (want[clear] == got_sel[b, u][clear]).all(), (b, u)
    assert ambiguous == 0


def test_mass_rows_sum(sv):
    cfg = INF2B
    q, kc = _struct(cfg, 3, 2, cfg["S"])
    _, mass = sv.predict_pattern(cfg["sides"], cfg["S"], 128, 5, q, kc, 0, 5)
    torch.cuda.synchronize()
    s = mass.sum(-1).cpu().numpy()
    rows = np.array([128] * 12 + [64], dtype=float)
    assert np.abs(s - rows).max() < 1e-3


def test_topk_all_and_sink(sv):
    cfg = EQ256
    q, kc = _struct(cfg, 4, 2, cfg["S"])
    sched = Schedule(cfg["sides"])
    gkv = ceil_div(sched.C(cfg["S"]), 32)
    mask, _ = sv.predict_pattern(cfg["sides"], cfg["S"], 32, 3, q, kc, 0, 1000)
    torch.cuda.synchronize()
    assert bits_to_bool(mask.cpu().numpy(), gkv).all()
    mask, _ = sv.predict_pattern(cfg["sides"], cfg["S"], 32, 3, q, kc, 1, 0, 1e9)
    torch.cuda.synchronize()
    sel = bits_to_bool(mask.cpu().numpy(), gkv)
    nsb = sink_blocks(sched, 3, 32)
    assert sel[..., :nsb].all() and not sel[..., nsb:].any()


@pytest.mark.parametrize("cfg", [EQ256, INF2B], ids=["256eq", "2b"])
def test_predict_then_map(sv, cfg):
    """GPU predictor -> GPU map == oracle map of the GPU's source pattern (bit exact)."""
    S, K, B = cfg["S"], cfg["K"], cfg["B"]
    bh = 3
    sched = Schedule(cfg["sides"])
    q, kc = _struct(cfg, 5, bh, S)
    src, _ = sv.predict_pattern(cfg["sides"], S, B, cfg["sink"], q, kc, 0, 3)
    dst = sv.map_indices(cfg["sides"], S, K, B, cfg["sink"], src, 0)
    torch.cuda.synchronize()
    src_b = bits_to_bool(src.cpu().numpy(), ceil_div(sched.C(S), B))
    dst_b = bits_to_bool(dst.cpu().numpy(), ceil_div(sched.C(K), B))
    for b in range(bh):
        assert (dst_b[b] == map_pattern(src_b[b], sched, S, K, B, cfg["sink"], "footprint")).all()


@pytest.mark.parametrize("mode,k,tau", [(0, 5, 0.0), (1, 0, 0.015)])
def test_predictor_three_slots(sv, mode, k, tau):
    """The three-slot form (predictor.cu, used above two query tiles per SM): 24 (b,h) at the 2B
    decision scale = 312 tiles of 128 rows, so every CTA runs full three-slot rounds and the
    K stages are shared and not shared across slots (13 tiles per (b,h)).  Same protocol as
    test_predictor_parity: masses (iii) and the strict selection (i) on every unit."""
    cfg, B, bh = INF2B, 128, 24
    S = cfg["S"]
    sched = Schedule(cfg["sides"])
    q, kc = _struct(cfg, SEED, bh, S)
    mask, mass = sv.predict_pattern(cfg["sides"], S, B, cfg["sink"], q, kc, mode, max(k, 1), tau)
    torch.cuda.synchronize()
    gq, gkv = ceil_div(sched.N(S), B), ceil_div(sched.C(S), B)
    got_sel = bits_to_bool(mask.cpu().numpy(), gkv)
    got_mass = mass.cpu().numpy().astype(np.float64)
    nsb = sink_blocks(sched, cfg["sink"], B)
    rows = np.array([min((u + 1) * B, sched.N(S)) - u * B for u in range(gq)], dtype=float)
    for b in range(bh):
        want_mass = block_mass(to_np(q[b]), to_np(kc[b]), sched, S, B)
        err = np.abs(got_mass[b] - want_mass)
        assert (err <= 1e-4 * np.abs(want_mass) + 1e-7 * rows[:, None]).all(), (b, err.max())
        for u in range(gq):
            if mode == 0:
                strict = _select(got_mass[b, u].astype(np.float32).astype(np.float64), mode, k,
                                 tau, rows[u], nsb)
            else:
                strict = got_mass[b, u].astype(np.float32) >= np.float32(tau) * np.float32(rows[u])
                strict[:nsb] = True
            assert (strict == got_sel[b, u]).all(), (b, u)


@pytest.mark.parametrize("bh", [24, 4])
def test_predictor_deterministic_repeats(sv, bh):
    """Repeat runs are bit-identical (fixed-order reductions, no atomics): 24 (b,h) runs the
    three-slot form, 4 the two-slot form.  Five launches back to back also exercise the
    persistent pipelines' barrier phases across launches (a race would show as a mismatch)."""
    cfg = INF2B
    q, kc = _struct(cfg, SEED, bh, cfg["S"])
    runs = []
    for _ in range(5):
        mask, mass = sv.predict_pattern(cfg["sides"], cfg["S"], 128, cfg["sink"], q, kc, 0, 5, 0.0)
        runs.append((mask.clone(), mass.clone()))
    torch.cuda.synchronize()
    for mask, mass in runs[1:]:
        assert torch.equal(mask, runs[0][0])
        assert torch.equal(mass, runs[0][1])
