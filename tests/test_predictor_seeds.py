"""CPU check of the predictor parity protocol's precondition (SURVEY.md §8c protocol (ii)):
on the standard seeds and (k, tau) values of tests/test_gpu_predictor.py, the fp64 oracle's
selection has no decision within 1e-4 relative of its boundary, so the GPU's fp32 selection is
required to match it everywhere.  Uses the oracle only (no GPU, no CUDA path)."""
import numpy as np
import pytest

from oracle.geometry import Schedule, ceil_div
from oracle.predictor import block_mass
from synth import structured_qkv
from tests.test_gpu_predictor import CASES, SEED, _margins


@pytest.mark.parametrize("cfg,B,mode,k,tau", CASES)
def test_standard_seed_has_no_ambiguous_decision(cfg, B, mode, k, tau):
    S = cfg["S"]
    bh = min(cfg["bh"], 4)
    sched = Schedule(cfg["sides"])
    q, kc, _ = structured_qkv(SEED, cfg["sides"], S, S, 0, bh, cfg["D"], sink_scales=cfg["sink"])
    gq = ceil_div(sched.N(S), B)
    rows = [min((u + 1) * B, sched.N(S)) - u * B for u in range(gq)]
    n_sb = ceil_div(sched.C(cfg["sink"]), B)
    for b in range(bh):
        m = block_mass(q[b].double().numpy(), kc[b].double().numpy(), sched, S, B)
        for u in range(gq):
            marg = _margins(m[u], mode, k, tau, rows[u])
            assert (marg[n_sb:] > 1e-4).all(), (b, u, float(marg[n_sb:].min()))
