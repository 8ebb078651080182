"""Pins for oracle/predictor.py (O4)."""
import itertools
import math

import numpy as np

from oracle.geometry import Schedule
from oracle.predictor import block_mass, predict_pattern, select_threshold, select_topk, sink_blocks
from synth import q_iid, kv_cache_iid

SCHED = Schedule([1, 2, 4, 6, 8, 12])      # C = 1, 5, 21, 57, 121, 265


def _inputs(S, D=16, seed=0):
    q = q_iid(seed, S, 0, 1, SCHED.N(S), D)[0].float().numpy()
    k, _ = kv_cache_iid(seed, 0, 1, SCHED.C(S), D)
    return q.astype(np.float64), k[0].double().numpy()


def test_mass_rows_sum_to_block_size():
    """sum_v mass[u, v] = |u|: softmax rows sum to one."""
    q, k = _inputs(6)
    for B in (1, 7, 16, 32, 144):
        m = block_mass(q, k, SCHED, 6, B)
        sizes = [min((u + 1) * B, 144) - u * B for u in range(m.shape[0])]
        assert np.allclose(m.sum(1), sizes, rtol=0, atol=1e-12)


def test_mass_bruteforce():
    """Brute-force double loop over (q, j) with an explicit per-element softmax."""
    q, k = _inputs(4, D=4)
    n_q, n_kv, B = 36, 57, 8
    m = block_mass(q, k, SCHED, 4, B)
    for u in range(m.shape[0]):
        for v in range(m.shape[1]):
            tot = 0.0
            for t in range(u * B, min((u + 1) * B, n_q)):
                z = [sum(q[t, d] * k[j, d] for d in range(4)) / 2.0 for j in range(n_kv)]
                mx = max(z)
                den = sum(math.exp(x - mx) for x in z)
                tot += sum(math.exp(z[j] - mx) / den for j in range(v * B, min((v + 1) * B, n_kv)))
            assert abs(tot - m[u, v]) < 1e-12


def test_topk_tie_rule():
    assert list(select_topk(np.array([0.1, 0.5, 0.5, 0.2]), 2)) == [1, 2]
    assert list(select_topk(np.array([0.5, 0.1, 0.5, 0.5]), 2)) == [0, 2]
    assert list(select_topk(np.array([1.0, 1.0, 1.0]), 1)) == [0]


def test_topk_against_subset_search():
    """Exhaustive: the selected set maximises the total mass, and among maximisers it is the
    lexicographically smallest index set (ties to smaller v)."""
    rng = np.random.default_rng(1)
    for trial in range(200):
        G = int(rng.integers(1, 8))
        row = rng.integers(0, 4, size=G).astype(float)      # many ties
        k = int(rng.integers(1, G + 1))
        best = max(itertools.combinations(range(G), k), key=lambda c: (sum(row[list(c)]),
                                                                        [-x for x in c]))
        assert list(select_topk(row, k)) == list(best)


def test_topk_all():
    q, k = _inputs(6)
    m = block_mass(q, k, SCHED, 6, 16)
    for u in range(m.shape[0]):
        assert list(select_topk(m[u], m.shape[1])) == list(range(m.shape[1]))


def test_threshold_inclusive():
    assert list(select_threshold(np.array([0.5, 0.25, 1.0]), 0.5, 1)) == [0, 2]
    assert list(select_threshold(np.array([8.0, 7.99]), 0.5, 16)) == [0]


def test_planted_dominant_key():
    """A key that dominates every query's attention is selected at k = 1."""
    q, k = _inputs(6)
    j_star = 200                                  # in block 200 // 16 = 12
    k = k.copy()
    k[j_star] = 50.0 * q.mean(0) / np.linalg.norm(q.mean(0))
    q = q + 3.0 * k[j_star] / np.linalg.norm(k[j_star])
    pat, mass = predict_pattern(q, k, SCHED, 6, 16, 0, "topk", 1)
    assert pat[:, 12].all() and (pat.sum(1) == 1).all()


def test_sink_union_after_selection():
    q, k = _inputs(6)
    pat, mass = predict_pattern(q, k, SCHED, 6, 16, 5, "topk", 1)
    nsb = sink_blocks(SCHED, 5, 16)
    assert nsb == 8                                # ceil(121 / 16)
    assert pat[:, :nsb].all()
    for u in range(pat.shape[0]):                  # the top-1 is still there
        assert pat[u, select_topk(mass[u], 1)[0]]
