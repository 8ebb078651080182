"""Pins for oracle/cs4a.py: the order in which the CS4A pattern takes the sink (READING 25).

Paper-literal (default): inds^(S) = TopK only; the sink is added at the
target after the mapping, inds^(K) = A_sink U M(inds^(S)).
Alternative (`sink_in_source`): the sink OR-ed at S and mapped along with the Top-K."""
import numpy as np
import pytest

from oracle.cs4a import cs4a_patterns
from oracle.geometry import INFINITY_1K_SIDES, Schedule, ceil_div
from oracle.mapping import map_pattern
from oracle.predictor import sink_blocks
from oracle.token_cs4a import map_tokens
from synth import structured_qkv

INF = Schedule(INFINITY_1K_SIDES)
EQ = Schedule([1, 2, 4, 6, 8, 12, 16])


def test_empty_source_maps_to_exactly_the_sink():
    """A_sink U M(empty) = A_sink: at 11 -> 13, B = 128, sink <= 5 (C_5 = 121 tokens)
    every target row is exactly {0}."""
    src = np.zeros((ceil_div(INF.N(11), 128), ceil_div(INF.C(11), 128)), dtype=bool)
    dst = map_pattern(src, INF, 11, 13, 128, 5, "footprint")
    assert dst.shape == (32, 83)
    assert dst[:, 0].all() and not dst[:, 1:].any()


def test_sink_block_of_S_maps_to_blocks_0_to_4():
    """Worked by hand: source block 0 at S = 11 holds tokens 0..127 = scales 1..5 (121 tokens) and
    tokens 0..6 of row 0 of scale 6 (side 12).  Relative alignment l' = l + 2 sends scales 1..5 to
    scales 3..7, whose footprints tile them: tokens [C_2, C_7) = [5, 521).  Scale 6 row 0, cols
    0..6 goes to scale 8 (side 20): row [0, 20/12) = {0}, cols [0, floor(7*20/12)) = 0..10 ->
    tokens 521..531.  Blocks of 128: tokens 5..531 -> blocks 0..4 (plus the sink block 0)."""
    src = np.zeros((ceil_div(INF.N(11), 128), ceil_div(INF.C(11), 128)), dtype=bool)
    src[:, 0] = True
    dst = map_pattern(src, INF, 11, 13, 128, 5, "footprint")
    for g in range(dst.shape[0]):
        assert list(np.nonzero(dst[g])[0]) == [0, 1, 2, 3, 4]


@pytest.mark.parametrize("k", [1, 3])
def test_paper_order_S_pattern_is_topk_only(k):
    S, K, B, sink = 5, 7, 32, 3
    q, kc, _ = structured_qkv(2, EQ.sides, S, S, 0, 1, 32, sink_scales=sink)
    q, kc = q[0].double().numpy(), kc[0].double().numpy()
    src, dst, _ = cs4a_patterns(q, kc, EQ, S, K, B, sink, "topk", k)
    assert (src.sum(1) == k).all()                      # no sink forced in at S
    nsb = sink_blocks(EQ, sink, B)
    assert dst[:, :nsb].all()                            # the sink is present at the target
    src2, dst2, _ = cs4a_patterns(q, kc, EQ, S, K, B, sink, "topk", k, sink_in_source=True)
    assert src2[:, :nsb].all() and (src2 | ~src).all()


def test_compositions_differ_by_the_image_of_the_sink():
    """sink_in_source = paper-literal U M({sink blocks}): the mapping is a union over source
    blocks, so the two orders differ exactly by the sink blocks' image."""
    S, K, B, sink = 11, 13, 128, 5
    rng = np.random.default_rng(5)
    gq, gkv = ceil_div(INF.N(S), B), ceil_div(INF.C(S), B)
    topk = np.zeros((gq, gkv), dtype=bool)
    for u in range(gq):
        topk[u, rng.choice(np.arange(1, gkv), 5, replace=False)] = True
    paper = map_pattern(topk, INF, S, K, B, sink, "footprint")
    with_sink = topk.copy()
    with_sink[:, :sink_blocks(INF, sink, B)] = True
    alt = map_pattern(with_sink, INF, S, K, B, sink, "footprint")
    sink_only = np.zeros_like(topk)
    sink_only[:, 0] = True
    assert np.array_equal(alt, paper | map_pattern(sink_only, INF, S, K, B, sink, "footprint"))
    assert alt.sum() > paper.sum()


def test_token_path_sink_order():
    """Token granularity, the same two orders: an empty token selection maps to exactly the sink
    tokens j < C_5 = 121; the sink tokens of S = 11 (scales 1..5) map to scales 3..7, i.e. with
    the target sink the tokens [0, C_7) = [0, 521)."""
    C = 192
    G_S = ceil_div(INF.N(11), C)
    empty = np.zeros((G_S, INF.C(11)), dtype=bool)
    dst = map_tokens(empty, INF, 11, 13, C, 5)
    assert dst[:, :121].all() and not dst[:, 121:].any()
    sink_src = empty.copy()
    sink_src[:, :121] = True
    dst = map_tokens(sink_src, INF, 11, 13, C, 5)
    assert dst[:, :521].all() and not dst[:, 521:].any()
    assert INF.C(7) == 521
