"""NEXT(3) benchmark: the sparsified attention tail of one generation step across all layers
(paper_2602_04361_b200/step.py), Infinity-2B shape: 32 layers x 16 heads, D=128, schedule to
64x64, decision scale S=11, targets 12 and 13, B=128, CS4A:CSLA = 6:4 with CS4A on
the shallowest layers, top-5 blocks per query block at S, the predictor
fused into the decision scale's dense pass (sparvar_dense_attn_mass; the unfused variant is
timed beside it).  Synthetic
seeded iid bf16 Q/K/V per layer (no weights: attention only; QKV projections, FFN and the rest
of the transformer are outside the hot path).  Inputs (1.0 GB of Q + 2.8 GB of K/V) exceed L2.

Timed on the device with CUDA events, W warm-up steps, median of K steps; the dense denominator
is the same scales with the build's own dense kernel.  Prints one JSON line (also appended to
--out).
    python scripts/step_bench.py [--layers 32] [--steps 10] [--warmup 3] [--out profiles/r01_step.jsonl]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

SIDES = [1, 2, 4, 6, 8, 12, 16, 20, 24, 32, 40, 48, 64]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    import paper_2602_04361_b200.step as step
    from synth import kv_cache_iid, q_iid

    S, K, B, D, bh, L = 11, 13, 128, 128, args.heads, args.layers
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    n_kv = sum(s * s for s in SIDES[:K])
    qs, ks, vs = [], [], []
    for l in range(L):
        qs.append({k: q_iid(1000 + l, k, 0, bh, SIDES[k - 1] ** 2, D, device=dev)
                   for k in range(S, K + 1)})
        k_, v_ = kv_cache_iid(1000 + l, 0, bh, n_kv, D, device=dev)
        ks.append(k_)
        vs.append(v_)
    st = step.SparsifiedStep(SIDES, S, K, B, bh, L, head_dim=D, topk=5)
    outs = st.alloc_outputs()

    def timed(fn, n):
        ts = []
        for _ in range(n):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    for _ in range(args.warmup):
        st.run(qs, ks, vs, outs)
    torch.cuda.synchronize()
    assert st.status.item() == 0
    sparse_ms = timed(lambda: st.run(qs, ks, vs, outs), args.steps)
    for _ in range(max(1, args.warmup // 2)):
        st.run_dense(qs, ks, vs, outs)
    dense_ms = timed(lambda: st.run_dense(qs, ks, vs, outs), max(3, args.steps // 2))

    # the same step captured once into a CUDA graph and replayed (no per-call host work: the
    # library's host side is validation and tensor-map encoding, done at capture)
    graph_ms = None
    try:
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            st.run(qs, ks, vs, outs)            # warm the lazily set kernel attributes
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            st.run(qs, ks, vs, outs)
        g.replay()
        torch.cuda.synchronize()
        graph_ms = timed(lambda: g.replay(), args.steps)
    except Exception as e:  # reported, not fatal
        graph_ms = f"capture failed: {e}"

    # the unfused variant: dense attention at S plus the stand-alone predictor
    st_u = step.SparsifiedStep(SIDES, S, K, B, bh, L, head_dim=D, topk=5, fused=False)
    for _ in range(args.warmup):
        st_u.run(qs, ks, vs, outs)
    unfused_ms = timed(lambda: st_u.run(qs, ks, vs, outs), args.steps)

    # CS4A layers at the paper's token granularity (NEXT(2): C = 192, alpha = 0.2)
    st_t = step.SparsifiedStep(SIDES, S, K, B, bh, L, head_dim=D, topk=5, granularity="token",
                               query_block=192, alpha=0.2)
    for _ in range(args.warmup):
        st_t.run(qs, ks, vs, outs)
    torch.cuda.synchronize()
    assert st_t.status.item() == 0
    token_ms = timed(lambda: st_t.run(qs, ks, vs, outs), args.steps)

    # per layer kind (one layer of each, repeated), for the breakdown
    st.csla_patterns()
    lay = {}
    for kind, l in (("cs4a", 0), ("csla", L - 1)):
        lay[kind] = timed(lambda: st.layer(l, qs[l], ks[l], vs[l], outs[l]), args.steps)
    rec = {"metric": "sparsified attention tail of one generation step (scales 11-13, all layers) ms",
           "value": round(sparse_ms, 4), "unit": "ms/step", "higher_is_better": False,
           "dense_ms": round(dense_ms, 4), "speedup_vs_dense": round(dense_ms / sparse_ms, 3),
           "unfused_predictor_ms": round(unfused_ms, 4),
           "token_granularity_ms": round(token_ms, 4),
           "graph_replay_ms": graph_ms if not isinstance(graph_ms, float) else round(graph_ms, 4),
           "layers": L, "cs4a_layers": st.n_cs4a, "csla_layers": L - st.n_cs4a,
           "cs4a_layer_ms": round(lay["cs4a"], 4), "csla_layer_ms": round(lay["csla"], 4),
           "config": {"workload": "infinity2b_sparsified_tail", "heads": bh, "head_dim": D,
                      "decision_scale": S, "targets": [12, 13], "block": B, "topk": 5,
                      "sink_scales": 5, "windows": [7, 5, 3, 1, 1], "split": "6:4 CS4A:CSLA",
                      "data": "synthetic seeded iid bf16 per layer", "l2": "inputs > L2"},
           "dtype": "bf16", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup}
    line = json.dumps(rec)
    print(line, flush=True)
    if args.out:
        with open(args.out, "a") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
