"""NEXT(2) measurement: token-granular CS4A at the bench workload's shape (Infinity-1K, 4 x 24 =
96 (b,h) units, D=128, S=11 -> K=13), query blocks of C=192 rows, top-k of
alpha=0.2 of the keys per block, sink scales <= 5.  Each kernel is timed alone
with CUDA events (median of --reps launches after warm-up) on seeded iid bf16 inputs; FLOPs are
counted per launch (colsum: the K Q^T products; token attention: 4 D x rows x listed tokens,
executed = padded to 128-row tiles and 128-token chunks).  One JSON line, appended to --out.
    python scripts/token_bench.py [--reps 20] [--out profiles/r01_token.jsonl]
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
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--bh", type=int, default=96)
    ap.add_argument("--C", type=int, default=192)
    ap.add_argument("--alpha", type=float, default=0.2)
    ap.add_argument("--out", default=None)
    ap.add_argument("--sink-in-source", action="store_true",
                    help="OR the sink tokens into the S-level selection (READING 25's alternative)")
    args = ap.parse_args()
    import paper_2602_04361_b200 as sv
    from synth import kv_cache_iid, q_iid

    S, K, D, bh, C, sink = 11, 13, 128, args.bh, args.C, 5
    dev = torch.device("cuda", 0)
    NS, NK = SIDES[S - 1] ** 2, SIDES[K - 1] ** 2
    CS, CK = sum(s * s for s in SIDES[:S]), sum(s * s for s in SIDES[:K])
    qS = q_iid(0, S, 0, bh, NS, D, device=dev)
    qK = q_iid(0, K, 0, bh, NK, D, device=dev)
    k, v = kv_cache_iid(0, 0, bh, CK, D, device=dev)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    peak = peaks["bf16_tflops"]

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    lse = torch.empty((bh, NS), dtype=torch.float32, device=dev)
    oS = torch.empty_like(qS)
    t_dense_S = timed(lambda: sv.dense_attn(SIDES, S, qS, k, v, o=oS, lse=lse))
    G_S, G_K = -(-NS // C), -(-NK // C)
    cs = torch.empty((bh, G_S, CS), dtype=torch.float32, device=dev)
    t_col = timed(lambda: sv.token_colsum(SIDES, S, C, qS, k, lse, out=cs))
    import math
    k_tok = max(1, math.ceil(args.alpha * CS))
    sel = torch.empty((bh, G_S, -(-CS // 32)), dtype=torch.int32, device=dev)
    sink_S = sink if args.sink_in_source else 0          # READING 25: paper order by default
    t_sel = timed(lambda: sv.token_select(SIDES, S, C, sink_S, cs, k_tok, out=sel))
    dst = torch.empty((bh, G_K, -(-CK // 32)), dtype=torch.int32, device=dev)
    t_map = timed(lambda: sv.token_map(SIDES, S, K, C, sink, sel, out=dst))
    cap = bh * G_K * CK
    rp = torch.empty(bh * G_K + 1, dtype=torch.int32, device=dev)
    ci = torch.empty(cap, dtype=torch.int32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    t_lists = timed(lambda: sv.build_block_lists(bh, G_K, CK, [(dst, False)], cap, rp, ci, status))
    o = torch.empty_like(qK)
    t_attn = timed(lambda: sv.token_sparse_attn(SIDES, K, C, qK, k, v, rp, ci, o=o))
    torch.cuda.synchronize()
    assert status.item() == 0
    counts = (rp[1:] - rp[:-1]).view(bh, G_K).double().cpu()
    rows = torch.tensor([min((g + 1) * C, NK) - g * C for g in range(G_K)], dtype=torch.float64)
    subs = -(-C // 128)
    algo = 4.0 * D * float((counts * rows).sum())
    executed = 4.0 * D * 128 * subs * float((torch.ceil(counts / 128) * 128).sum())
    col_flops = 2.0 * D * bh * G_S * C * (-(-CS // 128) * 128)
    t_dense_K = timed(lambda: sv.dense_attn(SIDES, K, qK, k, v, o=o))
    rec = {
        "metric": "token-granular CS4A (NEXT 2) per-kernel ms", "unit": "ms",
        "config": {"workload": "infinity8b_shape_token_cs4a", "units_bh": bh, "decision_scale": S,
                   "target_scale": K, "query_block_C": C, "alpha": args.alpha, "topk_tokens": k_tok,
                   "sink_scales": sink, "head_dim": D, "data": "synthetic seeded iid bf16",
                   "sink_order": "sink_in_source" if args.sink_in_source else "paper"},
        "dense_attn_S_with_lse_ms": round(t_dense_S, 4),
        "colsum_ms": round(t_col, 4), "colsum_tflops": round(col_flops / t_col / 1e9, 1),
        "colsum_gexp_per_s": round(bh * NS * CS / t_col / 1e6, 1),
        "select_ms": round(t_sel, 4), "map_ms": round(t_map, 4), "lists_ms": round(t_lists, 4),
        "token_attn_ms": round(t_attn, 4),
        "tokens_per_query_block": round(float(counts.mean()), 1),
        "token_density": round(float(counts.mean()) / CK, 4),
        "token_attn_tflops_executed": round(executed / t_attn / 1e9, 1),
        "token_attn_tensor_util_executed": round(executed / t_attn / 1e9 / peak, 4),
        "token_attn_tflops_algorithmic": round(algo / t_attn / 1e9, 1),
        "dense_attn_K_ms": round(t_dense_K, 4),
        "speedup_vs_dense": round(t_dense_K / t_attn, 3),
        "peak_tflops": peak, "reps": args.reps,
    }
    line = json.dumps(rec)
    print(line, flush=True)
    if args.out:
        with open(args.out, "a") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
