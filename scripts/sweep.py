"""Sparsity sweep, SURVEY.md §8(d) "Sweep (config 5)": the scale-skip combo (last scale only,
K=11 with decision scale S=10) and the K=13 last scale, on `structured` synthetic inputs
(DESIGN.md §4), Infinity-2B shape (1 x 16 heads, D=128).

Points:
  * CSLA window rows of Table csla_ablation: (a,b,c) on scales 11,12,13,
    scales 9,10 window 1, 6-8 masked; sink <= 5, 6, 7, 8 and none.
  * Predictor (CS4A lists: sink + mapped, the paper's sink order) top-k in {2,3,5,7,10} and tau in
    {0.005,0.01,0.02,0.05} at S=11 -> K=13 and S=10 -> K=11.
  * Block size B in {64, 128}.
Each point reports the attention ms (CUDA events, median), listed and executed FLOPs, tensor
utilisation on executed FLOPs against MEASURED_PEAKS.json, and the method error of the
block-sparse output against the build's own dense kernel (relative Frobenius, max abs).  Kernel
parity against the fp64 oracle is the tests' job (tests/test_gpu_*.py); this script does not
touch oracle/.

    python scripts/sweep.py [--reps 20] [--out profiles/r01_sweep.jsonl]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

SIDES = [1, 2, 4, 6, 8, 12, 16, 20, 24, 32, 40, 48, 64]   # Infinity 1024x1024
D = 128
HEADS = 16
WINDOW_ROWS = [(1, 3, 5), (3, 3, 3), (3, 5, 7), (5, 5, 5), (5, 7, 9), (7, 7, 7), (7, 9, 11)]
SINKS = [5, 6, 7, 8, 0]
TOPKS = [2, 3, 5, 7, 10]
TAUS = [0.005, 0.01, 0.02, 0.05]


def windows_of(row):
    """(a,b,c) on scales 11,12,13 -> the ABI's window vector relative to K=13 (index 0 = K)."""
    a, b, c = row
    return (c, b, a, 1, 1)


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def executed_steps(row_ptr, col_idx, bh, g_q, B):
    """KV steps the kernel executes: per 128-row tile, the union of its G = 128/B blocks' lists."""
    rp = row_ptr.cpu().numpy()
    ci = col_idx.cpu().numpy()
    G = max(1, 128 // B)
    steps = 0
    for b in range(bh):
        for t0 in range(0, g_q, G):
            s = set()
            for u in range(t0, min(t0 + G, g_q)):
                r = b * g_q + u
                s.update(ci[rp[r]:rp[r + 1]].tolist())
            steps += len(s)
    return steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.jsonl"))
    ap.add_argument("--quick", action="store_true", help="a few points only (smoke)")
    args = ap.parse_args()

    import paper_2602_04361_b200 as sv
    from synth import structured_qkv

    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    peak = peaks["bf16_tflops"]           # kernels timed alone: the burst peak
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)

    # one structured input set: K/V cache over all 13 scales, queries of scales 10, 11 and 13
    _, k, v = structured_qkv(args.seed, SIDES, 13, 13, 0, HEADS, D, device=dev)
    q_of = {s: structured_qkv(args.seed, SIDES, s, 13, 0, HEADS, D, device=dev)[0].contiguous()
            for s in (10, 11, 13)}
    k, v = k.contiguous(), v.contiguous()

    dense_cache = {}

    def dense_out(K):
        if K not in dense_cache:
            n_kv = sum(s * s for s in SIDES[:K])
            o = sv.dense_attn(SIDES, K, q_of[K], k, v)
            ms = timed(lambda: sv.dense_attn(SIDES, K, q_of[K], k, v, o=o), args.reps)
            dense_cache[K] = (o.float(), ms, 4.0 * D * q_of[K].shape[1] * n_kv * HEADS)
        return dense_cache[K]

    out = open(args.out, "w")
    rows = []

    def point(kind, K, B, masks, extra, lists_tag=None):
        g = sv.geometry(SIDES, K, B)
        rp, ci, st = sv.build_block_lists(HEADS, g["G_q"], g["G_kv"], masks)
        torch.cuda.synchronize()
        assert st.item() == 0, f"list status {st.item()}"
        nnz = int(rp[-1].item())
        q = q_of[K]
        o = sv.block_sparse_attn(SIDES, K, B, q, k, v, rp, ci)
        ms = timed(lambda: sv.block_sparse_attn(SIDES, K, B, q, k, v, rp, ci, o=o), args.reps)
        od, dms, dflops = dense_out(K)
        diff = o.float() - od
        rel_f = (torch.linalg.norm(diff) / torch.linalg.norm(od)).item()
        max_abs = diff.abs().max().item()
        ex_steps = executed_steps(rp, ci, HEADS, g["G_q"], B)
        listed = 4.0 * D * B * B * nnz
        executed = 4.0 * D * 128 * B * ex_steps
        rec = {"kind": kind, "K": K, "B": B, **extra,
               "active_blocks_per_head": nnz / HEADS,
               "grid_density": nnz / (HEADS * g["G_q"] * g["G_kv"]),
               "flex_sparsity": 1.0 - nnz * B * B / (HEADS * g["N"] * g["C"]),
               "ms": round(ms, 4), "dense_ms": round(dms, 4), "speedup_vs_dense": round(dms / ms, 3),
               "listed_gflop": round(listed / 1e9, 2), "executed_gflop": round(executed / 1e9, 2),
               "tflops_executed": round(executed / ms / 1e9, 1),
               "tensor_util_executed": round(executed / ms / 1e9 / peak, 4),
               "err_rel_fro_vs_dense": rel_f, "err_max_abs_vs_dense": max_abs}
        out.write(json.dumps(rec) + "\n")
        out.flush()
        rows.append(rec)
        print(json.dumps(rec), flush=True)
        return o, rp, ci

    blocks = (128,) if args.quick else (128, 64)
    for B in blocks:
        # ---- K=13 CSLA: window rows (sink <= 5) and sink rows (default windows)
        combos = [(r, 5) for r in WINDOW_ROWS] + [((3, 5, 7), s) for s in SINKS if s != 5]
        if args.quick:
            combos = [((3, 5, 7), 5)]
        for wr, sink in combos:
            local = sv.local_mask(SIDES, 13, B, sink, windows_of(wr))
            point("csla", 13, B, [(local, True)],
                  {"windows_11_12_13": list(wr), "sink_scales": sink})
        # ---- predictor (CS4A lists = sink + mapped) at S=11 -> K=13 and S=10 -> K=11 (skip)
        for S, K in ((11, 13), (10, 11)):
            gS = sv.geometry(SIDES, S, B)
            qS = q_of[S]
            sels = [("topk", kk) for kk in TOPKS] + [("threshold", t) for t in TAUS]
            if args.quick:
                sels = [("topk", 5)]
            for mode, val in sels:
                # READING 25: Top-K alone at S, the sink added by the map at K
                src, _ = sv.predict_pattern(SIDES, S, B, 0, qS, k,
                                            sv.SELECT_TOPK if mode == "topk" else sv.SELECT_THRESHOLD,
                                            topk=int(val) if mode == "topk" else 1,
                                            threshold=float(val) if mode == "threshold" else 0.0)
                mapped = sv.map_indices(SIDES, S, K, B, 5, src)
                point("cs4a", K, B, [(mapped, False)],
                      {"decision_scale": S, "select": mode, "value": val,
                       "src_blocks_per_head": int(sv.unpack_bits(src, gS["G_kv"]).sum().item()) / HEADS})
                if mode == "topk" and val == 5:
                    # the union policy (READING 19) at the same point
                    local = sv.local_mask(SIDES, K, B, 5, (7, 5, 3, 1, 1))
                    point("union", K, B, [(local, True), (mapped, False)],
                          {"decision_scale": S, "select": mode, "value": val})
        # ---- skip combo CSLA (K=11, relative windows (7,5,3,1,1))
        local = sv.local_mask(SIDES, 11, B, 5, (7, 5, 3, 1, 1))
        point("csla", 11, B, [(local, True)], {"windows_rel": [7, 5, 3, 1, 1], "sink_scales": 5})
    out.close()
    print(f"wrote {len(rows)} points to {args.out}")


if __name__ == "__main__":
    main()
