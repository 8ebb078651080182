"""NEXT(4) measurement: CSLA attention over the compressed KV cache (sink + windowed scales,
PAPER.md:1170) against the full cache, bench workload shape (96 (b,h), K = 13, B = 128, default
windows), median CUDA-event time per launch.  One JSON line, appended to --out."""
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
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import paper_2602_04361_b200 as sv
    from synth import kv_cache_iid, q_iid
    K, B, D, bh, sink, win = 13, 128, 128, 96, 5, (7, 5, 3, 1, 1)
    dev = torch.device("cuda", 0)
    n_q, n_kv = SIDES[K - 1] ** 2, sum(s * s for s in SIDES[:K])
    q = q_iid(0, K, 0, bh, n_q, D, device=dev)
    k, v = kv_cache_iid(0, 0, bh, n_kv, D, device=dev)

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

    g_q = -(-n_q // B)
    full_mask = sv.local_mask(SIDES, K, B, sink, win)
    rpf, cif, st = sv.build_block_lists(bh, g_q, -(-n_kv // B), [(full_mask, True)])
    o = torch.empty_like(q)
    t_full = timed(lambda: sv.block_sparse_attn(SIDES, K, B, q, k, v, rpf, cif, o=o))
    kept = sv.csla_kept_rows(SIDES, K, sink, win)
    kc = sv.compress_kv(SIDES, K, k, sink, win)
    vc = sv.compress_kv(SIDES, K, v, sink, win)
    t_copy = timed(lambda: (sv.compress_kv(SIDES, K, k, sink, win, out=kc),
                            sv.compress_kv(SIDES, K, v, sink, win, out=vc)))
    cmask = sv.local_mask_compressed(SIDES, K, B, sink, win)
    rpc, cic, st2 = sv.build_block_lists(bh, g_q, -(-kept // B), [(cmask, True)])
    t_comp = timed(lambda: sv.block_sparse_attn_rows(SIDES, K, B, q, kc, vc, kept, rpc, cic, o=o))
    torch.cuda.synchronize()
    assert st.item() == 0 and st2.item() == 0
    nnz_f, nnz_c = int(rpf[-1].item()) // bh, int(rpc[-1].item()) // bh
    rec = {"metric": "CSLA attention over the compressed KV cache (NEXT 4) ms", "unit": "ms",
           "config": {"workload": "infinity8b_last_scale_kv_compressed", "units_bh": bh,
                      "target_scale": K, "block": B, "sink_scales": sink, "windows": list(win)},
           "kv_rows_full": n_kv, "kv_rows_compressed": kept,
           "kv_bytes_full": 2 * bh * n_kv * D * 2, "kv_bytes_compressed": 2 * bh * kept * D * 2,
           "blocks_per_head_full": nnz_f, "blocks_per_head_compressed": nnz_c,
           "csla_attn_full_ms": round(t_full, 4), "csla_attn_compressed_ms": round(t_comp, 4),
           "compress_copy_k_and_v_ms": round(t_copy, 4), "reps": args.reps}
    line = json.dumps(rec)
    print(line, flush=True)
    if args.out:
        with open(args.out, "a") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
