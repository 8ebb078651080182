"""Run every kernel of libsparvar.so once at a small configuration, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck), SURVEY.md:292, 301.

    compute-sanitizer --tool memcheck python scripts/sanitize.py tiny|256eq [kernel ...]

Kernels: mask, predict, map, lists, sparse, dense, mass, cached, rows, colsum, token_sel,
token_map, token_attn, token_cached.  Default: all.  No output checking here (the parity tests do
that); the point is the sanitizer's report on the same launch configurations.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2602_04361_b200 as sv  # noqa: E402
from synth import kv_cache_iid, q_iid, structured_qkv  # noqa: E402

CFGS = {
    "tiny": dict(sides=[1, 2, 4, 8], K=4, S=3, B=16, D=64, bh=2, sink=2, windows=(3, 3), C=16),
    "256eq": dict(sides=[1, 2, 4, 6, 8, 12, 16], K=7, S=5, B=32, D=128, bh=3, sink=3,
                  windows=(7, 5, 3, 1, 1), C=64),
}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
    want = set(sys.argv[2:]) or None
    c = CFGS[name]
    sides, K, S, B, D, bh, sink = c["sides"], c["K"], c["S"], c["B"], c["D"], c["bh"], c["sink"]
    nK, nS = sides[K - 1] ** 2, sides[S - 1] ** 2
    cK, cS = sum(s * s for s in sides[:K]), sum(s * s for s in sides[:S])
    dev = torch.device("cuda", 0)
    q = q_iid(0, K, 0, bh, nK, D, device=dev)
    qs, ks, _ = structured_qkv(1, sides, S, K, 0, bh, D, sink_scales=sink)
    qS = qs.to(dev)
    k, v = kv_cache_iid(0, 0, bh, cK, D, device=dev)
    k[:, :cS] = ks[:, :cS].to(dev)
    ran = []

    def on(n):
        if want is None or n in want:
            ran.append(n)
            return True
        return False

    gk, gs = sv.geometry(sides, K, B), sv.geometry(sides, S, B)
    local = sv.local_mask(sides, K, B, sink, c["windows"]) if on("mask") else \
        sv.local_mask(sides, K, B, sink, c["windows"])
    src, _ = sv.predict_pattern(sides, S, B, 0, qS, k, sv.SELECT_TOPK, 2)
    if on("predict"):
        sv.predict_pattern(sides, S, B, sink, qS, k, sv.SELECT_THRESHOLD, 0, 0.02)
    mapped = sv.map_indices(sides, S, K, B, sink, src)
    on("map")
    rp, ci, st = sv.build_block_lists(bh, gk["G_q"], gk["G_kv"], [(local, True), (mapped, False)])
    on("lists")
    rpS, ciS, _ = sv.build_block_lists(bh, gs["G_q"], gs["G_kv"], [(src, False)])
    if on("sparse"):
        lse = torch.empty((bh, nK), dtype=torch.float32, device=dev)
        sv.block_sparse_attn(sides, K, B, q, k, v, rp, ci, lse=lse)
    if on("dense"):
        sv.dense_attn(sides, K, q, k, v)
    oS = torch.empty_like(qS)
    if on("mass"):
        sv.dense_attn_mass(sides, S, B, 0, qS, k, v, sv.SELECT_TOPK, 2, o=oS)
    else:
        sv.dense_attn(sides, S, qS, k, v, o=oS)
    if on("cached"):
        oc = sv.cache_residual_from_dense(sides, S, B, qS, k, v, rpS, ciS, oS)
        sv.block_sparse_attn_cached(sides, K, B, q, k, v, rp, ci, oc, S)
        sv.cache_residual(sides, S, B, qS, k, v, rpS, ciS)
    if on("rows"):
        kc = sv.compress_kv(sides, K, k, sink, c["windows"])
        vc = sv.compress_kv(sides, K, v, sink, c["windows"])
        kept = kc.shape[1]
        lm = sv.local_mask_compressed(sides, K, B, sink, c["windows"])
        rpc, cic, _ = sv.build_block_lists(bh, gk["G_q"], -(-kept // B), [(lm, True)])
        sv.block_sparse_attn_rows(sides, K, B, q, kc, vc, kept, rpc, cic)
    C = c["C"]
    lseS = torch.empty((bh, nS), dtype=torch.float32, device=dev)
    sv.dense_attn(sides, S, qS, k, v, o=oS, lse=lseS)
    cs = sv.token_colsum(sides, S, C, qS, k, lseS) if on("colsum") else \
        sv.token_colsum(sides, S, C, qS, k, lseS)
    ktok = max(1, (cS + 4) // 5)
    tsel = sv.token_select(sides, S, C, 0, cs, ktok)
    on("token_sel")
    tmap = sv.token_map(sides, S, K, C, sink, tsel)
    on("token_map")
    G_K = -(-nK // C)
    trp, tci, _ = sv.build_block_lists(bh, G_K, cK, [(tmap, False)])
    if on("token_attn"):
        sv.token_sparse_attn(sides, K, C, q, k, v, trp, tci)
    if on("token_cached"):
        G_S = -(-nS // C)
        srp, sci, _ = sv.build_block_lists(bh, G_S, cS, [(tsel, False)])
        toc = sv.token_cache_residual(sides, S, C, qS, k, v, srp, sci, oS)
        sv.token_sparse_attn_cached(sides, K, C, q, k, v, trp, tci, toc, S)
    torch.cuda.synchronize()
    print(f"sanitize {name}: ran {' '.join(ran)}; status {st.item()}")


if __name__ == "__main__":
    main()
