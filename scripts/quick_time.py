"""Quick device timing of the attention kernels (development aid, not the bench)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_04361_b200 as sv
from synth import q_iid, kv_cache_iid

sides = [1, 2, 4, 6, 8, 12, 16, 20, 24, 32, 40, 48, 64]
K, B, D = 13, 128, 128
for bh in (16, 96):
    q = torch.randn(bh, 4096, D, device="cuda").bfloat16()
    k = torch.randn(bh, 10521, D, device="cuda").bfloat16()
    v = torch.randn(bh, 10521, D, device="cuda").bfloat16()
    g = sv.geometry(sides, K, B)
    mask = sv.local_mask(sides, K, B, 5, (7, 5, 3, 1, 1))
    rp, ci, st = sv.build_block_lists(bh, g["G_q"], g["G_kv"], [(mask, True)])
    for name, fn in (("sparse", lambda: sv.block_sparse_attn(sides, K, B, q, k, v, rp, ci)),
                     ("dense", lambda: sv.dense_attn(sides, K, q, k, v))):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 20
        e0.record()
        for _ in range(n): fn()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        tiles = 435 * bh if name == "sparse" else 32 * 83 * bh
        fl = 4 * D * 128 * 128 * tiles
        print(f"bh={bh} {name}: {ms:.4f} ms  {fl/ms/1e9:.1f} TFLOP/s executed", flush=True)
