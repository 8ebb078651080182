"""Development aid: run one attention variant on the 8B-shaped last scale for ncu / timing.
    python scripts/prof_attn.py [csla|cs4a|dense] [reps]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_04361_b200 as sv

which = sys.argv[1] if len(sys.argv) > 1 else "csla"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
sides = [1, 2, 4, 6, 8, 12, 16, 20, 24, 32, 40, 48, 64]
K, S, B, D, bh = 13, 11, 128, 128, 96
torch.manual_seed(0)
q = torch.randn(bh, 4096, D, device="cuda").bfloat16()
qS = torch.randn(bh, 1600, D, device="cuda").bfloat16()
k = torch.randn(bh, 10521, D, device="cuda").bfloat16()
v = torch.randn(bh, 10521, D, device="cuda").bfloat16()
layer = sv.SparseLayer(sides, K, S, B, bh, sink_scales=5, topk=5)
layer.build_patterns(qS, k)
if which == "dense":
    fn = lambda: sv.dense_attn(sides, K, q, k, v)
elif which == "pred":
    fn = lambda: sv.predict_pattern(sides, S, B, 5, qS, k, sv.SELECT_TOPK, 5, mask_out=layer.src,
                                    mass_out=layer.mass)
elif which == "step":
    fn = lambda: (layer.build_patterns(qS, k), layer.attend("csla", q, k, v), layer.attend("cs4a", q, k, v))
else:
    fn = lambda: layer.attend(which, q, k, v)
for _ in range(reps):
    fn()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    fn()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
if which in ("csla", "cs4a", "dense"):
    nnz = int(layer.lists[which][0][-1].item()) if which != "dense" else 32 * 83 * bh
    print(f"{which}: {ms:.4f} ms, {4 * D * B * B * nnz / ms / 1e9:.1f} TFLOP/s executed", flush=True)
elif which == "pred":
    exps = bh * 1600 * 4121
    print(f"pred: {ms:.4f} ms, {exps / ms / 1e6:.1f} Gexp/s, {2 * D * exps / ms / 1e9:.1f} TFLOP/s (QK)", flush=True)
else:
    print(f"{which}: {ms:.4f} ms", flush=True)

if which == "step":
    # warm per-kernel CUDA-event times of every launch of one step
    g = layer.gk
    parts = {
        "local_mask": lambda: sv.local_mask(sides, K, B, 5, (7, 5, 3, 1, 1), out=layer.local),
        "predict": lambda: sv.predict_pattern(sides, S, B, 5, qS, k, sv.SELECT_TOPK, 5,
                                              mask_out=layer.src, mass_out=layer.mass),
        "map": lambda: sv.map_indices(sides, S, K, B, 5, layer.src, out=layer.mapped),
        "lists_csla": lambda: sv.build_block_lists(bh, g["G_q"], g["G_kv"], [(layer.local, True)],
                                                   layer.cap, *layer.lists["csla"], layer.status),
        "lists_cs4a": lambda: sv.build_block_lists(bh, g["G_q"], g["G_kv"], [(layer.mapped, False)],
                                                   layer.cap, *layer.lists["cs4a"], layer.status),
        "attn_csla": lambda: layer.attend("csla", q, k, v),
        "attn_cs4a": lambda: layer.attend("cs4a", q, k, v),
    }
    for name, f in parts.items():
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            f()
        e1.record()
        torch.cuda.synchronize()
        print(f"  {name:12s} {e0.elapsed_time(e1) / 20 * 1e3:8.1f} us", flush=True)
