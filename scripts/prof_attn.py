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
fn = (lambda: sv.dense_attn(sides, K, q, k, v)) if which == "dense" else \
     (lambda: layer.attend(which, q, k, v))
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
nnz = int(layer.lists[which][0][-1].item()) if which != "dense" else 32 * 83 * bh
print(f"{which}: {ms:.4f} ms, {4 * D * B * B * nnz / ms / 1e9:.1f} TFLOP/s executed", flush=True)
