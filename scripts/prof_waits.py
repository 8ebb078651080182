"""Development aid: where the attention roles block (SM clocks summed per CTA) from a -DSV_PROF
variant library.   SPARVAR_LIB=variants/lib_prof.so python scripts/prof_waits.py [csla|cs4a|dense]"""
import ctypes
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2602_04361_b200 as sv

which = sys.argv[1] if len(sys.argv) > 1 else "csla"
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
for _ in range(3):
    fn()
torch.cuda.synchronize()
sv.lib.sparvar_prof_reset()
fn()
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 24576)()
sv.lib.sparvar_prof_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
sv.lib.sparvar_prof_read(buf, 24576)
a = np.array(buf[:], dtype=np.int64)
g = lambda base: a[base:base + 148].astype(np.float64)
ops = g(7000)
tot = g(6800)
print(f"{os.path.basename(sv.LIB_PATH)} {which}: slot-ops per CTA median {np.median(ops):.0f} (min {ops.min():.0f} max {ops.max():.0f})")
print(f"  MMA loop clk per op (median CTA): {np.median(tot / np.maximum(ops, 1)):.0f}  "
      f"(tensor work per op at 100%: {int(os.environ.get("SV_OP_CLK", "1024"))} clk)")
LABELS = {
    "v6": [("MMA wait kv_full", 6000), ("MMA wait P", 6200), ("MMA wait o_free", 6400),
           ("MMA wait q_full", 6600), ("loader wait kv_empty", 5000),
           ("softmax wait S (2 thr)", 5200), ("epilogue wait O (2 thr)", 5400),
           ("MMA issue block P.V", 7200), ("MMA issue block QK", 7400),
           ("softmax compute (2 thr)", 7600), ("softmax wait prev P.V (8 w)", 7800)],
    "pairs": [("MMA wait K stage", 6000), ("MMA wait V stage", 5400), ("MMA wait S free", 6200),
              ("MMA wait P written", 5600), ("MMA wait o_free", 6400), ("MMA wait q_full", 6600),
              ("loader wait stage empty", 5000), ("softmax wait S (2 thr)", 5200),
              ("softmax compute (2 thr)", 7600), ("softmax wait P buffer (8 w)", 7800)],
}[os.environ.get("SV_PROF_LABELS", "v6")]
for name, base in LABELS:
    v = g(base)
    print(f"  {name:26s} per op {np.median(v / np.maximum(ops, 1)):7.0f} clk   share of MMA loop "
          f"{np.median(v / np.maximum(tot, 1)):.3f}")
