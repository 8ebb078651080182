"""Development aid: blocked-clock breakdown of the predictor roles (-DSV_PRED_PROF build).
    SPARVAR_LIB=variants/lib_pprof.so python scripts/pred_prof.py"""
import ctypes
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_04361_b200 as sv

sides = [1, 2, 4, 6, 8, 12, 16, 20, 24, 32, 40, 48, 64]
S, B, D, bh = 11, 128, 128, 96
qS = torch.randn(bh, 1600, D, device="cuda").bfloat16()
k = torch.randn(bh, 10521, D, device="cuda").bfloat16()
fn = lambda: sv.predict_pattern(sides, S, B, 5, qS, k, sv.SELECT_TOPK, 5)
fn(); torch.cuda.synchronize()
sv.lib.sparvar_pred_prof_reset()
reps = 5
for _ in range(reps):
    fn()
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 16)()
sv.lib.sparvar_pred_prof_read.argtypes = [ctypes.c_void_p]
sv.lib.sparvar_pred_prof_read(buf)
ncta = 148 * reps
names = {0: "MMA wait s_free", 1: "MMA wait kv_full", 2: "MMA wait q_full", 3: "K loader wait kv_empty",
         4: "softmax(q0 warps) wait s_full", 5: "MMA loop total", 6: "softmax(q0) step bodies",
         7: "softmax(q0 warps) tile-end", 9: "softmax(q0) whole", 12: "softmax(other warps) wait s_full", 8: "MMA issue of 8 tcgen05.mma (leader)"}
for i, n in names.items():
    per = buf[i] / ncta
    if i in (4, 6, 7, 9):
        per /= 2      # the two quarter-0 softmax warps per CTA (one per slot)
    if i == 12:
        per /= 6      # the other six softmax warps
    print(f"{n:36s} {per:12.0f} clk per CTA-launch")
