"""Development aid: softmax phase timings (SM clocks) from a -DSV_PROF variant library.
    SPARVAR_LIB=variants/lib_prof.so python scripts/prof_phases.py [csla|cs4a|dense]"""
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
n = int((a != 0).sum() // 5)
st = a[:5 * n].reshape(n, 5)
st = st[st[:, 0] > 0]
d = np.diff(st, axis=1)
gap = st[1:, 0] - st[:-1, 4]
print(f"{which}: steps recorded {len(st)}")
print("median clk: wait %.0f  pass1(max) %.0f  pass2(exp) %.0f  tail %.0f  gap->next %.0f  period %.0f" % (
    np.median(d[:, 0]), np.median(d[:, 1]), np.median(d[:, 2]), np.median(d[:, 3]), np.median(gap),
    np.median(np.diff(st[:, 0]))))
print("first 12 steps (wait, pass1, pass2, tail):")
print(d[:12])

st0 = a[7400:7400 + 148]; su = a[7600:7600 + 148]; en = a[7800:7800 + 148]
if st0.min() > 0:
    t0 = st0.min()
    print("CTA start spread us: %.2f   setup (median) us: %.2f   end: min %.2f median %.2f max %.2f us" % (
        (st0.max() - t0) / 1e3, np.median(su - st0) / 1e3, (en.min() - t0) / 1e3, np.median(en - t0) / 1e3,
        (en.max() - t0) / 1e3))

def cta(base):
    return a[base:base + 148].astype(np.float64)
sm_wait, sm_tot = cta(5000), cta(5200)
pw, kw, ow, qw, mt = cta(5400), cta(5600), cta(5800), cta(6000), cta(6200)
print("per-CTA medians (clk): softmax(slot0,thr0) total %.0f wait-S %.0f (%.0f%%)" % (
    np.median(sm_tot), np.median(sm_wait), 100 * np.median(sm_wait / np.maximum(sm_tot, 1))))
print("  MMA total %.0f: wait P %.0f (%.0f%%)  wait KV %.0f (%.0f%%)  wait O-free %.0f  wait Q %.0f" % (
    np.median(mt), np.median(pw), 100 * np.median(pw / np.maximum(mt, 1)), np.median(kw),
    100 * np.median(kw / np.maximum(mt, 1)), np.median(ow), np.median(qw)))
lt, lw = cta(6400), cta(6600)
print("  KV loader total %.0f: wait empty stage %.0f (%.0f%%)" % (np.median(lt), np.median(lw), 100 * np.median(lw / np.maximum(lt, 1))))

tr = a[2048:2048 + 5 * 400].reshape(-1, 5)
tr = tr[tr[:, 0] > 0]
if len(tr) > 20:
    # v3 MMA warp per step: [t0 before V stage wait, t1 after, t2 after P wait, t3 after PV issue, t4 after QK(g+2) issue]
    d = np.diff(tr, axis=1)
    print("MMA step trace (CTA0) medians clk: V-stage wait %.0f | P wait %.0f | PV issue %.0f | QK issue %.0f | gap %.0f | period %.0f" % (
        np.median(d[:, 0]), np.median(d[:, 1]), np.median(d[:, 2]), np.median(d[:, 3]),
        np.median(tr[1:, 0] - tr[:-1, 4]), np.median(np.diff(tr[:, 0]))))
