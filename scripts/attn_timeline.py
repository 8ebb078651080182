"""Development aid: both slots' softmax step timelines in CTA 0 (thread 0 of each slot's warpgroup,
the two warps of SM sub-partition 0) from a -DSV_PROF variant library.
    SPARVAR_LIB=variants/lib_prof.so python scripts/attn_timeline.py [csla|dense]"""
import ctypes
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2602_04361_b200 as sv  # noqa: E402

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
sl = []
for t in range(2):
    x = a[t * 2500:(t + 1) * 2500].reshape(500, 5)
    x = x[x[:, 0] > 0]
    sl.append(x)
t0 = min(x[:, 0].min() for x in sl)
for t, x in enumerate(sl):
    d = np.diff(x, axis=1)
    print(f"slot {t}: {len(x)} steps; median wait {np.median(d[:, 0]):.0f} max-pass {np.median(d[:, 1]):.0f} "
          f"exp-pass {np.median(d[:, 2]):.0f} tail {np.median(d[:, 3]):.0f} gap {np.median(x[1:, 0] - x[:-1, 4]):.0f} "
          f"period {np.median(np.diff(x[:, 0])):.0f}")
# overlap of the exp passes (stamp 2 -> 3) and of the whole bodies (1 -> 4)
def overlap(i0, i1):
    ev = []
    for x in sl:
        for r in x:
            ev.append((r[i0], 1))
            ev.append((r[i1], -1))
    ev.sort()
    cur, last, acc = 0, ev[0][0], [0, 0, 0]
    for tt, dd in ev:
        acc[min(cur, 2)] += tt - last
        cur += dd
        last = tt
    return acc
e = overlap(2, 3)
b = overlap(1, 4)
span = max(x[:, 4].max() for x in sl) - t0
print(f"span {span} clk; exp passes: both {e[2]} one {e[1]}; bodies: both {b[2]} one {b[1]}")
print("steps 20..31 rel clk [wait, body, maxdone, expdone, end] slot0 | slot1")
for g in range(20, 32):
    r = [list(x[g] - t0) if g < len(x) else None for x in sl]
    print(g, r[0], "|", r[1])
# MMA issuer ops of CTA 0 (slot alternates 0, 1 while both slots have tiles):
# [0 before P wait, 1 P seen, 2 PV issued, 3 QK issued, 4 loop top, 5 V stage ready, 6 K stage ready]
op = a[8192:8192 + 8 * 1000].reshape(1000, 8)
op = op[op[:, 0] > 0]
if len(op):
    m = lambda x: float(np.median(x))  # noqa: E731
    print(f"MMA ops {len(op)}: V-stage wait {m(op[:, 5] - op[:, 4]):.0f}  K-stage wait {m(op[:, 6] - op[:, 5]):.0f}  "
          f"to P wait {m(op[:, 0] - op[:, 6]):.0f}  P wait {m(op[:, 1] - op[:, 0]):.0f}  PV {m(op[:, 2] - op[:, 1]):.0f}  "
          f"QK {m(op[:, 3] - op[:, 2]):.0f}  QK->next top {m(op[1:, 4] - op[:-1, 3]):.0f}  period {m(np.diff(op[:, 0])):.0f}")
    print("ops 40..48 rel clk [P wait, P seen, PV, QK, top, V ok, K ok]:")
    for i in range(40, min(48, len(op))):
        print(i, [int(x - t0) for x in op[i][:7]])
# K/V stages of CTA 0: loader [wait-empty start, TMA issue], issuer [stage observed full]
ld = a[16384:16384 + 4000].reshape(2000, 2)
use = a[20480:20480 + 2000]
n = int(min((ld[:, 0] > 0).sum(), (use > 0).sum()))
if n > 50:
    ld, use = ld[:n], use[:n]
    m = lambda x: float(np.median(x))  # noqa: E731
    print(f"stages {n}: loader wait-empty {m(ld[:, 1] - ld[:, 0]):.0f}  issue->issuer sees full {m(use - ld[:, 1]):.0f} "
          f"(p10 {np.percentile(use - ld[:, 1], 10):.0f} p90 {np.percentile(use - ld[:, 1], 90):.0f})  "
          f"loads per 1000 clk {1000 * n / (ld[-1, 1] - ld[0, 1]):.2f}")
    print("stage 100..110 rel: [loader wait start, issue, issuer sees full]")
    for i in range(100, 110):
        print(i, int(ld[i, 0] - t0), int(ld[i, 1] - t0), int(use[i] - t0))
# issuer tile starts of CTA 0: [enter, K stage ready, Q ready, QK issued]
ts = a[22528:22528 + 2000].reshape(500, 4)
ts = ts[ts[:, 0] > 0]
if len(ts):
    m = lambda x: float(np.median(x))  # noqa: E731
    print(f"tile starts {len(ts)}: K-stage wait {m(ts[:, 1] - ts[:, 0]):.0f} (max {int((ts[:, 1] - ts[:, 0]).max())})  "
          f"Q wait {m(ts[:, 2] - ts[:, 1]):.0f} (max {int((ts[:, 2] - ts[:, 1]).max())})  QK issue {m(ts[:, 3] - ts[:, 2]):.0f}")
# step-period outliers per slot: how much time the long periods (tile boundaries) add
for t, x in enumerate(sl):
    per = np.diff(x[:, 1])
    med = np.median(per)
    big = per[per > 1.4 * med]
    print(f"slot {t}: periods median {med:.0f} p90 {np.percentile(per, 90):.0f} max {per.max()}; "
          f"{len(big)} long periods add {int((big - med).sum())} clk of {int(per.sum())} "
          f"({100 * (big - med).sum() / per.sum():.1f}%)")
