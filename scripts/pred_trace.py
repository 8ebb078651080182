"""Development aid: one CTA's timeline of the predictor (-DSV_PRED_PROF -DSV_PRED_TRACE=<cta> build).
    SPARVAR_LIB=variants/lib_ptrace.so python scripts/pred_trace.py"""
import ctypes
import os
import statistics
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2602_04361_b200 as sv  # noqa: E402

sides = [1, 2, 4, 6, 8, 12, 16, 20, 24, 32, 40, 48, 64]
S, B, D, bh = 11, 128, 128, 96
qS = torch.randn(bh, 1600, D, device="cuda").bfloat16()
k = torch.randn(bh, 10521, D, device="cuda").bfloat16()
fn = lambda: sv.predict_pattern(sides, S, B, 5, qS, k, sv.SELECT_TOPK, 5)  # noqa: E731
for _ in range(3):
    fn()
torch.cuda.synchronize()
sm = (ctypes.c_longlong * (2 * 400 * 3))()
mma = (ctypes.c_longlong * (2 * 400 * 2))()
te = (ctypes.c_longlong * (2 * 16 * 2))()
sv.lib.sparvar_pred_trace_read.argtypes = [ctypes.c_void_p] * 3
assert sv.lib.sparvar_pred_trace_read(sm, mma, te) == 0
done = (ctypes.c_longlong * (2 * 400))()   # S completion times, when the build records them
if hasattr(sv.lib, "sparvar_pred_trace_done"):
    sv.lib.sparvar_pred_trace_done.argtypes = [ctypes.c_void_p]
    assert sv.lib.sparvar_pred_trace_done(done) == 0
DN = lambda t, g: done[t * 400 + g]  # noqa: E731
SM = lambda t, g, i: sm[(t * 400 + g) * 3 + i]  # noqa: E731
MM = lambda t, g, i: mma[(t * 400 + g) * 2 + i]  # noqa: E731
steps = [max(g for g in range(400) if SM(t, g, 2) != 0) + 1 if SM(t, 0, 2) else 0 for t in range(2)]
t0 = min(x for x in list(sm) + list(mma) if x != 0)
t1 = max(x for x in list(sm) + list(mma) + list(te))
print(f"steps per slot {steps}, span {t1 - t0} clk")
for t in range(2):
    body = [SM(t, g, 2) - SM(t, g, 1) for g in range(steps[t])]
    wait = [SM(t, g, 1) - SM(t, g, 0) for g in range(steps[t])]
    issue = [MM(t, g, 1) - MM(t, g, 0) for g in range(steps[t])]
    lag = [SM(t, g, 1) - MM(t, g, 1) for g in range(steps[t])]   # softmax body start - MMA issue end
    ex = [DN(t, g) - MM(t, g, 1) for g in range(steps[t])]       # S complete - MMA issue end
    dw = [SM(t, g, 1) - DN(t, g) for g in range(steps[t])]       # softmax body start - S complete
    dd = [DN(t if t == 1 else 1, g) - DN(0, g) for g in range(steps[t])]
    print(f"  S complete - issue end med {statistics.median(ex)}; body start - S complete med "
          f"{statistics.median(dw)}; done(1,g)-done(0,g) med {statistics.median(dd)}; "
          f"done(t,g+1)-done(t,g) med {statistics.median([DN(t, g + 1) - DN(t, g) for g in range(steps[t] - 1)])}")
    gap = [SM(t, g, 0) - SM(t, g - 1, 2) for g in range(1, steps[t])]
    print(f"slot {t}: body med {statistics.median(body)} sum {sum(body)} | s_full wait med "
          f"{statistics.median(wait)} sum {sum(wait)} | issue med {statistics.median(issue)} | "
          f"body-start minus issue-end med {statistics.median(lag)} | gap end->next wait med "
          f"{statistics.median(gap)} sum {sum(gap)}")
    tes = [(te[(t * 16 + i) * 2], te[(t * 16 + i) * 2 + 1]) for i in range(16) if te[(t * 16 + i) * 2]]
    print(f"  tile ends: {[b - a for a, b in tes]}")
# overlap of the two slots' bodies
ev = []
for t in range(2):
    for g in range(steps[t]):
        ev.append((SM(t, g, 1), 1))
        ev.append((SM(t, g, 2), -1))
ev.sort()
cur, last, both, one = 0, t0, 0, 0
for x, d in ev:
    if cur == 2:
        both += x - last
    elif cur == 1:
        one += x - last
    cur += d
    last = x
print(f"time with 2 bodies active {both}, 1 active {one}, none {t1 - t0 - both - one}")
print("first 12 steps of each slot (rel clk): [mma issue start, end, S done] [wait, body start, end]")
for g in range(12):
    print(g, [(MM(t, g, 0) - t0, MM(t, g, 1) - t0, DN(t, g) - t0, SM(t, g, 0) - t0, SM(t, g, 1) - t0, SM(t, g, 2) - t0)
              for t in range(2)])
for g in range(60, 66):
    print(g, [(MM(t, g, 0) - t0, MM(t, g, 1) - t0, DN(t, g) - t0, SM(t, g, 0) - t0, SM(t, g, 1) - t0, SM(t, g, 2) - t0)
              for t in range(2)])
