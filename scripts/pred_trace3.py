"""Development aid: one CTA's predictor timeline (-DSV_PRED_TRACE=<cta> build): per slot and S use,
issuer [s_free wait start, MMA issue start, issue end] and softmax [s_full wait start, S seen,
step end].   SPARVAR_LIB=variants/lib_ptr.so python scripts/pred_trace3.py"""
import ctypes
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2602_04361_b200 as sv  # noqa: E402

sides = [1, 2, 4, 6, 8, 12, 16, 20, 24, 32, 40, 48, 64]
qS = torch.randn(96, 1600, 128, device="cuda").bfloat16()
k = torch.randn(96, 10521, 128, device="cuda").bfloat16()
for _ in range(3):
    sv.predict_pattern(sides, 11, 128, 5, qS, k, sv.SELECT_TOPK, 5)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (3 * 320 * 6))()
sv.lib.sparvar_pred_trace3.argtypes = [ctypes.c_void_p]
assert sv.lib.sparvar_pred_trace3(buf) == 0
a = np.array(buf[:], dtype=np.int64).reshape(3, 320, 6)
t0 = a[a > 0].min()
m = lambda x: float(np.median(x))  # noqa: E731
for t in range(3):
    x = a[t]
    n = int((x[:, 5] > 0).sum())
    x = x[:n]
    print(f"slot {t}: {n} steps | issuer s_free wait {m(x[:, 1] - x[:, 0]):.0f} issue {m(x[:, 2] - x[:, 1]):.0f} | "
          f"softmax S wait {m(x[:, 4] - x[:, 3]):.0f} body {m(x[:, 5] - x[:, 4]):.0f} | "
          f"S seen - issue end {m(x[:, 4] - x[:, 2]):.0f} | period {m(np.diff(x[:, 4])):.0f}")
print("steps 40..44 rel clk per slot: [free-wait, issue, issued, S-wait, S seen, end]")
for g in range(40, 45):
    print(g, [list(int(v - t0) for v in a[t, g]) for t in range(3)])
