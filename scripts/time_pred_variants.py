"""Development aid: shuffled-order timing of the decision-scale predictor in several libsparvar
builds (8B shape, S = 11, B = 128, top-5).   python scripts/time_pred_variants.py lib1.so ..."""
import os
import random
import statistics
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_04361_b200 as sv

libs = sys.argv[1:]
handles = {os.path.basename(p): sv._load(os.path.abspath(p), partial=True) for p in libs}
sides = [1, 2, 4, 6, 8, 12, 16, 20, 24, 32, 40, 48, 64]
S, B, D, bh = 11, 128, 128, 96
torch.manual_seed(0)
qS = torch.randn(bh, 1600, D, device="cuda").bfloat16()
k = torch.randn(bh, 10521, D, device="cuda").bfloat16()
res = {n: [] for n in handles}
rng = random.Random(7)
for rep in range(9):
    order = list(handles)
    rng.shuffle(order)
    for name in order:
        sv.lib = handles[name]
        time.sleep(0.05)
        fn = lambda: sv.predict_pattern(sides, S, B, 5, qS, k, sv.SELECT_TOPK, 5)
        for _ in range(2):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name].append(e0.elapsed_time(e1) / 20)
for n, v in res.items():
    print(f"{n:20s} predictor {statistics.median(v):.4f} [{min(v):.4f}] ms")
