"""Development aid: interleaved timing of several libsparvar builds on the 8B-shaped last scale.
    python scripts/time_variants.py lib1.so lib2.so ...   (default: the in-tree library)"""
import os
import statistics
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_04361_b200 as sv

libs = sys.argv[1:] or [sv.LIB_PATH]
handles = {os.path.basename(p): sv._load(os.path.abspath(p), partial=True) for p in libs}
sides = [1, 2, 4, 6, 8, 12, 16, 20, 24, 32, 40, 48, 64]
K, S, B, D, bh = 13, 11, 128, 128, int(os.environ.get("SV_BH", "96"))
torch.manual_seed(0)
q = torch.randn(bh, 4096, D, device="cuda").bfloat16()
qS = torch.randn(bh, 1600, D, device="cuda").bfloat16()
k = torch.randn(bh, 10521, D, device="cuda").bfloat16()
v = torch.randn(bh, 10521, D, device="cuda").bfloat16()
layer = sv.SparseLayer(sides, K, S, B, bh, sink_scales=5, topk=5)
layer.build_patterns(qS, k)
torch.cuda.synchronize()
nnz = {w: int(layer.lists[w][0][-1].item()) for w in ("csla", "cs4a")}
nnz["dense"] = 32 * 83 * bh
try:
    import pynvml
    pynvml.nvmlInit()
    hnd = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    clk = lambda: pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM)
except Exception:
    clk = lambda: -1
res = {(n, w): [] for n in handles for w in nnz}
clks = []
import random
import time
rng = random.Random(1234)
names = list(handles)
for rep in range(int(os.environ.get("SV_ROUNDS", "9"))):
    # random order per round and a short idle gap before each library: no position bias from
    # the power / clock state the previous library left behind
    order = names[:]
    rng.shuffle(order)
    for name in order:
        L = handles[name]
        time.sleep(0.05)
        sv.lib = L
        for w in ("csla", "cs4a", "dense"):
            fn = (lambda: sv.dense_attn(sides, K, q, k, v)) if w == "dense" else \
                 (lambda: layer.attend(w, q, k, v))
            reps = 5 if w == "dense" else 20
            for _ in range(2):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            clks.append(clk())
            res[(name, w)].append(e0.elapsed_time(e1) / reps)
print("SM clock MHz during runs: median %s min %s  (times: median [min] over %d rounds, shuffled order)" % (statistics.median(clks), min(clks), len(res[next(iter(res))])))
for name in handles:
    line = [name.ljust(18)]
    for w in ("csla", "cs4a", "dense"):
        ms = statistics.median(res[(name, w)])
        line.append(f"{w} {ms:.4f} [{min(res[(name, w)]):.4f}] ms ({4 * D * B * B * nnz[w] / ms / 1e9:.0f} TF)")
    d, c = statistics.median(res[(name, "dense")]), statistics.median(res[(name, "csla")])
    line.append(f"x{d / c:.2f}")
    print("  ".join(line), flush=True)
