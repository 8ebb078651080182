"""Development aid: shuffled-order timing of the pattern work (a1 local mask, a4 map, a5 lists for
CSLA and CS4A; the predictor excluded) in several libsparvar builds, 8B shape.
    python scripts/time_patterns.py lib1.so lib2.so ..."""
import os
import random
import statistics
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2602_04361_b200 as sv  # noqa: E402

libs = sys.argv[1:]
handles = {os.path.basename(p): sv._load(os.path.abspath(p), partial=True) for p in libs}
sides = [1, 2, 4, 6, 8, 12, 16, 20, 24, 32, 40, 48, 64]
torch.manual_seed(0)
qS = torch.randn(96, 1600, 128, device="cuda").bfloat16()
k = torch.randn(96, 10521, 128, device="cuda").bfloat16()
layer = sv.SparseLayer(sides, 13, 11, 128, 96, sink_scales=5, topk=5)
layer.build_patterns(qS, k)
torch.cuda.synchronize()
ref = {w: [x.clone() for x in layer.lists[w]] for w in ("csla", "cs4a")}
res = {n: [] for n in handles}
rng = random.Random(5)
for rep in range(9):
    order = list(handles)
    rng.shuffle(order)
    for name in order:
        sv.lib = handles[name]
        fn = lambda: layer.build_patterns(qS, k, predict=False)  # noqa: E731
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name].append(e0.elapsed_time(e1) / 20 * 1e3)
        for w in ("csla", "cs4a"):
            rp, ci = layer.lists[w]
            n = int(rp[-1].item())
            assert torch.equal(rp, ref[w][0]) and torch.equal(ci[:n], ref[w][1][:n]), (name, w)
for n, v in res.items():
    print(f"{n:24s} pattern work {statistics.median(v):.1f} [{min(v):.1f}] us (lists identical)")
