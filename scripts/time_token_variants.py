"""Development aid: shuffled-order timing of the token-list attention kernel (NEXT(2)) in several
libsparvar builds, at the bench shape (96 (b,h), S = 11 -> K = 13, C = 192, alpha = 0.2).
    python scripts/time_token_variants.py lib1.so lib2.so ..."""
import math
import os
import random
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_04361_b200 as sv  # noqa: E402

libs = sys.argv[1:]
handles = {os.path.basename(p): sv._load(os.path.abspath(p), partial=True) for p in libs}
sides = [1, 2, 4, 6, 8, 12, 16, 20, 24, 32, 40, 48, 64]
S, K, C, D, bh, sink = 11, 13, 192, 128, 96, 5
nS, nK = sides[S - 1] ** 2, sides[K - 1] ** 2
cS, cK = sum(x * x for x in sides[:S]), sum(x * x for x in sides[:K])
torch.manual_seed(0)
qS = torch.randn(bh, nS, D, device="cuda").bfloat16()
q = torch.randn(bh, nK, D, device="cuda").bfloat16()
k = torch.randn(bh, cK, D, device="cuda").bfloat16()
v = torch.randn(bh, cK, D, device="cuda").bfloat16()
lse = torch.empty((bh, nS), dtype=torch.float32, device="cuda")
sv.dense_attn(sides, S, qS, k, v, lse=lse)
cs = sv.token_colsum(sides, S, C, qS, k, lse)
sel = sv.token_select(sides, S, C, 0, cs, max(1, math.ceil(0.2 * cS)))
dst = sv.token_map(sides, S, K, C, sink, sel)
G = -(-nK // C)
rp, ci, st = sv.build_block_lists(bh, G, cK, [(dst, False)])
torch.cuda.synchronize()
tokens = int(rp[-1].item())
res = {n: [] for n in handles}
rng = random.Random(3)
for rep in range(int(os.environ.get("SV_ROUNDS", "7"))):
    order = list(handles)
    rng.shuffle(order)
    for name in order:
        sv.lib = handles[name]
        time.sleep(0.05)
        fn = lambda: sv.token_sparse_attn(sides, K, C, q, k, v, rp, ci)
        for _ in range(2):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name].append(e0.elapsed_time(e1) / 10)
print(f"token attention: {tokens / (bh * G):.0f} tokens per 192-row block of {cK}")
for n, vv in res.items():
    ms = statistics.median(vv)
    print(f"{n:22s} token_attn {ms:.4f} [{min(vv):.4f}] ms")
