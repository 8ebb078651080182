"""Development aid: per-CTA work quantisation probe.  Times the decision-scale predictor and the
CSLA attention of the 8B-shaped last scale for several (b,h) counts: with 148 persistent CTAs and
two lock-stepped predictor slots, the predictor's makespan is ceil(13 bh / 148 / 2) rounds, so
its time should step at bh = 92 (1196 tiles > 148 x 8) if a half-empty round costs a full one.
    python scripts/quant_probe.py [bh ...]"""
import os
import statistics
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_04361_b200 as sv

sides = [1, 2, 4, 6, 8, 12, 16, 20, 24, 32, 40, 48, 64]
K, S, B, D = 13, 11, 128, 128
bhs = [int(x) for x in sys.argv[1:]] or [74, 80, 86, 91, 92, 96]


def timed(fn, n=20, reps=5):
    for _ in range(3):
        fn()
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / n)
    return statistics.median(out)


torch.manual_seed(0)
for bh in bhs:
    q = torch.randn(bh, 4096, D, device="cuda").bfloat16()
    qS = torch.randn(bh, 1600, D, device="cuda").bfloat16()
    k = torch.randn(bh, 10521, D, device="cuda").bfloat16()
    v = torch.randn(bh, 10521, D, device="cuda").bfloat16()
    layer = sv.SparseLayer(sides, K, S, B, bh, sink_scales=5, topk=5)
    layer.build_patterns(qS, k)
    t_pred = timed(lambda: sv.predict_pattern(sides, S, B, 5, qS, k, sv.SELECT_TOPK, 5))
    t_csla = timed(lambda: layer.attend("csla", q, k, v))
    t_cs4a = timed(lambda: layer.attend("cs4a", q, k, v))
    print(f"bh {bh:3d}  pred tiles {13 * bh:5d} ({13 * bh / 148:5.2f}/CTA)  predictor {t_pred:.4f} ms "
          f"({t_pred / bh * 1e3:.2f} us/bh)  attn tiles {32 * bh:5d} ({32 * bh / 148:5.2f}/CTA)  "
          f"csla {t_csla:.4f} ms ({t_csla / bh * 1e3:.2f} us/bh)  cs4a {t_cs4a:.4f} ms "
          f"({t_cs4a / bh * 1e3:.2f} us/bh)", flush=True)
    del q, qS, k, v, layer
    torch.cuda.empty_cache()
