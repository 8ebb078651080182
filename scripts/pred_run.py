"""Development aid: run the predictor a few times at the 8B shape (S = 11, B = 128, top-5), for
ncu captures of one build.   SPARVAR_LIB=<lib> python scripts/pred_run.py"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2602_04361_b200 as sv  # noqa: E402

sides = [1, 2, 4, 6, 8, 12, 16, 20, 24, 32, 40, 48, 64]
qS = torch.randn(96, 1600, 128, device="cuda").bfloat16()
k = torch.randn(96, 10521, 128, device="cuda").bfloat16()
for _ in range(5):
    sv.predict_pattern(sides, 11, 128, 5, qS, k, sv.SELECT_TOPK, 5)
torch.cuda.synchronize()
