"""Context measurement (not a product path): the library FlashAttention-4 CuTe-DSL forward
(vllm.vllm_flash_attn.cute, installed in the image) on the bench's dense shape, next to this
build's own dense kernel — how good the speed-up denominator is.  Optionally FA4's block-sparse
forward on the CSLA block lists of the bench (every listed block a full 128 x 128 tile).
    python scripts/fa4_compare.py"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_04361_b200 as sv  # noqa: E402

SIDES = [1, 2, 4, 6, 8, 12, 16, 20, 24, 32, 40, 48, 64]
B, H, D, NQ, NKV = 4, 24, 128, 4096, 10521


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / reps)
    return statistics.median(ts)


def main():
    torch.manual_seed(0)
    q = torch.randn(B * H, NQ, D, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(B * H, NKV, D, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(B * H, NKV, D, device="cuda", dtype=torch.bfloat16)
    flops = 4.0 * D * NQ * NKV * B * H
    ours = timeit(lambda: sv.dense_attn(SIDES, 13, q, k, v))
    print(f"ours dense : {ours:.4f} ms  {flops / ours / 1e9:.0f} TFLOP/s")
    # FA4 wants (batch, seqlen, heads, dim)
    qf = q.view(B, H, NQ, D).transpose(1, 2).contiguous()
    kf = k.view(B, H, NKV, D).transpose(1, 2).contiguous()
    vf = v.view(B, H, NKV, D).transpose(1, 2).contiguous()
    try:
        from vllm.vllm_flash_attn.cute.interface import flash_attn_func
        out = flash_attn_func(qf, kf, vf)
        o = out[0] if isinstance(out, tuple) else out
        fa = timeit(lambda: flash_attn_func(qf, kf, vf))
        print(f"FA4 dense  : {fa:.4f} ms  {flops / fa / 1e9:.0f} TFLOP/s   ours/FA4 time {ours / fa:.3f}")
        ref = sv.dense_attn(SIDES, 13, q, k, v).view(B, H, NQ, D).transpose(1, 2)
        print(f"max |ours - FA4| = {(ref.float() - o.float()).abs().max().item():.4f}")
    except Exception as e:  # noqa: BLE001
        print("FA4 unavailable:", type(e).__name__, str(e)[:300])
    try:
        from flash_attn import flash_attn_func as fa2
        t2 = timeit(lambda: fa2(qf, kf, vf))
        print(f"FA2 dense  : {t2:.4f} ms  {flops / t2 / 1e9:.0f} TFLOP/s")
    except Exception as e:  # noqa: BLE001
        print("FA2 unavailable:", type(e).__name__, str(e)[:200])


if __name__ == "__main__":
    main()
