"""Shared test configurations and comparison helpers."""
import numpy as np
import torch

from oracle.geometry import INFINITY_1K_SIDES

TINY = dict(sides=[1, 2, 4, 8], K=4, S=3, B=16, D=64, bh=1, sink=2, windows=(3, 3))
EQ256 = dict(sides=[1, 2, 4, 6, 8, 12, 16], K=7, S=5, B=32, D=128, bh=8, sink=3,
             windows=(7, 5, 3, 1, 1))
INF2B = dict(sides=list(INFINITY_1K_SIDES), K=13, S=11, B=128, D=128, bh=16, sink=5,
             windows=(7, 5, 3, 1, 1))

# north_star tolerance for attention on bf16-rounded inputs
MAX_ABS, MEAN_ABS = 1e-2, 1e-3


def bits_to_bool(words, n):
    w = np.asarray(words, dtype=np.int64) & 0xFFFFFFFF
    bits = (w[..., :, None] >> np.arange(32)) & 1
    return bits.reshape(*w.shape[:-1], -1)[..., :n].astype(bool)


def bool_to_bits(mask):
    """bool (..., n) -> int32 words (..., ceil(n/32))"""
    mask = np.asarray(mask, dtype=bool)
    n = mask.shape[-1]
    W = -(-n // 32)
    pad = np.zeros((*mask.shape[:-1], W * 32), dtype=np.int64)
    pad[..., :n] = mask
    words = (pad.reshape(*mask.shape[:-1], W, 32) << np.arange(32)).sum(-1)
    return ((words + 2 ** 31) % 2 ** 32 - 2 ** 31).astype(np.int32)


def csr_lists(row_ptr, col_idx, rows):
    rp = row_ptr.cpu().numpy()
    ci = col_idx.cpu().numpy()
    return [ci[rp[r]:rp[r + 1]] for r in range(rows)]


def attn_errors(gpu_out, ref):
    d = np.abs(gpu_out.astype(np.float64) - ref)
    return float(d.max()), float(d.mean())


def to_np(t: torch.Tensor):
    return t.detach().float().cpu().numpy().astype(np.float64)
