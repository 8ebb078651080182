"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the SparVAR method (no masks, no softmax, no mapping).  It
only turns (seed, tensor tag, element counter) into bf16 numbers, so that the CPU oracle
(`oracle/`) and the CUDA path (`paper_2602_04361_b200/`) can be fed the *same* values while
sharing no other code (DESIGN.md §"Inputs").

Generator (counter based, so any (batch x head) shard regenerates independently):
    key   = splitmix64(seed * 0x9E3779B97F4A7C15 + tag)
    a, b  = splitmix64(key + 2*i), splitmix64(key + 2*i + 1)          i = global element index
    u1    = ((a >>> 11) + 1) * 2^-53  in (0, 1]      u2 = (b >>> 11) * 2^-53  in [0, 1)
    z     = sqrt(-2 ln u1) * cos(2 pi u2)            (Box-Muller, fp64)
    value = bf16_rne(fp32_rne(z))
Element i of a (BH, rows, D) tensor is ((bh * rows) + row) * D + d with `bh` the GLOBAL
(batch*heads + head) index, so a rank holding heads [h0, h1) gets exactly the rows a single GPU
would have generated for them.

The integer part is exact on every device; the fp64 log/cos may differ in the last ulp between
CPU and GPU libm, so a parity test always feeds both sides ONE generated copy (generated on one
device, copied to the other).  Never compare values generated independently on two devices.

Modes
  iid         Q, K, V ~ N(0, 1)                       (timing; attention parity)
  structured  q = g*phi(p_q) + eps, k = g*phi(p_k) + eps with phi random Fourier features of the
              token's normalised 2-D centre, plus a shared "sink" direction on the keys of the
              first `sink_scales` scales and on all queries (predictor / mapping tests, where iid
              attention is too flat to make top-k well conditioned).  SURVEY.md §8(d).
"""
from __future__ import annotations

import math
from typing import Sequence

import torch

__all__ = [
    "TAG_Q", "TAG_K", "TAG_V", "splitmix64", "normal_f64", "normal_bf16",
    "qkv_iid", "kv_cache_iid", "q_iid", "structured_qkv",
]

TAG_Q = 0x51      # + 0x100 * scale index (queries of different scales are different tensors)
TAG_K = 0x4B
TAG_V = 0x56
TAG_OMEGA = 0x0F
TAG_PHASE = 0x0E
TAG_SINK = 0x0D
TAG_EPS_Q = 0x1E
TAG_EPS_K = 0x2E

_GOLDEN = -7046029254386353131          # 0x9E3779B97F4A7C15 as int64
_M1 = -4658895280553007687              # 0xBF58476D1CE4E5B9
_M2 = -7723592293110705685              # 0x94D049BB133111EB


def _srl(x: torch.Tensor, s: int) -> torch.Tensor:
    """Logical right shift of int64 viewed as uint64."""
    return (x >> s) & ((1 << (64 - s)) - 1)


def splitmix64(x: torch.Tensor) -> torch.Tensor:
    """SplitMix64 finaliser on int64 tensors (two's complement wrap == uint64 arithmetic)."""
    z = x + _GOLDEN
    z = (z ^ _srl(z, 30)) * _M1
    z = (z ^ _srl(z, 27)) * _M2
    return z ^ _srl(z, 31)


def _key(seed: int, tag: int) -> int:
    t = torch.tensor([(seed * 0x9E3779B97F4A7C15 + tag) & 0xFFFFFFFFFFFFFFFF], dtype=torch.uint64)
    return int(splitmix64(t.view(torch.int64))[0])


def normal_f64(seed: int, tag: int, start: int, count: int, device="cpu") -> torch.Tensor:
    """`count` standard normals for element counters start .. start+count-1 (fp64)."""
    key = _key(seed, tag)
    i = torch.arange(start, start + count, dtype=torch.int64, device=device)
    a = splitmix64(key + 2 * i)
    b = splitmix64(key + 2 * i + 1)
    u1 = (_srl(a, 11) + 1).to(torch.float64) * (2.0 ** -53)
    u2 = _srl(b, 11).to(torch.float64) * (2.0 ** -53)
    return torch.sqrt(-2.0 * torch.log(u1)) * torch.cos((2.0 * math.pi) * u2)


def normal_bf16(seed: int, tag: int, start: int, count: int, device="cpu") -> torch.Tensor:
    return normal_f64(seed, tag, start, count, device).to(torch.float32).to(torch.bfloat16)


def _bh_tensor(seed, tag, bh_start, bh_count, rows, D, device, capacity=None):
    cap = rows if capacity is None else capacity
    out = torch.zeros((bh_count, cap, D), dtype=torch.bfloat16, device=device)
    for i in range(bh_count):
        bh = bh_start + i
        out[i, :rows] = normal_bf16(seed, tag, bh * rows * D, rows * D, device).view(rows, D)
    return out


def q_iid(seed, scale, bh_start, bh_count, n_q, D, device="cpu"):
    """Queries of scale `scale` (1-based), (bh_count, n_q, D) bf16."""
    return _bh_tensor(seed, TAG_Q + 0x100 * scale, bh_start, bh_count, n_q, D, device)


def kv_cache_iid(seed, bh_start, bh_count, n_kv, D, device="cpu", capacity=None):
    """History K/V cache (concatenated scales, schedule order), (bh_count, capacity, D) bf16.
    Rows >= n_kv (spare capacity) are zero."""
    k = _bh_tensor(seed, TAG_K, bh_start, bh_count, n_kv, D, device, capacity)
    v = _bh_tensor(seed, TAG_V, bh_start, bh_count, n_kv, D, device, capacity)
    return k, v


def qkv_iid(seed, scale, bh_start, bh_count, n_q, n_kv, D, device="cpu"):
    q = q_iid(seed, scale, bh_start, bh_count, n_q, D, device)
    k, v = kv_cache_iid(seed, bh_start, bh_count, n_kv, D, device)
    return q, k, v


def _centres(sides: Sequence[int], scales: Sequence[int], device) -> torch.Tensor:
    """Normalised token centres ((x+.5)/s, (y+.5)/s), row-major, scales concatenated."""
    pts = []
    for k in scales:
        s = sides[k - 1]
        r = (torch.arange(s, dtype=torch.float64, device=device) + 0.5) / s
        xx, yy = torch.meshgrid(r, r, indexing="ij")
        pts.append(torch.stack([xx.reshape(-1), yy.reshape(-1)], 1))
    return torch.cat(pts, 0)


def structured_qkv(seed, sides: Sequence[int], q_scale: int, kv_scales: int, bh_start, bh_count,
                   D, sink_scales=5, gamma=9.0, sigma_f=3.0, eps=0.3, sink_amp=2.0,
                   device="cpu"):
    """Locality-structured inputs (SURVEY.md §8(d) 'structured').  Returns bf16
    q (bh, N_{q_scale}, D), k, v (bh, C_{kv_scales}, D).  Random draws all come from the
    counter generator above (tags OMEGA/PHASE/SINK/EPS_*), per global bh."""
    pq = _centres(sides, [q_scale], device)
    pk = _centres(sides, list(range(1, kv_scales + 1)), device)
    n_sink = sum(s * s for s in sides[:sink_scales])
    F = D // 2
    qs, ks, vs = [], [], []
    for i in range(bh_count):
        bh = bh_start + i
        omega = normal_f64(seed, TAG_OMEGA, bh * F * 2, F * 2, device).view(F, 2) * sigma_f
        phase = normal_f64(seed, TAG_PHASE, bh * F, F, device)
        u = normal_f64(seed, TAG_SINK, bh * D, D, device)
        u = u / torch.linalg.norm(u)

        def feat(p):
            a = 2.0 * math.pi * (p @ omega.T) + phase
            return torch.cat([torch.cos(a), torch.sin(a)], 1) * math.sqrt(1.0 / F)

        nq, nk = pq.shape[0], pk.shape[0]
        q = gamma * feat(pq) + eps * normal_f64(seed, TAG_EPS_Q + 0x100 * q_scale, bh * nq * D,
                                                nq * D, device).view(nq, D)
        k = gamma * feat(pk) + eps * normal_f64(seed, TAG_EPS_K, bh * nk * D, nk * D,
                                                device).view(nk, D)
        q = q + sink_amp * u
        k[:n_sink] += sink_amp * u
        v = normal_f64(seed, TAG_V, bh * nk * D, nk * D, device).view(nk, D)
        qs.append(q.to(torch.float32).to(torch.bfloat16))
        ks.append(k.to(torch.float32).to(torch.bfloat16))
        vs.append(v.to(torch.float32).to(torch.bfloat16))
    return torch.stack(qs), torch.stack(ks), torch.stack(vs)
