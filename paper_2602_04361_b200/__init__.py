"""Python binding of libsparvar.so — SparVAR's block-sparse cross-scale attention hot path on
sm_100a (B200).  Argument marshalling only: every step of the path runs in the CUDA kernels of
the C ABI declared in include/sparvar.h; PyTorch only provides device memory and streams.

There is no CPU or PyTorch fallback.  If libsparvar.so is missing the import of this module
raises (build it with `python -m paper_2602_04361_b200.build` or `__graft_entry__.build()`).

Functions mirror the ABI names:
    local_mask, predict_pattern, map_indices, build_block_lists, block_sparse_attn, dense_attn
plus `geometry()` (block counts of a schedule) and `SparseLayer`, the user-facing composition of
the whole path for one layer at the target scale.
"""
from __future__ import annotations

import ctypes
import math
import os
from typing import Optional, Sequence, Tuple

import torch

__all__ = [
    "lib", "SparVARError", "geometry", "local_mask", "predict_pattern", "map_indices",
    "build_block_lists", "block_sparse_attn", "dense_attn", "cache_residual",
    "block_sparse_attn_cached", "cache_residual_from_dense", "dense_attn_mass",
    "dense_attn_mass_workspace", "token_colsum", "token_select", "token_map", "token_sparse_attn",
    "token_cache_residual", "token_sparse_attn_cached", "csla_kept_rows", "compress_kv",
    "local_mask_compressed", "block_sparse_attn_rows",
    "SparseLayer", "unpack_bits",
    "SELECT_TOPK", "SELECT_THRESHOLD", "MAP_FOOTPRINT", "MAP_POINT",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPARVAR_LIB") or os.path.join(_HERE, "libsparvar.so")

SELECT_TOPK, SELECT_THRESHOLD = 0, 1
MAP_FOOTPRINT, MAP_POINT = 0, 1
_STATUS = {0: "OK", 1: "INVALID_ARG", 2: "SCHEDULE", 3: "UNSUPPORTED", 4: "CAPACITY",
           5: "EMPTY_ROW", 6: "CUDA"}


class SparVARError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"sparvar {_STATUS.get(status, status)}: {msg}")
        self.status = status


class _Schedule(ctypes.Structure):
    _fields_ = [("num_scales", ctypes.c_int32), ("sides", ctypes.POINTER(ctypes.c_int32))]


class _Shape(ctypes.Structure):
    _fields_ = [("batch_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("q_stride_bh", ctypes.c_int64), ("kv_stride_bh", ctypes.c_int64),
                ("o_stride_bh", ctypes.c_int64)]


def _load(path: str = LIB_PATH, partial: bool = False):
    """Bind the C ABI of libsparvar.so.  `partial` (development timing of older variant builds
    only) skips entry points the library does not export."""
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python -m paper_2602_04361_b200.build`")
    L = ctypes.CDLL(path)
    P, I32, I64, F32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float
    S = ctypes.POINTER(_Schedule)
    SH = ctypes.POINTER(_Shape)
    sig = {
        "sparvar_local_mask": [S, I32, I32, I32, P, I32, P, P],
        "sparvar_predict_pattern": [S, I32, I32, I32, SH, P, P, F32, I32, I32, F32, P, P, P],
        "sparvar_map_indices": [S, I32, I32, I32, I32, I32, I32, P, P, P],
        "sparvar_build_block_lists": [I32, I32, I32, P, P, I32, P, P, I64, P, P],
        "sparvar_block_sparse_attn": [S, I32, I32, SH, P, P, P, P, P, F32, P, P, P],
        "sparvar_dense_attn": [S, I32, SH, P, P, P, F32, P, P, P],
        "sparvar_cache_residual": [S, I32, I32, SH, P, P, P, P, P, F32, P, P, P],
        "sparvar_block_sparse_attn_cached": [S, I32, I32, SH, P, P, P, P, P, F32, P, I32, I64, P,
                                             P, P],
        "sparvar_cache_residual_from_dense": [S, I32, I32, SH, P, P, P, P, P, F32, P, P, P],
        "sparvar_dense_attn_mass": [S, I32, I32, I32, SH, P, P, P, F32, I32, I32, F32, P, P, P, P,
                                    P, ctypes.c_size_t, P],
        "sparvar_token_colsum": [S, I32, I32, SH, P, P, P, F32, P, P],
        "sparvar_token_select": [S, I32, I32, I32, I32, P, I32, P, P],
        "sparvar_token_map": [S, I32, I32, I32, I32, I32, I32, P, P, P],
        "sparvar_token_sparse_attn": [S, I32, I32, SH, P, P, P, P, P, F32, P, P],
        "sparvar_token_cache_residual": [S, I32, I32, SH, P, P, P, P, P, F32, P, P, P],
        "sparvar_compress_kv": [S, I32, I32, P, I32, I32, I32, P, I64, P, I64, P],
        "sparvar_local_mask_compressed": [S, I32, I32, I32, P, I32, P, P],
        "sparvar_block_sparse_attn_rows": [S, I32, I32, SH, P, P, P, I64, P, P, F32, P, P, P],
        "sparvar_token_sparse_attn_cached": [S, I32, I32, SH, P, P, P, P, P, F32, P, I32, I64, P,
                                             P],
    }
    for name, args in sig.items():
        if partial and not hasattr(L, name):
            continue
        f = getattr(L, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    if hasattr(L, "sparvar_csla_kept_rows"):
        L.sparvar_csla_kept_rows.argtypes = [S, I32, I32, P, I32]
        L.sparvar_csla_kept_rows.restype = ctypes.c_int64
    if hasattr(L, "sparvar_dense_attn_mass_workspace"):
        L.sparvar_dense_attn_mass_workspace.argtypes = [S, I32, I32, I32]
        L.sparvar_dense_attn_mass_workspace.restype = ctypes.c_size_t
    L.sparvar_last_error.restype = ctypes.c_char_p
    L.sparvar_version.restype = ctypes.c_int32
    return L


lib = _load()


def _check(status: int):
    if status != 0:
        raise SparVARError(status, lib.sparvar_last_error().decode())


def _sched(sides: Sequence[int]):
    arr = (ctypes.c_int32 * len(sides))(*[int(s) for s in sides])
    s = _Schedule(len(sides), arr)
    s._keep = arr
    return s


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _ptr(t: Optional[torch.Tensor]):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _bh_view(t: torch.Tensor, name: str):
    if t.dim() != 3 or t.dtype != torch.bfloat16 or not t.is_cuda:
        raise ValueError(f"{name} must be a (BH, rows, D) bf16 CUDA tensor")
    if t.stride(2) != 1 or t.stride(1) != t.shape[2]:
        raise ValueError(f"{name}: rows must be contiguous (stride (.., D, 1))")
    return t.stride(0)


def _dev_tensor(t, name: str, dtype, min_numel: int = 0, exact_numel: Optional[int] = None):
    """The C ABI cannot see allocation sizes: check dtype, device, layout and size here."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != dtype:
        raise ValueError(f"{name} must be a CUDA {dtype} tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if exact_numel is not None and t.numel() != exact_numel:
        raise ValueError(f"{name} has {t.numel()} elements, {exact_numel} required")
    if t.numel() < min_numel:
        raise ValueError(f"{name} has {t.numel()} elements, at least {min_numel} required")
    return t


def _csr(row_ptr, col_idx, rows: int):
    """CSR lists of `rows` query blocks: int32 row_ptr[rows + 1] and int32 col_idx."""
    _dev_tensor(row_ptr, "row_ptr", torch.int32, exact_numel=rows + 1)
    _dev_tensor(col_idx, "col_idx", torch.int32, min_numel=1)


def _kv_rows(sides, scale: int) -> int:
    return sum(int(s) * int(s) for s in sides[:scale])


def geometry(sides: Sequence[int], scale: int, block: int) -> dict:
    """Sizes of scale `scale` (1-based): N, C, G_q, G_kv and the bit-row width W."""
    N = sides[scale - 1] ** 2
    C = sum(s * s for s in sides[:scale])
    g_q, g_kv = -(-N // block), -(-C // block)
    return {"N": N, "C": C, "G_q": g_q, "G_kv": g_kv, "W": -(-g_kv // 32)}


def unpack_bits(words: torch.Tensor, n: int) -> torch.Tensor:
    """Bit rows (..., W) uint32/int32 -> bool (..., n), bit v%32 of word v/32."""
    w = words.to(torch.int64) & 0xFFFFFFFF
    bits = (w.unsqueeze(-1) >> torch.arange(32, device=w.device)) & 1
    return bits.reshape(*w.shape[:-1], -1)[..., :n].bool()


def local_mask(sides, target: int, block: int, sink_scales: int = 5,
               windows: Sequence[int] = (7, 5, 3, 1, 1), out: Optional[torch.Tensor] = None,
               stream=None) -> torch.Tensor:
    g = geometry(sides, target, block)
    if out is None:
        out = torch.empty((g["G_q"], g["W"]), dtype=torch.int32, device="cuda")
    w = (ctypes.c_int32 * max(1, len(windows)))(*[int(x) for x in windows])
    _check(lib.sparvar_local_mask(ctypes.byref(_sched(sides)), target, block, sink_scales, w,
                                  len(windows), _ptr(out), _stream(stream)))
    return out


def predict_pattern(sides, decision_scale: int, block: int, sink_scales: int, q_S: torch.Tensor,
                    k_cache: torch.Tensor, mode: int = SELECT_TOPK, topk: int = 1,
                    threshold: float = 0.0, softmax_scale: float = 0.0, want_mass: bool = True,
                    mask_out=None, mass_out=None, stream=None):
    g = geometry(sides, decision_scale, block)
    bh, D = q_S.shape[0], q_S.shape[2]
    sh = _Shape(bh, D, _bh_view(q_S, "q_S"), _bh_view(k_cache, "k_cache"), 0)
    if k_cache.shape[0] < bh or k_cache.shape[1] < g["C"] or k_cache.shape[2] != D:
        raise ValueError(f"k_cache must be (>= {bh}, >= {g['C']}, {D})")
    if q_S.shape[1] < g["N"]:
        raise ValueError(f"q_S needs >= {g['N']} rows")
    if mask_out is None:
        mask_out = torch.empty((bh, g["G_q"], g["W"]), dtype=torch.int32, device="cuda")
    if want_mass and mass_out is None:
        mass_out = torch.empty((bh, g["G_q"], g["G_kv"]), dtype=torch.float32, device="cuda")
    _dev_tensor(mask_out, "mask_out", torch.int32, min_numel=bh * g["G_q"] * g["W"])
    if want_mass:
        _dev_tensor(mass_out, "mass_out", torch.float32, min_numel=bh * g["G_q"] * g["G_kv"])
    _check(lib.sparvar_predict_pattern(ctypes.byref(_sched(sides)), decision_scale, block,
                                       sink_scales, ctypes.byref(sh), _ptr(q_S), _ptr(k_cache),
                                       softmax_scale, mode, topk, threshold,
                                       _ptr(mass_out if want_mass else None), _ptr(mask_out),
                                       _stream(stream)))
    return mask_out, (mass_out if want_mass else None)


def map_indices(sides, src_scale: int, dst_scale: int, block: int, sink_scales: int,
                src_mask: torch.Tensor, mode: int = MAP_FOOTPRINT, out=None, stream=None):
    bh = src_mask.shape[0]
    g = geometry(sides, dst_scale, block)
    gs = geometry(sides, src_scale, block)
    _dev_tensor(src_mask, "src_mask", torch.int32, min_numel=bh * gs["G_q"] * gs["W"])
    if out is None:
        out = torch.empty((bh, g["G_q"], g["W"]), dtype=torch.int32, device="cuda")
    _dev_tensor(out, "out", torch.int32, min_numel=bh * g["G_q"] * g["W"])
    _check(lib.sparvar_map_indices(ctypes.byref(_sched(sides)), src_scale, dst_scale, block,
                                   sink_scales, mode, bh, _ptr(src_mask), _ptr(out),
                                   _stream(stream)))
    return out


def build_block_lists(bh: int, g_q: int, g_kv: int, masks: Sequence[Tuple[torch.Tensor, bool]],
                      capacity: Optional[int] = None, row_ptr=None, col_idx=None, status=None,
                      stream=None):
    """masks: [(bit-row tensor, broadcast)], broadcast masks are (g_q, W), others (bh, g_q, W).
    Returns (row_ptr, col_idx, status) — status is a device int32 (0 = OK)."""
    if capacity is None:
        capacity = bh * g_q * g_kv
    if row_ptr is None:
        row_ptr = torch.empty(bh * g_q + 1, dtype=torch.int32, device="cuda")
    if col_idx is None:
        col_idx = torch.empty(max(1, capacity), dtype=torch.int32, device="cuda")
    if status is None:
        status = torch.zeros(1, dtype=torch.int32, device="cuda")
    W = -(-g_kv // 32)
    for i, (m, bc) in enumerate(masks):
        _dev_tensor(m, f"masks[{i}]", torch.int32, min_numel=(1 if bc else bh) * g_q * W)
    _dev_tensor(row_ptr, "row_ptr", torch.int32, min_numel=bh * g_q + 1)
    _dev_tensor(col_idx, "col_idx", torch.int32, min_numel=min(max(1, capacity), 1))
    if col_idx.numel() < capacity:
        raise ValueError(f"col_idx has {col_idx.numel()} elements < capacity {capacity}")
    _dev_tensor(status, "status", torch.int32, min_numel=1)
    ptrs = (ctypes.c_void_p * len(masks))(*[m.data_ptr() for m, _ in masks])
    bc = (ctypes.c_int32 * len(masks))(*[1 if b else 0 for _, b in masks])
    _check(lib.sparvar_build_block_lists(bh, g_q, g_kv, ptrs, bc, len(masks), _ptr(row_ptr),
                                         _ptr(col_idx), capacity, _ptr(status), _stream(stream)))
    return row_ptr, col_idx, status


def _attn_shape(q, k, o, v=None, kv_rows: Optional[int] = None, n_q: Optional[int] = None):
    """Shape struct of an attention call, after checking every tensor against q's (b,h) count:
    K/V/O with fewer (b,h) slabs (e.g. GQA-shaped K/V) or K/V with fewer than kv_rows rows
    would make the kernels' TMA / loads read past the allocations."""
    qs, ks, os_ = _bh_view(q, "q"), _bh_view(k, "k_cache"), _bh_view(o, "o")
    bh, D = q.shape[0], q.shape[2]
    for t, name in ((k, "k_cache"), (o, "o")) + (((v, "v_cache"),) if v is not None else ()):
        if t.shape[0] < bh or t.shape[2] != D:
            raise ValueError(f"{name} must be (>= {bh}, rows, {D}) like q")
    if v is not None and _bh_view(v, "v_cache") != ks:
        raise ValueError("k_cache and v_cache must share a (b,h) stride")
    if kv_rows is not None:
        for t, name in ((k, "k_cache"), (v, "v_cache")):
            if t is not None and t.shape[1] < kv_rows:
                raise ValueError(f"{name} has {t.shape[1]} rows, the call reads {kv_rows}")
    if n_q is not None and (q.shape[1] < n_q or o.shape[1] < n_q):
        raise ValueError(f"q / o need >= {n_q} rows")
    return _Shape(bh, D, qs, ks, os_)


def _cache_in(o_cache, bh: int, n_S: int, D: int):
    _bh_view(o_cache, "o_cache")
    if o_cache.shape[0] < bh or o_cache.shape[1] < n_S or o_cache.shape[2] != D:
        raise ValueError(f"o_cache must be (>= {bh}, >= {n_S}, {D})")


def _lse(lse, bh: int, n_q: int):
    if lse is not None:
        _dev_tensor(lse, "lse", torch.float32, min_numel=bh * n_q)


def block_sparse_attn(sides, target: int, block: int, q: torch.Tensor, k_cache: torch.Tensor,
                      v_cache: torch.Tensor, row_ptr: torch.Tensor, col_idx: torch.Tensor,
                      softmax_scale: float = 0.0, o=None, lse=None, stream=None):
    if o is None:
        o = torch.empty_like(q)
    g = geometry(sides, target, block)
    sh = _attn_shape(q, k_cache, o, v_cache, g["C"], g["N"])
    _csr(row_ptr, col_idx, q.shape[0] * g["G_q"])
    _lse(lse, q.shape[0], g["N"])
    _check(lib.sparvar_block_sparse_attn(ctypes.byref(_sched(sides)), target, block,
                                         ctypes.byref(sh), _ptr(q), _ptr(k_cache), _ptr(v_cache),
                                         _ptr(row_ptr), _ptr(col_idx), softmax_scale, _ptr(o),
                                         _ptr(lse), _stream(stream)))
    return o


def dense_attn(sides, target: int, q, k_cache, v_cache, softmax_scale: float = 0.0, o=None,
               lse=None, stream=None):
    if o is None:
        o = torch.empty_like(q)
    g = geometry(sides, target, 128)
    sh = _attn_shape(q, k_cache, o, v_cache, g["C"], g["N"])
    _lse(lse, q.shape[0], g["N"])
    _check(lib.sparvar_dense_attn(ctypes.byref(_sched(sides)), target, ctypes.byref(sh), _ptr(q),
                                  _ptr(k_cache), _ptr(v_cache), softmax_scale, _ptr(o), _ptr(lse),
                                  _stream(stream)))
    return o


def cache_residual(sides, decision_scale: int, block: int, q_S, k_cache, v_cache, row_ptr_S,
                   col_idx_S, softmax_scale: float = 0.0, o_cache=None, o_scratch=None,
                   stream=None):
    """NEXT(1): O_cache = O_dense - O_sparse at the decision scale."""
    if o_cache is None:
        o_cache = torch.empty_like(q_S)
    if o_scratch is None:
        o_scratch = torch.empty_like(q_S)
    if o_scratch.stride(0) != o_cache.stride(0):
        raise ValueError("o_scratch and o_cache must share a (b,h) stride")
    g = geometry(sides, decision_scale, block)
    sh = _attn_shape(q_S, k_cache, o_cache, v_cache, g["C"], g["N"])
    _attn_shape(q_S, k_cache, o_scratch, v_cache, g["C"], g["N"])
    _csr(row_ptr_S, col_idx_S, q_S.shape[0] * g["G_q"])
    _check(lib.sparvar_cache_residual(ctypes.byref(_sched(sides)), decision_scale, block,
                                      ctypes.byref(sh), _ptr(q_S), _ptr(k_cache), _ptr(v_cache),
                                      _ptr(row_ptr_S), _ptr(col_idx_S), softmax_scale,
                                      _ptr(o_scratch), _ptr(o_cache), _stream(stream)))
    return o_cache


def cache_residual_from_dense(sides, decision_scale: int, block: int, q_S, k_cache, v_cache,
                              row_ptr_S, col_idx_S, o_dense, softmax_scale: float = 0.0,
                              o_cache=None, stream=None):
    """NEXT(1)/NEXT(3): O_cache = o_dense - O_sparse at S, reusing the decision scale's dense
    output instead of recomputing it."""
    if o_cache is None:
        o_cache = torch.empty_like(q_S)
    if _bh_view(o_dense, "o_dense") != o_cache.stride(0):
        raise ValueError("o_dense and o_cache must share a (b,h) stride")
    g = geometry(sides, decision_scale, block)
    sh = _attn_shape(q_S, k_cache, o_cache, v_cache, g["C"], g["N"])
    _attn_shape(q_S, k_cache, o_dense, v_cache, g["C"], g["N"])
    _csr(row_ptr_S, col_idx_S, q_S.shape[0] * g["G_q"])
    _check(lib.sparvar_cache_residual_from_dense(
        ctypes.byref(_sched(sides)), decision_scale, block, ctypes.byref(sh), _ptr(q_S),
        _ptr(k_cache), _ptr(v_cache), _ptr(row_ptr_S), _ptr(col_idx_S), softmax_scale,
        _ptr(o_dense), _ptr(o_cache), _stream(stream)))
    return o_cache


def dense_attn_mass(sides, decision_scale: int, block: int, sink_scales: int, q_S, k_cache,
                    v_cache, mode: int = SELECT_TOPK, topk: int = 1, threshold: float = 0.0,
                    softmax_scale: float = 0.0, o=None, lse=None, want_mass: bool = True,
                    mass_out=None, mask_out=None, workspace=None, stream=None):
    """NEXT(3): dense attention at the decision scale with the predictor fused in.  Returns
    (o, mask, mass or None); mask / mass as predict_pattern's."""
    g = geometry(sides, decision_scale, block)
    bh = q_S.shape[0]
    if o is None:
        o = torch.empty_like(q_S)
    if mask_out is None:
        mask_out = torch.empty((bh, g["G_q"], g["W"]), dtype=torch.int32, device="cuda")
    if want_mass and mass_out is None:
        mass_out = torch.empty((bh, g["G_q"], g["G_kv"]), dtype=torch.float32, device="cuda")
    need = dense_attn_mass_workspace(sides, decision_scale, block, bh)
    if workspace is None:
        workspace = torch.empty(max(1, need), dtype=torch.uint8, device="cuda")
    sh = _attn_shape(q_S, k_cache, o, v_cache, g["C"], g["N"])
    _lse(lse, bh, g["N"])
    _dev_tensor(mask_out, "mask_out", torch.int32, min_numel=bh * g["G_q"] * g["W"])
    if want_mass:
        _dev_tensor(mass_out, "mass_out", torch.float32, min_numel=bh * g["G_q"] * g["G_kv"])
    _dev_tensor(workspace, "workspace", torch.uint8)     # size: checked by the ABI (CAPACITY)
    _check(lib.sparvar_dense_attn_mass(
        ctypes.byref(_sched(sides)), decision_scale, block, sink_scales, ctypes.byref(sh),
        _ptr(q_S), _ptr(k_cache), _ptr(v_cache), softmax_scale, mode, topk, threshold, _ptr(o),
        _ptr(lse), _ptr(mass_out if want_mass else None), _ptr(mask_out), _ptr(workspace),
        workspace.numel() * workspace.element_size(), _stream(stream)))
    return o, mask_out, (mass_out if want_mass else None)


def dense_attn_mass_workspace(sides, decision_scale: int, block: int, bh: int) -> int:
    """Bytes of device workspace dense_attn_mass needs."""
    return int(lib.sparvar_dense_attn_mass_workspace(ctypes.byref(_sched(sides)), decision_scale,
                                                      block, bh))


# ------------------------------------------------------------------ NEXT(2): token-level CS4A
def token_colsum(sides, decision_scale: int, C: int, q_S, k_cache, lse_S, softmax_scale=0.0,
                 out=None, stream=None):
    """A[bh, g, j] = sum over query block g (C rows) of P[q, j] at S."""
    N, Ck = sides[decision_scale - 1] ** 2, sum(s * s for s in sides[:decision_scale])
    bh, D = q_S.shape[0], q_S.shape[2]
    if out is None:
        out = torch.empty((bh, -(-N // C), Ck), dtype=torch.float32, device="cuda")
    sh = _Shape(bh, D, _bh_view(q_S, "q_S"), _bh_view(k_cache, "k_cache"), 0)
    if k_cache.shape[0] < bh or k_cache.shape[1] < Ck or q_S.shape[1] < N:
        raise ValueError("k_cache / q_S too small for the decision scale")
    _lse(lse_S, bh, N)
    if lse_S is None:
        raise ValueError("lse_S is required")
    _dev_tensor(out, "out", torch.float32, min_numel=bh * -(-N // C) * Ck)
    _check(lib.sparvar_token_colsum(ctypes.byref(_sched(sides)), decision_scale, C,
                                    ctypes.byref(sh), _ptr(q_S), _ptr(k_cache), _ptr(lse_S),
                                    softmax_scale, _ptr(out), _stream(stream)))
    return out


def token_select(sides, decision_scale: int, C: int, sink_scales: int, colsum, topk_tokens: int,
                 out=None, stream=None):
    bh, G, Ck = colsum.shape
    if G != -(-(sides[decision_scale - 1] ** 2) // C) or Ck != _kv_rows(sides, decision_scale):
        raise ValueError("colsum must be (bh, ceil(N_S / C), C_S)")
    _dev_tensor(colsum, "colsum", torch.float32)
    if out is None:
        out = torch.empty((bh, G, -(-Ck // 32)), dtype=torch.int32, device="cuda")
    _dev_tensor(out, "out", torch.int32, min_numel=bh * G * -(-Ck // 32))
    _check(lib.sparvar_token_select(ctypes.byref(_sched(sides)), decision_scale, C, sink_scales, bh,
                                    _ptr(colsum), topk_tokens, _ptr(out), _stream(stream)))
    return out


def token_map(sides, src_scale: int, dst_scale: int, C: int, sink_scales: int, src_mask,
              mode: int = MAP_FOOTPRINT, out=None, stream=None):
    bh = src_mask.shape[0]
    G_K = -(-(sides[dst_scale - 1] ** 2) // C)
    Ck = sum(s * s for s in sides[:dst_scale])
    G_S = -(-(sides[src_scale - 1] ** 2) // C)
    _dev_tensor(src_mask, "src_mask", torch.int32,
                min_numel=bh * G_S * -(-_kv_rows(sides, src_scale) // 32))
    if out is None:
        out = torch.empty((bh, G_K, -(-Ck // 32)), dtype=torch.int32, device="cuda")
    _dev_tensor(out, "out", torch.int32, min_numel=bh * G_K * -(-Ck // 32))
    _check(lib.sparvar_token_map(ctypes.byref(_sched(sides)), src_scale, dst_scale, C, sink_scales,
                                 mode, bh, _ptr(src_mask), _ptr(out), _stream(stream)))
    return out


def token_sparse_attn(sides, target: int, C: int, q, k_cache, v_cache, row_ptr, col_idx,
                      softmax_scale: float = 0.0, o=None, stream=None):
    if o is None:
        o = torch.empty_like(q)
    n_q = sides[target - 1] ** 2
    sh = _attn_shape(q, k_cache, o, v_cache, _kv_rows(sides, target), n_q)
    _csr(row_ptr, col_idx, q.shape[0] * -(-n_q // C))
    _check(lib.sparvar_token_sparse_attn(ctypes.byref(_sched(sides)), target, C, ctypes.byref(sh),
                                         _ptr(q), _ptr(k_cache), _ptr(v_cache), _ptr(row_ptr),
                                         _ptr(col_idx), softmax_scale, _ptr(o), _stream(stream)))
    return o


def token_cache_residual(sides, decision_scale: int, C: int, q_S, k_cache, v_cache, row_ptr_S,
                         col_idx_S, o_dense, softmax_scale: float = 0.0, o_cache=None,
                         stream=None):
    """Token-level O_cache = o_dense - token attention at S over the selected tokens."""
    if o_cache is None:
        o_cache = torch.empty_like(q_S)
    if _bh_view(o_dense, "o_dense") != o_cache.stride(0):
        raise ValueError("o_dense and o_cache must share a (b,h) stride")
    n_q = sides[decision_scale - 1] ** 2
    sh = _attn_shape(q_S, k_cache, o_cache, v_cache, _kv_rows(sides, decision_scale), n_q)
    _attn_shape(q_S, k_cache, o_dense, v_cache, _kv_rows(sides, decision_scale), n_q)
    _csr(row_ptr_S, col_idx_S, q_S.shape[0] * -(-n_q // C))
    _check(lib.sparvar_token_cache_residual(
        ctypes.byref(_sched(sides)), decision_scale, C, ctypes.byref(sh), _ptr(q_S), _ptr(k_cache),
        _ptr(v_cache), _ptr(row_ptr_S), _ptr(col_idx_S), softmax_scale, _ptr(o_dense),
        _ptr(o_cache), _stream(stream)))
    return o_cache


def token_sparse_attn_cached(sides, target: int, C: int, q, k_cache, v_cache, row_ptr, col_idx,
                             o_cache, cache_scale: int, softmax_scale: float = 0.0, o=None,
                             stream=None):
    """Token-list attention at K plus the NN-upsampled token-level O_cache."""
    if o is None:
        o = torch.empty_like(q)
    cstride = _bh_view(o_cache, "o_cache")
    n_q = sides[target - 1] ** 2
    sh = _attn_shape(q, k_cache, o, v_cache, _kv_rows(sides, target), n_q)
    _csr(row_ptr, col_idx, q.shape[0] * -(-n_q // C))
    _cache_in(o_cache, q.shape[0], sides[cache_scale - 1] ** 2, q.shape[2])
    _check(lib.sparvar_token_sparse_attn_cached(
        ctypes.byref(_sched(sides)), target, C, ctypes.byref(sh), _ptr(q), _ptr(k_cache),
        _ptr(v_cache), _ptr(row_ptr), _ptr(col_idx), softmax_scale, _ptr(o_cache), cache_scale,
        cstride, _ptr(o), _stream(stream)))
    return o


# ------------------------------------------------------------------ NEXT(4): compressed KV
def _win(windows):
    return (ctypes.c_int32 * max(1, len(windows)))(*[int(x) for x in windows])


def csla_kept_rows(sides, target: int, sink_scales: int = 5, windows=(7, 5, 3, 1, 1)) -> int:
    """Rows of the compressed cache of a CSLA layer at `target` (sink + windowed scales)."""
    n = int(lib.sparvar_csla_kept_rows(ctypes.byref(_sched(sides)), target, sink_scales,
                                       _win(windows), len(windows)))
    if n < 0:
        raise SparVARError(1, "invalid arguments")
    return n


def compress_kv(sides, target: int, cache, sink_scales: int = 5, windows=(7, 5, 3, 1, 1),
                out=None, stream=None):
    """(bh, >= C_K, D) bf16 cache -> (bh, kept, D): the CSLA layer's sink + local scales."""
    bh, _, D = cache.shape
    kept = csla_kept_rows(sides, target, sink_scales, windows)
    if cache.shape[1] < _kv_rows(sides, target):
        raise ValueError(f"cache needs >= {_kv_rows(sides, target)} rows")
    if out is None:
        out = torch.empty((bh, kept, D), dtype=cache.dtype, device=cache.device)
    if out.shape[0] < bh or out.shape[1] < kept or out.shape[2] != D:
        raise ValueError(f"out must be (>= {bh}, >= {kept}, {D})")
    _check(lib.sparvar_compress_kv(ctypes.byref(_sched(sides)), target, sink_scales, _win(windows),
                                   len(windows), bh, D, _ptr(cache), _bh_view(cache, "cache"),
                                   _ptr(out), _bh_view(out, "out"), _stream(stream)))
    return out


def local_mask_compressed(sides, target: int, block: int, sink_scales: int = 5,
                          windows=(7, 5, 3, 1, 1), out=None, stream=None):
    kept = csla_kept_rows(sides, target, sink_scales, windows)
    g_q = -(-(sides[target - 1] ** 2) // block)
    W = -(-(-(-kept // block)) // 32)
    if out is None:
        out = torch.empty((g_q, W), dtype=torch.int32, device="cuda")
    _check(lib.sparvar_local_mask_compressed(ctypes.byref(_sched(sides)), target, block, sink_scales,
                                             _win(windows), len(windows), _ptr(out),
                                             _stream(stream)))
    return out


def block_sparse_attn_rows(sides, target: int, block: int, q, k_cache, v_cache, kv_rows: int,
                           row_ptr, col_idx, softmax_scale: float = 0.0, o=None, lse=None,
                           stream=None):
    """block_sparse_attn over a cache with kv_rows valid rows (e.g. the compressed cache)."""
    if o is None:
        o = torch.empty_like(q)
    g = geometry(sides, target, block)
    sh = _attn_shape(q, k_cache, o, v_cache, int(kv_rows), g["N"])
    _csr(row_ptr, col_idx, q.shape[0] * g["G_q"])
    _lse(lse, q.shape[0], g["N"])
    _check(lib.sparvar_block_sparse_attn_rows(ctypes.byref(_sched(sides)), target, block,
                                              ctypes.byref(sh), _ptr(q), _ptr(k_cache),
                                              _ptr(v_cache), kv_rows, _ptr(row_ptr), _ptr(col_idx),
                                              softmax_scale, _ptr(o), _ptr(lse), _stream(stream)))
    return o


def block_sparse_attn_cached(sides, target: int, block: int, q, k_cache, v_cache, row_ptr,
                             col_idx, o_cache, cache_scale: int, softmax_scale: float = 0.0,
                             o=None, lse=None, stream=None):
    """NEXT(1): O^(K) = NN-upsample(O_cache) + Delta O^(K), fused epilogue."""
    if o is None:
        o = torch.empty_like(q)
    cstride = _bh_view(o_cache, "o_cache")
    g = geometry(sides, target, block)
    sh = _attn_shape(q, k_cache, o, v_cache, g["C"], g["N"])
    _csr(row_ptr, col_idx, q.shape[0] * g["G_q"])
    _lse(lse, q.shape[0], g["N"])
    _cache_in(o_cache, q.shape[0], sides[cache_scale - 1] ** 2, q.shape[2])
    _check(lib.sparvar_block_sparse_attn_cached(
        ctypes.byref(_sched(sides)), target, block, ctypes.byref(sh), _ptr(q), _ptr(k_cache),
        _ptr(v_cache), _ptr(row_ptr), _ptr(col_idx), softmax_scale, _ptr(o_cache), cache_scale,
        cstride, _ptr(o), _ptr(lse), _stream(stream)))
    return o


class SparseLayer:
    """The whole hot path for one attention layer at target scale K:

        CSLA layer : local_mask(K) -> build_block_lists([local]) -> block_sparse_attn
        CS4A layer : predict_pattern(S) -> map_indices(S->K) -> build_block_lists([mapped])
                     -> block_sparse_attn
        union      : all three masks OR-ed (READING 19)

    Sink order (DESIGN.md READING 25): by default the S-level pattern is the Top-K alone
     and the sink is added by the mapping at K (A_sink U M(inds^(S)),
    PAPER.md:883-890).  sink_in_source=True ORs the sink into the S-level pattern as well, so
    the mapping also carries the sink blocks' footprint to K.

    Buffers for masks and lists are allocated once (sized from the geometry) and reused, so a
    step is kernel launches only.
    """

    def __init__(self, sides, target: int, decision: int, block: int, bh: int,
                 sink_scales: int = 5, windows=(7, 5, 3, 1, 1), select_mode=SELECT_TOPK,
                 topk: int = 5, threshold: float = 0.01, map_mode=MAP_FOOTPRINT,
                 kinds: Sequence[str] = ("csla", "cs4a", "union"), sink_in_source: bool = False):
        self.sides, self.K, self.S, self.B, self.bh = list(sides), target, decision, block, bh
        self.sink, self.windows = sink_scales, tuple(windows)
        self.sink_in_source = bool(sink_in_source)
        self.sink_S = sink_scales if sink_in_source else 0      # READING 25
        self.kinds = tuple(kinds)   # list sets built by build_patterns (READING 19 policies)
        self.select_mode, self.topk, self.threshold, self.map_mode = select_mode, topk, threshold, map_mode
        gk, gs = geometry(sides, target, block), geometry(sides, decision, block)
        self.gk, self.gs = gk, gs
        dev = "cuda"
        self.local = torch.empty((gk["G_q"], gk["W"]), dtype=torch.int32, device=dev)
        self.src = torch.empty((bh, gs["G_q"], gs["W"]), dtype=torch.int32, device=dev)
        self.mass = torch.empty((bh, gs["G_q"], gs["G_kv"]), dtype=torch.float32, device=dev)
        self.mapped = torch.empty((bh, gk["G_q"], gk["W"]), dtype=torch.int32, device=dev)
        cap = bh * gk["G_q"] * gk["G_kv"]
        self.lists = {}
        for name in self.kinds:
            self.lists[name] = (torch.empty(bh * gk["G_q"] + 1, dtype=torch.int32, device=dev),
                                torch.empty(cap, dtype=torch.int32, device=dev))
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.cap = cap

    def build_patterns(self, q_S, k_cache, stream=None, predict: bool = True):
        """a1-a5: CSLA mask, decision-scale prediction, mapping, and the CSR list sets.
        predict=False reuses the S-level pattern already in self.src (bench.py times the
        predictor launch on its own)."""
        local_mask(self.sides, self.K, self.B, self.sink, self.windows, out=self.local, stream=stream)
        if predict:
            self.predict(q_S, k_cache, stream)
        map_indices(self.sides, self.S, self.K, self.B, self.sink, self.src, self.map_mode,
                    out=self.mapped, stream=stream)
        g = self.gk
        for name in self.kinds:
            rp, ci = self.lists[name]
            build_block_lists(self.bh, g["G_q"], g["G_kv"], self._masks(name), self.cap, rp, ci,
                              self.status, stream=stream)

    def predict(self, q_S, k_cache, stream=None):
        """a2/a3: the S-level pattern (Top-K alone unless sink_in_source, READING 25)."""
        predict_pattern(self.sides, self.S, self.B, self.sink_S, q_S, k_cache, self.select_mode,
                        self.topk, self.threshold, mask_out=self.src, mass_out=self.mass,
                        stream=stream)

    def _masks(self, which):
        return {"csla": [(self.local, True)], "cs4a": [(self.mapped, False)],
                "union": [(self.local, True), (self.mapped, False)]}[which]

    def attend(self, which: str, q, k_cache, v_cache, o=None, lse=None, stream=None):
        """a6 on the lists `which` in {'csla', 'cs4a', 'union'}."""
        rp, ci = self.lists[which]
        return block_sparse_attn(self.sides, self.K, self.B, q, k_cache, v_cache, rp, ci, o=o,
                                 lse=lse, stream=stream)
