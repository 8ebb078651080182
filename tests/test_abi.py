"""CPU-only checks of the C ABI library: it loads, exports every symbol include/sparvar.h
declares, and rejects bad arguments on the host (no kernel is launched on these paths)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sparvar.h")


@pytest.fixture(scope="module")
def sv():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2602_04361_b200 as pkg
    return pkg


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(sparvar_[a-z_]+)\s*\(", txt)))


def test_exports_every_declared_symbol(sv):
    names = _declared()
    assert "sparvar_block_sparse_attn" in names and len(names) == 23
    L = ctypes.CDLL(sv.LIB_PATH)
    for n in names:
        assert hasattr(L, n), n


def test_version_and_error_string(sv):
    assert sv.lib.sparvar_version() == 105
    assert isinstance(sv.lib.sparvar_last_error(), bytes)


def _sched(sv, sides):
    return ctypes.byref(sv._sched(sides))


def test_schedule_validation(sv):
    out = ctypes.c_void_p(16)   # never dereferenced: validation fails first
    w = (ctypes.c_int32 * 1)(3)
    st = sv.lib.sparvar_local_mask(_sched(sv, [2, 1]), 2, 16, 0, w, 1, out, None)
    assert st == 2 and b"non-decreasing" in sv.lib.sparvar_last_error()
    st = sv.lib.sparvar_local_mask(_sched(sv, [1, 2]), 3, 16, 0, w, 1, out, None)
    assert st == 1
    w2 = (ctypes.c_int32 * 1)(4)
    st = sv.lib.sparvar_local_mask(_sched(sv, [1, 2]), 2, 16, 0, w2, 1, out, None)
    assert st == 1 and b"odd" in sv.lib.sparvar_last_error()


def test_attention_validation(sv):
    sh = sv._Shape(1, 96, 64 * 96, 85 * 96, 64 * 96)     # head_dim 96 unsupported
    p = ctypes.c_void_p(256)
    st = sv.lib.sparvar_dense_attn(_sched(sv, [1, 2, 4, 8]), 4, ctypes.byref(sh), p, p, p, 0.0,
                                   p, None, None)
    assert st == 3
    sh = sv._Shape(1, 64, 64 * 64, 80 * 64, 64 * 64)     # kv stride < C_K * D
    st = sv.lib.sparvar_block_sparse_attn(_sched(sv, [1, 2, 4, 8]), 4, 16, ctypes.byref(sh), p, p,
                                          p, p, p, 0.0, p, None, None)
    assert st == 1 and b"kv_stride" in sv.lib.sparvar_last_error()
    sh = sv._Shape(1, 64, 64 * 64, 85 * 64 + 3, 64 * 64)  # stride not a multiple of 8
    st = sv.lib.sparvar_dense_attn(_sched(sv, [1, 2, 4, 8]), 4, ctypes.byref(sh), p, p, p, 0.0,
                                   p, None, None)
    assert st == 1
    sh = sv._Shape(1, 64, 64 * 64, 88 * 64, 64 * 64)
    st = sv.lib.sparvar_block_sparse_attn(_sched(sv, [1, 2, 4, 8]), 4, 48, ctypes.byref(sh), p, p,
                                          p, p, p, 0.0, p, None, None)
    assert st == 3                                         # block 48 unsupported


def test_predict_and_map_validation(sv):
    p = ctypes.c_void_p(256)
    sh = sv._Shape(1, 64, 16 * 64, 21 * 64, 0)
    st = sv.lib.sparvar_predict_pattern(_sched(sv, [1, 2, 4, 8]), 3, 16, 0, ctypes.byref(sh), p, p,
                                        0.0, 0, 0, 0.0, None, p, None)
    assert st == 1 and b"topk" in sv.lib.sparvar_last_error()
    st = sv.lib.sparvar_map_indices(_sched(sv, [1, 2, 4, 8]), 4, 3, 16, 0, 0, 1, p, p, None)
    assert st == 1
    st = sv.lib.sparvar_map_indices(_sched(sv, [1, 2, 4, 8]), 3, 4, 16, 0, 7, 1, p, p, None)
    assert st == 1


def test_build_lists_validation(sv):
    p = ctypes.c_void_p(256)
    masks = (ctypes.c_void_p * 1)(256)
    bc = (ctypes.c_int32 * 1)(0)
    st = sv.lib.sparvar_build_block_lists(1, 1, 1, masks, bc, 0, p, p, 10, None, None)
    assert st == 1
    st = sv.lib.sparvar_build_block_lists(0, 1, 1, masks, bc, 1, p, p, 10, None, None)
    assert st == 1


def test_no_fallback_when_library_missing(tmp_path, monkeypatch):
    """The binding raises on import when libsparvar.so is absent (no CPU fallback)."""
    import importlib.util
    import shutil
    pkg = tmp_path / "paper_2602_04361_b200"
    pkg.mkdir()
    shutil.copy(os.path.join(ROOT, "paper_2602_04361_b200", "__init__.py"), pkg / "__init__.py")
    spec = importlib.util.spec_from_file_location("sv_nolib", pkg / "__init__.py")
    mod = importlib.util.module_from_spec(spec)
    with pytest.raises(ImportError):
        spec.loader.exec_module(mod)


def test_next_rows_validation(sv):
    """Host-side validation of the NEXT(1)-(4) entry points (no device work is reached)."""
    p = ctypes.c_void_p(256)
    S4 = _sched(sv, [1, 2, 4, 8])
    sh = sv._Shape(1, 64, 64 * 64, 85 * 64, 64 * 64)
    # token path: query_block outside {64, 128, 192}
    st = sv.lib.sparvar_token_colsum(S4, 3, 100, ctypes.byref(sh), p, p, p, 0.0, p, None)
    assert st == 3 and b"query_block" in sv.lib.sparvar_last_error()
    st = sv.lib.sparvar_token_sparse_attn(S4, 4, 96, ctypes.byref(sh), p, p, p, p, p, 0.0, p, None)
    assert st == 3
    st = sv.lib.sparvar_token_select(S4, 3, 64, 0, 1, p, 0, p, None)      # topk_tokens < 1
    assert st == 1
    st = sv.lib.sparvar_token_map(S4, 4, 3, 64, 0, 0, 1, p, p, None)      # src > dst
    assert st == 1
    # cached paths: cache_scale above the target, o_dense aliasing o_cache
    st = sv.lib.sparvar_token_sparse_attn_cached(S4, 3, 64, ctypes.byref(sh), p, p, p, p, p, 0.0,
                                                 p, 4, 64 * 64, p, None)
    assert st == 1
    st = sv.lib.sparvar_cache_residual_from_dense(S4, 3, 16, ctypes.byref(sh), p, p, p, p, p, 0.0,
                                                  p, p, None)
    assert st == 1 and b"alias" in sv.lib.sparvar_last_error()
    # fused dense + mass: workspace too small -> CAPACITY before any launch
    need = sv.lib.sparvar_dense_attn_mass_workspace(S4, 3, 16, 1)
    assert need > 0
    st = sv.lib.sparvar_dense_attn_mass(S4, 3, 16, 1, ctypes.byref(sh), p, p, p, 0.0, 0, 2, 0.0,
                                        p, None, None, p, p, need - 16, None)
    assert st == 4
    # compressed KV: kept rows and window validation
    w = (ctypes.c_int32 * 2)(3, 1)
    assert sv.lib.sparvar_csla_kept_rows(S4, 4, 1, w, 2) == 1 + 16 + 64
    bad = (ctypes.c_int32 * 1)(2)
    assert sv.lib.sparvar_csla_kept_rows(S4, 4, 1, bad, 1) == -1
    st = sv.lib.sparvar_local_mask_compressed(S4, 4, 16, 1, bad, 1, p, None)
    assert st == 1 and b"odd" in sv.lib.sparvar_last_error()
    st = sv.lib.sparvar_block_sparse_attn_rows(S4, 4, 16, ctypes.byref(sh), p, p, p, 86, p, p, 0.0,
                                               p, None, None)   # more rows than C_K = 85
    assert st == 1


def test_kv_step_bound_and_cached_schedule_checks(sv):
    """the attention kernel holds a tile's KV step count in 16 bits, so a cache of more
    than 65535 blocks is rejected up front (UNSUPPORTED); the cached entry points validate the
    schedule before reading it (a NULL `sides` is INVALID_ARG, not a crash)."""
    p = ctypes.c_void_p(256)
    big = _sched(sv, [1024, 1025])                      # C_2 = 2,099,201 rows -> 131,201 blocks
    sh = sv._Shape(1, 64, 1025 * 1025 * 64, 2099201 * 64, 1025 * 1025 * 64)
    st = sv.lib.sparvar_block_sparse_attn(big, 2, 16, ctypes.byref(sh), p, p, p, p, p, 0.0, p,
                                          None, None)
    assert st == 3 and b"steps per tile" in sv.lib.sparvar_last_error()
    null = sv._Schedule(2, ctypes.POINTER(ctypes.c_int32)())
    st = sv.lib.sparvar_block_sparse_attn_cached(ctypes.byref(null), 2, 16, ctypes.byref(sh), p, p,
                                                 p, p, p, 0.0, p, 1, 64, p, None, None)
    assert st == 1 and b"null schedule" in sv.lib.sparvar_last_error()
    st = sv.lib.sparvar_token_sparse_attn_cached(ctypes.byref(null), 2, 64, ctypes.byref(sh), p, p,
                                                 p, p, p, 0.0, p, 1, 64, p, None)
    assert st == 1 and b"null schedule" in sv.lib.sparvar_last_error()


def test_binding_rejects_bad_tensors(sv):
    """the Python wrappers check what the C ABI cannot see (allocation sizes, dtypes,
    devices) before passing raw pointers; CPU tensors and wrong dtypes are refused."""
    import torch
    q = torch.zeros((2, 64, 64), dtype=torch.bfloat16)
    with pytest.raises(ValueError):
        sv.dense_attn([1, 2, 4, 8], 4, q, q, q)                  # not CUDA
    with pytest.raises(ValueError):
        sv._dev_tensor(torch.zeros(4, dtype=torch.int64), "row_ptr", torch.int32)
    with pytest.raises(ValueError):
        sv._dev_tensor(torch.zeros(4, dtype=torch.int32), "row_ptr", torch.int32)   # CPU
