// api.cu — the C ABI of libsparvar.so (include/sparvar.h): host-side validation, scale geometry,
// TMA tensor-map construction and kernel launches.  No state is kept between calls.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/sparvar.h"
#include "kernels.h"

namespace {

thread_local std::string g_err;

sparvar_status fail(sparvar_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

sparvar_status cuda_fail(cudaError_t e, const char* what) {
  return fail(SPARVAR_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

sparvar_status ok() {
  g_err.clear();
  return SPARVAR_OK;
}

// Schedule -> Geo.  Sides non-decreasing, >= 1.
sparvar_status make_geo(const sparvar_schedule* s, sv::Geo* g) {
  if (s == nullptr || s->sides == nullptr) return fail(SPARVAR_ERR_INVALID_ARG, "null schedule");
  if (s->num_scales < 1 || s->num_scales > sv::kMaxScales)
    return fail(SPARVAR_ERR_SCHEDULE, "num_scales %d not in [1, %d]", s->num_scales, sv::kMaxScales);
  *g = sv::Geo{};
  g->K = s->num_scales;
  long long c = 0;
  g->cum[0] = 0;
  for (int i = 0; i < s->num_scales; ++i) {
    const int side = s->sides[i];
    if (side < 1) return fail(SPARVAR_ERR_SCHEDULE, "side[%d] = %d < 1", i, side);
    if (i > 0 && side < s->sides[i - 1])
      return fail(SPARVAR_ERR_SCHEDULE, "sides must be non-decreasing (side[%d] = %d < %d)", i,
                  side, s->sides[i - 1]);
    if (side > 46340) return fail(SPARVAR_ERR_SCHEDULE, "side[%d] too large", i);
    g->side[i] = side;
    c += (long long)side * side;
    if (c >= (1LL << 31)) return fail(SPARVAR_ERR_SCHEDULE, "schedule exceeds 2^31 tokens");
    g->cum[i + 1] = (int)c;
  }
  return SPARVAR_OK;
}

int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

bool attn_block_ok(int b) { return b == 16 || b == 32 || b == 64 || b == 128; }

// ---------------------------------------------------------------------------- TMA descriptors
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (fn == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// bf16 tensor viewed as (D, rows, bh): box (64, box_rows, 1), 128-byte swizzle.  Rows >= `rows`
// of a slab are out of bounds and read as zeros (never the next slab's data).
sparvar_status make_tmap(CUtensorMap* m, const void* base, int D, long long rows, int bh,
                         long long stride_bh_elems, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (fn == nullptr) return fail(SPARVAR_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)rows, (cuuint64_t)bh};
  cuuint64_t strides[2] = {(cuuint64_t)D * 2, (cuuint64_t)stride_bh_elems * 2};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SPARVAR_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return SPARVAR_OK;
}

sparvar_status check_shape(const sparvar_attn_shape* sh, long long n_q, long long n_kv, bool need_o) {
  if (sh == nullptr) return fail(SPARVAR_ERR_INVALID_ARG, "null shape");
  if (sh->head_dim != 64 && sh->head_dim != 128)
    return fail(SPARVAR_ERR_UNSUPPORTED, "head_dim %d not in {64, 128}", sh->head_dim);
  if (sh->batch_heads < 1 || sh->batch_heads > 65535)
    return fail(SPARVAR_ERR_INVALID_ARG, "batch_heads %d not in [1, 65535]", sh->batch_heads);
  const long long D = sh->head_dim;
  if (sh->q_stride_bh < n_q * D || sh->q_stride_bh % 8)
    return fail(SPARVAR_ERR_INVALID_ARG, "q_stride_bh must be >= N*D and a multiple of 8");
  if (sh->kv_stride_bh < n_kv * D || sh->kv_stride_bh % 8)
    return fail(SPARVAR_ERR_INVALID_ARG, "kv_stride_bh must be >= C_k*D and a multiple of 8");
  if (need_o && (sh->o_stride_bh < n_q * D || sh->o_stride_bh % 8))
    return fail(SPARVAR_ERR_INVALID_ARG, "o_stride_bh must be >= N*D and a multiple of 8");
  return SPARVAR_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

extern "C" {

const char* sparvar_last_error(void) { return g_err.c_str(); }

int32_t sparvar_version(void) { return 105; }   // 1.05: + compressed KV for CSLA layers (NEXT(4))

sparvar_status sparvar_local_mask(const sparvar_schedule* sched, int32_t target_scale,
                                  int32_t block, int32_t sink_scales, const int32_t* windows,
                                  int32_t num_windows, uint32_t* mask_out, void* stream) {
  sv::Geo g;
  sparvar_status s = make_geo(sched, &g);
  if (s != SPARVAR_OK) return s;
  if (target_scale < 1 || target_scale > g.K)
    return fail(SPARVAR_ERR_INVALID_ARG, "target_scale %d not in [1, %d]", target_scale, g.K);
  if (block < 1) return fail(SPARVAR_ERR_INVALID_ARG, "block %d < 1", block);
  if (sink_scales < 0 || sink_scales > target_scale)
    return fail(SPARVAR_ERR_INVALID_ARG, "sink_scales %d not in [0, %d]", sink_scales, target_scale);
  if (num_windows < 0 || num_windows > sv::kMaxScales || (num_windows > 0 && windows == nullptr))
    return fail(SPARVAR_ERR_INVALID_ARG, "bad windows array");
  if (mask_out == nullptr) return fail(SPARVAR_ERR_INVALID_ARG, "null mask_out");
  int rel[sv::kMaxScales] = {0};
  for (int i = 0; i < num_windows; ++i) {
    if (windows[i] < 0 || (windows[i] > 0 && windows[i] % 2 == 0))
      return fail(SPARVAR_ERR_INVALID_ARG, "window %d must be 0 or odd", windows[i]);
    rel[i] = windows[i];
  }
  cudaError_t e = sv::launch_local_mask(g, target_scale, block, sink_scales, rel, mask_out,
                                        (cudaStream_t)stream);
  if (e == cudaErrorInvalidValue)
    return fail(SPARVAR_ERR_UNSUPPORTED, "mask row too wide for shared memory");
  if (e != cudaSuccess) return cuda_fail(e, "local_mask launch");
  return ok();
}

// ---------------------------------------------------------------- NEXT(4): compressed KV
static sparvar_status csla_windows(const int32_t* windows, int32_t num_windows, int* rel) {
  if (num_windows < 0 || num_windows > sv::kMaxScales || (num_windows > 0 && windows == nullptr))
    return fail(SPARVAR_ERR_INVALID_ARG, "bad windows array");
  for (int i = 0; i < sv::kMaxScales; ++i) rel[i] = 0;
  for (int i = 0; i < num_windows; ++i) {
    if (windows[i] < 0 || (windows[i] > 0 && windows[i] % 2 == 0))
      return fail(SPARVAR_ERR_INVALID_ARG, "window %d must be 0 or odd", windows[i]);
    rel[i] = windows[i];
  }
  return SPARVAR_OK;
}

int64_t sparvar_csla_kept_rows(const sparvar_schedule* sched, int32_t target_scale,
                               int32_t sink_scales, const int32_t* windows, int32_t num_windows) {
  sv::Geo g;
  int rel[sv::kMaxScales];
  if (make_geo(sched, &g) != SPARVAR_OK || target_scale < 1 || target_scale > g.K ||
      csla_windows(windows, num_windows, rel) != SPARVAR_OK)
    return -1;
  long long n = 0;
  for (int h = 1; h <= target_scale; ++h)
    if (h <= sink_scales || rel[target_scale - h] > 0) n += (long long)g.side[h - 1] * g.side[h - 1];
  return n;
}

sparvar_status sparvar_local_mask_compressed(const sparvar_schedule* sched, int32_t target_scale,
                                             int32_t block, int32_t sink_scales,
                                             const int32_t* windows, int32_t num_windows,
                                             uint32_t* mask_out, void* stream) {
  sv::Geo g;
  sparvar_status s = make_geo(sched, &g);
  if (s != SPARVAR_OK) return s;
  if (target_scale < 1 || target_scale > g.K)
    return fail(SPARVAR_ERR_INVALID_ARG, "target_scale %d not in [1, %d]", target_scale, g.K);
  if (block < 1) return fail(SPARVAR_ERR_INVALID_ARG, "block %d < 1", block);
  if (sink_scales < 0 || sink_scales > target_scale)
    return fail(SPARVAR_ERR_INVALID_ARG, "sink_scales %d not in [0, %d]", sink_scales, target_scale);
  int rel[sv::kMaxScales];
  if ((s = csla_windows(windows, num_windows, rel)) != SPARVAR_OK) return s;
  if (mask_out == nullptr) return fail(SPARVAR_ERR_INVALID_ARG, "null mask_out");
  cudaError_t e = sv::launch_local_mask(g, target_scale, block, sink_scales, rel, mask_out,
                                        (cudaStream_t)stream, true);
  if (e == cudaErrorInvalidValue)
    return fail(SPARVAR_ERR_UNSUPPORTED, "mask row too wide for shared memory");
  if (e != cudaSuccess) return cuda_fail(e, "local_mask launch");
  return ok();
}

sparvar_status sparvar_compress_kv(const sparvar_schedule* sched, int32_t target_scale,
                                   int32_t sink_scales, const int32_t* windows,
                                   int32_t num_windows, int32_t batch_heads, int32_t head_dim,
                                   const uint16_t* cache_in, int64_t in_stride_bh,
                                   uint16_t* cache_out, int64_t out_stride_bh, void* stream) {
  sv::Geo g;
  sparvar_status s = make_geo(sched, &g);
  if (s != SPARVAR_OK) return s;
  if (target_scale < 1 || target_scale > g.K)
    return fail(SPARVAR_ERR_INVALID_ARG, "target_scale %d not in [1, %d]", target_scale, g.K);
  if (sink_scales < 0 || sink_scales > target_scale)
    return fail(SPARVAR_ERR_INVALID_ARG, "sink_scales %d not in [0, %d]", sink_scales, target_scale);
  int rel[sv::kMaxScales];
  if ((s = csla_windows(windows, num_windows, rel)) != SPARVAR_OK) return s;
  if (batch_heads < 1 || (head_dim != 64 && head_dim != 128))
    return fail(SPARVAR_ERR_INVALID_ARG, "batch_heads %d / head_dim %d", batch_heads, head_dim);
  if (cache_in == nullptr || cache_out == nullptr) return fail(SPARVAR_ERR_INVALID_ARG, "null cache");
  const long long kept = sparvar_csla_kept_rows(sched, target_scale, sink_scales, windows, num_windows);
  if (in_stride_bh < (long long)g.cum[target_scale] * head_dim || out_stride_bh < kept * head_dim)
    return fail(SPARVAR_ERR_INVALID_ARG, "stride too small for the (compressed) cache");
  // one 2-D copy (rows of every (b,h)) per maximal run of kept scales
  long long dst_row = 0;
  for (int h = 1; h <= target_scale;) {
    const bool keep = h <= sink_scales || rel[target_scale - h] > 0;
    if (!keep) { ++h; continue; }
    int h1 = h;
    while (h1 + 1 <= target_scale && (h1 + 1 <= sink_scales || rel[target_scale - h1 - 1] > 0)) ++h1;
    const long long r0 = g.cum[h - 1], rows = g.cum[h1] - g.cum[h - 1];
    cudaError_t e = cudaMemcpy2DAsync(cache_out + dst_row * head_dim, out_stride_bh * 2,
                                      cache_in + r0 * head_dim, in_stride_bh * 2,
                                      rows * head_dim * 2, batch_heads, cudaMemcpyDeviceToDevice,
                                      (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "compress copy");
    dst_row += rows;
    h = h1 + 1;
  }
  return ok();
}

sparvar_status sparvar_predict_pattern(const sparvar_schedule* sched, int32_t decision_scale,
                                       int32_t block, int32_t sink_scales,
                                       const sparvar_attn_shape* shape, const uint16_t* q_S,
                                       const uint16_t* k_cache, float softmax_scale,
                                       int32_t select_mode, int32_t topk, float threshold,
                                       float* mass_out, uint32_t* mask_out, void* stream) {
  sv::Geo g;
  sparvar_status s = make_geo(sched, &g);
  if (s != SPARVAR_OK) return s;
  const int S = decision_scale;
  if (S < 1 || S > g.K) return fail(SPARVAR_ERR_INVALID_ARG, "decision_scale %d not in [1, %d]", S, g.K);
  if (!attn_block_ok(block))
    return fail(SPARVAR_ERR_UNSUPPORTED, "block %d not in {16, 32, 64, 128}", block);
  if (sink_scales < 0 || sink_scales > S)
    return fail(SPARVAR_ERR_INVALID_ARG, "sink_scales %d not in [0, %d]", sink_scales, S);
  const long long n_q = (long long)g.side[S - 1] * g.side[S - 1];
  const long long n_kv = g.cum[S];
  s = check_shape(shape, n_q, n_kv, false);
  if (s != SPARVAR_OK) return s;
  if (q_S == nullptr || k_cache == nullptr || mask_out == nullptr)
    return fail(SPARVAR_ERR_INVALID_ARG, "null tensor pointer");
  if (!aligned16(q_S) || !aligned16(k_cache))
    return fail(SPARVAR_ERR_INVALID_ARG, "tensor pointers must be 16-byte aligned");
  if (select_mode != SPARVAR_SELECT_TOPK && select_mode != SPARVAR_SELECT_THRESHOLD)
    return fail(SPARVAR_ERR_INVALID_ARG, "select_mode %d", select_mode);
  if (select_mode == SPARVAR_SELECT_TOPK && topk < 1)
    return fail(SPARVAR_ERR_INVALID_ARG, "topk %d < 1", topk);
  if (select_mode == SPARVAR_SELECT_THRESHOLD && !std::isfinite(threshold))
    return fail(SPARVAR_ERR_INVALID_ARG, "threshold must be finite");
  const int D = shape->head_dim;
  sv::PredArgs a{};
  a.n_q = (int)n_q;
  a.n_kv = (int)n_kv;
  a.g_q = ceil_div(n_q, block);
  a.g_kv = ceil_div(n_kv, block);
  a.bh = shape->batch_heads;
  const float scale = softmax_scale > 0.f ? softmax_scale : 1.0f / std::sqrt((float)D);
  a.scale_log2 = scale * 1.4426950408889634f;
  a.mode = select_mode;
  a.topk = topk;
  a.tau = threshold;
  a.n_sink_blocks = sink_scales > 0 ? ceil_div(g.cum[sink_scales], block) : 0;
  a.mass = mass_out;
  a.mask = mask_out;
  if (sv::predictor_smem_bytes(D, block, a.g_kv) > 227 * 1024)
    return fail(SPARVAR_ERR_UNSUPPORTED,
                "predictor statistics for %d KV blocks do not fit in shared memory", a.g_kv);
  CUtensorMap tq, tk;
  if ((s = make_tmap(&tq, q_S, D, n_q, a.bh, shape->q_stride_bh, 128)) != SPARVAR_OK) return s;
  if ((s = make_tmap(&tk, k_cache, D, n_kv, a.bh, shape->kv_stride_bh, block)) != SPARVAR_OK) return s;
  cudaError_t e = sv::launch_predictor(D, block, tq, tk, a, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "predictor launch");
  return ok();
}

sparvar_status sparvar_map_indices(const sparvar_schedule* sched, int32_t src_scale,
                                   int32_t dst_scale, int32_t block, int32_t sink_scales,
                                   int32_t map_mode, int32_t batch_heads,
                                   const uint32_t* src_mask, uint32_t* dst_mask, void* stream) {
  sv::Geo g;
  sparvar_status s = make_geo(sched, &g);
  if (s != SPARVAR_OK) return s;
  if (src_scale < 1 || dst_scale > g.K || src_scale > dst_scale)
    return fail(SPARVAR_ERR_INVALID_ARG, "need 1 <= src_scale (%d) <= dst_scale (%d) <= %d",
                src_scale, dst_scale, g.K);
  if (block < 1) return fail(SPARVAR_ERR_INVALID_ARG, "block %d < 1", block);
  if (sink_scales < 0 || sink_scales > dst_scale)
    return fail(SPARVAR_ERR_INVALID_ARG, "sink_scales %d not in [0, %d]", sink_scales, dst_scale);
  if (map_mode != SPARVAR_MAP_FOOTPRINT && map_mode != SPARVAR_MAP_POINT)
    return fail(SPARVAR_ERR_INVALID_ARG, "map_mode %d", map_mode);
  if (batch_heads < 1 || batch_heads > 65535)
    return fail(SPARVAR_ERR_INVALID_ARG, "batch_heads %d", batch_heads);
  if (src_mask == nullptr || dst_mask == nullptr)
    return fail(SPARVAR_ERR_INVALID_ARG, "null mask pointer");
  cudaError_t e = sv::launch_map_indices(g, src_scale, dst_scale, block, sink_scales, map_mode,
                                         batch_heads, src_mask, dst_mask, (cudaStream_t)stream);
  if (e == cudaErrorInvalidValue)
    return fail(SPARVAR_ERR_UNSUPPORTED, "mask row too wide for shared memory");
  if (e != cudaSuccess) return cuda_fail(e, "map launch");
  return ok();
}

sparvar_status sparvar_build_block_lists(int32_t batch_heads, int32_t g_q, int32_t g_kv,
                                         const uint32_t* const* masks, const int32_t* broadcast,
                                         int32_t num_masks, int32_t* row_ptr, int32_t* col_idx,
                                         int64_t col_capacity, int32_t* status_dev, void* stream) {
  if (batch_heads < 1 || g_q < 1 || g_kv < 1)
    return fail(SPARVAR_ERR_INVALID_ARG, "batch_heads, g_q, g_kv must be >= 1");
  if ((long long)batch_heads * g_q >= (1LL << 31))
    return fail(SPARVAR_ERR_INVALID_ARG, "too many rows");
  if (num_masks < 1 || num_masks > 8 || masks == nullptr || broadcast == nullptr)
    return fail(SPARVAR_ERR_INVALID_ARG, "need 1..8 masks");
  if (row_ptr == nullptr || (col_idx == nullptr && col_capacity > 0) || col_capacity < 0)
    return fail(SPARVAR_ERR_INVALID_ARG, "null row_ptr / col_idx");
  sv::MaskSet ms{};
  ms.n = num_masks;
  for (int i = 0; i < num_masks; ++i) {
    if (masks[i] == nullptr) return fail(SPARVAR_ERR_INVALID_ARG, "masks[%d] is null", i);
    ms.ptr[i] = masks[i];
    ms.broadcast[i] = broadcast[i] ? 1 : 0;
  }
  cudaError_t e = sv::launch_build_lists(batch_heads, g_q, g_kv, ms, row_ptr, col_idx,
                                         col_capacity, status_dev, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "build_lists launch");
  return ok();
}

static sparvar_status attn_common(const sparvar_schedule* sched, int32_t target_scale,
                                  int32_t block, const sparvar_attn_shape* shape,
                                  const uint16_t* q, const uint16_t* k, const uint16_t* v,
                                  const int32_t* row_ptr, const int32_t* col_idx, float scale_in,
                                  uint16_t* o, float* lse, void* stream,
                                  const uint16_t* add = nullptr, int32_t add_scale = 0,
                                  int64_t add_stride = 0, float* mass_s = nullptr,
                                  float* mass_m = nullptr, long long n_kv_rows = -1) {
  sv::Geo g;
  sparvar_status s = make_geo(sched, &g);
  if (s != SPARVAR_OK) return s;
  if (target_scale < 1 || target_scale > g.K)
    return fail(SPARVAR_ERR_INVALID_ARG, "target_scale %d not in [1, %d]", target_scale, g.K);
  if (!attn_block_ok(block))
    return fail(SPARVAR_ERR_UNSUPPORTED, "block %d not in {16, 32, 64, 128}", block);
  const long long n_q = (long long)g.side[target_scale - 1] * g.side[target_scale - 1];
  const long long n_kv = n_kv_rows >= 0 ? n_kv_rows : g.cum[target_scale];
  if (n_kv < 1 || n_kv > g.cum[target_scale])
    return fail(SPARVAR_ERR_INVALID_ARG, "kv rows %lld not in [1, C_K]", n_kv);
  // a tile's KV step count is kept in 16 bits by the kernel (attention.cu, Small::n): with at
  // most ceil(n_kv / block) steps per tile, bound that here
  if (ceil_div(n_kv, block) > sv::kMaxKvSteps)
    return fail(SPARVAR_ERR_UNSUPPORTED, "%d KV blocks of %d rows exceed the kernel's %d steps per "
                "tile", ceil_div(n_kv, block), block, sv::kMaxKvSteps);
  s = check_shape(shape, n_q, n_kv, true);
  if (s != SPARVAR_OK) return s;
  if (q == nullptr || k == nullptr || v == nullptr || o == nullptr)
    return fail(SPARVAR_ERR_INVALID_ARG, "null tensor pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o))
    return fail(SPARVAR_ERR_INVALID_ARG, "tensor pointers must be 16-byte aligned");
  const int D = shape->head_dim;
  sv::AttnArgs a{};
  a.n_q = (int)n_q;
  a.n_kv = (int)n_kv;
  a.g_q = ceil_div(n_q, block);
  a.bh = shape->batch_heads;
  a.row_ptr = row_ptr;
  a.col_idx = col_idx;
  const float scale = scale_in > 0.f ? scale_in : 1.0f / std::sqrt((float)D);
  a.scale_log2 = scale * 1.4426950408889634f;
  a.o = o;
  a.o_stride = shape->o_stride_bh;
  a.lse = lse;
  a.add = add;
  a.add_stride = add_stride;
  a.s_dst = g.side[target_scale - 1];
  a.s_src = add != nullptr ? g.side[add_scale - 1] : 1;
  a.mass_s = mass_s;
  a.mass_m = mass_m;
  CUtensorMap tq, tk, tv;
  if ((s = make_tmap(&tq, q, D, n_q, a.bh, shape->q_stride_bh, 128)) != SPARVAR_OK) return s;
  if ((s = make_tmap(&tk, k, D, n_kv, a.bh, shape->kv_stride_bh, block)) != SPARVAR_OK) return s;
  if ((s = make_tmap(&tv, v, D, n_kv, a.bh, shape->kv_stride_bh, block)) != SPARVAR_OK) return s;
  cudaError_t e = sv::launch_attention(D, block, tq, tk, tv, a, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "attention launch");
  return ok();
}

sparvar_status sparvar_block_sparse_attn(const sparvar_schedule* sched, int32_t target_scale,
                                         int32_t block, const sparvar_attn_shape* shape,
                                         const uint16_t* q, const uint16_t* k_cache,
                                         const uint16_t* v_cache, const int32_t* row_ptr,
                                         const int32_t* col_idx, float softmax_scale,
                                         uint16_t* o, float* lse, void* stream) {
  if (row_ptr == nullptr || col_idx == nullptr)
    return fail(SPARVAR_ERR_INVALID_ARG, "null row_ptr / col_idx");
  return attn_common(sched, target_scale, block, shape, q, k_cache, v_cache, row_ptr, col_idx,
                     softmax_scale, o, lse, stream);
}

sparvar_status sparvar_cache_residual(const sparvar_schedule* sched, int32_t decision_scale,
                                     int32_t block, const sparvar_attn_shape* shape,
                                     const uint16_t* q_S, const uint16_t* k_cache,
                                     const uint16_t* v_cache, const int32_t* row_ptr_S,
                                     const int32_t* col_idx_S, float softmax_scale,
                                     uint16_t* o_scratch, uint16_t* o_cache, void* stream) {
  if (row_ptr_S == nullptr || col_idx_S == nullptr || o_scratch == nullptr || o_cache == nullptr)
    return fail(SPARVAR_ERR_INVALID_ARG, "null row_ptr / col_idx / output pointer");
  if (o_scratch == o_cache) return fail(SPARVAR_ERR_INVALID_ARG, "o_scratch must not alias o_cache");
  sparvar_status s = attn_common(sched, decision_scale, 128, shape, q_S, k_cache, v_cache, nullptr,
                                 nullptr, softmax_scale, o_cache, nullptr, stream);
  if (s != SPARVAR_OK) return s;
  s = attn_common(sched, decision_scale, block, shape, q_S, k_cache, v_cache, row_ptr_S, col_idx_S,
                  softmax_scale, o_scratch, nullptr, stream);
  if (s != SPARVAR_OK) return s;
  const int side = sched->sides[decision_scale - 1];
  cudaError_t e = sv::launch_residual(shape->batch_heads, side * side, shape->head_dim, o_cache,
                                      shape->o_stride_bh, o_scratch, shape->o_stride_bh, o_cache,
                                      shape->o_stride_bh, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "residual launch");
  return ok();
}

sparvar_status sparvar_cache_residual_from_dense(const sparvar_schedule* sched,
                                                int32_t decision_scale, int32_t block,
                                                const sparvar_attn_shape* shape,
                                                const uint16_t* q_S, const uint16_t* k_cache,
                                                const uint16_t* v_cache, const int32_t* row_ptr_S,
                                                const int32_t* col_idx_S, float softmax_scale,
                                                const uint16_t* o_dense, uint16_t* o_cache,
                                                void* stream) {
  if (row_ptr_S == nullptr || col_idx_S == nullptr || o_dense == nullptr || o_cache == nullptr)
    return fail(SPARVAR_ERR_INVALID_ARG, "null row_ptr / col_idx / o_dense / o_cache");
  if (o_dense == o_cache) return fail(SPARVAR_ERR_INVALID_ARG, "o_cache must not alias o_dense");
  if (!aligned16(o_dense)) return fail(SPARVAR_ERR_INVALID_ARG, "o_dense must be 16-byte aligned");
  // the sparse term lands in o_cache, then o_cache = o_dense - o_cache element by element
  sparvar_status s = attn_common(sched, decision_scale, block, shape, q_S, k_cache, v_cache,
                                 row_ptr_S, col_idx_S, softmax_scale, o_cache, nullptr, stream);
  if (s != SPARVAR_OK) return s;
  const int side = sched->sides[decision_scale - 1];
  cudaError_t e = sv::launch_residual(shape->batch_heads, side * side, shape->head_dim, o_dense,
                                      shape->o_stride_bh, o_cache, shape->o_stride_bh, o_cache,
                                      shape->o_stride_bh, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "residual launch");
  return ok();
}

// ---------------------------------------------------------------- NEXT(2): token-level CS4A
static bool token_c_ok(int C) { return C == 64 || C == 128 || C == 192; }

sparvar_status sparvar_token_colsum(const sparvar_schedule* sched, int32_t decision_scale,
                                    int32_t query_block, const sparvar_attn_shape* shape,
                                    const uint16_t* q_S, const uint16_t* k_cache,
                                    const float* lse_S, float softmax_scale, float* colsum_out,
                                    void* stream) {
  sv::Geo g;
  sparvar_status s = make_geo(sched, &g);
  if (s != SPARVAR_OK) return s;
  const int S = decision_scale;
  if (S < 1 || S > g.K) return fail(SPARVAR_ERR_INVALID_ARG, "decision_scale %d not in [1, %d]", S, g.K);
  if (!token_c_ok(query_block))
    return fail(SPARVAR_ERR_UNSUPPORTED, "query_block %d not in {64, 128, 192}", query_block);
  const long long n_q = (long long)g.side[S - 1] * g.side[S - 1];
  const long long n_kv = g.cum[S];
  s = check_shape(shape, n_q, n_kv, false);
  if (s != SPARVAR_OK) return s;
  if (q_S == nullptr || k_cache == nullptr || lse_S == nullptr || colsum_out == nullptr)
    return fail(SPARVAR_ERR_INVALID_ARG, "null pointer");
  if (!aligned16(q_S) || !aligned16(k_cache))
    return fail(SPARVAR_ERR_INVALID_ARG, "tensor pointers must be 16-byte aligned");
  const int D = shape->head_dim;
  const float scale = softmax_scale > 0.f ? softmax_scale : 1.0f / std::sqrt((float)D);
  CUtensorMap tk, tq;
  if ((s = make_tmap(&tk, k_cache, D, n_kv, shape->batch_heads, shape->kv_stride_bh, 128)) != SPARVAR_OK)
    return s;
  if ((s = make_tmap(&tq, q_S, D, n_q, shape->batch_heads, shape->q_stride_bh, query_block)) != SPARVAR_OK)
    return s;
  cudaError_t e = sv::launch_colsum(D, query_block, tk, tq, shape->batch_heads, (int)n_q, (int)n_kv,
                                    scale * 1.4426950408889634f, lse_S, colsum_out,
                                    (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "colsum launch");
  return ok();
}

sparvar_status sparvar_token_select(const sparvar_schedule* sched, int32_t decision_scale,
                                    int32_t query_block, int32_t sink_scales, int32_t batch_heads,
                                    const float* colsum, int32_t topk_tokens, uint32_t* mask_out,
                                    void* stream) {
  sv::Geo g;
  sparvar_status s = make_geo(sched, &g);
  if (s != SPARVAR_OK) return s;
  const int S = decision_scale;
  if (S < 1 || S > g.K) return fail(SPARVAR_ERR_INVALID_ARG, "decision_scale %d not in [1, %d]", S, g.K);
  if (query_block < 1) return fail(SPARVAR_ERR_INVALID_ARG, "query_block %d < 1", query_block);
  if (sink_scales < 0 || sink_scales > S)
    return fail(SPARVAR_ERR_INVALID_ARG, "sink_scales %d not in [0, %d]", sink_scales, S);
  if (topk_tokens < 1) return fail(SPARVAR_ERR_INVALID_ARG, "topk_tokens %d < 1", topk_tokens);
  if (batch_heads < 1 || batch_heads > 65535)
    return fail(SPARVAR_ERR_INVALID_ARG, "batch_heads %d", batch_heads);
  if (colsum == nullptr || mask_out == nullptr) return fail(SPARVAR_ERR_INVALID_ARG, "null pointer");
  const long long n_q = (long long)g.side[S - 1] * g.side[S - 1];
  const int G = ceil_div(n_q, query_block);
  const int n_sink = sink_scales > 0 ? g.cum[sink_scales] : 0;
  cudaError_t e = sv::launch_topk_tokens(batch_heads * G, g.cum[S], topk_tokens, n_sink, colsum,
                                         mask_out, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "token select launch");
  return ok();
}

sparvar_status sparvar_token_map(const sparvar_schedule* sched, int32_t src_scale,
                                 int32_t dst_scale, int32_t query_block, int32_t sink_scales,
                                 int32_t map_mode, int32_t batch_heads, const uint32_t* src_mask,
                                 uint32_t* dst_mask, void* stream) {
  sv::Geo g;
  sparvar_status s = make_geo(sched, &g);
  if (s != SPARVAR_OK) return s;
  if (src_scale < 1 || dst_scale > g.K || src_scale > dst_scale)
    return fail(SPARVAR_ERR_INVALID_ARG, "need 1 <= src_scale (%d) <= dst_scale (%d) <= %d",
                src_scale, dst_scale, g.K);
  if (query_block < 1) return fail(SPARVAR_ERR_INVALID_ARG, "query_block %d < 1", query_block);
  if (sink_scales < 0 || sink_scales > dst_scale)
    return fail(SPARVAR_ERR_INVALID_ARG, "sink_scales %d not in [0, %d]", sink_scales, dst_scale);
  if (map_mode != SPARVAR_MAP_FOOTPRINT && map_mode != SPARVAR_MAP_POINT)
    return fail(SPARVAR_ERR_INVALID_ARG, "map_mode %d", map_mode);
  if (batch_heads < 1 || batch_heads > 65535)
    return fail(SPARVAR_ERR_INVALID_ARG, "batch_heads %d", batch_heads);
  if (src_mask == nullptr || dst_mask == nullptr) return fail(SPARVAR_ERR_INVALID_ARG, "null mask pointer");
  cudaError_t e = sv::launch_map_tokens(g, src_scale, dst_scale, query_block, sink_scales, map_mode,
                                        batch_heads, src_mask, dst_mask, (cudaStream_t)stream);
  if (e == cudaErrorInvalidValue)
    return fail(SPARVAR_ERR_UNSUPPORTED, "token row of %d bits too wide for shared memory", g.cum[dst_scale]);
  if (e != cudaSuccess) return cuda_fail(e, "token map launch");
  return ok();
}

static sparvar_status token_attn_common(const sparvar_schedule* sched, int32_t target_scale,
                                        int32_t query_block, const sparvar_attn_shape* shape,
                                        const uint16_t* q, const uint16_t* k_cache,
                                        const uint16_t* v_cache, const int32_t* row_ptr,
                                        const int32_t* col_idx, float softmax_scale, uint16_t* o,
                                        void* stream, const uint16_t* add = nullptr,
                                        int32_t add_scale = 0, int64_t add_stride = 0) {
  sv::Geo g;
  sparvar_status s = make_geo(sched, &g);
  if (s != SPARVAR_OK) return s;
  const int K = target_scale;
  if (K < 1 || K > g.K) return fail(SPARVAR_ERR_INVALID_ARG, "target_scale %d not in [1, %d]", K, g.K);
  if (!token_c_ok(query_block))
    return fail(SPARVAR_ERR_UNSUPPORTED, "query_block %d not in {64, 128, 192}", query_block);
  const long long n_q = (long long)g.side[K - 1] * g.side[K - 1];
  s = check_shape(shape, n_q, g.cum[K], true);
  if (s != SPARVAR_OK) return s;
  if (q == nullptr || k_cache == nullptr || v_cache == nullptr || o == nullptr ||
      row_ptr == nullptr || col_idx == nullptr)
    return fail(SPARVAR_ERR_INVALID_ARG, "null pointer");
  if (!aligned16(q) || !aligned16(k_cache) || !aligned16(v_cache) || !aligned16(o))
    return fail(SPARVAR_ERR_INVALID_ARG, "tensor pointers must be 16-byte aligned");
  const int D = shape->head_dim;
  const float scale = softmax_scale > 0.f ? softmax_scale : 1.0f / std::sqrt((float)D);
  CUtensorMap tq;
  if ((s = make_tmap(&tq, q, D, n_q, shape->batch_heads, shape->q_stride_bh, 128)) != SPARVAR_OK)
    return s;
  cudaError_t e = sv::launch_token_attn(D, tq, k_cache, v_cache, shape->kv_stride_bh,
                                        shape->batch_heads, (int)n_q, query_block,
                                        scale * 1.4426950408889634f, row_ptr, col_idx, o,
                                        shape->o_stride_bh, add, add_stride,
                                        add != nullptr ? g.side[add_scale - 1] : 1, g.side[K - 1],
                                        (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "token attention launch");
  return ok();
}

sparvar_status sparvar_token_sparse_attn(const sparvar_schedule* sched, int32_t target_scale,
                                         int32_t query_block, const sparvar_attn_shape* shape,
                                         const uint16_t* q, const uint16_t* k_cache,
                                         const uint16_t* v_cache, const int32_t* row_ptr,
                                         const int32_t* col_idx, float softmax_scale, uint16_t* o,
                                         void* stream) {
  return token_attn_common(sched, target_scale, query_block, shape, q, k_cache, v_cache, row_ptr,
                           col_idx, softmax_scale, o, stream);
}

sparvar_status sparvar_token_cache_residual(const sparvar_schedule* sched, int32_t decision_scale,
                                            int32_t query_block, const sparvar_attn_shape* shape,
                                            const uint16_t* q_S, const uint16_t* k_cache,
                                            const uint16_t* v_cache, const int32_t* row_ptr_S,
                                            const int32_t* col_idx_S, float softmax_scale,
                                            const uint16_t* o_dense, uint16_t* o_cache,
                                            void* stream) {
  if (o_dense == nullptr || o_cache == nullptr)
    return fail(SPARVAR_ERR_INVALID_ARG, "null o_dense / o_cache");
  if (o_dense == o_cache) return fail(SPARVAR_ERR_INVALID_ARG, "o_cache must not alias o_dense");
  if (!aligned16(o_dense)) return fail(SPARVAR_ERR_INVALID_ARG, "o_dense must be 16-byte aligned");
  sparvar_status s = token_attn_common(sched, decision_scale, query_block, shape, q_S, k_cache,
                                       v_cache, row_ptr_S, col_idx_S, softmax_scale, o_cache, stream);
  if (s != SPARVAR_OK) return s;
  const int side = sched->sides[decision_scale - 1];
  cudaError_t e = sv::launch_residual(shape->batch_heads, side * side, shape->head_dim, o_dense,
                                      shape->o_stride_bh, o_cache, shape->o_stride_bh, o_cache,
                                      shape->o_stride_bh, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "residual launch");
  return ok();
}

sparvar_status sparvar_token_sparse_attn_cached(
    const sparvar_schedule* sched, int32_t target_scale, int32_t query_block,
    const sparvar_attn_shape* shape, const uint16_t* q, const uint16_t* k_cache,
    const uint16_t* v_cache, const int32_t* row_ptr, const int32_t* col_idx, float softmax_scale,
    const uint16_t* o_cache, int32_t cache_scale, int64_t cache_stride_bh, uint16_t* o,
    void* stream) {
  if (o_cache == nullptr) return fail(SPARVAR_ERR_INVALID_ARG, "null o_cache");
  sv::Geo g;
  sparvar_status s = make_geo(sched, &g);          // validates the schedule before any read
  if (s != SPARVAR_OK) return s;
  if (cache_scale < 1 || cache_scale > target_scale || cache_scale > g.K)
    return fail(SPARVAR_ERR_INVALID_ARG, "cache_scale %d not in [1, target_scale]", cache_scale);
  if (shape == nullptr) return fail(SPARVAR_ERR_INVALID_ARG, "null shape");
  const long long n_S = (long long)g.side[cache_scale - 1] * g.side[cache_scale - 1];
  if (cache_stride_bh < n_S * shape->head_dim || cache_stride_bh % 8 != 0 || !aligned16(o_cache))
    return fail(SPARVAR_ERR_INVALID_ARG, "cache_stride_bh must be >= N_S*D, a multiple of 8, "
                "and o_cache 16-byte aligned");
  return token_attn_common(sched, target_scale, query_block, shape, q, k_cache, v_cache, row_ptr,
                           col_idx, softmax_scale, o, stream, o_cache, cache_scale, cache_stride_bh);
}

size_t sparvar_dense_attn_mass_workspace(const sparvar_schedule* sched, int32_t decision_scale,
                                         int32_t block, int32_t batch_heads) {
  sv::Geo g;
  if (make_geo(sched, &g) != SPARVAR_OK || decision_scale < 1 || decision_scale > g.K ||
      block < 1 || batch_heads < 1)
    return 0;
  const long long n_q = (long long)g.side[decision_scale - 1] * g.side[decision_scale - 1];
  const long long g_kv = ceil_div(g.cum[decision_scale], block);
  return (size_t)(batch_heads * (2 * g_kv * n_q + n_q)) * sizeof(float);
}

sparvar_status sparvar_dense_attn_mass(const sparvar_schedule* sched, int32_t decision_scale,
                                       int32_t block, int32_t sink_scales,
                                       const sparvar_attn_shape* shape, const uint16_t* q_S,
                                       const uint16_t* k_cache, const uint16_t* v_cache,
                                       float softmax_scale, int32_t select_mode, int32_t topk,
                                       float threshold, uint16_t* o, float* lse, float* mass_out,
                                       uint32_t* mask_out, void* workspace, size_t workspace_bytes,
                                       void* stream) {
  sv::Geo g;
  sparvar_status s = make_geo(sched, &g);
  if (s != SPARVAR_OK) return s;
  if (decision_scale < 1 || decision_scale > g.K)
    return fail(SPARVAR_ERR_INVALID_ARG, "decision_scale %d not in [1, %d]", decision_scale, g.K);
  if (sink_scales < 0 || sink_scales > decision_scale)
    return fail(SPARVAR_ERR_INVALID_ARG, "sink_scales %d not in [0, %d]", sink_scales, decision_scale);
  if (select_mode != SPARVAR_SELECT_TOPK && select_mode != SPARVAR_SELECT_THRESHOLD)
    return fail(SPARVAR_ERR_INVALID_ARG, "select_mode %d", select_mode);
  if (select_mode == SPARVAR_SELECT_TOPK && topk < 1)
    return fail(SPARVAR_ERR_INVALID_ARG, "topk %d < 1", topk);
  if (select_mode == SPARVAR_SELECT_THRESHOLD && !std::isfinite(threshold))
    return fail(SPARVAR_ERR_INVALID_ARG, "threshold must be finite");
  if (shape == nullptr) return fail(SPARVAR_ERR_INVALID_ARG, "null shape");
  if (mask_out == nullptr || workspace == nullptr)
    return fail(SPARVAR_ERR_INVALID_ARG, "null mask_out / workspace");
  const size_t need = sparvar_dense_attn_mass_workspace(sched, decision_scale, block,
                                                        shape->batch_heads);
  if (need == 0 || workspace_bytes < need)
    return fail(SPARVAR_ERR_CAPACITY, "workspace of %zu bytes < %zu", workspace_bytes, need);
  if (reinterpret_cast<uintptr_t>(workspace) % 16 != 0)
    return fail(SPARVAR_ERR_INVALID_ARG, "workspace must be 16-byte aligned");
  const long long n_q = (long long)g.side[decision_scale - 1] * g.side[decision_scale - 1];
  const int g_kv = ceil_div(g.cum[decision_scale], block);
  const int g_q = ceil_div(n_q, block);
  if (5LL * g_kv * sizeof(float) > 48 * 1024)
    return fail(SPARVAR_ERR_UNSUPPORTED, "%d key blocks: mass row too wide for shared memory", g_kv);
  float* ms = static_cast<float*>(workspace);
  float* mm = ms + (long long)shape->batch_heads * g_kv * n_q;
  float* lse_ws = mm + (long long)shape->batch_heads * g_kv * n_q;
  float* lse_use = lse != nullptr ? lse : lse_ws;
  s = attn_common(sched, decision_scale, block, shape, q_S, k_cache, v_cache, nullptr, nullptr,
                  softmax_scale, o, lse_use, stream, nullptr, 0, 0, ms, mm);
  if (s != SPARVAR_OK) return s;
  const int n_sink_blocks = sink_scales > 0 ? ceil_div(g.cum[sink_scales], block) : 0;
  cudaError_t e = sv::launch_mass_select(shape->batch_heads, (int)n_q, g_q, g_kv, block, ms, mm,
                                         lse_use, select_mode, topk, threshold, n_sink_blocks,
                                         mass_out, mask_out, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "mass select launch");
  return ok();
}

sparvar_status sparvar_block_sparse_attn_cached(
    const sparvar_schedule* sched, int32_t target_scale, int32_t block,
    const sparvar_attn_shape* shape, const uint16_t* q, const uint16_t* k_cache,
    const uint16_t* v_cache, const int32_t* row_ptr, const int32_t* col_idx, float softmax_scale,
    const uint16_t* o_cache, int32_t cache_scale, int64_t cache_stride_bh, uint16_t* o, float* lse,
    void* stream) {
  if (row_ptr == nullptr || col_idx == nullptr || o_cache == nullptr)
    return fail(SPARVAR_ERR_INVALID_ARG, "null row_ptr / col_idx / o_cache");
  sv::Geo g;
  sparvar_status s = make_geo(sched, &g);          // validates the schedule before any read
  if (s != SPARVAR_OK) return s;
  if (cache_scale < 1 || cache_scale > target_scale || cache_scale > g.K)
    return fail(SPARVAR_ERR_INVALID_ARG, "cache_scale %d not in [1, target_scale]", cache_scale);
  if (shape == nullptr) return fail(SPARVAR_ERR_INVALID_ARG, "null shape");
  const long long n_S = (long long)g.side[cache_scale - 1] * g.side[cache_scale - 1];
  if (cache_stride_bh < n_S * shape->head_dim || cache_stride_bh % 8 != 0 || !aligned16(o_cache))
    return fail(SPARVAR_ERR_INVALID_ARG, "cache_stride_bh must be >= N_S*D, a multiple of 8, "
                "and o_cache 16-byte aligned");
  return attn_common(sched, target_scale, block, shape, q, k_cache, v_cache, row_ptr, col_idx,
                     softmax_scale, o, lse, stream, o_cache, cache_scale, cache_stride_bh);
}

sparvar_status sparvar_block_sparse_attn_rows(const sparvar_schedule* sched,
                                              int32_t target_scale, int32_t block,
                                              const sparvar_attn_shape* shape, const uint16_t* q,
                                              const uint16_t* k_cache, const uint16_t* v_cache,
                                              int64_t kv_rows, const int32_t* row_ptr,
                                              const int32_t* col_idx, float softmax_scale,
                                              uint16_t* o, float* lse, void* stream) {
  if (row_ptr == nullptr || col_idx == nullptr)
    return fail(SPARVAR_ERR_INVALID_ARG, "null row_ptr / col_idx");
  return attn_common(sched, target_scale, block, shape, q, k_cache, v_cache, row_ptr, col_idx,
                     softmax_scale, o, lse, stream, nullptr, 0, 0, nullptr, nullptr, kv_rows);
}

sparvar_status sparvar_dense_attn(const sparvar_schedule* sched, int32_t target_scale,
                                  const sparvar_attn_shape* shape, const uint16_t* q,
                                  const uint16_t* k_cache, const uint16_t* v_cache,
                                  float softmax_scale, uint16_t* o, float* lse, void* stream) {
  return attn_common(sched, target_scale, 128, shape, q, k_cache, v_cache, nullptr, nullptr,
                     softmax_scale, o, lse, stream, nullptr, 0, 0);
}

}  // extern "C"
