// token.cu — NEXT(2), token-granular CS4A (the paper's own CS4A granularity) for sm_100a.
//
//  * colsum_kernel: A^(S)[g, j] = sum_{q in query block g} P[q, j]
//    over query blocks of C rows.  Computed transposed, S^T = K Q_g^T (tcgen05, M = 128 keys,
//    N = C queries, double-buffered accumulators in TMEM), so each thread owns one key row and
//    the column sum of P is the row sum sum_q 2^(s_jq * scale * log2 e - L_q) with
//    L_q = lse_q * log2 e from the decision scale's dense pass: no cross-thread reduction, fp32.
//  * token_attn_kernel: Delta O^(K) over per-query-block token lists (PAPER.md:318-328,
//    824-830 "gathers discrete, non-contiguous key and value vectors ... packed into contiguous
//    dense tiles within shared memory"): a producer warp gathers 128 listed K and V rows per
//    chunk with cp.async straight into the 128-byte-swizzled layout the tensor core reads,
//    tcgen05 computes S = Q K^T and O += P V with S / P / O in TMEM, and one softmax thread per
//    query row runs the fp32 online softmax (exp2 domain, lazy rescale).  One CTA per
//    (b,h, query block): the block's 128-row sub-tiles are two slots sharing every gathered
//    chunk; seven gather warps fill double-buffered K/V chunks.
#include <cuda_bf16.h>
#include <algorithm>
#include <cstdio>

#include "kernels.h"
#include "ptx.cuh"
#include "kernel_util.cuh"

namespace sv {
namespace {

constexpr int TBM = 128;           // key rows per colsum tile / query rows per attention tile

// ------------------------------------------------------------------------------- column sums
// One CTA per (b,h, query block g, range of key tiles).  Warp 8 loads the block's Q once and
// streams 128-key tiles of K through a 2-stage TMA ring; it issues S^T = K Q_g^T into one of two
// TMEM accumulators (C columns each).  Warpgroup s (warps 4s..4s+3) exponentiates the tiles of
// accumulator s (one key row per thread: sum_q 2^(s * scale * log2 e - L_q)), so two softmax
// warps per SM sub-partition keep the MUFU pipe busy while the next MMA runs.
template <int D, int C>
struct ColCfg {
  static constexpr int NBOX = D / 64;
  static constexpr int K_BYTES = TBM * D * 2;
  static constexpr int Q_BYTES = C * D * 2;
  static constexpr int SMEM = 2 * K_BYTES + Q_BYTES + C * 4 + 1024;   // + alignment slack
};

template <int D, int C>
__global__ void __launch_bounds__(288, 1) colsum_kernel(const __grid_constant__ CUtensorMap tmap_k,
                                                        const __grid_constant__ CUtensorMap tmap_q,
                                                        int n_q, int n_kv, int G, int n_kt,
                                                        int tiles_per_cta, float scale_log2,
                                                        const float* __restrict__ lse,
                                                        float* __restrict__ out) {
  using CF = ColCfg<D, C>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));       // SW128 tiles: 1 KB aligned
  uint8_t* sQ = smem;
  uint8_t* sK = smem + CF::Q_BYTES;                          // [2]
  float* sL = reinterpret_cast<float*>(sK + 2 * CF::K_BYTES);
  __shared__ uint64_t q_full, k_full[2], k_free[2], acc_full[2], acc_free[2];
  __shared__ uint32_t tslot;
  const int kt0 = blockIdx.x * tiles_per_cta;
  const int nt = min(tiles_per_cta, n_kt - kt0);
  const int g = blockIdx.y, bh = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&q_full, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&k_full[b], 1);
      mbar_init(&k_free[b], 1);
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_free[b], TBM);
    }
    fence_barrier_init();
  }
  if (warp == 8) {
    tmem_alloc(&tslot, 512);
    tmem_relinquish();
  }
  // L_q of the block's queries; rows past N_S contribute 2^-inf = 0
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const int q = g * C + c;
    sL[c] = q < n_q ? lse[(long long)bh * n_q + q] * 1.4426950408889634f : INFINITY;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;                              // accumulator b: cols [256 b, +C)
  if (warp == 8) {
    if (lane == 0) {
      mbar_arrive_expect_tx(&q_full, CF::Q_BYTES);
#pragma unroll
      for (int b = 0; b < CF::NBOX; ++b)
        tma_load_3d(sQ + b * (C * 128), &tmap_q, &q_full, b * 64, g * C, bh);
      // K ring: the load of tile i+2 waits for the MMA of tile i to have read its stage
      for (int i = 0; i < min(nt, 2); ++i) {
        mbar_arrive_expect_tx(&k_full[i], CF::K_BYTES);
#pragma unroll
        for (int b = 0; b < CF::NBOX; ++b)
          tma_load_3d(sK + i * CF::K_BYTES + b * (TBM * 128), &tmap_k, &k_full[i], b * 64,
                      (kt0 + i) * TBM, bh);
      }
    }
    __syncwarp();
    constexpr uint32_t IDESC = idesc_bf16_f32(TBM, C, 0, 0);
    const uint64_t db = sdesc_sw128(smem_u32(sQ), 16, 1024);
    mbar_wait(&q_full, 0);
    for (int i = 0; i < nt; ++i) {
      const int s = i & 1;
      mbar_wait(&k_full[s], (i >> 1) & 1);
      if (i >= 2) mbar_wait(&acc_free[s], ((i >> 1) - 1) & 1);
      tc_fence_after();
      const uint64_t da = sdesc_sw128(smem_u32(sK + s * CF::K_BYTES), 16, 1024);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t oa = ((kk >> 2) * (TBM * 128) + (kk & 3) * 32) >> 4;
          const uint32_t ob = ((kk >> 2) * (C * 128) + (kk & 3) * 32) >> 4;
          mma_ss(tmem + s * 256, da + oa, db + ob, IDESC, kk > 0);
        }
        mma_commit(&acc_full[s]);
        mma_commit(&k_free[s]);
      }
      __syncwarp();
      if (i + 2 < nt && lane == 0) {
        mbar_wait(&k_free[s], (i >> 1) & 1);
        mbar_arrive_expect_tx(&k_full[s], CF::K_BYTES);
#pragma unroll
        for (int b = 0; b < CF::NBOX; ++b)
          tma_load_3d(sK + s * CF::K_BYTES + b * (TBM * 128), &tmap_k, &k_full[s], b * 64,
                      (kt0 + i + 2) * TBM, bh);
      }
      __syncwarp();
    }
  } else {
    // warpgroup s exponentiates the tiles of accumulator s (tiles i with i % 2 == s)
    const int s = warp >> 2;
    const uint32_t t_row = tmem + (uint32_t((warp & 3) * 32) << 16);
    for (int i = s; i < nt; i += 2) {
      mbar_wait(&acc_full[s], (i >> 1) & 1);
      tc_fence_after();
      float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
      for (int c0 = 0; c0 < C; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(t_row + s * 256 + c0, v);
        tmem_wait_ld();
#pragma unroll
        for (int t = 0; t < 32; t += 2) {
          acc0 += ex2(__uint_as_float(v[t]) * scale_log2 - sL[c0 + t]);
          acc1 += ex2(__uint_as_float(v[t + 1]) * scale_log2 - sL[c0 + t + 1]);
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_free[s]);
      const int j = (kt0 + i) * TBM + (warp & 3) * 32 + lane;
      if (j < n_kv) out[((long long)bh * G + g) * n_kv + j] = acc0 + acc1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ------------------------------------------------------------------------ token-list attention
template <int D>
struct TokCfg {
  static constexpr int NBOX = D / 64;
  static constexpr int TILE_BYTES = TBM * D * 2;
  static constexpr int SMEM = 6 * TILE_BYTES + 1024;    // 2 Q tiles, 2 K and 2 V chunks (+ align)
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// One CTA per (b,h, query block g).  The block's rows run as NS = ceil(C / 128) tile slots
// (C = 192: rows 0-127 and 128-191) that share every gathered K/V chunk.  Warps 0-3 / 4-7:
// softmax of slot 0 / 1 (one query row per thread) and its epilogue; warp 8: tcgen05 issue;
// warps 9-15: gather into double-buffered chunks of 128 tokens.  Issue order per chunk c and
// slot t: O_t += P_t,c-1 V_c-1, then S_t = Q_t K_c^T (S/P alias in TMEM and the tensor pipe runs
// one thread's ops in order, so S_t,c complete also means P_t,c-1 V_c-1 is, which the softmax
// needs before an O rescale).  The two slots' softmax chains interleave on the tensor pipe.
// Optional NEXT(1) residual for the token path: out += NN-upsample(add) over the query grid
// (READING 22): output query (x, y) of side s_dst adds cache row
// (floor(x s_src / s_dst), floor(y s_src / s_dst)) of side s_src.
struct TokCache {
  const uint16_t* add;   // bf16 [bh][s_src * s_src][D] or nullptr
  long long add_stride;  // elements between (b,h) slabs
  int s_src, s_dst;
};

#ifndef SV_TOK_ROW_GATHER
#define SV_TOK_ROW_GATHER 0   // 1: one list row per lane (round-1 gather), 0: coalesced rows
#endif
constexpr int TOK_WARPS = 16;
constexpr int TOK_THREADS = TOK_WARPS * 32;
constexpr int TOK_WARP_MMA = 8, TOK_WARP_GATHER0 = 9;
constexpr int TOK_GATHER_WARPS = TOK_WARPS - TOK_WARP_GATHER0;
constexpr int TOK_REG_SOFTMAX = 184, TOK_REG_OTHER = 72;
static_assert(8 * (TOK_REG_SOFTMAX - 128) <= 8 * (128 - TOK_REG_OTHER), "register pool");

template <int D, int NS>
__global__ void __launch_bounds__(TOK_THREADS, 1) token_attn_kernel(
    const __grid_constant__ CUtensorMap tmap_q, const uint16_t* __restrict__ k,
    const uint16_t* __restrict__ v, long long kv_stride, int n_q, int C, int G,
    float scale_log2, const int* __restrict__ row_ptr, const int* __restrict__ col_idx,
    uint16_t* __restrict__ o, long long o_stride, const TokCache cache) {
  using TC = TokCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;                                       // [NS]
  uint8_t* sK = smem + 2 * TC::TILE_BYTES;                  // [2] chunk buffers
  uint8_t* sV = smem + 4 * TC::TILE_BYTES;                  // [2]
  __shared__ uint64_t q_full, s_bar[2], p_bar[2], pv_done[2], kv_full[2], kv_empty[2];
  __shared__ uint32_t tslot;
  const int g = blockIdx.x % G, bh = blockIdx.x / G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = bh * G + g;
  const int beg = __ldg(row_ptr + r), n = __ldg(row_ptr + r + 1) - beg;
  const int chunks = (n + TBM - 1) / TBM;
  const int row_end = min(g * C + C, n_q);                  // rows of block g
  if (threadIdx.x == 0) {
    mbar_init(&q_full, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_bar[b], 1);
      mbar_init(&p_bar[b], TBM);
      mbar_init(&pv_done[b], 1);
      mbar_init(&kv_full[b], TOK_GATHER_WARPS);
      mbar_init(&kv_empty[b], 1);
    }
    fence_barrier_init();
  }
  if (warp == TOK_WARP_MMA) {
    tmem_alloc(&tslot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;            // slot t: S/P cols [128t, 128t+128), O [256+128t, +D)
  if (warp >= TOK_WARP_MMA) {
    reg_dealloc<TOK_REG_OTHER>();
    if (warp >= TOK_WARP_GATHER0) {
      // ---------------------------------------------------------- packed gather (cp.async)
      // list entry c*128 + i -> row i of buffer c&1, 16-byte pieces in the SW128 order the
      // tensor core reads; rows past the list are zero-filled (their logits are masked)
      const int gw = warp - TOK_WARP_GATHER0;
      const uint16_t* kb = k + (long long)bh * kv_stride;
      const uint16_t* vb = v + (long long)bh * kv_stride;
      for (int c = 0; c < chunks; ++c) {
        const int b = c & 1;
        if (c >= 2) mbar_wait(&kv_empty[b], ((c >> 1) - 1) & 1);
        const uint32_t dK = smem_u32(sK + b * TC::TILE_BYTES), dV = smem_u32(sV + b * TC::TILE_BYTES);
#if SV_TOK_ROW_GATHER
        for (int i = gw * 32 + lane; i < TBM; i += TOK_GATHER_WARPS * 32) {
          const int e = c * TBM + i;
          const bool ok = e < n;
          const int tok = ok ? __ldg(col_idx + beg + e) : 0;
          const uint16_t* ks = kb + (long long)tok * D;
          const uint16_t* vs = vb + (long long)tok * D;
#pragma unroll
          for (int p = 0; p < D / 8; ++p) {
            const uint32_t off = (p >> 3) * (TBM * 128) + i * 128 + (((p & 7) ^ (i & 7)) << 4);
            cp_async16(dK + off, ks + p * 8, ok);
            cp_async16(dV + off, vs + p * 8, ok);
          }
        }
#else
        // coalesced: the D/8 16-byte pieces of a row go to consecutive lanes, so a warp
        // instruction reads 32 * 16 B from 32 / (D/8) whole rows (2 at D = 128) instead of one
        // piece of 32 different rows (32 L1 wavefronts)
        constexpr int PIECES = D / 8, RPI = 32 / PIECES;         // rows per warp instruction
        const int p = lane % PIECES, ri = lane / PIECES;
        for (int i0 = gw * RPI; i0 < TBM; i0 += TOK_GATHER_WARPS * RPI) {
          const int i = i0 + ri;
          const int e = c * TBM + i;
          const bool ok = e < n;
          const int tok = ok ? __ldg(col_idx + beg + e) : 0;
          const uint32_t off = (p >> 3) * (TBM * 128) + i * 128 + (((p & 7) ^ (i & 7)) << 4);
          cp_async16(dK + off, kb + (long long)tok * D + p * 8, ok);
          cp_async16(dV + off, vb + (long long)tok * D + p * 8, ok);
        }
#endif
        cp_async_wait_all();
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&kv_full[b]);
      }
    } else {
      // ---------------------------------------------------------- tcgen05 issue
      if (lane == 0) {
        mbar_arrive_expect_tx(&q_full, NS * TC::TILE_BYTES);
#pragma unroll
        for (int t = 0; t < NS; ++t)
#pragma unroll
          for (int b = 0; b < TC::NBOX; ++b)
            tma_load_3d(sQ + t * TC::TILE_BYTES + b * (TBM * 128), &tmap_q, &q_full, b * 64,
                        g * C + t * TBM, bh);
      }
      constexpr uint32_t IDESC_QK = idesc_bf16_f32(TBM, TBM, 0, 0);
      constexpr uint32_t IDESC_PV = idesc_bf16_f32(TBM, D, 0, 1);
      mbar_wait(&q_full, 0);
      auto pv = [&](int t, int c) {                         // O_t += P_t,c V_c
        mbar_wait(&p_bar[t], c & 1);
        tc_fence_after();
        const int b = c & 1;
        const uint64_t dv = sdesc_sw128(smem_u32(sV + b * TC::TILE_BYTES), TBM * 128, 1024);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < TBM / 16; ++kk)
            mma_ts(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, dv + ((uint32_t)(kk * 2048) >> 4),
                   IDESC_PV, (c > 0 || kk > 0) ? 1u : 0u);
          if (t == NS - 1) mma_commit(&kv_empty[b]);       // last reader of chunk c's buffers
          mma_commit(&pv_done[t]);
        }
        __syncwarp();
      };
      auto qk = [&](int t, int c) {                         // S_t = Q_t K_c^T
        const uint64_t dq = sdesc_sw128(smem_u32(sQ + t * TC::TILE_BYTES), 16, 1024);
        const uint64_t dk = sdesc_sw128(smem_u32(sK + (c & 1) * TC::TILE_BYTES), 16, 1024);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t oa = ((kk >> 2) * (TBM * 128) + (kk & 3) * 32) >> 4;
            mma_ss(tmem + t * 128, dq + oa, dk + oa, IDESC_QK, kk > 0);
          }
          mma_commit(&s_bar[t]);
        }
        __syncwarp();
      };
      for (int c = 0; c < chunks; ++c) {
#pragma unroll
        for (int t = 0; t < NS; ++t) {
          if (c > 0) pv(t, c - 1);
          // P_0,c-1 V_c-1 only needs chunk c-1: issue it before waiting for chunk c's gather
          if (t == 0) {
            mbar_wait(&kv_full[c & 1], (c >> 1) & 1);
            tc_fence_after();
          }
          qk(t, c);
        }
      }
      if (chunks > 0)
#pragma unroll
        for (int t = 0; t < NS; ++t) pv(t, chunks - 1);
    }
  } else if (warp < 4 * NS) {
    // ------------------------------------------------------------ softmax, one row per thread
    reg_alloc<TOK_REG_SOFTMAX>();
    const int t = warp >> 2;
    const int row = (warp & 3) * 32 + lane;
    const uint32_t t_row = tmem + (uint32_t((warp & 3) * 32) << 16);
    const uint32_t s_col = t * 128, o_col = 256 + t * 128;
    float m = -INFINITY, l = 0.f;
    for (int c = 0; c < chunks; ++c) {
      mbar_wait(&s_bar[t], c & 1);
      tc_fence_after();
      uint32_t s[TBM];
#pragma unroll
      for (int c0 = 0; c0 < TBM; c0 += 32) tmem_ld32(t_row + s_col + c0, s + c0);
      tmem_wait_ld();
      const int valid = min(TBM, n - c * TBM);
      if (valid < TBM) {
#pragma unroll
        for (int i = 0; i < TBM; ++i)
          if (i >= valid) s[i] = __float_as_uint(-INFINITY);
      }
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < TBM; i += 2) mx = fmax3(mx, __uint_as_float(s[i]), __uint_as_float(s[i + 1]));
      const float mx_s = mx * scale_log2;
      const bool need = mx_s > m + 8.0f;
      float alpha = 1.f;
      if (need) {
        alpha = ex2(m - mx_s);
        l *= alpha;
        m = mx_s;
      }
      // S_t,c complete => P_t,c-1 V_c-1 complete (issued before it): O may be rescaled now
      if (c > 0 && __any_sync(0xffffffffu, need)) {
#pragma unroll 1
        for (int c0 = 0; c0 < D; c0 += 32) {
          uint32_t ov[32];
          tmem_ld32(t_row + o_col + c0, ov);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
          tmem_st32(t_row + o_col + c0, ov);
        }
      }
      const float mref = (m == -INFINITY) ? 0.f : m;
      float sum = 0.f;
#pragma unroll
      for (int c0 = 0; c0 < TBM; c0 += 32) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float p0 = ex2(__uint_as_float(s[c0 + i]) * scale_log2 - mref);
          const float p1 = ex2(__uint_as_float(s[c0 + i + 1]) * scale_log2 - mref);
          sum += p0 + p1;
          pk[i / 2] = pack_bf16x2(p0, p1);
        }
        tmem_st16(t_row + s_col + c0 / 2, pk);
      }
      l += sum;
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&p_bar[t]);
    }
    // epilogue: O / l -> bf16 rows of this query block
    const int q = g * C + t * TBM + row;
    const bool store = q < row_end && t * TBM + row < C;
    uint16_t* orow = o + (long long)bh * o_stride + (long long)q * D;
    const uint16_t* arow = nullptr;
    if (cache.add != nullptr && store) {
      const int x = q / cache.s_dst, y = q % cache.s_dst;
      const int src = (x * cache.s_src / cache.s_dst) * cache.s_src + (y * cache.s_src / cache.s_dst);
      arow = cache.add + (long long)bh * cache.add_stride + (long long)src * D;
    }
    if (chunks > 0) {
      mbar_wait(&pv_done[t], (chunks - 1) & 1);
      tc_fence_after();
      const float inv = 1.f / l;
#pragma unroll 1
      for (int c0 = 0; c0 < D; c0 += 16) {
        uint32_t ov[16];
        tmem_ld16(t_row + o_col + c0, ov);
        tmem_wait_ld();
        float ad[16];
        if (arow != nullptr) {
          const uint4 u0 = *reinterpret_cast<const uint4*>(arow + c0);
          const uint4 u1 = *reinterpret_cast<const uint4*>(arow + c0 + 8);
          const uint32_t w[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            ad[2 * i] = __uint_as_float(w[i] << 16);
            ad[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) ad[i] = 0.f;
        }
        uint32_t pk[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          pk[i] = pack_bf16x2(fmaf(__uint_as_float(ov[2 * i]), inv, ad[2 * i]),
                              fmaf(__uint_as_float(ov[2 * i + 1]), inv, ad[2 * i + 1]));
        if (store) {
          uint4* dst = reinterpret_cast<uint4*>(orow + c0);
          dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        }
      }
    } else if (store) {
      // empty list: the output is the (upsampled) cache row, if any
      for (int c0 = 0; c0 < D; c0 += 8)
        *reinterpret_cast<uint4*>(orow + c0) =
            arow != nullptr ? *reinterpret_cast<const uint4*>(arow + c0) : make_uint4(0, 0, 0, 0);
    }
    reg_dealloc<128>();
  } else {
    // warps of an unused second slot (C <= 128)
    reg_alloc<TOK_REG_SOFTMAX>();
    reg_dealloc<128>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == TOK_WARP_MMA) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace

cudaError_t launch_colsum(int head_dim, int C, const CUtensorMap& tk, const CUtensorMap& tq,
                          int bh, int n_q, int n_kv, float scale_log2, const float* lse,
                          float* out, cudaStream_t st) {
  const int G = (n_q + C - 1) / C;
  const int n_kt = (n_kv + TBM - 1) / TBM;
  // whole rows of key tiles per CTA (the Q load and pipeline fill amortised over the row) unless
  // there are too few (b,h,g) rows to give every SM two CTAs' worth of work
  const long long rows = (long long)G * bh;
  const int splits = (int)std::min<long long>(n_kt, std::max<long long>(1, (2LL * 148 + rows - 1) / rows));
  const int tpc = (n_kt + splits - 1) / splits;
  const dim3 grid((n_kt + tpc - 1) / tpc, G, bh);
#define SV_COL(D_, C_)                                                                       \
  if (head_dim == D_ && C == C_) {                                                           \
    auto kern = colsum_kernel<D_, C_>;                                                       \
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                                         ColCfg<D_, C_>::SMEM);                              \
    if (e != cudaSuccess) return e;                                                          \
    kern<<<grid, 288, ColCfg<D_, C_>::SMEM, st>>>(tk, tq, n_q, n_kv, G, n_kt, tpc, scale_log2, lse, out); \
    return cudaGetLastError();                                                               \
  }
  SV_COL(128, 192) SV_COL(128, 128) SV_COL(128, 64) SV_COL(64, 192) SV_COL(64, 128) SV_COL(64, 64)
#undef SV_COL
  return cudaErrorInvalidValue;
}

cudaError_t launch_token_attn(int head_dim, const CUtensorMap& tq, const uint16_t* k,
                              const uint16_t* v, long long kv_stride, int bh, int n_q, int C,
                              float scale_log2, const int* row_ptr, const int* col_idx,
                              uint16_t* o, long long o_stride, const uint16_t* add,
                              long long add_stride, int s_src, int s_dst, cudaStream_t st) {
  const int G = (n_q + C - 1) / C;
  const int ns = (C + TBM - 1) / TBM;
  const TokCache cache{add, add_stride, s_src, s_dst};
  const long long items = (long long)bh * G;
  if (items <= 0) return cudaSuccess;
  if (items > (1LL << 31) - 1 || ns > 2) return cudaErrorInvalidValue;
#define SV_TOK(D_, NS_)                                                                       \
  if (head_dim == D_ && ns == NS_) {                                                          \
    auto kern = token_attn_kernel<D_, NS_>;                                                   \
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                                         TokCfg<D_>::SMEM);                                   \
    if (e != cudaSuccess) return e;                                                           \
    kern<<<(unsigned)items, TOK_THREADS, TokCfg<D_>::SMEM, st>>>(tq, k, v, kv_stride, n_q, C, G, \
                                                              scale_log2, row_ptr, col_idx, o, \
                                                              o_stride, cache);               \
    return cudaGetLastError();                                                                \
  }
  SV_TOK(128, 1) SV_TOK(128, 2) SV_TOK(64, 1) SV_TOK(64, 2)
#undef SV_TOK
  return cudaErrorInvalidValue;
}

}  // namespace sv
