// attention.cu — block-sparse (and dense) cross-scale attention forward for sm_100a.
//
// Computes, for every (b,h) and query block u, o_t = softmax_J(q_t . k_j * scale) V_J over the
// real tokens J of the KV blocks listed for u (PAPER.md:204-212 Eq. attn_cross_scale,
// PAPER.md:318-328 Eq. sparse_update, PAPER.md:397-407 Eq. block_mask; READINGS 9, 17, 20).
//
// Design:
//  * one CTA = one 128-row query tile of one (b,h); two CTAs are co-resident per SM (96 KB smem,
//    256 TMEM columns each), so one CTA's softmax overlaps the other CTA's tensor-core work.
//  * warp 0: TMA producer (Q once, then K_v / V_v of each listed block into a 2-stage ring)
//    warp 1: tcgen05 issuer (S = Q K^T into TMEM, then O += P V with P read from TMEM)
//    warps 2-5: softmax / correction / epilogue, one TMEM lane (= query row) per thread.
//  * S (fp32, <=128 cols) and O (fp32, D cols) live in TMEM; P (bf16) overwrites S in place and
//    is the TMEM A operand of the P.V MMA.  Online softmax in fp32 with a lazy rescale of O
//    (only when the running max grows by more than 2^8).
//  * Block sizes below 128: a 128-row tile holds G = 128/B query blocks; the KV steps are the
//    ascending union of their lists and each row masks the steps its own block does not list,
//    so every row sees exactly its own list (exact semantics, extra work only for B < 128).
#include <cuda_bf16.h>
#include <cstdio>

#include "kernels.h"
#include "ptx.cuh"

namespace sv {
namespace {

constexpr int BM = 128;                 // query rows per tile (TMEM lanes)
constexpr int NUM_THREADS = 192;        // 6 warps
constexpr uint32_t TMEM_COLS = 256;
constexpr uint32_t S_COL = 0;           // S / P
constexpr uint32_t O_COL = 128;         // O accumulator

template <int D, int BLK>
struct Cfg {
  static constexpr int NBOX = D / 64;                       // 64-element (128 B) TMA boxes per row
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int STAGE_BYTES = BLK * D * 2;
  static constexpr int NST = (2 * 32768 / STAGE_BYTES) < 2 ? 2
                           : ((2 * 32768 / STAGE_BYTES) > 8 ? 8 : (2 * 32768 / STAGE_BYTES));
  static constexpr int G = BM / BLK;                        // query blocks per tile
  static constexpr int SMEM = 1024 /*align slack*/ + Q_BYTES + NST * STAGE_BYTES + 256;
};

// Enumerates the KV steps of a tile: ascending union of the lists of its G query blocks, with
// the bitmask of the groups that list each step.  Every role runs its own copy in lockstep.
template <int G>
struct Steps {
  int cur[G], end[G];
  int dense_next, dense_end;
  bool dense;
  __device__ void init(const AttnArgs& a, int bh, int tile, int g_kv) {
    dense = (a.row_ptr == nullptr);
    dense_next = 0;
    dense_end = g_kv;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int u = tile * G + g;
      if (!dense && u < a.g_q) {
        const int r = bh * a.g_q + u;
        cur[g] = __ldg(a.row_ptr + r);
        end[g] = __ldg(a.row_ptr + r + 1);
      } else {
        cur[g] = 0;
        end[g] = 0;
      }
    }
  }
  __device__ bool next(const AttnArgs& a, int& v, uint32_t& gmask) {
    if (dense) {
      if (dense_next >= dense_end) return false;
      v = dense_next++;
      gmask = (1u << G) - 1u;
      return true;
    }
    if (G == 1) {
      if (cur[0] >= end[0]) return false;
      v = __ldg(a.col_idx + cur[0]);
      ++cur[0];
      gmask = 1u;
      return true;
    }
    int best = 0x7fffffff;
#pragma unroll
    for (int g = 0; g < G; ++g)
      if (cur[g] < end[g]) best = min(best, __ldg(a.col_idx + cur[g]));
    if (best == 0x7fffffff) return false;
    gmask = 0;
#pragma unroll
    for (int g = 0; g < G; ++g)
      if (cur[g] < end[g] && __ldg(a.col_idx + cur[g]) == best) {
        gmask |= 1u << g;
        ++cur[g];
      }
    v = best;
    return true;
  }
  __device__ int count(const AttnArgs& a) {
    Steps<G> c = *this;
    int n = 0, v;
    uint32_t m;
    while (c.next(a, v, m)) ++n;
    return n;
  }
};

template <int D, int BLK>
__global__ void __launch_bounds__(NUM_THREADS, 2)
attn_fwd_kernel(const __grid_constant__ CUtensorMap tmap_q,
                const __grid_constant__ CUtensorMap tmap_k,
                const __grid_constant__ CUtensorMap tmap_v, const AttnArgs a) {
  using C = Cfg<D, BLK>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + C::Q_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + C::NST * C::STAGE_BYTES);
  uint64_t* bar_q = bars;
  uint64_t* bar_full = bars + 1;
  uint64_t* bar_empty = bars + 1 + C::NST;
  uint64_t* bar_s = bars + 1 + 2 * C::NST;
  uint64_t* bar_p = bar_s + 1;
  uint64_t* bar_o = bar_s + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_s + 3);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int tile = blockIdx.x;
  const int bh = blockIdx.y;
  const int g_kv = (a.n_kv + BLK - 1) / BLK;

  if (threadIdx.x == 0) {
    mbar_init(bar_q, 1);
    for (int i = 0; i < C::NST; ++i) {
      mbar_init(bar_full + i, 1);
      mbar_init(bar_empty + i, 1);
    }
    mbar_init(bar_s, 1);
    mbar_init(bar_p, BM);
    mbar_init(bar_o, 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap_q);
    prefetch_tmap(&tmap_k);
    prefetch_tmap(&tmap_v);
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  Steps<C::G> steps;
  steps.init(a, bh, tile, g_kv);

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      mbar_arrive_expect_tx(bar_q, C::Q_BYTES);
#pragma unroll
      for (int b = 0; b < C::NBOX; ++b)
        tma_load_3d(sQ + b * (BM * 128), &tmap_q, bar_q, b * 64, tile * BM, bh);
      int v;
      uint32_t gm;
      int idx = 0;
      while (steps.next(a, v, gm)) {
#pragma unroll
        for (int which = 0; which < 2; ++which, ++idx) {
          const int st = idx % C::NST;
          const uint32_t ph = (idx / C::NST) & 1;
          mbar_wait(bar_empty + st, ph ^ 1);
          uint8_t* dst = sKV + st * C::STAGE_BYTES;
          mbar_arrive_expect_tx(bar_full + st, C::STAGE_BYTES);
          const CUtensorMap* m = which == 0 ? &tmap_k : &tmap_v;
#pragma unroll
          for (int b = 0; b < C::NBOX; ++b)
            tma_load_3d(dst + b * (BLK * 128), m, bar_full + st, b * 64, v * BLK, bh);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- tcgen05 issuer
    if (lane == 0) {
      const int n = steps.count(a);
      constexpr uint32_t IDESC_QK = idesc_bf16_f32(BM, BLK, 0, 0);
      constexpr uint32_t IDESC_PV = idesc_bf16_f32(BM, D, 0, 1);
      const uint32_t q_base = smem_u32(sQ);
      const uint32_t kv_base = smem_u32(sKV);
      mbar_wait(bar_q, 0);
      tc_fence_after();
      int idx = 0;
      for (int j = 0; j < n; ++j) {
        {  // S = Q K^T
          const int st = idx % C::NST;
          const uint32_t ph = (idx / C::NST) & 1;
          ++idx;
          mbar_wait(bar_full + st, ph);
          tc_fence_after();
          const uint32_t kb = kv_base + st * C::STAGE_BYTES;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint64_t da = sdesc_sw128(q_base + (kk >> 2) * (BM * 128) + (kk & 3) * 32, 16, 1024);
            const uint64_t db = sdesc_sw128(kb + (kk >> 2) * (BLK * 128) + (kk & 3) * 32, 16, 1024);
            mma_ss(tmem + S_COL, da, db, IDESC_QK, kk > 0);
          }
          mma_commit(bar_empty + st);
          mma_commit(bar_s);
        }
        mbar_wait(bar_p, j & 1);
        tc_fence_after();
        {  // O += P V
          const int st = idx % C::NST;
          const uint32_t ph = (idx / C::NST) & 1;
          ++idx;
          mbar_wait(bar_full + st, ph);
          tc_fence_after();
          const uint32_t vb = kv_base + st * C::STAGE_BYTES;
#pragma unroll
          for (int kk = 0; kk < BLK / 16; ++kk) {
            const uint64_t db = sdesc_sw128(vb + kk * 2048, BLK * 128, 1024);
            mma_ts(tmem + O_COL, tmem + S_COL + kk * 8, db, IDESC_PV, (j > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(bar_empty + st);
        }
      }
      mma_commit(bar_o);
    }
  } else {
    // ---------------------------------------------------------------- softmax warps
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t t_row = tmem + (uint32_t(quarter * 32) << 16);
    const int grp = row / BLK;
    const float sl2 = a.scale_log2;
    float m = -INFINITY;   // running max of s * scale * log2(e)
    float l = 0.f;         // running sum of exp2(s * sl2 - m)
    int v;
    uint32_t gm;
    int j = 0;
    while (steps.next(a, v, gm)) {
      mbar_wait(bar_s, j & 1);
      tc_fence_after();
      uint32_t sr[BLK];
      if constexpr (BLK >= 32) {
#pragma unroll
        for (int c = 0; c < BLK; c += 32) tmem_ld32(t_row + S_COL + c, sr + c);
      } else {
#pragma unroll
        for (int c = 0; c < BLK; c += 8) tmem_ld8(t_row + S_COL + c, sr + c);
      }
      tmem_wait_ld();
      float s[BLK];
#pragma unroll
      for (int c = 0; c < BLK; ++c) s[c] = __uint_as_float(sr[c]);
      const bool row_on = (gm >> grp) & 1u;
      const int valid = row_on ? min(BLK, a.n_kv - v * BLK) : 0;
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < BLK; ++c) {
        if (c >= valid) s[c] = -INFINITY;
        mx = fmaxf(mx, s[c]);
      }
      const float mx_s = mx * sl2;
      const bool need = mx_s > m + 8.0f;
      float alpha = 1.f;
      if (need) {
        alpha = ex2(m - mx_s);
        m = mx_s;
        l *= alpha;
      }
      const float mref = (m == -INFINITY) ? 0.f : m;
      uint32_t p[BLK / 2];
      float sum = 0.f;
#pragma unroll
      for (int c = 0; c < BLK; c += 2) {
        const float p0 = ex2(fmaf(s[c], sl2, -mref));
        const float p1 = ex2(fmaf(s[c + 1], sl2, -mref));
        sum += p0 + p1;
        p[c / 2] = pack_bf16x2(p0, p1);
      }
      l += sum;
      if constexpr (BLK / 2 >= 32) {
#pragma unroll
        for (int c = 0; c < BLK / 2; c += 32) tmem_st32(t_row + S_COL + c, p + c);
      } else {
#pragma unroll
        for (int c = 0; c < BLK / 2; c += 8) tmem_st8(t_row + S_COL + c, p + c);
      }
      if (j > 0 && __any_sync(0xffffffffu, need)) {
#pragma unroll 1
        for (int c = 0; c < D; c += 32) {
          uint32_t o[32];
          tmem_ld32(t_row + O_COL + c, o);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st32(t_row + O_COL + c, o);
        }
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(bar_p);
      ++j;
    }
    // ---------------------------------------------------------------- epilogue
    mbar_wait(bar_o, 0);
    tc_fence_after();
    const int n_row = tile * BM + row;
    const bool store = n_row < a.n_q;
    const float inv = l > 0.f ? 1.f / l : 0.f;
    uint16_t* orow = a.o + (long long)bh * a.o_stride + (long long)n_row * D;
#pragma unroll 1
    for (int c = 0; c < D; c += 32) {
      uint32_t o[32];
      tmem_ld32(t_row + O_COL + c, o);
      tmem_wait_ld();
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i)
        pk[i] = (l > 0.f) ? pack_bf16x2(__uint_as_float(o[2 * i]) * inv,
                                        __uint_as_float(o[2 * i + 1]) * inv)
                          : 0u;
      if (store) {
        uint4* dst = reinterpret_cast<uint4*>(orow + c);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
      }
    }
    if (a.lse != nullptr && store)
      a.lse[(long long)bh * a.n_q + n_row] =
          l > 0.f ? (m * 0.69314718055994531f + logf(l)) : -INFINITY;
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem, TMEM_COLS);
  }
}

template <int D, int BLK>
cudaError_t launch_t(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                     const AttnArgs& a, cudaStream_t st) {
  using C = Cfg<D, BLK>;
  auto kern = attn_fwd_kernel<D, BLK>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  if (e != cudaSuccess) return e;
  dim3 grid((a.n_q + BM - 1) / BM, a.bh);
  kern<<<grid, NUM_THREADS, C::SMEM, st>>>(tq, tk, tv, a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attention(int head_dim, int block, const CUtensorMap& tq, const CUtensorMap& tk,
                             const CUtensorMap& tv, const AttnArgs& a, cudaStream_t st) {
#define SV_CASE(D_, B_) \
  if (head_dim == D_ && block == B_) return launch_t<D_, B_>(tq, tk, tv, a, st);
  SV_CASE(128, 128) SV_CASE(128, 64) SV_CASE(128, 32) SV_CASE(128, 16)
  SV_CASE(64, 128) SV_CASE(64, 64) SV_CASE(64, 32) SV_CASE(64, 16)
#undef SV_CASE
  return cudaErrorInvalidValue;
}

}  // namespace sv
