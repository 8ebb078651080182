// predictor.cu — decision-scale sparse-pattern predictor for sm_100a (a2 + a3 in DESIGN.md).
//
// For each (b,h) and query block u at the decision scale S (
// READINGS 10-13):
//     P = softmax(Q_S K_{<=S}^T * scale)               (fp32 logits from bf16, fp32 exp)
//     mass[u, v] = sum_{q in u} sum_{j in v, j < C_S} P[q, j]
//     keep TOPK(k) (ties to the smaller v) or mass >= tau * |u|, then OR the sink blocks.
//
// One pass: a CTA owns a 128-row Q tile (G = 128/B query blocks).  Warp 0 streams K blocks with
// TMA, warp 1 issues S_j = Q K_j^T into one of two TMEM buffers (so QK of step j+1 overlaps the
// softmax of step j), warps 2-5 (one query row per thread) keep, for every KV block j, the
// block-local max m_j and sum_j = sum exp2(s*scale*log2e - m_j) in shared memory.  At the end
// each row rescales them to its final max/normaliser (exact: P = 2^(s' - m_j) 2^(m_j - m) / l),
// rows are reduced per query block in a fixed order (deterministic), and one warp per query block
// selects with ballots into bit rows.
#include <cuda_bf16.h>
#include <cstdio>

#include "kernels.h"
#include "ptx.cuh"

namespace sv {
namespace {

constexpr int BM = 128;
constexpr int NUM_THREADS = 192;
constexpr uint32_t TMEM_COLS = 256;

template <int D, int BLK>
struct PCfg {
  static constexpr int NBOX = D / 64;
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int STAGE_BYTES = BLK * D * 2;
  static constexpr int NST = (2 * 32768 / STAGE_BYTES) > 8 ? 8 : (2 * 32768 / STAGE_BYTES);
  static constexpr int G = BM / BLK;
  static constexpr int SEG = BLK < 32 ? BLK : 32;        // rows reduced by one shuffle segment
  static constexpr int NSEG = BM / SEG;
  static size_t smem(int g_kv) {
    return 1024 + Q_BYTES + NST * STAGE_BYTES + 256 + size_t(2) * g_kv * BM * 4 +
           size_t(NSEG) * g_kv * 4;
  }
};

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int D, int BLK>
__global__ void __launch_bounds__(NUM_THREADS, 1)
predict_kernel(const __grid_constant__ CUtensorMap tmap_q,
               const __grid_constant__ CUtensorMap tmap_k, const PredArgs a) {
  using C = PCfg<D, BLK>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = smem + C::Q_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sK + C::NST * C::STAGE_BYTES);
  uint64_t* bar_q = bars;
  uint64_t* bar_full = bars + 1;
  uint64_t* bar_empty = bars + 1 + C::NST;
  uint64_t* bar_s = bars + 1 + 2 * C::NST;     // [2]
  uint64_t* bar_free = bar_s + 2;              // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_free + 2);
  float* st_m = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 256);
  float* st_s = st_m + a.g_kv * BM;
  float* part = st_s + a.g_kv * BM;            // [NSEG][g_kv]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int tile = blockIdx.x;
  const int bh = blockIdx.y;
  const int n = a.g_kv;

  if (threadIdx.x == 0) {
    mbar_init(bar_q, 1);
    for (int i = 0; i < C::NST; ++i) {
      mbar_init(bar_full + i, 1);
      mbar_init(bar_empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar_s + i, 1);
      mbar_init(bar_free + i, BM);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap_q);
    prefetch_tmap(&tmap_k);
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(bar_q, C::Q_BYTES);
#pragma unroll
      for (int b = 0; b < C::NBOX; ++b)
        tma_load_3d(sQ + b * (BM * 128), &tmap_q, bar_q, b * 64, tile * BM, bh);
      for (int j = 0; j < n; ++j) {
        const int st = j % C::NST;
        const uint32_t ph = (j / C::NST) & 1;
        mbar_wait(bar_empty + st, ph ^ 1);
        mbar_arrive_expect_tx(bar_full + st, C::STAGE_BYTES);
#pragma unroll
        for (int b = 0; b < C::NBOX; ++b)
          tma_load_3d(sK + st * C::STAGE_BYTES + b * (BLK * 128), &tmap_k, bar_full + st, b * 64,
                      j * BLK, bh);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t IDESC = idesc_bf16_f32(BM, BLK, 0, 0);
      const uint32_t q_base = smem_u32(sQ);
      const uint32_t k_base = smem_u32(sK);
      mbar_wait(bar_q, 0);
      tc_fence_after();
      for (int j = 0; j < n; ++j) {
        const int st = j % C::NST;
        const uint32_t ph = (j / C::NST) & 1;
        const int buf = j & 1;
        mbar_wait(bar_free + buf, ((j >> 1) & 1) ^ 1);   // softmax done with S[buf] of step j-2
        mbar_wait(bar_full + st, ph);
        tc_fence_after();
        const uint32_t kb = k_base + st * C::STAGE_BYTES;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t da = sdesc_sw128(q_base + (kk >> 2) * (BM * 128) + (kk & 3) * 32, 16, 1024);
          const uint64_t db = sdesc_sw128(kb + (kk >> 2) * (BLK * 128) + (kk & 3) * 32, 16, 1024);
          mma_ss(tmem + buf * 128, da, db, IDESC, kk > 0);
        }
        mma_commit(bar_empty + st);
        mma_commit(bar_s + buf);
      }
    }
  } else {
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t t_row = tmem + (uint32_t(quarter * 32) << 16);
    const float sl2 = a.scale_log2;
    for (int j = 0; j < n; ++j) {
      const int buf = j & 1;
      mbar_wait(bar_s + buf, (j >> 1) & 1);
      tc_fence_after();
      uint32_t sr[BLK];
      if constexpr (BLK >= 32) {
#pragma unroll
        for (int c = 0; c < BLK; c += 32) tmem_ld32(t_row + buf * 128 + c, sr + c);
      } else {
#pragma unroll
        for (int c = 0; c < BLK; c += 8) tmem_ld8(t_row + buf * 128 + c, sr + c);
      }
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(bar_free + buf);
      const int valid = min(BLK, a.n_kv - j * BLK);
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < BLK; ++c)
        if (c < valid) mx = fmaxf(mx, __uint_as_float(sr[c]));
      const float mref = mx * sl2;
      float sum = 0.f;
#pragma unroll
      for (int c = 0; c < BLK; ++c)
        if (c < valid) sum += ex2(fmaf(__uint_as_float(sr[c]), sl2, -mref));
      st_m[j * BM + row] = mref;
      st_s[j * BM + row] = sum;
    }
    // final max / normaliser of this row, then its share of every block mass
    float m = -INFINITY;
    for (int j = 0; j < n; ++j) m = fmaxf(m, st_m[j * BM + row]);
    float l = 0.f;
    for (int j = 0; j < n; ++j) l += st_s[j * BM + row] * ex2(st_m[j * BM + row] - m);
    const bool row_valid = tile * BM + row < a.n_q;
    const float inv = row_valid ? 1.f / l : 0.f;
    // reduce over the rows of each query block, fixed order (deterministic)
    for (int j = 0; j < n; ++j) {
      float w = st_s[j * BM + row] * ex2(st_m[j * BM + row] - m) * inv;
#pragma unroll
      for (int off = C::SEG / 2; off > 0; off >>= 1) w += __shfl_xor_sync(0xffffffffu, w, off);
      if ((lane % C::SEG) == 0) part[(row / C::SEG) * n + j] = w;
    }
    named_bar(1, BM);
    // selection: one softmax warp per query block (loop)
    const int W = (n + 31) / 32;
    constexpr int SEG_PER_G = BLK / C::SEG;
    for (int g = quarter; g < C::G; g += 4) {
      const int u = tile * C::G + g;
      if (u >= a.g_q) continue;
      // mass of block v = sum of its segments, fixed order; stored into st_m (free now)
      float* mrow = st_m + g * n;
      for (int v = lane; v < n; v += 32) {
        float acc = 0.f;
        for (int sgi = 0; sgi < SEG_PER_G; ++sgi) acc += part[(g * SEG_PER_G + sgi) * n + v];
        mrow[v] = acc;
      }
      __syncwarp();
      const long long r = (long long)bh * a.g_q + u;
      const int rows_u = min(BLK, a.n_q - u * BLK);
      const float thr = a.tau * float(rows_u);
      for (int w0 = 0; w0 < W; ++w0) {
        const int v = w0 * 32 + lane;
        bool sel = false;
        if (v < n) {
          const float mv = mrow[v];
          if (a.mode == 0) {
            int rank = 0;
            for (int t = 0; t < n; ++t) {
              const float mt = mrow[t];
              rank += (mt > mv) || (mt == mv && t < v);
            }
            sel = rank < a.topk;
          } else {
            sel = mv >= thr;
          }
          sel = sel || (v < a.n_sink_blocks);
          if (a.mass) a.mass[r * n + v] = mv;
        }
        const uint32_t word = __ballot_sync(0xffffffffu, sel);
        if (lane == 0) a.mask[r * W + w0] = word;
      }
    }
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
cudaError_t launch_t(const CUtensorMap& tq, const CUtensorMap& tk, const PredArgs& a,
                     cudaStream_t st) {
  using C = PCfg<D, BLK>;
  const size_t smem = C::smem(a.g_kv);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  auto kern = predict_kernel<D, BLK>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((a.n_q + BM - 1) / BM, a.bh);
  kern<<<grid, NUM_THREADS, smem, st>>>(tq, tk, a);
  return cudaGetLastError();
}

}  // namespace

size_t predictor_smem_bytes(int head_dim, int block, int g_kv) {
#define SV_CASE(D_, B_) \
  if (head_dim == D_ && block == B_) return PCfg<D_, B_>::smem(g_kv);
  SV_CASE(128, 128) SV_CASE(128, 64) SV_CASE(128, 32) SV_CASE(128, 16)
  SV_CASE(64, 128) SV_CASE(64, 64) SV_CASE(64, 32) SV_CASE(64, 16)
#undef SV_CASE
  return ~size_t(0);
}

cudaError_t launch_predictor(int head_dim, int block, const CUtensorMap& tq, const CUtensorMap& tk,
                             const PredArgs& a, cudaStream_t st) {
#define SV_CASE(D_, B_) \
  if (head_dim == D_ && block == B_) return launch_t<D_, B_>(tq, tk, a, st);
  SV_CASE(128, 128) SV_CASE(128, 64) SV_CASE(128, 32) SV_CASE(128, 16)
  SV_CASE(64, 128) SV_CASE(64, 64) SV_CASE(64, 32) SV_CASE(64, 16)
#undef SV_CASE
  return cudaErrorInvalidValue;
}

}  // namespace sv
