// predictor.cu — decision-scale sparse-pattern predictor for sm_100a (a2 + a3 in DESIGN.md).
//
// For each (b,h) and query block u at the decision scale S (
// READINGS 10-13):
//     P = softmax(Q_S K_{<=S}^T * scale)               (fp32 logits from bf16, fp32 exp)
//     mass[u, v] = sum_{q in u} sum_{j in v, j < C_S} P[q, j]
//     keep TOPK(k) (ties to the smaller v) or mass >= tau * |u|, then OR the sink blocks.
//
// Design (DESIGN.md §7 "predict_kernel"):
//  * Persistent, one CTA per SM, two tile SLOTS (128 query rows each) with their own softmax
//    warpgroup and a double-buffered S in TMEM (4 x 128 columns): the tensor core computes
//    S_{j+1} while the softmax warps reduce S_j, so the kernel runs at the exp2 throughput.
//  * Every tile has the same G_kvS KV steps, so the MMA warp and the K loader alternate the two
//    slots in lockstep; when both slots work on the same (b,h) they share each K stage.
//  * Per (row, KV block) the softmax warps keep the block sum of 2^(s*scale*log2e - m) relative
//    to the row's running max m (lazy: the stored sums are rescaled only when m grows by more
//    than 2^8).  At the tile end each row normalises by l = sum of its block sums (exact:
//    P[q, j] = 2^(s' - m) / l), rows are reduced per query block in a fixed order
//    (deterministic), and one warp per query block selects with ballots into bit rows.
//  * One in four exp2 pairs runs as a degree-4 polynomial on the FMA pipe (relative error
//    2.6e-6, well inside the 1e-4 mass tolerance) to take load off the MUFU pipe.
#include <cuda_bf16.h>
#include <cstdio>
#include <type_traits>

#include "kernels.h"
#include "ptx.cuh"
#include "kernel_util.cuh"

#ifndef SV_PRED_QB
#define SV_PRED_QB 4     // preferred number of Q buffers (2..4); fewer if shared memory is short
#endif
#ifndef SV_PRED_ORDER
#define SV_PRED_ORDER 0   // 0: contiguous tile ranges; 1: same-head tile pairs in strided windows
#endif
#ifndef SV_PRED_EMU_EVERY
#define SV_PRED_EMU_EVERY 4   // 1 in 4 exp2 pairs as a degree-4 polynomial on the FMA pipe
#endif

#ifdef SV_PRED_PROF
// Development instrumentation (variant libraries only, -DSV_PRED_PROF): clocks summed over CTAs.
__device__ unsigned long long sv_pred_prof[16];
extern "C" int sparvar_pred_prof_read(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, sv_pred_prof, sizeof(sv_pred_prof)) == cudaSuccess ? 0 : 1;
}
extern "C" int sparvar_pred_prof_reset() {
  static unsigned long long z[16];
  return cudaMemcpyToSymbol(sv_pred_prof, z, sizeof(z)) == cudaSuccess ? 0 : 1;
}
#ifdef SV_PRED_TRACE
// one CTA's timeline: softmax (quarter-0 warp of each slot) wait/body/end per step, the issuer's
// MMA block per slot-step, tile ends
__device__ long long sv_pred_tr_sm[2][400][3];
__device__ long long sv_pred_tr_mma[2][400][2];
__device__ long long sv_pred_tr_te[2][16][2];
extern "C" int sparvar_pred_trace_read(long long* sm, long long* mma, long long* te) {
  return (cudaMemcpyFromSymbol(sm, sv_pred_tr_sm, sizeof(sv_pred_tr_sm)) == cudaSuccess &&
          cudaMemcpyFromSymbol(mma, sv_pred_tr_mma, sizeof(sv_pred_tr_mma)) == cudaSuccess &&
          cudaMemcpyFromSymbol(te, sv_pred_tr_te, sizeof(sv_pred_tr_te)) == cudaSuccess) ? 0 : 1;
}
#define TR_ON (blockIdx.x == SV_PRED_TRACE)
#endif
#define PP_T0() const long long pp0_ = clock64();
#ifdef SV_PRED_TRACE_ONLY
#define PP_ATOMIC(i_, v_)
#else
#define PP_ATOMIC(i_, v_) atomicAdd(&sv_pred_prof[i_], (unsigned long long)(v_));
#endif
#define PP_ADD(i_) if ((threadIdx.x & 31) == 0) { PP_ATOMIC(i_, clock64() - pp0_) }
#else
#define PP_T0()
#define PP_ADD(i_)
#endif

namespace sv {
namespace {

__host__ __device__ inline int gcd_pred(int a, int b) {
  while (b) { const int t = a % b; a = b; b = t; }
  return a;
}

constexpr int BM = 128;
constexpr int NUM_WARPS = 12;   // WG0/WG1 softmax slot 0/1, warp 8 MMA, 9 K, 10 Q, 11 selection
constexpr int NUM_THREADS = NUM_WARPS * 32;
constexpr int WARP_MMA = 8, WARP_K = 9, WARP_Q = 10, WARP_SEL = 11;
constexpr int REG_LAUNCH = 168;
constexpr int REG_SOFTMAX = 208;
constexpr int REG_OTHER = 88;
static_assert(8 * (REG_SOFTMAX - REG_LAUNCH) <= 4 * (REG_LAUNCH - REG_OTHER), "register pool");
constexpr uint32_t TMEM_COLS = 512;
constexpr int EMU_EVERY = SV_PRED_EMU_EVERY;
constexpr int SMEM_LIMIT = 232448;
constexpr int MAXQ = 4;
// q full/empty, kv full/empty, s full/free [2][2], part full/free [2][2]
constexpr int NBARS = 2 * MAXQ + 2 * 8 + 8 + 8;

template <int D, int BLK>
struct PCfg {
  static constexpr int NBOX = D / 64;
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int STAGE_BYTES = BLK * D * 2;
  static constexpr int G = BM / BLK;                     // query blocks per tile
  static constexpr int SEG = BLK < 32 ? BLK : 32;        // rows reduced by one shuffle segment
  static constexpr int NSEG = BM / SEG;
  // bytes of everything but the Q buffers and the K ring
  static size_t fixed(int g_kv) {
    return size_t(2) * g_kv * BM * 4 /* block sums */ + size_t(4) * NSEG * g_kv * 4 /* parts */ +
           size_t((g_kv + 1) & ~1) * 4 /* selection row */ + NBARS * 8 + 16;
  }
  // (Q buffers, K stages) that fit, preferring 4 Q buffers (both tiles of the next round
  // prefetched); nst = 0 if nothing fits
  static void plan(int g_kv, int& nqb, int& nst) {
    for (nqb = SV_PRED_QB; nqb >= 2; --nqb) {
      const long long left = SMEM_LIMIT - (long long)fixed(g_kv) - (long long)nqb * Q_BYTES;
      nst = left > 0 ? (int)(left / STAGE_BYTES) : 0;
      if (nst > 8) nst = 8;
      if (nst >= 2) return;
    }
    nst = 0;
  }
  static size_t smem(int g_kv, int nqb, int nst) {
    return size_t(nqb) * Q_BYTES + size_t(nst) * STAGE_BYTES + fixed(g_kv);
  }
};

template <int D, int BLK>
__global__ void __launch_bounds__(NUM_THREADS, 1)
predict_kernel(const __grid_constant__ CUtensorMap tmap_q,
               const __grid_constant__ CUtensorMap tmap_k, const PredArgs a, int nqb, int nst) {
  using C = PCfg<D, BLK>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int n = a.g_kv;                                  // KV steps of every tile
  uint8_t* sQ = smem;
  uint8_t* sK = smem + nqb * C::Q_BYTES;
  float* sums = reinterpret_cast<float*>(sK + nst * C::STAGE_BYTES);   // [2][n][BM]
  float* part = sums + 2 * n * BM;                              // [2 slots][2 bufs][NSEG][n]
  float* sel_row = part + 4 * C::NSEG * n;                      // [n] selection warp's mass row
  uint64_t* bars = reinterpret_cast<uint64_t*>(sel_row + ((n + 1) & ~1));   // 8-byte aligned
  uint64_t* q_full = bars;           // [MAXQ]
  uint64_t* q_empty = q_full + MAXQ; // [MAXQ]
  uint64_t* kv_full = q_empty + MAXQ;// [8]
  uint64_t* kv_empty = kv_full + 8;  // [8]
  uint64_t* s_full = kv_empty + 8;   // [2 slots][2 bufs]
  uint64_t* s_free = s_full + 4;     // [2 slots][2 bufs] (128 arrivals)
  uint64_t* part_full = s_free + 4;  // [2 slots][2 bufs] (128 arrivals)
  uint64_t* part_free = part_full + 4;   // [2 slots][2 bufs]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + NBARS);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_tiles = (a.n_q + BM - 1) / BM;
  const int items = n_tiles * a.bh;
#if SV_PRED_ORDER == 0
  // contiguous, equal-size range of tiles (every tile costs the same n steps)
  const int lo = (int)((long long)items * blockIdx.x / gridDim.x);
  const int hi = (int)((long long)items * (blockIdx.x + 1) / gridDim.x);
  const int T = hi - lo;
  // global tile (head * n_tiles + tile) of slot use k (slot k & 1, round k >> 1), or -1
  auto tile_of = [&](int k) -> int { return k < T ? lo + k : -1; };
#else
  // Rounds of two tiles (one per slot).  FULL rounds take pairs of adjacent tiles of one (b,h)
  // (both slots share every K stage), dealt in strided windows: round r of CTA c takes pair
  // r * grid + (c + rot * r) mod grid, so the grid works on ~grid consecutive pairs at a time (a
  // few heads, their K_{<=S} L2-resident).  For an odd tile count the last tile of every head is
  // a SINGLE round (slot 1 idle), dealt one per CTA starting with the CTAs that have one full
  // round fewer.
  (void)items;
  const int fp = n_tiles / 2;
  const int n_full = fp * a.bh;
  const int n_single = (n_tiles & 1) ? a.bh : 0;
  const int grid = gridDim.x;
  int rot = 59;
  while (grid > 1 && gcd_pred(rot % grid, grid) != 1) rot += 2;
  const int k_full = n_full / grid, rem = n_full - k_full * grid;
  const int pos = (int)((blockIdx.x + (long long)k_full * rot) % grid);
  const int mine_full = k_full + (pos < rem ? 1 : 0);
  const int s_first = (pos - rem + grid) % grid;
  const int mine_single = s_first < n_single ? (n_single - s_first + grid - 1) / grid : 0;
  const int T = 2 * (mine_full + mine_single);
  auto tile_of = [&](int k) -> int {
    const int r = k >> 1, t = k & 1;
    if (r < mine_full) {
      const int pr = r * grid + (int)((blockIdx.x + (long long)r * rot) % grid);
      return (pr / fp) * n_tiles + 2 * (pr % fp) + t;
    }
    if (t == 1 || r - mine_full >= mine_single) return -1;
    const int sg = s_first + (r - mine_full) * grid;
    return sg * n_tiles + n_tiles - 1;
  };
#endif

  if (threadIdx.x == 0) {
    if ((smem_u32(smem) & 1023u) != 0) {
      printf("sparvar: dynamic shared memory not 1024-byte aligned\n");
      __trap();
    }
    for (int i = 0; i < MAXQ; ++i) {
      mbar_init(q_full + i, 1);
      mbar_init(q_empty + i, 1);
    }
    for (int i = 0; i < 8; ++i) {
      mbar_init(kv_full + i, 1);
      mbar_init(kv_empty + i, 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(s_free + i, BM);
      mbar_init(part_full + i, BM);
      mbar_init(part_free + i, 1);
    }
    fence_barrier_init();
  }
  if (warp == WARP_K && lane == 0) prefetch_tmap(&tmap_k);
  if (warp == WARP_Q && lane == 0) prefetch_tmap(&tmap_q);
  if (warp == WARP_MMA) {
    tmem_alloc(tmem_slot, TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // slot use k (tile tile_of(k)) runs in slot k & 1, round k >> 1; the valid uses take the Q
  // buffers in order (the q-th valid one buffer q % nqb).  Both slots of a round start and end
  // together (equal step counts); a round without slot 1 has tile_of(2r + 1) < 0.

  if (warp >= 8) {
    reg_dealloc<REG_OTHER>();
    if (warp == WARP_Q) {
      // ---------------------------------------------------------------- Q loader
      if (lane == 0) {
        int q = 0;
        for (int k = 0; k < T; ++k) {
          const int it = tile_of(k);
          if (it < 0) continue;
          const int b = q % nqb;
          if (q >= nqb) mbar_wait(q_empty + b, ((q / nqb) - 1) & 1);
          ++q;
          mbar_arrive_expect_tx(q_full + b, C::Q_BYTES);
#pragma unroll
          for (int x = 0; x < C::NBOX; ++x)
            tma_load_3d(sQ + b * C::Q_BYTES + x * (BM * 128), &tmap_q, q_full + b, x * 64,
                        (it % n_tiles) * BM, it / n_tiles);
        }
      }
    } else if (warp == WARP_K) {
      // ---------------------------------------------------------------- K loader
      if (lane == 0) {
        const uint64_t pol = policy_evict_last();
        int idx = 0;
        for (int r = 0; 2 * r < T; ++r) {
          const int it0 = tile_of(2 * r), it1 = tile_of(2 * r + 1);
          const int bh0 = it0 / n_tiles;
          const bool two = it1 >= 0;
          const bool shared = two && it1 / n_tiles == bh0;
          for (int j = 0; j < n; ++j) {
            for (int t = 0; t < (two && !shared ? 2 : 1); ++t) {
              const int bh = (t ? it1 : it0) / n_tiles;
              const int s = idx % nst;
              const uint32_t ph = (idx / nst) & 1;
              ++idx;
              { PP_T0() mbar_wait(kv_empty + s, ph ^ 1); PP_ADD(3) }
              mbar_arrive_expect_tx(kv_full + s, C::STAGE_BYTES);
#pragma unroll
              for (int x = 0; x < C::NBOX; ++x)
                tma_load_3d_hint(sK + s * C::STAGE_BYTES + x * (BLK * 128), &tmap_k, kv_full + s,
                                 x * 64, j * BLK, bh, pol);
            }
          }
        }
      }
    } else if (warp == WARP_SEL) {
      // ---------------------------------------------------------------- selection
      // Tile k's per-warp partial masses arrive in part[k & 1][(k >> 1) & 1]; this warp sums the
      // segments of each query block into its mass row and selects with ballots into bit rows,
      // off the softmax warps' critical path.
      const int W = (n + 31) / 32;
      constexpr int SEG_PER_G = BLK / C::SEG;
      for (int k = 0; k < T; ++k) {
        const int t = k & 1, kk = k >> 1, pb = kk & 1;
        const float* pt = part + (t * 2 + pb) * C::NSEG * n;
        const int it = tile_of(k);
        if (it < 0) continue;
        mbar_wait(part_full + 2 * t + pb, (kk >> 1) & 1);
        const int bh = it / n_tiles, tile = it % n_tiles;
        for (int gq = 0; gq < C::G; ++gq) {
          const int u = tile * C::G + gq;
          if (u >= a.g_q) break;
          for (int v = lane; v < n; v += 32) {
            float acc = 0.f;
            for (int sgi = 0; sgi < SEG_PER_G; ++sgi) acc += pt[(gq * SEG_PER_G + sgi) * n + v];
            sel_row[v] = acc;
          }
          __syncwarp();
          const long long r = (long long)bh * a.g_q + u;
          const int rows_u = min(BLK, a.n_q - u * BLK);
          const float thr = a.tau * float(rows_u);
          for (int w0 = 0; w0 < W; ++w0) {
            const int v = w0 * 32 + lane;
            bool sel = false;
            if (v < n) {
              const float mv = sel_row[v];
              if (a.mode == 0) {
                int rank = 0;
#pragma unroll 8
                for (int tt = 0; tt < n; ++tt) {
                  const float mt = sel_row[tt];
                  rank += (mt > mv) || (mt == mv && tt < v);
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
          __syncwarp();   // sel_row is rewritten by the next query block
        }
        if (lane == 0) mbar_arrive(part_free + 2 * t + pb);
      }
    } else if (warp == WARP_MMA) {
      // ---------------------------------------------------------------- tcgen05 issuer
      constexpr uint32_t IDESC = idesc_bf16_f32(BM, BLK, 0, 0);
      const bool leader = elect_one();
      const uint64_t dq0 = sdesc_sw128(smem_u32(sQ), 16, 1024);
      const uint64_t dk0 = sdesc_sw128(smem_u32(sK), 16, 1024);
      // ring positions and Q buffer indices as incremental counters: no integer division on the
      // issue path (the issuer shares its SM sub-partition with two softmax warps)
      int ring_s = 0;
      uint32_t ring_ph = 0;
      int qbuf = 0;                        // Q buffer of slot use k = 2r (round r's first tile)
      uint32_t qph = 0;                    // its use parity
      uint32_t step0 = 0, step1 = 0;   // S buffer uses per slot
      PP_T0()
      for (int r = 0; 2 * r < T; ++r) {
        const int it0 = tile_of(2 * r), it1 = tile_of(2 * r + 1);
        const bool two = it1 >= 0;
        const bool shared = two && it1 / n_tiles == it0 / n_tiles;
        // Q buffers of the round's tiles (the q-th valid use: buffer q % nqb, parity (q / nqb) & 1)
        int qb[2];
        uint32_t qp[2];
        qb[0] = qbuf;
        qp[0] = qph;
        qb[1] = qbuf + 1 == nqb ? 0 : qbuf + 1;
        qp[1] = qbuf + 1 == nqb ? qph ^ 1 : qph;
        for (int t = 0; t < (two ? 2 : 1); ++t) {
          PP_T0() mbar_wait(q_full + qb[t], qp[t]); PP_ADD(2)
        }
        for (int u = 0; u < (two ? 2 : 1); ++u)
          if (++qbuf == nqb) { qbuf = 0; qph ^= 1; }
        for (int j = 0; j < n; ++j) {
          int s = 0;
          for (int t = 0; t < (two ? 2 : 1); ++t) {
            const uint32_t g = t ? step1 : step0;
            if (t) ++step1; else ++step0;
            const int buf = g & 1;
            // softmax of this slot is done reading S[buf] (step g - 2)
            { PP_T0() mbar_wait(s_free + 2 * t + buf, ((g >> 1) & 1) ^ 1); PP_ADD(0) }
            if (t == 0 || !shared) {
              s = ring_s;
              { PP_T0() mbar_wait(kv_full + s, ring_ph); PP_ADD(1) }
              if (++ring_s == nst) { ring_s = 0; ring_ph ^= 1; }
            }
            tc_fence_after();
            const uint64_t da = dq0 + ((uint64_t)(qb[t] * C::Q_BYTES) >> 4);
            const uint64_t db = dk0 + ((uint64_t)(s * C::STAGE_BYTES) >> 4);
            {
            PP_T0()
            if (leader) {
#pragma unroll
              for (int kk = 0; kk < D / 16; ++kk) {
                const uint32_t oa = ((kk >> 2) * (BM * 128) + (kk & 3) * 32) >> 4;
                const uint32_t ob = ((kk >> 2) * (BLK * 128) + (kk & 3) * 32) >> 4;
                mma_ss(tmem + (2 * t + buf) * 128, da + oa, db + ob, IDESC, kk > 0);
              }
              if (t == 1 || !shared || !two) mma_commit(kv_empty + s);
              mma_commit(s_full + 2 * t + buf);
              if (j == n - 1) mma_commit(q_empty + qb[t]);
            }
            PP_ADD(8)
#ifdef SV_PRED_TRACE
            if (TR_ON && leader && g < 400) {
              sv_pred_tr_mma[t][g][0] = pp0_;
              sv_pred_tr_mma[t][g][1] = clock64();
            }
#endif
            }
            __syncwarp();
          }
        }
      }
      PP_ADD(5)
    }
    // no re-grow here: a loader that finished early would race the softmax warps' growth for
    // the CTA's register pool (setmaxnreg.inc blocks), and nothing after this needs registers
  } else {
    // ---------------------------------------------------------------- softmax warpgroups
    reg_alloc<REG_SOFTMAX>();
    const int t = warp >> 2;
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t t_row = tmem + (uint32_t(quarter * 32) << 16);
    const float sl2 = a.scale_log2;
    const uint64_t sl2x2 = f2_pack(sl2, sl2);
    float* my_sums = sums + t * n * BM;
    uint32_t g = 0;
#ifdef SV_PRED_PROF
    const long long ppk_ = clock64();
#endif
    for (int k = t; k < T; k += 2) {
      const int it = tile_of(k);
      if (it < 0) continue;
      const int tile = it % n_tiles;
      float m = -INFINITY;
      float l = 0.f;   // running sum of the stored block sums (relative to m)
      for (int j = 0; j < n; ++j, ++g) {
        const int buf = g & 1;
        { PP_T0()
          mbar_wait(s_full + 2 * t + buf, (g >> 1) & 1);
          if (quarter == 0) { PP_ADD(4) } else { PP_ADD(12) }
#ifdef SV_PRED_TRACE
          if (TR_ON && quarter == 0 && lane == 0 && g < 400) sv_pred_tr_sm[t][g][0] = pp0_;
#endif
        }
#ifdef SV_PRED_PROF
        const long long pps_ = clock64();
#endif
        tc_fence_after();
        uint32_t sr[BLK];
        if constexpr (BLK >= 32) {
#pragma unroll
          for (int c = 0; c < BLK; c += 32) tmem_ld32(t_row + (2 * t + buf) * 128 + c, sr + c);
        } else {
#pragma unroll
          for (int c = 0; c < BLK; c += 8) tmem_ld8(t_row + (2 * t + buf) * 128 + c, sr + c);
        }
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(s_free + 2 * t + buf);
        const int valid = min(BLK, a.n_kv - j * BLK);   // ragged last KV block (READING 20)
        if (__builtin_expect(valid < BLK, 0)) {
#pragma unroll
          for (int c = 0; c < BLK; ++c)
            if (c >= valid) sr[c] = __float_as_uint(-INFINITY);
        }
        float mm[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < BLK; c += 4) {
          const int q = (c >> 2) & 3;
          mm[q] = fmax3(mm[q], __uint_as_float(sr[c]), __uint_as_float(sr[c + 1]));
          mm[q] = fmax3(mm[q], __uint_as_float(sr[c + 2]), __uint_as_float(sr[c + 3]));
        }
        const float mx_s = fmax3(fmaxf(mm[0], mm[1]), mm[2], mm[3]) * sl2;
        if (mx_s > m + 8.0f) {
          // lazy rescale of the row's stored block sums (rare after the first blocks)
          const float alpha = ex2(m - mx_s);
          for (int jj = 0; jj < j; ++jj) my_sums[jj * BM + row] *= alpha;
          l *= alpha;
          m = mx_s;
        }
        const uint64_t negm = f2_pack(-m, -m);
        uint64_t acc[4] = {0, 0, 0, 0};
        auto exp_sum = [&](auto emu) {
          constexpr int E = decltype(emu)::value;
#pragma unroll
          for (int c = 0; c < BLK; c += 2) {
            const uint64_t x =
                ffma2(f2_pack(__uint_as_float(sr[c]), __uint_as_float(sr[c + 1])), sl2x2, negm);
            float p0, p1;
            if (E > 0 && (c / 2) % (E > 0 ? E : 1) == E - 1) {
              ex2_emu2<4>(x, p0, p1);
            } else {
              float x0, x1;
              f2_unpack(x, x0, x1);
              p0 = ex2(x0);
              p1 = ex2(x1);
            }
            acc[(c >> 1) & 3] = fadd2(acc[(c >> 1) & 3], f2_pack(p0, p1));
          }
        };
        // the polynomial exp2 clamps -inf logits to 2^-126, so it only runs on unmasked steps
        // (warp-uniform branch; masked = the ragged last KV block)
        if (EMU_EVERY > 0 && __all_sync(0xffffffffu, valid == BLK))
          exp_sum(std::integral_constant<int, EMU_EVERY>());
        else
          exp_sum(std::integral_constant<int, 0>());
        const uint64_t s2 = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
        float s0, s1;
        f2_unpack(s2, s0, s1);
        my_sums[j * BM + row] = s0 + s1;
        l += s0 + s1;
#ifdef SV_PRED_PROF
        if (quarter == 0 && lane == 0) { PP_ATOMIC(6, clock64() - pps_) }
#ifdef SV_PRED_TRACE
        if (TR_ON && quarter == 0 && lane == 0 && g < 400) {
          sv_pred_tr_sm[t][g][1] = pps_;
          sv_pred_tr_sm[t][g][2] = clock64();
        }
#endif
#endif
      }
#ifdef SV_PRED_PROF
      const long long ppe_ = clock64();
#endif
      // ------------------------------------------------------------ tile end: masses
      // P[q, j] = 2^(s' - m) / l: each row's normalised block sums, reduced over the warp's 32
      // rows into part[t][pb][quarter][.] for the selection warp (double-buffered per slot)
      const bool row_valid = tile * BM + row < a.n_q;
      const float inv = row_valid ? 1.f / l : 0.f;
      const int kk = k >> 1, pb = kk & 1;
      float* pt = part + (t * 2 + pb) * C::NSEG * n;
      if (kk >= 2) mbar_wait(part_free + 2 * t + pb, ((kk >> 1) - 1) & 1);
      if constexpr (C::SEG == 32) {
        // transpose-reduce: 31 shuffles per 32 blocks; lane i ends with the sum of block j0 + i
        for (int j0 = 0; j0 < n; j0 += 32) {
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = j0 + i < n ? my_sums[(j0 + i) * BM + row] * inv : 0.f;
#pragma unroll
          for (int sh = 16; sh >= 1; sh >>= 1) {
            const bool up = (lane & sh) != 0;
#pragma unroll
            for (int i = 0; i < sh; ++i) {
              const float send = up ? v[i] : v[i + sh];
              const float keep = up ? v[i + sh] : v[i];
              v[i] = keep + __shfl_xor_sync(0xffffffffu, send, sh);
            }
          }
          if (j0 + lane < n) pt[quarter * n + j0 + lane] = v[0];
        }
      } else {
        for (int j = 0; j < n; ++j) {
          float w = my_sums[j * BM + row] * inv;
#pragma unroll
          for (int off = C::SEG / 2; off > 0; off >>= 1) w += __shfl_xor_sync(0xffffffffu, w, off);
          if ((lane % C::SEG) == 0) pt[(row / C::SEG) * n + j] = w;
        }
      }
      mbar_arrive(part_full + 2 * t + pb);
#ifdef SV_PRED_PROF
      if (quarter == 0 && lane == 0) { PP_ATOMIC(7, clock64() - ppe_) }
#ifdef SV_PRED_TRACE
      if (TR_ON && quarter == 0 && lane == 0 && (k >> 1) < 16) {
        sv_pred_tr_te[t][k >> 1][0] = ppe_;
        sv_pred_tr_te[t][k >> 1][1] = clock64();
      }
#endif
#endif
    }
#ifdef SV_PRED_PROF
    if (quarter == 0 && lane == 0) { PP_ATOMIC(9, clock64() - ppk_) }
#endif
    reg_dealloc<REG_LAUNCH>();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == WARP_MMA) {
    tc_fence_after();
    tmem_dealloc(tmem, TMEM_COLS);
  }
}

int num_sms_pred() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}

template <int D, int BLK>
cudaError_t launch_t(const CUtensorMap& tq, const CUtensorMap& tk, const PredArgs& a,
                     cudaStream_t st) {
  using C = PCfg<D, BLK>;
  int nqb, nst;
  C::plan(a.g_kv, nqb, nst);
  if (nst < 2) return cudaErrorInvalidValue;
  const size_t smem = C::smem(a.g_kv, nqb, nst);
  auto kern = predict_kernel<D, BLK>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
#if SV_PRED_ORDER == 0
  const long long items = (long long)((a.n_q + BM - 1) / BM) * a.bh;
#else
  const long long items = 2 * (((long long)((a.n_q + BM - 1) / BM) * a.bh + 1) / 2);
#endif
  if (items <= 0) return cudaSuccess;
  const int sms = num_sms_pred();
  const int grid = (int)(items >= 2LL * sms ? sms : (items + 1) / 2);
  kern<<<grid, NUM_THREADS, smem, st>>>(tq, tk, a, nqb, nst);
  return cudaGetLastError();
}

}  // namespace

size_t predictor_smem_bytes(int head_dim, int block, int g_kv) {
#define SV_CASE(D_, B_)                            \
  if (head_dim == D_ && block == B_) {             \
    int nqb, nst;                                  \
    PCfg<D_, B_>::plan(g_kv, nqb, nst);            \
    return nst < 2 ? ~size_t(0) : PCfg<D_, B_>::smem(g_kv, nqb, nst); \
  }
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
