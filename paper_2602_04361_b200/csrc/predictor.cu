// predictor.cu — decision-scale sparse-pattern predictor for sm_100a (a2 + a3 in DESIGN.md).
//
// For each (b,h) and query block u at the decision scale S (
// READINGS 10-13):
//     P = softmax(Q_S K_{<=S}^T * scale)               (fp32 logits from bf16, fp32 exp)
//     mass[u, v] = sum_{q in u} sum_{j in v, j < C_S} P[q, j]
//     keep TOPK(k) (ties to the smaller v) or mass >= tau * |u|, then OR the sink blocks.
//
// Design (DESIGN.md §7 "predict_kernel"):
//  * Persistent, one CTA per SM, NS tile SLOTS of 128 query rows, each with its own softmax
//    warpgroup and its own S accumulator in TMEM.  NS = 3 where shared memory allows it (three
//    softmax warps per SM sub-partition keep the MUFU pipe busier than two), else NS = 2 with a
//    double-buffered S per slot.  The tensor core computes a slot's next S while its softmax
//    reduces the current one (the softmax releases S as soon as its last TMEM load lands).
//  * Every tile has the same G_kvS KV steps, so the MMA warp and the K loader run the slots of a
//    round in lockstep; slots of a round on the same (b,h) share each K stage.
//  * Per (row, KV block) the softmax keeps the block sum of 2^(s*scale*log2e - m) relative to
//    the row's running max m (lazy: rescaled only when m grows by more than 2^8) and the row
//    total l in a register.  With NS = 3 a 128-key step is read from TMEM in two 64-column
//    chunks twice (max pass, then exp2 pass) to fit 152 registers per thread.  At the tile end
//    the rows are normalised by 1/l (exact: P[q, j] = 2^(s' - m) / l) and reduced per KV block
//    with a transpose-reduce into a partial-mass buffer; a selection warp sums the partials in a
//    fixed order (deterministic) and selects with ballots into bit rows.
//  * One in four exp2 pairs runs as a degree-4 polynomial on the FMA pipe (relative error
//    2.6e-6, well inside the 1e-4 mass tolerance) to take load off the MUFU pipe.
#include <cuda_bf16.h>
#include <cstdio>
#include <type_traits>

#include "kernels.h"
#include "ptx.cuh"
#include "kernel_util.cuh"

#ifndef SV_PRED_EMU_EVERY
#define SV_PRED_EMU_EVERY 4   // 1 in 4 exp2 pairs as a degree-4 polynomial on the FMA pipe
#endif
#ifndef SV_PRED_STRIDED
#define SV_PRED_STRIDED 1     // 1: groups of NS tiles dealt round-robin (K L2-resident), 0: ranges
#endif
#ifndef SV_PRED_MAX_SLOTS
#define SV_PRED_MAX_SLOTS 3   // 3: use three slots when shared memory allows, 2: always two
#endif

#ifdef SV_PRED_TRACE
// development timeline of one CTA (variant builds only): per slot and S use g, the issuer's
// s_free-wait start / MMA issue start / issue end and the softmax's s_full-wait start / S seen /
// step end (warp `quarter 0` of the slot, lane 0)
__device__ long long sv_ptr[3][320][6];
extern "C" int sparvar_pred_trace3(long long* out) {
  return cudaMemcpyFromSymbol(out, sv_ptr, sizeof(sv_ptr)) == cudaSuccess ? 0 : 1;
}
#define PTR(t_, g_, i_) if (blockIdx.x == SV_PRED_TRACE && (g_) < 320) sv_ptr[t_][g_][i_] = clock64();
#else
#define PTR(t_, g_, i_)
#endif

namespace sv {
namespace {

constexpr int BM = 128;
constexpr uint32_t TMEM_COLS = 512;
constexpr int EMU_EVERY = SV_PRED_EMU_EVERY;
constexpr int SMEM_LIMIT = 232448;
constexpr int MAXQ = 6;
// q full/empty [MAXQ], kv full/empty [8], s full/free [NS * NB <= 4], part full/free [NS][2]
constexpr int NBARS = 2 * MAXQ + 2 * 8 + 2 * 4 + 2 * 6;

template <int D, int BLK, int NS>
struct PCfg {
  static_assert(NS == 2 || NS == 3, "slots");
  static constexpr int NB = NS == 2 ? 2 : 1;              // S buffers per slot
  static constexpr int NUM_WARPS = 4 * NS + 4;           // softmax WGs, MMA, K, Q, selection
  static constexpr int NUM_THREADS = NUM_WARPS * 32;
  static constexpr int WARP_MMA = 4 * NS, WARP_K = 4 * NS + 1, WARP_Q = 4 * NS + 2,
                       WARP_SEL = 4 * NS + 3;
  static constexpr int REG_LAUNCH = NS == 2 ? 168 : 128;
  static constexpr int REG_OTHER = 88;
  // 208 / 136 (ptxas compiles every role within REG_LAUNCH; the softmax code of NS = 3 fits 128)
  static constexpr int REG_SOFTMAX = REG_LAUNCH + ((REG_LAUNCH - REG_OTHER) / NS) / 8 * 8;
  static_assert(NUM_THREADS * REG_LAUNCH <= 65536, "register file");
  static_assert(4 * NS * (REG_SOFTMAX - REG_LAUNCH) <= 4 * (REG_LAUNCH - REG_OTHER), "pool");
  static_assert(NS * NB * 128 <= (int)TMEM_COLS, "TMEM");
  static constexpr int HC = (NS == 2 || BLK <= 64) ? BLK : 64;   // S columns per TMEM read
  static constexpr int NCH = BLK / HC;                   // reads per pass
  static constexpr int NBOX = D / 64;
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int STAGE_BYTES = BLK * D * 2;
  static constexpr int G = BM / BLK;                     // query blocks per tile
  static constexpr int SEG = BLK < 32 ? BLK : 32;        // rows reduced by one shuffle segment
  static constexpr int NSEG = BM / SEG;
  // bytes of everything but the Q buffers and the K ring
  static size_t fixed(int g_kv) {
    return size_t(NS) * g_kv * BM * 4 /* block sums */ +
           size_t(2 * NS) * NSEG * g_kv * 4 /* partial masses */ +
           size_t((g_kv + 1) & ~1) * 4 /* selection row */ + NBARS * 8 + 16;
  }
  // (Q buffers, K stages) that fit: one Q buffer per slot plus as many prefetch buffers as fit
  // (up to one round ahead), then the K ring; nst = 0 if nothing fits
  static void plan(int g_kv, int& nqb, int& nst) {
    for (nqb = 2 * NS; nqb >= NS; --nqb) {
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

template <int D, int BLK, int NS>
__global__ void __launch_bounds__(PCfg<D, BLK, NS>::NUM_THREADS, 1)
predict_kernel(const __grid_constant__ CUtensorMap tmap_q,
               const __grid_constant__ CUtensorMap tmap_k, const PredArgs a, int nqb, int nst) {
  using C = PCfg<D, BLK, NS>;
  constexpr int NB = C::NB;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int n = a.g_kv;                                  // KV steps of every tile
  uint8_t* sQ = smem;
  uint8_t* sK = smem + nqb * C::Q_BYTES;
  float* sums = reinterpret_cast<float*>(sK + nst * C::STAGE_BYTES);   // [NS][n][BM]
  float* part = sums + NS * n * BM;                             // [NS slots][2 bufs][NSEG][n]
  float* sel_row = part + 2 * NS * C::NSEG * n;                 // [n] selection warp's mass row
  uint64_t* bars = reinterpret_cast<uint64_t*>(sel_row + ((n + 1) & ~1));   // 8-byte aligned
  uint64_t* q_full = bars;                 // [MAXQ]
  uint64_t* q_empty = q_full + MAXQ;       // [MAXQ]
  uint64_t* kv_full = q_empty + MAXQ;      // [8]
  uint64_t* kv_empty = kv_full + 8;        // [8]
  uint64_t* s_full = kv_empty + 8;         // [NS][NB]
  uint64_t* s_free = s_full + 4;           // [NS][NB] (128 arrivals)
  uint64_t* part_full = s_free + 4;        // [NS][2] (128 arrivals)
  uint64_t* part_free = part_full + 6;     // [NS][2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + NBARS);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_tiles = (a.n_q + BM - 1) / BM;
  const int items = n_tiles * a.bh;
  // slot use k runs in slot k % NS, round k / NS; tile_of(k) is its global query tile
  // (head * n_tiles + tile) or -1 (the valid slots of a round are a prefix)
#if SV_PRED_STRIDED
  // groups of NS consecutive tiles dealt round-robin over the CTAs: round r of CTA c takes group
  // r * grid + c, so at any time the grid works on ~grid * NS consecutive tiles (a few heads,
  // whose K_{<=S} stays L2-resident and is read from DRAM about once)
  const int n_groups = (items + NS - 1) / NS;
  const int rounds = (int)blockIdx.x < n_groups ? (n_groups - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int T = rounds * NS;
  auto tile_of = [&](int k) -> int {
    const int it = ((k / NS) * (int)gridDim.x + (int)blockIdx.x) * NS + k % NS;
    return it < items ? it : -1;
  };
#else
  // contiguous, equal-size range of tiles (every tile costs the same n steps)
  const int lo = (int)((long long)items * blockIdx.x / gridDim.x);
  const int hi = (int)((long long)items * (blockIdx.x + 1) / gridDim.x);
  const int T = hi - lo;
  auto tile_of = [&](int k) -> int { return k < T ? lo + k : -1; };
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
    }
    for (int i = 0; i < 6; ++i) {
      mbar_init(part_full + i, BM);
      mbar_init(part_free + i, 1);
    }
    fence_barrier_init();
  }
  if (warp == C::WARP_K && lane == 0) prefetch_tmap(&tmap_k);
  if (warp == C::WARP_Q && lane == 0) prefetch_tmap(&tmap_q);
  if (warp == C::WARP_MMA) {
    tmem_alloc(tmem_slot, TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= 4 * NS) {
    reg_dealloc<C::REG_OTHER>();
    if (warp == C::WARP_Q) {
      // ---------------------------------------------------------------- Q loader
      // the q-th valid use takes Q buffer q % nqb
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
    } else if (warp == C::WARP_K) {
      // ---------------------------------------------------------------- K loader
      // per round and KV step: one stage per distinct (b,h) among the round's slots, in slot order
      if (lane == 0) {
        const uint64_t pol = policy_evict_last();
        int ring_s = 0;
        uint32_t ring_ph = 0;
        for (int k0 = 0; k0 < T; k0 += NS) {
          int dh[NS], nd = 0;
#pragma unroll
          for (int t = 0; t < NS; ++t) {
            const int it = tile_of(k0 + t);
            if (it < 0) break;
            const int bh = it / n_tiles;
            bool seen = false;
            for (int d = 0; d < nd; ++d) seen = seen || dh[d] == bh;
            if (!seen) dh[nd++] = bh;
          }
          for (int j = 0; j < n; ++j) {
            for (int d = 0; d < nd; ++d) {
              const int s = ring_s;
              mbar_wait(kv_empty + s, ring_ph ^ 1);
              if (++ring_s == nst) { ring_s = 0; ring_ph ^= 1; }
              mbar_arrive_expect_tx(kv_full + s, C::STAGE_BYTES);
#pragma unroll
              for (int x = 0; x < C::NBOX; ++x)
                tma_load_3d_hint(sK + s * C::STAGE_BYTES + x * (BLK * 128), &tmap_k, kv_full + s,
                                 x * 64, j * BLK, dh[d], pol);
            }
          }
        }
      }
    } else if (warp == C::WARP_SEL) {
      // ---------------------------------------------------------------- selection
      // Use k's per-warp partial masses arrive in part[k % NS][(k / NS) & 1]; this warp sums the
      // segments of each query block into its mass row and selects with ballots into bit rows,
      // off the softmax warps' critical path.
      const int W = (n + 31) / 32;
      constexpr int SEG_PER_G = BLK / C::SEG;
      for (int k = 0; k < T; ++k) {
        const int t = k % NS, kk = k / NS, pb = kk & 1;
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
    } else if (warp == C::WARP_MMA) {
      // ---------------------------------------------------------------- tcgen05 issuer
      constexpr uint32_t IDESC = idesc_bf16_f32(BM, BLK, 0, 0);
      const bool leader = elect_one();
      const uint64_t dq0 = sdesc_sw128(smem_u32(sQ), 16, 1024);
      const uint64_t dk0 = sdesc_sw128(smem_u32(sK), 16, 1024);
      // ring positions and Q-buffer indices as incremental counters: no integer division on the
      // issue path (the issuer shares its SM sub-partition with softmax warps)
      int ring_s = 0;
      uint32_t ring_ph = 0;
      int qbuf = 0;                        // Q buffer of use k0 (the round's first slot)
      uint32_t qph = 0;                    // its use parity
      uint32_t step[NS];                   // S uses per slot
#pragma unroll
      for (int t = 0; t < NS; ++t) step[t] = 0;
      for (int k0 = 0; k0 < T; k0 += NS) {
        int ns = 0;                        // slots working this round (a prefix)
#pragma unroll
        for (int t = 0; t < NS; ++t)
          if (tile_of(k0 + t) >= 0) ns = t + 1;
        int qb[NS];
        bool first_is0[NS], first_self[NS], last_self[NS];   // K-stage sharing (same (b,h))
        uint32_t qp[NS];
        {
          int b = qbuf;
          uint32_t p = qph;
#pragma unroll
          for (int t = 0; t < NS; ++t) {
            qb[t] = b;
            qp[t] = p;
            if (++b == nqb) { b = 0; p ^= 1; }
          }
        }
        {
          int bhs[NS];
#pragma unroll
          for (int t = 0; t < NS; ++t) bhs[t] = t < ns ? tile_of(k0 + t) / n_tiles : -1 - t;
#pragma unroll
          for (int t = 0; t < NS; ++t) {
            int first = t;
#pragma unroll
            for (int u = t - 1; u >= 0; --u)
              if (bhs[u] == bhs[t]) first = u;
            bool later = false;
#pragma unroll
            for (int u = t + 1; u < NS; ++u) later = later || bhs[u] == bhs[t];
            first_self[t] = first == t;
            first_is0[t] = first == 0;
            last_self[t] = !later;
          }
        }
        for (int t = 0; t < ns; ++t) mbar_wait(q_full + qb[t], qp[t]);
        for (int u = 0; u < ns; ++u)
          if (++qbuf == nqb) { qbuf = 0; qph ^= 1; }
        for (int j = 0; j < n; ++j) {
          int stg0 = 0, stg1 = 0, stg_t = 0;   // ring stages of slots 0 and 1 this step
#pragma unroll
          for (int t = 0; t < NS; ++t) {
            if (t >= ns) break;
            const uint32_t g = step[t]++;
            const int buf = NB == 2 ? int(g & 1) : 0;
            const uint32_t fpar = (NB == 2 ? (g >> 1) : g) & 1;
            // the softmax of this slot is done reading this S buffer (use g - NB)
            if (lane == 0) { PTR(t, g, 0) }
            mbar_wait(s_free + t * NB + buf, fpar ^ 1);
            if (first_self[t]) {
              stg_t = ring_s;
              mbar_wait(kv_full + ring_s, ring_ph);
              if (++ring_s == nst) { ring_s = 0; ring_ph ^= 1; }
            } else {
              stg_t = first_is0[t] ? stg0 : stg1;
            }
            if (t == 0) stg0 = stg_t;
            if (t == 1) stg1 = stg_t;
            tc_fence_after();
            const uint64_t da = dq0 + ((uint64_t)(qb[t] * C::Q_BYTES) >> 4);
            const uint64_t db = dk0 + ((uint64_t)(stg_t * C::STAGE_BYTES) >> 4);
            if (leader) {
              PTR(t, g, 1)
#pragma unroll
              for (int kk = 0; kk < D / 16; ++kk) {
                const uint32_t oa = ((kk >> 2) * (BM * 128) + (kk & 3) * 32) >> 4;
                const uint32_t ob = ((kk >> 2) * (BLK * 128) + (kk & 3) * 32) >> 4;
                mma_ss(tmem + (t * NB + buf) * 128, da + oa, db + ob, IDESC, kk > 0);
              }
              PTR(t, g, 2)
              if (last_self[t]) mma_commit(kv_empty + stg_t);
              mma_commit(s_full + t * NB + buf);
              if (j == n - 1) mma_commit(q_empty + qb[t]);
            }
            __syncwarp();
          }
        }
      }
    }
    // no re-grow here: a loader that finished early would race the softmax warps' growth for
    // the CTA's register pool (setmaxnreg.inc blocks), and nothing after this needs registers
  } else {
    // ---------------------------------------------------------------- softmax warpgroups
    reg_alloc<C::REG_SOFTMAX>();
    constexpr int HC = C::HC, NCH = C::NCH;
    const int t = warp >> 2;
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t t_row = tmem + (uint32_t(quarter * 32) << 16);
    const float sl2 = a.scale_log2;
    const uint64_t sl2x2 = f2_pack(sl2, sl2);
    float* my_sums = sums + t * n * BM;
    uint32_t g = 0;
    auto load_chunk = [&](uint32_t col, uint32_t* sr) {
      if constexpr (HC >= 32) {
#pragma unroll
        for (int c = 0; c < HC; c += 32) tmem_ld32(t_row + col + c, sr + c);
      } else {
#pragma unroll
        for (int c = 0; c < HC; c += 8) tmem_ld8(t_row + col + c, sr + c);
      }
    };
    auto mask_chunk = [&](uint32_t* sr, int c0, int valid) {
      if (__builtin_expect(valid < c0 + HC, 0)) {
#pragma unroll
        for (int c = 0; c < HC; ++c)
          if (c0 + c >= valid) sr[c] = __float_as_uint(-INFINITY);
      }
    };
    auto max_chunk = [&](const uint32_t* sr, float* mm) {
#pragma unroll
      for (int c = 0; c < HC; c += 4) {
        const int q = (c >> 2) & 3;
        mm[q] = fmax3(mm[q], __uint_as_float(sr[c]), __uint_as_float(sr[c + 1]));
        mm[q] = fmax3(mm[q], __uint_as_float(sr[c + 2]), __uint_as_float(sr[c + 3]));
      }
    };
    // sum of 2^(s * sl2 - m) over a chunk; column c0 + c of the step picks the emulated pairs
    auto exp_chunk = [&](const uint32_t* sr, int c0, uint64_t negm, uint64_t* acc, auto emu) {
      constexpr int E = decltype(emu)::value;
#pragma unroll
      for (int c = 0; c < HC; c += 2) {
        const uint64_t x =
            ffma2(f2_pack(__uint_as_float(sr[c]), __uint_as_float(sr[c + 1])), sl2x2, negm);
        float p0, p1;
        if (E > 0 && ((c0 + c) / 2) % (E > 0 ? E : 1) == E - 1) {
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
    for (int k = t; k < T; k += NS) {
      const int it = tile_of(k);
      if (it < 0) continue;
      const int tile = it % n_tiles;
      float m = -INFINITY;
      float l = 0.f;   // running sum of the stored block sums (relative to m)
      for (int j = 0; j < n; ++j, ++g) {
        const int buf = NB == 2 ? int(g & 1) : 0;
        const uint32_t spar = (NB == 2 ? (g >> 1) : g) & 1;
        const uint32_t s_col = (t * NB + buf) * 128;
        if (quarter == 0 && lane == 0) { PTR(t, g, 3) }
        mbar_wait(s_full + t * NB + buf, spar);
        if (quarter == 0 && lane == 0) { PTR(t, g, 4) }
        tc_fence_after();
        const int valid = min(BLK, a.n_kv - j * BLK);   // ragged last KV block (READING 20)
        uint32_t sr[HC];
        float mm[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        if constexpr (NCH == 1) {
          load_chunk(s_col, sr);
          tmem_wait_ld();
          tc_fence_before();
          mbar_arrive(s_free + t * NB + buf);
          mask_chunk(sr, 0, valid);
          max_chunk(sr, mm);
        } else {
          // pass 1: the row max over the step, one chunk at a time
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) {
            load_chunk(s_col + ch * HC, sr);
            tmem_wait_ld();
            mask_chunk(sr, ch * HC, valid);
            max_chunk(sr, mm);
          }
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
        // the polynomial exp2 clamps -inf logits to 2^-126, so it only runs on unmasked steps
        // (valid depends on j only: CTA-uniform)
        const bool emu_ok = EMU_EVERY > 0 && valid == BLK;
        if constexpr (NCH == 1) {
          if (emu_ok) exp_chunk(sr, 0, negm, acc, std::integral_constant<int, EMU_EVERY>());
          else exp_chunk(sr, 0, negm, acc, std::integral_constant<int, 0>());
        } else {
          // pass 2: exp2 sums, starting with the last chunk, still in registers from pass 1;
          // S is released once the other chunks are in registers
          if (emu_ok) exp_chunk(sr, (NCH - 1) * HC, negm, acc, std::integral_constant<int, EMU_EVERY>());
          else exp_chunk(sr, (NCH - 1) * HC, negm, acc, std::integral_constant<int, 0>());
#pragma unroll
          for (int ch = 0; ch < NCH - 1; ++ch) {
            load_chunk(s_col + ch * HC, sr);
            tmem_wait_ld();
            if (ch == NCH - 2) {
              tc_fence_before();
              mbar_arrive(s_free + t * NB + buf);
            }
            mask_chunk(sr, ch * HC, valid);
            if (emu_ok) exp_chunk(sr, ch * HC, negm, acc, std::integral_constant<int, EMU_EVERY>());
            else exp_chunk(sr, ch * HC, negm, acc, std::integral_constant<int, 0>());
          }
        }
        const uint64_t s2 = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
        float s0, s1;
        f2_unpack(s2, s0, s1);
        my_sums[j * BM + row] = s0 + s1;
        if (quarter == 0 && lane == 0) { PTR(t, g, 5) }
        l += s0 + s1;
      }
      // ------------------------------------------------------------ tile end: masses
      // P[q, j] = 2^(s' - m) / l: each row's normalised block sums, reduced over the warp's 32
      // rows into part[t][pb][quarter][.] for the selection warp (double-buffered per slot)
      const bool row_valid = tile * BM + row < a.n_q;
      const float inv = row_valid ? 1.f / l : 0.f;
      const int kk = k / NS, pb = kk & 1;
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
    }
    reg_dealloc<C::REG_LAUNCH>();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == C::WARP_MMA) {
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

// slot count for a shape's shared memory: three slots when their statistics and one Q buffer
// per slot fit (launch_t also requires more than two tiles per SM)
template <int D, int BLK>
int pick_slots(int g_kv) {
  int nqb, nst;
  if (SV_PRED_MAX_SLOTS >= 3) {
    PCfg<D, BLK, 3>::plan(g_kv, nqb, nst);
    if (nst >= 2) return 3;
  }
  PCfg<D, BLK, 2>::plan(g_kv, nqb, nst);
  return nst >= 2 ? 2 : 0;
}

template <int D, int BLK, int NS>
cudaError_t launch_ns(const CUtensorMap& tq, const CUtensorMap& tk, const PredArgs& a,
                      cudaStream_t st) {
  using C = PCfg<D, BLK, NS>;
  int nqb, nst;
  C::plan(a.g_kv, nqb, nst);
  if (nst < 2) return cudaErrorInvalidValue;
  const size_t smem = C::smem(a.g_kv, nqb, nst);
  auto kern = predict_kernel<D, BLK, NS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long long items = (long long)((a.n_q + BM - 1) / BM) * a.bh;
  if (items <= 0) return cudaSuccess;
  const int sms = num_sms_pred();
  const int grid = (int)(items >= (long long)NS * sms ? sms : (items + NS - 1) / NS);
  kern<<<grid, C::NUM_THREADS, smem, st>>>(tq, tk, a, nqb, nst);
  return cudaGetLastError();
}

template <int D, int BLK>
cudaError_t launch_t(const CUtensorMap& tq, const CUtensorMap& tk, const PredArgs& a,
                     cudaStream_t st) {
  // three slots only pay with more than two tiles per SM: a lone three-slot round is ~1.2x
  // the time of a two-slot round (the third softmax warp shares the sub-partition's MUFU)
  const long long items = (long long)((a.n_q + BM - 1) / BM) * a.bh;
  int ns = pick_slots<D, BLK>(a.g_kv);
  if (ns == 3 && items <= 2LL * num_sms_pred()) ns = 2;
  if (ns == 3) return launch_ns<D, BLK, 3>(tq, tk, a, st);
  if (ns == 2) return launch_ns<D, BLK, 2>(tq, tk, a, st);
  return cudaErrorInvalidValue;
}

}  // namespace

size_t predictor_smem_bytes(int head_dim, int block, int g_kv) {
#define SV_CASE(D_, B_)                                                        \
  if (head_dim == D_ && block == B_) {                                         \
    int nqb, nst;                                                              \
    const int ns = pick_slots<D_, B_>(g_kv);                                   \
    if (ns == 3) {                                                             \
      PCfg<D_, B_, 3>::plan(g_kv, nqb, nst);                                   \
      return PCfg<D_, B_, 3>::smem(g_kv, nqb, nst);                            \
    }                                                                          \
    if (ns == 2) {                                                             \
      PCfg<D_, B_, 2>::plan(g_kv, nqb, nst);                                   \
      return PCfg<D_, B_, 2>::smem(g_kv, nqb, nst);                            \
    }                                                                          \
    return ~size_t(0);                                                         \
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
