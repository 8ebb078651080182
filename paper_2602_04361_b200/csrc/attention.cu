// attention.cu — block-sparse (and dense) cross-scale attention forward for sm_100a.
//
// Computes, for every (b,h) and query block u, o_t = softmax_J(q_t . k_j * scale) V_J over the
// real tokens J of the KV blocks listed for u (PAPER.md:204-212 Eq. attn_cross_scale,
// PAPER.md:318-328 Eq. sparse_update, PAPER.md:397-407 Eq. block_mask; READINGS 9, 17, 20).
//
// Design (DESIGN.md §7 "attn_fwd_kernel"):
//  * Persistent, one CTA per SM (all 512 TMEM columns).  The 128-row query tiles ("items",
//    (b,h)-major) are dealt in strided windows: CTA c takes position (c + 59 k) mod grid of the
//    k-th window of `grid` consecutive items, so at any time the grid works on a few heads whose
//    K/V stay in L2 (SV_ORDER=0: cost-balanced contiguous ranges found by a warp-parallel search
//    over row_ptr).
//  * Two tile SLOTS per CTA, each with its own S/P (128 TMEM cols) and O (D cols) accumulators
//    and its own softmax warpgroup: the tensor core works on one slot while the other slot's
//    softmax runs.  The MMA warp issues in a fixed round-robin order (per round and slot:
//    O += P_j V_j once all of P is written, then S = Q K_{j+1}^T or the next tile's first S), and
//    every role derives the same order from a per-CTA schedule (thread 0 simulates the
//    round-robin once per batch of up to MAX_TILES tiles), so one KV ring serves both slots.
//    The issuer polls its barriers (a suspended try_wait wakes late and idles the tensor pipe).
//  * Q lives in 3 shared buffers (two current tiles + one prefetched); a buffer is released by
//    the commit of its tile's last Q K^T and the schedule gives each new tile the earliest
//    pending release (that release precedes the tile's first MMA, so no deadlock).
//  * S (fp32) and O (fp32) live in TMEM; P (bf16) overwrites S in place and is the TMEM A operand
//    of P.V (tcgen05 ops of one thread execute in issue order, so the next Q K^T cannot clobber P
//    early).  fp32 online softmax in the exp2 domain with lazy rescale of O (only when the running
//    max grows by more than 2^8); the S_j commit also covers P_{j-1} V_{j-1}.
//  * A separate epilogue warpgroup drains each finished tile (TMEM O -> 1/l -> bf16 -> global,
//    LSE) in completion order, so the softmax warpgroup starts the slot's next tile at once; the
//    next tile's first P.V waits on "O drained".  Q loads and O stores carry an L2 evict-first
//    policy (read / written once), K/V loads evict-last (re-read by other tiles of the head).
//  * MASS instantiation (NEXT(3), sparvar_dense_attn_mass): the softmax warps also store each
//    step's block sum and reference max for the fused predictor (mass_select_kernel).
//  * NEXT(1): an optional NN-upsampled residual is added in the epilogue.
//  * Block sizes below 128: a 128-row tile holds G = 128/B query blocks; the KV steps are the
//    ascending union of their lists and each row masks the steps its own block does not list.
//    The ragged last KV block is masked to -inf (READING 20): TMA zero fill alone gives logit 0.
#include <cuda_bf16.h>
#include <cstdio>

#include "kernels.h"
#include "ptx.cuh"
#include "kernel_util.cuh"

#ifdef SV_PROF
// Development instrumentation (variant libraries only, scripts/build_variant.sh).
__device__ long long sv_prof_buf[24576];
extern "C" int sparvar_prof_read(long long* host, int n) {
  return cudaMemcpyFromSymbol(host, sv_prof_buf, sizeof(long long) * n) == cudaSuccess ? 0 : 1;
}
#define SV_STAMP(i_) \
  if (blockIdx.x == 0 && (threadIdx.x & 127) == 0 && threadIdx.x < 256 && (i_) < 2500) \
    sv_prof_buf[(i_) + (threadIdx.x >> 7) * 2500] = clock64();
#define SV_STAMP_CTA(base_) \
  if (threadIdx.x == 0 && blockIdx.x < 192) sv_prof_buf[(base_) + blockIdx.x] = (long long)globaltimer_ns();
#ifdef SV_PROF_LITE   // timeline stamps only: no per-wait atomics
#define SV_ACC(base_, v_) {}
#else
#define SV_ACC(base_, v_) \
  if (blockIdx.x < 192) atomicAdd((unsigned long long*)&sv_prof_buf[(base_) + blockIdx.x], (unsigned long long)(v_));
#endif
#define SV_CLK() clock64()
// MMA issuer op trace of CTA 0: [8192 + 4 * op + {0: before P wait, 1: after, 2: PV issued, 3: QK issued}]
#define SV_OPSTAMP(op_, k_) \
  if (blockIdx.x == 0 && lane == 0 && (op_) < 1000) sv_prof_buf[8192 + 8 * (op_) + (k_)] = clock64();
extern "C" int sparvar_prof_reset() {
  static long long z[24576];
  return cudaMemcpyToSymbol(sv_prof_buf, z, sizeof(z)) == cudaSuccess ? 0 : 1;
}
#else
#define SV_STAMP(i_) {}
#define SV_STAMP_CTA(base_) {}
#define SV_ACC(base_, v_) {}
#define SV_CLK() 0LL
#define SV_OPSTAMP(op_, k_) {}
#endif

#ifndef SV_EMU_EVERY
#define SV_EMU_EVERY 0
#endif

namespace sv {
namespace {

constexpr int BM = 128;                  // query rows per tile (TMEM lanes)
constexpr int NUM_WARPS = 16;            // WG0/WG1 softmax slot 0/1, WG2 MMA/KV/Q/zero, WG3 epilogue
constexpr int NUM_THREADS = NUM_WARPS * 32;
constexpr int WARP_MMA = 8, WARP_KV = 9, WARP_Q = 10, WARP_ZERO = 11, WARP_EPI = 12;
// setmaxnreg moves registers inside the CTA's own pool (launch: 16 warps x 128): the 8 softmax
// warps take 8 x 72 more, WG2 gives 4 x 64 and WG3 4 x 80 back.
constexpr int REG_LAUNCH = 128;
#ifndef SV_REG_SOFTMAX
#define SV_REG_SOFTMAX 200
#endif
#ifndef SV_REG_PRODUCER
#define SV_REG_PRODUCER 64
#endif
#ifndef SV_REG_EPILOGUE
#define SV_REG_EPILOGUE 48
#endif
constexpr int REG_SOFTMAX = SV_REG_SOFTMAX;
constexpr int REG_PRODUCER = SV_REG_PRODUCER;   // WG2: MMA issuer, loaders
constexpr int REG_EPILOGUE = SV_REG_EPILOGUE;   // WG3
static_assert(8 * (REG_SOFTMAX - REG_LAUNCH) <=
                  4 * (REG_LAUNCH - REG_PRODUCER) + 4 * (REG_LAUNCH - REG_EPILOGUE),
              "register pool");
constexpr int EMU_EVERY = SV_EMU_EVERY;  // 1 in EMU_EVERY exp2 pairs on the FMA pipe (0 = none)
constexpr uint32_t TMEM_COLS = 512;
#ifndef SV_NQB
#define SV_NQB 3
#endif
constexpr int NQB = SV_NQB;              // Q buffers
constexpr int MAX_TILES = 96;            // tiles per schedule batch
constexpr int TILE_OVERHEAD = 2;         // per-tile cost, in KV steps, for the balanced partition
constexpr int SMEM_LIMIT = 232448;       // 227 KB opt-in
constexpr uint8_t EMPTY_TILE = 0xFF;
#ifndef SV_ORDER
#define SV_ORDER 1
#endif
// Work order.  0: cost-balanced contiguous item ranges (one head per CTA at a time: every head is
// active at once, K/V working set far above L2).  1: strided windows -- at any time the CTAs work
// on ~grid consecutive items (a few heads, L2-resident K/V); CTA c takes position
// (c + k*R) mod grid of window k so a CTA does not keep drawing the same query-tile index.
constexpr int ORDER = SV_ORDER;
#ifndef SV_LEAN
#define SV_LEAN 1      // lean MMA issue loop (one P wait per op, no warp syncs)
#endif
// Q tiles are read once and O rows written once per launch: both carry an L2 evict-first
// policy so they do not push out the K/V blocks other CTAs are about to re-read (together
// -1% CSLA time in shuffled-order timing).
#ifndef SV_Q_EVICT_FIRST
#define SV_Q_EVICT_FIRST 1
#endif
#ifndef SV_O_EVICT_FIRST
#define SV_O_EVICT_FIRST 1
#endif
#ifndef SV_MMA_POLL
#define SV_MMA_POLL 1
#endif
#ifndef SV_MMA_SHADOW
#define SV_MMA_SHADOW 1
#endif
#ifndef SV_SFX_SHADOW
#define SV_SFX_SHADOW 1
#endif
// The MMA issuer polls its barriers (mbarrier.test_wait) instead of try_wait, which may
// suspend the thread: a suspended issuer wakes late and leaves the tensor pipe idle (-2.3% CSLA
// time in shuffled-order timing; polling in the K/V loader or the softmax warps gains nothing).
#if SV_MMA_POLL
#define SV_MMA_WAIT mbar_wait_spin
#elif SV_MMA_DBG
#define SV_MMA_WAIT(bar_, par_) mma_wait_dbg((bar_), (par_), kv_idx, (int)p_cnt0, (int)p_cnt1, jn0, jn1, icur0, icur1, __LINE__)
#else
#define SV_MMA_WAIT mbar_wait
#endif
// profiling builds: clocks the MMA issuer spends blocked, per barrier kind (base index)
#define SV_MMA_WAIT_T(bar_, par_, base_)                                   \
  {                                                                        \
    const long long t0_ = SV_CLK();                                        \
    SV_MMA_WAIT(bar_, par_);                                               \
    if ((threadIdx.x & 31) == 0) SV_ACC(base_, SV_CLK() - t0_)             \
  }

__host__ __device__ inline int gcd_int(int a, int b) {
  while (b) { const int t = a % b; a = b; b = t; }
  return a;
}

// Small shared state after the Q / KV buffers.
static_assert(kMaxKvSteps <= 0xFFFF, "Small::n holds a tile's KV step count in 16 bits");
struct Small {
  float2 stats[2][BM];          // per slot, per row: (1/l or 0, lse) handed softmax -> epilogue
  uint16_t n[MAX_TILES];        // KV steps of the batch's i-th tile (<= kMaxKvSteps, api.cu)
  uint8_t meta[MAX_TILES];      // slot | buf << 1 | (use parity of buf) << 3, or EMPTY_TILE
  uint8_t eord[MAX_TILES];      // completion order (for the epilogue)
  int T, Tn, lo, hi, uses;
  int mma_st[5];                // SV_MMA_SHADOW: issuer state between schedule batches
  int sfx_st[2][2];             // SV_SFX_SHADOW: per-slot softmax (S phases, tiles done)
  uint32_t tmem_slot;
  uint64_t bars[2 * NQB + 2 * 8 + 14];
};

template <int D, int BLK>
struct Cfg {
  static constexpr int NBOX = D / 64;                       // 64-element (128 B) TMA boxes per row
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int STAGE_BYTES = BLK * D * 2;
  static constexpr int AVAIL = SMEM_LIMIT - (int)sizeof(Small) - NQB * Q_BYTES;
  static constexpr int NST = AVAIL / STAGE_BYTES > 8 ? 8 : AVAIL / STAGE_BYTES;
  static constexpr int G = BM / BLK;                        // query blocks per tile
  static constexpr int SMEM = NQB * Q_BYTES + NST * STAGE_BYTES + (int)sizeof(Small);
  static_assert(NST >= 2, "KV ring too small");
  static_assert(NST <= 8, "barrier array sized for 8 stages");
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
    if (dense) return dense_end;
    if (G == 1) return end[0] - cur[0];
    Steps<G> c = *this;
    int n = 0, v;
    uint32_t m;
    while (c.next(a, v, m)) ++n;
    return n;
  }
};

// NEXT(1): source row of the nearest-neighbour upsampled cache residual for output query
// n_row of scale K: (x, y) = divmod(n_row, s_K) -> (floor(x s_S / s_K), floor(y s_S / s_K))
// (READING 22); nullptr when no residual is fused.
template <int D>
__device__ __forceinline__ const uint16_t* cache_row(const AttnArgs& a, int bh, int n_row) {
  if (a.add == nullptr) return nullptr;
  const int x = n_row / a.s_dst, y = n_row % a.s_dst;
  const int src = (x * a.s_src / a.s_dst) * a.s_src + (y * a.s_src / a.s_dst);
  return a.add + (long long)bh * a.add_stride + (long long)src * D;
}
__device__ __forceinline__ void load_cache16(const uint16_t* p, float* out) {
  if (p == nullptr) {
#pragma unroll
    for (int i = 0; i < 16; ++i) out[i] = 0.f;
    return;
  }
  const uint4 u0 = *reinterpret_cast<const uint4*>(p);
  const uint4 u1 = *reinterpret_cast<const uint4*>(p + 8);
  const uint32_t w[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    out[2 * i] = __uint_as_float(w[i] << 16);
    out[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

__device__ __forceinline__ void mma_wait_dbg(uint64_t* bar, uint32_t par, int kv, int p0, int p1,
                                             int j0, int j1, int i0, int i1, int line) {
  const uint32_t a = smem_u32(bar);
  if (mbar_try_wait(a, par)) return;
  const uint64_t t0 = globaltimer_ns();
  bool said = false;
  while (!mbar_try_wait(a, par)) {
    if (!said && globaltimer_ns() - t0 > 1000000000ull) {
      said = true;
      if ((threadIdx.x & 31) == 0) printf("MMA stuck: block %d lane %d line %d bar 0x%x par %u kv_idx %d p_cnt %d %d jn %d %d icur %d %d\n",
             blockIdx.x, threadIdx.x & 31, line, a, par, kv, p0, p1, j0, j1, i0, i1);
    }
  }
}

// Cost prefix F(i) of the first i items of [item_begin, item_end) (monotone in i): listed blocks
// (row_ptr prefix sums) + TILE_OVERHEAD per tile.
template <int G>
__device__ __forceinline__ long long cost_prefix(const AttnArgs& a, int item_begin, int i,
                                                 int n_tiles, int g_kv, int base_row) {
  if (a.row_ptr == nullptr) return (long long)(g_kv + TILE_OVERHEAD) * i;
  const int item = item_begin + i;
  const int bh = item / n_tiles, tile = item % n_tiles;
  const int row = bh * a.g_q + min(tile * G, a.g_q);
  return (long long)(__ldg(a.row_ptr + row) - base_row) + (long long)TILE_OVERHEAD * i;
}

// MASS (NEXT(3), decision-scale dense pass with fused block mass): every softmax thread also
// stores, per KV step (= key block v), its row's block sum sum_{j in v} 2^(x_j - m) and the m it
// is relative to (exp2 domain), for mass_select_kernel to normalise with the row's final LSE.
template <int D, int BLK, bool MASS = false>
__global__ void __launch_bounds__(NUM_THREADS, 1)
attn_fwd_kernel(const __grid_constant__ CUtensorMap tmap_q,
                const __grid_constant__ CUtensorMap tmap_k,
                const __grid_constant__ CUtensorMap tmap_v, const AttnArgs a, int item_begin,
                int item_end) {
  using C = Cfg<D, BLK>;
  constexpr int G = C::G;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ = smem;                                       // NQB x Q_BYTES
  uint8_t* sKV = smem + NQB * C::Q_BYTES;                   // NST x STAGE_BYTES
  Small* sm = reinterpret_cast<Small*>(sKV + C::NST * C::STAGE_BYTES);
  uint64_t* q_full = sm->bars;             // [NQB] Q tile landed
  uint64_t* q_empty = q_full + NQB;        // [NQB] last Q K^T of the buffer's tile complete
  uint64_t* kv_full = q_empty + NQB;       // [NST]
  uint64_t* kv_empty = kv_full + 8;        // [NST]
  uint64_t* s_bar = kv_empty + 8;          // [2] S_j of slot ready (also covers P_{j-1}V_{j-1})
  uint64_t* p_bar = s_bar + 2;             // [2][2] first / second half of P_j written (128)
  uint64_t* o_bar = p_bar + 4;             // [2] last P.V of the slot's tile complete
  uint64_t* o_free = o_bar + 2;            // [2] epilogue drained O of the slot (128)
  uint64_t* st_bar = o_free + 2;           // [2] softmax wrote the tile's row stats (128)
  uint64_t* st_free = st_bar + 2;          // [2] epilogue read them (128)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int g_kv = (a.n_kv + BLK - 1) / BLK;
  const int n_tiles = (a.n_q + BM - 1) / BM;
  SV_STAMP_CTA(7400)

  // ------------------------------------------------------------------ setup
  if (threadIdx.x == 0) {
    if ((smem_u32(smem) & 1023u) != 0) {
      printf("sparvar: dynamic shared memory not 1024-byte aligned\n");
      __trap();
    }
    for (int i = 0; i < NQB; ++i) {
      mbar_init(q_full + i, 1);
      mbar_init(q_empty + i, 1);
    }
    for (int i = 0; i < C::NST; ++i) {
      mbar_init(kv_full + i, 1);
      mbar_init(kv_empty + i, 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(s_bar + t, 1);
      mbar_init(p_bar + 2 * t, BM);
      mbar_init(p_bar + 2 * t + 1, BM);
      mbar_init(o_bar + t, 1);
      mbar_init(o_free + t, BM);
      mbar_init(st_bar + t, BM);
      mbar_init(st_free + t, BM);
    }
    sm->uses = 0;
#if SV_MMA_SHADOW
    for (int i = 0; i < 5; ++i) sm->mma_st[i] = 0;
#endif
#if SV_SFX_SHADOW
    for (int i = 0; i < 4; ++i) (&sm->sfx_st[0][0])[i] = 0;
#endif
    fence_barrier_init();
  }
  if (warp == WARP_KV && lane == 0) {
    prefetch_tmap(&tmap_k);
    prefetch_tmap(&tmap_v);
  }
  if (warp == WARP_Q && lane == 0) prefetch_tmap(&tmap_q);
  if (warp == WARP_MMA) {
    tmem_alloc(&sm->tmem_slot, TMEM_COLS);
    tmem_relinquish();
  }
  if (ORDER == 0 && warp == 1) {
    // balanced contiguous range [lo, hi) of this CTA: lanes 0-15 search the lower boundary,
    // lanes 16-31 the upper one, 16 probes per round (min i with F(i) >= target)
    const int N = item_end - item_begin;
    const int base_row =
        a.row_ptr == nullptr ? 0
                             : __ldg(a.row_ptr + (item_begin / n_tiles) * a.g_q +
                                     min((item_begin % n_tiles) * G, a.g_q));
    const long long total = cost_prefix<G>(a, item_begin, N, n_tiles, g_kv, base_row);
    const int half = lane >> 4, hl = lane & 15;
    const int c = blockIdx.x + half;
    const long long target = total * c / (long long)gridDim.x;
    int lo = -1, hi = N;                   // F(lo) < target <= F(hi)  (F(-1) = -inf)
    if (c == 0) hi = 0;
    if (c == (int)gridDim.x) lo = N - 1;
    while (__any_sync(0xffffffffu, hi - lo > 1)) {
      const int span = hi - lo;
      const int p = lo + (int)(((long long)span * (hl + 1)) / 17);
      const bool ok = span > 1 && p > lo && p < hi &&
                      cost_prefix<G>(a, item_begin, p, n_tiles, g_kv, base_row) >= target;
      const uint32_t m = __ballot_sync(0xffffffffu, ok) >> (half * 16) & 0xFFFFu;
      if (span > 1) {
        if (m != 0) {
          const int f = __ffs(m) - 1;
          hi = lo + (int)(((long long)span * (f + 1)) / 17);
          if (f > 0) lo = lo + (int)(((long long)span * f) / 17);
        } else {
          lo = lo + (int)(((long long)span * 16) / 17);
        }
      }
    }
    const int lo_res = __shfl_sync(0xffffffffu, hi, 0);
    const int hi_res = __shfl_sync(0xffffffffu, hi, 16);
    if (lane == 0) {
      sm->lo = item_begin + lo_res;
      sm->hi = item_begin + hi_res;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm->tmem_slot;
  // this CTA's items: item_at(li) for li in [0, n_mine), increasing
  const int N_items = item_end - item_begin;
  const int grid = gridDim.x;
  int rot = 59;
  while (gcd_int(rot % grid, grid) != 1 && grid > 1) rot += 2;
  const int k_full = N_items / grid;
  const int n_mine = ORDER == 0 ? sm->hi - sm->lo
                                : k_full + (((blockIdx.x + (long long)k_full * rot) % grid) <
                                                    N_items - k_full * grid ? 1 : 0);
  const int range_lo = ORDER == 0 ? sm->lo : 0;
  auto item_at = [&](int li) -> int {
    if (ORDER == 0) return range_lo + li;
    return item_begin + li * grid + (int)((blockIdx.x + (long long)li * rot) % grid);
  };
  SV_STAMP_CTA(7600)

  // role state that persists across schedule batches (barrier phases, ring positions)
  int kv_idx = 0;                  // KV loader / MMA: ring position
  uint32_t p_cnt0 = 0, p_cnt1 = 0; // MMA: P phases consumed per slot
  int tiles0 = 0, tiles1 = 0;      // MMA / softmax / epilogue: tiles done per slot
  uint32_t s_cnt = 0;              // softmax: S phases consumed
  uint32_t q_used = 0;             // Q loader: buffers used at least once (bits)

  for (int b0 = 0; b0 < n_mine; b0 += MAX_TILES) {
    const int T = min(MAX_TILES, n_mine - b0);
    for (int i = threadIdx.x; i < T; i += NUM_THREADS) {
      const int it = item_at(b0 + i);
      Steps<G> st;
      st.init(a, it / n_tiles, it % n_tiles, g_kv);
      sm->n[i] = (uint16_t)st.count(a);
    }
    __syncthreads();
    // round-robin simulation of the MMA order -> slot, Q buffer, start and completion order
    if (threadIdx.x == 0) {
      uint32_t uses = (uint32_t)sm->uses;
      int r0 = 0, r1 = 0, r2 = 0;          // pending release key per Q buffer
      int fin0 = 0, fin1 = 0;              // finish key of each slot's current tile
      int rend0 = 0, rend1 = 0;            // round at which it finishes
      int cur0 = -1, cur1 = -1;            // its index
      int k = 0, e = 0;
      for (int i = 0; i < T; ++i) {
        const int n = sm->n[i];
        if (n == 0) {
          sm->meta[i] = EMPTY_TILE;
          continue;
        }
        int slot, R;
        if (k < 2) {
          slot = k;
          R = -1;
        } else {
          slot = fin0 < fin1 ? 0 : 1;
          R = slot ? rend1 : rend0;
          sm->eord[e++] = (uint8_t)(slot ? cur1 : cur0);   // its predecessor completes now
        }
        int buf;
        if (k < NQB) {
          buf = k;
        } else if (NQB == 2) {
          buf = r0 <= r1 ? 0 : 1;
        } else {
          buf = (r0 <= r1 && r0 <= r2) ? 0 : (r1 <= r2 ? 1 : 2);
        }
        // op (round r, slot s) has key 2*(r+1)+s; last Q K^T at round R+n-1, last P.V at R+n
        const int rk = 2 * (R + n) + slot;
        if (buf == 0) r0 = rk; else if (buf == 1) r1 = rk; else r2 = rk;
        const int fk = 2 * (R + n + 1) + slot;
        if (slot) { fin1 = fk; rend1 = R + n; cur1 = i; } else { fin0 = fk; rend0 = R + n; cur0 = i; }
        sm->meta[i] = (uint8_t)(slot | (buf << 1) | (((uses >> buf) & 1u) << 3));
        uses ^= 1u << buf;
        ++k;
      }
      if (cur0 >= 0 && cur1 >= 0) {
        sm->eord[e++] = (uint8_t)(fin0 < fin1 ? cur0 : cur1);
        sm->eord[e++] = (uint8_t)(fin0 < fin1 ? cur1 : cur0);
      } else if (cur0 >= 0) {
        sm->eord[e++] = (uint8_t)cur0;
      }
      sm->uses = (int)uses;
      sm->T = T;
      sm->Tn = k;
    }
    __syncthreads();
    const int Tn = sm->Tn;

    if (warp >= WARP_EPI) {
      reg_dealloc<REG_EPILOGUE>();
      // -------------------------------------------------------------- epilogue warpgroup
      const int quarter = warp & 3;
      const int row = quarter * 32 + lane;
      const uint32_t t_row = tmem + (uint32_t(quarter * 32) << 16);
#if SV_O_EVICT_FIRST
      const uint64_t o_pol = policy_evict_first();   // O is written once: keep K/V in L2
#endif
      for (int e = 0; e < Tn; ++e) {
        const int i = sm->eord[e];
        const int t = sm->meta[i] & 1;
        const int it = item_at(b0 + i);
        const int bh = it / n_tiles, tile = it % n_tiles;
        const uint32_t par = (t ? tiles1 : tiles0) & 1;
        if (t) ++tiles1; else ++tiles0;
        mbar_wait(st_bar + t, par);
        const float2 stt = sm->stats[t][row];
        mbar_arrive(st_free + t);
        const long long te0_ = SV_CLK();
        mbar_wait(o_bar + t, par);
        if ((threadIdx.x & 127) == 0) SV_ACC(5400, SV_CLK() - te0_)
        tc_fence_after();
        const int n_row = tile * BM + row;
        const bool store = n_row < a.n_q;
        uint16_t* orow = a.o + (long long)bh * a.o_stride + (long long)n_row * D;
        const uint16_t* arow = cache_row<D>(a, bh, n_row);
#pragma unroll 1
        for (int c = 0; c < D; c += 16) {
          uint32_t o[16];
          tmem_ld16(t_row + 256 + t * D + c, o);
          tmem_wait_ld();
          if (c + 16 == D) {
            tc_fence_before();
            mbar_arrive(o_free + t);      // O of this slot may be overwritten now
          }
          float add[16];
          load_cache16(arow != nullptr && store ? arow + c : nullptr, add);
          uint32_t pk[8];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            pk[q] = pack_bf16x2(fmaf(__uint_as_float(o[2 * q]), stt.x, add[2 * q]),
                                fmaf(__uint_as_float(o[2 * q + 1]), stt.x, add[2 * q + 1]));
          if (store) {
#if SV_O_EVICT_FIRST
            st_global_v4_hint(orow + c, pk, o_pol);
            st_global_v4_hint(orow + c + 8, pk + 4, o_pol);
#else
            uint4* dst = reinterpret_cast<uint4*>(orow + c);
            dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
#endif
          }
        }
        if (a.lse != nullptr && store) a.lse[(long long)bh * a.n_q + n_row] = stt.y;
      }
    } else if (warp >= 8) {
      reg_dealloc<REG_PRODUCER>();
      if (warp == WARP_KV) {
        // -------------------------------------------------------------- KV loader
        if (lane == 0) {
          const uint64_t pol = policy_evict_last();
          int icur[2] = {-1, -1}, jn[2] = {0, 0}, nn[2] = {0, 0}, vcur[2] = {0, 0}, bhs[2] = {0, 0};
          Steps<G> st[2];
          auto load = [&](const CUtensorMap* m, int v, int bh) {
            const int s = kv_idx % C::NST;
            const uint32_t ph = (kv_idx / C::NST) & 1;
            ++kv_idx;
            {
              const long long t0_ = SV_CLK();
              mbar_wait(kv_empty + s, ph ^ 1);
              SV_ACC(5000, SV_CLK() - t0_)
#ifdef SV_PROF
              if (blockIdx.x == 0 && kv_idx <= 2000) {
                sv_prof_buf[16384 + 2 * (kv_idx - 1)] = t0_;
                sv_prof_buf[16384 + 2 * (kv_idx - 1) + 1] = clock64();
              }
#endif
            }
            uint8_t* dst = sKV + s * C::STAGE_BYTES;
            mbar_arrive_expect_tx(kv_full + s, C::STAGE_BYTES);
#pragma unroll
            for (int b = 0; b < C::NBOX; ++b)
              tma_load_3d_hint(dst + b * (BLK * 128), m, kv_full + s, b * 64, v * BLK, bh, pol);
          };
          auto start = [&](int t, int from) {
            int i = from;
            while (i < T && (sm->meta[i] == EMPTY_TILE || (sm->meta[i] & 1) != t)) ++i;
            icur[t] = i < T ? i : -1;
            if (icur[t] < 0) return;
            const int it = item_at(b0 + i);
            bhs[t] = it / n_tiles;
            st[t].init(a, bhs[t], it % n_tiles, g_kv);
            nn[t] = sm->n[i];
            jn[t] = 0;
            uint32_t gm;
            st[t].next(a, vcur[t], gm);
            load(&tmap_k, vcur[t], bhs[t]);
          };
          start(0, 0);
          start(1, 0);
          while (icur[0] >= 0 || icur[1] >= 0) {
            for (int t = 0; t < 2; ++t) {
              if (icur[t] < 0) continue;
              load(&tmap_v, vcur[t], bhs[t]);
              if (++jn[t] < nn[t]) {
                uint32_t gm;
                st[t].next(a, vcur[t], gm);
                load(&tmap_k, vcur[t], bhs[t]);
              } else {
                start(t, icur[t] + 1);
              }
            }
          }
        }
      } else if (warp == WARP_Q) {
        // -------------------------------------------------------------- Q loader (start order)
        if (lane == 0) {
          for (int i = 0; i < T; ++i) {
            const int meta = sm->meta[i];
            if (meta == EMPTY_TILE) continue;
            const int buf = (meta >> 1) & 3;
            const uint32_t use_par = (meta >> 3) & 1;
            if (q_used & (1u << buf)) mbar_wait(q_empty + buf, use_par ^ 1);
            q_used |= 1u << buf;
            const int it = item_at(b0 + i);
            uint8_t* dst = sQ + buf * C::Q_BYTES;
            mbar_arrive_expect_tx(q_full + buf, C::Q_BYTES);
#pragma unroll
            for (int b = 0; b < C::NBOX; ++b)
#if SV_Q_EVICT_FIRST
              tma_load_3d_hint(dst + b * (BM * 128), &tmap_q, q_full + buf, b * 64,
                               (it % n_tiles) * BM, it / n_tiles, policy_evict_first());
#else
              tma_load_3d(dst + b * (BM * 128), &tmap_q, q_full + buf, b * 64,
                          (it % n_tiles) * BM, it / n_tiles);
#endif
          }
        }
      } else if (warp == WARP_ZERO) {
        // -------------------------------------------------------------- empty tiles
        // no listed block in any of the tile's query blocks: zero output, lse = -inf
        for (int i = 0; i < T; ++i) {
          if (sm->meta[i] != EMPTY_TILE) continue;
          const int it = item_at(b0 + i);
          const int bh = it / n_tiles, tile = it % n_tiles;
          for (int r = lane; r < BM; r += 32) {
            const int row = tile * BM + r;
            if (row >= a.n_q) continue;
            uint4* dst =
                reinterpret_cast<uint4*>(a.o + (long long)bh * a.o_stride + (long long)row * D);
            // empty sparse part: the output is the (upsampled) cache residual, if any
            const uint16_t* arow = cache_row<D>(a, bh, row);
            for (int c = 0; c < D / 8; ++c)
              dst[c] = arow != nullptr ? reinterpret_cast<const uint4*>(arow)[c] : make_uint4(0, 0, 0, 0);
            if (a.lse != nullptr) a.lse[(long long)bh * a.n_q + row] = -INFINITY;
          }
        }
      } else if (warp == WARP_MMA) {
        // -------------------------------------------------------------- tcgen05 issuer
        // The whole warp runs the control flow so descriptors stay warp-uniform (uniform
        // registers); one elected lane issues each tcgen05 instruction.
#if SV_MMA_SHADOW
        // The persistent role state is live across every role's branch, so ptxas keeps it on
        // the stack (the kernel is compiled at 128 registers; setmaxnreg does not change that)
        // and the issuer paid an LDL/STL per op.  Shadow copies scoped to this branch stay in
        // registers; they are written back once per schedule batch.
        // (Plain shadow copies are folded away in SSA form: the state is kept in shared memory
        // between batches instead, so it is not live across the other roles' branches at all.)
        {
        int kv_idx = sm->mma_st[0], tiles0 = sm->mma_st[1], tiles1 = sm->mma_st[2];
        uint32_t p_cnt0 = (uint32_t)sm->mma_st[3], p_cnt1 = (uint32_t)sm->mma_st[4];
#endif
        constexpr uint32_t IDESC_QK = idesc_bf16_f32(BM, BLK, 0, 0);
        constexpr uint32_t IDESC_PV = idesc_bf16_f32(BM, D, 0, 1);
        constexpr int KH = BLK >= 64 ? BLK / 32 : BLK / 16;  // P.V K-steps of the first P half
        const bool leader = elect_one();
        const uint64_t dq0 = sdesc_sw128(smem_u32(sQ), 16, 1024);
        const uint64_t dk0 = sdesc_sw128(smem_u32(sKV), 16, 1024);
        const uint64_t dv0 = sdesc_sw128(smem_u32(sKV), BLK * 128, 1024);
        int icur0 = -1, icur1 = -1, jn0 = 0, jn1 = 0, nn0 = 0, nn1 = 0, qb0 = 0, qb1 = 0;
        // ring position as (stage, phase) counters: no div/mod on the issue path
        int ring_s = kv_idx % C::NST;
        uint32_t ring_ph = (kv_idx / C::NST) & 1;
        auto next_stage = [&]() -> uint32_t {
          const int s = ring_s;
          SV_MMA_WAIT_T(kv_full + s, ring_ph, 6000);
#ifdef SV_PROF
          if (blockIdx.x == 0 && lane == 0 && kv_idx < 2000) sv_prof_buf[20480 + kv_idx] = clock64();
#endif
          if (++ring_s == C::NST) { ring_s = 0; ring_ph ^= 1; }
          ++kv_idx;
          return (uint32_t)s;
        };
        auto issue_qk = [&](int t, uint32_t s, int qb, bool last) {
          const uint64_t da = dq0 + ((uint64_t)(qb * C::Q_BYTES) >> 4);
          const uint64_t db = dk0 + ((uint64_t)(s * C::STAGE_BYTES) >> 4);
          if (leader) {
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint32_t oa = ((kk >> 2) * (BM * 128) + (kk & 3) * 32) >> 4;
              const uint32_t ob = ((kk >> 2) * (BLK * 128) + (kk & 3) * 32) >> 4;
              mma_ss(tmem + t * 128, da + oa, db + ob, IDESC_QK, kk > 0);
            }
            mma_commit(kv_empty + s);
            mma_commit(s_bar + t);
            if (last) mma_commit(q_empty + qb);   // last use of this Q buffer
          }
#if !SV_LEAN
          __syncwarp();
#endif
        };
        auto start = [&](int t, int from) {
          int i = from;
          while (i < T && (sm->meta[i] == EMPTY_TILE || (sm->meta[i] & 1) != t)) ++i;
          const int ic = i < T ? i : -1;
          if (t) icur1 = ic; else icur0 = ic;
          if (ic < 0) return;
          const int meta = sm->meta[ic];
          const int qb = (meta >> 1) & 3;
          const int n = sm->n[ic];
          if (t) { qb1 = qb; nn1 = n; jn1 = 0; } else { qb0 = qb; nn0 = n; jn0 = 0; }
#ifdef SV_PROF
          const int st_ = tiles0 + tiles1;
          if (blockIdx.x == 0 && lane == 0 && st_ < 500) sv_prof_buf[22528 + 4 * st_] = clock64();
#endif
          const uint32_t s = next_stage();
#ifdef SV_PROF
          if (blockIdx.x == 0 && lane == 0 && st_ < 500) sv_prof_buf[22528 + 4 * st_ + 1] = clock64();
#endif
          SV_MMA_WAIT_T(q_full + qb, (meta >> 3) & 1, 6600);
#ifdef SV_PROF
          if (blockIdx.x == 0 && lane == 0 && st_ < 500) sv_prof_buf[22528 + 4 * st_ + 2] = clock64();
#endif
          tc_fence_after();
          issue_qk(t, s, qb, n == 1);
#ifdef SV_PROF
          if (blockIdx.x == 0 && lane == 0 && st_ < 500) sv_prof_buf[22528 + 4 * st_ + 3] = clock64();
#endif
        };
        const long long tm0_ = SV_CLK();
        start(0, 0);
        start(1, 0);
        while (icur0 >= 0 || icur1 >= 0) {
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const int icur = t ? icur1 : icur0;
            if (icur < 0) continue;
            const int jn = t ? jn1 : jn0, nn = t ? nn1 : nn0, qb = t ? qb1 : qb0;
            const int tdone = t ? tiles1 : tiles0;
            // the stages this op reads are (normally) resident already: check them before P
#ifdef SV_PROF
            SV_OPSTAMP((int)(p_cnt0 + p_cnt1), 4)
#endif
            const uint32_t sv = next_stage();
#ifdef SV_PROF
            SV_OPSTAMP((int)(p_cnt0 + p_cnt1), 5)
#endif
            const bool more = jn + 1 < nn;
            const uint32_t sk = more ? next_stage() : 0u;
#ifdef SV_PROF
            SV_OPSTAMP((int)(p_cnt0 + p_cnt1), 6)
#endif
            const uint32_t par = (t ? p_cnt1 : p_cnt0) & 1;
            if (t) ++p_cnt1; else ++p_cnt0;
            if (lane == 0) SV_ACC(7000, 1)
            const uint64_t dv = dv0 + ((uint64_t)(sv * C::STAGE_BYTES) >> 4);
            const uint32_t o_tmem = tmem + 256 + t * D;
            const uint32_t p_tmem = tmem + t * 128;
            // the tile's first P.V overwrites O: the epilogue must have drained the previous one
            if (jn == 0 && tdone > 0) SV_MMA_WAIT_T(o_free + t, (tdone - 1) & 1, 6400);
#ifdef SV_PROF
            const int op_ = (int)(p_cnt0 + p_cnt1) - 1;
            SV_OPSTAMP(op_, 0)
#endif
#if SV_LEAN
            // O_t += P_t V_j: every softmax thread arrives on the first-half barrier before the
            // second, so waiting on the second covers all of P (one wait + fence per op: the
            // issue queue is shallow, every instruction here is tensor-pipe idle time)
            SV_MMA_WAIT_T(p_bar + 2 * t + 1, par, 6200);
#ifdef SV_PROF
            SV_OPSTAMP(op_, 1)
#endif
            tc_fence_after();
            if (leader) {
#pragma unroll
              for (int kk = 0; kk < BLK / 16; ++kk)
                mma_ts(o_tmem, p_tmem + kk * 8, dv + ((uint32_t)(kk * 2048) >> 4), IDESC_PV,
                       (jn > 0 || kk > 0) ? 1u : 0u);
              mma_commit(kv_empty + sv);
            }
#ifdef SV_PROF
            SV_OPSTAMP(op_, 2)
#endif
#else
            // O_t += P_t V_j in two halves: the first as soon as half of P is in TMEM
            SV_MMA_WAIT(p_bar + 2 * t, par);
            tc_fence_after();
            if (leader) {
#pragma unroll
              for (int kk = 0; kk < KH; ++kk)
                mma_ts(o_tmem, p_tmem + kk * 8, dv + ((uint32_t)(kk * 2048) >> 4), IDESC_PV,
                       (jn > 0 || kk > 0) ? 1u : 0u);
            }
            __syncwarp();
            SV_MMA_WAIT(p_bar + 2 * t + 1, par);
            tc_fence_after();
            if (leader) {
#pragma unroll
              for (int kk = KH; kk < BLK / 16; ++kk)
                mma_ts(o_tmem, p_tmem + kk * 8, dv + ((uint32_t)(kk * 2048) >> 4), IDESC_PV, 1u);
              mma_commit(kv_empty + sv);
            }
            __syncwarp();
#endif
            if (more) {
              if (t) ++jn1; else ++jn0;
              issue_qk(t, sk, qb, jn + 2 == nn);
#ifdef SV_PROF
              SV_OPSTAMP(op_, 3)
#endif
            } else {
              if (leader) mma_commit(o_bar + t);
              __syncwarp();
              if (t) ++tiles1; else ++tiles0;
              start(t, icur + 1);
            }
          }
        }
        if (lane == 0) SV_ACC(6800, SV_CLK() - tm0_)
#if SV_MMA_SHADOW
        __syncwarp();
        if (lane == 0) {
          sm->mma_st[0] = kv_idx; sm->mma_st[1] = tiles0; sm->mma_st[2] = tiles1;
          sm->mma_st[3] = (int)p_cnt0; sm->mma_st[4] = (int)p_cnt1;
        }
        __syncwarp();
        }
#endif
      }
    } else {
      // ---------------------------------------------------------------- softmax warpgroups
      reg_alloc<REG_SOFTMAX>();
      const int t = warp >> 2;                 // slot
#if SV_SFX_SHADOW
      // as for the issuer: this warpgroup's loop-carried counters live in shared memory between
      // batches (one copy per slot), not across the other roles' branches
      {
      uint32_t s_cnt = (uint32_t)sm->sfx_st[t][0];
      int tiles0 = sm->sfx_st[t][1], tiles1 = sm->sfx_st[t][1];
#endif
      const int quarter = warp & 3;
      const int row = quarter * 32 + lane;
      const uint32_t t_row = tmem + (uint32_t(quarter * 32) << 16);
      const uint32_t s_col = t * 128;
      const uint32_t o_col = 256 + t * D;
      const int grp = row / BLK;
      const float sl2 = a.scale_log2;
      const uint64_t sl2x2 = f2_pack(sl2, sl2);
      for (int i = 0; i < T; ++i) {
        const int meta = sm->meta[i];
        if (meta == EMPTY_TILE || (meta & 1) != t) continue;
        const int it = item_at(b0 + i);
        Steps<G> st;
        st.init(a, it / n_tiles, it % n_tiles, g_kv);
        const int mass_row = (it % n_tiles) * BM + row;                    // MASS only
        const long long mass_base = (long long)(it / n_tiles) * g_kv * a.n_q + mass_row;
        float m = -INFINITY;   // running max of s * scale * log2(e)
        float l = 0.f;         // running sum of exp2(s * sl2 - m)
        int v;
        uint32_t gm;
        bool have = st.next(a, v, gm);
        int j = 0;
        while (have) {
          SV_STAMP(5 * s_cnt + 0)
          const long long ts0_ = SV_CLK();
          mbar_wait(s_bar + t, s_cnt & 1);
          if ((threadIdx.x & 127) == 0) SV_ACC(5200, SV_CLK() - ts0_)
          SV_STAMP(5 * s_cnt + 1)
          ++s_cnt;
          tc_fence_after();
          uint32_t sr[BLK];
          // next step's block index: the load's latency hides under this step
          int v_n;
          uint32_t gm_n;
          bool have_n;
          const bool row_on = (gm >> grp) & 1u;
          const int valid = row_on ? min(BLK, a.n_kv - v * BLK) : 0;
          float mx;
          {
            float mm[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
            auto mask_and_max = [&](int c_lo, int c_hi) {
              // ragged last KV block / rows whose query block does not list this step
              // (warp-uniform branch, rarely taken)
              if (__builtin_expect(__any_sync(0xffffffffu, valid < c_hi), 0)) {
#pragma unroll
                for (int c = 0; c < BLK; ++c)
                  if (c >= c_lo && c < c_hi && c >= valid) sr[c] = __float_as_uint(-INFINITY);
              }
#pragma unroll
              for (int c = 0; c + 8 <= BLK; c += 8) {
                if (c < c_lo || c >= c_hi) continue;
                const int q = (c >> 3) & 3;
                mm[q] = fmax3(mm[q], __uint_as_float(sr[c]), __uint_as_float(sr[c + 1]));
                mm[q] = fmax3(mm[q], __uint_as_float(sr[c + 2]), __uint_as_float(sr[c + 3]));
                mm[q] = fmax3(mm[q], __uint_as_float(sr[c + 4]), __uint_as_float(sr[c + 5]));
                mm[q] = fmax3(mm[q], __uint_as_float(sr[c + 6]), __uint_as_float(sr[c + 7]));
              }
            };
            if constexpr (BLK >= 64) {
              // one batch of TMEM loads for the whole step's S and one wait (two half batches
              // with the first half's max between them paid two load latencies: 1-3% slower)
#pragma unroll
              for (int c = 0; c < BLK; c += 32) tmem_ld32(t_row + s_col + c, sr + c);
              have_n = st.next(a, v_n, gm_n);
              tmem_wait_ld();
              mask_and_max(0, BLK);
            } else {
              if constexpr (BLK == 32) {
                tmem_ld32(t_row + s_col, sr);
              } else {
#pragma unroll
                for (int c = 0; c < BLK; c += 8) tmem_ld8(t_row + s_col + c, sr + c);
              }
              have_n = st.next(a, v_n, gm_n);
              tmem_wait_ld();
              mask_and_max(0, BLK);
            }
            mx = fmax3(fmaxf(mm[0], mm[1]), mm[2], mm[3]);
          }
          SV_STAMP(5 * (s_cnt - 1) + 2)
          const float mx_s = mx * sl2;
          const bool need = mx_s > m + 8.0f;
          float alpha = 1.f;
          if (need) {
            alpha = ex2(m - mx_s);
            m = mx_s;
            l *= alpha;
          }
          // lazy rescale of O (rare): P_{j-1} V_{j-1} is complete (covered by the S_j commit) and
          // P_j V_j is not issued before this thread arrives on p_bar
          if (j > 0 && __any_sync(0xffffffffu, need)) {
#pragma unroll 1
            for (int c = 0; c < D; c += 32) {
              uint32_t o[32];
              tmem_ld32(t_row + o_col + c, o);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
              tmem_st32(t_row + o_col + c, o);
            }
          }
          const float mref = (m == -INFINITY) ? 0.f : m;
          const uint64_t negm = f2_pack(-mref, -mref);
          uint64_t acc[4] = {0, 0, 0, 0};
          constexpr int CH = BLK < 32 ? BLK : 32;
#pragma unroll
          for (int c0 = 0; c0 < BLK; c0 += CH) {
            uint32_t p[CH / 2];
#pragma unroll
            for (int c = 0; c < CH; c += 2) {
              const uint64_t x = ffma2(f2_pack(__uint_as_float(sr[c0 + c]), __uint_as_float(sr[c0 + c + 1])),
                                       sl2x2, negm);
              float p0, p1;
              if (EMU_EVERY > 0 && ((c0 + c) / 2) % (EMU_EVERY > 0 ? EMU_EVERY : 1) == EMU_EVERY - 1) {
                ex2_emu2<3>(x, p0, p1);
              } else {
                float x0, x1;
                f2_unpack(x, x0, x1);
                p0 = ex2(x0);
                p1 = ex2(x1);
              }
              acc[(c >> 1) & 3] = fadd2(acc[(c >> 1) & 3], f2_pack(p0, p1));
              p[c / 2] = pack_bf16x2(p0, p1);
            }
            // P chunk c0 lands in columns [c0/2, c0/2 + CH/2) of S, all already read
            if constexpr (CH == 32) {
              tmem_st16(t_row + s_col + c0 / 2, p);
            } else {
#pragma unroll
              for (int c = 0; c < CH / 2; c += 8) tmem_st8(t_row + s_col + c0 / 2 + c, p + c);
            }
#if !SV_LEAN
            if (BLK >= 64 && c0 + CH == BLK / 2) {
              // first half of P is in TMEM: let the MMA warp start P.V on it
              tmem_wait_st();
              tc_fence_before();
              mbar_arrive(p_bar + 2 * t);
            }
#endif
          }
          {
            SV_STAMP(5 * (s_cnt - 1) + 3)
            const uint64_t s2 = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
            float s0, s1;
            f2_unpack(s2, s0, s1);
            l += s0 + s1;
            if constexpr (MASS) {
              if (mass_row < a.n_q) {
                const long long off = mass_base + (long long)v * a.n_q;
                a.mass_s[off] = s0 + s1;
                a.mass_m[off] = mref;
              }
            }
          }
          tmem_wait_st();
          tc_fence_before();
#if !SV_LEAN
          if (BLK < 64) mbar_arrive(p_bar + 2 * t);
#endif
          mbar_arrive(p_bar + 2 * t + 1);   // the lean issuer waits on this one only
          SV_STAMP(5 * (s_cnt - 1) + 4)
          ++j;
          v = v_n;
          gm = gm_n;
          have = have_n;
        }
        // hand the row statistics to the epilogue warpgroup
        const int tdone = t ? tiles1 : tiles0;
        if (tdone > 0) mbar_wait(st_free + t, (tdone - 1) & 1);
        if (t) ++tiles1; else ++tiles0;
        const bool live = m != -INFINITY;      // the row saw at least one valid logit
        sm->stats[t][row] = make_float2(live ? 1.f / l : 0.f,
                                        live ? (m * 0.69314718055994531f + logf(l)) : -INFINITY);
        mbar_arrive(st_bar + t);
      }
#if SV_SFX_SHADOW
      if ((threadIdx.x & 127) == 0) {        // read back only after the batch's __syncthreads
        sm->sfx_st[t][0] = (int)s_cnt;
        sm->sfx_st[t][1] = t ? tiles1 : tiles0;
      }
      }
#endif
      reg_dealloc<REG_LAUNCH>();
    }
    __syncthreads();
    // WG2/WG3 take their registers back only once every softmax warp has returned its share:
    // a producer that finished early and re-grew inside its branch could starve a softmax warp
    // that had not grown yet (setmaxnreg.inc blocks until the CTA pool has the registers).
    if (warp >= WARP_MMA) reg_alloc<REG_LAUNCH>();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == WARP_MMA) {
    tc_fence_after();
    tmem_dealloc(tmem, TMEM_COLS);
  }
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}

template <int D, int BLK, bool MASS = false>
cudaError_t launch_t(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                     const AttnArgs& a, cudaStream_t st) {
  using C = Cfg<D, BLK>;
  auto kern = attn_fwd_kernel<D, BLK, MASS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  if (e != cudaSuccess) return e;
  const int n_tiles = (a.n_q + BM - 1) / BM;
  const long long items = (long long)n_tiles * a.bh;
  if (items <= 0) return cudaSuccess;
  if (items > (1LL << 30)) return cudaErrorInvalidValue;
  const int sms = num_sms();
  // two tile slots per CTA: fewer CTAs than SMs when there is little work
  const int grid = (int)(items >= 2LL * sms ? sms : (items + 1) / 2);
  kern<<<grid, NUM_THREADS, C::SMEM, st>>>(tq, tk, tv, a, 0, (int)items);
  return cudaGetLastError();
}

// o_cache = o_dense - o_sparse (NEXT(1)): bf16 in, fp32 difference, bf16 out;
// 8 elements (16 B) per thread per iteration, grid-stride over all (b,h) rows.
__global__ void __launch_bounds__(256) residual_kernel(int bh, int rows, int D, const uint16_t* dense,
                                                       long long ds, const uint16_t* sparse,
                                                       long long ss, uint16_t* out, long long os) {
  const long long per_bh = (long long)rows * D / 8;
  const long long total = per_bh * bh;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long b = i / per_bh, e = (i % per_bh) * 8;
    const uint4 x = *reinterpret_cast<const uint4*>(dense + b * ds + e);
    const uint4 y = *reinterpret_cast<const uint4*>(sparse + b * ss + e);
    const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
    uint32_t r[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float lo = __uint_as_float(xs[k] << 16) - __uint_as_float(ys[k] << 16);
      const float hi = __uint_as_float(xs[k] & 0xffff0000u) - __uint_as_float(ys[k] & 0xffff0000u);
      r[k] = pack_bf16x2(lo, hi);
    }
    *reinterpret_cast<uint4*>(out + b * os + e) = make_uint4(r[0], r[1], r[2], r[3]);
  }
}

// NEXT(3): block masses from the MASS pass and the predictor's selection (same rules as
// predict_kernel: top-k by rank with ties to the smaller v, or mass >= tau |u|, then the sinks).
// One CTA per (b,h, query block u), thread r = row u*B + r:
//   mass[u, v] = sum_r s[v][q] * 2^(m[v][q] - lse[q] * log2 e)   (= sum_r sum_{j in v} P[q, j])
// reduced in a fixed order (warp shuffles, then the 4 warp partials in order): deterministic.
__global__ void __launch_bounds__(128) mass_select_kernel(int n_q, int g_q, int g_kv, int B,
                                                          const float* __restrict__ s,
                                                          const float* __restrict__ m,
                                                          const float* __restrict__ lse, int mode,
                                                          int topk, float tau, int n_sink_blocks,
                                                          float* mass_out, uint32_t* mask_out) {
  extern __shared__ float shm[];
  float* part = shm;                  // [4][g_kv]
  float* mass = shm + 4 * g_kv;       // [g_kv]
  const int bh = blockIdx.x / g_q, u = blockIdx.x % g_q;
  const int r = threadIdx.x, warp = r >> 5, lane = r & 31;
  const int q = u * B + r;
  const bool valid = r < B && q < n_q;
  const float L = valid ? lse[(long long)bh * n_q + q] * 1.4426950408889634f : 0.f;
  const long long base = (long long)bh * g_kv * n_q + q;
  for (int v = 0; v < g_kv; ++v) {
    float w = 0.f;
    if (valid) {
      const long long off = base + (long long)v * n_q;
      w = s[off] * exp2f(m[off] - L);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    if (lane == 0) part[warp * g_kv + v] = w;
  }
  __syncthreads();
  for (int v = r; v < g_kv; v += blockDim.x)
    mass[v] = ((part[v] + part[g_kv + v]) + part[2 * g_kv + v]) + part[3 * g_kv + v];
  __syncthreads();
  if (warp != 0) return;
  const long long row = (long long)bh * g_q + u;
  const int W = (g_kv + 31) / 32;
  const int rows_u = min(B, n_q - u * B);
  const float thr = tau * float(rows_u);
  for (int w0 = 0; w0 < W; ++w0) {
    const int v = w0 * 32 + lane;
    bool sel = false;
    if (v < g_kv) {
      const float mv = mass[v];
      if (mode == 0) {
        int rank = 0;
        for (int t = 0; t < g_kv; ++t) {
          const float mt = mass[t];
          rank += (mt > mv) || (mt == mv && t < v);
        }
        sel = rank < topk;
      } else {
        sel = mv >= thr;
      }
      sel = sel || (v < n_sink_blocks);
      if (mass_out != nullptr) mass_out[row * g_kv + v] = mv;
    }
    const uint32_t word = __ballot_sync(0xffffffffu, sel);
    if (lane == 0) mask_out[row * W + w0] = word;
  }
}

}  // namespace

cudaError_t launch_mass_select(int bh, int n_q, int g_q, int g_kv, int B, const float* s,
                               const float* m, const float* lse, int mode, int topk, float tau,
                               int n_sink_blocks, float* mass_out, uint32_t* mask_out,
                               cudaStream_t st) {
  const size_t shmem = size_t(5) * g_kv * sizeof(float);
  if (shmem > 48 * 1024) return cudaErrorInvalidValue;
  if ((long long)bh * g_q <= 0) return cudaSuccess;
  mass_select_kernel<<<bh * g_q, 128, shmem, st>>>(n_q, g_q, g_kv, B, s, m, lse, mode, topk, tau,
                                                   n_sink_blocks, mass_out, mask_out);
  return cudaGetLastError();
}

cudaError_t launch_residual(int bh, int rows, int D, const uint16_t* dense, long long dense_stride,
                            const uint16_t* sparse, long long sparse_stride, uint16_t* out,
                            long long out_stride, cudaStream_t st) {
  const long long vec = (long long)bh * rows * D / 8;
  if (vec <= 0) return cudaSuccess;
  const int grid = (int)((vec + 255) / 256 < 4L * num_sms() ? (vec + 255) / 256 : 4L * num_sms());
  residual_kernel<<<grid, 256, 0, st>>>(bh, rows, D, dense, dense_stride, sparse, sparse_stride,
                                        out, out_stride);
  return cudaGetLastError();
}

cudaError_t launch_attention(int head_dim, int block, const CUtensorMap& tq, const CUtensorMap& tk,
                             const CUtensorMap& tv, const AttnArgs& a, cudaStream_t st) {
#define SV_CASE(D_, B_)                                                   \
  if (head_dim == D_ && block == B_)                                      \
    return a.mass_s != nullptr ? launch_t<D_, B_, true>(tq, tk, tv, a, st) \
                               : launch_t<D_, B_>(tq, tk, tv, a, st);
  SV_CASE(128, 128) SV_CASE(128, 64) SV_CASE(128, 32) SV_CASE(128, 16)
  SV_CASE(64, 128) SV_CASE(64, 64) SV_CASE(64, 32) SV_CASE(64, 16)
#undef SV_CASE
  return cudaErrorInvalidValue;
}

}  // namespace sv
