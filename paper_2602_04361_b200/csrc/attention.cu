// attention.cu — block-sparse (and dense) cross-scale attention forward for sm_100a.
//
// Computes, for every (b,h) and query block u, o_t = softmax_J(q_t . k_j * scale) V_J over the
// real tokens J of the KV blocks listed for u (PAPER.md:204-212 Eq. attn_cross_scale,
// PAPER.md:318-328 Eq. sparse_update, PAPER.md:397-407 Eq. block_mask; READINGS 9, 17, 20).
//
// Design (DESIGN.md §7 "attn_fwd_kernel v1"):
//  * Persistent: one CTA per SM (512 TMEM columns), CTA c walks the 128-row query tiles
//    ("items", (b,h)-major) c, c+grid, ...  Two tile SLOTS run concurrently in a CTA, each with
//    its own S/P (128 TMEM cols) and O (D cols) accumulators and its own softmax warpgroup, so
//    the tensor core works on one slot while the other slot's softmax runs (ping-pong).
//  * The MMA warp issues in a fixed round-robin order: per round and slot, O += P_j V_j then
//    S = Q K_{j+1}^T (or the next tile's first S).  Every role (KV loader, Q loader, MMA, softmax)
//    derives the same order from a per-CTA schedule built once in shared memory, so a single KV
//    ring (TMA, mbarrier full/empty) serves both slots and no role needs to talk to another
//    except through the ring / tile barriers.
//  * Q lives in 3 shared buffers: two slots' current tiles plus one prefetched tile.  A buffer is
//    released by the commit of its tile's last Q K^T, and the schedule assigns each new tile the
//    earliest pending release (deadlock-free: that release precedes the tile's start in the MMA
//    order).
//  * S (fp32) and O (fp32) live in TMEM; P (bf16) overwrites S in place and is the TMEM A operand
//    of the P.V MMA (tcgen05 ops of one thread execute in issue order, so the next S = Q K^T issued
//    after P.V cannot clobber P early).  Online softmax in fp32, exp2 domain, with a lazy rescale
//    of O (only when the running max grows by more than 2^8).  The commit that signals S_j also
//    covers P_{j-1} V_{j-1}, so a rescale of O never races the tensor core.
//  * Block sizes below 128: a 128-row tile holds G = 128/B query blocks; the KV steps are the
//    ascending union of their lists and each row masks the steps its own block does not list, so
//    every row sees exactly its own list.  The ragged last KV block is masked to -inf
//    (READING 20): TMA zero fill alone would give logit 0.
#include <cuda_bf16.h>
#include <cstdio>

#include "kernels.h"
#include "ptx.cuh"

#ifdef SV_PROF
// Development instrumentation (built only into variant libraries, scripts/build_variant.sh):
// globaltimer-free SM clock stamps of the softmax phases of CTA 0 / slot 0 / row 0.
__device__ long long sv_prof_buf[8192];
extern "C" int sparvar_prof_read(long long* host, int n) {
  return cudaMemcpyFromSymbol(host, sv_prof_buf, sizeof(long long) * n) == cudaSuccess ? 0 : 1;
}
#define SV_STAMP(slot_, i_) \
  if (blockIdx.x == 0 && threadIdx.x == 0 && (i_) < 8192) sv_prof_buf[(i_)] = clock64();
#define SV_STAMP_MMA(i_) \
  if (blockIdx.x == 0 && (i_) < 4096) sv_prof_buf[4096 + (i_)] = clock64();
#else
#define SV_STAMP(slot_, i_)
#define SV_STAMP_MMA(i_)
#endif

namespace sv {
namespace {

constexpr int BM = 128;                  // query rows per tile (TMEM lanes)
constexpr int NUM_WARPS = 12;            // WG0 softmax slot 0, WG1 softmax slot 1, WG2: MMA, KV, Q, idle
constexpr int NUM_THREADS = NUM_WARPS * 32;
constexpr int WARP_MMA = 8, WARP_KV = 9, WARP_Q = 10;
// setmaxnreg moves registers inside the CTA's own pool (launch: 12 warps x 168): the 8 softmax warps
// take 8 x 56 more, the 4 other warps give 4 x 112 back.
constexpr int REG_LAUNCH = 168;
constexpr int REG_SOFTMAX = 224;
constexpr int REG_OTHER = 56;
static_assert(8 * (REG_SOFTMAX - REG_LAUNCH) <= 4 * (REG_LAUNCH - REG_OTHER), "register pool");
#ifndef SV_EMU_EVERY
#define SV_EMU_EVERY 4
#endif
constexpr int EMU_EVERY = SV_EMU_EVERY;  // 1 in EMU_EVERY exp2 pairs on the FMA pipe (0 = none)
constexpr uint32_t TMEM_COLS = 512;
constexpr int NQB = 3;                   // Q buffers
constexpr int MAX_TILES = 128;           // tiles per CTA per launch (the host splits bigger jobs)
constexpr int SMEM_LIMIT = 232448;       // 227 KB opt-in
constexpr int SMEM_SMALL = 1600;         // schedule + barriers
constexpr int SMEM_SLACK = 1024;         // alignment of the dynamic smem base to 1024

template <int D, int BLK>
struct Cfg {
  static constexpr int NBOX = D / 64;                       // 64-element (128 B) TMA boxes per row
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int STAGE_BYTES = BLK * D * 2;
  static constexpr int AVAIL = SMEM_LIMIT - SMEM_SMALL - SMEM_SLACK - NQB * Q_BYTES;
  static constexpr int NST = AVAIL / STAGE_BYTES > 8 ? 8 : AVAIL / STAGE_BYTES;
  static constexpr int G = BM / BLK;                        // query blocks per tile
  static constexpr int SMEM = SMEM_SLACK + NQB * Q_BYTES + NST * STAGE_BYTES + SMEM_SMALL;
  static_assert(NST >= 2, "KV ring too small");
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

// Per-CTA schedule in shared memory.  ord[k] (k = start order) indexes the CTA's non-empty tiles;
// meta[k] = slot | buf << 1 | (use parity of buf) << 3.
struct Sched {
  int item[MAX_TILES];     // global item id of the CTA's i-th tile (CTA order)
  int n[MAX_TILES];        // KV steps of that tile
  uint8_t ord[MAX_TILES];  // start order -> CTA-order index
  uint8_t meta[MAX_TILES];
  int T;                   // tiles of this CTA
  int Tn;                  // non-empty tiles
};
static_assert(((sizeof(Sched) + 15) & ~15ull) + 8 * (2 * NQB + 2 * 8 + 6) + 16 <= SMEM_SMALL,
              "schedule + barriers exceed SMEM_SMALL");

__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t r, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(r));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

template <int N>
__device__ __forceinline__ void reg_alloc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void reg_dealloc() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}

// 2^x for a pair on the FMA/ALU pipes (offloads MUFU): x = n + f, n = rint(x) via the 1.5*2^23
// magic add, f in [-1/2, 1/2], 2^f by a degree-3 polynomial (max rel. error 7.5e-5, far below
// the bf16 rounding P gets), 2^n added to the exponent field.  x is clamped at -126 so masked
// (-inf) logits give 2^-126 instead of 0: negligible against l >= 1, and rows that never see a
// valid logit are zeroed by the epilogue (m stays -inf).
__device__ __forceinline__ void ex2_emu2(uint64_t x2, float& p0, float& p1) {
  constexpr float MAGIC = 12582912.0f;   // 1.5 * 2^23
  float x0, x1;
  f2_unpack(x2, x0, x1);
  x0 = fmaxf(x0, -126.f);
  x1 = fmaxf(x1, -126.f);
  const uint64_t xc = f2_pack(x0, x1);
  const uint64_t t = fadd2(xc, f2_pack(MAGIC, MAGIC));
  const uint64_t r = fadd2(t, f2_pack(-MAGIC, -MAGIC));
  const uint64_t f = ffma2(r, f2_pack(-1.f, -1.f), xc);   // x - rint(x)
  uint64_t q = ffma2(f2_pack(0.05517166f, 0.05517166f), f, f2_pack(0.24261113f, 0.24261113f));
  q = ffma2(q, f, f2_pack(0.69326097f, 0.69326097f));
  q = ffma2(q, f, f2_pack(0.99992806f, 0.99992806f));
  float q0, q1, t0, t1;
  f2_unpack(q, q0, q1);
  f2_unpack(t, t0, t1);
  p0 = __int_as_float(__float_as_int(q0) + (__float_as_int(t0) << 23));
  p1 = __int_as_float(__float_as_int(q1) + (__float_as_int(t1) << 23));
}

template <int D, int BLK>
__global__ void __launch_bounds__(NUM_THREADS, 1)
attn_fwd_kernel(const __grid_constant__ CUtensorMap tmap_q,
                const __grid_constant__ CUtensorMap tmap_k,
                const __grid_constant__ CUtensorMap tmap_v, const AttnArgs a, int item_begin,
                int item_end) {
  using C = Cfg<D, BLK>;
  constexpr int G = C::G;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;                                       // NQB x Q_BYTES
  uint8_t* sKV = smem + NQB * C::Q_BYTES;                   // NST x STAGE_BYTES
  Sched* sch = reinterpret_cast<Sched*>(sKV + C::NST * C::STAGE_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sch) +
                                               ((sizeof(Sched) + 15) & ~size_t(15)));
  uint64_t* q_full = bars;                 // [NQB]
  uint64_t* q_empty = bars + NQB;          // [NQB]
  uint64_t* kv_full = bars + 2 * NQB;      // [NST]
  uint64_t* kv_empty = kv_full + C::NST;   // [NST]
  uint64_t* s_bar = kv_empty + C::NST;     // [2] S_j of slot ready (also covers P_{j-1}V_{j-1})
  uint64_t* p_bar = s_bar + 2;             // [2] P_j of slot written (128 arrivals)
  uint64_t* o_bar = p_bar + 2;             // [2] last P.V of a slot's tile complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int g_kv = (a.n_kv + BLK - 1) / BLK;
  const int n_tiles = (a.n_q + BM - 1) / BM;

  // ------------------------------------------------------------------ setup
  if (threadIdx.x == 0) {
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
      mbar_init(p_bar + t, BM);
      mbar_init(o_bar + t, 1);
    }
    fence_barrier_init();
  }
  if (warp == WARP_KV && lane == 0) {
    prefetch_tmap(&tmap_k);
    prefetch_tmap(&tmap_v);
  }
  if (warp == WARP_Q && lane == 0) prefetch_tmap(&tmap_q);
  if (warp == WARP_MMA) {
    tmem_alloc(tmem_slot, TMEM_COLS);
    tmem_relinquish();
  }
  // tile lengths, in parallel
  int T = 0;
  {
    const int first = item_begin + blockIdx.x;
    if (first < item_end) T = (item_end - first + gridDim.x - 1) / gridDim.x;
    for (int i = threadIdx.x; i < T; i += NUM_THREADS) {
      const int it = first + i * gridDim.x;
      Steps<G> st;
      st.init(a, it / n_tiles, it % n_tiles, g_kv);
      sch->item[i] = it;
      sch->n[i] = st.count(a);
    }
  }
  tc_fence_before();
  __syncthreads();
  // round-robin simulation of the MMA order -> slot, Q buffer and start order of every tile
  if (threadIdx.x == 0) {
    long long fin_key[2] = {0, 0};   // key of the op that finishes the slot's current tile
    int round_end[2] = {0, 0};       // round at which the slot's current tile finishes
    bool busy[2] = {false, false};
    int pend_key[NQB + 1], pend_buf[NQB + 1], npend = 0;
    int uses[NQB] = {0, 0, 0};
    int k = 0;
    for (int i = 0; i < T; ++i) {
      const int n = sch->n[i];
      if (n == 0) continue;
      int slot, R;
      if (k < 2) {
        slot = k;
        R = -1;
      } else {
        slot = (!busy[1] || (busy[0] && fin_key[0] < fin_key[1])) ? 0 : 1;
        R = round_end[slot];
      }
      int buf;
      if (k < NQB) {
        buf = k;
      } else {
        int best = 0;
        for (int p = 1; p < npend; ++p)
          if (pend_key[p] < pend_key[best]) best = p;
        buf = pend_buf[best];
        pend_key[best] = pend_key[npend - 1];
        pend_buf[best] = pend_buf[npend - 1];
        --npend;
      }
      // op (round r, slot s) has key 2*(r+1)+s; last Q K^T at round R+n-1, last P.V at R+n
      pend_key[npend] = 2 * (R + n) + slot;
      pend_buf[npend] = buf;
      ++npend;
      busy[slot] = true;
      round_end[slot] = R + n;
      fin_key[slot] = 2LL * (R + n + 1) + slot;
      sch->ord[k] = (uint8_t)i;
      sch->meta[k] = (uint8_t)(slot | (buf << 1) | ((uses[buf] & 1) << 3));
      ++uses[buf];
      ++k;
    }
    sch->T = T;
    sch->Tn = k;
  }
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int Tn = sch->Tn;

  if (warp >= 8) {
  reg_dealloc<REG_OTHER>();
  if (warp == WARP_KV) {
    // ---------------------------------------------------------------- KV loader
    if (lane == 0) {
      const uint64_t pol = policy_evict_last();
      int kcur[2] = {-1, -1};
      int jn[2] = {0, 0}, nn[2] = {0, 0}, vcur[2] = {0, 0}, bhs[2] = {0, 0};
      Steps<G> st[2];
      int idx = 0;
      auto load = [&](const CUtensorMap* m, int v, int bh) {
        const int s = idx % C::NST;
        const uint32_t ph = (idx / C::NST) & 1;
        ++idx;
        mbar_wait(kv_empty + s, ph ^ 1);
        uint8_t* dst = sKV + s * C::STAGE_BYTES;
        mbar_arrive_expect_tx(kv_full + s, C::STAGE_BYTES);
#pragma unroll
        for (int b = 0; b < C::NBOX; ++b)
          tma_load_3d_hint(dst + b * (BLK * 128), m, kv_full + s, b * 64, v * BLK, bh, pol);
      };
      auto start = [&](int t, int from) {
        int k = from;
        while (k < Tn && (sch->meta[k] & 1) != t) ++k;
        kcur[t] = k < Tn ? k : -1;
        if (kcur[t] < 0) return;
        const int it = sch->item[sch->ord[k]];
        bhs[t] = it / n_tiles;
        st[t].init(a, bhs[t], it % n_tiles, g_kv);
        nn[t] = sch->n[sch->ord[k]];
        jn[t] = 0;
        uint32_t gm;
        st[t].next(a, vcur[t], gm);
        load(&tmap_k, vcur[t], bhs[t]);
      };
      start(0, 0);
      start(1, 0);
      while (kcur[0] >= 0 || kcur[1] >= 0) {
        for (int t = 0; t < 2; ++t) {
          if (kcur[t] < 0) continue;
          load(&tmap_v, vcur[t], bhs[t]);
          if (++jn[t] < nn[t]) {
            uint32_t gm;
            st[t].next(a, vcur[t], gm);
            load(&tmap_k, vcur[t], bhs[t]);
          } else {
            start(t, kcur[t] + 1);
          }
        }
      }
    }
  } else if (warp == WARP_Q) {
    // ---------------------------------------------------------------- Q loader (start order)
    if (lane == 0) {
      for (int k = 0; k < Tn; ++k) {
        const int meta = sch->meta[k];
        const int buf = (meta >> 1) & 3;
        const uint32_t use_par = (meta >> 3) & 1;
        if (k >= NQB) mbar_wait(q_empty + buf, use_par ^ 1);
        const int it = sch->item[sch->ord[k]];
        uint8_t* dst = sQ + buf * C::Q_BYTES;
        mbar_arrive_expect_tx(q_full + buf, C::Q_BYTES);
#pragma unroll
        for (int b = 0; b < C::NBOX; ++b)
          tma_load_3d(dst + b * (BM * 128), &tmap_q, q_full + buf, b * 64, (it % n_tiles) * BM,
                      it / n_tiles);
      }
    }
    // empty tiles (no listed block in any of their query blocks): zero output, lse = -inf
    for (int i = 0; i < sch->T; ++i) {
      if (sch->n[i] != 0) continue;
      const int it = sch->item[i];
      const int bh = it / n_tiles, tile = it % n_tiles;
      for (int r = lane; r < BM; r += 32) {
        const int row = tile * BM + r;
        if (row >= a.n_q) continue;
        uint4* dst = reinterpret_cast<uint4*>(a.o + (long long)bh * a.o_stride + (long long)row * D);
        for (int c = 0; c < D / 8; ++c) dst[c] = make_uint4(0, 0, 0, 0);
        if (a.lse != nullptr) a.lse[(long long)bh * a.n_q + row] = -INFINITY;
      }
    }
  } else if (warp == WARP_MMA) {
    // ---------------------------------------------------------------- tcgen05 issuer
    // The whole warp runs the control flow so descriptors stay warp-uniform (uniform registers,
    // no per-instruction ELECT/R2UR loops); one elected lane issues each tcgen05 instruction.
    constexpr uint32_t IDESC_QK = idesc_bf16_f32(BM, BLK, 0, 0);
    constexpr uint32_t IDESC_PV = idesc_bf16_f32(BM, D, 0, 1);
    const bool leader = elect_one();
    const uint32_t kv_base = smem_u32(sKV);
    const uint32_t q_base0 = smem_u32(sQ);
    // descriptor "lo" words advance by (bytes >> 4); the hi word is constant per operand kind
    const uint64_t dq0 = sdesc_sw128(q_base0, 16, 1024);
    const uint64_t dk0 = sdesc_sw128(kv_base, 16, 1024);
    const uint64_t dv0 = sdesc_sw128(kv_base, BLK * 128, 1024);
    int kcur[2] = {-1, -1}, jn[2] = {0, 0}, nn[2] = {0, 0}, qb[2] = {0, 0};
    uint32_t p_cnt[2] = {0, 0};
    int idx = 0;
    auto next_stage = [&]() -> uint32_t {
      const int s = idx % C::NST;
      const uint32_t ph = (idx / C::NST) & 1;
      ++idx;
      mbar_wait(kv_full + s, ph);
      tc_fence_after();
      return (uint32_t)s;
    };
    auto issue_qk = [&](int t) {
      const uint32_t s = next_stage();
      const uint64_t da = dq0 + ((uint64_t)(qb[t] * C::Q_BYTES) >> 4);
      const uint64_t db = dk0 + ((uint64_t)(s * C::STAGE_BYTES) >> 4);
      const uint32_t d_tmem = tmem + t * 128;
      if (leader) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t oa = ((kk >> 2) * (BM * 128) + (kk & 3) * 32) >> 4;
          const uint32_t ob = ((kk >> 2) * (BLK * 128) + (kk & 3) * 32) >> 4;
          mma_ss(d_tmem, da + oa, db + ob, IDESC_QK, kk > 0);
        }
        mma_commit(kv_empty + s);
        mma_commit(s_bar + t);
        if (jn[t] == nn[t] - 1) mma_commit(q_empty + qb[t]);   // last use of this Q buffer
      }
      __syncwarp();
    };
    auto start = [&](int t, int from) {
      int k = from;
      while (k < Tn && (sch->meta[k] & 1) != t) ++k;
      kcur[t] = k < Tn ? k : -1;
      if (kcur[t] < 0) return;
      const int meta = sch->meta[k];
      qb[t] = (meta >> 1) & 3;
      nn[t] = sch->n[sch->ord[k]];
      jn[t] = 0;
      mbar_wait(q_full + qb[t], (meta >> 3) & 1);
      tc_fence_after();
      issue_qk(t);
    };
    start(0, 0);
    start(1, 0);
    while (kcur[0] >= 0 || kcur[1] >= 0) {
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        if (kcur[t] < 0) continue;
        mbar_wait(p_bar + t, p_cnt[t] & 1);
        ++p_cnt[t];
        tc_fence_after();
        {  // O_t += P_t V_j
          const uint32_t s = next_stage();
          const uint64_t dv = dv0 + ((uint64_t)(s * C::STAGE_BYTES) >> 4);
          const uint32_t o_tmem = tmem + 256 + t * D;
          const uint32_t p_tmem = tmem + t * 128;
          if (leader) {
#pragma unroll
            for (int kk = 0; kk < BLK / 16; ++kk)
              mma_ts(o_tmem, p_tmem + kk * 8, dv + ((uint32_t)(kk * 2048) >> 4), IDESC_PV,
                     (jn[t] > 0 || kk > 0) ? 1u : 0u);
            mma_commit(kv_empty + s);
          }
          __syncwarp();
        }
        if (++jn[t] < nn[t]) {
          issue_qk(t);
        } else {
          if (leader) mma_commit(o_bar + t);
          __syncwarp();
          start(t, kcur[t] + 1);
        }
      }
    }
  }
  } else {
    // ---------------------------------------------------------------- softmax warpgroups
    reg_alloc<REG_SOFTMAX>();
    const int t = warp >> 2;                 // slot
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t t_row = tmem + (uint32_t(quarter * 32) << 16);
    const uint32_t s_col = t * 128;
    const uint32_t o_col = 256 + t * D;
    const int grp = row / BLK;
    const float sl2 = a.scale_log2;
    const uint64_t sl2x2 = f2_pack(sl2, sl2);
    uint32_t s_cnt = 0, o_cnt = 0;
    for (int k = 0; k < Tn; ++k) {
      if ((sch->meta[k] & 1) != t) continue;
      const int it = sch->item[sch->ord[k]];
      const int bh = it / n_tiles, tile = it % n_tiles;
      Steps<G> st;
      st.init(a, bh, tile, g_kv);
      float m = -INFINITY;   // running max of s * scale * log2(e)
      float l = 0.f;         // running sum of exp2(s * sl2 - m)
      int v;
      uint32_t gm;
      bool have = st.next(a, v, gm);
      int j = 0;
      while (have) {
        SV_STAMP(0, 5 * s_cnt + 0)
        mbar_wait(s_bar + t, s_cnt & 1);
        SV_STAMP(0, 5 * s_cnt + 1)
        ++s_cnt;
        tc_fence_after();
        uint32_t sr[BLK];
        if constexpr (BLK >= 32) {
#pragma unroll
          for (int c = 0; c < BLK; c += 32) tmem_ld32(t_row + s_col + c, sr + c);
        } else {
#pragma unroll
          for (int c = 0; c < BLK; c += 8) tmem_ld8(t_row + s_col + c, sr + c);
        }
        // next step's block index: the load's latency hides under this step
        int v_n;
        uint32_t gm_n;
        const bool have_n = st.next(a, v_n, gm_n);
        tmem_wait_ld();
        const bool row_on = (gm >> grp) & 1u;
        const int valid = row_on ? min(BLK, a.n_kv - v * BLK) : 0;
        // ragged last KV block / rows whose query block does not list this step (warp-uniform
        // branch, rarely taken)
        if (__builtin_expect(__any_sync(0xffffffffu, valid < BLK), 0)) {
#pragma unroll
          for (int c = 0; c < BLK; ++c)
            if (c >= valid) sr[c] = __float_as_uint(-INFINITY);
        }
        float mx;
        {
          float mm[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int c = 0; c + 8 <= BLK; c += 8) {
            const int q = (c >> 3) & 3;
            mm[q] = fmax3(mm[q], __uint_as_float(sr[c]), __uint_as_float(sr[c + 1]));
            mm[q] = fmax3(mm[q], __uint_as_float(sr[c + 2]), __uint_as_float(sr[c + 3]));
            mm[q] = fmax3(mm[q], __uint_as_float(sr[c + 4]), __uint_as_float(sr[c + 5]));
            mm[q] = fmax3(mm[q], __uint_as_float(sr[c + 6]), __uint_as_float(sr[c + 7]));
          }
          mx = fmax3(fmaxf(mm[0], mm[1]), mm[2], mm[3]);
        }
        SV_STAMP(0, 5 * (s_cnt - 1) + 2)
        const float mx_s = mx * sl2;
        const bool need = mx_s > m + 8.0f;
        float alpha = 1.f;
        if (need) {
          alpha = ex2(m - mx_s);
          m = mx_s;
          l *= alpha;
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
              ex2_emu2(x, p0, p1);
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
        }
        {
          SV_STAMP(0, 5 * (s_cnt - 1) + 3)
          const uint64_t s2 = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
          float s0, s1;
          f2_unpack(s2, s0, s1);
          l += s0 + s1;
        }
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
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(p_bar + t);
        SV_STAMP(0, 5 * (s_cnt - 1) + 4)
        ++j;
        v = v_n;
        gm = gm_n;
        have = have_n;
      }
      // ------------------------------------------------------------ epilogue of this tile
      mbar_wait(o_bar + t, o_cnt & 1);
      ++o_cnt;
      tc_fence_after();
      const int n_row = tile * BM + row;
      const bool store = n_row < a.n_q;
      const bool live = m != -INFINITY;        // the row saw at least one valid logit
      const float inv = live ? 1.f / l : 0.f;
      uint16_t* orow = a.o + (long long)bh * a.o_stride + (long long)n_row * D;
#pragma unroll 1
      for (int c = 0; c < D; c += 32) {
        uint32_t o[32];
        tmem_ld32(t_row + o_col + c, o);
        tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          pk[i] = pack_bf16x2(__uint_as_float(o[2 * i]) * inv, __uint_as_float(o[2 * i + 1]) * inv);
        if (store) {
          uint4* dst = reinterpret_cast<uint4*>(orow + c);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
        }
      }
      if (a.lse != nullptr && store)
        a.lse[(long long)bh * a.n_q + n_row] =
            live ? (m * 0.69314718055994531f + logf(l)) : -INFINITY;
      tc_fence_before();
    }
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

template <int D, int BLK>
cudaError_t launch_t(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                     const AttnArgs& a, cudaStream_t st) {
  using C = Cfg<D, BLK>;
  auto kern = attn_fwd_kernel<D, BLK>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  if (e != cudaSuccess) return e;
  const int n_tiles = (a.n_q + BM - 1) / BM;
  const long long items = (long long)n_tiles * a.bh;
  const int sms = num_sms();
  for (long long b0 = 0; b0 < items; b0 += (long long)sms * MAX_TILES) {
    const long long b1 = b0 + (long long)sms * MAX_TILES < items ? b0 + (long long)sms * MAX_TILES : items;
    const long long cnt = b1 - b0;
    // two tile slots per CTA: fewer CTAs than SMs when there is little work
    const int grid = (int)(cnt >= 2LL * sms ? sms : (cnt + 1) / 2);
    kern<<<grid, NUM_THREADS, C::SMEM, st>>>(tq, tk, tv, a, (int)b0, (int)b1);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
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
