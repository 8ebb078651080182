// masks.cu — integer kernels of the hot path: CSLA local block mask (a1), cross-scale index
// mapping (a4), and merge + compaction of bit-row masks into CSR block lists (a5).
//
// All three are exact integer computations and are parity-tested bit for bit against the fp64 /
// integer oracle (oracle/csla.py, oracle/mapping.py, oracle/attention.py), which follows the
// paper token by token; these kernels instead mark contiguous flat-index ranges (a clipped window
// row or a footprint row is one contiguous run of a scale's row-major layout) and so touch every
// block a token run covers without visiting tokens one by one.
#include <cstdio>

#include "kernels.h"

namespace sv {
namespace {

// round-half-to-even of p/q, q > 0, p of any sign (READING 3 / READING 15)
__device__ __forceinline__ int rne_div(long long p, long long q) {
  long long fl = p / q;
  if ((p % q != 0) && ((p < 0) != (q < 0))) --fl;     // floor division
  const long long rem2 = 2 * (p - fl * q);            // in [0, 2q)
  if (rem2 > q || (rem2 == q && (fl & 1))) ++fl;
  return static_cast<int>(fl);
}

// Set bits [b0, b1] of a shared bit row.
__device__ __forceinline__ void set_bit_range(uint32_t* row, int b0, int b1) {
  for (int w = b0 >> 5; w <= (b1 >> 5); ++w) {
    const int lo = max(b0, w * 32) - w * 32;
    const int hi = min(b1, w * 32 + 31) - w * 32;
    const uint32_t m = (hi == 31 ? 0xffffffffu : ((1u << (hi + 1)) - 1u)) & ~((1u << lo) - 1u);
    atomicOr(row + w, m);
  }
}

// Flat token range [t0, t1] of the cache -> blocks.
__device__ __forceinline__ void set_token_range(uint32_t* row, int t0, int t1, int B) {
  set_bit_range(row, t0 / B, t1 / B);
}

// ------------------------------------------------------------------------------------ a1
// One CTA per query block u.  Each thread takes query tokens of u; for every scale h with a
// window it clips the Chebyshev square around the aligned coordinate and marks
// the blocks each square row covers.  The sink prefix [0, C_sink) is a single range.
struct WinArr {
  int w[kMaxScales];   // w[i] = window of scale K - i
  int base[kMaxScales];  // first cache row of scale h at [h-1]: C_{h-1}, or the compressed
                         // offset when the cache keeps only the CSLA scales (NEXT(4))
};

__global__ void local_mask_kernel(const Geo g, int K, int B, int sink_scales, const WinArr win,
                                  int W, uint32_t* __restrict__ out) {
  extern __shared__ uint32_t srow[];
  const int u = blockIdx.x;
  for (int w = threadIdx.x; w < W; w += blockDim.x) srow[w] = 0;
  __syncthreads();
  const int sK = g.side[K - 1];
  const int nq = sK * sK;
  if (threadIdx.x == 0 && sink_scales > 0) set_token_range(srow, 0, g.cum[sink_scales] - 1, B);
  for (int t = u * B + threadIdx.x; t < min((u + 1) * B, nq); t += blockDim.x) {
    const int x = t / sK, y = t % sK;
    for (int h = 1; h <= K; ++h) {
      const int w = win.w[K - h];
      if (w <= 0) continue;
      const int r = w / 2;
      const int sh = g.side[h - 1];
      const int xt = min(rne_div((long long)x * sh, sK), sh - 1);
      const int yt = min(rne_div((long long)y * sh, sK), sh - 1);
      const int x0 = max(0, xt - r), x1 = min(sh - 1, xt + r);
      const int y0 = max(0, yt - r), y1 = min(sh - 1, yt + r);
      const int base = win.base[h - 1];
      for (int xr = x0; xr <= x1; ++xr)
        set_token_range(srow, base + xr * sh + y0, base + xr * sh + y1, B);
    }
  }
  __syncthreads();
  for (int w = threadIdx.x; w < W; w += blockDim.x) out[(long long)u * W + w] = srow[w];
}

// ------------------------------------------------------------------------------------ a4
// Mapping is a union over tokens, so it is the OR, over the active blocks v of the source row
// phi(g), of the image T[v] of block v: the target blocks holding a projection of one of v's real
// tokens.  T depends only on the geometry, not on (b,h) or the row, so each CTA
// builds T for all source blocks in shared memory, then emits the target rows of its (b,h) range.
//
// Token j of source block v: decompose (READING 2), align l' = l + (K - S)
// (PAPER.md:870), project (READING 14).  A footprint row is a contiguous run of the
// target scale's row-major layout, marked as one block range.
__device__ void mark_image(const Geo& g, int j, int shift, int mode, int B, uint32_t* trow) {
  int l = 1;
  while (g.cum[l] <= j) ++l;                               // C_{l-1} <= j < C_l
  const int delta = j - g.cum[l - 1];
  const int lp = l + shift;
  const int s = g.side[l - 1], sp = g.side[lp - 1];
  const int x = delta / s, y = delta % s;
  const int base = g.cum[lp - 1];
  if (mode == 1) {                                         // POINT
    const int xp = x * sp / s, yp = y * sp / s;
    set_token_range(trow, base + xp * sp + yp, base + xp * sp + yp, B);
  } else {                                                 // FOOTPRINT (READING 14)
    const int x0 = x * sp / s, x1 = (x + 1) * sp / s - 1;
    const int y0 = y * sp / s, y1 = (y + 1) * sp / s - 1;
    for (int xp = x0; xp <= x1; ++xp)
      set_token_range(trow, base + xp * sp + y0, base + xp * sp + y1, B);
  }
}

__device__ __forceinline__ uint32_t range_word(int b0, int b1, int w) {
  const int lo = max(b0, w * 32), hi = min(b1, w * 32 + 31);
  if (lo > hi) return 0u;
  const int len = hi - lo + 1;
  return (len == 32 ? 0xffffffffu : ((1u << len) - 1u)) << (lo - w * 32);
}

// Image of source block v in the target bit row: OR over v's real tokens (see mark_image).
// MW > 0: one warp per source block, each lane ORs its tokens' footprint into MW register words,
// then a warp OR-reduction (no atomics).  MW == 0: shared-memory atomics (wide rows).
template <int MW>
__device__ void build_block_image(const Geo& g, int v, int S, int K, int B, int mode, int W_K,
                                  uint32_t* trow, int lane) {
  const int n_kvS = g.cum[S];
  const int shift = K - S;
  uint32_t acc[MW > 0 ? MW : 1];
#pragma unroll
  for (int w = 0; w < (MW > 0 ? MW : 1); ++w) acc[w] = 0u;
  for (int j = v * B + lane; j < min((v + 1) * B, n_kvS); j += 32) {
    if constexpr (MW == 0) {
      mark_image(g, j, shift, mode, B, trow);
    } else {
      int l = 1;
      while (g.cum[l] <= j) ++l;                             // C_{l-1} <= j < C_l
      const int delta = j - g.cum[l - 1];
      const int lp = l + shift;
      const int s = g.side[l - 1], sp = g.side[lp - 1];
      const int x = delta / s, y = delta % s;
      const int base = g.cum[lp - 1];
      int x0, x1, y0, y1;
      if (mode == 1) {                                       // POINT
        x0 = x1 = x * sp / s;
        y0 = y1 = y * sp / s;
      } else {                                               // FOOTPRINT (READING 14)
        x0 = x * sp / s; x1 = (x + 1) * sp / s - 1;
        y0 = y * sp / s; y1 = (y + 1) * sp / s - 1;
      }
      for (int xp = x0; xp <= x1; ++xp) {
        const int b0 = (base + xp * sp + y0) / B, b1 = (base + xp * sp + y1) / B;
#pragma unroll
        for (int w = 0; w < MW; ++w) acc[w] |= range_word(b0, b1, w);
      }
    }
  }
  if constexpr (MW > 0) {
#pragma unroll
    for (int w = 0; w < MW; ++w) {
      const uint32_t r = __reduce_or_sync(0xffffffffu, acc[w]);
      if (lane == 0 && w < W_K) trow[w] = r;
    }
  }
}

template <int MW>
__global__ void __launch_bounds__(1024) map_table_kernel(const Geo g, int S, int K, int B,
                                                        int sink_scales, int mode, int G_S,
                                                        int G_K, int G_kvS, int W_S, int W_K,
                                                        int bh_total, int bh_per_cta,
                                                        const uint32_t* __restrict__ src,
                                                        uint32_t* __restrict__ dst) {
  extern __shared__ uint32_t table[];                      // [G_kvS][W_K]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (MW == 0) {
    for (int i = threadIdx.x; i < G_kvS * W_K; i += blockDim.x) table[i] = 0;
    __syncthreads();
  }
  for (int v = warp; v < G_kvS; v += nw)
    build_block_image<MW>(g, v, S, K, B, mode, W_K, table + v * W_K, lane);
  __syncthreads();
  // sink blocks v < ceil(C_sink / B) (READING 13)
  const int n_sb = sink_scales > 0 ? (g.cum[sink_scales] + B - 1) / B : 0;
  const int bh0 = blockIdx.x * bh_per_cta;
  const int bh1 = min(bh_total, bh0 + bh_per_cta);
  const int items = (bh1 - bh0) * G_K * W_K;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int w = it % W_K;
    const int gq = (it / W_K) % G_K;
    const int bh = bh0 + it / (W_K * G_K);
    int gs = rne_div(2LL * gq * G_S + G_S - G_K, 2LL * G_K);   // phi
    gs = min(max(gs, 0), G_S - 1);
    const uint32_t* srow = src + ((long long)bh * G_S + gs) * W_S;
    uint32_t acc = 0;
    for (int ws = 0; ws < W_S; ++ws) {
      uint32_t bits = __ldg(srow + ws);
      while (bits) {
        const int v = ws * 32 + __ffs(bits) - 1;
        bits &= bits - 1;
        if (v < G_kvS) acc |= table[v * W_K + w];
      }
    }
    const int lo = w * 32;
    if (lo < n_sb) acc |= (n_sb - lo >= 32) ? 0xffffffffu : ((1u << (n_sb - lo)) - 1u);
    dst[((long long)bh * G_K + gq) * W_K + w] = acc;
  }
}

// Fallback when the block-image table does not fit in shared memory (tiny blocks, e.g. B = 1).
// One CTA per (target query block gq, bh).  Source row phi(gq); every real token of
// every active source block is decomposed, aligned to l' = l + (K - S)
// and projected (READING 14).
__global__ void map_kernel(const Geo g, int S, int K, int B, int sink_scales, int mode, int G_S,
                           int G_K, int W_S, int W_K, const uint32_t* __restrict__ src,
                           uint32_t* __restrict__ dst) {
  extern __shared__ uint32_t srow[];
  const int gq = blockIdx.x;
  const int bh = blockIdx.y;
  for (int w = threadIdx.x; w < W_K; w += blockDim.x) srow[w] = 0;
  __syncthreads();
  int gs = rne_div(2LL * gq * G_S + G_S - G_K, 2LL * G_K);
  gs = min(max(gs, 0), G_S - 1);
  const uint32_t* srcrow = src + ((long long)bh * G_S + gs) * W_S;
  const int n_kvS = g.cum[S];
  const int shift = K - S;
  for (int w = 0; w < W_S; ++w) {
    uint32_t bits = __ldg(srcrow + w);
    while (bits) {
      const int v = w * 32 + __ffs(bits) - 1;
      bits &= bits - 1;
      for (int j = v * B + threadIdx.x; j < min((v + 1) * B, n_kvS); j += blockDim.x)
        mark_image(g, j, shift, mode, B, srow);
    }
  }
  if (threadIdx.x == 0 && sink_scales > 0) set_token_range(srow, 0, g.cum[sink_scales] - 1, B);
  __syncthreads();
  uint32_t* drow = dst + ((long long)bh * G_K + gq) * W_K;
  for (int w = threadIdx.x; w < W_K; w += blockDim.x) drow[w] = srow[w];
}

// ------------------------------------------------------------------------ NEXT(2): token level
// TopK of one column-sum row A^(S)[g, :] (READING 11): one CTA per
// (b,h,g).  The k-th largest value is found by a 4 x 8-bit radix select on the float bits
// (column sums are >= 0, so their bit patterns order like the values); every value above it is
// kept, and of the values equal to it the ones with the smallest indices (ties to the smaller
// j), then the sink tokens j < C_sink are added.  Output: bit row of ceil(n/32) words.
constexpr int TK_THREADS = 256;

__global__ void __launch_bounds__(TK_THREADS) topk_tokens_kernel(const float* __restrict__ a, int n,
                                                                 int k_tok, int n_sink,
                                                                 uint32_t* __restrict__ out) {
  __shared__ unsigned hist[256];
  __shared__ unsigned s_prefix, s_remaining;
  __shared__ int s_warp[TK_THREADS / 32];
  const long long row = blockIdx.x;
  const float* x = a + row * n;
  const int W = (n + 31) / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned prefix = 0, mask = 0, remaining = (unsigned)min(k_tok, n);
  const bool all = k_tok >= n;
  if (!all) {
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0;
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const unsigned key = __float_as_uint(x[i]);
        if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        unsigned cum = 0;
        int b = 255;
        for (; b > 0; --b) {
          if (cum + hist[b] >= remaining) break;
          cum += hist[b];
        }
        s_prefix = prefix | ((unsigned)b << shift);
        s_remaining = remaining - cum;
      }
      __syncthreads();
      prefix = s_prefix;
      remaining = s_remaining;
      mask |= 255u << shift;
      __syncthreads();
    }
  }
  // prefix = bits of the k-th largest value T; keep x > T, and the first `remaining` x == T
  unsigned eq_before = 0;                                   // equal values in earlier chunks
  for (int c0 = 0; c0 < W * 32; c0 += blockDim.x) {
    const int i = c0 + threadIdx.x;
    const unsigned key = i < n ? __float_as_uint(x[i]) : 0u;
    const bool eq = !all && i < n && key == prefix;
    const unsigned eb = __ballot_sync(0xffffffffu, eq);
    if (lane == 0) s_warp[warp] = __popc(eb);
    __syncthreads();
    unsigned before = eq_before;
    unsigned tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      if (w < warp) before += s_warp[w];
      tot += s_warp[w];
    }
    before += __popc(eb & ((1u << lane) - 1u));
    bool sel = i < n && (all || key > prefix || (eq && before < remaining));
    sel = sel || (i < n_sink);
    const unsigned word = __ballot_sync(0xffffffffu, sel);
    if (lane == 0 && (i >> 5) < W) out[row * W + (i >> 5)] = word;
    eq_before += tot;
    __syncthreads();
  }
}

// Token-level M_{S->K} (READING 14): one CTA per (b,h, target query block g_K).
// Every selected token of source block phi(g_K) is projected by Decompose-Align-Project with the
// forward-interval footprint (mark_image at block size 1, i.e. token granularity), then the sink
// tokens j < C_sink are added.
__global__ void map_tokens_kernel(const Geo g, int S, int K, int C, int sink_scales, int mode,
                                  const uint32_t* __restrict__ src, uint32_t* __restrict__ dst) {
  extern __shared__ uint32_t trow[];
  const int G_S = (g.side[S - 1] * g.side[S - 1] + C - 1) / C;
  const int G_K = (g.side[K - 1] * g.side[K - 1] + C - 1) / C;
  const int bh = blockIdx.x / G_K, gk = blockIdx.x % G_K;
  const int n_S = g.cum[S], n_K = g.cum[K];
  const int W_S = (n_S + 31) / 32, W_K = (n_K + 31) / 32;
  for (int w = threadIdx.x; w < W_K; w += blockDim.x) trow[w] = 0;
  __syncthreads();
  // phi(g_K) = clamp(rne(((2 g_K + 1) G_S - G_K) / (2 G_K)), 0, G_S - 1)
  const int gs = min(max(rne_div((long long)(2 * gk + 1) * G_S - G_K, 2LL * G_K), 0), G_S - 1);
  const uint32_t* srow = src + ((long long)bh * G_S + gs) * W_S;
  for (int j = threadIdx.x; j < n_S; j += blockDim.x)
    if ((__ldg(srow + (j >> 5)) >> (j & 31)) & 1u) mark_image(g, j, K - S, mode, 1, trow);
  if (threadIdx.x == 0 && sink_scales > 0) set_bit_range(trow, 0, g.cum[sink_scales] - 1);
  __syncthreads();
  uint32_t* drow = dst + ((long long)bh * G_K + gk) * W_K;
  for (int w = threadIdx.x; w < W_K; w += blockDim.x) drow[w] = trow[w];
}

// ------------------------------------------------------------------------------------ a5
// Up to 32 CTAs, each owning a contiguous range of rows.  A CTA first counts the set bits of all
// rows before its range (coalesced over words; at most a few thousand L2 hits) to get its base
// offset — no inter-CTA communication, deterministic.  Then, in chunks of blockDim rows: one
// thread per row ORs the masks' words and counts, a block scan gives row_ptr, and one WARP per
// row writes the ascending list (ballot prefix per word, coalesced stores).
constexpr int BL_THREADS = 256;
constexpr int BL_MAX_CTAS = 32;
constexpr int BL_WMAX = 8;

__device__ __forceinline__ uint32_t row_word(const MaskSet& ms, int r, int u, int w, int W) {
  uint32_t x = 0;
  for (int i = 0; i < ms.n; ++i)
    x |= __ldg(ms.ptr[i] + (long long)(ms.broadcast[i] ? u : r) * W + w);
  return x;
}

__device__ __forceinline__ int block_sum(int v, int* s_warp) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) s_warp[warp] = v;
  __syncthreads();
  int tot = 0;
  for (int i = 0; i < nw; ++i) tot += s_warp[i];
  return tot;
}

__global__ void __launch_bounds__(BL_THREADS) build_lists_kernel(int rows, int g_q, int g_kv,
                                                                 MaskSet ms, int* __restrict__ row_ptr,
                                                                 int* __restrict__ col_idx,
                                                                 long long cap, int* status,
                                                                 int rows_per_cta) {
  __shared__ int s_warp[32];
  __shared__ int s_off[BL_THREADS + 1];
  __shared__ uint32_t s_words[BL_THREADS * BL_WMAX];   // the chunk's OR-ed rows (W <= BL_WMAX)
  const int W = (g_kv + 31) / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int r0 = blockIdx.x * rows_per_cta;
  const int r1 = min(rows, r0 + rows_per_cta);
  if (r0 >= r1) return;
  // base offset: set bits of rows [0, r0)
  int mine = 0;
  // rows [0, r0), 4 rows per thread per round so several loads are in flight
  for (int rb = threadIdx.x; rb < r0; rb += 4 * blockDim.x) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = rb + q * blockDim.x;
      if (r < r0) {
        const int u = r % g_q;
        for (int w = 0; w < W; ++w) mine += __popc(row_word(ms, r, u, w, W));
      }
    }
  }
  long long base = block_sum(mine, s_warp);
  if (blockIdx.x == 0 && threadIdx.x == 0) row_ptr[0] = 0;
  int err = 0;
  for (int c0 = r0; c0 < r1; c0 += blockDim.x) {
    const int r = c0 + threadIdx.x;
    int c = 0;
    if (r < r1) {
      for (int w = 0; w < W; ++w) {
        const uint32_t x = row_word(ms, r, r % g_q, w, W);
        if (W <= BL_WMAX) s_words[threadIdx.x * BL_WMAX + w] = x;
        c += __popc(x);
      }
      if (c == 0) err = 5;                                  // SPARVAR_ERR_EMPTY_ROW
    }
    // block exclusive scan of c
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    __syncthreads();
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    int wpre = 0, tot = 0;
    for (int i = 0; i < nw; ++i) {
      if (i < warp) wpre += s_warp[i];
      tot += s_warp[i];
    }
    const int excl = wpre + inc - c;
    s_off[threadIdx.x] = excl;
    if (threadIdx.x == 0) s_off[blockDim.x] = tot;
    if (r < r1) row_ptr[r + 1] = (int)(base + excl + c);
    __syncthreads();
    if (base + tot > cap) {
      if (threadIdx.x == 0 && status) atomicCAS(status, 0, 4);   // SPARVAR_ERR_CAPACITY
      return;
    }
    // one warp per row: coalesced list stores
    for (int rr = warp; rr < min((int)blockDim.x, r1 - c0); rr += nw) {
      const int row = c0 + rr;
      long long pos = base + s_off[rr];
      for (int w = 0; w < W; ++w) {
        const uint32_t x = W <= BL_WMAX ? s_words[rr * BL_WMAX + w]   // warp-uniform
                                        : row_word(ms, row, row % g_q, w, W);
        if ((x >> lane) & 1u) col_idx[pos + __popc(x & ((1u << lane) - 1u))] = w * 32 + lane;
        pos += __popc(x);
      }
    }
    base += tot;
    __syncthreads();
  }
  if (err && status) atomicCAS(status, 0, err);
}

// Wide rows (W > BL_WMAX words, e.g. token bit rows of NEXT(2)): three passes instead of one
// kernel that re-counts every earlier row.  (1) one warp per row writes its popcount (OR of the
// masks) to row_ptr[r + 1]; (2) one CTA scans row_ptr in place (chunked, deterministic) and
// flags empty rows / capacity; (3) one CTA per row writes the ascending column list, a block
// scan of the per-word counts giving each word's offset.
__global__ void __launch_bounds__(256) wide_count_kernel(int rows, int g_q, int W, MaskSet ms,
                                                         int* __restrict__ row_ptr) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  int c = 0;
  for (int w = lane; w < W; w += 32) c += __popc(row_word(ms, warp, warp % g_q, w, W));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) row_ptr[warp + 1] = c;
}

__global__ void __launch_bounds__(1024) wide_scan_kernel(int rows, int* __restrict__ row_ptr,
                                                         long long cap, int* status) {
  __shared__ int s_warp[32];
  __shared__ long long s_carry;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { s_carry = 0; row_ptr[0] = 0; }
  __syncthreads();
  int err = 0;
  for (int c0 = 0; c0 < rows; c0 += blockDim.x) {
    const int r = c0 + threadIdx.x;
    const int c = r < rows ? row_ptr[r + 1] : 0;
    if (r < rows && c == 0) err = 5;                        // SPARVAR_ERR_EMPTY_ROW
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    int wpre = 0, tot = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      if (i < warp) wpre += s_warp[i];
      tot += s_warp[i];
    }
    const long long carry = s_carry;
    if (r < rows) row_ptr[r + 1] = (int)(carry + wpre + inc);
    __syncthreads();
    if (threadIdx.x == 0) s_carry = carry + tot;
    __syncthreads();
  }
  if (s_carry > cap && threadIdx.x == 0 && status) atomicCAS(status, 0, 4);   // CAPACITY
  if (err && status) atomicCAS(status, 0, err);
}

__global__ void __launch_bounds__(256) wide_write_kernel(int g_q, int W, MaskSet ms,
                                                         const int* __restrict__ row_ptr,
                                                         int* __restrict__ col_idx, long long cap) {
  __shared__ int s_warp[8];
  __shared__ int s_carry;
  const int r = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long base = row_ptr[r];
  if ((long long)row_ptr[r + 1] > cap) return;             // capacity error already flagged
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int w0 = 0; w0 < W; w0 += blockDim.x) {
    const int w = w0 + threadIdx.x;
    const uint32_t x = w < W ? row_word(ms, r, r % g_q, w, W) : 0u;
    const int c = __popc(x);
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    int wpre = 0, tot = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      if (i < warp) wpre += s_warp[i];
      tot += s_warp[i];
    }
    long long pos = base + s_carry + wpre + inc - c;
    for (uint32_t y = x; y; y &= y - 1) col_idx[pos++] = w * 32 + __ffs(y) - 1;
    __syncthreads();
    if (threadIdx.x == 0) s_carry += tot;
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_local_mask(const Geo& g, int target, int block, int sink_scales,
                              const int* windows_rel, uint32_t* out, cudaStream_t st,
                              bool compressed) {
  WinArr win;
  for (int i = 0; i < kMaxScales; ++i) win.w[i] = windows_rel[i];
  // compressed cache (NEXT(4)): only the sink scales and the windowed scales, in scale order
  int n_kv = 0;
  for (int h = 1; h <= target; ++h) {
    const bool keep = !compressed || h <= sink_scales || windows_rel[target - h] > 0;
    win.base[h - 1] = compressed ? n_kv : g.cum[h - 1];
    if (keep) n_kv += g.side[h - 1] * g.side[h - 1];
  }
  if (!compressed) n_kv = g.cum[target];
  const int nq = g.side[target - 1] * g.side[target - 1];
  const int gq = (nq + block - 1) / block;
  const int gkv = (n_kv + block - 1) / block;
  const int W = (gkv + 31) / 32;
  const size_t smem = size_t(W) * 4;
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(local_mask_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const int threads = block >= 256 ? 256 : (block >= 64 ? block : 64);
  local_mask_kernel<<<gq, threads, smem, st>>>(g, target, block, sink_scales, win, W, out);
  return cudaGetLastError();
}

cudaError_t launch_map_indices(const Geo& g, int S, int K, int block, int sink_scales, int mode,
                               int bh, const uint32_t* src, uint32_t* dst, cudaStream_t st) {
  const int nS = g.side[S - 1] * g.side[S - 1], nK = g.side[K - 1] * g.side[K - 1];
  const int G_S = (nS + block - 1) / block, G_K = (nK + block - 1) / block;
  const int G_kvS = (g.cum[S] + block - 1) / block;
  const int W_S = (G_kvS + 31) / 32;
  const int W_K = ((g.cum[K] + block - 1) / block + 31) / 32;
  const size_t smem = size_t(G_kvS) * W_K * 4;
  if (smem > 100 * 1024) {
    const size_t row_smem = size_t(W_K) * 4;
    if (row_smem > 200 * 1024) return cudaErrorInvalidValue;
    if (row_smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(map_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)row_smem);
      if (e != cudaSuccess) return e;
    }
    dim3 grid(G_K, bh);
    map_kernel<<<grid, block >= 128 ? 128 : 64, row_smem, st>>>(g, S, K, block, sink_scales, mode,
                                                                G_S, G_K, W_S, W_K, src, dst);
    return cudaGetLastError();
  }
  // Enough CTAs to cover the SMs; each CTA rebuilds the (identical) table for its (b,h) range.
  const int bh_per_cta = bh <= 148 ? 1 : (bh + 147) / 148;
  const int ctas = (bh + bh_per_cta - 1) / bh_per_cta;
  auto launch = [&](auto kern) -> cudaError_t {
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
      if (e != cudaSuccess) return e;
    }
    kern<<<ctas, 1024, smem, st>>>(g, S, K, block, sink_scales, mode, G_S, G_K, G_kvS, W_S, W_K,
                                  bh, bh_per_cta, src, dst);
    return cudaGetLastError();
  };
  if (W_K <= 4) return launch(map_table_kernel<4>);
  if (W_K <= 8) return launch(map_table_kernel<8>);
  return launch(map_table_kernel<0>);
}

cudaError_t launch_build_lists(int bh, int g_q, int g_kv, const MaskSet& ms, int* row_ptr,
                               int* col_idx, long long cap, int* status, cudaStream_t st) {
  const int rows = bh * g_q;
  const int W = (g_kv + 31) / 32;
  if (W > BL_WMAX) {
    wide_count_kernel<<<(rows * 32 + 255) / 256, 256, 0, st>>>(rows, g_q, W, ms, row_ptr);
    wide_scan_kernel<<<1, 1024, 0, st>>>(rows, row_ptr, cap, status);
    wide_write_kernel<<<rows, 256, 0, st>>>(g_q, W, ms, row_ptr, col_idx, cap);
    return cudaGetLastError();
  }
  int ctas = (rows + 63) / 64;
  if (ctas > BL_MAX_CTAS) ctas = BL_MAX_CTAS;
  const int per = (rows + ctas - 1) / ctas;
  ctas = (rows + per - 1) / per;
  build_lists_kernel<<<ctas, BL_THREADS, 0, st>>>(rows, g_q, g_kv, ms, row_ptr, col_idx, cap, status,
                                                  per);
  return cudaGetLastError();
}

cudaError_t launch_topk_tokens(int rows, int n, int k_tok, int n_sink, const float* a,
                               uint32_t* out, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  topk_tokens_kernel<<<rows, TK_THREADS, 0, st>>>(a, n, k_tok, n_sink, out);
  return cudaGetLastError();
}

cudaError_t launch_map_tokens(const Geo& g, int S, int K, int C, int sink_scales, int mode,
                              int bh, const uint32_t* src, uint32_t* dst, cudaStream_t st) {
  const int G_K = (g.side[K - 1] * g.side[K - 1] + C - 1) / C;
  const size_t shm = size_t((g.cum[K] + 31) / 32) * 4;
  if (shm > 48 * 1024) return cudaErrorInvalidValue;
  const long long grid = (long long)bh * G_K;
  if (grid <= 0) return cudaSuccess;
  map_tokens_kernel<<<(unsigned)grid, 256, shm, st>>>(g, S, K, C, sink_scales, mode, src, dst);
  return cudaGetLastError();
}

}  // namespace sv
