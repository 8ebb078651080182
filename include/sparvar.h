/* sparvar.h — C ABI of libsparvar.so, the sm_100a (B200) hot path of SparVAR
 * (arXiv 2602.04361, "block-sparse cross-scale attention" for next-scale image generators).
 *
 * Citations "PAPER.md:<line>" refer to the paper text; READING n refers to the numbered readings
 * of ambiguous passages in DESIGN.md ("Readings") / SURVEY.md §8(c).
 *
 * Conventions shared by every entry point
 *  - Scales are 1-based (READING 1).  A schedule is the list of square grid sides s_1..s_K
 *    (non-decreasing, s_1 >= 1); N_k = s_k^2 tokens, C_k = N_1 + ... + N_k (PAPER.md:200-204,
 *    860).  The KV cache of scale k is the first C_k rows of a cache that may hold more rows
 *    (PAPER.md:211, 854).
 *  - Blocks: query block u covers tokens [uB, min((u+1)B, N_k)), KV block v covers
 *    flat cache rows [vB, min((v+1)B, C_k)).  G_q = ceil(N_k/B), G_kv = ceil(C_k/B).
 *  - A block mask is stored as BIT ROWS: row r has W = ceil(G_kv/32) uint32 words
 *    [r*W, (r+1)*W); block v is active iff bit (v % 32) of word (v / 32) is set.  Bits >= G_kv
 *    are zero on output.
 *  - Tensors are BHND: element (bh, n, d) of Q at q[bh*q_stride_bh + n*D + d];
 *    bh = batch*H + head.  bf16 tensors are passed as uint16_t pointers to the bf16 bit patterns.
 *  - Ownership: every pointer is caller-owned DEVICE memory unless marked "host".  The library
 *    allocates nothing, keeps no state between calls, and builds its TMA descriptors per call on
 *    the host.
 *  - Asynchrony: every call validates its arguments on the host, enqueues its kernels on
 *    `stream` (a cudaStream_t; NULL = legacy default stream) and returns.  Argument errors are
 *    returned synchronously and nothing is enqueued; errors only detectable on the device (an
 *    empty block-list row, CSR capacity overflow) are written to `status_dev`.
 *  - Every call returns a sparvar_status; on a non-OK status sparvar_last_error() returns a
 *    thread-local message.
 *  - Determinism: masks, block lists, selections and attention outputs are bitwise identical run
 *    to run (no atomics with order-dependent results, no split-KV reductions).
 */
#ifndef SPARVAR_H_
#define SPARVAR_H_

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SPARVAR_OK = 0,
  SPARVAR_ERR_INVALID_ARG = 1,   /* null pointer, out-of-range scale/block/k, misaligned stride */
  SPARVAR_ERR_SCHEDULE = 2,      /* empty / non-monotone schedule, side < 1 */
  SPARVAR_ERR_UNSUPPORTED = 3,   /* valid but not implemented here (head_dim, block, smem size) */
  SPARVAR_ERR_CAPACITY = 4,      /* (device) CSR col_idx capacity exceeded */
  SPARVAR_ERR_EMPTY_ROW = 5,     /* (device) a query block with no active KV block */
  SPARVAR_ERR_CUDA = 6           /* a CUDA runtime/driver call failed */
} sparvar_status;

typedef enum { SPARVAR_SELECT_TOPK = 0, SPARVAR_SELECT_THRESHOLD = 1 } sparvar_select_mode;
typedef enum { SPARVAR_MAP_FOOTPRINT = 0, SPARVAR_MAP_POINT = 1 } sparvar_map_mode;

/* Scale schedule; `sides` is a HOST array of num_scales int32. */
typedef struct {
  int32_t num_scales;
  const int32_t* sides;
} sparvar_schedule;

/* Shape of one attention call.  head_dim D in {64, 128}.  Strides are in ELEMENTS between
 * consecutive (b,h) slabs and must be multiples of 8 (16-byte TMA alignment); q_stride_bh >= N*D,
 * kv_stride_bh >= C_k*D (the cache capacity may exceed C_k), o_stride_bh >= N*D.
 * Pointers must be 16-byte aligned. */
typedef struct {
  int32_t batch_heads;      /* B*H: number of independent (batch, head) units */
  int32_t head_dim;
  int64_t q_stride_bh;
  int64_t kv_stride_bh;
  int64_t o_stride_bh;
} sparvar_attn_shape;

/* (a1) CSLA cross-scale local block mask B^(K)(u,v)  (Eq. block_mask).
 *   Token mask M(q, j) = sink OR local: key j is active for query q = (x, y) of scale K iff
 *   j < C_{sink_scales}, or j = (h, x_k, y_k) with window w_h > 0 and
 *   |x~ - x_k| <= floor(w_h/2), |y~ - y_k| <= floor(w_h/2), where x~ = min(rne(x s_h / s_K), s_h-1)
 *   (READINGS 3-5).  B(u,v) = OR over the real tokens of tile (u,v).
 *   windows:  HOST array; windows[i] is w for scale target_scale - i (i = 0: the target scale);
 *             0 = scale masked; nonzero windows must be odd.  Scales not covered are masked.
 *             Paper default: {7,5,3,1,1} with sink_scales = 5 (READING 5).
 *   block:    B >= 1.   sink_scales in [0, target_scale].
 *   mask_out: [G_q][W] bit rows (one mask, identical for every (b,h)).
 */
sparvar_status sparvar_local_mask(const sparvar_schedule* sched, int32_t target_scale,
                                  int32_t block, int32_t sink_scales, const int32_t* windows,
                                  int32_t num_windows, uint32_t* mask_out, void* stream);

/* (a2, a3) Decision-scale predictor  (READINGS 10-13).
 *   For each (b,h): P = softmax(Q_S K_{<=S}^T * softmax_scale) over keys j < C_S in fp32 from
 *   bf16 inputs (fp32 logits, fp32 exp);  mass[u,v] = sum_{q in u} sum_{j in v} P[q,j].
 *   Row u keeps TOPK(topk): the topk largest masses, ties to the smaller v (topk >= G_kvS keeps
 *   all), or THRESHOLD: mass[u,v] >= threshold * |u| (fp32 compare); then OR the sink blocks
 *   v < ceil(C_{sink_scales} / B).
 *   shape:    head_dim, batch_heads, q_stride_bh (Q_S slabs), kv_stride_bh (cache slabs).
 *   q_S:      bf16 [BH][N_S][D];  k_cache: bf16 cache, rows [0, C_S) of each slab are read.
 *   softmax_scale <= 0 selects 1/sqrt(D).   block in {16, 32, 64, 128}.
 *   mass_out: nullable fp32 [BH][G_S][G_kvS].    mask_out: [BH][G_S][W_S] bit rows.
 *   Returns SPARVAR_ERR_UNSUPPORTED if the per-row statistics (G_kvS * 8 bytes per query row)
 *   do not fit in shared memory.
 */
sparvar_status sparvar_predict_pattern(const sparvar_schedule* sched, int32_t decision_scale,
                                       int32_t block, int32_t sink_scales,
                                       const sparvar_attn_shape* shape, const uint16_t* q_S,
                                       const uint16_t* k_cache, float softmax_scale,
                                       int32_t select_mode, int32_t topk, float threshold,
                                       float* mass_out, uint32_t* mask_out, void* stream);

/* (a4) Cross-scale index mapping M_{S->K}  (READINGS 2, 10, 14, 15).
 *   Target query block g takes the pattern of source row phi(g) = clamp(rne(((2g+1) G_S - G_K)
 *   / (2 G_K)), 0, G_S-1) (Query Block Homography).  Every real token j < C_S of
 *   every active source block is decomposed to (l, delta), aligned to l' = K - (S - l)
 *    and projected: POINT  (x', y') = (floor(x s_l'/s_l), floor(y s_l'/s_l))
 *   (PAPER.md:878); FOOTPRINT (default, READING 14) all (x', y') with
 *   floor(x s_l'/s_l) <= x' < floor((x+1) s_l'/s_l), likewise y'.  A target block is active iff
 *   it holds a projected token; then OR the sink blocks v < ceil(C_{sink_scales}/B).
 *   src_mask: [batch_heads][G_S][W_S] bit rows (from sparvar_predict_pattern, same block).
 *   dst_mask: [batch_heads][G_K][W_K] bit rows.   src_scale <= dst_scale.
 */
sparvar_status sparvar_map_indices(const sparvar_schedule* sched, int32_t src_scale,
                                   int32_t dst_scale, int32_t block, int32_t sink_scales,
                                   int32_t map_mode, int32_t batch_heads,
                                   const uint32_t* src_mask, uint32_t* dst_mask, void* stream);

/* (a5) Merge + compact to CSR block lists  (READING 19: union of the masks in use).
 *   Row r = bh*g_q + u of the output is the ascending list of set bits of
 *   OR_i masks[i][row r or row u if broadcast[i]].
 *   masks:     HOST array of num_masks DEVICE pointers to bit-row masks with W = ceil(g_kv/32);
 *   broadcast: HOST array; 1 = masks[i] is a single [g_q][W] mask shared by all bh (CSLA),
 *              0 = masks[i] is [batch_heads][g_q][W].
 *   row_ptr:   int32 [batch_heads*g_q + 1];  col_idx: int32 [col_capacity].
 *   status_dev: nullable int32 on the device; set to SPARVAR_ERR_EMPTY_ROW if a row is empty or
 *              SPARVAR_ERR_CAPACITY if nnz > col_capacity (col_idx is then not written), left
 *              untouched otherwise (initialise it to 0).
 *   1 <= num_masks <= 8.
 */
sparvar_status sparvar_build_block_lists(int32_t batch_heads, int32_t g_q, int32_t g_kv,
                                         const uint32_t* const* masks, const int32_t* broadcast,
                                         int32_t num_masks, int32_t* row_ptr, int32_t* col_idx,
                                         int64_t col_capacity, int32_t* status_dev, void* stream);

/* (a6) Block-sparse cross-scale attention forward  (PAPER.md:204-212 Eq. attn_cross_scale
 *   restricted as in Eq. sparse_update PAPER.md:318-328 and Eq. block_mask).
 *   For query t of query block u of (b,h): o_t = sum_{j in J} softmax_J(q_t.k_j * scale) v_j with
 *   J = union over v in col_idx[row_ptr[r]..row_ptr[r+1]) of [vB, min((v+1)B, C_K)),
 *   r = bh*G_q + u (READINGS 9, 17, 20).  Lists must be ascending and duplicate-free.
 *   bf16 inputs, fp32 logits / online softmax / accumulation, bf16 output.
 *   q:  bf16 [BH][N_K][D];  k_cache, v_cache: bf16 caches (rows [0, C_K) read);
 *   o:  bf16 [BH][N_K][D];  lse: nullable fp32 [BH][N_K] natural-log sum-exp of the scaled logits.
 *   block in {16, 32, 64, 128}; head_dim in {64, 128}; softmax_scale <= 0 -> 1/sqrt(D).
 *   An empty list row yields a zero output row and lse = -inf.
 */
sparvar_status sparvar_block_sparse_attn(const sparvar_schedule* sched, int32_t target_scale,
                                         int32_t block, const sparvar_attn_shape* shape,
                                         const uint16_t* q, const uint16_t* k_cache,
                                         const uint16_t* v_cache, const int32_t* row_ptr,
                                         const int32_t* col_idx, float softmax_scale,
                                         uint16_t* o, float* lse, void* stream);

/* (a7) Dense cross-scale attention forward, Eq. attn_cross_scale: the same kernel
 *   with every KV block of [0, C_K) listed.  The denominator of the speed-up figure. */
sparvar_status sparvar_dense_attn(const sparvar_schedule* sched, int32_t target_scale,
                                  const sparvar_attn_shape* shape, const uint16_t* q,
                                  const uint16_t* k_cache, const uint16_t* v_cache,
                                  float softmax_scale, uint16_t* o, float* lse, void* stream);

/* NEXT(1) — CS4A dense-attention cache residual at the decision scale S:
 *   O_cache = O_dense - Softmax(Q_S K_inds^T) V_inds, the sparse term being the block-sparse
 *   attention over the decision-scale lists (row_ptr_S / col_idx_S, e.g. built from the
 *   predictor's mask with sparvar_build_block_lists).  Runs the dense kernel into o_cache, the
 *   block-sparse kernel into o_scratch, then subtracts in fp32 (bf16 result).
 *   q_S: bf16 [BH][N_S][D]; o_scratch, o_cache: caller-owned bf16 [BH][N_S][D] with the shape's
 *   o_stride_bh, must not alias.  block as for sparvar_block_sparse_attn.
 */
sparvar_status sparvar_cache_residual(const sparvar_schedule* sched, int32_t decision_scale,
                                     int32_t block, const sparvar_attn_shape* shape,
                                     const uint16_t* q_S, const uint16_t* k_cache,
                                     const uint16_t* v_cache, const int32_t* row_ptr_S,
                                     const int32_t* col_idx_S, float softmax_scale,
                                     uint16_t* o_scratch, uint16_t* o_cache, void* stream);

/* NEXT(1)/NEXT(3) — the same O_cache when the dense attention at S has already been computed
 *   (the decision scale runs dense attention in every layer): o_dense is that
 *   output (bf16 [BH][N_S][D], o_stride_bh), read only; o_cache receives
 *   o_dense - Softmax(Q K_inds^T) V_inds (the block-sparse term is computed into o_cache and
 *   subtracted in place, fp32, bf16 result).  o_cache must not alias o_dense.  Errors as for
 *   sparvar_cache_residual.
 */
sparvar_status sparvar_cache_residual_from_dense(const sparvar_schedule* sched,
                                                int32_t decision_scale, int32_t block,
                                                const sparvar_attn_shape* shape,
                                                const uint16_t* q_S, const uint16_t* k_cache,
                                                const uint16_t* v_cache, const int32_t* row_ptr_S,
                                                const int32_t* col_idx_S, float softmax_scale,
                                                const uint16_t* o_dense, uint16_t* o_cache,
                                                void* stream);

/* NEXT(3) — the decision-scale dense pass with the predictor fused in (the
 *   model runs full attention at S, and the block masses are read off that same softmax):
 *   o = dense attention at decision_scale (as sparvar_dense_attn, but the key-block size is
 *   `block`), lse (nullable, fp32 [BH][N_S]) its log-sum-exp, and mass_out (nullable,
 *   fp32 [BH][G_S][G_kvS]) / mask_out (bit rows [BH][G_S][W_S]) exactly as
 *   sparvar_predict_pattern defines them (same selection rules and tie breaks; masses from the
 *   fp32 probabilities before the bf16 rounding of P).  workspace: caller-owned device memory
 *   of at least sparvar_dense_attn_mass_workspace() bytes, 16-byte aligned (per-row block sums
 *   and their reference maxima, and the LSE if lse is null).  Errors as for
 *   sparvar_predict_pattern; SPARVAR_ERR_CAPACITY if the workspace is too small.
 */
size_t sparvar_dense_attn_mass_workspace(const sparvar_schedule* sched, int32_t decision_scale,
                                         int32_t block, int32_t batch_heads);
sparvar_status sparvar_dense_attn_mass(const sparvar_schedule* sched, int32_t decision_scale,
                                       int32_t block, int32_t sink_scales,
                                       const sparvar_attn_shape* shape, const uint16_t* q_S,
                                       const uint16_t* k_cache, const uint16_t* v_cache,
                                       float softmax_scale, int32_t select_mode, int32_t topk,
                                       float threshold, uint16_t* o, float* lse, float* mass_out,
                                       uint32_t* mask_out, void* workspace, size_t workspace_bytes,
                                       void* stream);

/* NEXT(2) — token-granular CS4A, the paper's own CS4A granularity.
 *   Query blocks are query_block = C contiguous rows (C = 192 in the paper, PAPER.md:842;
 *   C in {64, 128, 192}); G_k = ceil(N_k / C).  Token bit rows: uint32 words, bit j%32 of word
 *   j/32 = key token j, ceil(C_k / 32) words per row.
 * sparvar_token_colsum: A[bh][g][j] = sum_{q in block g} P[q][j] over the keys j < C_S
 *    in fp32, P = softmax(Q_S K^T * scale); lse_S (fp32 [BH][N_S]) is the
 *   log-sum-exp of those rows, e.g. the lse output of sparvar_dense_attn at S.  colsum_out: fp32
 *   [BH][G_S][C_S].  K is read through the same shape/stride rules as the attention calls.
 * sparvar_token_select: per row g, the topk_tokens largest column sums (ties to the smaller j,
 *   k >= C_S keeps all) plus the sink tokens j < C_{sink_scales} -> mask_out [BH][G_S][W].
 * sparvar_token_map: target query block g_K reads source block phi(g_K); every
 *   selected source token is projected by Decompose-Align-Project (footprint or point mode,
 *   PAPER.md:853-881) and the sink tokens are added -> dst_mask [BH][G_K][ceil(C_K/32)].
 *   Compact it to per-block token lists with sparvar_build_block_lists(bh, G_K, C_K, ...).
 * sparvar_token_sparse_attn: rows of query block g attend exactly the listed tokens
 *   col_idx[row_ptr[bh*G_K+g] .. row_ptr[bh*G_K+g+1]) (ascending token indices < C_K):
 *   o = softmax(q K_J^T * scale) V_J, fp32 online softmax, bf16 out; empty lists give 0 rows.
 */
sparvar_status sparvar_token_colsum(const sparvar_schedule* sched, int32_t decision_scale,
                                    int32_t query_block, const sparvar_attn_shape* shape,
                                    const uint16_t* q_S, const uint16_t* k_cache,
                                    const float* lse_S, float softmax_scale, float* colsum_out,
                                    void* stream);
sparvar_status sparvar_token_select(const sparvar_schedule* sched, int32_t decision_scale,
                                    int32_t query_block, int32_t sink_scales, int32_t batch_heads,
                                    const float* colsum, int32_t topk_tokens, uint32_t* mask_out,
                                    void* stream);
sparvar_status sparvar_token_map(const sparvar_schedule* sched, int32_t src_scale,
                                 int32_t dst_scale, int32_t query_block, int32_t sink_scales,
                                 int32_t map_mode, int32_t batch_heads, const uint32_t* src_mask,
                                 uint32_t* dst_mask, void* stream);
sparvar_status sparvar_token_sparse_attn(const sparvar_schedule* sched, int32_t target_scale,
                                         int32_t query_block, const sparvar_attn_shape* shape,
                                         const uint16_t* q, const uint16_t* k_cache,
                                         const uint16_t* v_cache, const int32_t* row_ptr,
                                         const int32_t* col_idx, float softmax_scale, uint16_t* o,
                                         void* stream);
/* Token-level O_cache (PAPER.md:289-334 on the token path): sparvar_token_cache_residual runs
 *   the token-list attention at the decision scale over its own selection (lists of
 *   sparvar_token_select's rows) into o_cache and subtracts it from o_dense (the dense output at
 *   S) in place: o_cache = o_dense - Softmax(Q K_inds^T) V_inds.  sparvar_token_sparse_attn_cached
 *   is sparvar_token_sparse_attn with the nearest-neighbour upsampled o_cache (side of
 *   cache_scale, cache_stride_bh elements per (b,h)) added in its epilogue (READING 22); empty
 *   lists give the cache row.  Errors as for sparvar_cache_residual / _block_sparse_attn_cached.
 */
sparvar_status sparvar_token_cache_residual(const sparvar_schedule* sched, int32_t decision_scale,
                                            int32_t query_block, const sparvar_attn_shape* shape,
                                            const uint16_t* q_S, const uint16_t* k_cache,
                                            const uint16_t* v_cache, const int32_t* row_ptr_S,
                                            const int32_t* col_idx_S, float softmax_scale,
                                            const uint16_t* o_dense, uint16_t* o_cache,
                                            void* stream);
sparvar_status sparvar_token_sparse_attn_cached(
    const sparvar_schedule* sched, int32_t target_scale, int32_t query_block,
    const sparvar_attn_shape* shape, const uint16_t* q, const uint16_t* k_cache,
    const uint16_t* v_cache, const int32_t* row_ptr, const int32_t* col_idx, float softmax_scale,
    const uint16_t* o_cache, int32_t cache_scale, int64_t cache_stride_bh, uint16_t* o,
    void* stream);

/* NEXT(4) — compressed KV cache for CSLA layers ("retaining only sinks and local scales KV
 *   Cache"): a CSLA layer at target K reads only the sink scales (h <= sink_scales)
 *   and the scales with a window (windows[K - h] > 0); the compressed cache holds those scales'
 *   rows in scale order (READING 23).
 * sparvar_csla_kept_rows: its row count (-1 on invalid arguments).
 * sparvar_compress_kv: copies the kept rows of a full cache (rows C_{h-1}..C_h of every kept h,
 *   in_stride_bh elements per (b,h)) into cache_out (out_stride_bh >= kept rows * D), on stream.
 * sparvar_local_mask_compressed: sparvar_local_mask's block mask over the compressed index,
 *   [G_q][ceil(ceil(kept/block)/32)] words (blocks straddle kept scales as in the full cache).
 * sparvar_block_sparse_attn_rows: sparvar_block_sparse_attn over a cache of kv_rows valid rows
 *   (1 <= kv_rows <= C_K), e.g. the compressed cache with the compressed mask's lists.
 */
int64_t sparvar_csla_kept_rows(const sparvar_schedule* sched, int32_t target_scale,
                               int32_t sink_scales, const int32_t* windows, int32_t num_windows);
sparvar_status sparvar_compress_kv(const sparvar_schedule* sched, int32_t target_scale,
                                   int32_t sink_scales, const int32_t* windows,
                                   int32_t num_windows, int32_t batch_heads, int32_t head_dim,
                                   const uint16_t* cache_in, int64_t in_stride_bh,
                                   uint16_t* cache_out, int64_t out_stride_bh, void* stream);
sparvar_status sparvar_local_mask_compressed(const sparvar_schedule* sched, int32_t target_scale,
                                             int32_t block, int32_t sink_scales,
                                             const int32_t* windows, int32_t num_windows,
                                             uint32_t* mask_out, void* stream);
sparvar_status sparvar_block_sparse_attn_rows(const sparvar_schedule* sched,
                                              int32_t target_scale, int32_t block,
                                              const sparvar_attn_shape* shape, const uint16_t* q,
                                              const uint16_t* k_cache, const uint16_t* v_cache,
                                              int64_t kv_rows, const int32_t* row_ptr,
                                              const int32_t* col_idx, float softmax_scale,
                                              uint16_t* o, float* lse, void* stream);

/* NEXT(1) — cached block-sparse attention at scale K:
 *   O^(K) = Upsample(O_cache) + Delta O^(K), Delta O^(K) = sparvar_block_sparse_attn output.
 *   Upsample is nearest neighbour over the query grid: output query (x, y) of side s_K adds
 *   cache row (floor(x s_S / s_K), floor(y s_S / s_K)) of side s_S = side of cache_scale
 *   (READING 22).  The addition is fused into the attention epilogue (fp32, bf16 result); rows
 *   with an empty list get the cache row alone.  lse (nullable) is that of Delta O.
 *   o_cache: bf16 [BH][N_S][D] with cache_stride_bh elements between (b,h) slabs.
 */
sparvar_status sparvar_block_sparse_attn_cached(
    const sparvar_schedule* sched, int32_t target_scale, int32_t block,
    const sparvar_attn_shape* shape, const uint16_t* q, const uint16_t* k_cache,
    const uint16_t* v_cache, const int32_t* row_ptr, const int32_t* col_idx, float softmax_scale,
    const uint16_t* o_cache, int32_t cache_scale, int64_t cache_stride_bh, uint16_t* o, float* lse,
    void* stream);

/* Thread-local message for the last non-OK status of this thread ("" if none). */
const char* sparvar_last_error(void);

/* ABI version (major*100 + minor). */
int32_t sparvar_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SPARVAR_H_ */
