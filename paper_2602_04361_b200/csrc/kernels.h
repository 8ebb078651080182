// kernels.h — internal launch interface between api.cu (C ABI, validation, TMA descriptors) and
// the kernel translation units.  Not part of the public ABI (see include/sparvar.h).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace sv {

constexpr int kMaxScales = 32;
// attention kernel: a tile's KV step count is stored in 16 bits (attention.cu, Small::n);
// api.cu rejects ceil(n_kv / block) above this
constexpr int kMaxKvSteps = 65535;

// Scale geometry copied by value into kernels (a few hundred bytes of kernel parameters).
struct Geo {
  int K;                          // number of scales in the schedule
  int side[kMaxScales];           // s_1..s_K at [0..K)
  int cum[kMaxScales + 1];        // C_0..C_K at [0..K]
};

// ------------------------------------------------------------------ masks.cu
cudaError_t launch_local_mask(const Geo& g, int target, int block, int sink_scales,
                              const int* windows_rel /*[kMaxScales], index = target - h*/,
                              uint32_t* out, cudaStream_t st, bool compressed = false);
cudaError_t launch_map_indices(const Geo& g, int S, int K, int block, int sink_scales, int mode,
                               int bh, const uint32_t* src, uint32_t* dst, cudaStream_t st);
struct MaskSet {
  const uint32_t* ptr[8];
  int broadcast[8];
  int n;
};
cudaError_t launch_build_lists(int bh, int g_q, int g_kv, const MaskSet& ms, int* row_ptr,
                               int* col_idx, long long cap, int* status, cudaStream_t st);

// ------------------------------------------------------------------ attention.cu
struct AttnArgs {
  int n_q;            // N_K query rows per (b,h)
  int n_kv;           // C_K valid cache rows
  int g_q;            // ceil(N_K / block): CSR rows per (b,h)
  int bh;             // batch*heads
  const int* row_ptr; // nullptr -> dense (every block)
  const int* col_idx;
  float scale_log2;   // softmax_scale * log2(e)
  uint16_t* o;
  long long o_stride; // elements between (b,h) slabs of O
  float* lse;
  // optional NEXT(1) cache residual added in the epilogue: o += NN-upsample(add) (READING 22)
  const uint16_t* add;   // bf16 [bh][s_src*s_src][D] or nullptr
  long long add_stride;  // elements between (b,h) slabs of add
  int s_src, s_dst;      // query grid sides of the cache (S) and of the output (K)
  // optional NEXT(3) fused block mass (dense pass at the decision scale): per (bh, block v, row q)
  // at [(bh * g_kv + v) * n_q + q] the row's sum of 2^(x - m) over the block and that m
  float* mass_s;
  float* mass_m;
};
// NEXT(3): masses from the MASS pass (+ LSE) and top-k / threshold selection into bit rows
cudaError_t launch_mass_select(int bh, int n_q, int g_q, int g_kv, int B, const float* s,
                               const float* m, const float* lse, int mode, int topk, float tau,
                               int n_sink_blocks, float* mass_out, uint32_t* mask_out,
                               cudaStream_t st);
// o_cache = o_dense - o_sparse, bf16 in / out, fp32 arithmetic (NEXT(1))
cudaError_t launch_residual(int bh, int rows, int D, const uint16_t* dense, long long dense_stride,
                            const uint16_t* sparse, long long sparse_stride, uint16_t* out,
                            long long out_stride, cudaStream_t st);
cudaError_t launch_attention(int head_dim, int block, const CUtensorMap& tq, const CUtensorMap& tk,
                             const CUtensorMap& tv, const AttnArgs& a, cudaStream_t st);

// ------------------------------------------------------------------ NEXT(2): token-level CS4A
// masks.cu: top-k of column-sum rows -> token bit rows; token-level mapping S -> K
cudaError_t launch_topk_tokens(int rows, int n, int k_tok, int n_sink, const float* a,
                               uint32_t* out, cudaStream_t st);
cudaError_t launch_map_tokens(const Geo& g, int S, int K, int C, int sink_scales, int mode,
                              int bh, const uint32_t* src, uint32_t* dst, cudaStream_t st);
// token.cu: column sums at S (needs the LSE of the dense pass) and token-list attention at K
cudaError_t launch_colsum(int head_dim, int C, const CUtensorMap& tk, const CUtensorMap& tq,
                          int bh, int n_q, int n_kv, float scale_log2, const float* lse,
                          float* out, cudaStream_t st);
cudaError_t launch_token_attn(int head_dim, const CUtensorMap& tq, const uint16_t* k,
                              const uint16_t* v, long long kv_stride, int bh, int n_q, int C,
                              float scale_log2, const int* row_ptr, const int* col_idx,
                              uint16_t* o, long long o_stride, const uint16_t* add,
                              long long add_stride, int s_src, int s_dst, cudaStream_t st);

// ------------------------------------------------------------------ predictor.cu
struct PredArgs {
  int n_q;            // N_S
  int n_kv;           // C_S
  int g_q;            // ceil(N_S / block)
  int g_kv;           // ceil(C_S / block)
  int bh;
  float scale_log2;
  int mode;           // 0 top-k, 1 threshold
  int topk;
  float tau;
  int n_sink_blocks;  // ceil(C_sink / block)
  float* mass;        // nullable [bh][g_q][g_kv]
  uint32_t* mask;     // [bh][g_q][W]
};
// Returns cudaErrorInvalidValue if the statistics do not fit (caller maps it to UNSUPPORTED).
cudaError_t launch_predictor(int head_dim, int block, const CUtensorMap& tq, const CUtensorMap& tk,
                             const PredArgs& a, cudaStream_t st);
size_t predictor_smem_bytes(int head_dim, int block, int g_kv);

}  // namespace sv
