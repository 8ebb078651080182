// Microbenchmark: issue rate of tcgen05.mma kind::f16 (bf16 -> fp32) on one SM, back to back,
// for the shapes the attention kernel uses.  Operands are uninitialised smem (values do not
// matter for timing).  One CTA per SM on all SMs, reports clk per MMA instruction.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_04361_b200/csrc \
//        bench_micro/mma_rate.cu -o bench_micro/mma_rate -lcuda
#include <cstdio>
#include "ptx.cuh"
using namespace sv;

template <int N, bool TS, int NMMA>
__global__ void __launch_bounds__(128, 1) k_rate(long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    constexpr uint32_t idesc = idesc_bf16_f32(128, N, 0, TS ? 1 : 0);
    // warm up
    for (int i = 0; i < 64; ++i) {
      const uint64_t da = sdesc_sw128(a + (i & 7) * 32, 16, 1024);
      const uint64_t db = sdesc_sw128(b + (i & 7) * 32, TS ? N * 128 : 16, 1024);
      if (TS) mma_ts(tmem + 256, tmem + (i & 7) * 8, db, idesc, 1);
      else mma_ss(tmem, da, db, idesc, 1);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t0 = clock64();
    for (int i = 0; i < NMMA; ++i) {
      const uint64_t da = sdesc_sw128(a + (i & 7) * 32, 16, 1024);
      const uint64_t db = sdesc_sw128(b + (i & 7) * 32, TS ? N * 128 : 16, 1024);
      if (TS) mma_ts(tmem + 256, tmem + (i & 7) * 8, db, idesc, 1);
      else mma_ss(tmem, da, db, idesc, 1);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 1);
    const long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

// Attention-like mix: per iteration 8 SS MMAs (S = Q K^T into cols [0,128)) + commit, then 8 TS
// MMAs (O += P V, P from TMEM cols [0,64), O at [256,384)) + commit.  Optional background TMEM
// traffic from 4 other warps (LDTM of cols [128,256) and STTM back), like a softmax warpgroup.
template <int MODE>
__global__ void __launch_bounds__(160, 1) k_mix(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  __shared__ uint64_t done;
  __shared__ uint64_t never;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&done, 1); mbar_init(&never, 1); fence_barrier_init(); stop = 0; }
  __syncthreads();
  if (threadIdx.x == 0) mbar_arrive(&done);   // phase 0 of `done` completes immediately
  if (warp == 0) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    constexpr uint32_t idq = idesc_bf16_f32(128, 128, 0, 0);
    constexpr uint32_t idp = idesc_bf16_f32(128, 128, 0, 1);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t bs = (MODE & 32) ? b + (it & 3) * 32768u : b;   // rotate 4 "stages"
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        mma_ss(tmem, sdesc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
               sdesc_sw128(bs + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), idq, kk > 0);
      mma_commit(&bar);
      if (MODE & 16) { mbar_wait(&done, 0); tc_fence_after(); }
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        mma_ts(tmem + 256, tmem + kk * 8, sdesc_sw128(((MODE & 32) ? b + ((it + 2) & 3) * 32768u : b) + kk * 2048, 16384, 1024), idp, 1);
      mma_commit(&bar);
      if (MODE & 4) { mbar_wait(&bar, 1); }   // two commits per iteration: parity returns
      if (MODE & 8) { mbar_wait(&done, 0); tc_fence_after(); }   // completed barrier + fence
    }
    mma_commit(&bar);
    const long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    stop = 1;
  } else if (warp >= 1 && (MODE & 3)) {
    const uint32_t trow = tmem + (uint32_t(((warp - 1) & 3) * 32) << 16);
    uint32_t r[32];
    while (!stop) {
      if (MODE & 1) { tmem_ld32(trow + 128, r); tmem_wait_ld(); }
      if (MODE & 2) { tmem_st32(trow + 160, r); tmem_wait_st(); }
    }
  } else if (warp >= 1 && (MODE & 64)) {
    // background warps polling an mbarrier phase that never completes (like waiting softmax warps)
    const uint32_t nb = smem_u32(&never);
    while (!stop) {
      if (mbar_try_wait(nb, 0)) break;
      if (MODE & 128) { if (lane == 0) { } }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

// LDTM latency while the tensor pipe is busy: thread 0 keeps issuing SS MMAs into columns
// [0,128); warps 1-4 time "4 x tcgen05.ld 32x32b.x32 of columns [256,384) + wait::ld".
__global__ void __launch_bounds__(160, 1) k_ldtm_under_mma(long long* out, int iters, int busy) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) stop = 0;
  if (warp == 0) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    constexpr uint32_t idq = idesc_bf16_f32(128, 128, 0, 0);
    while (!stop && busy) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        mma_ss(tmem, sdesc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
               sdesc_sw128(b + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), idq, kk > 0);
    }
  } else if (warp >= 1) {
    const uint32_t trow = tmem + (uint32_t(((warp - 1) & 3) * 32) << 16);
    uint32_t r[128];
    uint32_t acc = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      tmem_ld32(trow + 256, r);
      tmem_ld32(trow + 288, r + 32);
      tmem_ld32(trow + 320, r + 64);
      tmem_ld32(trow + 352, r + 96);
      tmem_wait_ld();
      acc += r[0] ^ r[127];
    }
    long long t1 = clock64();
    if (lane == 0 && warp == 1) { out[blockIdx.x] = (t1 - t0) / iters; out[200 + blockIdx.x] = acc; }
    __syncwarp();
    if (warp == 1 && lane == 0) stop = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

// Attention-kernel MMA sequence without any waits: two slots (S at cols 0 / 128, O at 256 /
// 384, Q buffers 0 / 32 KB), K/V stages rotating over 4 x 32 KB; per round and slot:
// PV (8 TS into O_t, P = S_t cols), QK (8 SS into S_t), commits like the kernel.
template <int MODE_SEQ>
__global__ void __launch_bounds__(128, 1) k_attn_seq(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) mbar_init(bar + i, 1); fence_barrier_init(); }
  if (warp == 0) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t q0 = smem_u32(sm), kv = smem_u32(sm + 65536);
    constexpr uint32_t idq = idesc_bf16_f32(128, 128, 0, 0);
    constexpr uint32_t idp = idesc_bf16_f32(128, 128, 0, 1);
    int st = 0;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int t = 0; t < 2; ++t) {
        const uint32_t vb = kv + (st & 3) * 32768u; ++st;
        for (int kk = 0; kk < 8; ++kk)
          mma_ts(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, sdesc_sw128(vb + kk * 2048, 16384, 1024), idp, kk > 0 || it > 0);
        mma_commit(bar + 0);
        if (MODE_SEQ & 1) { mma_commit(bar + 1); mma_commit(bar + 2); }
        const uint32_t kb = kv + (st & 3) * 32768u; ++st;
        const uint32_t qb = q0 + t * 32768u;
        for (int kk = 0; kk < 8; ++kk)
          mma_ss(tmem + t * 128, sdesc_sw128(qb + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                 sdesc_sw128(kb + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), idq, kk > 0);
        mma_commit(bar + 1);
        mma_commit(bar + 2 + t);
      }
    }
    mma_commit(bar + 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

// tcgen05.mma issue queue depth: time each issue return of 24 back-to-back MMAs on an idle pipe
__global__ void __launch_bounds__(32, 1) k_qdepth(long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  tmem_alloc(&tslot, 512);
  tmem_relinquish();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    constexpr uint32_t idq = idesc_bf16_f32(128, 128, 0, 0);
    long long t[25];
    const uint64_t da = sdesc_sw128(a, 16, 1024), db = sdesc_sw128(b, 16, 1024);
    t[0] = clock64();
#pragma unroll
    for (int i = 0; i < 24; ++i) {
      mma_ss(tslot, da + (i & 3) * 2, db + (i & 3) * 2, idq, 1);
      t[i + 1] = clock64();
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long te = clock64();
    for (int i = 0; i < 25; ++i) out[i] = t[i] - t[0];
    out[25] = te - t[0];
  }
  __syncwarp();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tslot, 512);
}

template <int MODE>
void run_mix(const char* name, int sms) {
  const int iters = 256;
  long long* d; cudaMalloc(&d, sizeof(long long) * sms);
  auto k = k_mix<MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k<<<sms, 160, 200 * 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[256]; cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < sms; ++i) avg += h[i]; avg /= sms;
  printf("%-34s %s: %.1f clk per 16 MMAs (ideal 1024)\n", name,
         e == cudaSuccess ? "ok" : cudaGetErrorString(e), avg / iters);
  cudaFree(d);
}

template <int N, bool TS>
void run(const char* name, int sms) {
  constexpr int NMMA = 4096;
  long long* d; cudaMalloc(&d, sizeof(long long) * sms);
  auto k = k_rate<N, TS, NMMA>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k<<<sms, 128, 200 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[256]; cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < sms; ++i) avg += h[i]; avg /= sms;
  const double flop = 2.0 * 128 * N * 16;
  printf("%-22s %s: %.1f clk/MMA  -> %.0f flop/clk/SM (nominal 8192)\n", name,
         e == cudaSuccess ? "ok" : cudaGetErrorString(e), avg / NMMA, flop / (avg / NMMA));
  cudaFree(d);
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<128, false>("SS M128 N128 (QK)", 1);
  run<128, false>("SS M128 N128 all SMs", sms);
  run<256, false>("SS M128 N256", sms);
  run<64, false>("SS M128 N64", sms);
  run<128, true>("TS M128 N128 (PV)", sms);
  run<256, true>("TS M128 N256", sms);
  {
    long long* d; cudaMalloc(&d, sizeof(long long) * 32);
    cudaFuncSetAttribute(k_qdepth, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    k_qdepth<<<1, 32, 100 * 1024>>>(d);
    cudaDeviceSynchronize();
    long long h[26]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("issue-return times of 24 back-to-back MMAs (clk):");
    for (int i = 1; i < 25; ++i) printf(" %lld", h[i]);
    printf("  | all complete at %lld\n", h[25]);
    cudaFree(d);
  }
  for (int busy = 0; busy < 2; ++busy) {
    long long* d; cudaMalloc(&d, sizeof(long long) * 512);
    cudaFuncSetAttribute(k_ldtm_under_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    k_ldtm_under_mma<<<sms, 160, 200 * 1024>>>(d, 2000, busy);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < sms; ++i) avg += h[i]; avg /= sms;
    printf("4 x LDTM.x32 + wait, tensor pipe %s: %.0f clk (%s)\n", busy ? "busy" : "idle", avg,
           e == cudaSuccess ? "ok" : cudaGetErrorString(e));
    cudaFree(d);
  }
  {
    long long* d; cudaMalloc(&d, sizeof(long long) * 256);
    cudaFuncSetAttribute(k_attn_seq<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_attn_seq<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int iters = 256;
    k_attn_seq<1><<<sms, 128, 200 * 1024>>>(d, iters);
    cudaDeviceSynchronize();
    { long long h[148]; cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
      double avg = 0; for (int i = 0; i < sms; ++i) avg += h[i]; avg /= sms;
      printf("attention MMA sequence, 3 commits after PV: %.1f clk per round (ideal 2048)\n", avg / iters); }
    k_attn_seq<0><<<sms, 128, 200 * 1024>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < sms; ++i) avg += h[i]; avg /= sms;
    printf("attention MMA sequence (2 slots, no waits): %.1f clk per round of 32 MMAs (ideal 2048) %s\n",
           avg / iters, e == cudaSuccess ? "ok" : cudaGetErrorString(e));
    cudaFree(d);
  }
  run_mix<0>("mix SS8+TS8", sms);
  run_mix<1>("mix + LDTM background", sms);
  run_mix<3>("mix + LDTM/STTM background", sms);
  run_mix<4>("mix, wait each iteration", sms);
  run_mix<8>("mix + done-wait/fence per iteration", sms);
  run_mix<32>("mix, B rotating over 4 stages", sms);
  run_mix<64>("mix + 4 warps polling an mbarrier", sms);
  run_mix<24>("mix + done-wait/fence x2 per iteration", sms);
  return 0;
}
