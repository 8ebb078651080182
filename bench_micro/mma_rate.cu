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
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); stop = 0; }
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
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        mma_ss(tmem, sdesc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
               sdesc_sw128(b + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), idq, kk > 0);
      mma_commit(&bar);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        mma_ts(tmem + 256, tmem + kk * 8, sdesc_sw128(b + kk * 2048, 16384, 1024), idp, 1);
      mma_commit(&bar);
      if (MODE & 4) { mbar_wait(&bar, 1); }   // two commits per iteration: parity returns
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
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
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
  run_mix<0>("mix SS8+TS8", sms);
  run_mix<1>("mix + LDTM background", sms);
  run_mix<3>("mix + LDTM/STTM background", sms);
  run_mix<4>("mix, wait each iteration", sms);
  return 0;
}
