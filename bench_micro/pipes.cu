// Microbenchmark: latency of tcgen05.ld (TMEM -> registers) and throughput of MUFU.EX2,
// FFMA2 and F2FP per SM sub-partition, measured with clock64 on one SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_04361_b200/csrc \
//        bench_micro/pipes.cu -o bench_micro/pipes
#include <cstdio>
#include "ptx.cuh"
using namespace sv;

__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

__global__ void __launch_bounds__(128, 1) k_ldtm(long long* out, int iters) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t_row = tslot + (uint32_t(warp * 32) << 16);
  uint32_t r[128];
  uint32_t acc = 0;
  // 1 x32 load + wait
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    tmem_ld32(t_row + (i & 3) * 32, r);
    tmem_wait_ld();
    acc += r[0] ^ r[31];
  }
  long long t1 = clock64();
  // 4 x32 loads + one wait
  for (int i = 0; i < iters; ++i) {
    tmem_ld32(t_row + 0, r);
    tmem_ld32(t_row + 32, r + 32);
    tmem_ld32(t_row + 64, r + 64);
    tmem_ld32(t_row + 96, r + 96);
    tmem_wait_ld();
    acc += r[0] ^ r[127] ^ r[64];
  }
  long long t2 = clock64();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / iters; out[1] = (t2 - t1) / iters; out[9] = acc; }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tslot, 512); }
}

// warps_per_smsp warps on each of the 4 SMSPs run n MUFU.EX2 (independent chains of 8)
template <int OP>
__global__ void k_pipe(long long* out, int iters, float seed) {
  float x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = seed * (threadIdx.x + k) * 1e-6f;
  uint64_t y[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) { float a = x[k]; asm("mov.b64 %0, {%1,%1};" : "=l"(y[k]) : "f"(a)); }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) x[k] = ex2(x[k] * 0.999f);          // MUFU + FMUL
      if (OP == 1) y[k] = ffma2(y[k], y[k], y[k]);     // FFMA2
      if (OP == 2) { uint32_t p = pack_bf16x2(x[k], x[k] + 1.f); x[k] = __uint_as_float(p); }
      if (OP == 3) x[k] = fmaf(x[k], x[k], x[k]);      // FFMA
    }
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(y[k])); s += x[k] + a + b; }
  if (threadIdx.x == 0) out[0] = t1 - t0;
  if (s == 12345.f) out[1] = 1;
}

int main() {
  long long* d; cudaMalloc(&d, 64 * sizeof(long long));
  long long h[16];
  k_ldtm<<<1, 128>>>(d, 1000);
  cudaDeviceSynchronize();
  cudaMemcpy(h, d, 16 * sizeof(long long), cudaMemcpyDeviceToHost);
  printf("LDTM x32 + wait: %lld clk;  4 x LDTM x32 + wait: %lld clk\n", h[0], h[1]);
  const char* names[4] = {"MUFU.EX2(+FMUL)", "FFMA2", "F2FP.BF16x2", "FFMA"};
  for (int op = 0; op < 4; ++op) {
    for (int wps : {1, 2, 4}) {
      const int threads = 128 * wps;   // wps warps per SMSP
      const int iters = 1000;
      if (op == 0) k_pipe<0><<<1, threads>>>(d, iters, 1.f);
      if (op == 1) k_pipe<1><<<1, threads>>>(d, iters, 1.f);
      if (op == 2) k_pipe<2><<<1, threads>>>(d, iters, 1.f);
      if (op == 3) k_pipe<3><<<1, threads>>>(d, iters, 1.f);
      cudaDeviceSynchronize();
      cudaMemcpy(h, d, 2 * sizeof(long long), cudaMemcpyDeviceToHost);
      printf("%-18s %d warps/SMSP: %.2f clk per warp-instruction per SMSP\n", names[op], wps,
             (double)h[0] / (iters * 8.0 * wps));
    }
  }
  return 0;
}
