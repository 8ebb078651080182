// Microbenchmark: does a MUFU.EX2 stream from other warps slow tcgen05.mma issue/execution?
// One CTA per SM, 9 warps.  Warp 0 issues the attention op mix back to back (8 SS M128 N128 K16
// into S + 8 TS into O, one commit each) for `iters` ops; warps 1..8 (two per SM sub-partition,
// like the two slots' softmax warps) run a background stream until warp 0 is done:
//   MODE 0 idle, 1 MUFU.EX2 on all 8, 2 FFMA2 on all 8, 3 MUFU on warps off sub-partition 0,
//   4 MUFU on sub-partition 0 only (warps 4 and 8, beside the issuer), 5 MUFU on one warp per
//   sub-partition (warps 1..4).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_04361_b200/csrc \
//        bench_micro/mma_mufu.cu -o bench_micro/mma_mufu
#include <cstdio>
#include "ptx.cuh"
#include "kernel_util.cuh"
using namespace sv;

template <int MODE>
__global__ void __launch_bounds__(288, 1) k_mm(long long* out, float* sink, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar, fin;
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&fin, 1); fence_barrier_init(); stop = 0; }
  if (warp == 0) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0) {
    if (lane == 0) {
      const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
      constexpr uint32_t idq = idesc_bf16_f32(128, 128, 0, 0);
      constexpr uint32_t idp = idesc_bf16_f32(128, 128, 0, 1);
      const long long t0 = clock64();
      for (int it = 0; it < iters; ++it) {
        const uint32_t bs = b + (it & 3) * 32768u;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ts(tmem + 256, tmem + kk * 8, sdesc_sw128(bs + kk * 2048, 16384, 1024), idp, 1);
        mma_commit(&bar);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ss(tmem, sdesc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                 sdesc_sw128(bs + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), idq, kk > 0);
        mma_commit(&bar);
      }
      mma_commit(&fin);
      mbar_wait(&fin, 0);
      const long long t1 = clock64();
      out[blockIdx.x] = t1 - t0;
      stop = 1;
    }
  } else {
    const int sp = warp & 3;
    bool on = false;
    if (MODE == 1 || MODE == 2) on = true;
    if (MODE == 3) on = sp != 0;
    if (MODE == 4) on = sp == 0;
    if (MODE == 5) on = warp <= 4;
    if (on) {
      float x[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = -0.001f * (lane + i);
      uint64_t y[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) y[i] = f2_pack(x[2 * i], x[2 * i + 1]);
      const uint64_t c = f2_pack(0.999f, 0.999f);
      while (!stop) {
#pragma unroll 4
        for (int r = 0; r < 64; ++r) {
          if (MODE == 2) {
#pragma unroll
            for (int i = 0; i < 4; ++i) y[i] = ffma2(y[i], c, c);
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = ex2(x[i]) - 1.0f;
          }
        }
      }
      float s = 0.f;
      for (int i = 0; i < 8; ++i) s += x[i];
      float y0, y1;
      f2_unpack(y[0], y0, y1);
      sink[blockIdx.x * 288 + threadIdx.x] = s + y0 + y1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

// Latency of mbarrier.test_wait / try_wait on an already-completed barrier (and of a plain
// shared-memory load), timed by warp 1 while warp 0 keeps the tensor pipe busy with SS MMAs
// (BUSY = 1), TS MMAs (BUSY = 2) or idle (BUSY = 0).
template <int BUSY>
__global__ void __launch_bounds__(64, 1) k_lat(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t done;
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  __shared__ volatile int word;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { mbar_init(&done, 1); fence_barrier_init(); stop = 0; word = 1; }
  __syncthreads();
  if (threadIdx.x == 0) mbar_arrive(&done);   // phase 0 completes
  if (warp == 0) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0) {
    if (lane == 0 && BUSY) {
      const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
      constexpr uint32_t idq = idesc_bf16_f32(128, 128, 0, 0);
      constexpr uint32_t idp = idesc_bf16_f32(128, 128, 0, 1);
      while (!stop) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if (BUSY == 1)
            mma_ss(tmem, sdesc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                   sdesc_sw128(b + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), idq, 1);
          else
            mma_ts(tmem + 256, tmem + kk * 8, sdesc_sw128(b + kk * 2048, 16384, 1024), idp, 1);
        }
      }
    }
  } else {
    const uint32_t bar = smem_u32(&done);
    long long tt = 0, tr = 0, tl = 0;
    int acc = 0;
    for (int i = 0; i < iters; ++i) {
      long long t0 = clock64();
      acc += mbar_test_wait(bar, 0) ? 1 : 0;
      long long t1 = clock64();
      acc += mbar_try_wait(bar, 0) ? 1 : 0;
      long long t2 = clock64();
      acc += word;
      long long t3 = clock64();
      tt += t1 - t0; tr += t2 - t1; tl += t3 - t2;
    }
    if (lane == 0) {
      out[blockIdx.x * 4 + 0] = tt / iters;
      out[blockIdx.x * 4 + 1] = tr / iters;
      out[blockIdx.x * 4 + 2] = tl / iters;
      out[blockIdx.x * 4 + 3] = acc;
      stop = 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int BUSY>
void run_lat(const char* name, int sms) {
  long long* d; cudaMalloc(&d, sizeof(long long) * sms * 4);
  auto k = k_lat<BUSY>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k<<<sms, 64, 200 * 1024>>>(d, 2000);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[1024]; cudaMemcpy(h, d, sizeof(long long) * sms * 4, cudaMemcpyDeviceToHost);
  printf("%-28s %s: test_wait %lld  try_wait %lld  ld.shared %lld clk (incl. clock reads)\n", name,
         e == cudaSuccess ? "ok" : cudaGetErrorString(e), h[0], h[1], h[2]);
  cudaFree(d);
}

template <int MODE>
void run(const char* name, int sms) {
  const int iters = 512;
  long long* d; cudaMalloc(&d, sizeof(long long) * sms);
  float* s; cudaMalloc(&s, sizeof(float) * sms * 288);
  auto k = k_mm<MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int rep = 0; rep < 2; ++rep) k<<<sms, 288, 200 * 1024>>>(d, s, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[256]; cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < sms; ++i) avg += h[i]; avg /= sms;
  printf("%-44s %s: %.1f clk per op of 16 MMAs (ideal 1024)\n", name,
         e == cudaSuccess ? "ok" : cudaGetErrorString(e), avg / iters);
  cudaFree(d); cudaFree(s);
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("background idle", sms);
  run<1>("MUFU.EX2 on 8 warps (2 per sub-partition)", sms);
  run<2>("FFMA2 on 8 warps", sms);
  run<3>("MUFU on the 6 warps off the issuer's SMSP", sms);
  run<4>("MUFU on the 2 warps beside the issuer", sms);
  run<5>("MUFU on 4 warps (1 per sub-partition)", sms);
  run_lat<0>("barrier latency, pipe idle", sms);
  run_lat<1>("barrier latency, SS MMAs", sms);
  run_lat<2>("barrier latency, TS MMAs", sms);
  return 0;
}
