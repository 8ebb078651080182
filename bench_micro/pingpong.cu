// Microbenchmark: mbarrier hand-off latency between two warps of a CTA (arrive -> observed by a
// waiter in another warp), with try_wait (may suspend) and test_wait (pure polling); also the
// tcgen05.commit -> waiter latency after a single MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_04361_b200/csrc \
//        bench_micro/pingpong.cu -o bench_micro/pingpong
#include <cstdio>
#include "ptx.cuh"
using namespace sv;

template <bool POLL>
__device__ __forceinline__ void wait_(uint64_t* b, uint32_t par) {
  if (POLL) mbar_wait_spin(b, par); else mbar_wait(b, par);
}

template <bool POLL>
__global__ void k_pp(long long* out, int iters) {
  __shared__ uint64_t x, y;
  if (threadIdx.x == 0) { mbar_init(&x, 1); mbar_init(&y, 1); fence_barrier_init(); }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane != 0) return;
  if (warp == 0) {
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      mbar_arrive(&x);
      wait_<POLL>(&y, i & 1);
    }
    out[0] = (clock64() - t0) / iters;
  } else if (warp == 1) {
    for (int i = 0; i < iters; ++i) {
      wait_<POLL>(&x, i & 1);
      mbar_arrive(&y);
    }
  }
}

// thread 0: issue 1 MMA + commit, wait for it (its own commit), repeat: round trip per MMA
template <bool POLL>
__global__ void k_commit(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  tmem_alloc(&tslot, 512);
  tmem_relinquish();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    constexpr uint32_t idq = idesc_bf16_f32(128, 128, 0, 0);
    const uint64_t da = sdesc_sw128(a, 16, 1024), db = sdesc_sw128(b, 16, 1024);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      mma_ss(tslot, da, db, idq, 1);
      mma_commit(&bar);
      wait_<POLL>(&bar, i & 1);
    }
    out[0] = (clock64() - t0) / iters;
  }
  __syncwarp();
  tc_fence_after();
  tmem_dealloc(tslot, 512);
}

int main() {
  long long* d; cudaMalloc(&d, 64);
  long long h;
  k_pp<false><<<1, 64>>>(d, 10000); cudaDeviceSynchronize(); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("mbarrier ping-pong round trip, try_wait : %lld clk\n", h);
  k_pp<true><<<1, 64>>>(d, 10000); cudaDeviceSynchronize(); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("mbarrier ping-pong round trip, test_wait: %lld clk\n", h);
  cudaFuncSetAttribute(k_commit<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(k_commit<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k_commit<false><<<1, 32, 100 * 1024>>>(d, 2000); cudaDeviceSynchronize(); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("1 MMA + commit + wait (try_wait) : %lld clk\n", h);
  k_commit<true><<<1, 32, 100 * 1024>>>(d, 2000); cudaDeviceSynchronize(); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("1 MMA + commit + wait (test_wait): %lld clk\n", h);
  return 0;
}
