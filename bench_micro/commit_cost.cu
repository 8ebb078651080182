// Microbenchmark: tensor-pipe cost of tcgen05.commit.  One CTA per SM, one thread issues groups of
// 8 SS MMAs (M128 N128 K16, 512 clk of tensor work) followed by NC commits to distinct mbarriers
// that nobody waits on (MID: one of them between the two halves of the group instead).
// Reports clk per group (ideal 512).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_04361_b200/csrc \
//        bench_micro/commit_cost.cu -o bench_micro/commit_cost
#include <cstdio>
#include "ptx.cuh"
using namespace sv;

template <int NC, bool MID, bool TS>
__global__ void __launch_bounds__(32, 1) k_commit(long long* out, int groups) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bars[8], done;
  __shared__ uint32_t tslot;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(bars + i, 1);
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  tmem_alloc(&tslot, 512);
  tmem_relinquish();
  tc_fence_before();
  __syncwarp();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    constexpr uint32_t idesc = idesc_bf16_f32(128, 128, 0, TS ? 1 : 0);
    const long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t da = sdesc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
        const uint64_t db = sdesc_sw128(b + (kk >> 2) * 16384 + (kk & 3) * 32, TS ? 16384 : 16, 1024);
        if (TS) mma_ts(tmem + 256 + (g & 1) * 128, tmem + kk * 8, db, idesc, kk > 0);
        else mma_ss(tmem + (g & 1) * 128, da, db, idesc, kk > 0);
        if (MID && kk == 3) mma_commit(bars + 7);
      }
      for (int c = 0; c < NC - (MID ? 1 : 0); ++c) mma_commit(bars + c);
    }
    mma_commit(&done);
    mbar_wait(&done, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncwarp();
  tc_fence_after();
  tmem_dealloc(tmem, 512);
}

template <int NC, bool MID, bool TS>
void run(const char* name) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d; cudaMalloc(&d, 256 * sizeof(long long));
  auto k = k_commit<NC, MID, TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int groups = 2000;
  k<<<sms, 32, 100 * 1024>>>(d, groups);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[256]; cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < sms; ++i) avg += h[i]; avg /= sms;
  printf("%-40s %s: %.1f clk per group of 8 MMAs (ideal 512)\n", name,
         e == cudaSuccess ? "ok" : cudaGetErrorString(e), avg / groups);
  cudaFree(d);
}

int main() {
  run<0, false, false>("SS, no commit");
  run<1, false, false>("SS, 1 commit per group");
  run<2, false, false>("SS, 2 commits per group");
  run<3, false, false>("SS, 3 commits per group");
  run<2, true, false>("SS, 1 mid-group + 1 end commit");
  run<0, false, true>("TS, no commit");
  run<1, false, true>("TS, 1 commit per group");
  run<3, false, true>("TS, 3 commits per group");
  return 0;
}
