// Microbenchmark: does TMA traffic into shared memory slow tcgen05.mma that reads its operands
// from shared memory?  One CTA per SM: warp 0 issues NMMA back-to-back MMAs (SS M128 N128 K16,
// A+B = 8 KB of smem reads per MMA, or TS M128 N128 K16 with only B = 4 KB from smem); warp 1
// streams 32 KB TMA tiles from an L2-resident buffer into a separate 96 KB region (3-stage ring)
// for as long as warp 0 runs.  Reports clk per MMA and the TMA bytes per clock achieved.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_04361_b200/csrc \
//        bench_micro/smem_contention.cu -o bench_micro/smem_contention -lcuda
#include <cstdio>
#include <cuda.h>
#include "ptx.cuh"
using namespace sv;

constexpr int NMMA = 4096;

template <bool TS, bool TMA>
__global__ void __launch_bounds__(64, 1) k_cont(const __grid_constant__ CUtensorMap tm, long long* out,
                                              int rows_total) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar, full[3];
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 3; ++i) mbar_init(full + i, 1);
    stop = 0;
    fence_barrier_init();
  }
  if (warp == 0) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0 && threadIdx.x == 0) {
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    constexpr uint32_t idesc = idesc_bf16_f32(128, 128, 0, TS ? 1 : 0);
    for (int i = 0; i < 64; ++i) {
      const uint64_t da = sdesc_sw128(a + (i & 3) * 32, 16, 1024);
      const uint64_t db = sdesc_sw128(b + (i & 3) * 32, TS ? 128 * 128 : 16, 1024);
      if (TS) mma_ts(tmem + 256, tmem + (i & 7) * 8, db, idesc, 1);
      else mma_ss(tmem, da, db, idesc, 1);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t0 = clock64();
    for (int i = 0; i < NMMA; ++i) {
      const uint64_t da = sdesc_sw128(a + (i & 3) * 32, 16, 1024);
      const uint64_t db = sdesc_sw128(b + (i & 3) * 32, TS ? 128 * 128 : 16, 1024);
      if (TS) mma_ts(tmem + 256, tmem + (i & 7) * 8, db, idesc, 1);
      else mma_ss(tmem, da, db, idesc, 1);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 1);
    const long long t1 = clock64();
    stop = 1;
    out[2 * blockIdx.x] = t1 - t0;
  }
  if (TMA && warp == 1 && threadIdx.x == 32) {
    uint8_t* ring = sm + 65536;
    long long bytes = 0;
    const long long t0 = clock64();
    int i = 0;
    for (; !stop; ++i) {
      const int s = i % 3;
      if (i >= 3) mbar_wait(full + s, ((i / 3) - 1) & 1);
      const int row = ((blockIdx.x * 7 + i) * 128) % rows_total;
      mbar_arrive_expect_tx(full + s, 32768);
      tma_load_3d(ring + s * 32768, &tm, full + s, 0, row, 0);
      tma_load_3d(ring + s * 32768 + 16384, &tm, full + s, 64, row, 0);
      bytes += 32768;
    }
    for (int j = i - 3 > 0 ? i - 3 : 0; j < i; ++j) mbar_wait(full + j % 3, (j / 3) & 1);
    const long long t1 = clock64();
    out[2 * blockIdx.x + 1] = (long long)(bytes * 1000.0 / (double)(t1 - t0));   // milli-B per clk
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int rows = 8192 * 4;
  void* buf;
  cudaMalloc(&buf, (size_t)rows * 128 * 2);
  cudaMemset(buf, 0, (size_t)rows * 128 * 2);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[3] = {128, (cuuint64_t)rows, 1};
  cuuint64_t strides[2] = {256, (cuuint64_t)rows * 256};
  cuuint32_t box[3] = {64, 128, 1};
  cuuint32_t es[3] = {1, 1, 1};
  ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d;
  cudaMalloc(&d, 2 * 256 * sizeof(long long));
  auto run = [&](auto kern, const char* name) {
    const int smem = 65536 + 3 * 32768;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaMemset(d, 0, 2 * 256 * sizeof(long long));
    kern<<<sms, 64, smem>>>(tm, d, rows);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[512];
    cudaMemcpy(h, d, 2 * sms * sizeof(long long), cudaMemcpyDeviceToHost);
    double mma = 0, tma = 0;
    for (int i = 0; i < sms; ++i) { mma += h[2 * i]; tma += h[2 * i + 1]; }
    mma /= sms; tma /= sms;
    printf("%-28s %s: %.1f clk/MMA (ideal 64), smem read by MMA %.0f B/clk, TMA %.1f B/clk\n", name,
           e == cudaSuccess ? "ok" : cudaGetErrorString(e), mma / NMMA,
           (name[0] == 'S' ? 8192.0 : 4096.0) / (mma / NMMA), tma / 1000.0);
  };
  run(k_cont<false, false>, "SS M128 N128 alone");
  run(k_cont<false, true>, "SS M128 N128 + TMA stream");
  run(k_cont<true, false>, "TS M128 N128 alone");
  run(k_cont<true, true>, "TS M128 N128 + TMA stream");
  return 0;
}
