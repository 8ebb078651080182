// Microbenchmark: TMA (cp.async.bulk.tensor) load throughput into shared memory, per SM and
// chip-wide, for 128 x 128 bf16 tiles (2 boxes of 64 x 128, SWIZZLE_128B) from an
// L2-resident buffer — the K/V stage shape of the attention kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_04361_b200/csrc \
//        bench_micro/tma_rate.cu -o bench_micro/tma_rate -lcuda
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include "ptx.cuh"
using namespace sv;

template <int NST>
__global__ void __launch_bounds__(64, 1) k_tma(const __grid_constant__ CUtensorMap tm, long long* out,
                                              int iters, int rows_total) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[NST];
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) mbar_init(full + i, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const long long t0 = clock64();
    for (int i = 0; i < iters + NST; ++i) {
      const int s = i % NST;
      if (i >= NST) mbar_wait(full + s, ((i / NST) - 1) & 1);
      if (i < iters) {
        const int row = (int)((((long long)blockIdx.x * 7919 + (long long)i * 148) * 128) % rows_total);
        mbar_arrive_expect_tx(full + s, 32768);
        tma_load_3d(sm + s * 32768, &tm, full + s, 0, row, 0);
        tma_load_3d(sm + s * 32768 + 16384, &tm, full + s, 64, row, 0);
      }
    }
    out[blockIdx.x] = clock64() - t0;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  // default 8 MB of bf16 x 128 (L2-resident); argv[1] = MB for a DRAM-resident buffer
  const int mb = argc > 1 ? atoi(argv[1]) : 8;
  const int rows = mb * 4096;
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
  long long* d;
  cudaMalloc(&d, 256 * sizeof(long long));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 2000;
  auto run = [&](auto kern, int nst, int grid) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, nst * 32768);
    kern<<<grid, 64, nst * 32768>>>(tm, d, iters, rows);  // warm
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<grid, 64, nst * 32768>>>(tm, d, iters, rows);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long h[256]; cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < grid; ++i) avg += h[i]; avg /= grid;
    printf("NST %d grid %3d %s: %.1f B/clk/SM, chip %.2f TB/s\n", nst, grid,
           err == cudaSuccess ? "ok" : cudaGetErrorString(err), 32768.0 * iters / avg,
           32768.0 * iters * grid / (ms * 1e-3) / 1e12);
  };
  run(k_tma<2>, 2, 1); run(k_tma<4>, 4, 1); run(k_tma<6>, 6, 1);
  run(k_tma<2>, 2, sms); run(k_tma<4>, 4, sms); run(k_tma<6>, 6, sms);
  return 0;
}
