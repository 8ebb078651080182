// Microbenchmark: the attention MMA pipeline with its real cross-warp handshake but no softmax
// math and no loads, to measure what the barrier round trips cost the tensor pipe.
//   one tile, double-buffered S (v3 order): QK(0), QK(1), then per step g: [wait P(g)] PV(g),
//   QK(g+2); "softmax" warps 1..4 wait S(g) (commit), tcgen05.ld it, arrive P(g).
//   MODE bit 0: softmax warps skip the tcgen05.ld.  bit 1: MMA issuer polls (test_wait).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_04361_b200/csrc \
//        bench_micro/handshake.cu -o bench_micro/handshake
#include <cstdio>
#include "ptx.cuh"
using namespace sv;

template <int MODE, int NB>
__global__ void __launch_bounds__(160, 1) k_hs(long long* out, int steps) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t s_full[NB], p_full[NB];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NB; ++i) { mbar_init(s_full + i, 1); mbar_init(p_full + i, 128); }
    fence_barrier_init();
  }
  if (warp == 0) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0) {
    const uint32_t q = smem_u32(sm), kv = smem_u32(sm + 32768);
    constexpr uint32_t idq = idesc_bf16_f32(128, 128, 0, 0);
    constexpr uint32_t idp = idesc_bf16_f32(128, 128, 0, 1);
    const bool leader = lane == 0;
    auto qk = [&](int g) {
      const uint32_t buf = g % NB;
      const uint32_t kb = kv + (g % 4) * 32768u;
      if (leader) {
        for (int kk = 0; kk < 8; ++kk)
          mma_ss(tmem + buf * 128, sdesc_sw128(q + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                 sdesc_sw128(kb + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), idq, kk > 0);
        mma_commit(s_full + buf);
      }
      __syncwarp();
    };
    const long long t0 = clock64();
    for (int i = 0; i < NB; ++i) qk(i);
    for (int g = 0; g < steps; ++g) {
      const uint32_t buf = g % NB;
      if (MODE & 2) mbar_wait_spin(p_full + buf, (g / NB) & 1);
      else mbar_wait(p_full + buf, (g / NB) & 1);
      tc_fence_after();
      const uint32_t vb = kv + ((g + 2) % 4) * 32768u;
      if (leader) {
        for (int kk = 0; kk < 8; ++kk)
          mma_ts(tmem + 256, tmem + buf * 128 + kk * 8, sdesc_sw128(vb + kk * 2048, 16384, 1024), idp,
                 1);
      }
      __syncwarp();
      if (g + NB < steps) qk(g + NB);
    }
    if (leader) { mma_commit(p_full); }
    if (lane == 0) out[blockIdx.x] = clock64() - t0;
  } else {
    const uint32_t trow = tmem + (uint32_t(((warp - 1) & 3) * 32) << 16);
    for (int g = 0; g < steps; ++g) {
      const uint32_t buf = g % NB;
      mbar_wait(s_full + buf, (g / NB) & 1);
      tc_fence_after();
      if (!(MODE & 1)) {
        uint32_t r[32];
        tmem_ld32(trow + buf * 128, r);
        tmem_ld32(trow + buf * 128 + 32, r);
        tmem_wait_ld();
      }
      tc_fence_before();
      mbar_arrive(p_full + buf);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

// Two independent slots, each with its own issuer thread (warps 0 and 5) and its own 4 "softmax"
// warps (1-4 for slot 0, 6-9 for slot 1); per slot: S/P at cols t*128, O at 256 + t*128.
// Per step of a slot: wait P, PV (8 MMAs), QK (8 MMAs), commit S.  Softmax: wait S, ld, arrive P.
template <int ISSUERS, int NST>
__global__ void __launch_bounds__(352, 1) k_two(long long* out, int steps) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t s_full[2], p_full[2], kv_full[8], kv_empty[8];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) { mbar_init(s_full + i, 1); mbar_init(p_full + i, 128); }
    for (int i = 0; i < 8; ++i) { mbar_init(kv_full + i, 1); mbar_init(kv_empty + i, 1); }
    fence_barrier_init();
  }
  if (warp == 0) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  int ring = 0;   // issuer's ring position (NST > 0: a loader warp 10 cycles empty -> full)
  long long wt = 0, wp = 0;   // issuer clocks spent in stage waits / P waits
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t q = smem_u32(sm), kv = smem_u32(sm + 65536);
  constexpr uint32_t idq = idesc_bf16_f32(128, 128, 0, 0);
  constexpr uint32_t idp = idesc_bf16_f32(128, 128, 0, 1);
  auto stage = [&]() {
    if (NST > 0) {
      const int s = ring % NST;
      const long long w0 = clock64();
      if (ISSUERS == 3) mbar_wait_spin(kv_full + s, (ring / NST) & 1);
      else if (ISSUERS == 4 || ISSUERS == 7 || ISSUERS == 8 || ISSUERS == 10) { /* no wait: isolates the cost of the loader / commits */ }
      else if (ISSUERS == 5) { if (s == 0) mbar_wait(kv_full + s, (ring / NST) & 1); }
      else mbar_wait(kv_full + s, (ring / NST) & 1);
      wt += clock64() - w0;
      ++ring;
      return s;
    }
    return 0;
  };
  auto release = [&](int s) { if (NST > 0) mma_commit(kv_empty + s); };
  int deferred = -1;   // ISSUERS >= 8: the V stage's release commit moved after the QK group
  auto step_ops = [&](int t, int g, bool pv) {
    if (pv) {
      const int sv = stage();
      const uint32_t vb = kv + ((2 * g + t) % 4) * 32768u;
      for (int kk = 0; kk < 8; ++kk)
        mma_ts(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, sdesc_sw128(vb + kk * 2048, 16384, 1024), idp, 1);
      if (ISSUERS < 8) release(sv);
      else deferred = sv;
    }
    const int sk = stage();
    const uint32_t kb = kv + ((2 * g + t + 1) % 4) * 32768u;
    const uint32_t qb = q + t * 32768u;
    for (int kk = 0; kk < 8; ++kk)
      mma_ss(tmem + t * 128, sdesc_sw128(qb + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
             sdesc_sw128(kb + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), idq, kk > 0);
    if (ISSUERS == 10) {                      // s_full first, then the ring releases
      mma_commit(s_full + t);
      if (deferred >= 0) release(deferred);
      release(sk);
      deferred = -1;
      return;
    }
    if (deferred >= 0) release(deferred);
    deferred = -1;
    release(sk);
    mma_commit(s_full + t);
  };
  const long long t0 = clock64();
  if (ISSUERS == 2 && (warp == 0 || warp == 5)) {
    const int t = warp == 0 ? 0 : 1;
    if (lane == 0) {
      step_ops(t, 0, false);
      for (int g = 0; g < steps; ++g) {
        mbar_wait(p_full + t, g & 1);
        tc_fence_after();
        step_ops(t, g + 1, true);
      }
    }
  } else if ((ISSUERS == 1 || ISSUERS >= 3) && warp == 0) {
    if (lane == 0) {
      step_ops(0, 0, false);
      step_ops(1, 0, false);
      for (int g = 0; g < steps; ++g)
        for (int t = 0; t < 2; ++t) {
          const long long w1 = clock64();
          mbar_wait(p_full + t, g & 1);
          wp += clock64() - w1;
          tc_fence_after();
          step_ops(t, g + 1, true);
        }
    }
  } else if (warp == 10 && NST > 0) {
    if (lane == 0 && ISSUERS != 4) {
      const int total = 2 + 4 * steps;   // stages the issuer consumes
      for (int i = 0; i < total; ++i) {
        const int s = i % NST;
        if (ISSUERS == 6) mbar_wait_spin(kv_empty + s, ((i / NST) & 1) ^ 1);
        else mbar_wait(kv_empty + s, ((i / NST) & 1) ^ 1);
        mbar_arrive(kv_full + s);
      }
    }
  } else if ((warp >= 1 && warp <= 4) || (warp >= 6 && warp <= 9)) {
    const int t = warp >= 6 ? 1 : 0;
    const uint32_t trow = tmem + (uint32_t(((warp - (t ? 6 : 1)) & 3) * 32) << 16);
    for (int g = 0; g < steps; ++g) {
      mbar_wait(s_full + t, g & 1);
      tc_fence_after();
      uint32_t r[32];
      tmem_ld32(trow + t * 128, r);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(p_full + t);
    }
  }
  if (threadIdx.x == 0) { out[200 + blockIdx.x] = wt; out[400 + blockIdx.x] = wp; }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int ISSUERS, int NST>
void run_two(const char* name) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d; cudaMalloc(&d, 1024 * sizeof(long long));
  cudaFuncSetAttribute(k_two<ISSUERS, NST>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int steps = 256;
  k_two<ISSUERS, NST><<<sms, 352, 200 * 1024>>>(d, steps);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[600]; cudaMemcpy(h, d, 600 * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < sms; ++i) avg += h[i]; avg /= sms;
  printf("%-44s %s: %.0f clk per round of 32 MMAs (ideal 2048); issuer stage waits %.0f, P waits %.0f per round\n", name,
         e == cudaSuccess ? "ok" : cudaGetErrorString(e), avg / steps, (double)h[200] / steps, (double)h[400] / steps);
}

template <int MODE, int NB>
void run(const char* name) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d; cudaMalloc(&d, 256 * sizeof(long long));
  cudaFuncSetAttribute(k_hs<MODE, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int steps = 512;
  k_hs<MODE, NB><<<sms, 160, 200 * 1024>>>(d, steps);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < sms; ++i) avg += h[i]; avg /= sms;
  printf("%-44s %s: %.0f clk per step of 16 MMAs (ideal 1024)\n", name,
         e == cudaSuccess ? "ok" : cudaGetErrorString(e), avg / steps);
}

int main() {
  run<0, 2>("handshake, 2 S buffers (QK 2 steps ahead)");
  run<0, 3>("handshake, 3 S buffers (QK 3 steps ahead)");
  run<1, 2>("handshake, 2 S buffers, no tcgen05.ld");
  run_two<1, 0>("two slots, one issuer, no KV ring");
  run_two<1, 4>("two slots, one issuer, KV ring 4 stages");
  run_two<1, 6>("two slots, one issuer, KV ring 6 stages");
  run_two<1, 8>("two slots, one issuer, KV ring 8 stages");
  run_two<3, 8>("two slots, issuer polls, KV ring 8 stages");
  run_two<4, 8>("two slots, ring commits, no waits, no loader");
  run_two<5, 8>("two slots, ring, waits on 1 of 8 stages");
  run_two<6, 8>("two slots, ring 8, loader polls");
  run_two<7, 8>("two slots, ring 8, loader active, issuer never waits");
  run_two<2, 0>("two slots, two issuer warps, no KV ring");
  run_two<8, 8>("two slots, ring commits deferred, no waits");
  run_two<9, 8>("two slots, ring 8 + loader, commits deferred");
  run_two<10, 8>("two slots, ring commits after s_full, no waits");
  return 0;
}
