// kernel_util.cuh — small device helpers shared by the attention and predictor kernels
// (warp election, setmaxnreg, packed fp32x2 arithmetic, FMA-pipe exp2).  sm_100a only.
#pragma once
#include <cstdint>
#include "ptx.cuh"

namespace sv {

__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t r, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(r));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

template <int N>
__device__ __forceinline__ void reg_alloc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void reg_dealloc() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}

// 2^x for a pair on the FMA/ALU pipes (offloads MUFU): x = n + f, n = rint(x) via the 1.5*2^23
// magic add, f in [-1/2, 1/2], 2^f by a minimax polynomial of degree DEG (max relative error
// 7.5e-5 for DEG 3, 2.6e-6 for DEG 4), 2^n added to the exponent field.  x is clamped at -126
// so masked (-inf) logits give 2^-126 instead of 0: callers make that negligible (l >= 1) or
// exclude such rows.
template <int DEG>
__device__ __forceinline__ void ex2_emu2(uint64_t x2, float& p0, float& p1) {
  static_assert(DEG == 3 || DEG == 4, "degree");
  constexpr float MAGIC = 12582912.0f;   // 1.5 * 2^23
  float x0, x1;
  f2_unpack(x2, x0, x1);
  x0 = fmaxf(x0, -126.f);
  x1 = fmaxf(x1, -126.f);
  const uint64_t xc = f2_pack(x0, x1);
  const uint64_t t = fadd2(xc, f2_pack(MAGIC, MAGIC));
  const uint64_t r = fadd2(t, f2_pack(-MAGIC, -MAGIC));
  const uint64_t f = ffma2(r, f2_pack(-1.f, -1.f), xc);   // x - rint(x)
  uint64_t q;
  if constexpr (DEG == 3) {
    q = ffma2(f2_pack(0.05517166f, 0.05517166f), f, f2_pack(0.24261113f, 0.24261113f));
    q = ffma2(q, f, f2_pack(0.69326097f, 0.69326097f));
    q = ffma2(q, f, f2_pack(0.99992806f, 0.99992806f));
  } else {
    q = ffma2(f2_pack(0.0095701022f, 0.0095701022f), f, f2_pack(0.055917859f, 0.055917859f));
    q = ffma2(q, f, f2_pack(0.24024743f, 0.24024743f));
    q = ffma2(q, f, f2_pack(0.69312179f, 0.69312179f));
    q = ffma2(q, f, f2_pack(0.99999928f, 0.99999928f));
  }
  float q0, q1, t0, t1;
  f2_unpack(q, q0, q1);
  f2_unpack(t, t0, t1);
  p0 = __int_as_float(__float_as_int(q0) + (__float_as_int(t0) << 23));
  p1 = __int_as_float(__float_as_int(q1) + (__float_as_int(t1) << 23));
}

// Volatile variants: their relative program order is kept by the compiler, which lets a
// software-pipelined loop interleave the MUFU stream with FMA/ALU work by construction.
__device__ __forceinline__ uint64_t vffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t vfadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm volatile("add.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float vex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t vpack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

}  // namespace sv
