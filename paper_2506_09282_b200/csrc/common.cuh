// common.cuh -- small device helpers shared by the libhdc kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define HDC_DEV __device__ __forceinline__

namespace hdc {

// HardSign: +1 if v >= 0 else -1.  IEEE `>=`: -0.0 -> +1, NaN -> -1.
HDC_DEV float hardsign(float v) { return v >= 0.f ? 1.f : -1.f; }

// Streaming 128-bit load that does not allocate in L1 (B is read once).
HDC_DEV float4 ldg_stream(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

// Coherent-at-L2 load of data written by other CTAs of the same launch.
HDC_DEV float ld_cg(const float* p) { return __ldcg(p); }

// Packed fp32x2 FMA (sm_100a FFMA2): {a*b.x + c.x, a*b.y + c.y}, each correctly
// rounded exactly like fmaf -- half the FMA-pipe instructions of two fmaf.
HDC_DEV float2 ffma2(float a, float2 b, float2 c) {
  unsigned long long aa, bb, cc, dd;
  asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
  asm("mov.b64 %0, {%1, %2};" : "=l"(bb) : "f"(b.x), "f"(b.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(cc) : "f"(c.x), "f"(c.y));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(dd) : "l"(aa), "l"(bb), "l"(cc));
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(dd));
  return r;
}

HDC_DEV float warp_max_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <typename T>
HDC_DEV T warp_sum_xor(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Rigorous fp32 sign-decision bound coefficient:
// |fl32(x.b) - x.b| <= gamma_F sum|x_f b_f| <= gamma_F ||x|| ||b||,
// gamma_F = F u / (1 - F u), u = 2^-24.  We use (F + 32) u times a
// (1 + 2 F u + 2^-16) factor covering 1/(1 - F u), the fp32 evaluation of
// ||x||^2 (relative error <= F u, halved by the sqrt) and the two roundings of
// the product coef*||x||*||b||.  Valid for F <= 2^20 (checked by the API).
// Underflow of subnormal products is covered by kSignBoundAbs added to tau.
inline float sign_bound_coef(int64_t F) {
  const double u = 1.0 / 16777216.0;
  return (float)((double)(F + 32) * u * (1.0 + 2.0 * (double)F * u + 1.0 / 65536.0));
}
constexpr float kSignBoundAbs = 1e-37f;

}  // namespace hdc
