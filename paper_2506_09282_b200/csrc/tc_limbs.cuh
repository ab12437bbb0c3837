// tc_limbs.cuh -- the int8x3 limb image of the sign-exact tensor-core mode
// (HDC_PREC_FP32_TC) and the float64 re-evaluation of flagged signs,
// shared by the fused kernel (k_fused_tc.cu) and the small-batch tensor-core kernel
// (k_small_tc.cu) so both build bit-identical limbs and bounds.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace hdc {

// float64 re-evaluation of V[row, d] (fixed lane order, warp-cooperative).
__device__ __forceinline__ float recheck_dot(const float* __restrict__ xr, const float* __restrict__ br,
                                             int64_t F, int lane) {
  // lane sums f = lane, lane + 32, ... in f order (fixed), then a fixed butterfly; 32
  // independent loads in flight per chunk of 512 elements (one memory round trip each)
  constexpr int U = 16;
  double s = 0.0;
  for (int64_t f0 = 0; f0 < F; f0 += 32 * U) {
    float xv[U], bv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t f = f0 + 32 * u + lane;
      xv[u] = f < F ? __ldg(xr + f) : 0.f;
      bv[u] = f < F ? __ldg(br + f) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) s = fma((double)xv[u], (double)bv[u], s);   // 0 x 0 adds exactly 0
  }
  s = warp_sum_xor(s);
  return s >= 0.0 ? 1.f : -1.f;
}
// Balanced base-128 digits of the 21-bit integer image U = rint(x * c).
__device__ __forceinline__ void limbs_of(float x, float c, int& d0, int& d1, int& d2, int& U) {
  int u = __float2int_rn(x * c);
  u = max(-2080768, min(2080768, u));
  d2 = ((u + 64) & 127) - 64;
  const int u1 = (u - d2) >> 7;
  d1 = ((u1 + 64) & 127) - 64;
  d0 = (u1 - d1) >> 7;
  U = u;
}

__device__ __forceinline__ float scale_for(float amax) {
  if (!(amax > 0.f)) return 1.f;
  double c = 2080768.0 / (double)amax;
  if (c > 1e37) c = 1e37;
  return (float)c * (1.f - 9.5367431640625e-07f);  // (1 - 2^-20): keeps |x c| < 127*2^14
}

// Four consecutive elements f0..f0+3 of a source row (zero past F and for padding rows);
// one 16-byte load when the row start and f0 are 16-byte aligned and all four are < F.
__device__ __forceinline__ void load4(const float* __restrict__ row, int64_t f0, int64_t F, bool valid,
                                      bool vec, float* x) {
  if (valid && vec && f0 + 3 < F) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(row + f0));
    x[0] = v.x;
    x[1] = v.y;
    x[2] = v.z;
    x[3] = v.w;
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) x[e] = (valid && f0 + e < F) ? __ldg(row + f0 + e) : 0.f;
  }
}

// tau of a row from its L1(U): |c_x c_b x.b - U_x.U_b| <= 0.625 (L1(U_x) + L1(U_b)) +
// 0.3907 F and the dropped limb products (i + j >= 3) add <= F (2^20 + 2^12) (DESIGN.md
// §4).  The kernel compares I = A0 2^14 + A1 2^7 + A2 = (U_x.U_b - dropped) / 2^14, so
// tau is stored / 2^14, rounded up: ceil((5 l1 / 8 + tau_const) / 2^14)
// = (5 l1 + 8 tau_const + 2^17 - 1) >> 17.
__device__ __forceinline__ int64_t row_tau(long long l1, int64_t tau_const, bool valid) {
  return valid ? ((5 * l1 + 8 * tau_const + 131071) >> 17) + 1 : -(int64_t(1) << 62);
}

}  // namespace hdc
