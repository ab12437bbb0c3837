// Device twin of hdc_inputs/philox.py: Philox4x32-10 uniforms written straight
// into HBM (used by bench.py for the large X of cfg2/cfg4/cfg5). Integer
// arithmetic plus one exact fp32 affine map, so the bytes equal the numpy
// generator's (tests/test_inputs.py). Holds none of the method's arithmetic.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

constexpr uint32_t kM0 = 0xD2511F53u, kM1 = 0xCD9E8D57u;
constexpr uint32_t kW0 = 0x9E3779B9u, kW1 = 0xBB67AE85u;
constexpr uint32_t kKeyHi = 0x48444331u;  // must match philox.KEY_HI

__device__ __forceinline__ uint4 philox(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += kW0; k1 += kW1; }
    uint32_t hi0 = __umulhi(kM0, c.x), lo0 = kM0 * c.x;
    uint32_t hi1 = __umulhi(kM1, c.z), lo1 = kM1 * c.z;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
  }
  return c;
}

__global__ void uniform_kernel(float* __restrict__ out, uint64_t start, uint64_t count,
                               uint32_t seed, uint32_t tid, float a, float span) {
  const uint64_t b0 = start >> 2;
  const uint64_t nblk = ((start + count + 3) >> 2) - b0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nblk;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t blk = b0 + i;
    uint4 w = philox(make_uint4((uint32_t)blk, (uint32_t)(blk >> 32), tid, 0u), seed, kKeyHi);
    uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t idx = (blk << 2) + j;
      if (idx < start || idx >= start + count) continue;
      float u = (float)(ws[j] >> 8) * 5.9604644775390625e-08f;  // 2^-24, exact
      out[idx - start] = __fadd_rn(a, __fmul_rn(span, u));
    }
  }
}

}  // namespace

extern "C" int hdcgen_uniform_f32(float* out, uint64_t start, uint64_t count, uint32_t seed,
                                  uint32_t tid, float a, float b, void* stream) {
  if (count == 0) return 0;
  if (out == nullptr) return 1;
  const uint64_t nblk = ((start + count + 3) >> 2) - (start >> 2);
  uint64_t grid = (nblk + 255) / 256;
  if (grid > 148ull * 64) grid = 148ull * 64;
  uniform_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(out, start, count, seed, tid,
                                                                   a, b - a);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}
