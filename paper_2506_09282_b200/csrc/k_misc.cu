// k_misc.cu -- K5 row argmax and the model-setup kernels (padding copies, norms).
#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace hdc {
namespace {

// K5: one warp per row; (value, index) pairs combined so that the lowest index
// among equal maxima wins (eq. pred_batch; tie rule DESIGN.md R2).
__global__ void argmax_kernel(const float* __restrict__ S, int64_t N, int64_t K,
                              int32_t* __restrict__ labels) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (row >= N) return;
  const float* s = S + row * K;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int64_t k = lane; k < K; k += 32) {
    const float v = s[k];
    if (bi == 0x7fffffff || v > bv) { bv = v; bi = (int)k; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (oi != 0x7fffffff && (bi == 0x7fffffff || ov > bv || (ov == bv && oi < bi))) {
      bv = ov;
      bi = oi;
    }
  }
  if (lane == 0) labels[row] = bi;
}

__global__ void pad_copy_kernel(const float* __restrict__ src, int64_t rows, int64_t cols,
                                float* __restrict__ dst, int64_t dst_cols) {
  const int64_t total = rows * dst_cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / dst_cols, c = i % dst_cols;
    dst[i] = c < cols ? src[r * cols + c] : 0.f;
  }
}

__global__ void transpose_kernel(const float* __restrict__ src, int64_t rows, int64_t cols,
                                 float* __restrict__ dst) {
  __shared__ float t[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + k, c = c0 + threadIdx.x;
    t[k][threadIdx.x] = (r < rows && c < cols) ? src[r * cols + c] : 0.f;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t c = c0 + k, r = r0 + threadIdx.x;
    if (c < cols && r < rows) dst[c * rows + r] = t[threadIdx.x][k];
  }
}

// B4[u][f][j] = Bp[f][4u + j]: all rows of a 4-column unit contiguous.
__global__ void unit_major_kernel(const float4* __restrict__ Bp, int64_t Fp, int64_t U,
                                  float4* __restrict__ B4) {
  const int64_t total = Fp * U;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = i / Fp, f = i % Fp;
    B4[i] = Bp[f * U + u];
  }
}

// ||b_d||_2 in float64, rounded UP to fp32 (it only feeds an upper bound).
__global__ void col_norm_kernel(const float* __restrict__ Bp, int64_t F, int64_t Dp, int64_t D,
                                float* __restrict__ out) {
  const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (d >= Dp) return;
  double s = 0.0;
  if (d < D)
    for (int64_t f = 0; f < F; ++f) {
      const double b = Bp[f * Dp + d];
      s = fma(b, b, s);
    }
  out[d] = __double2float_ru(__dsqrt_ru(s));
}

// Diagnostic: read `bytes` once with 1-D bulk copies, each CTA one contiguous range through
// an 8 x 16 KB ring (the one-shot streaming ceiling the small-batch kernels are compared with).
__global__ void __launch_bounds__(64, 1) stream_read_kernel(const uint8_t* __restrict__ src, int64_t bytes,
                                                            unsigned* sink) {
  constexpr int NST = 8, CH = 16384;
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ uint64_t full[NST];
  const int64_t per = (bytes / gridDim.x + 15) / 16 * 16;
  const int64_t b0 = blockIdx.x * per, b1 = (b0 + per < bytes) ? b0 + per : bytes;
  const int64_t n = b1 > b0 ? (b1 - b0 + CH - 1) / CH : 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) ptx::mbar_init(&full[i], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  unsigned acc = 0;
  if (threadIdx.x == 0) {
    for (int64_t k = 0; k < n; ++k) {
      const int s = (int)(k % NST);
      if (k >= NST) {
        ptx::mbar_wait(&full[s], (uint32_t)(((k / NST) - 1) & 1));
        acc += ring[(size_t)s * CH];
      }
      const int64_t o = b0 + k * CH;
      const uint32_t nb = (uint32_t)((b1 - o) < CH ? ((b1 - o) + 15) / 16 * 16 : CH);
      ptx::mbar_arrive_expect_tx(&full[s], nb);
      ptx::bulk_load(ring + (size_t)s * CH, src + o, nb, &full[s]);
    }
    for (int64_t k = (n > NST ? n - NST : 0); k < n; ++k) {
      const int s = (int)(k % NST);
      ptx::mbar_wait(&full[s], (uint32_t)((k / NST) & 1));
      acc += ring[(size_t)s * CH];
    }
    if (acc == 0xFFFFFFFFu) *sink = acc;
  }
}

}  // namespace

cudaError_t launch_stream_read(const void* buf, int64_t bytes, int num_sms, cudaStream_t st) {
  const int smem = 8 * 16384;
  cudaError_t e = cudaFuncSetAttribute(stream_read_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  stream_read_kernel<<<num_sms, 64, smem, st>>>(static_cast<const uint8_t*>(buf), bytes, nullptr);
  return cudaGetLastError();
}

cudaError_t launch_argmax(const float* S, int64_t N, int64_t K, int32_t* labels, cudaStream_t st) {
  if (N <= 0) return cudaSuccess;
  const int warps = 8;
  argmax_kernel<<<(unsigned)((N + warps - 1) / warps), warps * 32, 0, st>>>(S, N, K, labels);
  return cudaGetLastError();
}

cudaError_t launch_pad_copy(const float* src, int64_t rows, int64_t cols, float* dst,
                            int64_t dst_cols, cudaStream_t st) {
  const int64_t total = rows * dst_cols;
  if (total <= 0) return cudaSuccess;
  int64_t grid = (total + 255) / 256;
  if (grid > 148 * 32) grid = 148 * 32;
  pad_copy_kernel<<<(unsigned)grid, 256, 0, st>>>(src, rows, cols, dst, dst_cols);
  return cudaGetLastError();
}

cudaError_t launch_transpose(const float* src, int64_t rows, int64_t cols, float* dst,
                             cudaStream_t st) {
  dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(src, rows, cols, dst);
  return cudaGetLastError();
}

cudaError_t launch_unit_major(const float* Bp, int64_t Fp, int64_t Dp, float* B4, cudaStream_t st) {
  const int64_t total = Fp * (Dp / 4);
  int64_t grid = (total + 255) / 256;
  if (grid > 148 * 32) grid = 148 * 32;
  unit_major_kernel<<<(unsigned)grid, 256, 0, st>>>(reinterpret_cast<const float4*>(Bp), Fp, Dp / 4,
                                                    reinterpret_cast<float4*>(B4));
  return cudaGetLastError();
}

cudaError_t launch_col_norms(const float* Bp, int64_t F, int64_t Dp, int64_t D, float* out,
                             cudaStream_t st) {
  col_norm_kernel<<<(unsigned)((Dp + 255) / 256), 256, 0, st>>>(Bp, F, Dp, D, out);
  return cudaGetLastError();
}

}  // namespace hdc
