// k_packed.cu -- kernels on a materialised, bit-packed H (N x D signs).
//
// Two uses of the encoded hypervectors outside the fused path:
//  * the unfused ablation of the paper's fusion: Stage II and the
//    argmax as a separate pass over H written to HBM by hdc_model_encode
//    (`packed_similarity_kernel`);
//  * single-pass training: class HVs by constrained bundling of
//    the encoded HVs of each class, m_k = HardSign(sum_{n: y_n = k} h_n)
//    (`label_sort_kernel`, `bundle_kernel`, `hardsign_i32_kernel`).
// Packing: row n, column d -> word n * ldw + d / 32, bit d % 32; bit set <=> h = -1.
#include <cstdint>
#include <cstdio>

#include "common.cuh"
#include "kernels.h"

namespace hdc {
namespace {

constexpr int kRows = 128;        // rows (threads) per CTA of the similarity kernel
constexpr int kDch = 64;          // columns per smem chunk (2 words per row)

// S[n, k] = sum_d h[n, d] C[k, d]  (d ascending, fp32 FMA; eq. batch_sim), then
// lowest-index argmax.  One thread per row; C chunks [kDch][KT] in smem are
// read as float4 broadcasts, H words of the CTA's rows staged through smem.
template <int KT>
__global__ void __launch_bounds__(kRows) packed_similarity_kernel(const uint32_t* __restrict__ H, int64_t ldw,
                                                                  int64_t N, int64_t D,
                                                                  const float* __restrict__ C, int64_t K,
                                                                  int32_t* labels, float* scores) {
  __shared__ __align__(16) float Cs[kDch][KT];
  __shared__ uint32_t Hs[kRows][kDch / 32 + 1];
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * kRows, row = r0 + tid;
  float2 acc[KT / 2];
#pragma unroll
  for (int k = 0; k < KT / 2; ++k) acc[k] = make_float2(0.f, 0.f);
  for (int64_t d0 = 0; d0 < D; d0 += kDch) {
    __syncthreads();
    for (int i = tid; i < kDch * KT; i += kRows) {
      const int dd = i / KT, k = i % KT;
      Cs[dd][k] = (k < K && d0 + dd < D) ? __ldg(C + (int64_t)k * D + d0 + dd) : 0.f;
    }
    for (int i = tid; i < kRows * (kDch / 32); i += kRows) {
      const int rr = i / (kDch / 32), w = i % (kDch / 32);
      const int64_t wi = d0 / 32 + w;
      Hs[rr][w] = (r0 + rr < N && wi < ldw) ? __ldg(H + (r0 + rr) * ldw + wi) : 0u;
    }
    __syncthreads();
    const int dn = (D - d0) < kDch ? (int)(D - d0) : kDch;
    for (int dd = 0; dd < dn; ++dd) {
      const float h = ((Hs[tid][dd >> 5] >> (dd & 31)) & 1u) ? -1.f : 1.f;
      const float4* c4 = reinterpret_cast<const float4*>(&Cs[dd][0]);
#pragma unroll
      for (int k4 = 0; k4 < KT / 4; ++k4) {
        const float4 cv = c4[k4];
        acc[2 * k4] = ffma2(h, make_float2(cv.x, cv.y), acc[2 * k4]);
        acc[2 * k4 + 1] = ffma2(h, make_float2(cv.z, cv.w), acc[2 * k4 + 1]);
      }
    }
  }
  if (row >= N) return;
  int best = 0;
  float bv = 0.f;
#pragma unroll
  for (int k = 0; k < KT; ++k) {
    if (k >= K) break;
    const float v = (k & 1) ? acc[k >> 1].y : acc[k >> 1].x;
    if (scores) scores[row * K + k] = v;
    if (k == 0 || v > bv) {
      bv = v;
      best = k;
    }
  }
  if (labels) labels[row] = best;
}

// Rows grouped by label (counting sort; the order inside a class is irrelevant: the
// bundle is an integer sum).  One CTA; offs[K + 1], perm[N]; labels outside [0, K) are
// counted in err.
__global__ void label_sort_kernel(const int32_t* __restrict__ y, int64_t N, int64_t K, int64_t* offs,
                                  int64_t* perm, unsigned* err) {
  extern __shared__ unsigned long long sh[];      // [K] counts then cursors
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) sh[k] = 0ull;
  __syncthreads();
  for (int64_t n = threadIdx.x; n < N; n += blockDim.x) {
    const int32_t k = y[n];
    if (k < 0 || k >= K) atomicAdd(err, 1u);
    else atomicAdd(&sh[k], 1ull);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long run = 0;
    for (int64_t k = 0; k < K; ++k) {
      const unsigned long long c = sh[k];
      offs[k] = (int64_t)run;
      sh[k] = run;
      run += c;
    }
    offs[K] = (int64_t)run;
  }
  __syncthreads();
  for (int64_t n = threadIdx.x; n < N; n += blockDim.x) {
    const int32_t k = y[n];
    if (k >= 0 && k < K) perm[atomicAdd(&sh[k], 1ull)] = n;
  }
}

// counts[k][d] += sum_{n: y_n = k} h[n, d] = n_k - 2 #{n in class k: h[n, d] = -1}: one
// thread per (class, 32-column word); per-bit counters in registers (exact integers).
__global__ void bundle_kernel(const uint32_t* __restrict__ H, int64_t ldw, int64_t D, int64_t K,
                              const int64_t* __restrict__ offs, const int64_t* __restrict__ perm,
                              int32_t* __restrict__ counts) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t k = blockIdx.y;
  if (w >= ldw || w * 32 >= D) return;
  const int64_t b = offs[k], e = offs[k + 1];
  int c[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) c[i] = 0;
  for (int64_t i = b; i < e; ++i) {
    const uint32_t bits = __ldg(H + perm[i] * ldw + w);
#pragma unroll
    for (int j = 0; j < 32; ++j) c[j] += (int)((bits >> j) & 1u);
  }
  const int nk = (int)(e - b);
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const int64_t d = w * 32 + j;
    if (d < D) counts[k * D + d] += nk - 2 * c[j];
  }
}

// constrained bundling: m = HardSign(count) (ties -> +1)
__global__ void hardsign_i32_kernel(const int32_t* __restrict__ counts, int64_t n, float* __restrict__ M) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    M[i] = counts[i] >= 0 ? 1.f : -1.f;
}

template <int KT>
cudaError_t launch_sim(const uint32_t* H, int64_t ldw, int64_t N, int64_t D, const float* C, int64_t K,
                       int32_t* labels, float* scores, cudaStream_t st) {
  packed_similarity_kernel<KT><<<(unsigned)((N + kRows - 1) / kRows), kRows, 0, st>>>(H, ldw, N, D, C, K,
                                                                                     labels, scores);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_packed_similarity(const uint32_t* H, int64_t ldw, int64_t N, int64_t D, const float* C,
                                     int64_t K, int32_t* labels, float* scores, cudaStream_t st) {
  if (K <= 8) return launch_sim<8>(H, ldw, N, D, C, K, labels, scores, st);
  if (K <= 16) return launch_sim<16>(H, ldw, N, D, C, K, labels, scores, st);
  if (K <= 32) return launch_sim<32>(H, ldw, N, D, C, K, labels, scores, st);
  if (K <= 64) return launch_sim<64>(H, ldw, N, D, C, K, labels, scores, st);
  return cudaErrorInvalidValue;     // the API checks K <= 64 for this diagnostic path
}

cudaError_t launch_bundle(const uint32_t* H, int64_t ldw, int64_t N, int64_t D, const int32_t* y, int64_t K,
                          int32_t* counts, float* M, unsigned* err, cudaStream_t st) {
  int64_t* offs = nullptr;
  int64_t* perm = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&offs, sizeof(int64_t) * (K + 1), st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&perm, sizeof(int64_t) * (N > 0 ? N : 1), st);
  if (e != cudaSuccess) return e;
  label_sort_kernel<<<1, 1024, sizeof(unsigned long long) * K, st>>>(y, N, K, offs, perm, err);
  e = cudaGetLastError();
  if (e == cudaSuccess) {
    dim3 grid((unsigned)((ldw + 127) / 128), (unsigned)K);
    bundle_kernel<<<grid, 128, 0, st>>>(H, ldw, D, K, offs, perm, counts);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && M) {
    hardsign_i32_kernel<<<148 * 4, 256, 0, st>>>(counts, K * D, M);
    e = cudaGetLastError();
  }
  cudaFreeAsync(offs, st);
  cudaFreeAsync(perm, st);
  return e;
}

}  // namespace hdc
