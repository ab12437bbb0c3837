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

constexpr int kRows = 64;         // rows per CTA of the similarity kernel
constexpr int kSimThreads = 128;  // 16 row groups x 8 class groups; 4 rows x 4 classes each
constexpr int kDw = 2;            // 32-column words per pipeline stage (64 columns)

// S[n, k] = sum_d h[n, d] C[k, d]  (fp32 FMA, d ascending; eq. batch_sim) and
// the lowest-index argmax, as a small GEMM over +-1 rows: per CTA 64 rows x
// KT classes; per stage 64 columns of H (2 words per row) and of C ([64][KT] in smem,
// double-buffered with cp.async); a thread keeps a 4-row x (KT/8)-class register tile.
template <int KT>
__global__ void __launch_bounds__(kSimThreads) packed_similarity_kernel(const uint32_t* __restrict__ H,
                                                                        int64_t ldw, int64_t N, int64_t D,
                                                                        const float* __restrict__ Ct,
                                                                        int64_t K, int32_t* labels,
                                                                        float* scores) {
  constexpr int KC = KT / 8;                         // classes per thread
  constexpr int CS_BYTES = 2 * kDw * 32 * KT * 4, SO_BYTES = kRows * (KT + 1) * 4;
  __shared__ __align__(16) uint8_t pool[CS_BYTES > SO_BYTES ? CS_BYTES : SO_BYTES];
  __shared__ uint32_t Hs[2][kRows][kDw];
  float (*Cs)[kDw * 32][KT] = reinterpret_cast<float (*)[kDw * 32][KT]>(pool);    // [2][64][KT]
  float (*Sout)[KT + 1] = reinterpret_cast<float (*)[KT + 1]>(pool);              // after the loop
  const int tid = threadIdx.x;
  const int rg = tid >> 3, cg = tid & 7;             // rows 4 rg .. 4 rg + 3, classes cg KC ..
  const int64_t r0 = (int64_t)blockIdx.x * kRows;
  const int64_t nst = (D + kDw * 32 - 1) / (kDw * 32);
  auto load = [&](int64_t st, int buf) {
    const int64_t d0 = st * kDw * 32;
    // C^T rows d (classes contiguous, KT floats, zero padded): 16-byte cp.async pieces
    for (int i = tid; i < kDw * 32 * (KT / 4); i += kSimThreads) {
      const int dd = i / (KT / 4), q = i % (KT / 4);
      float* dst = &Cs[buf][dd][4 * q];
      if (d0 + dd < D) {
        const float* src = Ct + (d0 + dd) * KT + 4 * q;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                     "l"(src) : "memory");
      } else {
        *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    for (int i = tid; i < kRows * kDw; i += kSimThreads) {
      const int rr = i / kDw, w = i % kDw;
      const int64_t wi = d0 / 32 + w;
      Hs[buf][rr][w] = (r0 + rr < N && wi < ldw) ? __ldg(H + (r0 + rr) * ldw + wi) : 0u;
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  float2 acc[4][KC / 2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < KC / 2; ++j) acc[i][j] = make_float2(0.f, 0.f);
  load(0, 0);
  for (int64_t st = 0; st < nst; ++st) {
    const int buf = (int)(st & 1);
    if (st + 1 < nst) {
      load(st + 1, buf ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    uint32_t hw[4][kDw];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int w = 0; w < kDw; ++w) hw[i][w] = Hs[buf][4 * rg + i][w];
    const int64_t d0 = st * kDw * 32;
    const int dn = (D - d0) < kDw * 32 ? (int)(D - d0) : kDw * 32;
    for (int dd = 0; dd < dn; ++dd) {
      float2 c2[KC / 2];
#pragma unroll
      for (int j = 0; j < KC / 2; ++j) c2[j] = *reinterpret_cast<const float2*>(&Cs[buf][dd][cg * KC + 2 * j]);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float h = ((hw[i][dd >> 5] >> (dd & 31)) & 1u) ? -1.f : 1.f;
#pragma unroll
        for (int j = 0; j < KC / 2; ++j) acc[i][j] = ffma2(h, c2[j], acc[i][j]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < KC / 2; ++j) {
      Sout[4 * rg + i][cg * KC + 2 * j] = acc[i][j].x;
      Sout[4 * rg + i][cg * KC + 2 * j + 1] = acc[i][j].y;
    }
  __syncthreads();
  if (tid >= kRows || r0 + tid >= N) return;
  const int64_t row = r0 + tid;
  int best = 0;
  float bv = 0.f;
  for (int k = 0; k < K; ++k) {
    const float v = Sout[tid][k];
    if (scores) scores[row * K + k] = v;
    if (k == 0 || v > bv) {
      bv = v;
      best = k;
    }
  }
  if (labels) labels[row] = best;
}

// C (K x D) -> C^T (D x KT), classes padded with zeros (the similarity kernel's operand)
__global__ void ct_pad_kernel(const float* __restrict__ C, int64_t K, int64_t D, int KT, float* __restrict__ Ct) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < D * KT; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = i / KT, k = i % KT;
    Ct[i] = k < K ? C[k * D + d] : 0.f;
  }
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

// counts[k][d] += sum_{n: y_n = k} h[n, d] = n_k - 2 #{n in class k: h[n, d] = -1}.  Rows
// in label order (perm) are cut into chunks of kBundleRows; thread = one 32-column word,
// per-bit counters in registers, flushed with integer atomics whenever the class changes
// (integer sums: exact and independent of the order the chunks run in).
constexpr int kBundleRows = 128;
__global__ void bundle_kernel(const uint32_t* __restrict__ H, int64_t ldw, int64_t N, int64_t D,
                              const int32_t* __restrict__ y, const int64_t* __restrict__ perm,
                              int32_t* __restrict__ counts, const unsigned* __restrict__ err) {
  if (*err) return;                    // a label outside [0, K): leave counts untouched
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t i0 = (int64_t)blockIdx.y * kBundleRows;
  const int64_t i1 = (i0 + kBundleRows) < N ? (i0 + kBundleRows) : N;
  if (w >= ldw || w * 32 >= D || i0 >= N) return;
  int c[32];
  int cur = -1, nk = 0;
  auto flush = [&]() {
    if (cur < 0) return;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int64_t d = w * 32 + j;
      if (d < D) atomicAdd(counts + (int64_t)cur * D + d, nk - 2 * c[j]);
    }
  };
  for (int64_t i = i0; i < i1; ++i) {
    const int64_t n = perm[i];
    const int k = y[n];
    if (k != cur) {
      flush();
      cur = k;
      nk = 0;
#pragma unroll
      for (int j = 0; j < 32; ++j) c[j] = 0;
    }
    const uint32_t bits = __ldg(H + n * ldw + w);
#pragma unroll
    for (int j = 0; j < 32; ++j) c[j] += (int)((bits >> j) & 1u);
    ++nk;
  }
  flush();
}

// constrained bundling: m = HardSign(count) (ties -> +1)
__global__ void hardsign_i32_kernel(const int32_t* __restrict__ counts, int64_t n, float* __restrict__ M,
                                    const unsigned* __restrict__ err) {
  if (*err) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    M[i] = counts[i] >= 0 ? 1.f : -1.f;
}

template <int KT>
cudaError_t launch_sim(const uint32_t* H, int64_t ldw, int64_t N, int64_t D, const float* C, int64_t K,
                       int32_t* labels, float* scores, cudaStream_t st) {
  float* Ct = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&Ct, sizeof(float) * D * KT, st);
  if (e != cudaSuccess) return e;
  ct_pad_kernel<<<148 * 4, 256, 0, st>>>(C, K, D, KT, Ct);
  packed_similarity_kernel<KT><<<(unsigned)((N + kRows - 1) / kRows), kSimThreads, 0, st>>>(H, ldw, N, D, Ct, K,
                                                                                          labels, scores);
  e = cudaGetLastError();
  cudaFreeAsync(Ct, st);
  return e;
}

}  // namespace

cudaError_t launch_packed_similarity(const uint32_t* H, int64_t ldw, int64_t N, int64_t D, const float* C,
                                     int64_t K, int32_t* labels, float* scores, cudaStream_t st) {
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
    dim3 grid((unsigned)((ldw + 127) / 128), (unsigned)((N + kBundleRows - 1) / kBundleRows));
    if (N > 0) bundle_kernel<<<grid, 128, 0, st>>>(H, ldw, N, D, y, perm, counts, err);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && M) {
    hardsign_i32_kernel<<<148 * 4, 256, 0, st>>>(counts, K * D, M, err);
    e = cudaGetLastError();
  }
  cudaFreeAsync(offs, st);
  cudaFreeAsync(perm, st);
  return e;
}

}  // namespace hdc
