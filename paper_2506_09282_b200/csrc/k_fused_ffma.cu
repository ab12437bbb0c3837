// k_fused_ffma.cu -- K1 (X staging) and K3: the fused large-batch fp32 kernel.
//
// K3 computes Alg. 1 for 128-row N-tiles without materialising H:
//   per (N-tile, D-tile 128 wide): V = X_tile B_tile by register-blocked FFMA
//   (8x8 outputs per thread, cp.async 4-stage smem pipeline over F),
//   HardSign in registers, fp64 re-evaluation of the rare |v| <= tau
//   (sign-exact fp32 path), then Stage II S_local += H C_tile^T
//    into an on-chip N-tile x K accumulator.  H lives only in shared
//   memory for the duration of one tile (the paper's "prohibitively large" H,
//   P:211, never reaches HBM).
// Each CTA owns one N-tile and a contiguous range of D-tiles (ScalableHD-L's
// row ownership, Alg. 4, combined with ScalableHD-S's D split, Alg. 3,
// so that the grid fills 148 SMs); the partial scores of the D ranges are summed
// in fixed order by the last-arriving CTA of the N-tile, which also takes the
// lowest-index argmax.  One launch (plus K1), bit-deterministic.
#include "common.cuh"
#include "kernels.h"

namespace hdc {
namespace {

#ifndef HDC_K3_BK
#define HDC_K3_BK 16
#endif
#ifndef HDC_K3_STAGES
#define HDC_K3_STAGES 4
#endif
constexpr int BM = 128, BN = 128, BK = HDC_K3_BK, STAGES = HDC_K3_STAGES, THREADS = 256;
constexpr int HS = BM + 4;           // Hs row stride (floats)
constexpr int LIST_CAP = 1024;       // flagged-element list per tile
constexpr int kSaccSmemMaxK = 64;    // larger K keeps the score accumulator in L2

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---------------------------------------------------------------- K1: X staging
// Xt[tile][f][m] (m fastest, zero-padded to 128 rows and Fp columns) so K3's
// A-operand tiles are contiguous 16-byte cp.async copies; xnorm[r] = ||x_r||_2
// (fp32, fixed summation order) for the sign bound.
__global__ void __launch_bounds__(256) prep_x_kernel(const float* __restrict__ X, int64_t N,
                                                     int64_t F, int64_t Fp,
                                                     float* __restrict__ Xt,
                                                     float* __restrict__ xnorm) {
  __shared__ float tile[32][BM + 1];
  const int t = threadIdx.x;
  const int64_t i = blockIdx.x;
  const int64_t row0 = i * BM;
  float ss = 0.f;
  for (int64_t f0 = 0; f0 < Fp; f0 += 32) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = t + 256 * u;
      const int r = e >> 5, c = e & 31;
      const int64_t row = row0 + r, f = f0 + c;
      tile[c][r] = (row < N && f < F) ? __ldg(X + row * F + f) : 0.f;
    }
    __syncthreads();
    if (t < BM) {
#pragma unroll 8
      for (int c = 0; c < 32; ++c) ss = fmaf(tile[c][t], tile[c][t], ss);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = t + 256 * u;
      const int c = e >> 7, r = e & 127;
      Xt[(i * Fp + f0 + c) * BM + r] = tile[c][r];
    }
    __syncthreads();
  }
  if (t < BM) xnorm[row0 + t] = sqrtf(ss);
}

// ---------------------------------------------------------------- K3
struct FusedParams {
  const float* Xt;
  const float* X;
  const float* xnorm;
  int64_t N, F, Fp, D, Dp, K;
  const float* Bp;
  const float* Bt;
  const float* Cp;
  const float* bnorm;
  float tau_coef;
  int recheck;
  int Tn, Td, R;
  float* S_part;
  unsigned* cnt;
  unsigned long long* recheck_count;
  float* scores;
  int32_t* labels;
};

// fp64 re-evaluation of one pre-activation by one warp (fixed reduction order).
__device__ __forceinline__ float recheck_sign_warp(const float* xr, const float* br, int64_t F,
                                                   int lane) {
  double s = 0.0;
  for (int64_t f = lane; f < F; f += 32) s = fma((double)__ldg(xr + f), (double)__ldg(br + f), s);
  s = warp_sum_xor(s);
  return s >= 0.0 ? 1.f : -1.f;
}

__global__ void __launch_bounds__(THREADS, 1) fused_ffma_kernel(const FusedParams p) {
  extern __shared__ __align__(16) float smem[];
  float* As = smem;                                  // [STAGES][BK][BM]
  float* Bs = As + STAGES * BK * BM;                 // [STAGES][BK][BN]
  float* Hs = Bs + STAGES * BK * BN;                 // [BN][HS]
  int* list = reinterpret_cast<int*>(Hs + BN * HS);  // [LIST_CAP]
  // On-chip N-tile x K score accumulator: shared memory [K][BM] when it fits,
  // else this CTA's own slice of the partial-score workspace ([BM][K], L2).
  const int64_t Np = (int64_t)p.Tn * BM;
  float* part = p.S_part + (int64_t)blockIdx.x * Np * p.K + (int64_t)blockIdx.y * BM * p.K;
  const bool sacc_smem = p.K <= kSaccSmemMaxK;
  float* Sacc = sacc_smem ? reinterpret_cast<float*>(list + LIST_CAP) : part;
  const int64_t sk = sacc_smem ? BM : 1, sm_ = sacc_smem ? 1 : p.K;
  __shared__ int s_nlist;
  __shared__ int s_last;

  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int tx = t & 15, ty = t >> 4;
  const int j = blockIdx.x;          // D split
  const int i = blockIdx.y;          // N tile
  const int td0 = (int)((int64_t)j * p.Td / p.R);
  const int td1 = (int)((int64_t)(j + 1) * p.Td / p.R);
  const int KS = (int)(p.Fp / BK);
  const int total = (td1 - td0) * KS;
  const float* Xtile = p.Xt + (int64_t)i * p.Fp * BM;

  for (int e = t; e < p.K * BM; e += THREADS) Sacc[e] = 0.f;  // same extent in both layouts
  if (t == 0) s_nlist = 0;

  auto load_stage = [&](int it, int stage) {
    const int tile = td0 + it / KS, ks = it % KS;
    const int64_t f0 = (int64_t)ks * BK;
    const int64_t d0 = (int64_t)tile * BN;
    float* as = As + stage * BK * BM;
    float* bs = Bs + stage * BK * BN;
    const float* xa = Xtile + f0 * BM;
#pragma unroll
    for (int u = 0; u < BK * BM / 4 / THREADS; ++u) {
      const int q = t + THREADS * u;       // float4 index 0..BK*32-1
      cp_async16(as + 4 * q, xa + 4 * q);
      const int row = q >> 5, c4 = q & 31;
      cp_async16(bs + row * BN + 4 * c4, p.Bp + (f0 + row) * p.Dp + d0 + 4 * c4);
    }
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < total) load_stage(s, s);
    cp_async_commit();
  }

  // 8 x 8 outputs as float2 pairs (b, b + 1): FFMA2, two FMAs per instruction, each
  // element still accumulated in k order
  float2 acc2[8][4];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc2[a][b] = make_float2(0.f, 0.f);
#define ACC(a, b) (((b) & 1) ? acc2[a][(b) >> 1].y : acc2[a][(b) >> 1].x)

  for (int it = 0; it < total; ++it) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nit = it + STAGES - 1;
      if (nit < total) load_stage(nit, nit % STAGES);
      cp_async_commit();
    }
    const float* as = As + (it % STAGES) * BK * BM;
    const float* bs = Bs + (it % STAGES) * BK * BN;
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      const float4 a0 = *reinterpret_cast<const float4*>(as + k * BM + ty * 4);
      const float4 a1 = *reinterpret_cast<const float4*>(as + k * BM + 64 + ty * 4);
      const float4 b0 = *reinterpret_cast<const float4*>(bs + k * BN + tx * 4);
      const float4 b1 = *reinterpret_cast<const float4*>(bs + k * BN + 64 + tx * 4);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float2 bp[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                            make_float2(b1.z, b1.w)};
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc2[a][b] = ffma2(av[a], bp[b], acc2[a][b]);
    }

    if (it % KS == KS - 1) {
      // ------------------------------------------------ epilogue of one D-tile
      const int tile = td0 + it / KS;
      const int64_t d0 = (int64_t)tile * BN;
      float xn[8], bn[8];
#pragma unroll
      for (int a = 0; a < 8; ++a)
        xn[a] = __ldg(p.xnorm + (int64_t)i * BM + (a < 4 ? ty * 4 + a : 64 + ty * 4 + a - 4));
#pragma unroll
      for (int b = 0; b < 8; ++b)
        bn[b] = __ldg(p.bnorm + d0 + (b < 4 ? tx * 4 + b : 64 + tx * 4 + b - 4));
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const int c = b < 4 ? tx * 4 + b : 64 + tx * 4 + b - 4;
        float h[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          const float v = ACC(a, b);
          h[a] = hardsign(v);
          const int r = a < 4 ? ty * 4 + a : 64 + ty * 4 + a - 4;
          if (p.recheck && fabsf(v) <= p.tau_coef * xn[a] * bn[b] + kSignBoundAbs &&
              (int64_t)i * BM + r < p.N && d0 + c < p.D) {
            const int slot = atomicAdd(&s_nlist, 1);
            if (slot < LIST_CAP) {
              list[slot] = r * BN + c;
            } else {  // list full: this thread re-evaluates on its own (rare)
              const int64_t row = (int64_t)i * BM + r;
              double s = 0.0;
              for (int64_t f = 0; f < p.F; ++f)
                s = fma((double)p.X[row * p.F + f], (double)p.Bt[(d0 + c) * p.Fp + f], s);
              h[a] = s >= 0.0 ? 1.f : -1.f;
            }
          }
        }
        *reinterpret_cast<float4*>(Hs + c * HS + ty * 4) = make_float4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<float4*>(Hs + c * HS + 64 + ty * 4) = make_float4(h[4], h[5], h[6], h[7]);
      }
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc2[a][b] = make_float2(0.f, 0.f);
      __syncthreads();
      const int nl = min(s_nlist, LIST_CAP);
      for (int q = warp; q < nl; q += THREADS / 32) {
        const int e = list[q];
        const int r = e / BN, c = e % BN;
        const float h = recheck_sign_warp(p.X + ((int64_t)i * BM + r) * p.F,
                                          p.Bt + (d0 + c) * p.Fp, p.F, lane);
        if (lane == 0) Hs[c * HS + r] = h;
      }
      if (t == 0 && s_nlist > 0) atomicAdd(p.recheck_count, (unsigned long long)s_nlist);
      __syncthreads();
      if (t == 0) s_nlist = 0;
      // Stage II: Sacc[k][m] += sum_c H[m, c] C[k, d0 + c]  (thread: row m, half of K)
      {
        const int m = t & (BM - 1), kh = t >> 7;
        const int kper = (int)((p.K + 1) / 2);
        const int k0 = kh * kper, k1 = min((int)p.K, k0 + kper);
        for (int kc = k0; kc < k1; kc += 8) {
          float s[8];
          const int kn = min(8, k1 - kc);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) s[kk] = kk < kn ? Sacc[(kc + kk) * sk + m * sm_] : 0.f;
          for (int c4 = 0; c4 < BN / 4; ++c4) {
            const float h0 = Hs[(4 * c4 + 0) * HS + m], h1 = Hs[(4 * c4 + 1) * HS + m];
            const float h2 = Hs[(4 * c4 + 2) * HS + m], h3 = Hs[(4 * c4 + 3) * HS + m];
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              if (kk < kn) {
                const float4 cv =
                    __ldg(reinterpret_cast<const float4*>(p.Cp + (int64_t)(kc + kk) * p.Dp + d0) + c4);
                s[kk] = fmaf(h0, cv.x, s[kk]);
                s[kk] = fmaf(h1, cv.y, s[kk]);
                s[kk] = fmaf(h2, cv.z, s[kk]);
                s[kk] = fmaf(h3, cv.w, s[kk]);
              }
            }
          }
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            if (kk < kn) Sacc[(kc + kk) * sk + m * sm_] = s[kk];
        }
      }
      // the next iteration's __syncthreads orders Stage II before the next Hs writes
    }
  }
  cp_async_wait<0>();
  __syncthreads();

  // ---- partial scores of this D range -> workspace; last CTA of the N-tile reduces.
  if (sacc_smem) {
    for (int e = t; e < BM * p.K; e += THREADS) {
      const int m = e / (int)p.K, k = e % (int)p.K;
      part[e] = Sacc[k * BM + m];
    }
  }
  __threadfence();
  __syncthreads();
  if (t == 0) s_last = (atomicAdd(p.cnt + i, 1u) == (unsigned)(p.R - 1));
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const float* base = p.S_part + (int64_t)i * BM * p.K;
  float* Sfin = Hs;  // [128][BM] scratch: classes handled in chunks of 128
  int best = 0;
  float bestv = 0.f;
  for (int kc = 0; kc < (int)p.K; kc += 128) {       // Hs holds 128 classes x BM rows
    const int kn = min(128, (int)p.K - kc);
    for (int e = t; e < BM * kn; e += THREADS) {
      const int m = e / kn, k = kc + e % kn;
      const int64_t off = (int64_t)m * p.K + k;
      float s = ld_cg(base + off);
      for (int jj = 1; jj < p.R; ++jj) s += ld_cg(base + (int64_t)jj * Np * p.K + off);
      Sfin[(k - kc) * BM + m] = s;
      const int64_t row = (int64_t)i * BM + m;
      if (p.scores && row < p.N) p.scores[row * p.K + k] = s;
    }
    __syncthreads();
    if (t < BM) {
      for (int k = 0; k < kn; ++k) {
        const float v = Sfin[k * BM + t];
        if ((kc == 0 && k == 0) || v > bestv) { bestv = v; best = kc + k; }
      }
    }
    __syncthreads();
  }
  if (t == 0) p.cnt[i] = 0u;
  if (p.labels && t < BM) {
    const int64_t row = (int64_t)i * BM + t;
    if (row < p.N) p.labels[row] = best;
  }
}

}  // namespace

size_t fused_ffma_smem_bytes(int64_t K) {
  return sizeof(float) * ((size_t)STAGES * BK * (BM + BN) + (size_t)BN * HS +
                          (K <= kSaccSmemMaxK ? (size_t)K * BM : 0)) +
         sizeof(int) * LIST_CAP;
}

int fused_choose_splits(int64_t Tn, int64_t Td, int num_sms) {
  // minimise waves * (D tiles per CTA) with one resident CTA per SM
  int best = 1;
  double best_cost = 1e30;
  for (int R = 1; R <= Td; ++R) {
    const double waves = (double)((Tn * R + num_sms - 1) / num_sms);
    const double per = (double)((Td + R - 1) / R);
    const double cost = waves * per + 0.02 * R;  // small penalty for more partials
    if (cost < best_cost) {
      best_cost = cost;
      best = R;
    }
  }
  return best;
}

cudaError_t launch_prep_x(const float* X, int64_t N, int64_t F, int64_t Fp, float* Xt, float* xnorm,
                          cudaStream_t st) {
  const int64_t Tn = (N + BM - 1) / BM;
  prep_x_kernel<<<(unsigned)Tn, 256, 0, st>>>(X, N, F, Fp, Xt, xnorm);
  return cudaGetLastError();
}

cudaError_t launch_fused_ffma(const ModelView& m, const FusedWorkspace& ws, const float* X, int64_t N,
                              float* scores, int32_t* labels, bool recheck, int R,
                              cudaStream_t st) {
  FusedParams p;
  p.Xt = ws.Xt;
  p.X = X;
  p.xnorm = ws.xnorm;
  p.N = N;
  p.F = m.F;
  p.Fp = m.Fp;
  p.D = m.D;
  p.Dp = m.Dp;
  p.K = m.K;
  p.Bp = m.Bp;
  p.Bt = m.Bt;
  p.Cp = m.Cp;
  p.bnorm = m.bnorm;
  p.tau_coef = m.tau_coef;
  p.recheck = recheck ? 1 : 0;
  p.Tn = (int)((N + BM - 1) / BM);
  p.Td = (int)((m.D + BN - 1) / BN);
  p.R = R;
  p.S_part = ws.S_part;
  p.cnt = ws.cnt;
  p.recheck_count = ws.recheck;
  p.scores = scores;
  p.labels = labels;
  const size_t sm = fused_ffma_smem_bytes(m.K);
  cudaError_t e = cudaFuncSetAttribute(fused_ffma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sm);
  if (e != cudaSuccess) return e;
  fused_ffma_kernel<<<dim3((unsigned)R, (unsigned)p.Tn), THREADS, sm, st>>>(p);
  return cudaGetLastError();
}

}  // namespace hdc
