// k_smallbatch.cu -- K2: bandwidth-bound small-batch HDC inference (N <= 32).
//
// Computes, for up to 32 rows of X, the whole of Alg. 1:
//   V = X B (fp32 FFMA), H = HardSign(V) (eq. hardsign), S = H C^T,
//   y = argmax_k S (lowest index on ties).
// Partitioning follows ScalableHD-S (Alg. 3; text P:355): the D axis
// is split across one CTA per SM; each CTA streams its contiguous column range
// of B (and C) from HBM exactly once with deep 128-bit load pipelining, forms
// the complete F-sum for its columns (HardSign needs all of F), applies
// HardSign, and contracts with its C columns into a partial S (the paper's
// S_local).  The last-arriving CTA sums the 148 partials in a FIXED order (the
// paper's critical-section `S += S_local`) and takes the row argmax
// (P:340-342): one launch, no floating-point atomics, bit-deterministic.
//
// HDC_PREC_FP32 sign exactness: every |v| <= tau = c_F ||x_n|| ||b_d|| is
// re-evaluated in float64 (warp-cooperative, fixed reduction order).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace hdc {
namespace {

constexpr int kThreads = 256;
constexpr int kPassUnits = 64;     // float4 column units per pass (256 columns)
constexpr int kMaxCTAs = 1024;

struct SmallParams {
  const float* X;
  int nrows;
  int64_t F, D, Dp, K;
  const float* Bp;
  const float* B4;       // unit-major copy of B: [units][Fp][4]
  int64_t Fp;
  const float* Cp;
  const float* bnorm;
  float tau_coef;
  int recheck;
  int G;                 // CTAs (contiguous column-unit ranges)
  int alias;             // single pass: the F-sum buffers reuse the X region
  int64_t units;         // ceil(D / 4) float4 column units
  float* S_part;         // [G][NB][K]
  unsigned* cnt;         // [1], zero between launches
  unsigned long long* recheck_count;
  unsigned long long* dbg;   // diagnostics (HDC_SMALL_DEBUG): per-phase cycle sums of thread 0
  float* scores;
  int32_t* labels;
};

// Diagnostics (HDC_SMALL_DEBUG): thread 0 of each CTA adds per-phase cycles.
#define PHASE(i)                                                              \
  do {                                                                        \
    if (p.dbg && tid == 0) {                                                  \
      const long long _t = clock64();                                         \
      atomicAdd(p.dbg + (i), (unsigned long long)(_t - tph));                 \
      tph = _t;                                                               \
    }                                                                         \
  } while (0)

template <int NB>
__host__ __device__ constexpr int chunk_rows() { return NB <= 4 ? 24 : (NB <= 8 ? 16 : 8); }

template <int NB>
__global__ void __launch_bounds__(kThreads, 1)
smallbatch_kernel(const SmallParams p) {
  constexpr int CH = chunk_rows<NB>();   // B rows per thread per pipeline chunk
  constexpr int XS = NB + 4;             // Xs row stride (f-major, float4 aligned)
  extern __shared__ __align__(16) float smem[];
  __shared__ float xnorm_s[NB];
  __shared__ int s_nlist;
  __shared__ int s_last;
  __shared__ int s_list[1024];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = blockIdx.x;
  const int64_t u0 = (int64_t)c * p.units / p.G, u1 = (int64_t)(c + 1) * p.units / p.G;
  const int nrows = p.nrows;
  const int64_t F = p.F;
  long long tph = clock64();

  // smem: [Sacc NB*K | Xs F*XS | (red | Hs)]; red/Hs overlay Xs when there is one pass.
  float* Sacc = smem;                                  // S_local accumulator, [NB][K]
  float* Xs = smem + ((NB * p.K + 3) & ~int64_t(3));
  // ---- X (nrows x F) -> smem, f-major [F][XS]; ||x_n||^2 by warp n (fixed order).
  for (int64_t f = tid; f < F; f += kThreads) {
    float xv[NB];
#pragma unroll
    for (int n = 0; n < NB; ++n) xv[n] = n < nrows ? __ldg(p.X + (int64_t)n * F + f) : 0.f;
#pragma unroll
    for (int n4 = 0; n4 < (NB + 3) / 4; ++n4) {
      float4 v;
      v.x = xv[4 * n4];
      v.y = 4 * n4 + 1 < NB ? xv[4 * n4 + 1] : 0.f;
      v.z = 4 * n4 + 2 < NB ? xv[4 * n4 + 2] : 0.f;
      v.w = 4 * n4 + 3 < NB ? xv[4 * n4 + 3] : 0.f;
      *reinterpret_cast<float4*>(Xs + f * XS + 4 * n4) = v;
    }
  }
  if (tid == 0) s_nlist = 0;
  __syncthreads();
  for (int n = warp; n < NB; n += kThreads / 32) {
    float ss = 0.f;
    for (int64_t f = lane; f < F; f += 32) ss = fmaf(Xs[f * XS + n], Xs[f * XS + n], ss);
    ss = warp_sum_xor(ss);
    if (lane == 0) xnorm_s[n] = sqrtf(ss);
  }
  __syncthreads();

  PHASE(0);
  float* red = p.alias ? Xs : Xs + F * XS;            // [RG][NB][PW*4] F-sum partials
  for (int i = tid; i < NB * p.K; i += kThreads) Sacc[i] = 0.f;

  for (int64_t pu0 = u0; pu0 < u1; pu0 += kPassUnits) {
    const int PW = (int)(u1 - pu0 < kPassUnits ? u1 - pu0 : kPassUnits);   // units in this pass
    const int RG = kThreads / PW;                            // row groups
    const int g = tid / PW, u = tid % PW;
    const bool active = g < RG;
    const float* bcol = p.Bp + (pu0 + u) * 4;

    float acc[NB][4];
#pragma unroll
    for (int n = 0; n < NB; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;

    // software-pipelined streaming of this thread's rows f = g, g+RG, ...:
    // CH loads in flight per thread while the previous chunk is consumed.
    float4 b0[CH], b1[CH];
    const int64_t rows_per = active ? (F - g + RG - 1) / RG : 0;
    const int64_t nch = (rows_per + CH - 1) / CH;
    auto issue = [&](int64_t ch, float4 (&buf)[CH]) {
#pragma unroll
      for (int r = 0; r < CH; ++r) {
        const int64_t f = g + (ch * CH + r) * (int64_t)RG;
        buf[r] = f < F ? ldg_stream(bcol + f * p.Dp) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    auto consume = [&](int64_t ch, const float4 (&buf)[CH]) {
#pragma unroll
      for (int r = 0; r < CH; ++r) {
        const int64_t f = g + (ch * CH + r) * (int64_t)RG;
        if (f < F) {
          const float4 b = buf[r];
          const float* xr = Xs + f * XS;
#pragma unroll
          for (int n4 = 0; n4 < (NB + 3) / 4; ++n4) {
            const float4 xv = *reinterpret_cast<const float4*>(xr + 4 * n4);
            const float xs[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int n = 4 * n4 + j;
              if (n < NB) {
                acc[n][0] = fmaf(xs[j], b.x, acc[n][0]);
                acc[n][1] = fmaf(xs[j], b.y, acc[n][1]);
                acc[n][2] = fmaf(xs[j], b.z, acc[n][2]);
                acc[n][3] = fmaf(xs[j], b.w, acc[n][3]);
              }
            }
          }
        }
      }
    };
    // two register buffers, statically indexed: loads of chunk c+1 are in flight
    // while chunk c is consumed
    if (nch > 0) issue(0, b0);
    for (int64_t ch = 0; ch < nch; ch += 2) {
      if (ch + 1 < nch) issue(ch + 1, b1);
      consume(ch, b0);
      if (ch + 1 < nch) {
        if (ch + 2 < nch) issue(ch + 2, b0);
        consume(ch + 1, b1);
      }
    }

    // ---- complete the F-sum over the RG row groups (fixed order g = 0..RG-1)
    __syncthreads();   // every thread is done with Xs (red may overlay it)
    PHASE(1);
    if (active) {
#pragma unroll
      for (int n = 0; n < NB; ++n)
        *reinterpret_cast<float4*>(red + ((int64_t)g * NB + n) * (PW * 4) + 4 * u) =
            make_float4(acc[n][0], acc[n][1], acc[n][2], acc[n][3]);
    }
    __syncthreads();
    float* Hs = red + (int64_t)RG * NB * PW * 4;            // [NB][PW*4] +-1
    const int PC = PW * 4;
    for (int e = tid; e < NB * PC; e += kThreads) {
      const int n = e / PC, col = e % PC;
      float v = red[(int64_t)n * PC + col];
      for (int gg = 1; gg < RG; ++gg) v += red[((int64_t)gg * NB + n) * PC + col];
      const int64_t d = pu0 * 4 + col;
      if (p.recheck && n < nrows && d < p.D) {
        const float tau = p.tau_coef * xnorm_s[n] * __ldg(p.bnorm + d) + kSignBoundAbs;
        if (fabsf(v) <= tau) {
          const int slot = atomicAdd(&s_nlist, 1);
          if (slot < 1024) s_list[slot] = e;
          else {  // list full: this thread re-evaluates (rare)
            double s = 0.0;
            for (int64_t f = 0; f < F; ++f) s = fma((double)p.X[(int64_t)n * F + f], (double)p.Bp[f * p.Dp + d], s);
            v = s >= 0.0 ? 1.f : -1.f;
          }
        }
      }
      Hs[e] = hardsign(v);
    }
    __syncthreads();
    PHASE(2);
    // ---- float64 re-evaluation of flagged pre-activations (one warp per item)
    const int nl = min(s_nlist, 1024);
    for (int i = warp; i < nl; i += kThreads / 32) {
      const int e = s_list[i];
      const int n = e / PC, col = e % PC;
      const int64_t d = pu0 * 4 + col;
      const float* xr = p.X + (int64_t)n * F;
      double s = 0.0;
      for (int64_t f = lane; f < F; f += 32) s = fma((double)__ldg(xr + f), (double)__ldg(p.Bp + f * p.Dp + d), s);
      s = warp_sum_xor(s);
      if (lane == 0) Hs[e] = s >= 0.0 ? 1.f : -1.f;
    }
    if (tid == 0 && s_nlist > 0) atomicAdd(p.recheck_count, (unsigned long long)s_nlist);
    __syncthreads();
    PHASE(3);
    if (tid == 0) s_nlist = 0;
    // ---- Stage II partial: Sacc[n, k] += sum_col H[n, col] C[k, d0 + col]
    for (int e = tid; e < nrows * p.K; e += kThreads) {
      const int n = e / (int)p.K, k = e % (int)p.K;
      const float* cr = p.Cp + (int64_t)k * p.Dp + pu0 * 4;
      const float* hr = Hs + (int64_t)n * PC;
      float s = Sacc[e];
      for (int c4 = 0; c4 < PW; ++c4) {
        const float4 cv = __ldg(reinterpret_cast<const float4*>(cr) + c4);
        s = fmaf(hr[4 * c4 + 0], cv.x, s);
        s = fmaf(hr[4 * c4 + 1], cv.y, s);
        s = fmaf(hr[4 * c4 + 2], cv.z, s);
        s = fmaf(hr[4 * c4 + 3], cv.w, s);
      }
      Sacc[e] = s;
    }
    __syncthreads();
  }

  PHASE(4);
  // ---- publish S_local; the last CTA sums all partials in CTA order and takes the argmax
  float* mypart = p.S_part + (int64_t)c * NB * p.K;
  for (int e = tid; e < nrows * p.K; e += kThreads) mypart[e] = Sacc[e];
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(p.cnt, 1u) == (unsigned)(p.G - 1));
  __syncthreads();
  PHASE(5);
  if (!s_last) return;
  __threadfence();
  const int nk = nrows * (int)p.K;
  float* Sfin = Sacc;  // reuse
  for (int e = warp; e < nk; e += kThreads / 32) {
    // lane j sums partials c = j, j+32, ... in order; then a fixed xor tree
    float s = 0.f;
    for (int cc = lane; cc < p.G; cc += 32) s += ld_cg(p.S_part + (int64_t)cc * NB * p.K + e);
    s = warp_sum_xor(s);
    if (lane == 0) {
      Sfin[e] = s;
      if (p.scores) p.scores[e] = s;
    }
  }
  if (tid == 0) *p.cnt = 0u;
  __syncthreads();
  PHASE(6);
  if (p.labels) {
    for (int n = tid; n < nrows; n += kThreads) {
      const float* sr = Sfin + (int64_t)n * p.K;
      int best = 0;
      float bv = sr[0];
      for (int k = 1; k < (int)p.K; ++k)
        if (sr[k] > bv) { bv = sr[k]; best = k; }
      p.labels[n] = best;
    }
  }
}

// ---------------------------------------------------------------------------
// K2w: warp-per-unit variant for NB <= 8 (bandwidth-bound regime).  B is read
// from the model's unit-major copy B4[u][f][4] (all F rows of a 4-column unit
// contiguous), so each warp streams one contiguous 16*F-byte run with fully
// coalesced 512-byte requests -- the access pattern that reaches the HBM copy
// rate (tools/stream_microbench.cu).  One warp per unit, one CTA per SM.
constexpr int kMaxUnitWarps = 17;   // 2500 units / 148 SMs at D = 10000

template <int NB>
__global__ void __launch_bounds__(32 * kMaxUnitWarps, 1)
smallbatch_warp_kernel(const SmallParams p) {
  constexpr int CH = NB <= 4 ? 8 : 4;
  constexpr int XS = ((NB + 3) / 4) * 4;
  extern __shared__ __align__(16) float smem[];
  __shared__ float xnorm_s[NB];
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nthreads = blockDim.x, W = nthreads >> 5;
  const int c = blockIdx.x;
  const int64_t u0 = (int64_t)c * p.units / p.G, u1 = (int64_t)(c + 1) * p.units / p.G;
  const int nrows = p.nrows;
  const int64_t F = p.F;
  const int K = (int)p.K;
  float* Xs = smem;                                        // [F][XS]
  float* Sw = smem + F * XS;                               // [W][NB*K] per-warp S_local
  long long tph = clock64();
  unsigned long long gt0 = 0;
  if (p.dbg && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt0));

  // start the HBM stream at once: each warp asks the TMA engine to prefetch its
  // first unit's contiguous run of B4 into L2 while X is staged
  if (lane == 0 && c + (int64_t)p.G * warp < p.units) {
    const float* bu = p.B4 + (c + (int64_t)p.G * warp) * p.Fp * 4;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(bu), "r"((uint32_t)(F * 16)) : "memory");
  }
  for (int64_t f = tid; f < F; f += nthreads) {
#pragma unroll
    for (int n = 0; n < XS; ++n)
      Xs[f * XS + n] = (n < NB && n < nrows) ? __ldg(p.X + (int64_t)n * F + f) : 0.f;
  }
  __syncthreads();
  for (int n = warp; n < NB; n += W) {
    float ss = 0.f;
    for (int64_t f = lane; f < F; f += 32) ss = fmaf(Xs[f * XS + n], Xs[f * XS + n], ss);
    ss = warp_sum_xor(ss);
    if (lane == 0) xnorm_s[n] = sqrtf(ss);
  }
  __syncthreads();
  PHASE(0);

  // units are dealt round-robin (unit u to CTA u mod G): each CTA's reads spread
  // over the whole of B, which evens out per-SM completion times
  for (int64_t jb = 0; c + p.G * jb < p.units; jb += W) {   // passes of W units
    const int64_t u = c + p.G * (jb + warp);
    const bool has = u < p.units;
    float* sw = Sw + (int64_t)warp * NB * K;
    if (has) {
      const float* bu = p.B4 + u * p.Fp * 4;
      float acc[NB][4];
#pragma unroll
      for (int n = 0; n < NB; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
      const int64_t R = (F + 31) / 32;                    // rows per lane
      const int64_t nch = (R + CH - 1) / CH;
      float4 b0[CH], b1[CH];
      auto issue = [&](int64_t ch, float4 (&buf)[CH]) {
#pragma unroll
        for (int r = 0; r < CH; ++r) {
          const int64_t f = lane + 32 * (ch * CH + r);
          buf[r] = f < F ? ldg_stream(bu + f * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      };
      auto consume = [&](int64_t ch, const float4 (&buf)[CH]) {
#pragma unroll
        for (int r = 0; r < CH; ++r) {
          const int64_t f = lane + 32 * (ch * CH + r);
          if (f < F) {
            const float4 b = buf[r];
#pragma unroll
            for (int n4 = 0; n4 < XS / 4; ++n4) {
              const float4 xv = *reinterpret_cast<const float4*>(Xs + f * XS + 4 * n4);
              const float xs[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const int n = 4 * n4 + j;
                if (n < NB) {
                  acc[n][0] = fmaf(xs[j], b.x, acc[n][0]);
                  acc[n][1] = fmaf(xs[j], b.y, acc[n][1]);
                  acc[n][2] = fmaf(xs[j], b.z, acc[n][2]);
                  acc[n][3] = fmaf(xs[j], b.w, acc[n][3]);
                }
              }
            }
          }
        }
      };
      if (nch > 0) issue(0, b0);
      for (int64_t ch = 0; ch < nch; ch += 2) {
        if (ch + 1 < nch) issue(ch + 1, b1);
        consume(ch, b0);
        if (ch + 1 < nch) {
          if (ch + 2 < nch) issue(ch + 2, b0);
          consume(ch + 1, b1);
        }
      }
      // complete the F-sum across lanes (fixed xor tree): every lane holds V[n][j]
#pragma unroll
      for (int n = 0; n < NB; ++n)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[n][j] = warp_sum_xor(acc[n][j]);
      // lane e < NB*4 owns element (n, j) = (e / 4, e % 4)
      float v = 0.f;
#pragma unroll
      for (int n = 0; n < NB; ++n)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (lane == n * 4 + j) v = acc[n][j];
      const int en = lane >> 2, ej = lane & 3;
      const int64_t d = u * 4 + ej;
      bool flag = false;
      if (p.recheck && lane < NB * 4 && en < nrows && d < p.D) {
        const float tau = p.tau_coef * xnorm_s[en] * __ldg(p.bnorm + d) + kSignBoundAbs;
        flag = fabsf(v) <= tau;
      }
      float h = hardsign(v);
      unsigned mask = __ballot_sync(0xffffffffu, flag);
      if (mask && lane == 0) atomicAdd(p.recheck_count, (unsigned long long)__popc(mask));
      while (mask) {            // float64 re-evaluation, fixed lane order
        const int src = __ffs(mask) - 1;
        mask &= mask - 1;
        const int sn = src >> 2, sj = src & 3;
        // X from shared memory, B from this warp's own unit run of B4 (just streamed,
        // L2-resident, 16-byte strided): no cold strided column gather
        const float* bu = p.B4 + u * p.Fp * 4 + sj;
        double s = 0.0;
#pragma unroll 8
        for (int64_t f = lane; f < F; f += 32)
          s = fma((double)Xs[f * XS + sn], (double)__ldg(bu + f * 4), s);
        s = warp_sum_xor(s);
        if (lane == src) h = s >= 0.0 ? 1.f : -1.f;
      }
      // Stage II partial of this unit: sw[n*K + k] = sum_j H[n][j] C[k][4u + j]
      for (int q0 = 0; q0 < nrows * K; q0 += 32) {   // warp-uniform trip count (shuffles)
        const int q = q0 + lane;
        const bool ok = q < nrows * K;
        const int n = ok ? q / K : 0, k = ok ? q % K : 0;
        // the 4 signs of row n live in lanes 4n .. 4n+3
        const float h0 = __shfl_sync(0xffffffffu, h, (4 * n + 0) & 31);
        const float h1 = __shfl_sync(0xffffffffu, h, (4 * n + 1) & 31);
        const float h2 = __shfl_sync(0xffffffffu, h, (4 * n + 2) & 31);
        const float h3 = __shfl_sync(0xffffffffu, h, (4 * n + 3) & 31);
        if (ok) {
          const float4 cv = __ldg(reinterpret_cast<const float4*>(p.Cp + (int64_t)k * p.Dp + u * 4));
          float s = fmaf(h0, cv.x, 0.f);
          s = fmaf(h1, cv.y, s);
          s = fmaf(h2, cv.z, s);
          s = fmaf(h3, cv.w, s);
          sw[q] = (jb == 0) ? s : sw[q] + s;
        }
      }
    } else if (jb == 0) {
      for (int q = lane; q < nrows * K; q += 32) sw[q] = 0.f;
    }
  }
  __syncthreads();
  PHASE(1);
  // CTA S_local = sum over warps in order; publish
  float* mypart = p.S_part + (int64_t)c * NB * p.K;
  for (int q = tid; q < nrows * K; q += nthreads) {
    float s = Sw[q];
    for (int w = 1; w < W; ++w) s += Sw[(int64_t)w * NB * K + q];
    mypart[q] = s;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(p.cnt, 1u) == (unsigned)(p.G - 1));
  __syncthreads();
  PHASE(2);
  if (p.dbg && tid == 0) {
    unsigned long long gt1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt1));
    atomicMin(p.dbg + 4, gt0);
    atomicMax(p.dbg + 5, gt0);
    atomicMin(p.dbg + 6, gt1);
    atomicMax(p.dbg + 7, gt1);
  }
  if (!s_last) return;
  __threadfence();
  // last CTA: pair q handled by an 8-lane group; lane s sums partials c = s, s+8, ...
  const int nk = nrows * K;
  float* Sfin = Sw;
  for (int q0 = 0; q0 < nk; q0 += nthreads / 8) {
    const int q = q0 + (tid >> 3), sl = tid & 7;
    float s = 0.f;
    if (q < nk)
      for (int cc = sl; cc < p.G; cc += 8) s += ld_cg(p.S_part + (int64_t)cc * NB * p.K + q);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    if (q < nk && sl == 0) {
      Sfin[q] = s;
      if (p.scores) p.scores[q] = s;
    }
  }
  if (tid == 0) *p.cnt = 0u;
  __syncthreads();
  if (p.labels) {
    for (int n = tid; n < nrows; n += nthreads) {
      const float* sr = Sfin + (int64_t)n * K;
      int best = 0;
      float bv = sr[0];
      for (int k = 1; k < K; ++k)
        if (sr[k] > bv) { bv = sr[k]; best = k; }
      p.labels[n] = best;
    }
  }
  PHASE(3);
}

template <int NB>
size_t smem_bytes(int64_t F, int64_t K, int64_t max_pass_units, bool alias) {
  const int64_t PW = max_pass_units, RG = kThreads / PW;
  const size_t xs = (size_t)F * (((NB + 3) / 4) * 4 + (NB >= 8 ? 4 : 0));
  const size_t rh = (size_t)RG * NB * PW * 4 + (size_t)NB * PW * 4;
  const size_t sacc = ((size_t)NB * K + 3) & ~size_t(3);
  return sizeof(float) * (sacc + (alias ? std::max(xs, rh) : xs + rh));
}

template <int NB>
cudaError_t launch_warp_nb(SmallParams p, cudaStream_t st) {
  const int64_t per = (p.units + p.G - 1) / p.G;
  const int W = (int)std::min<int64_t>(kMaxUnitWarps, per);
  constexpr int XS = ((NB + 3) / 4) * 4;
  const size_t sm = sizeof(float) * ((size_t)p.F * XS + (size_t)W * NB * p.K);
  if (sm > 220 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(smallbatch_warp_kernel<NB>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  static unsigned long long* dbg = nullptr;
  const bool debug = getenv("HDC_SMALL_DEBUG") != nullptr;
  if (debug) {
    if (!dbg) cudaMalloc((void**)&dbg, 8 * sizeof(unsigned long long));
    unsigned long long init[8] = {0, 0, 0, 0, ~0ull, 0, ~0ull, 0};
    cudaMemcpyAsync(dbg, init, sizeof(init), cudaMemcpyHostToDevice, st);
    cudaStreamSynchronize(st);
    p.dbg = dbg;
  }
  smallbatch_warp_kernel<NB><<<p.G, 32 * W, sm, st>>>(p);
  cudaError_t le = cudaGetLastError();
  if (debug && le == cudaSuccess) {
    unsigned long long h[8];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, dbg, sizeof(h), cudaMemcpyDeviceToHost);
    fprintf(stderr, "[hdc small-warp debug] NB=%d G=%d W=%d mean cycles/CTA: xfill=%.0f stream+unit=%.0f "
            "publish=%.0f | last CTA final=%.0f | CTA start spread %.2f us, end spread %.2f us, "
            "first start -> last publish %.2f us\n", NB, p.G, W, (double)h[0] / p.G, (double)h[1] / p.G,
            (double)h[2] / p.G, (double)h[3], (h[5] - h[4]) * 1e-3, (h[7] - h[6]) * 1e-3,
            (h[7] - h[4]) * 1e-3);
  }
  return le;
}

template <int NB>
cudaError_t launch_nb(SmallParams p, cudaStream_t st) {
  const int64_t per = (p.units + p.G - 1) / p.G;
  const int64_t maxpw = std::min<int64_t>(kPassUnits, per);
  p.alias = per <= kPassUnits ? 1 : 0;
  const size_t sm = smem_bytes<NB>(p.F, p.K, maxpw, p.alias != 0);
  if (sm > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(smallbatch_kernel<NB>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  static unsigned long long* dbg = nullptr;
  const bool debug = getenv("HDC_SMALL_DEBUG") != nullptr;
  if (debug) {
    if (!dbg) cudaMalloc((void**)&dbg, 8 * sizeof(unsigned long long));
    cudaMemsetAsync(dbg, 0, 8 * sizeof(unsigned long long), st);
    p.dbg = dbg;
  }
  smallbatch_kernel<NB><<<p.G, kThreads, sm, st>>>(p);
  cudaError_t le = cudaGetLastError();
  if (debug && le == cudaSuccess) {
    unsigned long long h[8];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, dbg, sizeof(h), cudaMemcpyDeviceToHost);
    fprintf(stderr, "[hdc small debug] NB=%d G=%d mean cycles/CTA: xfill=%.0f main=%.0f fsum=%.0f "
            "recheck=%.0f stage2=%.0f publish=%.0f | last CTA final=%.0f\n", NB, p.G,
            (double)h[0] / p.G, (double)h[1] / p.G, (double)h[2] / p.G, (double)h[3] / p.G,
            (double)h[4] / p.G, (double)h[5] / p.G, (double)h[6]);
  }
  return le;
}

}  // namespace

int64_t small_num_ctas(int64_t D, int num_sms) {
  const int64_t units = (D + 3) / 4;
  return std::min<int64_t>(units, std::min<int64_t>(num_sms, kMaxCTAs));
}

// Largest batch (of 1, 2, ..., 32 rows) the small kernel accepts for this shape
// (X and the F-sum buffers must fit in shared memory).
int small_max_rows(int64_t F, int64_t D, int64_t K, int num_sms) {
  const int64_t units = (D + 3) / 4, G = small_num_ctas(D, num_sms);
  const int64_t per = (units + G - 1) / G;
  const int64_t pw = std::min<int64_t>(kPassUnits, per);
  const bool alias = per <= kPassUnits;
  const size_t lim = 220 * 1024;
  if (smem_bytes<32>(F, K, pw, alias) <= lim) return 32;
  if (smem_bytes<16>(F, K, pw, alias) <= lim) return 16;
  if (smem_bytes<8>(F, K, pw, alias) <= lim) return 8;
  if (smem_bytes<4>(F, K, pw, alias) <= lim) return 4;
  if (smem_bytes<2>(F, K, pw, alias) <= lim) return 2;
  if (smem_bytes<1>(F, K, pw, alias) <= lim) return 1;
  return 0;
}

cudaError_t launch_smallbatch(const ModelView& m, const SmallWorkspace& ws, const float* X, int n,
                              float* scores, int32_t* labels, bool recheck, int num_sms,
                              cudaStream_t st) {
  SmallParams p;
  p.X = X;
  p.nrows = n;
  p.F = m.F;
  p.D = m.D;
  p.Dp = m.Dp;
  p.K = m.K;
  p.Bp = m.Bp;
  p.B4 = m.B4;
  p.Fp = m.Fp;
  p.Cp = m.Cp;
  p.bnorm = m.bnorm;
  p.tau_coef = m.tau_coef;
  p.recheck = recheck ? 1 : 0;
  p.units = (m.D + 3) / 4;
  p.G = (int)small_num_ctas(m.D, num_sms);
  p.S_part = ws.S_part;
  p.cnt = ws.cnt1;
  p.recheck_count = ws.recheck;
  p.dbg = nullptr;
  p.scores = scores;
  p.labels = labels;
  if (m.B4 && !getenv("HDC_SMALL_STRIPS")) {
    if (n <= 1) return launch_warp_nb<1>(p, st);
    if (n <= 2) return launch_warp_nb<2>(p, st);
    if (n <= 4) return launch_warp_nb<4>(p, st);
    if (n <= 8) return launch_warp_nb<8>(p, st);
  }
  if (n <= 1) return launch_nb<1>(p, st);
  if (n <= 2) return launch_nb<2>(p, st);
  if (n <= 4) return launch_nb<4>(p, st);
  if (n <= 8) return launch_nb<8>(p, st);
  if (n <= 16) return launch_nb<16>(p, st);
  return launch_nb<32>(p, st);
}

}  // namespace hdc
