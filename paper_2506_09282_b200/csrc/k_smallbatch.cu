// k_smallbatch.cu -- K2: bandwidth-bound small-batch HDC inference (N <= 32).
//
// Computes, for up to 32 rows of X, the whole of Alg. 1:
//   V = X B (fp32 FFMA), H = HardSign(V) (eq. hardsign), S = H C^T,
//   y = argmax_k S (lowest index on ties).
// Partitioning follows ScalableHD-S (Alg. 3; text P:355): the D axis
// is split across CTAs; each CTA streams its B[:, d-tile] and C[:, d-tile] from
// HBM exactly once, forms the complete F-sum for its columns (HardSign needs all
// of F), applies HardSign, and contracts with the C tile into a partial S
// (N x K, the paper's S_local).  Partials are summed in a FIXED order by the
// last-arriving CTA of each group of 16 tiles and then by the last group
// (the paper's critical-section `S += S_local`), which also takes the
// row argmax -- one launch, no float atomics, bit-deterministic.
//
// HDC_PREC_FP32 sign exactness: every |v| <= tau = c_F ||x_n|| ||b_d|| is
// re-evaluated in float64 (warp-cooperative, fixed reduction order).
#include "common.cuh"
#include "kernels.h"

namespace hdc {
namespace {

constexpr int kDT = 32;        // columns per CTA (8 lanes x float4)
constexpr int kThreads = 128;  // 4 warps x 4 row-groups
constexpr int kRG = 16;        // row groups (each owns U consecutive B rows per chunk)
constexpr int kU = 8;          // B rows per row-group per chunk
constexpr int kFC = kRG * kU;  // F rows per chunk (== kThreads: one X column per thread)
constexpr int kGS = 16;        // tiles per first-level reduction group
static_assert(kFC == kThreads, "X fill assumes one chunk column per thread");

struct SmallParams {
  const float* X;
  int nrows;
  int64_t F, D, Dp, K;
  const float* Bp;
  const float* Cp;
  const float* bnorm;
  float tau_coef;
  int recheck;
  int G, G1;
  float* S_part;
  float* S_grp;
  unsigned* cnt1;
  unsigned* cnt2;
  unsigned long long* recheck_count;
  float* scores;
  int32_t* labels;
};

template <int NB>
__global__ void __launch_bounds__(kThreads)
smallbatch_kernel(const SmallParams p) {
  extern __shared__ __align__(16) float smem[];
  float* Xs = smem;                                  // [NB][kFC]   (main loop)
  float* red = smem;                                 // [4][NB][kDT] (after the loop)
  float* Sfin = smem;                                // [NB][K]     (final reduction)
  const int union_floats = (int)(p.K > kFC ? NB * p.K : NB * kFC);
  float* Hs = smem + union_floats;                   // [NB][kDT+1]
  float* xsq_red = Hs + NB * (kDT + 1);              // [4][NB]
  float* xnorm = xsq_red + 4 * NB;                   // [NB]
  int* list = reinterpret_cast<int*>(xnorm + NB);    // [NB*kDT]
  __shared__ int s_nlist;
  __shared__ int s_last;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rg = warp * 4 + (lane >> 3);
  const int q = lane & 7;
  const int64_t d0 = (int64_t)blockIdx.x * kDT;
  const int nrows = p.nrows;
  if (tid == 0) s_nlist = 0;

  float acc[NB][4];
  float xsq[NB];
#pragma unroll
  for (int n = 0; n < NB; ++n) {
    acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
    xsq[n] = 0.f;
  }

  const float* bcol = p.Bp + d0 + 4 * q;
  for (int64_t f0 = 0; f0 < p.F; f0 += kFC) {
    // (1) issue this chunk's B loads first: they overlap the X fill below.
    float4 bv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t f = f0 + rg * kU + u;
      bv[u] = f < p.F ? ldg_stream(bcol + f * p.Dp) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    // (2) X chunk -> smem (row n, chunk column tid); ||x_n||^2 partials.
    __syncthreads();
    {
      const int64_t f = f0 + tid;
#pragma unroll
      for (int n = 0; n < NB; ++n) {
        const float x = (n < nrows && f < p.F) ? __ldg(p.X + (int64_t)n * p.F + f) : 0.f;
        Xs[n * kFC + tid] = x;
        xsq[n] = fmaf(x, x, xsq[n]);
      }
    }
    __syncthreads();
    // (3) V partials: acc[n][j] += x[n, f] * B[f, d0 + 4q + j], f ascending.
#pragma unroll
    for (int n = 0; n < NB; ++n) {
      const float4 xa = *reinterpret_cast<const float4*>(Xs + n * kFC + rg * kU);
      const float4 xb = *reinterpret_cast<const float4*>(Xs + n * kFC + rg * kU + 4);
      const float xs[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        acc[n][0] = fmaf(xs[u], bv[u].x, acc[n][0]);
        acc[n][1] = fmaf(xs[u], bv[u].y, acc[n][1]);
        acc[n][2] = fmaf(xs[u], bv[u].z, acc[n][2]);
        acc[n][3] = fmaf(xs[u], bv[u].w, acc[n][3]);
      }
    }
  }

  // ---- complete the F-sum: 4 row groups per warp (xor 8, 16), then 4 warps in smem.
#pragma unroll
  for (int n = 0; n < NB; ++n) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float v = acc[n][j];
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      acc[n][j] = v;
    }
    const float s = warp_sum_xor(xsq[n]);
    if (lane == 0) xsq_red[warp * NB + n] = s;
  }
  __syncthreads();  // Xs no longer read
  if (lane < 8) {
#pragma unroll
    for (int n = 0; n < NB; ++n)
      *reinterpret_cast<float4*>(red + (warp * NB + n) * kDT + 4 * q) =
          make_float4(acc[n][0], acc[n][1], acc[n][2], acc[n][3]);
  }
  if (tid < NB)
    xnorm[tid] = sqrtf(((xsq_red[tid] + xsq_red[NB + tid]) + xsq_red[2 * NB + tid]) +
                       xsq_red[3 * NB + tid]);
  __syncthreads();

  // ---- V, HardSign, flag sign decisions inside the fp32 error bound.
  for (int e = tid; e < NB * kDT; e += kThreads) {
    const int n = e / kDT, c = e % kDT;
    const float v = ((red[(0 * NB + n) * kDT + c] + red[(1 * NB + n) * kDT + c]) +
                     red[(2 * NB + n) * kDT + c]) +
                    red[(3 * NB + n) * kDT + c];
    if (p.recheck && n < nrows && d0 + c < p.D) {
      const float tau = p.tau_coef * xnorm[n] * __ldg(p.bnorm + d0 + c) + kSignBoundAbs;
      if (fabsf(v) <= tau) list[atomicAdd(&s_nlist, 1)] = e;
    }
    Hs[n * (kDT + 1) + c] = hardsign(v);
  }
  __syncthreads();

  // ---- float64 re-evaluation of the flagged pre-activations (one warp per item).
  const int nl = s_nlist;
  for (int i = warp; i < nl; i += kThreads / 32) {
    const int e = list[i];
    const int n = e / kDT, c = e % kDT;
    const float* xr = p.X + (int64_t)n * p.F;
    const float* bc = p.Bp + d0 + c;
    double s = 0.0;
    for (int64_t f = lane; f < p.F; f += 32) s = fma((double)__ldg(xr + f), (double)__ldg(bc + f * p.Dp), s);
    s = warp_sum_xor(s);
    if (lane == 0) Hs[n * (kDT + 1) + c] = s >= 0.0 ? 1.f : -1.f;
  }
  if (tid == 0 && nl > 0) atomicAdd(p.recheck_count, (unsigned long long)nl);
  __syncthreads();

  // ---- Stage II partial for this D tile: S_local[n, k] = sum_c H[n, c] C[k, d0 + c].
  float* mypart = p.S_part + (int64_t)blockIdx.x * NB * p.K;
  for (int e = tid; e < nrows * p.K; e += kThreads) {
    const int n = e / (int)p.K, k = e % (int)p.K;
    const float* cr = p.Cp + (int64_t)k * p.Dp + d0;
    const float* hr = Hs + n * (kDT + 1);
    float s = 0.f;
#pragma unroll
    for (int c4 = 0; c4 < kDT / 4; ++c4) {
      const float4 cv = __ldg(reinterpret_cast<const float4*>(cr) + c4);
      s = fmaf(hr[4 * c4 + 0], cv.x, s);
      s = fmaf(hr[4 * c4 + 1], cv.y, s);
      s = fmaf(hr[4 * c4 + 2], cv.z, s);
      s = fmaf(hr[4 * c4 + 3], cv.w, s);
    }
    mypart[e] = s;
  }

  // ---- level 1: last CTA of each group of kGS tiles sums the group in tile order.
  __threadfence();
  __syncthreads();
  const int g = blockIdx.x / kGS;
  const int gsz = min(kGS, p.G - g * kGS);
  if (tid == 0) s_last = (atomicAdd(p.cnt1 + g, 1u) == (unsigned)(gsz - 1));
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int nk = nrows * (int)p.K;
  const float* gpart = p.S_part + (int64_t)g * kGS * NB * p.K;
  for (int e = tid; e < nk; e += kThreads) {
    float s = ld_cg(gpart + e);
    for (int j = 1; j < gsz; ++j) s += ld_cg(gpart + (int64_t)j * NB * p.K + e);
    p.S_grp[(int64_t)g * NB * p.K + e] = s;
  }
  if (tid == 0) p.cnt1[g] = 0u;
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(p.cnt2, 1u) == (unsigned)(p.G1 - 1));
  __syncthreads();
  if (!s_last) return;
  __threadfence();

  // ---- level 2: the last group sums the group partials in group order; argmax.
  for (int e = tid; e < nk; e += kThreads) {
    float s = ld_cg(p.S_grp + e);
    for (int j = 1; j < p.G1; ++j) s += ld_cg(p.S_grp + (int64_t)j * NB * p.K + e);
    Sfin[e] = s;
    if (p.scores) p.scores[e] = s;
  }
  if (tid == 0) *p.cnt2 = 0u;
  __syncthreads();
  if (p.labels) {
    for (int n = tid; n < nrows; n += kThreads) {
      const float* sr = Sfin + n * p.K;
      int best = 0;
      float bv = sr[0];
      for (int k = 1; k < (int)p.K; ++k)
        if (sr[k] > bv) { bv = sr[k]; best = k; }
      p.labels[n] = best;
    }
  }
}

template <int NB>
size_t smem_bytes(int64_t K) {
  const int64_t uni = K > kFC ? NB * K : NB * kFC;
  return sizeof(float) * (uni + NB * (kDT + 1) + 4 * NB + NB) + sizeof(int) * NB * kDT;
}

template <int NB>
cudaError_t launch_nb(const SmallParams& p, cudaStream_t st) {
  const size_t sm = smem_bytes<NB>(p.K);  // <= 41 KB for NB = 32, K = 256: no opt-in
  smallbatch_kernel<NB><<<p.G, kThreads, sm, st>>>(p);
  return cudaGetLastError();
}

}  // namespace

int64_t small_num_tiles(int64_t D) { return (D + kDT - 1) / kDT; }
int64_t small_num_groups(int64_t D) { return (small_num_tiles(D) + kGS - 1) / kGS; }

cudaError_t launch_smallbatch(const ModelView& m, const SmallWorkspace& ws, const float* X, int n,
                              float* scores, int32_t* labels, bool recheck, cudaStream_t st) {
  SmallParams p;
  p.X = X;
  p.nrows = n;
  p.F = m.F;
  p.D = m.D;
  p.Dp = m.Dp;
  p.K = m.K;
  p.Bp = m.Bp;
  p.Cp = m.Cp;
  p.bnorm = m.bnorm;
  p.tau_coef = m.tau_coef;
  p.recheck = recheck ? 1 : 0;
  p.G = (int)small_num_tiles(m.D);
  p.G1 = (int)small_num_groups(m.D);
  p.S_part = ws.S_part;
  p.S_grp = ws.S_grp;
  p.cnt1 = ws.cnt1;
  p.cnt2 = ws.cnt2;
  p.recheck_count = ws.recheck;
  p.scores = scores;
  p.labels = labels;
  if (n <= 1) return launch_nb<1>(p, st);
  if (n <= 2) return launch_nb<2>(p, st);
  if (n <= 4) return launch_nb<4>(p, st);
  if (n <= 8) return launch_nb<8>(p, st);
  if (n <= 16) return launch_nb<16>(p, st);
  return launch_nb<32>(p, st);
}

}  // namespace hdc
