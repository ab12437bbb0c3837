// k_small_tc.cu -- K2t: small-batch (N <= 32) sign-exact HDC inference on the int8
// tensor cores (HDC_PREC_FP32_TC models), sm_100a.
//
// The whole of Alg. 1 for up to 32 rows of X in one launch, bound by
// reading B once from HBM (the paper's ScalableHD-S partitioning, Alg. 3 P:315-344:
// each CTA owns a contiguous D-range, forms complete F-sums for its columns, applies
// HardSign and contracts with its C columns into a partial S -- the paper's S_local;
// the partials are summed, the paper's `S += S_local`).
//
// B200 mapping (what differs from the fp32 streaming kernel K2s):
//  * B is streamed as the model's int8x3 limb image of B^T ([3][Dq][Fp], 3 bytes per
//    element instead of 4): one TMA box of this CTA's <= 128 columns x 64 K-bytes per
//    limb and ring stage (SWIZZLE_64B), up to 8 stages in flight.
//  * Stage I on the tensor cores with D on M: A = the CTA's B^T limbs (M = 128 rows; the
//    rows past its range read neighbouring shared memory and are ignored), B = X's limbs
//    (N = 16 / 32 rows, built by every CTA in shared memory from the caller's fp32 X
//    with the same limb code as the staging kernel, tc_limbs.cuh), three kind::i8 MMAs
//    per k-step with exact int32 accumulation (the i + j <= 2 limb products).
//  * HardSign from the exact integer image, float64 re-evaluation of the signs inside
//    the rigorous bound (as in K4) -> every sign equals the exact one.
//  * Stage II (68 x N x K MACs per CTA) in fp32 FFMA, fixed order; the partial scores are
//    converted to int64 fixed point (2^-shift units) and summed by atomics: exact and
//    order-independent, so the result is bit-deterministic with no last-arriver read of
//    148 partials; the last CTA only converts N x K sums and takes the argmax.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tc_limbs.cuh"
#include "tc_ptx.cuh"

namespace hdc {
namespace {

using namespace ptx;

constexpr int kWarpsT = 10;                      // warp 0 TMA, warp 1 MMA, warps 2..9 workers
constexpr int kThreadsT = 32 * kWarpsT;
constexpr int kWorkers = 32 * (kWarpsT - 2);
constexpr int kKB = 64;                          // K bytes per ring stage (SWIZZLE_64B rows)
constexpr int kStagesT = 12;
constexpr int kSmemLimitT = 225 * 1024;
constexpr size_t kRecheckScratch = 8 * 8208;      // 8 warps x (1028 + 1024 floats), see recheck_smem

struct SmallTcParams {
  const float* X;
  int nrows;
  int64_t F, Fp, D, Dp, Dq, K;
  int RB, RR, nst, G, KBn;   // columns per CTA, 8-row rounding, ring stages, CTAs, K-blocks
  const uint8_t* ximg;       // X's limb image ([3 NX][Fp] interleaved) + row taus, from xlimb_image_kernel
  const float* Bt;
  const float* Cp;
  const int64_t* coltau;
  int64_t tau_const;
  double scale, inv_scale;   // 2^shift, 2^-shift
  unsigned long long* acc;
  unsigned* cnt;
  unsigned long long* recheck_count;
  float* scores;
  int32_t* labels;
  unsigned long long* dbg;   // diagnostics (HDC_SMALL_DEBUG): [0] min start, [1..7] max phase ends, [8..] CTA 0 (ns)
};

__device__ __forceinline__ unsigned long long t_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define T_REC(i)                                               \
  do {                                                         \
    if (p.dbg && blockIdx.x == 0 && (threadIdx.x & 31) == 0) p.dbg[8 + (i)] = t_now(); \
  } while (0)
#define T_MARK(i)                                              \
  do {                                                         \
    if (p.dbg && (threadIdx.x & 31) == 0) atomicMax(p.dbg + (i), t_now()); \
  } while (0)

__host__ __device__ inline size_t t_align(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Shared memory: [ring stages][MMA over-read pad][X limbs | row taus][C columns][column taus][masks][S]
struct SmemT {
  size_t xl, rtau, cs, ctau, hm, fm, sfin, bars, total;
  int nst;
};
__host__ __device__ inline size_t ximg_bytes(int NX, int64_t Fp) { return (size_t)3 * NX * Fp + sizeof(int64_t) * NX; }
__host__ __device__ inline SmemT smem_plan(int NX, int RB, int64_t Fp, int64_t K) {
  SmemT s;
  const int RR = (RB + 7) / 8 * 8;
  const size_t stage = (size_t)3 * RR * kKB, pad = (size_t)(RR < 128 ? 128 - RR : 0) * kKB;
  const size_t rest = t_align(ximg_bytes(NX, Fp), 128) + t_align(sizeof(float) * K * RB, 16) +
                      sizeof(int64_t) * RB + 2 * sizeof(uint32_t) * RB + sizeof(float) * NX * K +
                      8 * (2 * kStagesT + 2) + 256;
  const size_t avail = (size_t)kSmemLimitT - 1024 - rest - pad;
  int nst = (int)(avail / stage);
  s.nst = nst > kStagesT ? kStagesT : nst;
  const size_t ring = (size_t)s.nst * stage + pad;
  s.xl = t_align(ring > kRecheckScratch ? ring : kRecheckScratch, 1024);   // ring doubles as recheck scratch
  s.rtau = s.xl + (size_t)3 * NX * Fp;                   // the image's row taus follow its limbs
  s.cs = t_align(s.xl + ximg_bytes(NX, Fp), 128);
  s.ctau = t_align(s.cs + sizeof(float) * K * RB, 16);
  s.hm = t_align(s.ctau + sizeof(int64_t) * RB, 16);
  s.fm = t_align(s.hm + sizeof(uint32_t) * RB, 16);
  s.sfin = t_align(s.fm + sizeof(uint32_t) * RB, 16);
  s.bars = t_align(s.sfin + sizeof(float) * NX * K, 16);
  s.total = s.bars + 8 * (2 * kStagesT + 2 + (kWarpsT - 2)) + 16;
  return s;
}

// X's limb image, computed once per call by NX warps (one row each) before the main
// kernel, in the main kernel's shared-memory layout (so one bulk copy stages it):
// operand rows R = l NX + n (limb-major [x0; x1; x2]) of K-major 8 x 16-byte core matrices,
// core (R / 8, f / 16) at ((R / 8) (Fp / 16) + f / 16) 128, then the NX row taus.  Same
// arithmetic as the staging kernel (tc_limbs.cuh).  Triggers the dependent (main) launch
// at once, so the main kernel's B stream starts while this runs (programmatic dependent
// launch).
__global__ void __launch_bounds__(256) xlimb_image_kernel(const float* __restrict__ X, int nrows, int NX, int64_t F,
                                                          int64_t Fp, int64_t tau_const, uint8_t* __restrict__ img) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int n = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (n >= NX) return;
  const bool valid = n < nrows;
  const float* xr = X + (int64_t)n * F;
  float amax = 0.f;
  if (valid)
    for (int64_t f = lane; f < F; f += 32) amax = fmaxf(amax, fabsf(__ldg(xr + f)));
  amax = warp_max_f(amax);
  const float c = scale_for(amax);
  long long l1 = 0;
  const int64_t gs = (Fp >> 4) * 128;                     // bytes per 8-row group
  for (int64_t g = lane; g < (Fp >> 2); g += 32) {
    uint32_t w[3] = {0u, 0u, 0u};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t f = 4 * g + e;
      int l0, l1d, l2, U;
      limbs_of(valid && f < F ? __ldg(xr + f) : 0.f, c, l0, l1d, l2, U);
      w[0] |= (uint32_t)(uint8_t)(int8_t)l0 << (8 * e);
      w[1] |= (uint32_t)(uint8_t)(int8_t)l1d << (8 * e);
      w[2] |= (uint32_t)(uint8_t)(int8_t)l2 << (8 * e);
      l1 += U < 0 ? -U : U;
    }
    const int64_t f0 = 4 * g, cb = (f0 >> 4) * 128 + (f0 & 15);
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      const int R = l * NX + n;
      *reinterpret_cast<uint32_t*>(img + (R >> 3) * gs + cb + (R & 7) * 16) = w[l];
    }
  }
  l1 = warp_sum_xor(l1);
  // an all-zero row has V = 0 exactly (HardSign +1 = the provisional sign of I = 0): no flags
  if (lane == 0)
    reinterpret_cast<int64_t*>(img + (size_t)3 * NX * Fp)[n] = row_tau(l1, tau_const, valid && amax > 0.f);
}

// float64 re-evaluation of V[n, d] = x_n . b_d (exact fp32 products, fixed order: lane
// partial sums over f = lane + 128 i + 32 q for q = 0..3 (four independent chains: a single
// chain of convert + FMA latencies cost ~1 us at F = 784), combined (q0 + q1) + (q2 + q3),
// then a fixed butterfly) from copies of the two rows staged in this warp's shared-memory
// scratch by bulk copies (one memory round trip for F <= 1024 and little code: rarely
// executed code is fetched cold).  `xs` and `bs` hold 1024 floats each (plus 4 of alignment
// slack for x).
__device__ __forceinline__ void recheck_issue(const float* __restrict__ xr, const float* __restrict__ br, int F,
                                              int f0, float* xs, float* bs, uint64_t* bar, int lane) {
  const int len = F - f0 < 1024 ? F - f0 : 1024;
  const uint64_t xa = reinterpret_cast<uint64_t>(xr + f0);
  const int xo = (int)((xa & 15u) >> 2);
  const uint32_t xb = (uint32_t)(((xo + len) * 4 + 15) & ~15), bb = (uint32_t)((len * 4 + 15) & ~15);
  __syncwarp();
  if (lane == 0) {
    mbar_arrive_expect_tx(bar, xb + bb);
    bulk_load(xs, reinterpret_cast<const void*>(xa & ~uint64_t(15)), xb, bar);
    bulk_load(bs, br + f0, bb, bar);              // B^T rows are 256-byte aligned (Fp % 64 == 0)
  }
}
// `issued`: the copies of the first 1024-element chunk were started earlier (recheck_issue).
__device__ __noinline__ float recheck_smem(const float* __restrict__ xr, const float* __restrict__ br, int F,
                                           float* xs, float* bs, uint64_t* bar, uint32_t& phase, int lane,
                                           bool issued = false) {
  double s = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  for (int f0 = 0; f0 < F; f0 += 1024) {
    const int len = F - f0 < 1024 ? F - f0 : 1024;
    const int xo = (int)((reinterpret_cast<uint64_t>(xr + f0) & 15u) >> 2);
    if (!(issued && f0 == 0)) recheck_issue(xr, br, F, f0, xs, bs, bar, lane);
    mbar_wait(bar, phase);
    phase ^= 1u;
    int f = lane;
#pragma unroll 1
    for (; f + 96 < len; f += 128) {
      s = fma((double)xs[xo + f], (double)bs[f], s);
      s1 = fma((double)xs[xo + f + 32], (double)bs[f + 32], s1);
      s2 = fma((double)xs[xo + f + 64], (double)bs[f + 64], s2);
      s3 = fma((double)xs[xo + f + 96], (double)bs[f + 96], s3);
    }
#pragma unroll 1
    for (; f < len; f += 32) s = fma((double)xs[xo + f], (double)bs[f], s);
  }
  s = (s + s1) + (s2 + s3);
  s = warp_sum_xor(s);
  return s >= 0.0 ? 1.f : -1.f;
}

// Stage II of one CTA (see the call site).  Thread item = (class k, row pair n0, n0 + 1):
// per 4 columns one 16-byte load of C[k] and one (broadcast) of the sign masks serve both
// rows -- the shared-memory wavefronts, not the adds, bound this loop (a thread per (n, k)
// took ~2900 cycles at N = 32, K = 10).  Per (n, k): four partial sums over the columns
// j = 4 i + q, combined (q0 + q1) + (q2 + q3): a fixed order.
__device__ __noinline__ void stage2_pass(const float* Cs, const uint32_t* hmask, int RB, int nrows, int K, int ncol,
                                         int wt, double scale, unsigned long long* acc) {
  const int items = K * ((nrows + 1) >> 1);
  for (int it = wt; it < items; it += kWorkers) {
    const int k = it % K, n0 = 2 * (it / K), n1 = n0 + 1;
    const float* cr = Cs + k * RB;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f, b0 = 0.f, b1 = 0.f, b2 = 0.f, b3 = 0.f;
    int j = 0;
#pragma unroll 4
    for (; j + 3 < ncol; j += 4) {
      const uint4 h4 = *reinterpret_cast<const uint4*>(hmask + j);
      const float4 c4 = *reinterpret_cast<const float4*>(cr + j);
      a0 += ((h4.x >> n0) & 1u) ? -c4.x : c4.x;
      a1 += ((h4.y >> n0) & 1u) ? -c4.y : c4.y;
      a2 += ((h4.z >> n0) & 1u) ? -c4.z : c4.z;
      a3 += ((h4.w >> n0) & 1u) ? -c4.w : c4.w;
      b0 += ((h4.x >> n1) & 1u) ? -c4.x : c4.x;
      b1 += ((h4.y >> n1) & 1u) ? -c4.y : c4.y;
      b2 += ((h4.z >> n1) & 1u) ? -c4.z : c4.z;
      b3 += ((h4.w >> n1) & 1u) ? -c4.w : c4.w;
    }
    for (; j < ncol; ++j) {
      a0 += ((hmask[j] >> n0) & 1u) ? -cr[j] : cr[j];
      b0 += ((hmask[j] >> n1) & 1u) ? -cr[j] : cr[j];
    }
    atomicAdd(acc + (int64_t)n0 * K + k, (unsigned long long)llrint((double)((a0 + a1) + (a2 + a3)) * scale));
    if (n1 < nrows)
      atomicAdd(acc + (int64_t)n1 * K + k, (unsigned long long)llrint((double)((b0 + b1) + (b2 + b3)) * scale));
  }
}

__device__ __forceinline__ void wbar() {          // the worker warps only (named barrier 1)
  asm volatile("bar.sync 1, %0;" ::"n"(kWorkers) : "memory");
}

// Code executed once per CTA is kept in rolled loops: straight-line unrolled code would be
// fetched from L2 instruction line by instruction line while the B stream saturates it.
template <int NX>
__global__ void __launch_bounds__(kThreadsT, 1)
small_tc_kernel(const __grid_constant__ CUtensorMap tmB, const SmallTcParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int RB = p.RB, RR = p.RR, nst = p.nst, K = (int)p.K;
  const SmemT L = smem_plan(NX, RB, p.Fp, p.K);
  uint8_t* ring = smem;                                    // [nst][3][RR][64] B^T limbs (TMA, SW64)
  uint8_t* xl = smem + L.xl;                               // [3 NX rows][Fp] X limbs, interleaved core matrices
  const int64_t* rtau = reinterpret_cast<const int64_t*>(smem + L.rtau);
  float* Cs = reinterpret_cast<float*>(smem + L.cs);       // [K][RB] this CTA's C columns
  int64_t* ctau = reinterpret_cast<int64_t*>(smem + L.ctau);
  uint32_t* hmask = reinterpret_cast<uint32_t*>(smem + L.hm);   // [RB] bit n set <=> h[n, d] = -1
  uint32_t* fmask = reinterpret_cast<uint32_t*>(smem + L.fm);   // [RB] bit n set <=> sign (n, d) flagged
  float* Sfin = reinterpret_cast<float*>(smem + L.sfin);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* empty = full + kStagesT;
  uint64_t* xfull = empty + kStagesT;                      // X limb image, C columns, column taus landed
  uint64_t* tfull = xfull + 1;
  uint64_t* rbar = tfull + 1;                               // [8] recheck row copies, one per worker warp
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + (kWarpsT - 2));
  int* s_last = reinterpret_cast<int*>(tmem_slot + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t d0 = (int64_t)blockIdx.x * RB;
  const int ncol = (int)((p.D - d0) < RB ? (p.D - d0) : RB);
  const int stage_bytes = 3 * RR * kKB;
  if (p.dbg && tid == 0) atomicMin(p.dbg, t_now());
  const uint32_t cbytes = (uint32_t)(((ncol + 3) & ~3) * 4), tbytes = (uint32_t)(((ncol + 1) & ~1) * 8);
  const uint32_t ibytes = (uint32_t)t_align(ximg_bytes(NX, p.Fp), 16);

  if (tid == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(xfull, 1);
    mbar_init(tfull, 1);
    for (int w = 0; w < kWarpsT - 2; ++w) mbar_init(rbar + w, 1);
    fence_mbar_init();
    // this CTA's C columns and column taus (independent of the X-limb kernel)
    mbar_arrive_expect_tx(xfull, (uint32_t)K * cbytes + tbytes + ibytes);
    for (int k = 0; k < K; ++k) bulk_load(Cs + k * RB, p.Cp + (int64_t)k * p.Dp + d0, cbytes, xfull);
    bulk_load(ctau, p.coltau + d0, tbytes, xfull);
  }
  if (warp == 1) tmem_alloc<128>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (tid == 0) T_REC(0);

  if (warp == 0) {
    // ===================================================== TMA producer: this CTA's B^T limbs
    if (lane == 0) {
      tma_prefetch_desc(&tmB);
      for (int kb = 0; kb < p.KBn; ++kb) {
        const int s = kb % nst;
        if (kb >= nst) mbar_wait(empty + s, (uint32_t)(((kb / nst) - 1) & 1));
        if (kb == nst) T_REC(1);
        mbar_arrive_expect_tx(full + s, (uint32_t)(3 * RB * kKB));
        for (int l = 0; l < 3; ++l)
          tma_load_2d(ring + (size_t)s * stage_bytes + (size_t)l * RR * kKB, &tmB, full + s, kb * kKB,
                      (int)(l * p.Dq + d0));
      }
    }
  } else if (warp == 1) {
    // ===================================================== MMA issuer (elected lane)
    // [A0|A1|A2] (+)= bt0 [x0;x1;x2]^T, [A1|A2] += bt1 [x0;x1]^T, A2 += bt2 x0^T: the six limb
    // products with i + j <= 2, exact in int32
    constexpr uint32_t I3 = make_idesc<2>(128, 3 * NX), I2 = make_idesc<2>(128, 2 * NX),
                       I1 = make_idesc<2>(128, NX);
    mbar_wait(xfull, 0);
    T_REC(2);
    tc_fence_after();
    const uint64_t a_base = smem_desc_sw(smem_u32(ring), 512, 4);     // SWIZZLE_64B, 8-row groups 512 B apart
    const uint32_t x_base = smem_u32(xl);
    const uint32_t sbo_x = (uint32_t)(8 * p.Fp);                        // 8-row core groups of xl
    for (int kb = 0; kb < p.KBn; ++kb) {
      const int s = kb % nst;
      mbar_wait(full + s, (uint32_t)((kb / nst) & 1));
      tc_fence_after();
      const uint64_t a_s = a_base + (uint64_t)(((size_t)s * stage_bytes) >> 4);
#pragma unroll
      for (int ks = 0; ks < kKB / 32; ++ks) {
        const uint64_t bdesc = smem_desc_interleaved(x_base + (uint32_t)(((kb * kKB + ks * 32) >> 4) * 128), 128, sbo_x);
        tc_mma_i8x3_elect(tmem, a_s + 2 * ks, a_s + ((RR * kKB + ks * 32) >> 4),
                          a_s + ((2 * RR * kKB + ks * 32) >> 4), bdesc, I3, I2, I1, NX,
                          (kb | ks) ? 1u : 0u);
      }
      tc_commit_elect(empty + s);
      if (kb == 0) T_REC(3);
    }
    T_REC(4);
    tc_commit_elect(tfull);
  } else {
    // ===================================================== workers (warps 2..9)
    const int ww = warp - 2;
    if (tid == 64) {
      // X's limb image is written by the preceding kernel (programmatic dependent launch):
      // wait for it to complete, then stage it with one bulk copy
      asm volatile("griddepcontrol.wait;" ::: "memory");
      T_REC(5);
      bulk_load(xl, p.ximg, ibytes, xfull);
    }
    mbar_wait(xfull, 0);
    T_MARK(1);
    if (ww == 0) T_REC(6);

    if (ww < 4) {
      // ---- epilogue: TMEM lane quarter q = warp % 4 holds columns 32 q .. 32 q + 31
      const int q = warp & 3, j = q * 32 + lane;
      const bool jok = j < ncol;
      const int64_t ct = jok ? ctau[j] : -(int64_t(1) << 62);
      mbar_wait(tfull, 0);
      tc_fence_after();
      T_MARK(2);
      if (ww == 0) T_REC(7);
      uint32_t hm = 0u, fm = 0u;
      const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int n0 = 0; n0 < NX; n0 += 16) {
        uint32_t r0[16], r1[16], r2[16];
        tmem_ld16(tb + n0, r0);
        tmem_ld16(tb + NX + n0, r1);
        tmem_ld16(tb + 2 * NX + n0, r2);
        tmem_ld_wait();
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const int n = n0 + jj;
          const int64_t I = (int64_t)(int32_t)r0[jj] * 16384 + (int64_t)(int32_t)r1[jj] * 128 + (int64_t)(int32_t)r2[jj];
          const int64_t aI = I < 0 ? -I : I;
          hm |= (uint32_t)(I < 0) << n;
          fm |= (uint32_t)(aI <= rtau[n] + ct) << n;
        }
      }
      tc_fence_before();
      if (jok) {
        hmask[j] = hm;
        fmask[j] = fm;                            // flagged signs, re-evaluated by all workers below
      }
      T_MARK(3);
      if (ww == 0) T_REC(8);
    }
    wbar();
    // float64 re-evaluation of the flagged signs, spread evenly over the 8 worker warps: every
    // warp scans the per-column flag counts (lane l: columns 4l .. 4l + 3) and takes flags
    // e = ww, ww + 8, ... in column-major order; one warp per sign (fixed lane order).  The
    // row copies of a warp's first flag go out before Stage II, which runs on the
    // provisional signs; a sign the re-evaluation flips then adds the exact correction
    // (h - h') C[k, d] = 2 h C[k, d] to the int64 sums (Stage II is linear in H),
    // so the recheck's round trip overlaps Stage II instead of preceding it.
    const int wt = tid - 64;
    const int nk = p.nrows * K;
    unsigned long long nrecheck = 0;
    uint32_t rphase = 0u;
    uint32_t fw[4];
    int cnt = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int jj = 4 * lane + u;
      fw[u] = jj < ncol ? fmask[jj] : 0u;
      cnt += __popc(fw[u]);
    }
    int incl = cnt;                                // inclusive prefix over lanes
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    auto select = [&](int e, int& jsel, int& nsel) {   // column and row of flag e
      const int L = __ffs(__ballot_sync(0xffffffffu, incl > e)) - 1;   // lane holding flag e
      jsel = 0;
      nsel = 0;
      if (lane == L) {
        int r = e - (incl - cnt);                  // rank of the flag within this lane's columns
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = __popc(fw[u]);
          if (r >= 0 && r < c) {
            uint32_t m = fw[u];
            for (int t = 0; t < r; ++t) m &= m - 1;
            jsel = 4 * lane + u;
            nsel = __ffs(m) - 1;
          }
          r -= c;
        }
      }
      jsel = __shfl_sync(0xffffffffu, jsel, L);
      nsel = __shfl_sync(0xffffffffu, nsel, L);
    };
    // the ring is free once the MMAs are done (tfull): 8 KB of it per warp as scratch
    float* xs = reinterpret_cast<float*>(ring + (size_t)ww * 8208);
    int j0 = 0, n0 = 0;
    if (ww < total) {
      select(ww, j0, n0);
      recheck_issue(p.X + (int64_t)n0 * p.F, p.Bt + (d0 + j0) * p.Fp, (int)p.F, 0, xs, xs + 1028, rbar + ww, lane);
    }
    if (ww == 0) T_REC(11);
    // ---- Stage II: S_local[n][k] = sum_{d in range} h[n, d] C[k, d] on the
    // provisional signs; exact int64 fixed-point accumulation across CTAs (Alg. 3
    // `S += S_local`).  Four independent partial sums over columns j = 4 i + q
    // (16-byte loads of C and the sign masks; RB is a multiple of 4), combined
    // (q0 + q1) + (q2 + q3): fixed order.
    stage2_pass(Cs, hmask, RB, p.nrows, K, ncol, wt, p.scale, p.acc);
    if (ww == 0) T_REC(12);
    for (int e = ww; e < total; e += kWarpsT - 2) {
      int jsel = j0, nsel = n0;
      if (e != ww) select(e, jsel, nsel);
      const float hv = recheck_smem(p.X + (int64_t)nsel * p.F, p.Bt + (d0 + jsel) * p.Fp, (int)p.F, xs,
                                    xs + 1028, rbar + ww, rphase, lane, e == ww);
      const bool prov_neg = (hmask[jsel] >> nsel) & 1u;
      if ((hv < 0.f) != prov_neg) {                 // flipped: S[n, k] += (h - h') C[k, d]
        const float dh = hv < 0.f ? -2.f : 2.f;
        for (int k = lane; k < K; k += 32) {
          const long long v = llrint((double)(dh * Cs[k * RB + jsel]) * p.scale);
          atomicAdd(p.acc + (int64_t)nsel * K + k, (unsigned long long)v);
        }
      }
      ++nrecheck;
    }
    if (lane == 0 && nrecheck) atomicAdd(p.recheck_count, nrecheck);
  }
  __syncthreads();                                   // TMEM reads, Stage II and rechecks done (all warps)
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<128>(tmem);
  }
  if (warp < 2) return;
  if (tid == 64) T_REC(13);
  const int wt = tid - 64;
  const int nk = p.nrows * K;
  T_MARK(4);
  if (wt == 0) T_REC(9);
  wbar();
  if (wt == 0) {
    // acq_rel: this CTA's reductions are ordered before its arrival is counted (release), and
    // the last arriver sees every other CTA's (acquire) -- one round trip
    unsigned prev;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(p.cnt) : "memory");
    *s_last = (prev == (unsigned)(p.G - 1)) ? 1 : 0;
  }
  wbar();
  if (!*s_last) return;
  for (int i = wt; i < nk; i += kWorkers) {
    const long long a = (long long)atomicExch(p.acc + i, 0ull);   // read and reset for the next call
    const float v = (float)((double)a * p.inv_scale);
    Sfin[i] = v;
    if (p.scores) p.scores[i] = v;
  }
  wbar();
  if (p.labels)
    for (int n = wt; n < p.nrows; n += kWorkers) {
      int best = 0;
      float bv = Sfin[n * K];
      for (int k = 1; k < K; ++k)
        if (Sfin[n * K + k] > bv) {   // lowest index on ties (DESIGN R2)
          bv = Sfin[n * K + k];
          best = k;
        }
      p.labels[n] = best;
    }
  if (wt == 0) *p.cnt = 0u;
  T_MARK(5);
  if (wt == 0) T_REC(10);
}

int rb_for(int64_t D, int num_sms) {
  int64_t rb = (D + num_sms - 1) / num_sms;
  rb = (rb + 3) / 4 * 4;                             // 16-byte rows of the C-column copies
  return (int)(rb < 4 ? 4 : (rb > 128 ? 128 : rb));
}

template <int NX>
cudaError_t launch_nx(const CUtensorMap& tm, SmallTcParams& p, uint8_t* img, cudaStream_t st) {
  const SmemT L = smem_plan(NX, p.RB, p.Fp, p.K);
  const size_t sm = L.total + 1024;
  if (sm > (size_t)kSmemLimitT || L.nst < 2) return cudaErrorInvalidValue;
  p.nst = L.nst;
  p.ximg = img;
  cudaError_t e = cudaFuncSetAttribute(small_tc_kernel<NX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  static unsigned long long* dbg = nullptr;
  const bool debug = getenv("HDC_SMALL_DEBUG") != nullptr;
  p.dbg = nullptr;
  if (debug) {
    if (!dbg) cudaMalloc((void**)&dbg, 32 * sizeof(unsigned long long));
    unsigned long long init[32] = {~0ull};
    cudaMemcpyAsync(dbg, init, sizeof(init), cudaMemcpyHostToDevice, st);
    p.dbg = dbg;
  }
  // (1) X's limb image (NX warps), (2) the streaming kernel as its programmatic dependent:
  // it may start as soon as (1) has started, so B's stream overlaps (1)
  xlimb_image_kernel<<<NX / 8, 256, 0, st>>>(p.X, p.nrows, NX, p.F, p.Fp, p.tau_const, img);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  cfg.gridDim = dim3(p.G, 1, 1);
  cfg.blockDim = dim3(kThreadsT, 1, 1);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = getenv("HDC_NO_PDL") ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, small_tc_kernel<NX>, tm, (const SmallTcParams)p);
  cudaError_t le = e != cudaSuccess ? e : cudaGetLastError();
  if (debug && le == cudaSuccess) {
    unsigned long long h[32];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, dbg, sizeof(h), cudaMemcpyDeviceToHost);
    fprintf(stderr, "[hdc small_tc cta0]");
    for (int i = 0; i < 14; ++i) fprintf(stderr, " %d:%.2f", i, h[8 + i] ? ((double)(long long)(h[8 + i] - h[0])) * 1e-3 : -1.0);
    fprintf(stderr, "\n[hdc small_tc debug] NX=%d G=%d RB=%d nst=%d: from first CTA start (us): X limbs %.2f, "
            "MMA done %.2f, signs %.2f, stage II %.2f, final %.2f\n", NX, p.G, p.RB, p.nst, (h[1] - h[0]) * 1e-3,
            (h[2] - h[0]) * 1e-3, (h[3] - h[0]) * 1e-3, (h[4] - h[0]) * 1e-3, h[5] ? (h[5] - h[0]) * 1e-3 : -1.0);
  }
  return le;
}

}  // namespace

int64_t small_tc_image_bytes(int64_t F) {
  const int64_t Fp = (F + kFPad - 1) / kFPad * kFPad;
  return (int64_t)t_align(ximg_bytes(32, Fp), 16);
}

bool small_tc_fits(int64_t F, int64_t D, int64_t K, int n, int num_sms) {
  if (n < 1 || n > 32 || K < 1 || K > 32 || F < 1) return false;
  const int NX = n <= 16 ? 16 : 32;
  const int64_t Fp = (F + kFPad - 1) / kFPad * kFPad;
  const SmemT L = smem_plan(NX, rb_for(D, num_sms), Fp, K);
  return L.total + 1024 <= (size_t)kSmemLimitT && L.nst >= 2 && Fp * 8 < (1 << 18) &&
         (int64_t)t_align(ximg_bytes(NX, Fp), 16) < (int64_t(1) << 20);   // one bulk copy (tx-count limit)
}

cudaError_t launch_small_tc(const SmallTcOperands& o, const float* X, int n, float* scores, int32_t* labels,
                            int num_sms, cudaStream_t st) {
  if (!small_tc_fits(o.F, o.D, o.K, n, num_sms) || !o.ximg) return cudaErrorInvalidValue;
  const int NX = n <= 16 ? 16 : 32;
  SmallTcParams p;
  p.X = X;
  p.nrows = n;
  p.F = o.F;
  p.Fp = o.Fp;
  p.D = o.D;
  p.Dp = o.Dp;
  p.Dq = o.Dq;
  p.K = o.K;
  p.RB = rb_for(o.D, num_sms);
  p.RR = (p.RB + 7) / 8 * 8;
  p.G = (int)((o.D + p.RB - 1) / p.RB);
  p.nst = 0;
  p.KBn = (int)(o.Fp / kKB);
  p.Bt = o.Bt;
  p.Cp = o.Cp;
  p.coltau = o.coltau;
  p.tau_const = tc_tau_const(o.F);
  p.scale = ldexp(1.0, o.shift);
  p.inv_scale = ldexp(1.0, -o.shift);
  p.acc = o.acc;
  p.cnt = o.cnt;
  p.recheck_count = o.recheck;
  p.scores = scores;
  p.labels = labels;
  CUtensorMap tm;
  if (!make_tensor_map_u8(&tm, o.Btc, (uint64_t)o.Fp, (uint64_t)3 * o.Dq, kKB, (uint32_t)p.RB, 64))
    return cudaErrorInvalidValue;
  return NX == 16 ? launch_nx<16>(tm, p, o.ximg, st) : launch_nx<32>(tm, p, o.ximg, st);
}

}  // namespace hdc
