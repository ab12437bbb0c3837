// k_smallstream.cu -- K2s: HBM-streaming small-batch HDC inference (N <= 32).
//
// The whole of Alg. 1 for up to 32 rows of X in one launch:
//   V = X B (fp32 FFMA), H = HardSign(V), S = H C^T,
//   y = argmax_k S, lowest index on ties.
// The work is bound by reading B (F x D fp32) once from HBM.  Partitioning is the
// paper's ScalableHD-S (Alg. 3): D is split into one contiguous range of
// 4-column units per CTA (148 CTAs); each CTA forms complete F-sums for its columns
// (HardSign needs all of F), applies HardSign and contracts with its C columns into
// a partial S (the paper's S_local); the partials are summed (the paper's `S += S_local`,
// P:336) in int64 fixed point by atomics -- exact, so order-free -- and the last-arriving
// CTA converts them and takes the argmax.
//
// B200 mapping.  The model keeps B unit-major (B4[u][f][4]: all F rows of a 4-column
// unit contiguous), so a CTA's share of B is one contiguous run of HBM.  A producer
// warp streams it with 1-D TMA bulk copies (cp.async.bulk, 4 KB chunks) through
// per-consumer-warp shared-memory rings (3-5 stages each, ~160-200 KB in flight per SM),
// started before X is staged; 10 consumer warps run the FFMA contraction from shared
// memory.  Sign-exact N = 1 streams the bf16 hi plane of B instead (half the bytes).
//
// Sign exactness (fp32 semantics): |v| <= tau (c_F ||x_n|| ||b_d||, or the hi plane's
// bound) is re-evaluated in float64 (warp-cooperative, fixed order) after the stream.
#include <atomic>
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace hdc {
namespace {

using namespace ptx;

// 10 consumer warps: a CTA's ~17 four-column units (D = 10^4 over 148 CTAs) take two
// rounds of units per warp instead of three with 8 warps (N=32: 59 -> 49 us per step);
// 12 or more warps exceed the register budget of the NB = 32 instantiation
#ifndef HDC_SMALL_CW
#define HDC_SMALL_CW 10
#endif
constexpr int kCw = HDC_SMALL_CW;              // consumer warps
constexpr int kCt = 32 * kCw;                  // consumer threads
constexpr int kThreadsS = kCt + 32;            // + producer warp (lane w feeds consumer warp w)
#ifndef HDC_SMALL_CHUNK
#define HDC_SMALL_CHUNK 256
#endif
constexpr int kChunkRows = HDC_SMALL_CHUNK;    // B4 rows per ring stage (4 KB)
constexpr int kStagesMax = 8;                  // per consumer warp
constexpr int kGroup = 8;                      // first-level reduction group (CTAs)
constexpr int kDefer = 256;                    // deferred rechecks per CTA
constexpr int kSlotsMax = 32;                  // of which with their Bt row bulk-copied to smem
// dynamic shared memory limit: 227 KB per CTA minus the static arrays (the defer list)
constexpr size_t kSmemDyn = 227 * 1024 - 1024 - (size_t)kDefer * 8;

struct StreamParams {
  const float* X;
  int nrows;
  int64_t F, D, Dp, K, Fp;
  const float* B4;       // [units][Fp][4]
  const uint16_t* B4h;   // [units][Fp][4] bf16 hi plane (HALF instantiation; N = 1 sign-exact)
  const float* Bt;       // [Dp][Fp] fp32 (float64 rechecks)
  const float* Cp;       // [K][Dp]
  const float* bnorm;    // [Dp]: ||b_d|| (fp32 B) or the hi-plane bound coefficient (HALF)
  float tau_coef;        // tau = tau_coef ||x_n|| bnorm[d] + kSignBoundAbs
  int recheck;
  int G;                 // CTAs
  int nst;               // ring stages per consumer warp
  int nslot;             // recheck row slots in shared memory (Bt rows bulk-copied when flagged)
  int max_cols;          // columns of the largest CTA range (4 ceil(units / G))
  int64_t units;
  float* S_part;         // [G + groups][NB][K] (unused: partials go to acc)
  unsigned long long* acc;   // [32][K] int64 fixed-point score sums, zero between launches
  double scale, inv_scale;   // 2^shift, 2^-shift
  unsigned* cnt;         // [1 + groups], zero between launches
  unsigned long long* recheck_count;
  float* scores;
  int32_t* labels;
  unsigned long long* dbg;   // diagnostics (HDC_SMALL_DEBUG): [0] min start, [1..7] max of phase ends (ns)
  // D-shard exchange (hdc_model_infer_dshard): xworld > 0 -> the last CTA sends this
  // rank's partial scores to every rank's exchange buffer and sums all ranks' partials
  float* const* xbufs;       // [xworld] device pointers (peer-mapped) of the exchange buffers
  int xrank, xworld;
  uint32_t xepoch;           // call number, identical on all ranks, increasing
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SS_MARK(i)                                           \
  do {                                                       \
    if (p.dbg && (tid & 31) == 0) atomicMax(p.dbg + (i), gtime()); \
  } while (0)

__device__ __forceinline__ void cbar() {       // consumer warps only (named barrier 1)
  asm volatile("bar.sync 1, %0;" ::"n"(kCt) : "memory");
}

// HALF: B is streamed as its bf16 hi plane (b_hi = RN_bf16(b), half the bytes) and the
// sign decisions are made exact by the float64 recheck of every |v_hi| <= tau, where tau
// bounds |v - v_hi| (the dropped x . b_lo plus the fp32 rounding; hi_bound_kernel).
// Both instantiations defer their rechecks to the end of the CTA's stream: a flagged sign's
// fp32 B^T row is bulk-copied into a shared-memory slot (or prefetched into L2 past the
// slots), Stage II runs on the provisional sign, and a sign the float64 dot changes adds
// (h - h_provisional) C[k][d] to the exact int64 score sums.
template <int NB, bool HALF>
__global__ void __launch_bounds__(kThreadsS, 1) smallstream_kernel(const StreamParams p) {
  constexpr int NBP = (NB + 3) / 4 * 4;        // rows padded to float4
  constexpr int kRows = HALF ? 2 * kChunkRows : kChunkRows;   // B4 rows per stage (4 KB)
  constexpr int kRowBytes = HALF ? 8 : 16;
  extern __shared__ __align__(128) uint8_t smem[];
  const int F = (int)p.F, K = (int)p.K, nst = p.nst;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);         // [kCw][kStagesMax]
  uint64_t* empty = full + kCw * kStagesMax;
  uint64_t* xfull = empty + kCw * kStagesMax;                 // X landed
  float* ring = reinterpret_cast<float*>(smem + (2 * kCw * kStagesMax + 2) * 8);   // [kCw][nst][R][4]
  // X rows as in global memory ([n][F], copied by one bulk copy from the 16-byte-aligned
  // address at or below X; xoff floats of slack in front)
  const uint64_t xaddr = reinterpret_cast<uint64_t>(p.X);
  const int xoff = (int)((xaddr & 15u) >> 2);
  const uint32_t xbytes = (uint32_t)(((xoff + p.nrows * F) * 4 + 15) & ~15);
  float* Xraw = ring + (size_t)kCw * nst * kChunkRows * 4;     // [xbytes / 4] (stage = 4 KB either way)
  const float* Xs = Xraw + xoff;                               // Xs[n * F + f]
  auto up4 = [](size_t x) { return (x + 3) & ~size_t(3); };  // float4-aligned regions
  float* Sw = Xraw + up4((size_t)NB * F + 4);                  // [kCw][NB][K] per-warp S_local
  float* Cs = Sw + up4((size_t)kCw * NB * K);                  // [K][ncol] this CTA's C columns
  float* bns = Cs + up4((size_t)K * p.max_cols);               // [ncol] ||b_d||
  float* fin = bns + up4(p.max_cols);                          // [NB K + 32 + 4 kCt] final sums
  const int slotf = (F + 3) & ~3;                              // floats per recheck row slot
  float* rows_s = fin + up4((size_t)NB * K + 32 + 4 * kCt + 32);   // [nslot][slotf] Bt rows
  __shared__ float xnorm_s[NBP];
  __shared__ int s_last;
  __shared__ int2 defer_s[kDefer];             // deferred rechecks: (n | provisional-negative << 31, d)
  __shared__ int ndefer_s;
  __shared__ __align__(8) uint64_t slotbar[kSlotsMax];   // row slot j landed (used once: parity 0)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = blockIdx.x;
  const int64_t u0 = (int64_t)c * p.units / p.G, u1 = (int64_t)(c + 1) * p.units / p.G;
  const int nch = (F + kRows - 1) / kRows;                   // chunks per unit

  if (p.dbg && tid == 0) atomicMin(p.dbg, gtime());
  if (tid < kCw * nst) {
    const int w = tid / nst, st = tid % nst;
    mbar_init(full + w * kStagesMax + st, 1);
    mbar_init(empty + w * kStagesMax + st, 1);
  }
  if (tid == 0) {
    mbar_init(xfull, 1);
    ndefer_s = 0;
  }
  if (tid < kSlotsMax) mbar_init(slotbar + tid, 1);
  fence_mbar_init();
  __syncthreads();

  if (warp == kCw) {
    // ===================================================== producer: lane w streams warp w's units
    if (lane == kCw) {
      // X (one bulk copy), this CTA's C columns (one per class) and ||b_d||, issued before
      // any of B so they are first in the memory queues (consumer loads issued at the same
      // time would wait behind the B stream)
      const int ncol_p = (int)(u1 - u0) * 4;
      const int64_t col0_p = u0 * 4;
      mbar_arrive_expect_tx(xfull, xbytes + (uint32_t)((K + 1) * ncol_p * 4));
      bulk_load(Xraw, reinterpret_cast<const void*>(xaddr & ~uint64_t(15)), xbytes, xfull);
      for (int k = 0; k < K; ++k)
        bulk_load(Cs + (size_t)k * ncol_p, p.Cp + (int64_t)k * p.Dp + col0_p, (uint32_t)(ncol_p * 4), xfull);
      bulk_load(bns, p.bnorm + col0_p, (uint32_t)(ncol_p * 4), xfull);
    }
    if (lane < kCw) {
      const int w = lane;
      int st = 0;
      uint32_t ph = 0;
      for (int64_t u = u0 + w; u < u1; u += kCw)
        for (int ch = 0; ch < nch; ++ch) {
          const int f0 = ch * kRows, rows = min(kRows, F - f0);
          mbar_wait(empty + w * kStagesMax + st, ph ^ 1);
          // bulk copies move multiples of 16 bytes: an odd HALF row count takes one zero
          // padding row along (Fp is a multiple of 64, so it exists)
          const uint32_t bytes = (uint32_t)((rows * kRowBytes + 15) & ~15);
          mbar_arrive_expect_tx(full + w * kStagesMax + st, bytes);
          const void* src = HALF ? static_cast<const void*>(p.B4h + (u * p.Fp + f0) * 4)
                                 : static_cast<const void*>(p.B4 + (u * p.Fp + f0) * 4);
          bulk_load(ring + ((size_t)w * nst + st) * kChunkRows * 4, src, bytes, full + w * kStagesMax + st);
          if (++st == nst) {
            st = 0;
            ph ^= 1;
          }
        }
    }
    return;   // the producer takes no part in the rest (consumer barriers are named)
  }

  // ===================================================== consumers
  // X, this CTA's columns of C (Cs[k][cols]) and of ||b_d|| (bns) arrive by the producer's
  // bulk copies (xfull), ahead of the B stream
  const int ncol = (int)(u1 - u0) * 4;
  const int64_t col0 = u0 * 4;
  float* sw = Sw + (size_t)warp * NB * K;
  for (int i = lane; i < NB * K; i += 32) sw[i] = 0.f;
  // float64 re-evaluation of v[n][d] (fixed order: lane l sums f = l, l + 32, ... in f
  // order, then a fixed butterfly), warp-uniform; 8 loads in flight per lane
  auto dot_smem = [&](const float* xr, const float* br) -> double {
    double a64 = 0.0;
    for (int f = lane; f < F; f += 32) a64 = fma((double)xr[f], (double)br[f], a64);
    return warp_sum_xor(a64);
  };
  auto dot_global = [&](const float* xr, const float* bt) -> double {
    double a64 = 0.0;
    for (int f0 = 0; f0 < F; f0 += 256) {
      float bv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int f = f0 + 32 * j + lane;
        bv[j] = f < F ? __ldg(bt + f) : 0.f;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int f = f0 + 32 * j + lane;
        if (f < F) a64 = fma((double)xr[f], (double)bv[j], a64);
      }
    }
    return warp_sum_xor(a64);
  };
  auto exact_sign = [&](int n, int64_t d, int slot) -> float {
    const float* xr = Xs + n * F;
    double a64;
    if (slot >= 0) {                                  // the row is in shared memory
      mbar_wait(slotbar + slot, 0);
      a64 = dot_smem(xr, rows_s + (size_t)slot * slotf);
    } else {
      a64 = dot_global(xr, p.Bt + d * p.Fp);
    }
    return a64 >= 0.0 ? 1.f : -1.f;
  };
  // Stage II runs on the provisional signs; a sign the recheck changes adds
  // (h - h_provisional) C[k][d] = +-2 C[k][d] straight into the exact int64 score sums (each
  // term rounded to 2^-shift on its own): the result does not depend on when, by which
  // warp, or in which order the rechecks run
  auto flip_correct = [&](int n, int64_t d, float hp, int slot) {
    const float h = exact_sign(n, d, slot);
    if (h != hp) {
      const double dh = (double)(h - hp);
      for (int k = lane; k < K; k += 32)
        atomicAdd(p.acc + n * K + k,
                  (unsigned long long)llrint(dh * (double)Cs[k * ncol + (int)(d - col0)] * p.scale));
    }
  };
  cbar();
  mbar_wait(xfull, 0);
  // zero rows nrows..NB-1 (also overwrites the bulk copy's tail slack past row nrows-1)
  for (int i = p.nrows * F + tid; i < NB * F; i += kCt) Xraw[xoff + i] = 0.f;
  for (int n = warp; n < p.nrows; n += kCw) {
    float ss = 0.f;
    for (int f = lane; f < F; f += 32) ss = fmaf(Xs[n * F + f], Xs[n * F + f], ss);
    ss = warp_sum_xor(ss);
    if (lane == 0) xnorm_s[n] = sqrtf(ss);
  }
  cbar();
  SS_MARK(1);

  // (n, q) elements a lane owns after the cross-lane reduction: e = EPL lane + i
  constexpr int NV = NB * 4;                          // V values of a unit
  constexpr int EPL = NV >= 32 ? NV / 32 : 1;         // per lane (reduce-scatter), else lane e < NV
  int st = 0;
  uint32_t ph = 0;
  unsigned long long nrecheck = 0;
  for (int64_t u = u0 + warp; u < u1; u += kCw) {
    // ---- V[n][0..3] for this unit, lanes over f (fp32 FMA, f ascending per lane)
    float acc[NV];
    float2 acc2[NV / 2];                          // packed (q0, q1), (q2, q3): FFMA2
#pragma unroll
    for (int e = 0; e < NV / 2; ++e) acc2[e] = make_float2(0.f, 0.f);
    for (int ch = 0; ch < nch; ++ch) {
      const int f0 = ch * kRows, rows = min(kRows, F - f0);
      mbar_wait(full + warp * kStagesMax + st, ph);
      const float* stage = ring + ((size_t)warp * nst + st) * kChunkRows * 4;
#pragma unroll 2
      for (int r = lane; r < rows; r += 32) {
        float2 b01, b23;
        if constexpr (HALF) {
          const uint2 b = reinterpret_cast<const uint2*>(stage)[r];   // 4 bf16: exact in fp32
          b01 = make_float2(__uint_as_float(b.x << 16), __uint_as_float(b.x & 0xffff0000u));
          b23 = make_float2(__uint_as_float(b.y << 16), __uint_as_float(b.y & 0xffff0000u));
        } else {
          const float4 b = reinterpret_cast<const float4*>(stage)[r];
          b01 = make_float2(b.x, b.y);
          b23 = make_float2(b.z, b.w);
        }
        const float* xc = Xs + f0 + r;                // column f of X: Xs[n F + f]
#pragma unroll
        for (int n = 0; n < NB; ++n) {
          const float x = *xc;                        // rows >= nrows are zero
          xc += F;
          acc2[n * 2 + 0] = ffma2(x, b01, acc2[n * 2 + 0]);   // each lane: fmaf(x, b_q, acc)
          acc2[n * 2 + 1] = ffma2(x, b23, acc2[n * 2 + 1]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + warp * kStagesMax + st);
      if (++st == nst) {
        st = 0;
        ph ^= 1;
      }
    }
#pragma unroll
    for (int e = 0; e < NV / 2; ++e) {
      acc[2 * e] = acc2[e].x;
      acc[2 * e + 1] = acc2[e].y;
    }
    // ---- complete the F-sums across lanes with a fixed pairwise tree
    float vv[EPL];
    if constexpr (NV >= 32) {
      // reduce-scatter: at offset o a lane keeps the half of its values selected by lane bit o
      // and adds the partner's copy of that half; after 5 steps lane l holds e = EPL l + i
#pragma unroll
      for (int o = 16, m = NV; o >= 1; o >>= 1, m >>= 1) {
        const bool hi = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < m / 2; ++i) {
          const float keep = hi ? acc[i + m / 2] : acc[i];
          const float send = hi ? acc[i] : acc[i + m / 2];
          acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
#pragma unroll
      for (int i = 0; i < EPL; ++i) vv[i] = acc[i];
    } else {
#pragma unroll
      for (int e = 0; e < NV; ++e) acc[e] = warp_sum_xor(acc[e]);
      vv[0] = 0.f;
#pragma unroll
      for (int e = 0; e < NV; ++e)
        if (lane == e) vv[0] = acc[e];
    }
    float hh[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) {
      const int e = (NV >= 32) ? EPL * lane + i : lane, n = e >> 2, q = e & 3;
      const int64_t d = u * 4 + q;
      bool flag = false;
      if (p.recheck && e < NV && n < p.nrows && d < p.D) {
        const float tau = p.tau_coef * xnorm_s[n] * bns[(int)(d - col0)] + kSignBoundAbs;
        flag = fabsf(vv[i]) <= tau;
      }
      hh[i] = hardsign(vv[i]);
      unsigned mask = __ballot_sync(0xffffffffu, flag);
      nrecheck += __popc(mask);
      while (mask) {            // float64 re-evaluation, fixed lane order
        const int src = __ffs(mask) - 1;
        mask &= mask - 1;
        const int se = (NV >= 32) ? EPL * src + i : src, sn = se >> 2, sq = se & 3;
        const int64_t sd = u * 4 + sq;
        // the provisional sign enters Stage II; the recheck is deferred to the end of the
        // CTA's stream, spread over all consumer warps (the Bt row fetched into L2 now, one
        // 128-byte line per lane), or run now when the CTA's list is full
        const float hp = __shfl_sync(0xffffffffu, hh[i], src);
        int slot = 0;
        if (lane == 0) slot = atomicAdd(&ndefer_s, 1);
        slot = __shfl_sync(0xffffffffu, slot, 0);
        if (slot < p.nslot) {
          // the Bt row by one bulk copy into row slot `slot` (queued behind the B stream;
          // it has landed by the end of the stream)
          if (lane == 0) {
            defer_s[slot] = make_int2(sn | (hp < 0.f ? int(0x80000000u) : 0), (int)sd);
            const uint32_t rb = (uint32_t)((F * 4 + 15) & ~15);   // Fp >= F rounded: in bounds
            mbar_arrive_expect_tx(slotbar + slot, rb);
            bulk_load(rows_s + (size_t)slot * slotf, p.Bt + sd * p.Fp, rb, slotbar + slot);
          }
        } else if (slot < kDefer) {
          if (lane == 0) defer_s[slot] = make_int2(sn | (hp < 0.f ? int(0x80000000u) : 0), (int)sd);
          const char* row = reinterpret_cast<const char*>(p.Bt + sd * p.Fp);
          for (int l = lane; l * 128 < F * 4; l += 32)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(row + l * 128));
        } else {
          flip_correct(sn, sd, hp, -1);
        }
      }
    }
    // ---- S_local[n][k] += sum_q H[n][q] C[k][4u + q]  (q ascending; padded C = 0)
    const int cl = (int)(u - u0) * 4;
    for (int i0 = 0; i0 < p.nrows * K; i0 += 32) {  // warp-uniform trip count (shuffles)
      const int i = i0 + lane;
      const bool ok = i < p.nrows * K;
      const int n = ok ? i / K : 0, k = ok ? i % K : 0;
      float h[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = n * 4 + q;                      // owner: lane e / EPL, slot e % EPL
        float hv = 0.f;
#pragma unroll
        for (int j = 0; j < EPL; ++j) {
          const float t = __shfl_sync(0xffffffffu, hh[j], (NV >= 32) ? (e / EPL) & 31 : e & 31);
          if (((NV >= 32) ? e % EPL : 0) == j) hv = t;
        }
        h[q] = hv;
      }
      if (ok) {
        const float* cr = Cs + k * ncol + cl;
        float a = sw[i];
        a = fmaf(h[0], cr[0], a);
        a = fmaf(h[1], cr[1], a);
        a = fmaf(h[2], cr[2], a);
        a = fmaf(h[3], cr[3], a);
        sw[i] = a;
      }
    }
  }
  SS_MARK(5);
  cbar();
  {
    const int nd = min(ndefer_s, kDefer);
    for (int j = warp; j < nd; j += kCw) {          // the deferred rechecks, over all warps
      const int2 e = defer_s[j];
      flip_correct(e.x & 0x7fffffff, (int64_t)e.y, e.x < 0 ? -1.f : 1.f, j < p.nslot ? j : -1);
    }
  }
  if (lane == 0 && nrecheck) atomicAdd(p.recheck_count, nrecheck);
  SS_MARK(2);
  cbar();

  // ---- CTA S_local = per-warp partials in warp order, converted to int64 fixed point
  // (2^-shift units) and added across CTAs with integer atomics: exact and order-free
  // (Alg. 3 `S += S_local`), so the last CTA only converts the N x K sums
  const int nk = p.nrows * K;
  for (int i = tid; i < nk; i += kCt) {
    float a = Sw[i];
    for (int w = 1; w < kCw; ++w) a += Sw[(size_t)w * NB * K + i];
    atomicAdd(p.acc + i, (unsigned long long)llrint((double)a * p.scale));
  }
  cbar();
  SS_MARK(3);
  if (tid == 0) {
    // acq_rel: this CTA's additions are ordered before its arrival is counted (release), and
    // the last arriver sees every other CTA's (acquire) -- one round trip
    unsigned prev;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(p.cnt) : "memory");
    s_last = (prev == (unsigned)(p.G - 1)) ? 1 : 0;
    if (s_last) p.cnt[0] = 0u;
  }
  cbar();
  if (!s_last) return;
  float* Sfin = fin;                                  // [nk]
  for (int i = tid; i < nk; i += kCt) {
    const long long a = (long long)atomicExch(p.acc + i, 0ull);   // read and reset for the next call
    const float v = (float)((double)a * p.inv_scale);
    Sfin[i] = v;
    if (p.scores) p.scores[i] = v;
  }
  cbar();
  SS_MARK(4);
  if (p.xworld > 0) {
    // ---- D-shard exchange over peer memory (Alg. 3 `S += S_local`, across GPUs):
    // buffer of rank r = xworld uint32 signals (padded to 4 words), then
    // [2 parities][xworld senders][xstride] floats.  (1) store this rank's S_local into slot (parity, xrank) of every
    // rank's buffer (peer stores over NVLink), (2) fence, release-store the epoch into
    // signal[xrank] of every rank, (3) acquire-wait until all signals of our own buffer
    // reached the epoch, (4) sum the slots in rank order: identical on every rank.
    // Parity double-buffering: a rank writes slot parity e & 1 of call e only after it
    // received every rank's call e-1 signal, i.e. after they finished reading call e-2.
    const int W = p.xworld, par = (int)(p.xepoch & 1u);
    const int xstride = (int)dshard_slot_floats(K), sigpad = (W + 3) & ~3;   // N-independent slots
    for (int r = 0; r < W; ++r) {
      float* dst = p.xbufs[r] + sigpad + ((size_t)par * W + p.xrank) * xstride;
      for (int i = tid; i < nk; i += kCt) dst[i] = Sfin[i];
    }
    __threadfence_system();
    cbar();
    if (tid < W) {
      uint32_t* sig = reinterpret_cast<uint32_t*>(p.xbufs[tid]);
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(sig + p.xrank), "r"(p.xepoch) : "memory");
    }
    if (tid < W) {
      const uint32_t* sig = reinterpret_cast<const uint32_t*>(p.xbufs[p.xrank]);
      uint32_t v;
      do {
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(sig + tid) : "memory");
      } while ((int32_t)(v - p.xepoch) < 0);
    }
    cbar();
    const float* own = p.xbufs[p.xrank] + sigpad + (size_t)par * W * xstride;
    for (int i = tid; i < nk; i += kCt) {
      float a = own[i];
      for (int r = 1; r < W; ++r) a += own[(size_t)r * xstride + i];
      Sfin[i] = a;
      if (p.scores) p.scores[i] = a;
    }
    cbar();
  }
  if (p.labels)
    for (int n = tid; n < p.nrows; n += kCt) {
      int best = 0;
      float bv = Sfin[n * K];
      for (int k = 1; k < K; ++k)
        if (Sfin[n * K + k] > bv) {
          bv = Sfin[n * K + k];
          best = k;
        }
      p.labels[n] = best;
    }
}

size_t stream_smem(int nst, int64_t F, int NB, int64_t K, int64_t max_cols, int nslot = 0) {
  auto up4 = [](size_t x) { return (x + 3) & ~size_t(3); };
  return (2 * kCw * kStagesMax + 2) * 8 +
         sizeof(float) * ((size_t)kCw * nst * kChunkRows * 4 + up4((size_t)F * NB + 4) + 4 +
                          up4((size_t)kCw * NB * K) + up4((size_t)K * max_cols) + up4(max_cols) +
                          up4((size_t)NB * K + 32 + 4 * kCt + 32) + (size_t)nslot * ((F + 3) & ~3) + 8);
}

template <int NB, bool HALF>
cudaError_t launch_stream_nb(StreamParams p, cudaStream_t st) {
  const size_t lim = kSmemDyn;
  int nst = kStagesMax;
  while (nst > 2 && stream_smem(nst, p.F, NB, p.K, p.max_cols) > lim) --nst;
  // recheck row slots in what is left: ring stages are traded (down to 3) for the slots a
  // CTA's flags need (cfg3, hi plane: ~2 flags per CTA at N = 1, max ~7; ~9 at N = 4, max
  // ~20 over 148 CTAs; fp32 B: ~0.1 per CTA); a flag beyond the slots reads its row from L2
  auto slots_at = [&](int ns) {
    const size_t used = stream_smem(ns, p.F, NB, p.K, p.max_cols);
    const size_t per = sizeof(float) * ((p.F + 3) & ~3);
    return used > lim ? 0 : (int)std::min<size_t>(kSlotsMax, (lim - used) / per);
  };
  const int want = HALF ? 12 : 4;
  while (nst > 3 && slots_at(nst) < want) --nst;
  p.nslot = slots_at(nst);
  const size_t sm = stream_smem(nst, p.F, NB, p.K, p.max_cols, p.nslot);
  if (sm > lim) return cudaErrorInvalidValue;
  p.nst = nst;
  // the attribute is per device context: set once per device (host call only then)
  constexpr int kMaxDev = 64;
  static std::atomic<size_t> attr_set[kMaxDev];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDev || sm > attr_set[dev].load()) {
    cudaError_t e = cudaFuncSetAttribute(smallstream_kernel<NB, HALF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)lim);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < kMaxDev) attr_set[dev] = lim;
  }
  static unsigned long long* dbg = nullptr;
  const bool debug = getenv("HDC_SMALL_DEBUG") != nullptr;
  if (debug) {
    if (!dbg) cudaMalloc((void**)&dbg, 8 * sizeof(unsigned long long));
    unsigned long long init[8] = {~0ull, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyAsync(dbg, init, sizeof(init), cudaMemcpyHostToDevice, st);
    p.dbg = dbg;
  }
  smallstream_kernel<NB, HALF><<<p.G, kThreadsS, sm, st>>>(p);
  cudaError_t le = cudaGetLastError();
  if (debug && le == cudaSuccess) {
    unsigned long long h[8];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, dbg, sizeof(h), cudaMemcpyDeviceToHost);
    fprintf(stderr, "[hdc smallstream debug] NB=%d nst=%d nslot=%d: from first CTA start (us): X staged %.2f, "
            "streams done %.2f, rechecks done %.2f, published %.2f, final %.2f\n", NB, p.nst, p.nslot,
            (h[1] - h[0]) * 1e-3, (h[5] - h[0]) * 1e-3, (h[2] - h[0]) * 1e-3, (h[3] - h[0]) * 1e-3, h[4] ? (h[4] - h[0]) * 1e-3 : -1.0);
  }
  return le;
}

// hi plane of B4 and its per-column sign bound (see smallstream_kernel HALF):
// |x.b - fl32(x.b_hi)| <= ||x|| ||b_lo|| + tau_F ||x|| ||b_hi||, b_lo = b - b_hi exact in fp32,
// tau_F = sign_bound_coef(F) (the fp32 evaluation, as for fp32 B); the factor
// (1 + 2 F u + 2^-10) covers the fp32 evaluation of ||x|| and the rounding of the bound.
__global__ void hi_plane_kernel(const float* __restrict__ B4, int64_t n4, uint16_t* __restrict__ B4h) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 b = reinterpret_cast<const float4*>(B4)[i];
    ushort4 h;
    h.x = __bfloat16_as_ushort(__float2bfloat16_rn(b.x));
    h.y = __bfloat16_as_ushort(__float2bfloat16_rn(b.y));
    h.z = __bfloat16_as_ushort(__float2bfloat16_rn(b.z));
    h.w = __bfloat16_as_ushort(__float2bfloat16_rn(b.w));
    reinterpret_cast<ushort4*>(B4h)[i] = h;
  }
}

__global__ void hi_bound_kernel(const float* __restrict__ Bt, int64_t F, int64_t Fp, int64_t Dp, double coef,
                                double slack, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t d = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (d >= Dp) return;
  double shi = 0.0, slo = 0.0;
  for (int64_t f = lane; f < F; f += 32) {
    const float b = Bt[d * Fp + f];
    const float hi = __bfloat162float(__float2bfloat16_rn(b));
    const double lo = (double)b - (double)hi;     // exact
    shi += (double)hi * (double)hi;
    slo += lo * lo;
  }
  shi = warp_sum_xor(shi);
  slo = warp_sum_xor(slo);
  if (lane == 0) out[d] = __double2float_ru((sqrt(slo) + coef * sqrt(shi)) * slack);
}

}  // namespace

cudaError_t launch_hi_plane(const float* B4, const float* Bt, int64_t F, int64_t Fp, int64_t Dp, uint16_t* B4h,
                            float* hibound, cudaStream_t st) {
  const int64_t n4 = Fp * Dp / 4;
  hi_plane_kernel<<<(unsigned)std::min<int64_t>((n4 + 255) / 256, 148 * 32), 256, 0, st>>>(B4, n4, B4h);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const double u = 1.0 / 16777216.0;
  const double slack = 1.0 + 2.0 * (double)F * u + 1.0 / 1024.0;
  hi_bound_kernel<<<(unsigned)((Dp * 32 + 255) / 256), 256, 0, st>>>(Bt, F, Fp, Dp, (double)sign_bound_coef(F),
                                                                     slack, hibound);
  return cudaGetLastError();
}

bool smallstream_fits(int64_t F, int64_t D, int64_t K, int n, int num_sms) {
  const int nb = n <= 1 ? 1 : n <= 4 ? 4 : n <= 8 ? 8 : n <= 16 ? 16 : 32;   // template NB used
  const int64_t units = (D + 3) / 4, G = std::min<int64_t>(units, num_sms);
  return stream_smem(2, F, nb, K, 4 * ((units + G - 1) / G)) <= kSmemDyn &&
         (int64_t)n * F * 4 + 16 < (int64_t(1) << 20);          // one bulk copy (tx-count limit)
}

cudaError_t launch_smallstream(const ModelView& m, const SmallWorkspace& ws, const float* X, int n,
                               float* scores, int32_t* labels, bool recheck, int num_sms,
                               cudaStream_t st, const DshardExchange* xc) {
  StreamParams p;
  p.xbufs = xc ? xc->bufs : nullptr;
  p.xrank = xc ? xc->rank : 0;
  p.xworld = xc ? xc->world : 0;
  p.xepoch = xc ? xc->epoch : 0u;
  p.X = X;
  p.nrows = n;
  p.F = m.F;
  p.D = m.D;
  p.Dp = m.Dp;
  p.K = m.K;
  p.Fp = m.Fp;
  p.B4 = m.B4;
  p.Bt = m.Bt;
  p.Cp = m.Cp;
  // sign-exact calls stream the bf16 hi plane when the model has one (half the bytes)
  // (HDC_SMALL_FULLB: stream the fp32 B4 instead, for measurements)
  // (n == 1 only: at cfg3 the hi plane's ~3% flags per element cost ~2 us of rechecks per
  // launch from N = 4 (18.5 vs 17.9 us), at N = 1 the halved stream wins (14.5 vs 16.5 us))
  // (HDC_SMALL_HALF4: also at 2 <= n <= 4, a measurement switch)
  const bool half = recheck && (n == 1 || (n <= 4 && getenv("HDC_SMALL_HALF4"))) && m.B4h && m.hibound &&
                    !getenv("HDC_SMALL_FULLB");
  p.B4h = half ? m.B4h : nullptr;
  p.bnorm = half ? m.hibound : m.bnorm;
  p.tau_coef = half ? 1.0f : m.tau_coef;
  p.recheck = recheck ? 1 : 0;
  p.units = (m.D + 3) / 4;
  p.G = (int)std::min<int64_t>(p.units, num_sms);
  p.max_cols = (int)(4 * ((p.units + p.G - 1) / p.G));
  p.nst = 0;
  p.S_part = ws.S_part;
  p.cnt = ws.cnt1;
  p.acc = ws.acc;
  p.scale = ldexp(1.0, ws.shift);
  p.inv_scale = ldexp(1.0, -ws.shift);
  p.recheck_count = ws.recheck;
  p.scores = scores;
  p.labels = labels;
  p.dbg = nullptr;
  if (half) {
    if (n <= 1) return launch_stream_nb<1, true>(p, st);
    if (n <= 4) return launch_stream_nb<4, true>(p, st);
    if (n <= 8) return launch_stream_nb<8, true>(p, st);
    if (n <= 16) return launch_stream_nb<16, true>(p, st);
    return launch_stream_nb<32, true>(p, st);
  }
  if (n <= 1) return launch_stream_nb<1, false>(p, st);
  if (n <= 4) return launch_stream_nb<4, false>(p, st);
  if (n <= 8) return launch_stream_nb<8, false>(p, st);
  if (n <= 16) return launch_stream_nb<16, false>(p, st);
  return launch_stream_nb<32, false>(p, st);
}

}  // namespace hdc
