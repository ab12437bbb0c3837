// k_fused_tc.cu -- K4: fused large-batch HDC inference on the 5th-gen tensor
// cores (tcgen05 + TMEM + TMA), sm_100a.
//
// Alg. 1 per (N-tile of 128 rows) x (D-tile of 80 columns):
//   Stage I   V_tile = X_tile B_tile: tcgen05.mma, accumulators in TMEM
//             (eq. batch_encode);
//   act       HardSign in the epilogue warps after tcgen05.ld, written
//             as exact bf16 +-1 into a shared-memory H tile;
//   Stage II  S[n, :] += H_tile C_tile^T as a second tcgen05.mma (bf16, C split
//             into hi + lo bf16 parts) into a TMEM accumulator that lives for the
//             CTA's whole run of D-tiles of one N-tile (eq. batch_sim P:180-183;
//             ScalableHD-L row ownership, Alg. 4).
// H never leaves the SM.
//
// Precision modes (hdc_precision_t):
//   BF16  X, B rounded to bf16 (RN); kind::f16, fp32 accumulate.
//   TF32  X, B rounded to tf32 (RNA); kind::tf32, fp32 accumulate.
//   INT8x3 (HDC_PREC_FP32_TC, sign-exact): per-row/column scaled 21-bit integer
//         images of X and B split into three balanced base-128 int8 limbs; the
//         six limb products with i + j <= 2 run as kind::i8 MMAs with EXACT int32
//         accumulation into three TMEM accumulators, combined in int64.  The
//         rigorous bound of that integer image flags the few
//         |I| <= tau, re-evaluated in float64 -> every HardSign decision equals
//         that of the exact product X B.
//
// Warp roles (384 threads, one CTA per SM, persistent over a contiguous range
// of the n-major tile sequence): warp 0 TMA producer, warp 1 MMA issuer (and
// TMEM owner), warps 4..11 epilogue (warp w reads TMEM lanes 32*(w%4).. and
// column half (w-4)/4).  smem: 4-stage ring of SWIZZLE_64B K-major operand
// tiles, 2 H tiles, 2 C tiles (interleaved K-major bf16 hi/lo); TMEM: two
// Stage I accumulator buffers + the Stage II accumulator.  Partial scores of
// N-tiles split between CTAs are summed in CTA order by the last-arriving CTA,
// which takes the lowest-index argmax: bit-deterministic.
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace hdc {
namespace {

using namespace ptx;

constexpr int BM = 128;              // rows per tile (MMA M)
constexpr int BN = 80;               // D columns per tile; 10000 = 125 x 80
constexpr int STAGES_MAX = 6;
#ifndef HDC_TC_EPI_WARPS
#define HDC_TC_EPI_WARPS 8
#endif
constexpr int NUM_EPI = HDC_TC_EPI_WARPS;           // epilogue warps: 4 lane quarters x NUM_CQ
constexpr int THREADS = 32 * (4 + NUM_EPI);         // + producer, MMA, C-producer, spare
constexpr int EPI_WARP0 = 4;
constexpr int NUM_CQ = NUM_EPI / 4;                 // column groups of the 80-wide tile
constexpr int EPI_COLS = BN / NUM_CQ;               // columns per epilogue warp
constexpr int MAX_LIMBS = 3;
constexpr int H_BYTES = BM * BN * 2;                 // bf16 H tile (interleaved K-major)
constexpr int CORE_LBO = 128;                        // K-adjacent 8x16B core matrices
constexpr int CORE_SBO = (BN / 8) * 128;             // 8-row groups (10 core matrices)
constexpr int KP_MAX_I8 = 32;                        // Stage II N (classes) limits
constexpr int KP_MAX_16 = 64;
constexpr int C_SLOT_MAX = 2 * KP_MAX_16 * BN * 2;   // bf16 hi + lo, [Kp][80] each

template <int MODE>
struct Cfg {
  static constexpr int NL = (MODE == 2) ? 3 : 1;
  static constexpr int ESZ = (MODE == 0) ? 2 : (MODE == 1) ? 4 : 1;
  // K bytes per stage = one swizzle-atom row: 128 B (SWIZZLE_128B) for the single-operand
  // modes, 64 B (SWIZZLE_64B) for the 3-limb int8 mode (smem budget).
  static constexpr int KBYTES = (MODE == 2) ? 64 : 128;
  static constexpr int SWZ = (MODE == 2) ? 4 : 2;                // descriptor layout type
  static constexpr int SBO = 8 * KBYTES;                         // 8-row core group
  static constexpr int A_LIMB_BYTES = BM * KBYTES;
  static constexpr int B_LIMB_BYTES = BN * KBYTES;
  static constexpr int KE = KBYTES / ESZ;                      // K elements per stage
  static constexpr int ACC_STRIDE = (MODE == 2) ? 3 * BN : 128;  // TMEM cols per Stage I buffer
  static constexpr int D2_COL = (MODE == 2) ? 480 : 256;          // Stage II accumulator
  static constexpr int KP_MAX = (MODE == 2) ? KP_MAX_I8 : KP_MAX_16;
  // Stage II operand per D-tile: int8 mode (FFMA Stage II in the epilogue) fp32 C^T [80][KPF]
  // + int64 column taus; other modes bf16 hi/lo [Kp][80] interleaved (Stage II MMA).
  static constexpr bool S2F = (MODE == 2);
  static constexpr int C_SLOT = S2F ? BN * KP_MAX * 4 + BN * 8 : 2 * KP_MAX * BN * 2;
  static constexpr int H_REGION = S2F ? BM * KP_MAX * 4 : 2 * H_BYTES;   // S reduction | H tiles
  static constexpr int STAGES_ = (MODE == 2) ? 4 : 5;
  static constexpr int A_STAGE = NL * A_LIMB_BYTES;
  static constexpr int B_STAGE = NL * B_LIMB_BYTES;
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = OFF_A + STAGES_ * A_STAGE;
  static constexpr int OFF_H = OFF_B + STAGES_ * B_STAGE;
  static constexpr int OFF_C = OFF_H + H_REGION;
  static constexpr int OFF_BAR = OFF_C + 2 * C_SLOT;
  static constexpr int TOTAL = OFF_BAR + 512;
  static_assert(OFF_B % 1024 == 0 && OFF_H % 1024 == 0 && OFF_C % 1024 == 0, "alignment");
  static_assert(TOTAL + 1024 <= 227 * 1024, "shared memory budget");
};

struct TcParams {
  int64_t N, F, Fp, D, Dp, Dq, K, Kp, Np;
  int Tn, Td, G;
  int64_t T;
  const float* X;          // caller's X (fp64 recheck)
  const float* Bt;         // fp32 B^T [Dp][Fp] (fp64 recheck)
  const int64_t* rowtau;   // int8 mode: per-row part of tau (units of 2^14)
  const int64_t* coltau;   // int8 mode: per-column part of tau
  const uint8_t* Cil;      // per D-tile Stage II operand (see Cfg::C_SLOT), c_tile_bytes each
  uint32_t c_tile_bytes;
  int kpf;                 // int8 mode: class stride of the fp32 C^T tiles (K rounded up to 4)
  float* S_part;           // [G][2][BM][K]
  unsigned* cnt;           // [Tn]
  unsigned long long* recheck_count;
  float* scores;
  int32_t* labels;
  int debug;               // diagnostics only (HDC_TC_DEBUG): 1 = no Stage I MMA, 2 = no operand TMA,
                           // 4 = per-role wait-cycle counters into dbg[]
  unsigned long long* dbg; // [16] cycle counters (debug & 4)
};

// Timed barrier wait (diagnostics): accumulates the cycles spent waiting.
#define TWAIT(slot, bar, par)                                        \
  do {                                                               \
    if (p.debug & 4) {                                               \
      const long long _t0 = clock64();                               \
      mbar_wait(bar, par);                                           \
      dbgc[slot] += (unsigned long long)(clock64() - _t0);           \
    } else {                                                         \
      mbar_wait(bar, par);                                           \
    }                                                                \
  } while (0)

__device__ __forceinline__ int64_t range_begin(int c, int64_t T, int G) { return (int64_t)c * T / G; }
__device__ __forceinline__ int owner_of(int64_t t, int64_t T, int G) {
  int c = (int)((t * G) / T);
  while (c + 1 < G && range_begin(c + 1, T, G) <= t) ++c;
  while (c > 0 && range_begin(c, T, G) > t) --c;
  return c;
}

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// float64 re-evaluation of V[row, d] (fixed lane order, warp-cooperative).
__device__ __forceinline__ float recheck_warp(const TcParams& p, int64_t row, int64_t d, int lane) {
  const float* xr = p.X + row * p.F;
  const float* br = p.Bt + d * p.Fp;
  double s = 0.0;
  for (int64_t f = lane; f < p.F; f += 32) s = fma((double)__ldg(xr + f), (double)__ldg(br + f), s);
  s = warp_sum_xor(s);
  return s >= 0.0 ? 1.f : -1.f;
}

__device__ __forceinline__ bool seg_last(int64_t t, int64_t t1, int Td) {
  return (t + 1 == t1) || ((t + 1) / Td != t / Td);
}

template <int MODE, int KT>
__global__ void __launch_bounds__(THREADS, 1)
fused_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const TcParams p) {
  using CF = Cfg<MODE>;
  constexpr bool S2F = CF::S2F;
  constexpr int NL = CF::NL;
  constexpr int KE = CF::KE;
  constexpr uint32_t IDESC = make_idesc<MODE>(BM, BN);
  constexpr uint32_t IDESC_N160 = make_idesc<MODE>(BM, 2 * BN);
  constexpr uint32_t IDESC_N240 = make_idesc<MODE>(BM, 3 * BN);
  constexpr uint32_t STAGE_TX = NL * (CF::A_LIMB_BYTES + CF::B_LIMB_BYTES);
  constexpr int A_LIMB_BYTES = CF::A_LIMB_BYTES;
  constexpr int KBYTES = CF::KBYTES;
  constexpr int STAGES = CF::STAGES_;
  auto sdesc = [](uint32_t addr) { return smem_desc_sw(addr, CF::SBO, CF::SWZ); };

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the swizzled tiles, keeping the pointer in the shared space
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem + CF::OFF_A;
  uint8_t* sB = smem + CF::OFF_B;
  uint8_t* sH = smem + CF::OFF_H;
  uint8_t* sC = smem + CF::OFF_C;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + CF::OFF_BAR);
  uint64_t* full = bars;                 // [STAGES] operands landed
  uint64_t* empty = bars + STAGES;       // [STAGES] operands consumed
  uint64_t* tfull = bars + 2 * STAGES;   // [2] Stage I accumulator ready
  uint64_t* tempty = tfull + 2;          // [2] Stage I accumulator drained
  uint64_t* cfull = tempty + 2;          // [2] C tile landed
  uint64_t* cempty = cfull + 2;          // [2] C tile consumed (Stage II MMA done)
  uint64_t* hfull = cempty + 2;          // [2] H tile written
  uint64_t* hempty = hfull + 2;          // [2] H tile consumed
  uint64_t* sfull = hempty + 2;          // [1] Stage II accumulator of a run complete
  uint64_t* sempty = sfull + 1;          // [1] Stage II accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sempty + 1);
  int* s_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x;
  const int64_t t0 = range_begin(c, p.T, p.G), t1 = range_begin(c + 1, p.T, p.G);
  const int KB = (int)(p.Fp / KE);
  unsigned long long dbgc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) dbgc[i] = 0;
  const long long t_start = clock64();
  const uint32_t c_tile_bytes = p.c_tile_bytes;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull + b, 1);
      mbar_init(tempty + b, NUM_EPI);
      mbar_init(cfull + b, 1);
      mbar_init(cempty + b, S2F ? NUM_EPI : 1);
      mbar_init(hfull + b, NUM_EPI);
      mbar_init(hempty + b, 1);
    }
    mbar_init(sfull, 1);
    mbar_init(sempty, 4);               // the 4 warps of column quarter 0 drain S
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================================================== TMA producer (operands)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = t0; t < t1; ++t) {
        const int ni = (int)(t / p.Td), di = (int)(t % p.Td);
        for (int kb = 0; kb < KB; ++kb) {
          TWAIT(0, empty + stage, phase ^ 1);
          if (p.debug & 2) {
            mbar_arrive(full + stage);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          mbar_arrive_expect_tx(full + stage, STAGE_TX);
#pragma unroll
          for (int l = 0; l < NL; ++l) {
            tma_load_2d(sA + stage * CF::A_STAGE + l * A_LIMB_BYTES, &tmA, full + stage, kb * KE,
                        (int)(l * p.Np + (int64_t)ni * BM));
            tma_load_2d(sB + stage * CF::B_STAGE + l * CF::B_LIMB_BYTES, &tmB, full + stage, kb * KE,
                        (int)(l * p.Dq + (int64_t)di * BN));
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 2) {
    // ===================================================== C-tile producer (Stage II B operand)
    // A separate warp, so the operand stream never waits for a C slot.
    if (lane == 0) {
      int cs = 0;
      uint32_t cphase = 0;
      for (int64_t t = t0; t < t1; ++t) {
        const int di = (int)(t % p.Td);
        mbar_wait(cempty + cs, cphase ^ 1);
        mbar_arrive_expect_tx(cfull + cs, c_tile_bytes + (MODE == 2 ? BN * 8 : 0));
        bulk_load(sC + cs * CF::C_SLOT, p.Cil + (int64_t)di * c_tile_bytes, c_tile_bytes, cfull + cs);
        if constexpr (MODE == 2)
          bulk_load(sC + cs * CF::C_SLOT + c_tile_bytes, p.coltau + (int64_t)di * BN, BN * 8,
                    cfull + cs);
        cs ^= 1;
        if (cs == 0) cphase ^= 1;
      }
    }
  } else if (warp == 1) {
    // ===================================================== MMA issuer (whole warp, elected lane issues)
    {
      int stage = 0, buf = 0, hb = 0, cs = 0;
      uint32_t phase = 0, bphase = 0, hphase = 0, cphase = 0, sphase = 0;
      bool seg_first = true;
      const uint32_t IDESC2 = make_idesc<0>(BM, (int)p.Kp);
      const uint32_t d2 = tmem_base + CF::D2_COL;
      // Stage II for tile tt: S += H(tt) [Chi(tt) + Clo(tt)]^T
      auto stage2 = [&](int64_t tt) {
        TWAIT(3, hfull + hb, hphase);
        TWAIT(4, cfull + cs, cphase);
        if (seg_first) TWAIT(5, sempty, sphase ^ 1);   // previous run's S drained
        tc_fence_after();
        const uint32_t h_base = smem_u32(sH + hb * H_BYTES);
        const uint32_t c_base = smem_u32(sC + cs * CF::C_SLOT);
#pragma unroll
        for (int s = 0; s < BN / 16; ++s) {
          const uint64_t ad = smem_desc_interleaved(h_base + s * 2 * CORE_LBO, CORE_LBO, CORE_SBO);
#pragma unroll
          for (int part = 0; part < 2; ++part) {
            const uint64_t bd = smem_desc_interleaved(
                c_base + part * (uint32_t)(p.Kp * BN * 2) + s * 2 * CORE_LBO, CORE_LBO, CORE_SBO);
            if (!(p.debug & 8)) tc_mma_elect<0>(d2, ad, bd, IDESC2, (seg_first && s == 0 && part == 0) ? 0u : 1u);
          }
        }
        seg_first = false;
        tc_commit_elect(hempty + hb);
        tc_commit_elect(cempty + cs);
        if (seg_last(tt, t1, p.Td)) {
          tc_commit_elect(sfull);
          seg_first = true;
          sphase ^= 1;
        }
        hb ^= 1;
        if (hb == 0) hphase ^= 1;
        cs ^= 1;
        if (cs == 0) cphase ^= 1;
      };
      for (int64_t t = t0; t < t1; ++t) {
        TWAIT(1, tempty + buf, bphase ^ 1);
        tc_fence_after();
        const uint32_t acc0 = tmem_base + buf * CF::ACC_STRIDE;
        const long long ts1 = clock64();
        for (int kb = 0; kb < KB; ++kb) {
          TWAIT(2, full + stage, phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * CF::A_STAGE);
          const uint32_t b_base = smem_u32(sB + stage * CF::B_STAGE);
#pragma unroll
          for (int ks = 0; ks < ((p.debug & 1) ? 0 : KBYTES / 32); ++ks) {
            const uint32_t acc = (kb == 0 && ks == 0) ? 0u : 1u;
            if constexpr (MODE == 2) {
              // The three B limb tiles are contiguous rows [b0; b1; b2] (240 x 64 B) and
              // the accumulators contiguous columns [A0 | A1 | A2], so one MMA per A limb:
              //   [A0|A1|A2] (+)= x0 [b0;b1;b2]^T,  [A1|A2] += x1 [b0;b1]^T,  A2 += x2 b0^T
              // (each A tile is read from shared memory once per k-step, not 3 times).
              const uint64_t bdesc = sdesc(b_base + ks * 32);
              tc_mma_elect<2>(acc0, sdesc(a_base + ks * 32), bdesc, IDESC_N240, acc);
              tc_mma_elect<2>(acc0 + BN, sdesc(a_base + A_LIMB_BYTES + ks * 32), bdesc,
                        IDESC_N160, 1u);
              tc_mma_elect<2>(acc0 + 2 * BN, sdesc(a_base + 2 * A_LIMB_BYTES + ks * 32), bdesc,
                        IDESC, 1u);
            } else {
              tc_mma_elect<MODE>(acc0, sdesc(a_base + ks * 32), sdesc(b_base + ks * 32),
                           IDESC, acc);
            }
          }
          tc_commit_elect(empty + stage);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit_elect(tfull + buf);
        if (p.debug & 4) dbgc[13] += (unsigned long long)(clock64() - ts1);
        buf ^= 1;
        if (buf == 0) bphase ^= 1;
        const long long ts2 = clock64();
        if constexpr (!S2F)
          if (t > t0) stage2(t - 1);        // overlaps the epilogue of tile t-1 with Stage I of t
        if (p.debug & 4) dbgc[14] += (unsigned long long)(clock64() - ts2);
      }
      if constexpr (!S2F)
        if (t1 > t0) stage2(t1 - 1);
    }
  } else if (warp >= EPI_WARP0) {
    // ===================================================== epilogue
    const int ew = warp - EPI_WARP0;
    const int q = warp & 3;                 // TMEM lane quarter (hardware: warp id % 4)
    const int cq = ew >> 2;                 // column quarter of the 80-wide tile
    const int m = q * 32 + lane;            // row within the N-tile
    const int K = (int)p.K;
    int buf = 0, hb = 0, cs = 0;
    uint32_t bphase = 0, hphase = 0, sphase = 0, cphase = 0;
    unsigned long long nrecheck = 0;
    const int first_ni = (int)(t0 / p.Td);
    float2 S2[KT / 2];                      // int8 mode: FFMA2 Stage II accumulators (this row)
#pragma unroll
    for (int k = 0; k < KT / 2; ++k) S2[k] = make_float2(0.f, 0.f);
#define SK(k) (((k) & 1) ? S2[(k) >> 1].y : S2[(k) >> 1].x)
    float* sRed = reinterpret_cast<float*>(sH);   // int8 mode: [K][BM] quarter reduction
    for (int64_t t = t0; t < t1; ++t) {
      const int ni = (int)(t / p.Td), di = (int)(t % p.Td);
      const int64_t row = (int64_t)ni * BM + m;
      const bool row_ok = row < p.N;
      int64_t rtau = -1;                    // int8 mode: row part of tau (-1: padded row, never flag)
      if constexpr (MODE == 2) rtau = row_ok ? __ldg(p.rowtau + row) : -(int64_t(1) << 62);
      TWAIT(6, tfull + buf, bphase);
      if constexpr (!S2F) TWAIT(7, hempty + hb, hphase ^ 1);
      const int64_t* sct = nullptr;         // column taus of this tile (int8 mode), in smem
      const float* sCt = nullptr;           // C^T tile [80][kpf] (int8 mode), in smem
      if constexpr (S2F) {
        TWAIT(15, cfull + cs, cphase);
        sCt = reinterpret_cast<const float*>(sC + cs * CF::C_SLOT);
        sct = reinterpret_cast<const int64_t*>(sC + cs * CF::C_SLOT + BN * KT * 4);
      }
      tc_fence_after();
      uint8_t* hrow = sH + hb * H_BYTES + (m >> 3) * CORE_SBO + (m & 7) * 16;
      const uint32_t tbase =
          tmem_base + ((uint32_t)(q * 32) << 16) + buf * CF::ACC_STRIDE + cq * EPI_COLS;
#pragma unroll 1
      for (int ch = 0; ch < ((p.debug & 16) ? 0 : EPI_COLS / 4); ++ch) {
        const int col0 = cq * EPI_COLS + ch * 4;   // column within the tile
        uint32_t hbits = 0;                         // bit j set -> h = -1
        if constexpr (MODE == 2) {
          uint32_t r0[4], r1[4], r2[4];
          tmem_ld4(tbase + ch * 4, r0);
          tmem_ld4(tbase + BN + ch * 4, r1);
          tmem_ld4(tbase + 2 * BN + ch * 4, r2);
          tmem_ld_wait();
          int64_t I[4];
          uint32_t fl = 0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            I[j] = (int64_t)(int32_t)r0[j] * 16384 + (int64_t)(int32_t)r1[j] * 128 +
                   (int64_t)(int32_t)r2[j];
            if (I[j] < 0) hbits |= 1u << j;
            const int64_t aI = I[j] < 0 ? -I[j] : I[j];
            if (aI <= rtau + sct[col0 + j]) fl |= 1u << j;   // coltau = -inf past D
          }
          if (__any_sync(0xffffffffu, fl != 0)) {
#pragma unroll 1
            for (int j = 0; j < 4; ++j) {
              unsigned mask = __ballot_sync(0xffffffffu, (fl >> j) & 1u);
              const int64_t d = (int64_t)di * BN + col0 + j;
              while (mask) {
                const int src = __ffs(mask) - 1;
                mask &= mask - 1;
                const int64_t srow = (int64_t)ni * BM + q * 32 + src;
                const float hv = recheck_warp(p, srow, d, lane);
                if (lane == src) hbits = hv < 0.f ? (hbits | (1u << j)) : (hbits & ~(1u << j));
                ++nrecheck;
              }
            }
          }
        } else {
          uint32_t r0[4];
          tmem_ld4(tbase + ch * 4, r0);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (!(__uint_as_float(r0[j]) >= 0.f)) hbits |= 1u << j;   // HardSign
        }
        if constexpr (S2F) {
          // Stage II on the FMA pipe: S[k] += h[c] C[k, d0 + c], c ascending (exact +-1 products;
          // padded columns have C = 0)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float h = ((hbits >> j) & 1u) ? -1.f : 1.f;
            const float4* ct = reinterpret_cast<const float4*>(sCt + (col0 + j) * KT);  // kpf == KT
#pragma unroll
            for (int k4 = 0; k4 < KT / 4; ++k4) {
              const float4 cv = ct[k4];
              S2[2 * k4 + 0] = ffma2(h, make_float2(cv.x, cv.y), S2[2 * k4 + 0]);
              S2[2 * k4 + 1] = ffma2(h, make_float2(cv.z, cv.w), S2[2 * k4 + 1]);
            }
          }
        } else {
          // 4 bf16 +-1 values (0x3F80 / 0xBF80) -> 8 bytes of a core-matrix row
          const uint32_t w0 = ((hbits & 1u) ? 0xBF80u : 0x3F80u) | (((hbits & 2u) ? 0xBF80u : 0x3F80u) << 16);
          const uint32_t w1 = ((hbits & 4u) ? 0xBF80u : 0x3F80u) | (((hbits & 8u) ? 0xBF80u : 0x3F80u) << 16);
          *reinterpret_cast<uint2*>(hrow + (col0 >> 3) * CORE_LBO + (col0 & 7) * 2) = make_uint2(w0, w1);
        }
      }
      tc_fence_before();
      if constexpr (!S2F) fence_proxy_async_smem();   // H writes -> visible to the tensor core
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(tempty + buf);
        if constexpr (S2F) mbar_arrive(cempty + cs);
        else mbar_arrive(hfull + hb);
      }
      buf ^= 1;
      if (buf == 0) bphase ^= 1;
      hb ^= 1;
      if (hb == 0) hphase ^= 1;
      cs ^= 1;
      if (cs == 0) cphase ^= 1;

      if (!seg_last(t, t1, p.Td)) continue;
      // ---- end of this CTA's run of D-tiles for N-tile ni: read S from TMEM
      const int c_first = owner_of((int64_t)ni * p.Td, p.T, p.G);
      const int c_last = owner_of((int64_t)(ni + 1) * p.Td - 1, p.T, p.G);
      const bool sole = (c_first == c_last);
      constexpr int FIN = S2F ? NUM_CQ - 1 : 0;   // column group that finalises the run's scores
      if constexpr (S2F) {
        // fixed-order reduction of the 4 column quarters: ((S0 + S1) + S2) + S3
        for (int qq = 0; qq < NUM_CQ - 1; ++qq) {
          if (cq == qq) {
#pragma unroll
            for (int k = 0; k < KT; ++k)
              if (k < K) sRed[k * BM + m] = (qq == 0) ? SK(k) : sRed[k * BM + m] + SK(k);
          }
          named_bar(1, NUM_EPI * 32);
        }
        if (cq == NUM_CQ - 1) {
#pragma unroll
          for (int k = 0; k < KT; ++k)
            if (k < K) SK(k) = sRed[k * BM + m] + SK(k);
        }
      }
      if (cq == FIN) {
        if constexpr (!S2F) TWAIT(8, sfull, sphase);
        tc_fence_after();
        const uint32_t sb = tmem_base + ((uint32_t)(q * 32) << 16) + CF::D2_COL;
        float* part = p.S_part + (((int64_t)c * 2 + ((ni == first_ni) ? 0 : 1)) * BM + m) * p.K;
        int best = 0;
        float bv = 0.f;
        auto take = [&](float v, int k) {
          if (sole) {
            if (row_ok && p.scores) p.scores[row * p.K + k] = v;
            if (k == 0 || v > bv) {
              bv = v;
              best = k;
            }
          } else {
            part[k] = v;
          }
        };
        if constexpr (S2F) {
#pragma unroll
          for (int k = 0; k < KT; ++k)
            if (k < K) take(SK(k), k);
        } else {
          for (int k0 = 0; k0 < K; k0 += 8) {
            uint32_t r[8];
            tmem_ld8(sb + k0, r);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (k0 + j < K) take(__uint_as_float(r[j]), k0 + j);
          }
        }
        tc_fence_before();
        __syncwarp();
        if constexpr (!S2F)
          if (lane == 0) mbar_arrive(sempty);
        if (sole && row_ok && p.labels) p.labels[row] = best;
        if (!sole) __threadfence();
      }
#pragma unroll
      for (int k = 0; k < KT; ++k) SK(k) = 0.f;
      sphase ^= 1;
      if (sole) continue;
      named_bar(1, NUM_EPI * 32);
      if (threadIdx.x == EPI_WARP0 * 32) {
        const unsigned prev = atomicAdd(p.cnt + ni, 1u);
        *s_flag = (prev == (unsigned)(c_last - c_first)) ? 1 : 0;
        if (*s_flag) p.cnt[ni] = 0u;
      }
      named_bar(1, NUM_EPI * 32);
      if (*s_flag && cq == FIN && row_ok) {
        __threadfence();
        int best = 0;
        float bv = 0.f;
        for (int k = 0; k < K; ++k) {
          float s = 0.f;
          for (int cc = c_first; cc <= c_last; ++cc) {
            const int slot = ((int)(range_begin(cc, p.T, p.G) / p.Td) == ni) ? 0 : 1;
            const float v = ld_cg(p.S_part + (((int64_t)cc * 2 + slot) * BM + m) * p.K + k);
            s = (cc == c_first) ? v : s + v;
          }
          if (p.scores) p.scores[row * p.K + k] = s;
          if (k == 0 || s > bv) {
            bv = s;
            best = k;
          }
        }
        if (p.labels) p.labels[row] = best;
      }
      named_bar(1, NUM_EPI * 32);     // s_flag reuse
    }
    if (MODE == 2 && lane == 0 && nrecheck) atomicAdd(p.recheck_count, nrecheck);
  }
  if ((p.debug & 4) && lane == 0 && (warp <= 2 || warp == EPI_WARP0)) {
    if (warp != 1) dbgc[13] = dbgc[14] = 0;
    if (warp != EPI_WARP0) dbgc[15] = 0;
    dbgc[9 + (warp == EPI_WARP0 ? 3 : warp)] = (unsigned long long)(clock64() - t_start);
    for (int i = 0; i < 16; ++i)
      if (dbgc[i]) atomicAdd(p.dbg + i, dbgc[i]);
  }
  __syncwarp();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

// ---------------------------------------------------------------- operand prep
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

// One warp per row of a row-major [rows][F] fp32 matrix (X rows, or B^T rows):
// int8 limbs into out[l][rows_p][Fp] and the per-row tau term.
__global__ void limb_rows_kernel(const float* __restrict__ src, int64_t rows, int64_t rows_p,
                                 int64_t F, int64_t ld_src, int64_t Fp, int8_t* __restrict__ out,
                                 int64_t* __restrict__ tau_part, int64_t tau_const) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= rows_p) return;
  const bool valid = r < rows;
  float amax = 0.f;
  if (valid)
    for (int64_t f = lane; f < F; f += 32) amax = fmaxf(amax, fabsf(src[r * ld_src + f]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  const float c = scale_for(amax);
  long long l1 = 0;
  for (int64_t f = lane; f < Fp; f += 32) {
    const float x = (valid && f < F) ? src[r * ld_src + f] : 0.f;
    int d0, d1, d2, U;
    limbs_of(x, c, d0, d1, d2, U);
    out[(0 * rows_p + r) * Fp + f] = (int8_t)d0;
    out[(1 * rows_p + r) * Fp + f] = (int8_t)d1;
    out[(2 * rows_p + r) * Fp + f] = (int8_t)d2;
    l1 += U < 0 ? -U : U;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) l1 += __shfl_xor_sync(0xffffffffu, l1, o);
  // |c_x c_b x.b - U_x.U_b| <= 0.625 (L1(U_x) + L1(U_b)) + 0.3907 F and the dropped limb
  // products (i + j >= 3) add <= F (2^20 + 2^12).  The kernel compares
  // I = A0 2^14 + A1 2^7 + A2 = (U_x.U_b - dropped) / 2^14, so tau is stored / 2^14,
  // rounded up: ceil((5 l1 / 8 + tau_const) / 2^14) = (5 l1 + 8 tau_const + 2^17 - 1) >> 17.
  if (lane == 0 && tau_part)
    tau_part[r] = valid ? ((5 * l1 + 8 * tau_const + 131071) >> 17) + 1 : -(int64_t(1) << 62);
}

// Rounded copies for the bf16 / tf32 modes: out[r][f] (rows_p x Fp, zero padded).
template <int MODE>
__global__ void round_rows_kernel(const float* __restrict__ src, int64_t rows, int64_t rows_p,
                                  int64_t F, int64_t ld_src, int64_t Fp, void* __restrict__ out) {
  const int64_t total = rows_p * Fp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / Fp, f = i % Fp;
    const float x = (r < rows && f < F) ? src[r * ld_src + f] : 0.f;
    if constexpr (MODE == 0) {
      reinterpret_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(x);
    } else {
      uint32_t y;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(y) : "f"(x));
      reinterpret_cast<uint32_t*>(out)[i] = y;
    }
  }
}


// C tiles for Stage II: per D-tile di, bf16 hi = RN(C), lo = RN(C - hi), each
// [Kp][80] in the interleaved K-major core-matrix layout the MMA B descriptor
// expects (core matrix (g, j) = rows 8g.., columns 8j.. at byte (10 g + j) * 128).
__global__ void c_interleave_kernel(const float* __restrict__ Cp, int64_t K, int64_t Kp, int64_t D,
                                    int64_t Dp, int64_t Td, __nv_bfloat16* __restrict__ out) {
  const int64_t per_part = Kp * BN;
  const int64_t total = Td * 2 * per_part;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t di = i / (2 * per_part);
    const int part = (int)((i / per_part) % 2);
    const int64_t e = i % per_part;          // element index inside the interleaved part
    const int64_t core = e / 64, inner = e % 64;
    const int64_t g = core / (BN / 8), j = core % (BN / 8);
    const int64_t r = g * 8 + inner / 8, cc = j * 8 + inner % 8;
    const int64_t d = di * BN + cc;
    const float v = (r < K && d < D) ? Cp[r * Dp + d] : 0.f;
    const __nv_bfloat16 hi = __float2bfloat16_rn(v);
    out[i] = part == 0 ? hi : __float2bfloat16_rn(v - __bfloat162float(hi));
  }
}

// int8 mode Stage II operand: fp32 C^T tiles [Td][80][kpf] (row = column d of the tile,
// classes contiguous, zero beyond K and beyond D).
__global__ void ct_tiles_kernel(const float* __restrict__ Cp, int64_t K, int64_t kpf, int64_t D,
                                int64_t Dp, int64_t Td, float* __restrict__ out) {
  const int64_t total = Td * BN * kpf;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i % kpf, dd = i / kpf;      // dd = global column index di * 80 + c
    out[i] = (k < K && dd < D) ? Cp[k * Dp + dd] : 0.f;
  }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

bool make_map_2d(CUtensorMap* m, CUtensorMapDataType dt, int esz, const void* base, uint64_t inner,
                 uint64_t outer, uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle sw) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * (uint64_t)esz};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  return enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int MODE, int KT>
cudaError_t launch_mode(const CUtensorMap& a, const CUtensorMap& b, const TcParams& p, cudaStream_t st) {
  const size_t sm = Cfg<MODE>::TOTAL + 1024;
  cudaError_t e = cudaFuncSetAttribute(fused_tc_kernel<MODE, KT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  fused_tc_kernel<MODE, KT><<<p.G, THREADS, sm, st>>>(a, b, p);
  return cudaGetLastError();
}

}  // namespace

int tc_tile_n() { return BN; }
int tc_max_k(int mode) { return mode == 2 ? KP_MAX_I8 : KP_MAX_16; }
int64_t tc_kp(int64_t K) { return (K + 15) / 16 * 16; }
int64_t tc_kpf(int64_t K) { return (K + 3) / 4 * 4; }
int64_t tc_c_tile_bytes(int mode, int64_t K) {
  return mode == 2 ? BN * tc_kpf(K) * 4 : 2 * tc_kp(K) * BN * 2;
}
int64_t tc_max_fp_int8() { return 100000; }

int64_t tc_tau_const(int64_t F) {
  // F (0.390625 + 2^20 + 2^12) + 1, in the integer units of U_x.U_b (before the 2^-14 scale)
  return (int64_t)F * 1052673 + 1;
}

cudaError_t launch_tc_limbs(const float* src, int64_t rows, int64_t rows_p, int64_t F, int64_t ld_src,
                            int64_t Fp, int8_t* out, int64_t* tau_part, int64_t tau_const,
                            cudaStream_t st) {
  const int warps = 8;
  limb_rows_kernel<<<(unsigned)((rows_p + warps - 1) / warps), warps * 32, 0, st>>>(
      src, rows, rows_p, F, ld_src, Fp, out, tau_part, tau_const);
  return cudaGetLastError();
}

cudaError_t launch_tc_round(int mode, const float* src, int64_t rows, int64_t rows_p, int64_t F,
                            int64_t ld_src, int64_t Fp, void* out, cudaStream_t st) {
  const int64_t total = rows_p * Fp;
  int64_t grid = (total + 255) / 256;
  if (grid > 148 * 16) grid = 148 * 16;
  if (mode == 0)
    round_rows_kernel<0><<<(unsigned)grid, 256, 0, st>>>(src, rows, rows_p, F, ld_src, Fp, out);
  else
    round_rows_kernel<1><<<(unsigned)grid, 256, 0, st>>>(src, rows, rows_p, F, ld_src, Fp, out);
  return cudaGetLastError();
}

cudaError_t launch_tc_c_tiles(int mode, const float* Cp, int64_t K, int64_t D, int64_t Dp, void* out,
                              cudaStream_t st) {
  const int64_t Td = (D + BN - 1) / BN;
  if (mode == 2) {
    const int64_t total = Td * BN * tc_kpf(K);
    int64_t grid = (total + 255) / 256;
    if (grid > 148 * 16) grid = 148 * 16;
    ct_tiles_kernel<<<(unsigned)grid, 256, 0, st>>>(Cp, K, tc_kpf(K), D, Dp, Td, (float*)out);
    return cudaGetLastError();
  }
  return launch_tc_c_interleave(Cp, K, tc_kp(K), D, Dp, out, st);
}

cudaError_t launch_tc_c_interleave(const float* Cp, int64_t K, int64_t Kp, int64_t D, int64_t Dp,
                                   void* out, cudaStream_t st) {
  const int64_t Td = (D + BN - 1) / BN;
  const int64_t total = Td * 2 * Kp * BN;
  int64_t grid = (total + 255) / 256;
  if (grid > 148 * 16) grid = 148 * 16;
  c_interleave_kernel<<<(unsigned)grid, 256, 0, st>>>(Cp, K, Kp, D, Dp, Td, (__nv_bfloat16*)out);
  return cudaGetLastError();
}

cudaError_t launch_fused_tc(int mode, const TcOperands& o, int64_t N, float* scores, int32_t* labels,
                            int num_sms, cudaStream_t st) {
  const int64_t Tn = o.N_p / BM;
  const int64_t Td = (o.D + BN - 1) / BN;
  TcParams p;
  p.N = N;
  p.F = o.F;
  p.Fp = o.Fp;
  p.D = o.D;
  p.Dp = o.Dp;
  p.Dq = o.Dq;
  p.K = o.K;
  p.Kp = tc_kp(o.K);
  p.Np = o.N_p;
  p.Tn = (int)Tn;
  p.Td = (int)Td;
  p.T = Tn * Td;
  p.G = (int)(p.T < num_sms ? p.T : num_sms);
  p.X = o.X;
  p.Bt = o.Bt;
  p.rowtau = o.rowtau;
  p.coltau = o.coltau;
  p.Cil = (const uint8_t*)o.Cil;
  p.kpf = (int)tc_kpf(o.K);
  p.c_tile_bytes = (uint32_t)tc_c_tile_bytes(mode, o.K);
  p.S_part = o.S_part;
  p.cnt = o.cnt;
  p.recheck_count = o.recheck;
  p.scores = scores;
  p.labels = labels;
  {
    const char* dbg = getenv("HDC_TC_DEBUG");
    p.debug = dbg ? atoi(dbg) : 0;
  }
  static unsigned long long* dbg_buf = nullptr;
  p.dbg = nullptr;
  if (p.debug & 4) {
    if (!dbg_buf) cudaMalloc((void**)&dbg_buf, 16 * sizeof(unsigned long long));
    cudaMemsetAsync(dbg_buf, 0, 16 * sizeof(unsigned long long), st);
    p.dbg = dbg_buf;
  }
  const int nl = (mode == 2) ? 3 : 1;
  const int esz = (mode == 0) ? 2 : (mode == 1) ? 4 : 1;
  const CUtensorMapDataType dt = (mode == 0)   ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                 : (mode == 1) ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                               : CU_TENSOR_MAP_DATA_TYPE_UINT8;
  CUtensorMap ma, mb;
  const uint32_t kbytes = (mode == 2) ? 64 : 128;
  const CUtensorMapSwizzle swz = (mode == 2) ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
  if (!make_map_2d(&ma, dt, esz, o.A, (uint64_t)o.Fp, (uint64_t)nl * o.N_p, kbytes / esz, BM, swz) ||
      !make_map_2d(&mb, dt, esz, o.B, (uint64_t)o.Fp, (uint64_t)nl * o.Dq, kbytes / esz, BN, swz))
    return cudaErrorInvalidValue;
  cudaError_t e;
  if (mode == 0) e = launch_mode<0, 4>(ma, mb, p, st);
  else if (mode == 1) e = launch_mode<1, 4>(ma, mb, p, st);
  else if (p.kpf <= 4) e = launch_mode<2, 4>(ma, mb, p, st);
  else if (p.kpf <= 8) e = launch_mode<2, 8>(ma, mb, p, st);
  else if (p.kpf <= 12) e = launch_mode<2, 12>(ma, mb, p, st);
  else if (p.kpf <= 16) e = launch_mode<2, 16>(ma, mb, p, st);
  else if (p.kpf <= 20) e = launch_mode<2, 20>(ma, mb, p, st);
  else if (p.kpf <= 24) e = launch_mode<2, 24>(ma, mb, p, st);
  else if (p.kpf <= 28) e = launch_mode<2, 28>(ma, mb, p, st);
  else e = launch_mode<2, 32>(ma, mb, p, st);
  if (e == cudaSuccess && (p.debug & 4)) {
    unsigned long long h[16];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, dbg_buf, sizeof(h), cudaMemcpyDeviceToHost);
    const char* names[16] = {"prod.empty", "mma.tempty", "mma.full", "mma.hfull", "mma.cfull",
                             "mma.sempty", "epi.tfull", "epi.hempty", "epi.sfull", "prod.total",
                             "mma.total", "cprod.total", "epi.total", "mma.SI", "mma.SII", "epi.cfull"};
    fprintf(stderr, "[hdc tc debug] mode %d, %d CTAs, %lld tiles; mean cycles per CTA:", mode, p.G,
            (long long)p.T);
    for (int i = 0; i < 16; ++i) fprintf(stderr, " %s=%.0f", names[i], (double)h[i] / p.G);
    fprintf(stderr, "\n");
  }
  return e;
}

}  // namespace hdc
