// k_fused_tc.cu -- K4: fused large-batch HDC inference on the 5th-gen tensor
// cores (tcgen05 + TMEM + TMA), sm_100a.
//
// Alg. 1 per (N-tile of 128 rows) x (D-tile of BN columns):
//   Stage I   V_tile = X_tile B_tile: tcgen05.mma, accumulators in TMEM
//             (eq. batch_encode);
//   act       HardSign in the epilogue warps after tcgen05.ld, written
//             as exact bf16 +-1 into TMEM (bf16/tf32) or a shared-memory H tile (int8);
//   Stage II  S_t = H_tile C_tile^T as a second tcgen05.mma (bf16; C split into
//             hi + lo bf16 parts, hi + mid + lo = C exactly in the int8 modes) into a
//             TMEM accumulator, drained per tile into exact int64 fixed-point row sums
//             that live for the CTA's whole run of D-tiles of one N-tile (eq. batch_sim
//             P:180-183; ScalableHD-L row ownership, Alg. 4).
// H never leaves the SM.
//
// Precision modes (hdc_precision_t):
//   BF16  X, B rounded to bf16 (RN); kind::f16, fp32 accumulate; BN = 160.
//   TF32  X, B rounded to tf32 (RNA); kind::tf32, fp32 accumulate; BN = 160.
//   INT8x3 (HDC_PREC_FP32_TC, sign-exact): per-row/column scaled 21-bit integer
//         images of X and B split into three balanced base-128 int8 limbs; the
//         six limb products with i + j <= 2 run as three N-concatenated kind::i8
//         MMAs with EXACT int32 accumulation into three TMEM accumulators (BN = 80,
//         double-buffered; or the "wide" mode for large F: BN = 160 as two 80-column
//         sub-tiles, one buffer), combined in int64.  The rigorous bound of that integer
//         image (DESIGN.md
//         §4) flags the few |I| <= tau; they are re-evaluated in float64 after the
//         kernel (tc_recheck_kernel), so every HardSign decision equals that of
//         the exact product X B and S is corrected exactly where a sign flips.
//
// Warp roles (384 threads, one CTA per SM, persistent over a contiguous range of the
// n-major tile sequence): warp 0 TMA producer, warp 1 Stage I MMA issuer (TMEM
// owner), warp 2 C-tile producer, warp 3 Stage II MMA issuer, warps 4..11 epilogue.
// Operand ring: SWIZZLE_128B K-major stages (64-byte SWIZZLE_64B int8 stages when
// Fp % 128 != 0).  Clusters: 2x1 CTAs sharing each B tile by TMA multicast (default),
// single CTAs for one N-tile, virtual 1 x 4 / 1 x 8 / 1 x 16 groups when the live X tiles
// plus B exceed L2, or a cta_group::2 pair (HDC_TC_CLUSTER=2x1p).  Partial scores of
// N-tiles split between clusters are exact int64 sums, added by the last arriver, which
// takes the lowest-index argmax: bit-deterministic and independent of N.
#include <cuda.h>
#include <cuda_bf16.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>

#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"
#include "tc_limbs.cuh"

namespace hdc {
namespace {

using namespace ptx;

constexpr int BM = 128;              // rows per tile (MMA M)
constexpr int STAGES_MAX = 6;
// K bytes per operand stage (one swizzle-atom row).  Fewer, larger stages mean fewer
// producer / MMA hand-offs: int8 at 128 B (2 stages of 78 KB) runs 8% faster than at
// 64 B (4 stages of 39 KB) at cfg2 (tc_kbytes); bf16/tf32 at 64 B was slower than 128 B.
#define HDC_TC_KB8 64                                // int8 mode default (launch picks 64 / 128 by Fp)
#ifndef HDC_TC_NAT16
#define HDC_TC_NAT16 1                               // bf16/tf32: swizzle atoms per stage
#endif
#ifndef HDC_TC_KB16
#define HDC_TC_KB16 128
#endif
#ifndef HDC_TC_EPI_WARPS
#define HDC_TC_EPI_WARPS 8
#endif
constexpr int NUM_EPI = HDC_TC_EPI_WARPS;           // epilogue warps: 4 lane quarters x NUM_CQ
constexpr int THREADS = 32 * (4 + NUM_EPI);         // + producer, MMA, C-producer, spare
constexpr int EPI_WARP0 = 4;
constexpr int NUM_CQ = NUM_EPI / 4;                 // column groups of the tile
constexpr int MAX_LIMBS = 3;
constexpr int CORE_LBO = 128;                        // K-adjacent 8x16B core matrices
constexpr int XCHG_BYTES = 128 * 8;                  // per-row (best value, index) of column group 1
constexpr int KP_MAX_I8 = 32;                        // Stage II N (classes) limits
constexpr int KP_MAX_16 = 64;

// D-tile width by mode and class count: 160 for bf16/tf32 with K <= 32 (an N=160
// MMA costs the same cycles as N=80, tools/mma_microbench.cu), else 80
// (int8: three limb accumulators x 80 columns x 2 buffers fill TMEM; wide: 2 x 3 x 80, one buffer).
// mode 3 = the int8 mode with 160-column tiles made of two 80-column sub-tiles and ONE
// accumulator buffer ("wide", large F only): each A (X limb) stage feeds twice the MMA work,
// so the operand stream per MMA cycle falls from 81 to 56 bytes per SM
__host__ __device__ constexpr int tile_n_for(int mode, int64_t K) {
  return (mode == 2) ? 80 : (mode == 3) ? 160 : (K <= 32 ? 160 : 80);
}

template <int MODE, int BN_, int KW = 0>
struct Cfg {
  static constexpr int BN = BN_;
  static constexpr bool I8 = MODE >= 2;                          // int8x3 limbs (modes 2, 3)
  static constexpr bool WIDE = MODE == 3;
  static constexpr int NSUB = WIDE ? 2 : 1;                      // 80-column sub-tiles of a tile
  static constexpr int SUBN = BN / NSUB;
  static constexpr int NACC = WIDE ? 1 : 2;                      // Stage I accumulator buffers
  static constexpr int NCS = WIDE ? 1 : 2;                       // C slots
  static constexpr int NL = I8 ? 3 : 1;
  static constexpr int ESZ = (MODE == 0) ? 2 : (MODE == 1) ? 4 : 1;
  // K bytes per stage = one swizzle-atom row (HDC_TC_KB8 / HDC_TC_KB16).
  static constexpr int KBYTES = KW ? KW : I8 ? HDC_TC_KB8 : HDC_TC_KB16;
  static constexpr int SWZ = (KBYTES == 64) ? 4 : 2;             // descriptor layout type
  static constexpr int SBO = 8 * KBYTES;                         // 8-row core group
  // bf16/tf32: NAT swizzle atoms (K blocks of KBYTES) per stage, each a [rows][KBYTES] tile
  static constexpr int NAT = I8 ? 1 : HDC_TC_NAT16;
  static constexpr int ATOM_A = BM * KBYTES, ATOM_B = BN * KBYTES;
  static constexpr int A_LIMB_BYTES = NAT * ATOM_A;
  static constexpr int B_LIMB_BYTES = NAT * ATOM_B;
  static constexpr int KA = KBYTES / ESZ;                        // K elements per atom
  static constexpr int KE = NAT * KA;                            // K elements per stage
  static constexpr int KP_MAX = WIDE ? 16 : (I8 || BN > 80) ? KP_MAX_I8 : KP_MAX_16;
  // TMEM columns: NACC Stage I accumulator buffers, the Stage II accumulator (the C parts
  // accumulate into the same Kp columns) and, for bf16/tf32, two H tiles as the Stage II
  // A operand (bf16 pairs, BN/2 columns each).
  static constexpr int ACC_STRIDE = I8 ? 3 * BN : (BN <= 128 ? 128 : BN);
  static constexpr int D2_COL = NACC * ACC_STRIDE;
  static constexpr bool H_TMEM = !I8;
  static constexpr int S_COLS = KP_MAX;
  static constexpr int H_COL = D2_COL + S_COLS;
  // H tile buffers: int8 (H in shared memory) one -- Stage II(t) completes long before the
  // epilogue writes H(t+1) -- which leaves room for the third C part
  static constexpr int NH = I8 ? 1 : 2;
  // C parts of the Stage II operand: bf16 hi + lo (+ a third for the int8 / fp32-semantics
  // modes, hi + mid + lo = C exactly for normal C)
  static constexpr int NCP = I8 ? 3 : 2;
  static_assert(H_COL + (H_TMEM ? NH * BN / 2 : 0) <= 512, "TMEM budget");
  static constexpr int H_BYTES = BM * BN * 2;                    // int8 mode: bf16 H tile in smem
  static constexpr int CORE_SBO = (BN / 8) * 128;                // 8-row groups of core matrices
  static constexpr int EPI_COLS = BN / NUM_CQ;                   // columns per epilogue thread
  static constexpr int CH = (EPI_COLS % 16 == 0) ? 16 : 8;       // columns per TMEM load
  static constexpr int NWB = (EPI_COLS + 31) / 32;               // bit words per thread
  // Stage II operand per D-tile: bf16 parts [NCP][Kp][BN] interleaved; int8 mode appends the
  // tile's coarse int32 column taus (coltau_m).
  static constexpr int C_SLOT = NCP * KP_MAX * BN * 2 + (I8 ? BN * 4 : 0);
  static constexpr int H_REGION = H_TMEM ? 0 : NH * H_BYTES;
  static constexpr int A_STAGE = NL * A_LIMB_BYTES;
  static constexpr int B_STAGE = NL * B_LIMB_BYTES;
  static constexpr int FIXED = H_REGION + NCS * C_SLOT + 512 + 1024 + 16 + XCHG_BYTES;
  static constexpr int STAGES_FIT = (227 * 1024 - FIXED) / (A_STAGE + B_STAGE);
  static constexpr int STAGES_ = STAGES_FIT < STAGES_MAX ? STAGES_FIT : STAGES_MAX;
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = OFF_A + STAGES_ * A_STAGE;
  static constexpr int OFF_H = OFF_B + STAGES_ * B_STAGE;
  static constexpr int OFF_C = OFF_H + H_REGION;
  static constexpr int OFF_X = (OFF_C + NCS * C_SLOT + 15) / 16 * 16;   // argmax exchange [BM] x (value, index)
  static constexpr int OFF_BAR = OFF_X + XCHG_BYTES;
  static constexpr int TOTAL = OFF_BAR + 512;
  static_assert(STAGES_ >= ((KBYTES == 128 && I8) || NAT > 1 ? 2 : 3), "pipeline depth");
  static_assert(OFF_B % 1024 == 0 && OFF_H % 1024 == 0 && OFF_C % 1024 == 0, "alignment");
  static_assert(C_SLOT % 16 == 0, "bulk-copy granule");
  static_assert(TOTAL + 1024 <= 227 * 1024, "shared memory budget");
};

struct TcParams {
  int64_t N, F, Fp, D, Dp, Dq, K, Kp, Np;
  int Tn, Td, G;            // G = clusters of the launch
  int TdG;                  // D-groups: a cluster tile = CLN N-tiles x CLD consecutive D-tiles
  int runit;                // range granularity in cluster tiles: TdG = whole N-tile rows per cluster
  int64_t T;                // cluster tiles (n-major), contiguous ranges per cluster
  const float* X;          // caller's X (fp64 recheck)
  const float* Bt;         // fp32 B^T [Dp][Fp] (fp64 recheck)
  const int64_t* rowtau;   // int8 mode: per-row part of tau (units of 2^14)
  const int64_t* coltau;   // int8 mode: per-column part of tau
  const int32_t* coltau_m; // int8 mode: ceil(coltau / 2^flag_shift), the epilogue's coarse column taus
  int flag_shift;          // int8 mode: the epilogue flags on floor(I / 2^flag_shift) (tc_flag_shift)
  const uint8_t* Cil;      // per D-tile Stage II operand (see Cfg::C_SLOT), c_tile_bytes each
  uint32_t c_tile_bytes;
  long long* S_part;       // [CTAs][nslot][BM][Kp] int64 fixed-point partial scores of split N-tiles
  long long* S_acc;        // [N_p][Kp] int64 sums of N-tiles split over > 8 CTAs (red.add), zero between calls
  double scale, inv_scale; // 2^shift, 2^-shift: the fixed point of the Stage II sums (tc_corr_shift)
  float scale_f;           // 2^shift as a normal float, else 0 (then the fp64 conversion)
  int64_t s_part_cap;      // capacity of S_part in [BM][K] slots
  int nslot;               // slots per CTA: 2 (CLD = 1: first / last N-group of the range),
                           // else one per N-group of the cluster's range
  unsigned* cnt;           // [Tn]
  unsigned long long* recheck_count;
  uint32_t* hout;                   // encode mode (hdc_model_encode): bit-packed H, bit set <=> h = -1;
  int64_t hout_ldw;                 //   row n, column d at word n * ldw + d / 32, bit d % 32; no Stage II
  uint2* flags;                     // int8 mode: (row, d | provisional-negative << 31) to re-evaluate
  unsigned long long* flag_count;   // appended entries (may exceed flag_cap: overflow re-evaluated inline)
  unsigned long long flag_cap;
  float* scores;
  int32_t* labels;
  int debug;               // diagnostics only (HDC_TC_DEBUG): 1 = no Stage I MMA, 2 = no operand TMA,
                           // 4 = per-role wait-cycle counters into dbg[]
  unsigned long long* dbg; // [16] cycle counters (debug & 4)
};

// Diagnostics (HDC_TC_DEBUG ablation / counter flags) exist only in side builds compiled
// with -DHDC_TC_DIAG=1 (tools/tc_timing.py); the product kernel has no debug branches.
#ifndef HDC_TC_DIAG
#define HDC_TC_DIAG 0
#endif
#ifndef HDC_I8_EPI_UNROLL
#define HDC_I8_EPI_UNROLL 1
#endif
constexpr int kI8EpiUnroll = HDC_I8_EPI_UNROLL;
#ifndef HDC_I8_EARLY
#define HDC_I8_EARLY 1
#endif
constexpr bool kI8Early = HDC_I8_EARLY;            // int8 epilogue: release the accumulator after J
#ifdef HDC_TC_DIAG_MASK
// compile-time ablation (no runtime checks): DBG(m) is a constant
#define DBG(mask) ((HDC_TC_DIAG_MASK) & (mask))
#else
#define DBG(mask) (HDC_TC_DIAG ? (p.debug & (mask)) : 0)
#endif

// Watchdog wait (diagnostics, debug & 16384): a wait that has not completed after ~1 s
// records (slot, CTA, warp, parity) in the host-mapped p.dbg buffer and sets an abort
// flag on which every later watchdog wait returns at once, so a protocol deadlock ends
// the kernel (with garbage results) and names the barrier instead of hanging the GPU.
template <class P>
__device__ __noinline__ void watchdog_wait(const P& p, uint64_t* bar, uint32_t par, int slot, long long t0) {
  volatile unsigned long long* d = p.dbg;
  const long long w0 = clock64();
  while (!mbar_test(bar, par)) {
    if (d[0]) return;
    if (clock64() - w0 > 2000000000ll) {
      const unsigned long long i =
          (threadIdx.x & 31) ? ~0ull : atomicAdd((unsigned long long*)p.dbg + 1, 1ull);
      if (i < 64) {
        unsigned long long* r = (unsigned long long*)p.dbg + 8 + 4 * i;
        r[0] = (unsigned long long)slot;
        r[1] = blockIdx.x;
        r[2] = threadIdx.x >> 5;
        r[3] = ((unsigned long long)par << 32) | (unsigned long long)((w0 - t0) >> 10);
      }
      __threadfence_system();
      d[0] = 1;
      return;
    }
  }
}

// Timed barrier wait (diagnostics): accumulates the cycles spent waiting.
#define TWAIT(slot, bar, par)                                        \
  do {                                                               \
    if (DBG(16384)) {                                                \
      watchdog_wait(p, bar, par, slot, t_start);                     \
    } else if (DBG(4)) {                                             \
      const long long _t0 = clock64();                               \
      mbar_wait(bar, par);                                           \
      dbgc[slot] += (unsigned long long)(clock64() - _t0);           \
    } else {                                                         \
      mbar_wait(bar, par);                                           \
    }                                                                \
  } while (0)

// Contiguous ranges of the n-major cluster-tile sequence, in units of U tiles (U = TdG: every
// range is whole N-tile rows, so the groups sweep the D-groups of B in step)
__device__ __forceinline__ int64_t range_begin(int c, int64_t T, int G, int U) {
  return (int64_t)c * (T / U) / G * U;
}
__device__ __forceinline__ int owner_of(int64_t t, int64_t T, int G, int U) {
  int c = (int)((t * G) / T);
  while (c + 1 < G && range_begin(c + 1, T, G, U) <= t) ++c;
  while (c > 0 && range_begin(c, T, G, U) > t) --c;
  return c;
}

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ float recheck_warp(const TcParams& p, int64_t row, int64_t d, int lane) {
  return recheck_dot(p.X + row * p.F, p.Bt + d * p.Fp, p.F, lane);
}

__device__ __forceinline__ bool seg_last(int64_t t, int64_t t1, int Td) {
  return (t + 1 == t1) || ((t + 1) / Td != t / Td);
}

template <int MODE, int BN, int CLN, int CLD, bool ENC, bool HWC, bool PAIR, int KW>
__global__ void __launch_bounds__(THREADS, 1)
fused_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmC, const TcParams p) {
  using CF = Cfg<MODE, BN, KW>;
  // PAIR: the 2 CTAs of a cluster run as one cta_group::2 MMA unit (M = 256: N-tiles
  // 2ng, 2ng+1; each CTA holds its 128 X rows and HALF of the B tile and of the C tile in
  // its own shared memory, so each SM ingests 128 + BN/2 operand rows per k-step instead of
  // 128 + BN).  The leader (rank 0) issues every MMA; the peer's epilogue signals the
  // leader's barriers remotely.
  static_assert(!PAIR || (CLN == 2 && CLD == 1 && HWC && !CF::I8 && !ENC), "pair mode: bf16/tf32 inference, 2x1 cluster");
  constexpr bool I8 = CF::I8;
  constexpr int KIND = I8 ? 2 : MODE;                // tcgen05 kind: 0 f16, 1 tf32, 2 i8
  constexpr int NSUB = CF::NSUB, SUBN = CF::SUBN;
  constexpr int NACC = CF::NACC, NCS = CF::NCS;
  constexpr int NL = CF::NL;
  constexpr int KE = CF::KE;
  constexpr int NH = CF::NH;
  constexpr int EPI_COLS = CF::EPI_COLS;
  constexpr int CH = CF::CH;
  constexpr int NWB = CF::NWB;
  constexpr int CORE_SBO = CF::CORE_SBO;
  constexpr uint32_t IDESC = make_idesc<KIND>(BM, SUBN);
  constexpr uint32_t IDESC_N160 = make_idesc<KIND>(BM, 2 * SUBN);
  constexpr uint32_t IDESC_N240 = make_idesc<KIND>(BM, 3 * SUBN);
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
  uint64_t* tempty = tfull + 2;          // [2] Stage I accumulator drained (read into registers)
  uint64_t* cfull = tempty + 2;          // [2] C tile (+ column taus) landed
  uint64_t* cempty = cfull + 2;          // [2] C tile consumed (Stage II MMA done)
  uint64_t* hfull = cempty + 2;          // [NH] H tile written
  uint64_t* hempty = hfull + 2;          // [NH] H tile consumed
  uint64_t* sfull = hempty + 2;          // [1] Stage II accumulator of a tile complete
  uint64_t* sempty = sfull + 1;          // [1] Stage II accumulator drained (int64 sums)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sempty + 1);
  int* s_flag = reinterpret_cast<int*>(tmem_slot + 1);

  // Cluster of CLN x CLD CTAs: rank (rn, rd) works on N-tile ng CLN + rn and D-tile
  // dg CLD + rd of cluster tile (ng, dg).  The CLD CTAs sharing an N-tile multicast
  // its X tile (each loads 128/CLD rows), the CLN CTAs sharing a D-tile multicast its
  // B tile (BN/CLN rows each): L2 -> SM traffic per tile falls by those factors.
  // HWC = false: a "virtual" cluster -- CLS consecutive CTAs share the tile schedule (the
  // CLD ranks work on the same N-tile at the same time, so its X tile is read from L2 by
  // all of them while few N-tiles are live: the L2 working set when X tiles are large,
  // DESIGN.md §2) but load their own tiles, with no hardware cluster or multicast.
  constexpr int CLS = CLN * CLD;
  constexpr bool MC = HWC && CLS > 1;              // hardware cluster with multicast
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x;                        // global CTA index (partial-score slots)
  const int rank = MC ? (int)cluster_ctarank() : (CLS > 1 ? c % CLS : 0);
  const int rn = rank / CLD, rd = rank % CLD;
  const int cl = c / CLS;                          // cluster index
  const uint16_t a_mask = (uint16_t)(((1u << CLD) - 1u) << (rn * CLD));   // same N-tile
  uint16_t b_mask = 0;                                                    // same D-tile
#pragma unroll
  for (int i = 0; i < CLN; ++i) b_mask |= (uint16_t)(1u << (i * CLD + rd));
  const int64_t t0 = range_begin(cl, p.T, p.G, p.runit), t1 = range_begin(cl + 1, p.T, p.G, p.runit);
  // K stages; the int8 mode's 128-byte stages may overhang Fp (a multiple of 64) by 64
  // elements: TMA zero-fills past the tensor's extent and the MMA skips those k-steps
  const int KB = (int)((p.Fp + KE - 1) / KE);
  const int last_ks = (int)(((p.Fp - (int64_t)(KB - 1) * KE) * CF::ESZ + 31) / 32);
  const int last_at = (int)((p.Fp - (int64_t)(KB - 1) * KE + CF::KA - 1) / CF::KA);   // atoms used
  const bool leader = !PAIR || rank == 0;
  // pair mode: barriers the leader's MMA warps wait on are the leader's
  auto arrive_lead = [&](uint64_t* bar) {
    if constexpr (PAIR) mbar_arrive_cluster(mapa_u32(bar, 0));
    else mbar_arrive(bar);
  };
  unsigned long long dbgc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) dbgc[i] = 0;
  const long long t_start = clock64();
  const uint32_t c_tile_bytes = p.c_tile_bytes;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, (MC && !PAIR) ? CLN + CLD - 1 : 1);   // MMA commits of every CTA this one multicasts to
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull + b, 1);
      mbar_init(tempty + b, PAIR ? 2 * NUM_EPI : NUM_EPI);   // pair: both CTAs' epilogues
      mbar_init(cfull + b, 1);
      mbar_init(cempty + b, (I8 && ENC) ? NUM_EPI : 1);   // encode: epilogue frees taus
      mbar_init(hfull + b, PAIR ? 2 * NUM_EPI : NUM_EPI);
      mbar_init(hempty + b, 1);
    }
    mbar_init(sfull, 1);
    mbar_init(sempty, PAIR ? 2 * NUM_EPI : NUM_EPI);   // every epilogue warp (of each CTA) drains its classes
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1) {
    if constexpr (PAIR) tmem_alloc_pair<512>(tmem_slot);
    else tmem_alloc<512>(tmem_slot);
  }
  tc_fence_before();
  if constexpr (MC) cluster_sync_all();   // peers' barriers initialised before any multicast
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================================================== TMA producer (operands)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      constexpr int AR = MC ? BM / CLD : BM, BR = MC ? SUBN / CLN : SUBN;   // rows this CTA loads
      const int ra = MC ? rd : 0, rb = MC ? rn : 0;       // its slice of the A / B tile
      for (int64_t t = t0; t < t1; ++t) {
        const int ni = (int)(t / p.TdG) * CLN + rn, di = (int)(t % p.TdG) * CLD + rd;
        for (int kb = 0; kb < KB; ++kb) {
          if (DBG(4096)) mbar_wait_spin(empty + stage, phase ^ 1);
          else TWAIT(0, empty + stage, phase ^ 1);
          if ((DBG(1024)) && c == 0) {
            const int64_t si = (t - t0) * KB + kb;
            if (si < 256) p.dbg[16 + 256 + si] = (unsigned long long)clock64();
          }
          if (DBG(2)) {
            mbar_arrive(full + stage);
          } else {
            if constexpr (PAIR) {
              // both CTAs' loads complete on the leader's barrier (the leader's MMA waits on it)
              const uint32_t fbar = mapa_u32(full + stage, 0);
              // (the leader's own barrier: a CTA-scope arrive, no cluster-scope release fence)
              if (leader) mbar_arrive_expect_tx(full + stage, 2 * CF::NAT * (CF::ATOM_A + (BN / 2) * KBYTES));
#pragma unroll
              for (int a = 0; a < CF::NAT; ++a) {
                tma_load_2d_pair(sA + stage * CF::A_STAGE + a * CF::ATOM_A, &tmA, fbar, kb * KE + a * CF::KA,
                                 (int)((int64_t)ni * BM));
                tma_load_2d_pair(sB + stage * CF::B_STAGE + a * CF::ATOM_B, &tmB, fbar, kb * KE + a * CF::KA,
                                 (int)((int64_t)di * BN + rank * (BN / 2)));
              }
            } else {
            mbar_arrive_expect_tx(full + stage, STAGE_TX);   // whole tiles: own + peers' slices
#pragma unroll
            for (int l = 0; l < NL; ++l)
#pragma unroll
              for (int a = 0; a < CF::NAT; ++a) {
              uint8_t* da = sA + stage * CF::A_STAGE + l * A_LIMB_BYTES + a * CF::ATOM_A + ra * AR * KBYTES;
              const int ya = (int)(l * p.Np + (int64_t)ni * BM + ra * AR);
              const int xk = kb * KE + a * CF::KA;
              if constexpr (MC && CLD > 1) tma_load_2d_mc(da, &tmA, full + stage, xk, ya, a_mask);
              else tma_load_2d(da, &tmA, full + stage, xk, ya);
              // B stage layout: [b0; b1; b2] (80-column mode), or the wide mode's row blocks
              // [b0s0 b0s1 b2s0 b2s1 b1s0 b1s1] (tc_mma_i8w5_elect)
#pragma unroll
              for (int h = 0; h < NSUB; ++h) {
                const int blk = CF::WIDE ? (l == 0 ? 0 : l == 2 ? 2 : 4) + h : l;
                uint8_t* db = sB + stage * CF::B_STAGE + blk * (CF::B_LIMB_BYTES / NSUB) +
                              a * CF::ATOM_B + rb * BR * KBYTES;
                const int yb = (int)(l * p.Dq + (int64_t)di * BN + h * SUBN + rb * BR);
                if constexpr (MC && CLN > 1) tma_load_2d_mc(db, &tmB, full + stage, xk, yb, b_mask);
                else tma_load_2d(db, &tmB, full + stage, xk, yb);
              }
            }
            }
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1 && leader) {
    // ===================================================== Stage I MMA issuer (elected lane)
    constexpr uint32_t IDESC_P = make_idesc<KIND>(2 * BM, BN);   // pair: M = 256
    int stage = 0, buf = 0;
    uint32_t phase = 0, bphase = 0;
    const uint64_t a_desc0 = sdesc(smem_u32(sA));
    const uint64_t b_desc0 = sdesc(smem_u32(sB));
    for (int64_t t = t0; t < t1; ++t) {
      if (!(DBG(8192))) TWAIT(1, tempty + buf, bphase ^ 1);   // 8192: diagnostics, no epilogue
      tc_fence_after();
      const uint32_t acc0 = tmem_base + buf * CF::ACC_STRIDE;
      for (int kb = 0; kb < KB; ++kb) {
        if (DBG(4096)) mbar_wait_spin(full + stage, phase);   // diagnostics: spin
        else TWAIT(2, full + stage, phase);
        if ((DBG(1024)) && c == 0 && lane == 0) {
          const int64_t si = (t - t0) * KB + kb;
          if (si < 256) p.dbg[16 + si] = (unsigned long long)clock64();
        }
        tc_fence_after();
        // descriptors = base descriptor + (byte offset >> 4) in the start-address field
        const uint64_t a_d = a_desc0 + (uint64_t)((stage * CF::A_STAGE) >> 4);
        const uint64_t b_d = b_desc0 + (uint64_t)((stage * CF::B_STAGE) >> 4);
        if (!(DBG(1))) {
          const uint32_t acc = (kb == 0) ? 0u : 1u;
          if constexpr (I8) {
            // The three B limb tiles are contiguous rows [b0; b1; b2] (240 x 64 B) and
            // the accumulators contiguous columns [A0 | A1 | A2], so one MMA per A limb:
            //   [A0|A1|A2] (+)= x0 [b0;b1;b2]^T,  [A1|A2] += x1 [b0;b1]^T,  A2 += x2 b0^T
            // (each A tile is read from shared memory once per k-step, not 3 times).
            // Wide mode: the same for each 80-column sub-tile h, accumulators at 240 h.
            // Wide mode: the five MMAs of tc_mma_i8w5_elect over both sub-tiles.
            const int nks = (kb == KB - 1) ? last_ks : KBYTES / 32;
#pragma unroll
            for (int ks = 0; ks < KBYTES / 32; ++ks)
              if (ks < nks) {
                if constexpr (CF::WIDE)
                  tc_mma_i8w5_elect(acc0, a_d + 2 * ks, a_d + ((A_LIMB_BYTES + ks * 32) >> 4),
                                    a_d + ((2 * A_LIMB_BYTES + ks * 32) >> 4), b_d + 2 * ks,
                                    b_d + ((3 * SUBN * KBYTES) >> 4) + 2 * ks,
                                    b_d + ((4 * SUBN * KBYTES) >> 4) + 2 * ks, IDESC_N240, IDESC_N160,
                                    ks == 0 ? acc : 1u);
                else
                  tc_mma_i8x3_elect(acc0, a_d + 2 * ks, a_d + ((A_LIMB_BYTES + ks * 32) >> 4),
                                    a_d + ((2 * A_LIMB_BYTES + ks * 32) >> 4), b_d + 2 * ks, IDESC_N240,
                                    IDESC_N160, IDESC, SUBN, ks == 0 ? acc : 1u);
              }
          } else {
            const int nat = (kb == KB - 1) ? last_at : CF::NAT;
#pragma unroll
            for (int at = 0; at < CF::NAT; ++at) {
              if (at >= nat) continue;
              const uint64_t aa = a_d + (uint64_t)((at * CF::ATOM_A) >> 4);
              const uint64_t bb = b_d + (uint64_t)((at * CF::ATOM_B) >> 4);
              const uint32_t ac = at == 0 ? acc : 1u;
              if constexpr (PAIR)
                tc_mma4_pair_elect<MODE>(acc0, aa, bb, aa + 2, bb + 2, aa + 4, bb + 4, aa + 6, bb + 6, IDESC_P, ac);
              else if constexpr (KBYTES == 128) {
                tc_mma4_elect<MODE>(acc0, aa, bb, aa + 2, bb + 2, aa + 4, bb + 4, aa + 6, bb + 6, IDESC, ac);
                if (DBG(32768))   // diagnostics: twice the MMA work per stage (wrong results)
                  tc_mma4_elect<MODE>(acc0, aa, bb, aa + 2, bb + 2, aa + 4, bb + 4, aa + 6, bb + 6, IDESC, 1u);
              }
              else
                tc_mma2_elect<MODE>(acc0, aa, bb, aa + 2, bb + 2, IDESC, ac);
            }
          }
        }
        if ((DBG(2049)) == 2049) {     // diagnostics (no MMAs): plain arrive instead of commit
          __syncwarp();
          if (lane == 0) mbar_arrive(empty + stage);
        } else if constexpr (PAIR) tc_commit_pair_mc_elect(empty + stage, (uint16_t)3);
        else if constexpr (MC) tc_commit_mc_elect(empty + stage, (uint16_t)(a_mask | b_mask));
        else tc_commit_elect(empty + stage);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if constexpr (PAIR) tc_commit_pair_mc_elect(tfull + buf, (uint16_t)3);
      else tc_commit_elect(tfull + buf);
      if (++buf == NACC) {
        buf = 0;
        bphase ^= 1;
      }
    }
  } else if (warp == 2) {
    if ((!ENC || I8) && !(DBG(8192))) {   // encode mode: only the int8 column taus
    // ===================================================== C-tile producer (Stage II B operand)
    // A separate warp, so the operand stream never waits for a C slot.
    if (lane == 0) {
      int cs = 0;
      uint32_t cphase = 0;
      for (int64_t t = t0; t < t1; ++t) {
        const int di = (int)(t % p.TdG) * CLD + rd;
        TWAIT(14, cempty + cs, cphase ^ 1);
        if constexpr (PAIR) {
          // this CTA's half of the class rows of each C part ([part][Kp/2][BN]), both halves
          // completing on the leader's barrier; rows of 128 B in the tmC view of Cil
          const uint32_t cbar = mapa_u32(cfull + cs, 0);
          const int half = (int)(p.Kp * BN);            // bytes of Kp/2 rows x BN bf16
          if (leader) mbar_arrive_expect_tx(cfull + cs, 2 * 2 * half);
#pragma unroll
          for (int part = 0; part < 2; ++part)
            tma_load_2d_pair(sC + cs * CF::C_SLOT + part * half, &tmC, cbar, 0,
                             (int)(((int64_t)di * c_tile_bytes + part * 2 * half + rank * half) / 128));
          cs ^= 1;
          if (cs == 0) cphase ^= 1;
          continue;
        }
        mbar_arrive_expect_tx(cfull + cs, (ENC ? 0u : c_tile_bytes) + (I8 ? BN * 4 : 0));
        if (!ENC)
          bulk_load(sC + cs * CF::C_SLOT, p.Cil + (int64_t)di * c_tile_bytes, c_tile_bytes, cfull + cs);
        if constexpr (I8)
          bulk_load(sC + cs * CF::C_SLOT + c_tile_bytes, p.coltau_m + (int64_t)di * BN, BN * 4,
                    cfull + cs);
        if (++cs == NCS) {
          cs = 0;
          cphase ^= 1;
        }
      }
    }
    }
  } else if (warp == 3 && leader) {
    if (!ENC && !(DBG(8192))) {
    // ===================================================== Stage II MMA issuer (elected lane)
    // A warp of its own: S(t) = H(t) [Chi(t) + Clo(t)]^T goes out the moment H(t) is written,
    // never waiting behind (or holding up) the Stage I issue loop.  Each tile's S(t) starts
    // from zero; the epilogue drains it into exact int64 fixed-point sums (sempty) before
    // the next tile's Stage II overwrites it, so scores do not depend on how the D-tiles of
    // a row are split between CTAs (hence not on N or the cluster shape).
    int hb = 0, cs = 0;
    uint32_t hphase = 0, cphase = 0, sphase = 0;
    const uint32_t IDESC2 = make_idesc<0>(PAIR ? 2 * BM : BM, (int)p.Kp);
    const uint32_t d2 = tmem_base + CF::D2_COL;
    const uint32_t part_bytes = PAIR ? (uint32_t)(p.Kp * BN) : (uint32_t)(p.Kp * BN * 2);   // pair: half the classes
    for (int64_t t = t0; t < t1; ++t) {
      TWAIT(3, hfull + hb, hphase);
      TWAIT(4, cfull + cs, cphase);
      TWAIT(5, sempty, sphase ^ 1);                 // S(t - 1) drained
      sphase ^= 1;
      tc_fence_after();
      const uint32_t c_base = smem_u32(sC + cs * CF::C_SLOT);
#pragma unroll
      for (int s = 0; s < BN / 16; ++s) {
        const uint32_t acc = (s == 0) ? 0u : 1u;
#pragma unroll
        for (int part = 0; part < (PAIR ? 2 : CF::NCP); ++part) {   // C = hi + lo (+ mid), one accumulator
          const uint64_t bd = smem_desc_interleaved(
              c_base + part * part_bytes + s * 2 * CORE_LBO, CORE_LBO, CORE_SBO);
          if (DBG(8)) continue;
          if constexpr (PAIR) {
            tc_mma_ts_pair_elect(d2, tmem_base + CF::H_COL + hb * (BN / 2) + s * 8, bd, IDESC2,
                                 part == 0 ? acc : 1u);
          } else if constexpr (CF::H_TMEM) {
            // A = H from TMEM (16 bf16 = 8 columns per k-step)
            tc_mma_ts_elect(d2, tmem_base + CF::H_COL + hb * (BN / 2) + s * 8, bd, IDESC2,
                            part == 0 ? acc : 1u);
          } else {
            const uint32_t h_base = smem_u32(sH + hb * CF::H_BYTES);
            const uint64_t ad = smem_desc_interleaved(h_base + s * 2 * CORE_LBO, CORE_LBO, CORE_SBO);
            tc_mma_elect<0>(d2, ad, bd, IDESC2, part == 0 ? acc : 1u);
          }
        }
      }
      if constexpr (PAIR) {
        tc_commit_pair_mc_elect(hempty + hb, (uint16_t)3);
        tc_commit_pair_mc_elect(cempty + cs, (uint16_t)3);
        tc_commit_pair_mc_elect(sfull, (uint16_t)3);
      } else {
        tc_commit_elect(hempty + hb);
        tc_commit_elect(cempty + cs);
        tc_commit_elect(sfull);
      }
      if (++hb == NH) {
        hb = 0;
        hphase ^= 1;
      }
      if (++cs == NCS) {
        cs = 0;
        cphase ^= 1;
      }
    }
    }
  } else if (warp >= EPI_WARP0 && !(DBG(8192))) {
    // ===================================================== epilogue
    const int ew = warp - EPI_WARP0;
    const int q = warp & 3;                 // TMEM lane quarter (hardware: warp id % 4)
    const int cq = ew >> 2;                 // column group of the tile
    const int m = q * 32 + lane;            // row within the N-tile
    const int K = (int)p.K;
    int buf = 0, hb = 0, cs = 0;
    uint32_t bphase = 0, hphase = 0, sphase = 0, cphase = 0;
    unsigned long long nrecheck = 0;
    const int first_ng = (int)(t0 / p.TdG);
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    // exact per-row sums of this thread's classes (column group cq: classes cq kq .. + kq - 1)
    // in int64 fixed point (2^-shift units): every tile's S(t) is added after it is complete
    static_assert(NUM_CQ <= 2, "argmax exchange of two column groups");
    constexpr int KQ_MAX = CF::KP_MAX / NUM_CQ;
    const int kq = (int)p.Kp / NUM_CQ;               // a multiple of 8
    long long sacc[KQ_MAX];
#pragma unroll
    for (int u = 0; u < KQ_MAX; ++u) sacc[u] = 0;
    auto drain_s = [&]() {
      TWAIT(8, sfull, sphase);
      sphase ^= 1;
      tc_fence_after();
      const uint32_t sb = tmem_base + lane_off + CF::D2_COL + cq * kq;
#pragma unroll
      for (int c0 = 0; c0 < KQ_MAX; c0 += 8) {
        if (c0 < kq) {
          uint32_t r[8];
          tmem_ld8(sb + c0, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float v = __uint_as_float(r[j]);
            // v 2^shift is exact (a power-of-two scaling) in fp32 when 2^shift is a normal
            // float, so both conversions round the same exact value
#ifdef HDC_S2_NOCVT
            sacc[c0 + j] += (long long)__float_as_int(v);   // diagnostics: cost of the conversion (wrong sums)
#else
            sacc[c0 + j] += p.scale_f > 0.f ? __float2ll_rn(v * p.scale_f) : llrint((double)v * p.scale);
#endif
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_lead(sempty);
    };
    // row argmax from the two column groups' (best value, lowest index) -- group 0 holds the
    // lower classes, so it wins ties; row < 0: padding row, no label
    float* xv = reinterpret_cast<float*>(smem + CF::OFF_X);
    int* xi = reinterpret_cast<int*>(smem + CF::OFF_X + 4 * BM);
    auto epi_argmax = [&](int best, float bv, int64_t row) {
      if constexpr (NUM_CQ == 2) {
        named_bar(1, NUM_EPI * 32);
        if (cq == 1) {
          xv[m] = bv;
          xi[m] = best;
        }
        named_bar(1, NUM_EPI * 32);
        if (cq == 0 && xi[m] >= 0 && (best < 0 || xv[m] > bv)) best = xi[m];
      }
      if (cq == 0 && row >= 0 && p.labels) p.labels[row] = best;
    };
    int64_t next_drain = t0;                          // next tile whose S(t) is to be added
    const int fsl = 14 - p.flag_shift, fs1 = p.flag_shift - 7, fs2 = p.flag_shift;   // int8 flag test
    for (int64_t t = t0; t < t1; ++t) {
      const int ng = (int)(t / p.TdG);
      const int ni = ng * CLN + rn, di = (int)(t % p.TdG) * CLD + rd;
      const int64_t row = (int64_t)ni * BM + m;
      const bool row_ok = row < p.N;
      // int8 mode: row part of the coarse tau, ceil(rowtau / 2^flag_shift); padding rows never flag
      int32_t mrow = -(1 << 28);
      if constexpr (I8)
        if (row_ok) mrow = (int32_t)((__ldg(p.rowtau + row) + (int64_t(1) << p.flag_shift) - 1) >> p.flag_shift);
      if (DBG(256)) {                  // diagnostics: sleep-polling instead of try_wait
        while (!mbar_test(tfull + buf, bphase)) __nanosleep(500);
      }
      TWAIT(6, tfull + buf, bphase);
      // wide mode (one accumulator buffer): the S drain and the wait for the column taus come
      // after the accumulator is handed back, off the Stage I issuer's critical path
      constexpr bool kLate = I8 && kI8Early && CF::WIDE;
      // Stage II of two tiles back: issued a whole tile ago, so complete; draining it lets the
      // Stage II MMAs of the previous tile go out (one TMEM accumulator, drained in order)
      if (!ENC && !kLate)
        while (next_drain <= t - 2) {
          drain_s();
          ++next_drain;
        }
      const int32_t* scm = nullptr;         // coarse column taus of this tile (int8 mode), in smem
      static_assert((EPI_COLS * 4) % 16 == 0, "16-byte column-tau loads");
      if constexpr (I8 && !kLate) {
        TWAIT(15, cfull + cs, cphase);
        scm = reinterpret_cast<const int32_t*>(sC + cs * CF::C_SLOT + c_tile_bytes) + cq * EPI_COLS;
      }
      tc_fence_after();
      // ---- phase 1: accumulator -> HardSign bits (bit set -> h = -1) and recheck flags
      uint32_t hbits[NWB], flags[NWB];
#pragma unroll
      for (int w = 0; w < NWB; ++w) hbits[w] = flags[w] = 0u;
      // int8: limb accumulators A0 | A1 | A2 of SUBN columns each at tbase + {0, 1, 2} SUBN;
      // wide mode: column group cq is sub-tile cq, its accumulators in the blocks
      // [A0s0 A0s1 A2s0 A2s1 A1s0 A1s1] (tc_mma_i8w5_elect): A0 at cq, A1 at 4 + cq, A2 at 2 + cq
      const uint32_t tbase = tmem_base + lane_off + buf * CF::ACC_STRIDE + (CF::WIDE ? cq * SUBN : cq * EPI_COLS);
      constexpr uint32_t OFF_A1 = CF::WIDE ? 4 * SUBN : SUBN, OFF_A2 = CF::WIDE ? 2 * SUBN : 2 * SUBN;
      bool released = false;                // accumulator buffer already handed back
      if constexpr (I8 && kI8Early && CF::WIDE) {
        // Two steps: (1) the accumulator -> J (four integer ops per element, J held in
        // registers), then the buffer goes back to the Stage I issuer at once (the wide mode
        // has one buffer, so this read is the part of the epilogue the MMAs wait for);
        // (2) signs and flags from J (the test of the loop below, same J).  Wide mode only:
        // with two buffers the read is hidden anyway, and the unrolled form cost cfg2 8%.
        int32_t Jv[EPI_COLS];
        constexpr int ECH = 8;              // columns per load group (registers: J + 3 x ECH)
#pragma unroll
        for (int ch = 0; ch < EPI_COLS / ECH; ++ch) {
          const int cl = ch * ECH;
          uint32_t r0[ECH], r1[ECH], r2[ECH];
          tmem_ld8(tbase + cl, r0);
          tmem_ld8(tbase + OFF_A1 + cl, r1);
          tmem_ld8(tbase + OFF_A2 + cl, r2);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < ECH; ++j)
            Jv[cl + j] = ((int32_t)r0[j] << fsl) + ((int32_t)r1[j] >> fs1) + ((int32_t)r2[j] >> fs2);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_lead(tempty + buf);
        released = true;
        if (!ENC)
          while (next_drain <= t - 2) {
            drain_s();
            ++next_drain;
          }
        TWAIT(15, cfull + cs, cphase);
        scm = reinterpret_cast<const int32_t*>(sC + cs * CF::C_SLOT + c_tile_bytes) + cq * EPI_COLS;
#pragma unroll
        for (int v = 0; v < EPI_COLS / 4; ++v) {
          const int4 q4 = reinterpret_cast<const int4*>(scm)[v];
          const int mq[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int b = 4 * v + e;
            const int32_t J = Jv[b];
            const int32_t sg = J >> 31;
            hbits[b >> 5] |= (uint32_t)sg & (1u << (b & 31));
            if ((J ^ sg) - mq[e] <= mrow) flags[b >> 5] |= 1u << (b & 31);
          }
        }
      } else if constexpr (I8) {
        // 64-bit masks (two for EPI_COLS = 80): register-resident under any unrolling
        static_assert(EPI_COLS <= 128, "int8 column group");
        uint64_t hb64 = 0, fl64 = 0, hb64x = 0, fl64x = 0;
#pragma unroll kI8EpiUnroll
        for (int ch = 0; ch < ((DBG(16)) ? 0 : EPI_COLS / CH); ++ch) {
          const int cl = ch * CH;             // column within this thread's group
          uint32_t r0[CH], r1[CH], r2[CH];
          if constexpr (CH == 16) {
            tmem_ld16(tbase + cl, r0);
            tmem_ld16(tbase + OFF_A1 + cl, r1);
            tmem_ld16(tbase + OFF_A2 + cl, r2);
          } else {
            tmem_ld8(tbase + cl, r0);
            tmem_ld8(tbase + OFF_A1 + cl, r1);
            tmem_ld8(tbase + OFF_A2 + cl, r2);
          }
          tmem_ld_wait();
          uint32_t hc = 0, fc = 0;            // this chunk's bits
          int32_t mc[CH];
#pragma unroll
          for (int v = 0; v < CH / 4; ++v) {
            const int4 q4 = reinterpret_cast<const int4*>(scm + cl)[v];
            mc[4 * v] = q4.x; mc[4 * v + 1] = q4.y; mc[4 * v + 2] = q4.z; mc[4 * v + 3] = q4.w;
          }
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            // I = r0 2^14 + r1 2^7 + r2 (exact, 64-bit) is only needed through
            // J = r0 2^(14-s) + floor(r1 / 2^(s-7)) + floor(r2 / 2^s), 7 <= s <= 14
            // (tc_flag_shift), which is floor(I / 2^s) or one less, |J| < 2^31.  With
            // J' = (J >= 0 ? J : -J - 1): |I| <= tau implies J' <= mrow + mcol (the ceilings
            // of tau's parts / 2^s), so every element of |I| <= tau is flagged;
            // an unflagged element has J' > mrow + mcol >= 2, where sign(J) = sign(I).
            const int32_t J = ((int32_t)r0[j] << fsl) + ((int32_t)r1[j] >> fs1) + ((int32_t)r2[j] >> fs2);
            const int32_t sg = J >> 31;
            hc |= (uint32_t)sg & (1u << j);
            if ((J ^ sg) - mc[j] <= mrow) fc |= 1u << j;   // past D: mcol = -2^28, never
          }
          if (EPI_COLS <= 64 || cl < 64) {
            hb64 |= (uint64_t)hc << cl;
            fl64 |= (uint64_t)fc << cl;
          } else {
            hb64x |= (uint64_t)hc << (cl - 64);
            fl64x |= (uint64_t)fc << (cl - 64);
          }
        }
        hbits[0] = (uint32_t)hb64;
        flags[0] = (uint32_t)fl64;
        if constexpr (NWB > 1) {
          hbits[1] = (uint32_t)(hb64 >> 32);
          flags[1] = (uint32_t)(fl64 >> 32);
        }
        if constexpr (NWB > 2) {
          hbits[2] = (uint32_t)hb64x;
          flags[2] = (uint32_t)fl64x;
        }
      } else {
#pragma unroll
        for (int ch = 0; ch < ((DBG(16)) ? 0 : EPI_COLS / CH); ++ch) {
          const int cl = ch * CH;             // column within this thread's group
          uint32_t r0[CH];
          if constexpr (CH == 16) tmem_ld16(tbase + cl, r0);
          else tmem_ld8(tbase + cl, r0);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            const int b = cl + j;
            if (!(__uint_as_float(r0[j]) >= 0.f)) hbits[b >> 5] |= 1u << (b & 31);   // HardSign
          }
        }
      }
      if (!released) {
        tc_fence_before();
        __syncwarp();
      }
      if (lane == 0) {
        if (!released) arrive_lead(tempty + buf);   // accumulator free for tile t + NACC
        if (I8 && ENC) mbar_arrive(cempty + cs);   // encode mode: taus read
      }
      // H buffer hb free (Stage II of tile t - 2 done)
      if constexpr (!ENC) {
        TWAIT(7, hempty + hb, hphase ^ 1);
        tc_fence_after();
      }
      // ---- phase 2 (int8 mode): flagged signs are appended to a global list with the
      // provisional sign used in H; hdc_recheck_kernel re-evaluates them in float64 after
      // this kernel and corrects S exactly where a sign flips (Stage II is linear in H).
      // Only a list overflow (e.g. many all-zero rows) falls back to re-evaluating here, and
      // small batches (no list: flag_cap == 0), whose ~1 flag per CTA costs less than the two
      // extra launches.
      if constexpr (I8) {
#pragma unroll
        for (int w = 0; w < NWB; ++w) {
          uint32_t fw = (DBG(512)) ? 0u : flags[w];   // 512: diagnostics, no rechecks
          uint32_t spill = 0u;
          while (fw) {
            const int bit = __ffs(fw) - 1;
            fw &= fw - 1;
            const int col = cq * EPI_COLS + w * 32 + bit;
            // flag_cap == 0: small batches re-evaluate every flag here (no list, no
            // recheck / finalize launches)
            const unsigned long long slot = p.flag_cap ? atomicAdd(p.flag_count, 1ull) : ~0ull;
            if (slot < p.flag_cap) {
              const uint32_t neg = (hbits[w] >> bit) & 1u;
              p.flags[slot] = make_uint2((uint32_t)row, (uint32_t)((int64_t)di * BN + col) | (neg << 31));
            } else {
              spill |= 1u << bit;
            }
          }
          unsigned lanes = __ballot_sync(0xffffffffu, spill != 0u);
          while (lanes) {
            const int src = __ffs(lanes) - 1;
            const int bit = __shfl_sync(0xffffffffu, __ffs(spill) - 1, src);
            const int col = cq * EPI_COLS + w * 32 + bit;
            const float hv = recheck_warp(p, (int64_t)ni * BM + q * 32 + src, (int64_t)di * BN + col, lane);
            if (lane == src) {
              hbits[w] = hv < 0.f ? (hbits[w] | (1u << bit)) : (hbits[w] & ~(1u << bit));
              spill &= spill - 1;
            }
            ++nrecheck;
            lanes = __ballot_sync(0xffffffffu, spill != 0u);
          }
        }
      }
      // ---- phase 3: H (exact bf16 +-1: 0x3F80 / 0xBF80) for the Stage II MMA
      if constexpr (ENC) {
        // encode mode: OR this thread's sign bits into the packed rows (column groups of
        // neighbouring threads / tiles share words; OR of disjoint bits is order-free)
        if (row_ok) {
          uint32_t* hr = p.hout + row * p.hout_ldw;
          const int64_t g0 = (int64_t)di * BN + cq * EPI_COLS;
#pragma unroll
          for (int w = 0; w < NWB; ++w) {
            const int nb = (EPI_COLS - 32 * w) < 32 ? (EPI_COLS - 32 * w) : 32;
            const uint32_t bits = hbits[w] & (nb == 32 ? 0xFFFFFFFFu : ((1u << nb) - 1u));
            if (!bits) continue;
            const int64_t gb = g0 + 32 * w, wi = gb >> 5;
            const int sh = (int)(gb & 31);
            if (wi < p.hout_ldw) atomicOr(hr + wi, bits << sh);
            if (sh && wi + 1 < p.hout_ldw && (bits >> (32 - sh))) atomicOr(hr + wi + 1, bits >> (32 - sh));
          }
        }
      } else if (DBG(128)) {
        // diagnostics: no H write
      } else if constexpr (CF::H_TMEM) {
        // packed bf16 pairs into TMEM columns H_COL + col / 2 of this thread's lane
        const uint32_t hbase = tmem_base + lane_off + CF::H_COL + hb * (BN / 2) + cq * (EPI_COLS / 2);
#pragma unroll
        for (int g = 0; g < EPI_COLS / 16; ++g) {
          uint32_t wv[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int b0 = g * 16 + 2 * j, b1 = b0 + 1;
            const uint32_t lo = ((hbits[b0 >> 5] >> (b0 & 31)) & 1u) ? 0xBF80u : 0x3F80u;
            const uint32_t hi = ((hbits[b1 >> 5] >> (b1 & 31)) & 1u) ? 0xBF80u : 0x3F80u;
            wv[j] = lo | (hi << 16);
          }
          tmem_st8(hbase + g * 8, wv);
        }
        if constexpr (EPI_COLS % 16 != 0) {
          // 8-column remainder (EPI_COLS = 40): four packed words
          uint32_t wv[8];
          const int g = EPI_COLS / 16;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int b0 = g * 16 + 2 * j, b1 = b0 + 1;
            const uint32_t lo = ((hbits[b0 >> 5] >> (b0 & 31)) & 1u) ? 0xBF80u : 0x3F80u;
            const uint32_t hi = ((hbits[b1 >> 5] >> (b1 & 31)) & 1u) ? 0xBF80u : 0x3F80u;
            wv[j] = lo | (hi << 16);
          }
          tmem_st4(hbase + g * 8, wv);
        }
        tmem_st_wait();
      } else {
        uint8_t* hrow = sH + hb * CF::H_BYTES + (m >> 3) * CORE_SBO + (m & 7) * 16;
#pragma unroll
        for (int g = 0; g < EPI_COLS / 8; ++g) {
          const int col0 = cq * EPI_COLS + g * 8;   // 8 columns = one 16-byte core-matrix row
          uint32_t wv[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int b0 = g * 8 + 2 * j, b1 = b0 + 1;
            const uint32_t lo = ((hbits[b0 >> 5] >> (b0 & 31)) & 1u) ? 0xBF80u : 0x3F80u;
            const uint32_t hi = ((hbits[b1 >> 5] >> (b1 & 31)) & 1u) ? 0xBF80u : 0x3F80u;
            wv[j] = lo | (hi << 16);
          }
          *reinterpret_cast<uint4*>(hrow + (col0 >> 3) * CORE_LBO) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        }
        fence_proxy_async_smem();           // H writes -> visible to the tensor core
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0 && !ENC) arrive_lead(hfull + hb);
      if (++buf == NACC) {
        buf = 0;
        bphase ^= 1;
      }
      if (++hb == NH) {
        hb = 0;
        hphase ^= 1;
      }
      if (++cs == NCS) {
        cs = 0;
        cphase ^= 1;
      }

      // ---- end of this CTA's run of D-tiles for N-tile ni: the last two tiles' S as well
      if (ENC || !seg_last(t, t1, p.TdG)) continue;
      while (next_drain <= t) {
        drain_s();
        ++next_drain;
      }
      // ---- end of this CTA's run of D-tiles for N-tile ni: sacc = this CTA's exact sums for
      // the row's classes of column group cq.  The N-tile's D-groups are split over clusters
      // c_first..c_last, each over its CLD ranks; the partial sums are integers, so their
      // total (and every score) is independent of the split.
      const int c_first = owner_of((int64_t)ng * p.TdG, p.T, p.G, p.runit);
      const int c_last = owner_of((int64_t)(ng + 1) * p.TdG - 1, p.T, p.G, p.runit);
      const bool sole = (c_first == c_last) && CLD == 1;
      const int kq0 = cq * kq;                // first class of this thread's group
      if (sole) {
        float bv = 0.f;
        int best = -1;
#pragma unroll
        for (int u = 0; u < KQ_MAX; ++u) {
          const int k = kq0 + u;
          if (u < kq && k < K) {
            const float v = (float)((double)sacc[u] * p.inv_scale);
            if (row_ok && p.scores) p.scores[row * p.K + k] = v;
            if (best < 0 || v > bv) {
              bv = v;
              best = k;
            }
          }
          sacc[u] = 0;
        }
        epi_argmax(best, bv, row_ok ? row : -1);
        continue;
      }
      const int myslot = (CLD == 1) ? ((ng == first_ng) ? 0 : 1) : (ng - first_ng);
      const int P = (c_last - c_first + 1) * CLD;     // partials per row of this N-tile
      // many partials (small N: the N-tile's D-range spread over many clusters): every
      // contributor adds its exact sums into the N-tile's int64 accumulator (red.add, spread
      // over the rows' L2 lines) instead of a partial slot, so the last arriver reads one sum
      // per (row, class) instead of P partials
      const bool many = P > 8 && p.S_acc != nullptr;
      if (many) {
#pragma unroll
        for (int u = 0; u < KQ_MAX; ++u) {
          if (u < kq && row_ok && kq0 + u < K)
            atomicAdd(reinterpret_cast<unsigned long long*>(p.S_acc + row * p.Kp + kq0 + u),
                      (unsigned long long)sacc[u]);
          sacc[u] = 0;
        }
      } else {
        long long* part = p.S_part + (((int64_t)c * p.nslot + myslot) * BM + m) * p.Kp + kq0;
#pragma unroll
        for (int u = 0; u < KQ_MAX; ++u) {
          if (u < kq) part[u] = sacc[u];
          sacc[u] = 0;
        }
      }
      __threadfence();
      named_bar(1, NUM_EPI * 32);
      if (threadIdx.x == EPI_WARP0 * 32) {
        const unsigned prev = atomicAdd(p.cnt + ni, 1u);
        *s_flag = (prev == (unsigned)((c_last - c_first + 1) * CLD - 1)) ? 1 : 0;
        if (*s_flag) p.cnt[ni] = 0u;
      }
      named_bar(1, NUM_EPI * 32);
      // slot of this N-tile in a contributing CTA's S_part: clusters after c_first start
      // inside N-group ng (slot 0); c_first may have started in an earlier one
      const int ng_first = (int)(range_begin(c_first, p.T, p.G, p.runit) / p.TdG);
      const int slot_first = (CLD == 1) ? ((ng_first == ng) ? 0 : 1) : (ng - ng_first);
      auto part_ptr = [&](int idx, int r, int k) {   // partial idx (cluster-major, then D rank)
        const int cc = c_first + idx / CLD, j = idx % CLD;
        const int64_t cta = (int64_t)cc * CLS + rn * CLD + j;
        return p.S_part + ((cta * p.nslot + (cc == c_first ? slot_first : 0)) * BM + r) * p.Kp + k;
      };
      const int64_t r0 = (int64_t)ni * BM;
      const int nv = (int)((p.N - r0) < BM ? (p.N - r0) : BM);
      const int pairs = nv > 0 ? nv * K : 0;          // (row, class) sums of this N-tile
      if (*s_flag && many) {
        // the N-tile's sums are complete in S_acc: read and reset them (for the next call),
        // scores to p.scores (always non-null here), then one thread per row takes the argmax
        __threadfence();
        if (row_ok) {
#pragma unroll
          for (int u = 0; u < KQ_MAX; ++u) {
            const int k = kq0 + u;
            if (u < kq && k < K) {
              const long long v = (long long)atomicExch(reinterpret_cast<unsigned long long*>(p.S_acc + row * p.Kp + k), 0ull);
              p.scores[row * p.K + k] = (float)((double)v * p.inv_scale);
            }
          }
        }
        named_bar(1, NUM_EPI * 32);
        if (cq == 0 && row_ok) {
          int best = 0;
          float bv = 0.f;
          for (int k = 0; k < K; ++k) {
            const float v = p.scores[row * p.K + k];
            if (k == 0 || v > bv) {
              bv = v;
              best = k;
            }
          }
          if (p.labels) p.labels[row] = best;
        }
      } else if (*s_flag && P > 8) {
        // Many partials (small N: the N-tile's D-range is spread over many clusters). The
        // sums go to p.scores (always non-null here), then one thread per row takes the
        // argmax.  Few pairs: a warp per pair, lanes splitting the partials; otherwise a
        // thread per pair, 8 partial loads in flight.  Integer sums: any order is exact.
        __threadfence();
        if (pairs <= 4 * NUM_EPI) {
          for (int pi = ew; pi < pairs; pi += NUM_EPI) {
            const int r = pi / K, k = pi - r * K;
            long long sum = 0;
            for (int idx = lane; idx < P; idx += 32) sum += (long long)__ldcg(part_ptr(idx, r, k));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            if (lane == 0) p.scores[(r0 + r) * p.K + k] = (float)((double)sum * p.inv_scale);
          }
        } else {
          for (int pi = ew * 32 + lane; pi < pairs; pi += NUM_EPI * 32) {
            const int r = pi / K, k = pi - r * K;
            long long sum = 0;
            for (int i0 = 0; i0 < P; i0 += 8) {
              long long v[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) v[u] = (i0 + u < P) ? (long long)__ldcg(part_ptr(i0 + u, r, k)) : 0ll;
#pragma unroll
              for (int u = 0; u < 8; ++u) sum += v[u];
            }
            p.scores[(r0 + r) * p.K + k] = (float)((double)sum * p.inv_scale);
          }
        }
        named_bar(1, NUM_EPI * 32);
        if (cq == 0 && row_ok) {
          int best = 0;
          float bv = 0.f;
          for (int k = 0; k < K; ++k) {
            const float v = p.scores[row * p.K + k];
            if (k == 0 || v > bv) {
              bv = v;
              best = k;
            }
          }
          if (p.labels) p.labels[row] = best;
        }
      } else if (*s_flag) {
        __threadfence();
        // this thread's classes, all partials' loads of a class group in flight together
        float bv = 0.f;
        int best = -1;
        for (int u = 0; u < kq; ++u) {
          const int k = kq0 + u;
          if (k >= K) break;
          long long sum = 0;
          for (int idx = 0; idx < P; ++idx) sum += row_ok ? (long long)__ldcg(part_ptr(idx, m, k)) : 0ll;
          const float v = (float)((double)sum * p.inv_scale);
          if (row_ok && p.scores) p.scores[row * p.K + k] = v;
          if (best < 0 || v > bv) {
            bv = v;
            best = k;
          }
        }
        epi_argmax(best, bv, row_ok ? row : -1);
      }
      named_bar(1, NUM_EPI * 32);     // s_flag reuse
    }
    if (I8 && lane == 0 && nrecheck) atomicAdd(p.recheck_count, nrecheck);
  }
  if ((DBG(4)) && lane == 0 && (warp <= 3 || warp == EPI_WARP0)) {
    if (warp != EPI_WARP0) dbgc[15] = 0;
    dbgc[warp == EPI_WARP0 ? 12 : (warp == 3 ? 13 : 9 + warp)] = (unsigned long long)(clock64() - t_start);
    for (int i = 0; i < 16; ++i)
      if (dbgc[i]) atomicAdd(p.dbg + i, dbgc[i]);
  }
  __syncwarp();
  if constexpr (MC) cluster_sync_all();   // no CTA leaves while peers may still signal it
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (PAIR) tmem_dealloc_pair<512>(tmem_base);
    else tmem_dealloc<512>(tmem_base);
  }
}

// ---------------------------------------------------------------- operand prep
// int8 limbs of four elements -> one 4-byte store per limb; returns their L1(U).
__device__ __forceinline__ long long emit_limbs4(const float* x, float c, int8_t* __restrict__ out,
                                                 int64_t rows_p, int64_t r, int64_t Fp, int64_t f0) {
  uint32_t w0 = 0, w1 = 0, w2 = 0;
  long long l1 = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    int d0, d1, d2, U;
    limbs_of(x[e], c, d0, d1, d2, U);
    w0 |= (uint32_t)(uint8_t)(int8_t)d0 << (8 * e);
    w1 |= (uint32_t)(uint8_t)(int8_t)d1 << (8 * e);
    w2 |= (uint32_t)(uint8_t)(int8_t)d2 << (8 * e);
    l1 += U < 0 ? -U : U;
  }
  *reinterpret_cast<uint32_t*>(out + (0 * rows_p + r) * Fp + f0) = w0;
  *reinterpret_cast<uint32_t*>(out + (1 * rows_p + r) * Fp + f0) = w1;
  *reinterpret_cast<uint32_t*>(out + (2 * rows_p + r) * Fp + f0) = w2;
  return l1;
}

// One warp per row of a row-major [rows][F] fp32 matrix (X rows, or B^T rows): int8
// limbs into out[l][rows_p][Fp] and the per-row tau term.  Lane `lane` owns the groups
// of four elements f0 = 4 lane + 128 g (Fp is a multiple of 64, so a group is entirely
// inside or outside [0, Fp)); the row is read once into registers (Fp <= 128 NG).
template <int NG>
__global__ void limb_rows_kernel(const float* __restrict__ src, int64_t rows, int64_t rows_p,
                                 int64_t F, int64_t ld_src, int64_t Fp, int8_t* __restrict__ out,
                                 int64_t* __restrict__ tau_part, int64_t tau_const, bool vec) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= rows_p) return;
  const bool valid = r < rows;
  const float* __restrict__ row = src + r * ld_src;
  float xs[4 * NG];
  float amax = 0.f;
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    load4(row, 4 * lane + 128 * g, F, valid, vec, xs + 4 * g);
#pragma unroll
    for (int e = 0; e < 4; ++e) amax = fmaxf(amax, fabsf(xs[4 * g + e]));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  const float c = scale_for(amax);
  long long l1 = 0;
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    const int64_t f0 = 4 * lane + 128 * g;
    if (f0 < Fp) l1 += emit_limbs4(xs + 4 * g, c, out, rows_p, r, Fp, f0);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) l1 += __shfl_xor_sync(0xffffffffu, l1, o);
  if (lane == 0 && tau_part) tau_part[r] = row_tau(l1, tau_const, valid);
}

// Long rows (Fp > 1024): one 256-thread block per row, thread t owning the groups
// f0 = 4 t + 1024 g (Fp <= 1024 NGB); block reductions for max |x| and L1(U).
template <int NGB>
__global__ void __launch_bounds__(256) limb_rows_block_kernel(const float* __restrict__ src, int64_t rows,
                                                              int64_t rows_p, int64_t F, int64_t ld_src,
                                                              int64_t Fp, int8_t* __restrict__ out,
                                                              int64_t* __restrict__ tau_part,
                                                              int64_t tau_const, bool vec) {
  __shared__ float s_max[8];
  __shared__ long long s_l1[8];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t r = blockIdx.x;
  const bool valid = r < rows;
  const float* __restrict__ row = src + r * ld_src;
  float xs[4 * NGB];
  float amax = 0.f;
#pragma unroll
  for (int g = 0; g < NGB; ++g) {
    load4(row, 4 * t + 1024 * g, F, valid, vec, xs + 4 * g);
#pragma unroll
    for (int e = 0; e < 4; ++e) amax = fmaxf(amax, fabsf(xs[4 * g + e]));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if (lane == 0) s_max[w] = amax;
  __syncthreads();
  amax = s_max[0];
#pragma unroll
  for (int i = 1; i < 8; ++i) amax = fmaxf(amax, s_max[i]);
  const float c = scale_for(amax);
  long long l1 = 0;
#pragma unroll
  for (int g = 0; g < NGB; ++g) {
    const int64_t f0 = 4 * t + 1024 * g;
    if (f0 < Fp) l1 += emit_limbs4(xs + 4 * g, c, out, rows_p, r, Fp, f0);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) l1 += __shfl_xor_sync(0xffffffffu, l1, o);
  if (lane == 0) s_l1[w] = l1;
  __syncthreads();
  if (t == 0 && tau_part) {
    long long s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += s_l1[i];
    tau_part[r] = row_tau(s, tau_const, valid);
  }
}

// Two-pass fallback for very long rows (Fp > 4096): one warp per row.
__global__ void limb_rows_2pass_kernel(const float* __restrict__ src, int64_t rows, int64_t rows_p, int64_t F,
                                       int64_t ld_src, int64_t Fp, int8_t* __restrict__ out,
                                       int64_t* __restrict__ tau_part, int64_t tau_const, bool vec) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= rows_p) return;
  const bool valid = r < rows;
  const float* __restrict__ row = src + r * ld_src;
  float amax = 0.f;
  for (int64_t f0 = 4 * lane; f0 < Fp; f0 += 128) {
    float x[4];
    load4(row, f0, F, valid, vec, x);
#pragma unroll
    for (int e = 0; e < 4; ++e) amax = fmaxf(amax, fabsf(x[e]));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  const float c = scale_for(amax);
  long long l1 = 0;
  for (int64_t f0 = 4 * lane; f0 < Fp; f0 += 128) {
    float x[4];
    load4(row, f0, F, valid, vec, x);
    l1 += emit_limbs4(x, c, out, rows_p, r, Fp, f0);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) l1 += __shfl_xor_sync(0xffffffffu, l1, o);
  if (lane == 0 && tau_part) tau_part[r] = row_tau(l1, tau_const, valid);
}

// Rounded copies for the bf16 / tf32 modes: out[r][f] (rows_p x Fp, zero padded), four
// elements per thread (16-byte loads when aligned, 8 / 16-byte stores).
template <int MODE>
__global__ void round_rows_kernel(const float* __restrict__ src, int64_t rows, int64_t rows_p,
                                  int64_t F, int64_t ld_src, int64_t Fp, void* __restrict__ out, bool vec) {
  const int64_t gpr = Fp / 4, total = rows_p * gpr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / gpr, f0 = 4 * (i - r * gpr);
    float x[4];
    load4(src + r * ld_src, f0, F, r < rows, vec, x);
    if constexpr (MODE == 0) {
      __nv_bfloat162 a = __floats2bfloat162_rn(x[0], x[1]), b = __floats2bfloat162_rn(x[2], x[3]);
      uint2 v;
      v.x = *reinterpret_cast<uint32_t*>(&a);
      v.y = *reinterpret_cast<uint32_t*>(&b);
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(out) + r * Fp + f0) = v;
    } else {
      uint32_t y[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(y[e]) : "f"(x[e]));
      *reinterpret_cast<uint4*>(reinterpret_cast<uint32_t*>(out) + r * Fp + f0) = make_uint4(y[0], y[1], y[2], y[3]);
    }
  }
}


// C tiles for Stage II: per D-tile di, bf16 hi = RN(C), lo = RN(C - hi) (two parts), or
// hi, mid = RN(C - hi), lo = RN(C - hi - mid) (three parts: C - hi and C - hi - mid are
// exact in fp32, and hi + mid + lo = C for normal C), each [Kp][bn] in the interleaved
// K-major core-matrix layout the MMA B descriptor expects (core matrix (g, j) = rows 8g..,
// columns 8j.. at byte (g bn/8 + j) * 128).
__global__ void c_interleave_kernel(const float* __restrict__ Cp, int64_t K, int64_t Kp, int64_t D,
                                    int64_t Dp, int64_t Td, int bn, int nparts, __nv_bfloat16* __restrict__ out) {
  const int64_t per_part = Kp * bn;
  const int64_t total = Td * nparts * per_part;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t di = i / (nparts * per_part);
    const int part = (int)((i / per_part) % nparts);
    const int64_t e = i % per_part;          // element index inside the interleaved part
    const int64_t core = e / 64, inner = e % 64;
    const int64_t g = core / (bn / 8), j = core % (bn / 8);
    const int64_t r = g * 8 + inner / 8, cc = j * 8 + inner % 8;
    const int64_t d = di * bn + cc;
    const float v = (r < K && d < D) ? Cp[r * Dp + d] : 0.f;
    const __nv_bfloat16 hi = __float2bfloat16_rn(v);
    const float r1 = v - __bfloat162float(hi);
    const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
    out[i] = part == 0 ? hi : (part == 1 ? mid : __float2bfloat16_rn(r1 - __bfloat162float(mid)));
  }
}

// ---------------------------------------------------------------- int8 mode: deferred rechecks
// (1) One warp per listed sign: float64 re-evaluation (the same fixed-order sum as the
// in-kernel fallback).  Where it differs from the provisional sign that went into H,
// S[row, :] is off by exactly (h - h') C[:, d] = 2 h C[:, d] (Stage II is linear in H,
// P:180-183); that correction is accumulated in int64 fixed point (2^-shift units), so
// the sum is exact and independent of the order the warps run in: bit-deterministic.
__global__ void tc_recheck_kernel(const float* __restrict__ X, const float* __restrict__ Bt, int64_t F,
                                  int64_t Fp, const float* __restrict__ Cp, int64_t Dp, int64_t K,
                                  int64_t Kp, const uint2* __restrict__ flags,
                                  const unsigned long long* __restrict__ flag_count,
                                  unsigned long long cap, int shift, long long* __restrict__ corr,
                                  unsigned* __restrict__ dirty, unsigned long long* recheck_count,
                                  uint32_t* __restrict__ hout, int64_t hout_ldw) {
  const int lane = threadIdx.x & 31;
  const unsigned long long cnt = *flag_count;
  const unsigned long long n = cnt < cap ? cnt : cap;
  const unsigned long long w0 = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
  const unsigned long long nw = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
  const double scale = ldexp(2.0, shift);
  for (unsigned long long i = w0; i < n; i += nw) {
    const uint2 e = flags[i];
    const int64_t row = e.x, d = e.y & 0x7FFFFFFFu;
    const bool neg_prov = (e.y >> 31) != 0u;
    const float hv = recheck_dot(X + row * F, Bt + d * Fp, F, lane);
    if ((hv < 0.f) != neg_prov && hout) {       // encode mode: flip the packed bit
      if (lane == 0) atomicXor(hout + row * hout_ldw + (d >> 5), 1u << (d & 31));
    } else if ((hv < 0.f) != neg_prov) {
      if (lane == 0) dirty[row] = 1u;
      for (int64_t k = lane; k < K; k += 32) {
        const double c = (double)__ldg(Cp + k * Dp + d) * scale;
        atomicAdd(reinterpret_cast<unsigned long long*>(corr + row * Kp + k),
                  (unsigned long long)(long long)llrint(hv < 0.f ? -c : c));
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(recheck_count, n);
}

// (2) Rows with a flipped sign: S = S' + corr 2^-shift, lowest-index argmax;
// clears the row's workspace and the list for the next call.
__global__ void tc_finalize_kernel(int64_t N, int64_t K, int64_t Kp, int shift, float* __restrict__ S,
                                   long long* __restrict__ corr, unsigned* __restrict__ dirty,
                                   int32_t* __restrict__ labels, unsigned long long* flag_count) {
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row == 0) *flag_count = 0ull;        // the recheck kernel has read it (stream order)
  if (row >= N || !dirty[row]) return;
  const double inv = ldexp(1.0, -shift);
  int best = 0;
  float bv = 0.f;
  for (int64_t k = 0; k < K; ++k) {
    const float v = (float)((double)S[row * K + k] + (double)corr[row * Kp + k] * inv);
    S[row * K + k] = v;
    corr[row * Kp + k] = 0;
    if (k == 0 || v > bv) {
      bv = v;
      best = (int)k;
    }
  }
  if (labels) labels[row] = best;
  dirty[row] = 0u;
}

// max |C| over the model (for the fixed-point shift of the corrections)
__global__ void absmax_kernel(const float* __restrict__ a, int64_t n, unsigned* __restrict__ out) {
  float m = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf(a[i]));
  m = warp_max_f(m);
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));   // non-negative floats order as uints
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static const EncodeTiledFn fn = []() -> EncodeTiledFn {   // thread-safe one-time lookup
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return (EncodeTiledFn)p;
    return nullptr;
  }();
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

template <int MODE, int BN, int CLN, int CLD, bool ENC, bool HWC = true, bool PAIR = false, int KW = 0>
cudaError_t launch_mode(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, TcParams& p,
                        int num_sms, cudaStream_t st) {
  constexpr int CLS = CLN * CLD;
  const size_t sm = Cfg<MODE, BN, KW>::TOTAL + 1024;
  auto kern = fused_tc_kernel<MODE, BN, CLN, CLD, ENC, HWC, PAIR, KW>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  cfg.blockDim = dim3(THREADS, 1, 1);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = HWC ? CLS : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // persistent: as many clusters as can be co-resident (148 SMs: 74 pairs, 33 quads);
  // computed once per instantiation and device (benign race: every thread computes the same)
  constexpr int kMaxDev = 64;
  static std::atomic<int> cache[kMaxDev];
  int dev = 0;
  cudaGetDevice(&dev);
  int max_clusters = (dev >= 0 && dev < kMaxDev) ? cache[dev].load() : 0;
  if (max_clusters <= 0) {
    cudaLaunchConfig_t q = cfg;
    q.gridDim = dim3(CLS * (num_sms / CLS), 1, 1);
    int n = 0;
    if (!HWC) {
      n = num_sms / CLS;                          // one CTA per SM, CLS CTAs per virtual cluster
    } else if (cudaOccupancyMaxActiveClusters(&n, kern, &q) != cudaSuccess || n < 1) {
      cudaGetLastError();
      n = num_sms / CLS;
    }
    max_clusters = n;
    if (dev >= 0 && dev < kMaxDev) cache[dev].store(n);
  }
  p.G = (int)(p.T < max_clusters ? p.T : max_clusters);
  // whole N-tile rows per range when there are many per cluster (imbalance <= 1/8 row): the
  // groups then sweep B's D-groups in step, so a B chunk fetched from DRAM serves all of them
  // from L2 (cfg5 int8 17.5 -> 17.1-17.3 ms, D = 20000 36.5 -> 34.1, bf16 6.95 -> 6.80);
  // HDC_TC_ALIGN=0 restores tile-granular ranges (measurements)
  {
    const char* al = getenv("HDC_TC_ALIGN");
    const bool align = al ? atoi(al) != 0 : true;
    p.runit = (align && p.TdG > 1 && p.T / p.TdG >= 8 * (int64_t)p.G) ? p.TdG : 1;
  }
  const int64_t per = (p.T / p.runit + p.G - 1) / p.G * p.runit;   // cluster tiles per range (at most)
  p.nslot = (CLD == 1) ? 2 : (int)((per + p.TdG - 1) / p.TdG + 1);
  if ((int64_t)p.G * CLS * p.nslot > p.s_part_cap) return cudaErrorInvalidValue;   // workspace bound
  cfg.gridDim = dim3(p.G * CLS, 1, 1);
  e = cudaLaunchKernelEx(&cfg, kern, a, b, c, (const TcParams)p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <int MODE, int BN, bool ENC, int KW>
cudaError_t launch_cluster_k(int cl_n, int cl_d, int virt, const CUtensorMap& a, const CUtensorMap& b,
                             const CUtensorMap& c, TcParams& p, int num_sms, cudaStream_t st) {
  if constexpr (MODE < 2 && !ENC) {
    if (virt == 2 && cl_n == 2 && cl_d == 1)   // CTA pair as one cta_group::2 MMA unit
      return launch_mode<MODE, BN, 2, 1, false, true, true>(a, b, c, p, num_sms, st);
  }
  if (virt == 2) virt = 0;                      // pair requested where it does not apply: 2x1 cluster
  if (virt) {
    if (cl_n == 1 && cl_d == 4) return launch_mode<MODE, BN, 1, 4, ENC, false, false, KW>(a, b, c, p, num_sms, st);
    if (cl_n == 1 && cl_d == 8) return launch_mode<MODE, BN, 1, 8, ENC, false, false, KW>(a, b, c, p, num_sms, st);
    if (cl_n == 1 && cl_d == 16) return launch_mode<MODE, BN, 1, 16, ENC, false, false, KW>(a, b, c, p, num_sms, st);
    return cudaErrorInvalidValue;
  }
  if (cl_n == 1 && cl_d == 1) return launch_mode<MODE, BN, 1, 1, ENC, true, false, KW>(a, b, c, p, num_sms, st);
  if (cl_n == 1 && cl_d == 2) return launch_mode<MODE, BN, 1, 2, ENC, true, false, KW>(a, b, c, p, num_sms, st);
  if (cl_n == 2 && cl_d == 1) return launch_mode<MODE, BN, 2, 1, ENC, true, false, KW>(a, b, c, p, num_sms, st);
  return cudaErrorInvalidValue;
}
// int8 mode: 128-byte K stages when Fp is a multiple of 128 (half the producer / MMA
// hand-offs), else 64-byte stages (a 128-byte last stage would load 64 bytes of zeros
// per row: cfg4, F = 784, ran 7% slower)
int tc_kbytes(int mode, int64_t Fp) {
  if (mode == 3) return 64;                            // wide: 3 stages of 54 KB
  if (mode != 2) return HDC_TC_KB16;
  const char* e = getenv("HDC_TC_KB8");              // measurements: force 64-byte int8 stages
  if (e && atoi(e) == 64) return 64;
  return (Fp % 128 == 0) ? 128 : 64;
}
template <int MODE, int BN, bool ENC>
cudaError_t launch_cluster_e(int cl_n, int cl_d, int virt, const CUtensorMap& a, const CUtensorMap& b,
                             const CUtensorMap& c, TcParams& p, int num_sms, cudaStream_t st) {
  if constexpr (MODE == 3) {
    return launch_cluster_k<MODE, BN, ENC, 64>(cl_n, cl_d, virt, a, b, c, p, num_sms, st);
  } else if constexpr (MODE == 2) {
    if (tc_kbytes(MODE, p.Fp) == 128)
      return launch_cluster_k<MODE, BN, ENC, 128>(cl_n, cl_d, virt, a, b, c, p, num_sms, st);
    return launch_cluster_k<MODE, BN, ENC, 64>(cl_n, cl_d, virt, a, b, c, p, num_sms, st);
  } else {
    return launch_cluster_k<MODE, BN, ENC, 0>(cl_n, cl_d, virt, a, b, c, p, num_sms, st);
  }
}
// ENC (encode mode, hdc_model_encode) is a separate instantiation so the inference kernel
// carries no encode branches.
template <int MODE, int BN>
cudaError_t launch_cluster(int cl_n, int cl_d, int virt, const CUtensorMap& a, const CUtensorMap& b,
                           const CUtensorMap& c, TcParams& p, int num_sms, cudaStream_t st) {
  return p.hout ? launch_cluster_e<MODE, BN, true>(cl_n, cl_d, virt, a, b, c, p, num_sms, st)
                : launch_cluster_e<MODE, BN, false>(cl_n, cl_d, virt, a, b, c, p, num_sms, st);
}

}  // namespace

bool make_tensor_map_u8(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint32_t box_inner,
                        uint32_t box_outer, int swizzle_bytes) {
  const CUtensorMapSwizzle sw = swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                                : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                      : CU_TENSOR_MAP_SWIZZLE_NONE;
  return make_map_2d(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, base, inner, outer, box_inner, box_outer, sw);
}

int tc_tile_n(int mode, int64_t K) { return tile_n_for(mode, K); }
int64_t tc_s_part_slots(int64_t Tn, int64_t Td, int cl_n, int cl_d, int virt, int num_sms) {
  if (cl_d == 1) return 2 * (int64_t)num_sms;
  const int64_t T = (Tn / cl_n) * (Td / cl_d), TdG = Td / cl_d;
  int64_t gmin = num_sms / (cl_n * cl_d) / 2 > 0 ? num_sms / (cl_n * cl_d) / 2 : 1;  // >= half co-resident
  if (virt) gmin = num_sms / (cl_n * cl_d);       // virtual clusters: exactly this many
  const int64_t per = (T + gmin - 1) / gmin;
  return (int64_t)num_sms * ((per + TdG - 1) / TdG + 1);
}
void tc_cluster_shape(int mode, int64_t K, int64_t F, int64_t D, int* cl_n, int* cl_d, int* virt) {
  // default: CTA pairs on two N-tiles of the same D-tile, multicasting the B tile
  // (measured best of 1x1 / 1x2 / 2x1 / 2x2 / 1x4 hardware clusters at cfg2, tools/tc_timing.py).
  // When the live X tiles of 148 CTAs plus B exceed the L2 (large F: cfg5 read 176 GB from
  // DRAM per launch), a virtual 1 x g group puts g CTAs on each N-tile (g = 4, 8, 16).
  const int bn = tile_n_for(mode, K);
  int n = 2, d = 1, v = 0;
  if (bn == 80 && mode < 2) n = 1;                // (bf16/tf32 with K > 32: no cluster)
  const int64_t Fp = (F + 63) / 64 * 64;
  const double esz_nl = (mode >= 2) ? 3.0 : (mode == 0 ? 2.0 : 4.0);
  const double a_tile = 128.0 * Fp * esz_nl, b_all = (double)(D + bn) * Fp * esz_nl;
  const double l2 = 120e6;                        // of the 126 MB L2, leaving room for C, S
  if (148.0 * a_tile + b_all > l2) {
    n = 1;
    v = 1;
    // group size g: the g-CTA groups' live X tiles plus B should leave L2 headroom
    // (measured at cfg5: 1x16 20.4 ms vs 1x8 21.1-21.8 ms int8, 6.51 vs 6.68 ms bf16)
    const double fit = 75e6;
    d = (37.0 * a_tile + b_all <= fit) ? 4 : (18.0 * a_tile + b_all <= fit) ? 8 : 16;
  }
  const char* env = getenv("HDC_TC_CLUSTER");
  int en = 0, ed = 0;
  char vc = 0;
  if (env) {
    const int got = sscanf(env, "%dx%d%c", &en, &ed, &vc);
    if (got >= 2 && !(bn == 80 && mode < 2)) {
      if (got == 3 && vc == 'v' && en == 1 && (ed == 4 || ed == 8 || ed == 16)) {
        n = 1; d = ed; v = 1;
      } else if (got == 3 && vc == 'p' && en == 2 && ed == 1 && mode < 2) {
        n = 2; d = 1; v = 2;                      // CTA pair (cta_group::2)
      } else if (got == 2 && ((en == 1 && (ed == 1 || ed == 2)) || (en == 2 && ed == 1))) {
        n = en; d = ed; v = 0;
      }
    }
  }
  *cl_n = n;
  *cl_d = d;
  *virt = v;
}
int tc_max_k(int mode) { return mode == 3 ? 16 : mode == 2 ? KP_MAX_I8 : KP_MAX_16; }
int64_t tc_kp(int64_t K) { return (K + 15) / 16 * 16; }
int64_t tc_c_tile_bytes(int mode, int64_t K) {
  const int64_t bn = tile_n_for(mode, K);
  return (mode >= 2 ? 3 : 2) * tc_kp(K) * bn * 2;   // bf16 parts (c_interleave_kernel), [Kp][bn] each
}
int64_t tc_max_fp_int8() { return 100000; }

// Shift of the epilogue's coarse flag test: |I| < 2^28.03 Fp (three int8 limb products per
// element), so floor(I / 2^s) with 2^s >= Fp / 2 fits in 30 bits; the granularity 2^s is
// at most ~3% of the smallest tau (>= 64 F), so the coarse test flags few extra elements.
int tc_flag_shift(int64_t Fp) {
  int s = 0;
  while ((int64_t(1) << (s + 1)) < Fp) ++s;          // 2^(s+1) >= Fp
  // 7 <= s <= 14 for the 32-bit form of the test (at Fp <= tc_max_fp_int8, |J| < 2^30.7)
  return s < 7 ? 7 : s > 14 ? 14 : s;
}

__global__ void coltau_m_kernel(const int64_t* __restrict__ coltau, int64_t Dq, int shift, int32_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= Dq) return;
  const int64_t t = coltau[i];
  // ceil(t / 2^shift); columns past D (t = -2^62) never flag
  out[i] = t < 0 ? -(1 << 28) : (int32_t)((t + (int64_t(1) << shift) - 1) >> shift);
}

cudaError_t launch_tc_coltau_m(const int64_t* coltau, int64_t Dq, int shift, int32_t* out, cudaStream_t st) {
  coltau_m_kernel<<<(unsigned)((Dq + 255) / 256), 256, 0, st>>>(coltau, Dq, shift, out);
  return cudaGetLastError();
}

int64_t tc_tau_const(int64_t F) {
  // F (0.390625 + 2^20 + 2^12) + 1, in the integer units of U_x.U_b (before the 2^-14 scale)
  return (int64_t)F * 1052673 + 1;
}

cudaError_t launch_tc_limbs(const float* src, int64_t rows, int64_t rows_p, int64_t F, int64_t ld_src,
                            int64_t Fp, int8_t* out, int64_t* tau_part, int64_t tau_const,
                            cudaStream_t st) {
  // 16-byte loads need 16-byte aligned rows
  const bool vec = ((reinterpret_cast<uintptr_t>(src) & 15) == 0) && (ld_src % 4 == 0);
  const int warps = 8;
  const unsigned grid = (unsigned)((rows_p + warps - 1) / warps);
  if (Fp <= 512)
    limb_rows_kernel<4><<<grid, warps * 32, 0, st>>>(src, rows, rows_p, F, ld_src, Fp, out, tau_part, tau_const, vec);
  else if (Fp <= 1024)
    limb_rows_kernel<8><<<grid, warps * 32, 0, st>>>(src, rows, rows_p, F, ld_src, Fp, out, tau_part, tau_const, vec);
  else if (Fp <= 2048)
    limb_rows_block_kernel<2><<<(unsigned)rows_p, 256, 0, st>>>(src, rows, rows_p, F, ld_src, Fp, out, tau_part,
                                                                 tau_const, vec);
  else if (Fp <= 4096)
    limb_rows_block_kernel<4><<<(unsigned)rows_p, 256, 0, st>>>(src, rows, rows_p, F, ld_src, Fp, out, tau_part,
                                                                 tau_const, vec);
  else
    limb_rows_2pass_kernel<<<grid, warps * 32, 0, st>>>(src, rows, rows_p, F, ld_src, Fp, out, tau_part, tau_const,
                                                        vec);
  return cudaGetLastError();
}

cudaError_t launch_tc_round(int mode, const float* src, int64_t rows, int64_t rows_p, int64_t F,
                            int64_t ld_src, int64_t Fp, void* out, cudaStream_t st) {
  const int64_t total = rows_p * Fp;
  int64_t grid = (total + 255) / 256;
  if (grid > 148 * 16) grid = 148 * 16;
  const bool vec = ((reinterpret_cast<uintptr_t>(src) & 15) == 0) && (ld_src % 4 == 0);
  if (mode == 0)
    round_rows_kernel<0><<<(unsigned)grid, 256, 0, st>>>(src, rows, rows_p, F, ld_src, Fp, out, vec);
  else
    round_rows_kernel<1><<<(unsigned)grid, 256, 0, st>>>(src, rows, rows_p, F, ld_src, Fp, out, vec);
  return cudaGetLastError();
}

cudaError_t launch_tc_c_tiles(int mode, const float* Cp, int64_t K, int64_t D, int64_t Dp, int64_t Dq,
                              void* out, cudaStream_t st) {
  const int bn = tile_n_for(mode, K);
  const int64_t Td = Dq / bn;                 // includes cluster padding tiles (all zero)
  const int64_t Kp = tc_kp(K);
  const int nparts = mode >= 2 ? 3 : 2;
  const int64_t total = Td * nparts * Kp * bn;
  int64_t grid = (total + 255) / 256;
  if (grid > 148 * 16) grid = 148 * 16;
  c_interleave_kernel<<<(unsigned)grid, 256, 0, st>>>(Cp, K, Kp, D, Dp, Td, bn, nparts, (__nv_bfloat16*)out);
  return cudaGetLastError();
}

cudaError_t launch_tc_recheck(const TcOperands& o, int64_t N, float* S, int32_t* labels, int shift,
                              cudaStream_t st) {
  tc_recheck_kernel<<<148 * 8, 256, 0, st>>>(o.X, o.Bt, o.F, o.Fp, o.Cp, o.Dp, o.K, tc_kp(o.K), o.flags,
                                             o.flag_count, o.flag_cap, shift, o.corr, o.dirty, o.recheck,
                                             o.hout, o.hout_ldw);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  tc_finalize_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(N, o.K, tc_kp(o.K), shift, S, o.corr,
                                                                  o.dirty, labels, o.flag_count);
  return cudaGetLastError();
}

int tc_corr_shift(const float* Cp, int64_t n, int64_t D) {
  unsigned* d = nullptr;
  unsigned h = 0;
  if (cudaMalloc((void**)&d, sizeof(unsigned)) != cudaSuccess) return 0;
  cudaMemset(d, 0, sizeof(unsigned));
  absmax_kernel<<<148, 256>>>(Cp, n, d);
  cudaMemcpy(&h, d, sizeof(unsigned), cudaMemcpyDeviceToHost);
  cudaFree(d);
  float cmax;
  memcpy(&cmax, &h, sizeof(float));
  // |sum of corrections| <= 2 D max|C| 2^shift < 2^62
  int ex = 0;
  frexp((double)cmax * 2.0 * (double)(D > 0 ? D : 1), &ex);   // 2 D max|C| < 2^ex
  int shift = 61 - ex;
  if (shift > 900) shift = 900;
  return shift;
}

cudaError_t launch_fused_tc(int mode, const TcOperands& o, int64_t N, float* scores, int32_t* labels,
                            int num_sms, cudaStream_t st) {
  const int bn = tile_n_for(mode, o.K);
  const int64_t Tn = o.N_p / BM;              // multiple of cl_n
  const int64_t Td = o.Dq / bn;               // multiple of cl_d
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
  p.TdG = (int)(Td / o.cl_d);
  p.T = (Tn / o.cl_n) * p.TdG;
  p.G = 0;                                    // set by launch_mode (co-resident clusters)
  p.X = o.X;
  p.Bt = o.Bt;
  p.rowtau = o.rowtau;
  p.coltau = o.coltau;
  p.coltau_m = o.coltau_m;
  p.flag_shift = o.flag_shift;
  p.Cil = (const uint8_t*)o.Cil;
  p.c_tile_bytes = (uint32_t)tc_c_tile_bytes(mode, o.K);
  p.S_part = o.S_part;
  p.S_acc = o.S_acc;
  p.s_part_cap = o.s_part_slots;
  p.scale = ldexp(1.0, o.shift);
  p.inv_scale = ldexp(1.0, -o.shift);
  p.scale_f = (o.shift >= -126 && o.shift <= 126) ? ldexpf(1.f, o.shift) : 0.f;
  p.cnt = o.cnt;
  p.recheck_count = o.recheck;
  p.hout = o.hout;
  p.hout_ldw = o.hout_ldw;
  p.flags = o.flags;
  p.flag_count = o.flag_count;
  p.flag_cap = o.flag_cap;
  p.scores = scores;
  p.labels = labels;
  {
    const char* dbg = getenv("HDC_TC_DEBUG");
    p.debug = dbg ? atoi(dbg) : 0;
  }
  static unsigned long long* dbg_buf = nullptr;
  p.dbg = nullptr;
  if (p.debug & (4 | 1024)) {
    if (!dbg_buf) cudaMalloc((void**)&dbg_buf, (16 + 512) * sizeof(unsigned long long));
    cudaMemsetAsync(dbg_buf, 0, (16 + 512) * sizeof(unsigned long long), st);
    p.dbg = dbg_buf;
  }
  static unsigned long long* wd_host = nullptr;   // watchdog records, host-mapped
  if (p.debug & 16384) {
    if (!wd_host) cudaHostAlloc((void**)&wd_host, (8 + 4 * 64) * sizeof(unsigned long long), cudaHostAllocMapped);
    memset(wd_host, 0, (8 + 4 * 64) * sizeof(unsigned long long));
    cudaHostGetDevicePointer((void**)&p.dbg, wd_host, 0);
  }
  const int nl = (mode >= 2) ? 3 : 1;
  const int subn = (mode == 3) ? bn / 2 : bn;  // wide: B loads per 80-column sub-tile
  const int esz = (mode == 0) ? 2 : (mode == 1) ? 4 : 1;
  const CUtensorMapDataType dt = (mode == 0)   ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                 : (mode == 1) ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                               : CU_TENSOR_MAP_DATA_TYPE_UINT8;
  CUtensorMap ma, mb, mc;
  const uint32_t kbytes = (uint32_t)tc_kbytes(mode, o.Fp);
  const CUtensorMapSwizzle swz = (kbytes == 64) ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
  // boxes: this CTA's slice of the tile (the rest arrives by multicast from cluster peers)
  const int a_rows = o.cl_virt == 1 ? BM : BM / o.cl_d, b_rows = o.cl_virt == 1 ? subn : subn / o.cl_n;
  if (!make_map_2d(&ma, dt, esz, o.A, (uint64_t)o.Fp, (uint64_t)nl * o.N_p, kbytes / esz, a_rows, swz) ||
      !make_map_2d(&mb, dt, esz, o.B, (uint64_t)o.Fp, (uint64_t)nl * o.Dq, kbytes / esz, b_rows, swz))
    return cudaErrorInvalidValue;
  // CTA-pair mode: each CTA loads half the class rows of a C tile part (rows of 128 B)
  memset(&mc, 0, sizeof(mc));
  if (o.cl_virt == 2 && o.Cil &&
      !make_map_2d(&mc, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, o.Cil, 128,
                   (uint64_t)(Td * (int64_t)p.c_tile_bytes / 128), 128, (uint32_t)(p.Kp * bn / 128),
                   CU_TENSOR_MAP_SWIZZLE_NONE))
    return cudaErrorInvalidValue;
  cudaError_t e;
  if (mode == 0 && bn == 160) e = launch_cluster<0, 160>(o.cl_n, o.cl_d, o.cl_virt, ma, mb, mc, p, num_sms, st);
  else if (mode == 1 && bn == 160) e = launch_cluster<1, 160>(o.cl_n, o.cl_d, o.cl_virt, ma, mb, mc, p, num_sms, st);
  else if (mode == 2) e = launch_cluster<2, 80>(o.cl_n, o.cl_d, o.cl_virt, ma, mb, mc, p, num_sms, st);
  else if (mode == 3) e = launch_cluster<3, 160>(o.cl_n, o.cl_d, o.cl_virt, ma, mb, mc, p, num_sms, st);
  else if (o.cl_n == 1 && o.cl_d == 1)
    e = (mode == 0) ? (p.hout ? launch_mode<0, 80, 1, 1, true>(ma, mb, mc, p, num_sms, st)
                              : launch_mode<0, 80, 1, 1, false>(ma, mb, mc, p, num_sms, st))
                    : (p.hout ? launch_mode<1, 80, 1, 1, true>(ma, mb, mc, p, num_sms, st)
                              : launch_mode<1, 80, 1, 1, false>(ma, mb, mc, p, num_sms, st));
  else e = cudaErrorInvalidValue;
  if (e == cudaSuccess && (p.debug & 16384)) {
    cudaStreamSynchronize(st);
    const unsigned long long n = wd_host[1] < 64 ? wd_host[1] : 64;
    fprintf(stderr, "[hdc tc watchdog] %s: %llu stalled waits\n", wd_host[0] ? "ABORTED" : "ok", wd_host[1]);
    for (unsigned long long i = 0; i < n; ++i) {
      const unsigned long long* r = wd_host + 8 + 4 * i;
      fprintf(stderr, "  slot %2llu  cta %4llu  warp %2llu  parity %llu  since %llu kcyc\n", r[0], r[1], r[2],
              r[3] >> 32, r[3] & 0xffffffffull);
    }
  }
  if (e == cudaSuccess && (p.debug & 1024)) {
    unsigned long long h[512];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, dbg_buf + 16, sizeof(h), cudaMemcpyDeviceToHost);
    fprintf(stderr, "[hdc tc timeline] CTA 0, KB=%d stages/tile; MMA full-wait exits / producer empty-wait exits (cycles from first):\n", (int)(p.Fp / (mode >= 2 ? 64 : (mode == 0 ? 64 : 32))));
    for (int i = 0; i < 64; ++i)
      fprintf(stderr, "  stage %3d: mma %8lld  prod %8lld\n", i, (long long)(h[i] - h[0]), (long long)(h[256 + i] - h[0]));
  }
  if (e == cudaSuccess && (p.debug & 4)) {
    unsigned long long h[16];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, dbg_buf, sizeof(h), cudaMemcpyDeviceToHost);
    const char* names[16] = {"prod.empty", "mma.tempty", "mma.full", "s2.hfull", "s2.cfull",
                             "s2.sempty", "epi.tfull", "epi.hempty", "epi.sfull", "prod.total",
                             "mma.total", "cprod.total", "epi.total", "s2.total", "cprod.cempty", "epi.cfull"};
    fprintf(stderr, "[hdc tc debug] mode %d, %d CTAs, %lld tiles; mean cycles per CTA:", mode, p.G,
            (long long)p.T);
    for (int i = 0; i < 16; ++i) fprintf(stderr, " %s=%.0f", names[i], (double)h[i] / p.G);
    fprintf(stderr, "\n");
  }
  return e;
}

}  // namespace hdc
