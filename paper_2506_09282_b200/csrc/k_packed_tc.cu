// k_packed_tc.cu -- the unfused ablation's Stage II at its own roofline: S = H C^T and the
// argmax from a bit-packed H in HBM (written by hdc_model_encode), on the tensor cores.
//
// The paper's fusion ablation compares keeping H on chip against
// materialising it.  A fair B200 comparison needs the second pass to be as good as the
// hardware allows: here Stage II is tcgen05 `kind::f16` over H unpacked to exact bf16 +-1
// in shared memory, C split into bf16 hi + lo (as in the fused kernel), fp32 accumulation
// in TMEM over the CTA's D-range in column order, and the CTAs of a row tile summed
// exactly in int64 fixed point (eq. batch_sim; lowest-index argmax P:187-190).
//
// CTA = 128 rows x a contiguous range of 64-column chunks.  Warps 2..5 (one per row
// quarter) unpack each chunk's 64 bits per row into the A stage (K-major core matrices,
// a 256-entry byte -> 8 x bf16 table); warp 0 bulk-copies the chunk's C hi/lo tile
// (prepared per call in the MMA's B layout); warp 1 issues 8 MMAs per chunk (4 k-steps x
// hi/lo); the unpack warps then read S from TMEM.
#include <cuda_bf16.h>

#include <cstdio>

#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace hdc {
namespace {

using namespace ptx;

constexpr int kPT_Threads = 192;                  // warp 0 C copies, warp 1 MMA, warps 2..5 unpack + epilogue
constexpr int kChunk = 64;                        // columns per chunk
constexpr int kAStages = 4;
constexpr int kCStages = 3;
constexpr int kABytes = 128 * kChunk * 2;         // bf16 H tile [128][64] in core matrices

struct PackedTcParams {
  const uint32_t* H;
  int64_t ldw, N, D, K, Kp;
  int nchunks, DS;                                // chunks of D, CTAs per row tile
  const uint8_t* ctiles;                          // per chunk: [2][Kp][64] bf16 core matrices
  uint32_t cbytes;                                // bytes per chunk (both parts)
  const unsigned* cmax;                           // max |C| (float bits): the fixed point's scale
  unsigned long long* acc;                        // [N][Kp] int64 sums, zero before the launch
  unsigned* cnt;                                  // [row tiles], zero before the launch
  int32_t* labels;
  float* scores;
};

// max |C| as the bits of a non-negative float (they order like the values)
__global__ void c_absmax_kernel(const float* __restrict__ C, int64_t n, unsigned* __restrict__ out) {
  float m = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf(C[i]));
  m = warp_max_f(m);
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

// fixed point 2^-shift with 2 D max|C| 2^shift < 2^62 (exact int64 sums, no overflow)
__device__ __forceinline__ int fixed_shift(float cmax, int64_t D) {
  int ex = 0;
  frexp((double)cmax * 2.0 * (double)(D > 0 ? D : 1), &ex);
  const int s = 61 - ex;
  return s > 900 ? 900 : s;
}

// C (K x D fp32, row-major) -> per 64-column chunk the bf16 hi / lo parts of C^T as the
// MMA's B operand: rows = classes (Kp, zero padded), K-major core matrices (g, j) =
// classes 8g.., columns 8j.. at byte (8 g + j) 128; lo = RN(c - hi)
__global__ void c_chunk_tiles_kernel(const float* __restrict__ C, int64_t K, int64_t Kp, int64_t D, int nchunks,
                                     __nv_bfloat16* __restrict__ out) {
  const int64_t per_part = Kp * kChunk, total = (int64_t)nchunks * 2 * per_part;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ch = i / (2 * per_part);
    const int part = (int)((i / per_part) % 2);
    const int64_t e = i % per_part;
    const int64_t core = e / 64, inner = e % 64;
    const int64_t g = core / 8, j = core % 8;
    const int64_t r = g * 8 + inner / 8, cc = j * 8 + inner % 8;
    const int64_t d = ch * kChunk + cc;
    const float v = (r < K && d < D) ? C[r * D + d] : 0.f;
    const __nv_bfloat16 hi = __float2bfloat16_rn(v);
    out[i] = part == 0 ? hi : __float2bfloat16_rn(v - __bfloat162float(hi));
  }
}

template <int KP>
__global__ void __launch_bounds__(kPT_Threads, 1) packed_similarity_tc_kernel(const PackedTcParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;                                         // [kAStages][kABytes]
  uint8_t* sC = sA + kAStages * kABytes;                      // [kCStages][cbytes]
  uint4* table = reinterpret_cast<uint4*>(sC + kCStages * 2 * KP * kChunk * 2);   // [256] byte -> 8 bf16 +-1
  uint64_t* bars = reinterpret_cast<uint64_t*>(table + 256);
  uint64_t* afull = bars;                                     // [kAStages] unpacked (4 warps)
  uint64_t* aempty = afull + kAStages;                        // [kAStages] MMAs done
  uint64_t* cfull = aempty + kAStages;                        // [kCStages]
  uint64_t* cempty = cfull + kCStages;
  uint64_t* sfull = cempty + kCStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sfull + 1);
  int* s_last = reinterpret_cast<int*>(tmem_slot + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tile = blockIdx.x / p.DS, part = blockIdx.x % p.DS;
  const int c0 = (int)((int64_t)part * p.nchunks / p.DS), c1 = (int)((int64_t)(part + 1) * p.nchunks / p.DS);
  const int64_t r0 = (int64_t)tile * 128;
  const uint32_t cb = (uint32_t)(2 * KP * kChunk * 2);        // C bytes per chunk
  const int shift = fixed_shift(__uint_as_float(*p.cmax), p.D);
  const double scale = ldexp(1.0, shift), inv_scale = ldexp(1.0, -shift);

  for (int i = tid; i < 256; i += kPT_Threads) {
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t lo = ((i >> (2 * q)) & 1) ? 0xBF80u : 0x3F80u;     // bit set <=> h = -1
      const uint32_t hi = ((i >> (2 * q + 1)) & 1) ? 0xBF80u : 0x3F80u;
      w[q] = lo | (hi << 16);
    }
    table[i] = make_uint4(w[0], w[1], w[2], w[3]);
  }
  if (tid == 0) {
    for (int s = 0; s < kAStages; ++s) {
      mbar_init(afull + s, 4);
      mbar_init(aempty + s, 1);
    }
    for (int s = 0; s < kCStages; ++s) {
      mbar_init(cfull + s, 1);
      mbar_init(cempty + s, 1);
    }
    mbar_init(sfull, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<KP < 32 ? 32 : KP>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int c = c0; c < c1; ++c) {
        const int i = c - c0, s = i % kCStages;
        if (i >= kCStages) mbar_wait(cempty + s, (uint32_t)(((i / kCStages) - 1) & 1));
        mbar_arrive_expect_tx(cfull + s, cb);
        bulk_load(sC + (size_t)s * cb, p.ctiles + (size_t)c * cb, cb, cfull + s);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t IDESC = make_idesc<0>(128, KP);
    for (int c = c0; c < c1; ++c) {
      const int i = c - c0, sa = i % kAStages, sc = i % kCStages;
      mbar_wait(afull + sa, (uint32_t)((i / kAStages) & 1));
      mbar_wait(cfull + sc, (uint32_t)((i / kCStages) & 1));
      tc_fence_after();
      const uint32_t a_base = smem_u32(sA + (size_t)sa * kABytes), c_base = smem_u32(sC + (size_t)sc * cb);
#pragma unroll
      for (int ks = 0; ks < kChunk / 16; ++ks) {
        const uint64_t ad = smem_desc_interleaved(a_base + ks * 2 * 128, 128, 1024);
#pragma unroll
        for (int hl = 0; hl < 2; ++hl) {
          const uint64_t bd = smem_desc_interleaved(c_base + hl * (KP * kChunk * 2) + ks * 2 * 128, 128, 1024);
          tc_mma_elect<0>(tmem, ad, bd, IDESC, (i | ks | hl) ? 1u : 0u);
        }
      }
      tc_commit_elect(aempty + sa);
      tc_commit_elect(cempty + sc);
    }
    tc_commit_elect(sfull);
  } else {
    // ===================================================== unpack (row r = thread) + epilogue
    const int q = warp & 3, r = q * 32 + lane;
    const int64_t row = r0 + r;
    const bool row_ok = row < p.N;
    const uint32_t* hr = p.H + (row_ok ? row : 0) * p.ldw;
    for (int c = c0; c < c1; ++c) {
      const int i = c - c0, sa = i % kAStages;
      if (i >= kAStages) mbar_wait(aempty + sa, (uint32_t)(((i / kAStages) - 1) & 1));
      const int64_t wi = (int64_t)c * 2;
      const uint32_t w0 = (row_ok && wi < p.ldw) ? __ldg(hr + wi) : 0u;
      const uint32_t w1 = (row_ok && wi + 1 < p.ldw) ? __ldg(hr + wi + 1) : 0u;
      // columns past D: their C is zero, any sign contributes 0
      uint8_t* dst = sA + (size_t)sa * kABytes + (size_t)(r >> 3) * 1024 + (r & 7) * 16;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t bits = ((j < 4 ? w0 : w1) >> (8 * (j & 3))) & 255u;
        *reinterpret_cast<uint4*>(dst + j * 128) = table[bits];
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(afull + sa);
    }
    mbar_wait(sfull, 0);
    tc_fence_after();
    // this CTA's sums: fp32 from TMEM -> int64 fixed point -> exact cross-CTA atomics
    const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16);
#pragma unroll
    for (int k0 = 0; k0 < KP; k0 += 8) {
      uint32_t v[8];
      tmem_ld8(tb + k0, v);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k = k0 + j;
        if (row_ok && k < p.K)
          atomicAdd(p.acc + row * p.Kp + k, (unsigned long long)llrint((double)__uint_as_float(v[j]) * scale));
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<KP < 32 ? 32 : KP>(tmem);
  }
  if (warp < 2) return;
  // the last CTA of the row tile converts the sums and takes the argmax
  asm volatile("bar.sync 1, 128;" ::: "memory");
  if (tid == 64) {
    unsigned prev;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(p.cnt + tile) : "memory");
    *s_last = (prev == (unsigned)(p.DS - 1)) ? 1 : 0;
  }
  asm volatile("bar.sync 1, 128;" ::: "memory");
  if (!*s_last) return;
  const int q = warp & 3, r = q * 32 + (tid & 31);
  const int64_t row = r0 + r;
  if (row >= p.N) return;
  int best = 0;
  float bv = 0.f;
  for (int k = 0; k < p.K; ++k) {
    const float v = (float)((double)(long long)__ldcg(reinterpret_cast<const long long*>(p.acc) + row * p.Kp + k) *
                            inv_scale);
    if (p.scores) p.scores[row * p.K + k] = v;
    if (k == 0 || v > bv) {
      bv = v;
      best = k;
    }
  }
  if (p.labels) p.labels[row] = best;
}

template <int KP>
cudaError_t launch_kp(PackedTcParams& p, int64_t tiles, cudaStream_t st) {
  const size_t sm = 1024 + (size_t)kAStages * kABytes + (size_t)kCStages * 2 * KP * kChunk * 2 + 256 * 16 + 256;
  cudaError_t e = cudaFuncSetAttribute(packed_similarity_tc_kernel<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sm);
  if (e != cudaSuccess) return e;
  packed_similarity_tc_kernel<KP><<<(unsigned)(tiles * p.DS), kPT_Threads, sm, st>>>(p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_packed_similarity_tc(const uint32_t* H, int64_t ldw, int64_t N, int64_t D, const float* C,
                                        int64_t K, int32_t* labels, float* scores, int num_sms, cudaStream_t st) {
  if (K < 1 || K > 64 || N < 1) return cudaErrorInvalidValue;
  const int64_t Kp = K <= 16 ? 16 : K <= 32 ? 32 : 64;
  const int nchunks = (int)((D + kChunk - 1) / kChunk);
  const int64_t tiles = (N + 127) / 128;
  int DS = (int)((2 * (int64_t)num_sms + tiles - 1) / tiles);     // >= 2 CTAs per SM of work
  if (DS > nchunks) DS = nchunks;
  if (DS < 1) DS = 1;
  PackedTcParams p;
  p.H = H;
  p.ldw = ldw;
  p.N = N;
  p.D = D;
  p.K = K;
  p.Kp = Kp;
  p.nchunks = nchunks;
  p.DS = DS;
  p.cbytes = (uint32_t)(2 * Kp * kChunk * 2);
  p.labels = labels;
  p.scores = scores;
  uint8_t* ct = nullptr;
  unsigned long long* acc = nullptr;
  unsigned* cnt = nullptr;                         // [tiles] counters, then max |C|
  cudaError_t e = cudaMallocAsync((void**)&ct, (size_t)nchunks * p.cbytes, st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&acc, sizeof(unsigned long long) * N * Kp, st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&cnt, sizeof(unsigned) * (tiles + 1), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(acc, 0, sizeof(unsigned long long) * N * Kp, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(cnt, 0, sizeof(unsigned) * (tiles + 1), st);
  if (e == cudaSuccess) {
    c_absmax_kernel<<<148, 256, 0, st>>>(C, K * D, cnt + tiles);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) {
    const int64_t total = (int64_t)nchunks * 2 * Kp * kChunk;
    int64_t grid = (total + 255) / 256;
    if (grid > 148 * 16) grid = 148 * 16;
    c_chunk_tiles_kernel<<<(unsigned)grid, 256, 0, st>>>(C, K, Kp, D, nchunks, (__nv_bfloat16*)ct);
    e = cudaGetLastError();
  }
  p.ctiles = ct;
  p.acc = acc;
  p.cnt = cnt;
  p.cmax = cnt + tiles;
  if (e == cudaSuccess)
    e = Kp == 16 ? launch_kp<16>(p, tiles, st) : Kp == 32 ? launch_kp<32>(p, tiles, st) : launch_kp<64>(p, tiles, st);
  cudaFreeAsync(ct, st);
  cudaFreeAsync(acc, st);
  cudaFreeAsync(cnt, st);
  return e;
}

}  // namespace hdc
