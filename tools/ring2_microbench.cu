// Microbenchmark: the K4 bf16 MMA-warp loop (5-stage ring of distinct SW128 operand
// tiles, 4 x M128 N160 K16 MMAs per stage, commit per stage, accumulator buffer
// alternating every 10 stages) with no data movement -- isolates MMA issue cost.
#include <cstdio>
#include <cstdint>
#include "../paper_2506_09282_b200/csrc/tc_ptx.cuh"
using namespace hdc::ptx;

template <int N, int VARIANT, bool RANDOM = false, int NT = 128, int DELAY = 0>   // VARIANT 0: elect-issue (kernel), 1: lane-0 issue, 2: elect, fixed D,
                                                     // 3: no MMA (commit only), 4: no MMA, plain arrive
__global__ void __launch_bounds__(NT, 1) ring2(int iters, unsigned long long* out) {
  // DELAY: dependent integer ops the MMA warp executes per stage after its commit
  // (probes how much per-stage issue work the tensor-core queue hides)
  constexpr int STAGES = 5, A_ST = 16384, B_ST = N * 128;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t slot;
  __shared__ uint64_t full[8], empty[8], done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < (STAGES * (A_ST + B_ST)) / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u + blockIdx.x * 97u;   // random-ish bf16 pairs, |v| ~ 1
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    const uint32_t v = RANDOM ? ((h & 0x807F807Fu) | 0x3F003F00u) : 0u;
    reinterpret_cast<uint32_t*>(smem)[i] = v;
  }
  if (warp == 1) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = slot;
  long long t0 = clock64();
  unsigned long long g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  if (warp == 0) {
    if (lane == 0) {
      int s = 0; uint32_t ph = 0;
      for (int i = 0; i < iters; ++i) {
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive(&full[s]);
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = make_idesc<0>(128, N);
    int s = 0; uint32_t ph = 0;
    if (VARIANT == 1 && lane != 0) goto skip;
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&full[s], ph);
      tc_fence_after();
      const uint32_t a = smem_u32(smem + s * A_ST), b = smem_u32(smem + STAGES * A_ST + s * B_ST);
      const uint32_t d = (VARIANT == 2) ? tb : tb + ((i / 10) & 1) * N;
      if (VARIANT == 5) {   // the K4 kernel's form: base descriptor + offset, 4 MMAs under one elect
        const uint64_t a_d = smem_desc_sw(smem_u32(smem), 1024, 2) + (uint64_t)((s * A_ST) >> 4);
        const uint64_t b_d = smem_desc_sw(smem_u32(smem + STAGES * A_ST), 1024, 2) + (uint64_t)((s * B_ST) >> 4);
        tc_mma4_elect<0>(d, a_d, b_d, a_d + 2, b_d + 2, a_d + 4, b_d + 4, a_d + 6, b_d + 6, idesc,
                         (i % 10 == 0) ? 0u : 1u);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (VARIANT >= 3) continue;
        if (VARIANT == 1)
          tc_mma<0>(d, smem_desc_sw(a + k * 32, 1024, 2), smem_desc_sw(b + k * 32, 1024, 2), idesc, (i % 10 == 0 && k == 0) ? 0u : 1u);
        else
          tc_mma_elect<0>(d, smem_desc_sw(a + k * 32, 1024, 2), smem_desc_sw(b + k * 32, 1024, 2), idesc, (i % 10 == 0 && k == 0) ? 0u : 1u);
      }
      if (VARIANT == 1) tc_commit(&empty[s]);
      else if (VARIANT == 4) { __syncwarp(); if (lane == 0) mbar_arrive(&empty[s]); }
      else tc_commit_elect(&empty[s]);
      if (DELAY) {
        uint32_t x = (uint32_t)i;
#pragma unroll 1
        for (int j = 0; j < DELAY; ++j) x = x * 1664525u + 1013904223u;
        if (x == 0x12345678u) out[1000 + blockIdx.x] = x;
      }
      if (++s == STAGES) { s = 0; ph ^= 1; }
    }
    if (VARIANT == 1) tc_commit(&done); else tc_commit_elect(&done);
    mbar_wait(&done, 0);
    unsigned long long g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    if (lane == 0) { out[blockIdx.x] = (unsigned long long)(clock64() - t0); out[148 + blockIdx.x] = g1 - g0; }
  skip:;
  }
  __syncwarp();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tb);
}

template <int N, int VARIANT, bool RANDOM = false, int NT = 128, int DELAY = 0>
void run(const char* name, int iters = 4000) {
  const int blocks = 148;
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * blocks * 2);
  auto k = ring2<N, VARIANT, RANDOM, NT, DELAY>;
  const int sm = 5 * (16384 + N * 128) + 2048;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  k<<<blocks, NT, sm>>>(iters, d);
  k<<<blocks, NT, sm>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[296];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0, ns = 0;
  for (int i = 0; i < blocks; ++i) { avg += h[i]; ns += h[148 + i]; }
  avg /= blocks; ns /= blocks;
  printf("%-40s cycles/MMA(stage/4)=%7.1f  ns/MMA=%7.2f  clock=%.0f MHz  err=%s\n", name, avg / iters / 4,
         ns / iters / 4, 1e3 * avg / ns, cudaGetErrorString(e));
}

int main() {
  run<160, 5>("N=160 K4-style mma4 (base+offset descriptors)");
  run<160, 5, true>("N=160 K4-style mma4, random data");
  run<160, 0>("N=160 elect, delay 0");
  run<160, 0, false, 128, 16>("N=160 elect, delay 16 dep-ops/stage");
  run<160, 0, false, 128, 32>("N=160 elect, delay 32 dep-ops/stage");
  run<160, 0, false, 128, 64>("N=160 elect, delay 64 dep-ops/stage");
  run<160, 0, false, 128, 128>("N=160 elect, delay 128 dep-ops/stage");
  run<160, 3, false, 128, 64>("no MMA, delay 64 dep-ops/stage");
  return 0;
}
