// Microbenchmark: back-to-back tcgen05.mma issue rate for the tile shapes the
// fused kernel uses (diagnostic tool, not part of libhdc).
#include <cstdio>
#include <cstdint>
#include "../paper_2506_09282_b200/csrc/tc_ptx.cuh"
using namespace hdc::ptx;

template <int KIND, int N, int SWZ, int SBO, bool INTERLEAVED = false, bool VARY = false>
__global__ void bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  for (int i = threadIdx.x; i < 196608 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    constexpr uint32_t idesc = make_idesc<KIND>(128, N);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t ks = (i & 1) * 32;
      if (INTERLEAVED)
        tc_mma<KIND>(tb, smem_desc_interleaved(a + (i % 5) * 256, 128, 1280),
                     smem_desc_interleaved(b + (i % 5) * 256, 128, 1280), idesc, 1u);
      else if (VARY) {   // distinct operand tiles every MMA: A in [0,96K), B in [96K, 192K)
        const uint32_t aoff = (uint32_t)((i % 6) * 16384 + ((i / 6) & 3) * 32);
        const uint32_t boff = (uint32_t)(98304 + (i % 3) * 32768 + ((i / 3) & 3) * 32);
        tc_mma<KIND>(tb, smem_desc_sw(smem_u32(smem) + aoff, SBO, SWZ),
                     smem_desc_sw(smem_u32(smem) + boff, SBO, SWZ), idesc, 1u);
      } else
        tc_mma<KIND>(tb, smem_desc_sw(a + ks, SBO, SWZ), smem_desc_sw(b + ks, SBO, SWZ), idesc, 1u);
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tb);
}

template <int KIND, int N, int SWZ, int SBO, bool IL = false, bool VARY = false>
void run(const char* name, int blocks) {
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * blocks);
  auto k = bench<KIND, N, SWZ, SBO, IL, VARY>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  const int iters = 4000;
  k<<<blocks, 128, 200000>>>(iters, d);
  k<<<blocks, 128, 200000>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(unsigned long long) * blocks, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < blocks; ++i) avg += h[i];
  avg /= blocks;
  const double kelem = KIND == 0 ? 16 : (KIND == 1 ? 8 : 32);
  const double macs = 128.0 * N * kelem;
  printf("%-28s blocks=%3d cycles/mma=%7.1f  MAC/clk/SM=%7.0f  err=%s\n", name, blocks, avg / iters,
         macs * iters / avg, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  const int blocks = 148;
  run<0, 80, 2, 1024, false, false>("bf16 N=80  same tiles", blocks);
  run<0, 80, 2, 1024, false, true>("bf16 N=80  distinct tiles", blocks);
  run<0, 160, 2, 1024, false, true>("bf16 N=160 distinct tiles", blocks);
  run<0, 256, 2, 1024, false, true>("bf16 N=256 distinct tiles", blocks);
  run<2, 80, 4, 512, false, true>("i8 N=80 SW64 distinct", blocks);
  run<2, 160, 4, 512, false, true>("i8 N=160 SW64 distinct", blocks);
  run<2, 240, 4, 512, false, true>("i8 N=240 SW64 distinct", blocks);
  run<2, 256, 4, 512, false, true>("i8 N=256 SW64 distinct", blocks);
  run<2, 240, 2, 1024, false, true>("i8 N=240 SW128 distinct", blocks);
  run<0, 32, 0, 0, true, false>("bf16 N=32 interleaved", blocks);
  return 0;
}
