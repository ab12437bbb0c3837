// Microbenchmark: back-to-back tcgen05.mma issue rate for the tile shapes the
// fused kernel uses (diagnostic tool, not part of libhdc).
#include <cstdio>
#include <cstdint>
#include "../paper_2506_09282_b200/csrc/tc_ptx.cuh"
using namespace hdc::ptx;

template <int KIND, int N, int SWZ, int SBO, bool INTERLEAVED = false>
__global__ void bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
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
      else
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

template <int KIND, int N, int SWZ, int SBO, bool IL = false>
void run(const char* name, int blocks) {
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * blocks);
  auto k = bench<KIND, N, SWZ, SBO, IL>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  const int iters = 4000;
  k<<<blocks, 128, 70000>>>(iters, d);
  k<<<blocks, 128, 70000>>>(iters, d);
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
  for (int blocks : {148}) {
    run<0, 32, 0, 0, true>("bf16 N=32 interleaved", blocks);
    run<0, 64, 0, 0, true>("bf16 N=64 interleaved", blocks);
    run<0, 32, 2, 1024>("bf16 N=32 SW128", blocks);
    run<0, 16, 2, 1024>("bf16 N=16 SW128", blocks);
    run<0, 80, 2, 1024>("bf16 N=80  SW128", blocks);
    run<0, 160, 2, 1024>("bf16 N=160 SW128", blocks);
    run<0, 256, 2, 1024>("bf16 N=256 SW128", blocks);
    run<0, 80, 4, 512>("bf16 N=80  SW64", blocks);
    run<0, 256, 4, 512>("bf16 N=256 SW64", blocks);
    run<1, 80, 2, 1024>("tf32 N=80  SW128", blocks);
    run<1, 256, 2, 1024>("tf32 N=256 SW128", blocks);
    run<2, 80, 4, 512>("i8 N=80  SW64", blocks);
    run<2, 160, 4, 512>("i8 N=160 SW64", blocks);
    run<2, 240, 4, 512>("i8 N=240 SW64", blocks);
    run<2, 256, 4, 512>("i8 N=256 SW64", blocks);
    run<2, 80, 2, 1024>("i8 N=80  SW128", blocks);
    run<2, 240, 2, 1024>("i8 N=240 SW128", blocks);
    run<2, 256, 2, 1024>("i8 N=256 SW128", blocks);
  }
  return 0;
}
