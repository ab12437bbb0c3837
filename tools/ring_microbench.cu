// Microbenchmark: producer/MMA mbarrier ring exactly as in the fused kernel,
// without data movement (diagnostic tool).
#include <cstdio>
#include <cstdint>
#include "../paper_2506_09282_b200/csrc/tc_ptx.cuh"
using namespace hdc::ptx;

template <int STAGES, int NMMA, int N, int VARIANT, int SPIN = 0>
__global__ void ring(int iters, unsigned long long* out) {
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
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (warp == 1) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = slot;
  long long t0 = clock64();
  if (warp == 0) {
    if (VARIANT == 1 || lane == 0) {
      int s = 0; uint32_t ph = 0;
      for (int i = 0; i < iters; ++i) {
        mbar_wait(&empty[s], ph ^ 1);
        if (VARIANT == 1) { if (lane == 0) mbar_arrive(&full[s]); } else mbar_arrive(&full[s]);
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    constexpr uint32_t idesc = make_idesc<0>(128, N);
    int s = 0; uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&full[s], ph);
      tc_fence_after();
#pragma unroll
      for (int k = 0; k < NMMA; ++k)
        tc_mma_elect<0>(tb, smem_desc_sw(a + (k & 3) * 32, 1024, 2), smem_desc_sw(b + (k & 3) * 32, 1024, 2), idesc, 1u);
      tc_commit_elect(&empty[s]);
      if (++s == STAGES) { s = 0; ph ^= 1; }
    }
    tc_commit_elect(&done);
    mbar_wait(&done, 0);
    if (lane == 0) out[blockIdx.x] = (unsigned long long)(clock64() - t0);
  }
  else if (warp >= 4 && SPIN) {
    if (SPIN == 1) mbar_wait(&done, 0);            // spin without suspend hint
    else {
      const uint32_t a = smem_u32(&done);
      asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, 1000000;\n\t@!P1 bra W_%=;\n\t}" ::"r"(a), "r"(0) : "memory");
    }
  }
  __syncwarp();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tb);
}

template <int STAGES, int NMMA, int N, int VARIANT, int SPIN = 0, int THREADS = 128>
void run(const char* name) {
  const int blocks = 148, iters = 2000;
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * blocks);
  auto k = ring<STAGES, NMMA, N, VARIANT, SPIN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  k<<<blocks, THREADS, 70000>>>(iters, d);
  k<<<blocks, THREADS, 70000>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < blocks; ++i) avg += h[i];
  avg /= blocks;
  const double mma_cyc = (N <= 80 ? 52.0 : N / 2.0) * NMMA;
  printf("%-36s cycles/stage=%7.1f  (pure MMA %5.0f)  eff=%.2f err=%s\n", name, avg / iters, mma_cyc,
         mma_cyc / (avg / iters), cudaGetErrorString(e));
}

int main() {
  run<5, 4, 80, 0>("5 stages, 4 x N=80");
  run<5, 4, 80, 1>("5 stages, 4 x N=80, prod whole warp");
  run<4, 4, 160, 0>("4 stages, 4 x N=160");
  run<4, 4, 240, 0>("4 stages, 4 x N=240");
  run<4, 8, 80, 0>("4 stages, 8 x N=80");
  run<4, 8, 240, 0>("4 stages, 8 x N=240");
  run<8, 4, 80, 0>("8 stages, 4 x N=80");
  run<3, 6, 240, 0>("3 stages, 6 x N=240");
  run<5, 4, 80, 0, 1, 640>("5st 4xN80 + 16 spinning warps");
  run<5, 4, 80, 0, 2, 640>("5st 4xN80 + 16 suspended warps");
  run<4, 6, 240, 0, 1, 640>("4st 6xN240 + 16 spinning warps");
  run<4, 6, 240, 0, 2, 640>("4st 6xN240 + 16 suspended warps");
  return 0;
}
