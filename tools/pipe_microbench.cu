// Microbenchmark: cost of the MMA-warp bookkeeping (tcgen05.commit, mbarrier
// waits) around tcgen05.mma, single CTA per SM (diagnostic tool).
#include <cstdio>
#include <cstdint>
#include "../paper_2506_09282_b200/csrc/tc_ptx.cuh"
using namespace hdc::ptx;

template <int MODE>
__global__ void bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t slot;
  __shared__ uint64_t bar[8];
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1); fence_mbar_init(); }
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    constexpr uint32_t idesc = make_idesc<0>(128, 80);
    long long t0 = clock64();
    uint32_t ph[8] = {0,0,0,0,0,0,0,0};
    for (int i = 0; i < iters; ++i) {
      const int s = i % 5;
      if (MODE == 6 || MODE == 7) {     // full[s]: arrive then wait (already complete), as the MMA warp does
        mbar_arrive(&bar[s]);
        mbar_wait(&bar[s], ph[s]);
        ph[s] ^= 1;
        if (MODE == 6) tc_fence_after();
      }
      if (MODE >= 1 && MODE != 5) {
        for (int k = 0; k < 4; ++k)
          tc_mma<0>(tb, smem_desc_sw(a + k * 32, 1024, 2), smem_desc_sw(b + k * 32, 1024, 2), idesc, 1u);
      }
      if (MODE != 1 && MODE != 6 && MODE != 7) tc_commit(&bar[s]);
      if (MODE == 6 || MODE == 7) tc_commit(&bar[5]);
      if (MODE == 4 || MODE == 5) {   // latency: wait for this iteration's own commit
        mbar_wait(&bar[s], ph[s]);
        ph[s] ^= 1;
      }
      if (MODE == 3 && i >= 4) {   // wait for the commit issued 4 iterations ago (ring of 5)
        const int w = (i - 4) % 5;
        mbar_wait(&bar[w], ph[w]);
        ph[w] ^= 1;
      }
    }
    tc_commit(&bar[7]);
    mbar_wait(&bar[7], 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tb);
}

template <int MODE>
void run(const char* name) {
  const int blocks = 148, iters = 2000;
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * blocks);
  cudaFuncSetAttribute(bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  bench<MODE><<<blocks, 128, 70000>>>(iters, d);
  bench<MODE><<<blocks, 128, 70000>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < blocks; ++i) avg += h[i];
  avg /= blocks;
  printf("%-40s cycles/iter=%7.1f err=%s\n", name, avg / iters, cudaGetErrorString(e));
}

int main() {
  run<0>("commit only");
  run<1>("4 MMA (N=80) no commit");
  run<2>("4 MMA + commit");
  run<3>("4 MMA + commit + wait(i-4)");
  run<4>("4 MMA + commit + wait(own) [latency]");
  run<5>("commit + wait(own) [latency]");
  run<6>("wait(done)+fence_after+4MMA+commit");
  run<7>("wait(done)+4MMA+commit (no fence)");
  return 0;
}
