// Microbenchmark: the K4 producer / MMA-issuer loop structure (tiles x stages, per-tile
// tfull commit and 64-bit tile-index division) with no data movement and no MMA, to
// compare with ring2's flat loop (diagnostic tool).
#include <cstdio>
#include <cstdint>
#include "../paper_2506_09282_b200/csrc/tc_ptx.cuh"
using namespace hdc::ptx;

struct P { int64_t T, TdG; int G; int KB; };

template <int VAR>
__global__ void __launch_bounds__(384, 1) ring3(const P p, unsigned long long* out) {
  constexpr int STAGES = 5;
  __shared__ uint32_t slot;
  __shared__ uint64_t full[8], empty[8], tfull[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(&tfull[0], 1); mbar_init(&tfull[1], 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const int c = blockIdx.x;
  const int64_t t0 = (int64_t)c * p.T / p.G, t1 = (int64_t)(c + 1) * p.T / p.G;
  long long c0 = clock64();
  if (warp == 0) {
    if (lane == 0) {
      int s = 0; uint32_t ph = 0;
      int acc = 0;
      for (int64_t t = t0; t < t1; ++t) {
        if (VAR & 1) acc += (int)(t / p.TdG) + (int)(t % p.TdG);   // per-tile 64-bit div
        for (int kb = 0; kb < p.KB; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive(&full[s]);
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
      if (acc == 123456789) out[1000] = acc;
    }
  } else if (warp == 1) {
    int s = 0; uint32_t ph = 0; int buf = 0;
    for (int64_t t = t0; t < t1; ++t) {
      for (int kb = 0; kb < p.KB; ++kb) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        tc_commit_elect(&empty[s]);
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
      if (VAR & 2) tc_commit_elect(&tfull[buf]);
      buf ^= 1;
    }
    if (lane == 0) out[c] = (unsigned long long)(clock64() - c0);
  }
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(slot);
}

template <int VAR>
void run(const char* name, int G, int64_t T, int64_t TdG, int KB, int smem = 0) {
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * 2048);
  P p{T, TdG, G, KB};
  cudaFuncSetAttribute(ring3<VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 230000);
  ring3<VAR><<<G, 384, smem>>>(p, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  ring3<VAR><<<G, 384, smem>>>(p, d);
  cudaEventRecord(e1);
  cudaError_t e = cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < G; ++i) avg += h[i]; avg /= G;
  const double stages = (double)T / G * KB;
  printf("%-36s %.3f ms, %.0f cycles/stage  err=%s\n", name, ms, avg / stages, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  // cfg2 bf16 geometry: 128 N-tiles x 63 D-tiles, 10 stages per tile, 148 CTAs
  run<0>("flat tiles", 148, 128 * 63, 63, 10);
  run<1>("+ per-tile 64-bit div", 148, 128 * 63, 63, 10);
  run<2>("+ per-tile tfull commit", 148, 128 * 63, 63, 10);
  run<3>("+ both", 148, 128 * 63, 63, 10);
  run<3>("+ both, 220 KB dynamic smem", 148, 128 * 63, 63, 10, 220 * 1024);
  return 0;
}
