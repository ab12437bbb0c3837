// Microbenchmark: streaming B (F x Dp fp32) column slices as the small-batch
// kernel does, to separate memory behaviour from the kernel's other phases.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include "../paper_2506_09282_b200/csrc/common.cuh"
#include "../paper_2506_09282_b200/csrc/tc_ptx.cuh"
using namespace hdc;

template <int CH, bool NC>
__global__ void __launch_bounds__(256, 1) colstream(const float* B, int64_t F, int64_t Dp, int64_t units, float* out) {
  const int tid = threadIdx.x, c = blockIdx.x, G = gridDim.x;
  const int64_t u0 = (int64_t)c * units / G, u1 = (int64_t)(c + 1) * units / G;
  const int PW = (int)(u1 - u0), RG = 256 / PW, g = tid / PW, u = tid % PW;
  float acc = 0.f;
  if (g < RG) {
    const float* bcol = B + (u0 + u) * 4;
    for (int64_t f0 = g; f0 < F; f0 += (int64_t)RG * CH) {
      float4 v[CH];
#pragma unroll
      for (int r = 0; r < CH; ++r) {
        const int64_t f = f0 + (int64_t)r * RG;
        if (NC) v[r] = f < F ? ldg_stream(bcol + f * Dp) : make_float4(0, 0, 0, 0);
        else v[r] = f < F ? *reinterpret_cast<const float4*>(bcol + f * Dp) : make_float4(0, 0, 0, 0);
      }
#pragma unroll
      for (int r = 0; r < CH; ++r) acc += v[r].x + v[r].y + v[r].z + v[r].w;
    }
  }
  if (acc == 12345.f) out[tid] = acc;
}

// unit-major layout: B4[u][f][4] (all F rows of a 4-column unit contiguous)
template <int CH>
__global__ void __launch_bounds__(256, 1) unitstream(const float* B4, int64_t F, int64_t Dp, int64_t units, float* out) {
  const int tid = threadIdx.x, c = blockIdx.x, G = gridDim.x;
  const int64_t u0 = (int64_t)c * units / G, u1 = (int64_t)(c + 1) * units / G;
  const int PW = (int)(u1 - u0), RG = 256 / PW, g = tid / PW, u = tid % PW;
  float acc = 0.f;
  if (g < RG) {
    const float* base = B4 + (u0 + u) * F * 4;
    for (int64_t f0 = g; f0 < F; f0 += (int64_t)RG * CH) {
      float4 v[CH];
#pragma unroll
      for (int r = 0; r < CH; ++r) {
        const int64_t f = f0 + (int64_t)r * RG;
        v[r] = f < F ? ldg_stream(base + f * 4) : make_float4(0, 0, 0, 0);
      }
#pragma unroll
      for (int r = 0; r < CH; ++r) acc += v[r].x + v[r].y + v[r].z + v[r].w;
    }
  }
  if (acc == 12345.f) out[tid] = acc;
}

// unit-major, thread reads consecutive rows of its unit (g-th contiguous block)
template <int CH>
__global__ void __launch_bounds__(256, 1) unitstream2(const float* B4, int64_t F, int64_t Dp, int64_t units, float* out) {
  const int tid = threadIdx.x, c = blockIdx.x, G = gridDim.x;
  const int64_t u0 = (int64_t)c * units / G, u1 = (int64_t)(c + 1) * units / G;
  const int64_t total = (u1 - u0) * F;           // float4 elements of this CTA, contiguous
  const float4* base = reinterpret_cast<const float4*>(B4 + u0 * F * 4);
  float acc = 0.f;
  for (int64_t i0 = tid; i0 < total; i0 += 256 * CH) {
    float4 v[CH];
#pragma unroll
    for (int r = 0; r < CH; ++r) {
      const int64_t i = i0 + (int64_t)r * 256;
      v[r] = i < total ? ldg_stream(reinterpret_cast<const float*>(base + i)) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int r = 0; r < CH; ++r) acc += v[r].x + v[r].y + v[r].z + v[r].w;
  }
  if (acc == 12345.f) out[tid] = acc;
}

// TMA bulk copies (1-D) of the CTA's contiguous region into a smem ring.
template <int NST, int CHUNK>
__global__ void __launch_bounds__(128, 1) bulkstream(const float* B4, int64_t F, int64_t Dp, int64_t units, float* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar[NST];
  const int tid = threadIdx.x, c = blockIdx.x, G = gridDim.x;
  const int64_t u0 = (int64_t)c * units / G, u1 = (int64_t)(c + 1) * units / G;
  const int64_t bytes = (u1 - u0) * F * 16;
  const uint8_t* src = reinterpret_cast<const uint8_t*>(B4 + u0 * F * 4);
  const int64_t nchunks = (bytes + CHUNK - 1) / CHUNK;
  if (tid == 0) { for (int i = 0; i < NST; ++i) hdc::ptx::mbar_init(&bar[i], 1); hdc::ptx::fence_mbar_init(); }
  __syncthreads();
  float acc = 0.f;
  if (tid == 0) {
    for (int64_t k = 0; k < nchunks && k < NST; ++k) {
      const uint32_t nb = (uint32_t)(bytes - k * CHUNK < CHUNK ? bytes - k * CHUNK : CHUNK);
      hdc::ptx::mbar_arrive_expect_tx(&bar[k], nb);
      hdc::ptx::bulk_load(sm + k * CHUNK, src + k * CHUNK, nb, &bar[k]);
    }
  }
  for (int64_t k = 0; k < nchunks; ++k) {
    const int s = (int)(k % NST);
    hdc::ptx::mbar_wait(&bar[s], (uint32_t)((k / NST) & 1));
    acc += reinterpret_cast<const float*>(sm + s * CHUNK)[tid];
    __syncthreads();
    if (tid == 0 && k + NST < nchunks) {
      const int64_t kk = k + NST;
      const uint32_t nb = (uint32_t)(bytes - kk * CHUNK < CHUNK ? bytes - kk * CHUNK : CHUNK);
      hdc::ptx::mbar_arrive_expect_tx(&bar[s], nb);
      hdc::ptx::bulk_load(sm + s * CHUNK, src + kk * CHUNK, nb, &bar[s]);
    }
  }
  if (acc == 12345.f) out[tid] = acc;
}

__global__ void flush(float* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] += 1.f;
}
__global__ void flush_read(const float* p, size_t n, float* out) {
  float a = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) a += p[i];
  if (a == 1234.5f) out[0] = a;
}
static int g_read_flush = 0;

int main(int argc, char** argv) {
  const int64_t F = argc > 1 ? atoll(argv[1]) : 784, D = 10000, Dp = 10240;
  float *B, *out, *fl;
  cudaMalloc(&B, F * Dp * 4);
  cudaMemset(B, 0, F * Dp * 4);
  cudaMalloc(&out, 4096);
  const size_t fn = 64 << 20;  // 256 MB flush buffer
  cudaMalloc(&fl, fn * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto bench = [&](const char* name, auto kern, int grid, int threads = 256, int smem = 0) {
    float best = 1e9, tot = 0;
    for (int it = 0; it < 12; ++it) {
      flush<<<1184, 256>>>(fl, fn);
      if (g_read_flush) flush_read<<<1184, 256>>>(fl + fn / 2, fn / 2, out);
      cudaEventRecord(e0);
      kern<<<grid, threads, smem>>>(B, F, Dp, (D + 3) / 4, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it >= 2) { best = ms < best ? ms : best; tot += ms; }
    }
    const double bytes = (double)F * D * 4;
    printf("%-32s grid=%4d best %.2f us (%.0f GB/s)  mean %.2f us\n", name, grid, best * 1e3,
           bytes / (best * 1e-3) / 1e9, tot / 10 * 1e3);
  };
  for (int rf = 0; rf < 2; ++rf) {
  g_read_flush = rf;
  printf("---- flush: write 256 MB%s\n", rf ? " + read 128 MB (clean L2)" : "");
  bench("nc CH=8", colstream<8, true>, 148);
  bench("nc CH=16", colstream<16, true>, 148);
  bench("nc CH=32", colstream<32, true>, 148);
  bench("nc CH=52 (all)", colstream<52, true>, 148);
  bench("plain CH=16", colstream<16, false>, 148);
  bench("nc CH=16 grid 296", colstream<16, true>, 296);
  bench("nc CH=16 grid 592", colstream<16, true>, 592);
  bench("unit-major CH=16", unitstream<16>, 148);
  bench("unit-major CH=32", unitstream<32>, 148);
  bench("unit-major contiguous CH=8", unitstream2<8>, 148);
  bench("unit-major contiguous CH=16", unitstream2<16>, 148);
  bench("unit-major contiguous CH=16 g296", unitstream2<16>, 296);
  }
  cudaFuncSetAttribute(bulkstream<4, 49152>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 49152);
  cudaFuncSetAttribute(bulkstream<8, 24576>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 24576);
  cudaFuncSetAttribute(bulkstream<6, 32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
  bench("bulk 4 x 48KB", bulkstream<4, 49152>, 148, 128, 4 * 49152);
  bench("bulk 8 x 24KB", bulkstream<8, 24576>, 148, 128, 8 * 24576);
  bench("bulk 6 x 32KB", bulkstream<6, 32768>, 148, 128, 6 * 32768);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
