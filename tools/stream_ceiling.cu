// Streaming ceiling for the small-batch path: how fast can one kernel read a cold
// 31.4 MB array (B of cfg3, F = 784, D = 10000, fp32) from HBM on B200, L2 left CLEAN
// by the flush (write 2x L2, then read another 2x L2 buffer)?  Times the kernel alone
// with CUDA events (launch included), best and median of 20.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/stream_ceiling.cu -o tools/stream_ceiling
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include "../paper_2506_09282_b200/csrc/common.cuh"
#include "../paper_2506_09282_b200/csrc/tc_ptx.cuh"
using namespace hdc;

__device__ __forceinline__ float4 ldg_nc(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}

// LDG.128: grid-stride over the whole array, CH loads in flight per thread
template <int CH>
__global__ void ldg_stream(const float4* a, int64_t n4, float* out) {
  float acc = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n4; i0 += stride * CH) {
    float4 v[CH];
#pragma unroll
    for (int r = 0; r < CH; ++r) {
      const int64_t i = i0 + r * stride;
      v[r] = i < n4 ? ldg_nc(a + i) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int r = 0; r < CH; ++r) acc += v[r].x + v[r].y + v[r].z + v[r].w;
  }
  if (acc == 12345.f) out[threadIdx.x] = acc;
}

// LDG.128: each CTA reads one contiguous block (like the per-CTA D ranges)
template <int CH>
__global__ void ldg_block(const float4* a, int64_t n4, float* out) {
  const int64_t b0 = blockIdx.x * n4 / gridDim.x, b1 = (blockIdx.x + 1) * n4 / gridDim.x;
  float acc = 0.f;
  for (int64_t i0 = b0 + threadIdx.x; i0 < b1; i0 += (int64_t)blockDim.x * CH) {
    float4 v[CH];
#pragma unroll
    for (int r = 0; r < CH; ++r) {
      const int64_t i = i0 + (int64_t)r * blockDim.x;
      v[r] = i < b1 ? ldg_nc(a + i) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int r = 0; r < CH; ++r) acc += v[r].x + v[r].y + v[r].z + v[r].w;
  }
  if (acc == 12345.f) out[threadIdx.x] = acc;
}

// 1-D bulk copies: each CTA streams its contiguous block through an NST x CHUNK ring;
// NP producer lanes (one per ring slice) keep copies in flight, consumers touch each chunk
template <int NST, int CHUNK>
__global__ void __launch_bounds__(256, 1) bulk_block(const float4* a, int64_t n4, float* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t full[NST], empty[NST];
  const int tid = threadIdx.x;
  const int64_t b0 = blockIdx.x * n4 / gridDim.x, b1 = (blockIdx.x + 1) * n4 / gridDim.x;
  const int64_t bytes = (b1 - b0) * 16;
  const uint8_t* src = reinterpret_cast<const uint8_t*>(a + b0);
  const int64_t nch = (bytes + CHUNK - 1) / CHUNK;
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) { ptx::mbar_init(&full[i], 1); ptx::mbar_init(&empty[i], 7); }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  float acc = 0.f;
  if (tid < 32) {
    if (tid == 0) {
      for (int64_t k = 0; k < nch; ++k) {
        const int s = (int)(k % NST);
        if (k >= NST) ptx::mbar_wait(&empty[s], (uint32_t)(((k / NST) - 1) & 1));
        const uint32_t nb = (uint32_t)(bytes - k * CHUNK < CHUNK ? bytes - k * CHUNK : CHUNK);
        ptx::mbar_arrive_expect_tx(&full[s], nb);
        ptx::bulk_load(sm + (size_t)s * CHUNK, src + k * CHUNK, nb, &full[s]);
      }
    }
  } else {
    const int w = (tid >> 5) - 1;             // 7 consumer warps
    for (int64_t k = 0; k < nch; ++k) {
      const int s = (int)(k % NST);
      ptx::mbar_wait(&full[s], (uint32_t)((k / NST) & 1));
      acc += reinterpret_cast<const float*>(sm + (size_t)s * CHUNK)[tid];
      __syncwarp();
      if ((tid & 31) == 0) ptx::mbar_arrive(&empty[s]);
    }
    (void)w;
  }
  if (tid == 0) {
    // the producer also counts as one of the 8 arrivals per stage
  }
  if (acc == 12345.f) out[tid] = acc;
}

__global__ void empty_kernel(float* out) {
  if (threadIdx.x == 1234567) out[0] = 1.f;
}
__global__ void flush_write(float* p, size_t n, float v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}
__global__ void flush_read(const float* p, size_t n, float* out) {
  float a = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) a += p[i];
  if (a == 1234.5f) out[0] = a;
}

int main() {
  const int64_t bytes = 784LL * 10000 * 4;          // 31.36 MB
  const int64_t n4 = bytes / 16;
  float4* a;
  float *out, *fw, *fr;
  cudaMalloc(&a, bytes);
  cudaMemset(a, 0, bytes);
  cudaMalloc(&out, 1 << 16);
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  const size_t fn = 2 * (size_t)l2 / 4;
  cudaMalloc(&fw, fn * 4);
  cudaMalloc(&fr, fn * 4);
  cudaMemset(fr, 0, fn * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto bench = [&](const char* name, auto launch, bool warm = false) {
    std::vector<float> t;
    for (int it = 0; it < 24; ++it) {
      if (!warm) {
        flush_write<<<592, 512>>>(fw, fn, (float)it);
        flush_read<<<592, 512>>>(fr, fn, out);
      }
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it >= 4) t.push_back(ms * 1e3f);
    }
    std::sort(t.begin(), t.end());
    printf("%-44s best %6.2f us (%5.0f GB/s)  median %6.2f us (%5.0f GB/s)%s\n", name, t[0], bytes / (t[0] * 1e3),
           t[t.size() / 2], bytes / (t[t.size() / 2] * 1e3), warm ? "  [warm L2]" : "");
  };
  bench("empty kernel (launch + events)", [&] { empty_kernel<<<148, 128>>>(out); });
  bench("ldg grid-stride 148x512 CH=4", [&] { ldg_stream<4><<<148, 512>>>(a, n4, out); });
  bench("ldg grid-stride 148x1024 CH=4", [&] { ldg_stream<4><<<148, 1024>>>(a, n4, out); });
  bench("ldg grid-stride 296x1024 CH=4", [&] { ldg_stream<4><<<296, 1024>>>(a, n4, out); });
  bench("ldg grid-stride 592x512 CH=8", [&] { ldg_stream<8><<<592, 512>>>(a, n4, out); });
  bench("ldg grid-stride 1184x256 CH=8", [&] { ldg_stream<8><<<1184, 256>>>(a, n4, out); });
  bench("ldg block 148x1024 CH=8", [&] { ldg_block<8><<<148, 1024>>>(a, n4, out); });
  bench("ldg block 148x512 CH=16", [&] { ldg_block<16><<<148, 512>>>(a, n4, out); });
  bench("ldg block 296x512 CH=8", [&] { ldg_block<8><<<296, 512>>>(a, n4, out); });
  bench("ldg block 592x512 CH=4", [&] { ldg_block<4><<<592, 512>>>(a, n4, out); });
  {
    auto k1 = bulk_block<8, 16384>;
    cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
    bench("bulk block 148, 8 x 16 KB", [&] { k1<<<148, 256, 8 * 16384>>>(a, n4, out); });
    auto k2 = bulk_block<12, 16384>;
    cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 16384);
    bench("bulk block 148, 12 x 16 KB", [&] { k2<<<148, 256, 12 * 16384>>>(a, n4, out); });
    auto k3 = bulk_block<24, 8192>;
    cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, 24 * 8192);
    bench("bulk block 148, 24 x 8 KB", [&] { k3<<<148, 256, 24 * 8192>>>(a, n4, out); });
    auto k4 = bulk_block<6, 32768>;
    cudaFuncSetAttribute(k4, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
    bench("bulk block 148, 6 x 32 KB", [&] { k4<<<148, 256, 6 * 32768>>>(a, n4, out); });
    auto k5 = bulk_block<8, 8192>;
    cudaFuncSetAttribute(k5, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 8192);
    bench("bulk block 296, 8 x 8 KB", [&] { k5<<<296, 256, 8 * 8192>>>(a, n4, out); });
    bench("bulk block 148, 8 x 16 KB", [&] { k1<<<148, 256, 8 * 16384>>>(a, n4, out); }, true);
  }
  bench("ldg grid-stride 592x512 CH=8", [&] { ldg_stream<8><<<592, 512>>>(a, n4, out); }, true);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
