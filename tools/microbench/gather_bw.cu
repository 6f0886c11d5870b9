// Microbenchmark: random 512-byte row gather bandwidth on B200 (the access
// pattern of the epoch kernel's neighbour rows), vs a sequential copy.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bw gather_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void gather(const float4* __restrict__ z, const uint32_t* __restrict__ idx,
                       uint64_t m, float* out, int inflight) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  float acc = 0.f;
  for (uint64_t i = w * 16; i < m; i += nw * 16) {
    float4 v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (k < inflight) v[k] = __ldg(z + uint64_t(idx[i + k]) * 32 + lane);
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (k < inflight) acc += v[k].x + v[k].y + v[k].z + v[k].w;
  }
  if (acc == 1234.5f) out[0] = acc;
}

__global__ void copy(const float4* __restrict__ a, float4* __restrict__ b, uint64_t n) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    b[i] = a[i];
}

int main() {
  const uint64_t rows = 3000000, d = 128;  // C3's Z: 1.5 GB
  const uint64_t m = 64ull << 20;          // 64 Mi row gathers (32 GB)
  float4* z;
  uint32_t* idx;
  float* out;
  cudaMalloc(&z, rows * d * 4);
  cudaMalloc(&idx, (m + 16) * 4);
  cudaMalloc(&out, 4);
  cudaMemset(z, 0, rows * d * 4);
  uint32_t* h = new uint32_t[m + 16];
  uint64_t s = 88172645463325252ull;
  for (uint64_t i = 0; i < m + 16; ++i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    h[i] = uint32_t(s % rows);
  }
  cudaMemcpy(idx, h, (m + 16) * 4, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int inflight : {1, 2, 4, 8, 16}) {
    for (int wps : {16, 32, 48, 64}) {  // warps per SM
      const int blocks = sms * (wps / 8);
      gather<<<blocks, 256>>>(z, idx, m, out, inflight);
      cudaEventRecord(e0);
      gather<<<blocks, 256>>>(z, idx, m, out, inflight);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      // rows actually gathered: inflight of every 16
      const double bytes = double(m) * inflight / 16 * 512;
      printf("gather inflight %2d warps/SM %2d: %.0f GB/s\n", inflight, wps, bytes / ms / 1e6);
    }
  }
  float4* b;
  cudaMalloc(&b, rows * d * 4);
  copy<<<sms * 8, 256>>>(z, b, rows * d / 4);
  cudaEventRecord(e0);
  copy<<<sms * 8, 256>>>(z, b, rows * d / 4);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("copy: %.0f GB/s (read+write)\n", 2.0 * rows * d * 4 / ms / 1e6);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
