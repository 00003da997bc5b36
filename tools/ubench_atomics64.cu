// Microbenchmark 3: red.shared.add.u64 (two packed 32-bit fixed-point fields
// per atomic) vs red.shared.add.s32, P2G box pattern (lanes = 2x4x4 cells).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_atomics64 ubench_atomics64.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int V, int SI>
__global__ void __launch_bounds__(256) scat(const uint32_t* __restrict__ seeds, float* out, int iters) {
  constexpr int FS = 8 * SI + 8;  // elements per field
  __shared__ __align__(16) unsigned long long ar[4 * FS];
  int* ar32 = reinterpret_cast<int*>(ar);
  for (int i = threadIdx.x; i < 4 * FS; i += blockDim.x) ar[i] = 0;
  __syncthreads();
  uint32_t s = seeds[blockIdx.x * blockDim.x + threadIdx.x];
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int ci = (warp & 1) * 2 + (lane >> 4) + 1, cj = ((lane >> 2) & 3) + 1, ck = (lane & 3) + 1;
  for (int it = 0; it < iters; ++it) {
    s = s * 1664525u + 1013904223u;
    float d = (s & 255) * (1.f / 256.f);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          int n = (ck + k) + 8 * (cj + j) + SI * (ci + i);
          float w = d * (i + 1) * (j + 2) * (k + 3);
          if (V == 0) {  // 8 x 32-bit
#pragma unroll
            for (int f = 0; f < 8; ++f) {
              int v = __float_as_int(w * (f + 1) * 1024.f + 12582912.f);
              unsigned a = (unsigned)__cvta_generic_to_shared(&ar32[f * 2 * FS + n]);
              asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
            }
          } else {  // 4 x 64-bit (two fields each)
#pragma unroll
            for (int f = 0; f < 4; ++f) {
              uint32_t lo = __float_as_uint(w * (2 * f + 1) * 1024.f + 12582912.f);
              uint32_t hi = __float_as_uint(w * (2 * f + 2) * 1024.f + 12582912.f);
              unsigned long long v = (unsigned long long)hi << 32 | lo;
              unsigned a = (unsigned)__cvta_generic_to_shared(&ar[f * FS + n]);
              asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
            }
          }
        }
  }
  __syncthreads();
  unsigned long long acc = 0;
  for (int i = threadIdx.x; i < 4 * FS; i += blockDim.x) acc += ar[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
}

int main() {
  int blocks = 148 * 8, threads = 256, iters = 64;
  size_t n = (size_t)blocks * threads;
  uint32_t* seeds;
  float* out;
  cudaMalloc(&seeds, n * 4);
  cudaMalloc(&out, n * 4);
  uint32_t* h = new uint32_t[n];
  for (size_t i = 0; i < n; ++i) h[i] = (uint32_t)(i * 2654435761u + 12345);
  cudaMemcpy(seeds, h, n * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](auto kern, const char* name) {
    kern<<<blocks, threads>>>(seeds, out, 2);
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(a);
      kern<<<blocks, threads>>>(seeds, out, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    double parts = double(n) * iters;
    printf("%-36s %8.3f ms  %.3e particles/s (8 fields x 27 nodes)\n", name, best, parts / (best * 1e-3));
  };
  run(scat<0, 68>, "8 x red.shared.add.s32, SI=68");
  run(scat<1, 68>, "4 x red.shared.add.u64, SI=68");
  run(scat<1, 64>, "4 x red.shared.add.u64, SI=64");
  run(scat<1, 72>, "4 x red.shared.add.u64, SI=72");
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
