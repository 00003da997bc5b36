// Throughput of FFMA vs FFMA2 (fma.rn.f32x2) on sm_100a, with and without an
// interleaved ALU stream.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_ffma2 ubench_ffma2.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

template <int MODE>
__global__ void k(float* out, int seed) {
  float a[16];
  unsigned u[4];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = float(threadIdx.x + i + seed) * 1e-3f;
#pragma unroll
  for (int i = 0; i < 4; ++i) u[i] = threadIdx.x * (i + 7) + seed;
  const float b = 0.999f, c = 1e-4f;
  const float2 b2 = make_float2(b, b), c2 = make_float2(c, c);
  for (int it = 0; it < ITERS; ++it) {
    if (MODE == 0 || MODE == 2) {  // 16 FFMA
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], b, c);
    } else {  // 8 FFMA2 = same flops
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float2 v = make_float2(a[2 * i], a[2 * i + 1]);
        v = __ffma2_rn(v, b2, c2);
        a[2 * i] = v.x;
        a[2 * i + 1] = v.y;
      }
    }
    if (MODE >= 2) {  // + 8 ALU ops
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        u[i] = (u[i] ^ (u[i] >> 3)) + 0x9E3779B9u;
        u[i] = __funnelshift_l(u[i], u[i], 5);
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + float(u[0] ^ u[1] ^ u[2] ^ u[3]);
}

template <int MODE>
void run(const char* name, float* d) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<MODE><<<148 * 4, 256>>>(d, 1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<MODE><<<148 * 4, 256>>>(d, r);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double fma = 5.0 * 148 * 4 * 256 * double(ITERS) * 16;
  printf("%-28s %8.3f ms  %7.2f TFMA/s (fp32 fma/s)\n", name, ms, fma / (ms * 1e-3) / 1e12);
}

int main() {
  float* d;
  cudaMalloc(&d, 148 * 4 * 256 * 4);
  run<0>("16 FFMA", d);
  run<1>("8 FFMA2", d);
  run<2>("16 FFMA + 8 ALU", d);
  run<3>("8 FFMA2 + 8 ALU", d);
  return 0;
}
