// FFMA vs FFMA2 throughput on sm_100a (scratch microbenchmark)
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r;
}
__global__ void k1(float* out, float s, int iters) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x + i;
  float b = s, c = s * 0.5f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], b, c);
    b += 1e-7f; c -= 1e-7f;
  }
  float t = 0; for (int i = 0; i < 16; ++i) t += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k2(float* out, float s, int iters) {
  u64 a[8];
  for (int i = 0; i < 8; ++i) { float2 v = make_float2(threadIdx.x + i, threadIdx.x - i); a[i] = *reinterpret_cast<u64*>(&v); }
  float2 bv = make_float2(s, s * 1.1f), cv = make_float2(s * 0.5f, s * 0.25f);
  u64 b = *reinterpret_cast<u64*>(&bv), c = *reinterpret_cast<u64*>(&cv);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma2(a[i], b, c);
    b ^= 1ull; c ^= 2ull;
  }
  float t = 0; for (int i = 0; i < 8; ++i) { float2 v = *reinterpret_cast<float2*>(&a[i]); t += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
int main() {
  float* o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000, blocks = 148 * 8, threads = 256;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(e0); k1<<<blocks, threads>>>(o, 1.0001f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fma = 16.0 * iters * blocks * threads;
    printf("FFMA : %.1f TFMA/s\n", fma / ms / 1e9);
    cudaEventRecord(e0); k2<<<blocks, threads>>>(o, 1.0001f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA2: %.1f TFMA/s\n", fma / ms / 1e9);
  }
  return 0;
}
