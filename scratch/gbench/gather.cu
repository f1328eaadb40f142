// gather bandwidth microbenchmark: sum of X[idx[i]] rows (128 B each)
#include <cuda_runtime.h>
#include <stdint.h>
extern "C" __global__ void gather_sum(const float4* __restrict__ x, const int* __restrict__ idx, int64_t m, int ld4, float* out, int unroll) {
  // 8 lanes per row (float4 each) -> 4 rows per warp instruction
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float4 acc = make_float4(0,0,0,0);
  for (int64_t base = warp * 32; base < m; base += nw * 32) {
    // 32 rows per iteration: 8 loads per lane
    float4 v[8];
    #pragma unroll
    for (int k = 0; k < 8; ++k) {
      int64_t i = base + k * 4 + (lane >> 3);
      int r = i < m ? __ldg(idx + i) : 0;
      v[k] = __ldg(x + (int64_t)r * ld4 + (lane & 7));
    }
    #pragma unroll
    for (int k = 0; k < 8; ++k) { acc.x += v[k].x; acc.y += v[k].y; acc.z += v[k].z; acc.w += v[k].w; }
  }
  out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}
extern "C" int run_gather(const float* x, const int* idx, int64_t m, int ld, float* out, int blocks, int threads, void* stream) {
  gather_sum<<<blocks, threads, 0, (cudaStream_t)stream>>>((const float4*)x, idx, m, ld / 4, out, 0);
  return (int)cudaGetLastError();
}
