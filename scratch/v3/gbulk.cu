// gather microbenchmark: 128-B rows X[idx[i]] into smem via per-lane cp.async.bulk (TMA 1D)
// vs LDG.128 (L1 path). Rows of arxiv-shaped random idx.
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
#ifndef NS
#define NS 4
#endif
#ifndef WPB
#define WPB 4
#endif
__global__ void __launch_bounds__(WPB * 32) gather_bulk(const float* __restrict__ x, const int* __restrict__ idx, int m, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned char* ring = sm + wid * (NS * 4096 + 64);
  uint64_t* bar = reinterpret_cast<uint64_t*>(ring + NS * 4096);
  if (lane == 0) for (int s = 0; s < NS; ++s) asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"(su(bar + s)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int gw = blockIdx.x * WPB + wid, nw = gridDim.x * WPB;
  const int chunks = (m + 31) / 32;
  float acc = 0.f;
  int it = 0;
  auto issue = [&](int c, int s) {
    if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(su(bar + s)), "r"(4096) : "memory");
    __syncwarp();
    const int i = c * 32 + lane;
    const int r = __ldg(idx + min(i, m - 1));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 128, [%2];"
                 :: "r"(su(ring + s * 4096 + lane * 128)), "l"(x + (int64_t)r * 32), "r"(su(bar + s)) : "memory");
  };
  int c = gw;
  for (int s = 0; s < NS; ++s) if (c + s * nw < chunks) issue(c + s * nw, s);
  for (int k = 0; c + k * nw < chunks; ++k) {
    const int s = k % NS;
    const uint32_t ph = (k / NS) & 1;
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W;}" :: "r"(su(bar + s)), "r"(ph) : "memory");
    const float4 v = *reinterpret_cast<const float4*>(ring + s * 4096 + lane * 128 + (lane & 7) * 16);
    acc += v.x + v.w;
    __syncwarp();
    if (c + (k + NS) * nw < chunks) issue(c + (k + NS) * nw, s);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void gather_ldg(const float4* __restrict__ x, const int* __restrict__ idx, int m, float* out) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int base = warp * 32; base < m; base += nw * 32) {
    float4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      int i = base + k * 4 + (lane >> 3);
      int r = i < m ? __ldg(idx + i) : 0;
      v[k] = __ldg(x + (int64_t)r * 8 + (lane & 7));
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) { acc.x += v[k].x; acc.w += v[k].w; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.w;
}
int main() {
  const int N = 169343, M = 1165855;
  std::mt19937 rng(1);
  std::vector<int> idx(M);
  for (auto& v : idx) v = rng() % N;
  float* x; int* di; float* out; char* fl;
  CK(cudaMalloc(&x, (size_t)N * 128)); CK(cudaMalloc(&di, 4 * M)); CK(cudaMalloc(&out, 1 << 24)); CK(cudaMalloc(&fl, 512 << 20));
  CK(cudaMemset(x, 0, (size_t)N * 128));
  CK(cudaMemcpy(di, idx.data(), 4 * M, cudaMemcpyHostToDevice));
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto timeit = [&](auto launch, const char* name) {
    std::vector<float> c, w;
    for (int cold = 1; cold >= 0; --cold) {
      std::vector<float>& v = cold ? c : w;
      for (int i = 0; i < 20; ++i) {
        if (cold) CK(cudaMemsetAsync(fl, i, 512 << 20));
        cudaEventRecord(a); launch(); cudaEventRecord(b); CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b); if (i > 2) v.push_back(ms * 1000);
      }
      std::sort(v.begin(), v.end());
    }
    printf("%-28s cold %6.1f us  warm %6.1f us  (%.0f GB/s warm)\n", name, c[c.size()/2], w[w.size()/2], M * 128.0 / (w[w.size()/2] * 1e3));
  };
  for (int cps : {2, 4, 8}) {
    const int smem = WPB * (NS * 4096 + 64);
    CK(cudaFuncSetAttribute(gather_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    char nm[64]; sprintf(nm, "bulk NS=%d ctas/sm=%d", NS, cps);
    timeit([&] { gather_bulk<<<nsm * cps, WPB * 32, smem>>>(x, di, M, out); }, nm);
  }
  for (int wps : {16, 32, 64}) {
    char nm[64]; sprintf(nm, "ldg warps/sm=%d", wps);
    timeit([&] { gather_ldg<<<nsm * wps / 8, 256>>>((const float4*)x, di, M, out); }, nm);
  }
  CK(cudaGetLastError());
  return 0;
}
