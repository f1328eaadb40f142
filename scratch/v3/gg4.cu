// gather4 TMA microbenchmark: rows of X (N x 32 fp32) by random idx into smem
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
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
#ifndef IL
#define IL 8   // issuing lanes per warp (each: 4 rows)
#endif
constexpr int STG = IL * 512;  // bytes per stage
__global__ void __launch_bounds__(WPB * 32) g4(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx, int m, float* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned char* ring = sm + wid * (NS * STG + 1024);
  uint64_t* bar = reinterpret_cast<uint64_t*>(ring + NS * STG);
  if (lane == 0) for (int s = 0; s < NS; ++s) asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"(su(bar + s)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int gw = blockIdx.x * WPB + wid, nw = gridDim.x * WPB;
  const int rows_per = IL * 4;
  const int chunks = (m + rows_per - 1) / rows_per;
  float acc = 0.f;
  auto issue = [&](int c, int s) {
    if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(su(bar + s)), "r"(STG) : "memory");
    __syncwarp();
    if (lane < IL) {
      const int i = c * rows_per + lane * 4;
      const int4 r = __ldg(reinterpret_cast<const int4*>(idx) + min(i, m - 4) / 4);
      asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                   :: "r"(su(ring + s * STG + lane * 512)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w), "r"(su(bar + s)) : "memory");
    }
  };
  int c = gw;
  for (int s = 0; s < NS; ++s) if (c + s * nw < chunks) issue(c + s * nw, s);
  for (int k = 0; c + k * nw < chunks; ++k) {
    const int s = k % NS;
    const uint32_t ph = (k / NS) & 1;
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W;}" :: "r"(su(bar + s)), "r"(ph) : "memory");
    const float4 v = *reinterpret_cast<const float4*>(ring + s * STG + (lane * 16) % STG);
    acc += v.x + v.w;
    __syncwarp();
    if (c + (k + NS) * nw < chunks) issue(c + (k + NS) * nw, s);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
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
  void* fp = nullptr; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  CUtensorMap tm;
  cuuint64_t gd[2] = {32, (cuuint64_t)N}; cuuint64_t gs[1] = {128}; cuuint32_t box[2] = {32, 1}, es[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("encode failed\n"); return 1; }
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int smem = WPB * (NS * STG + 1024);
  CK(cudaFuncSetAttribute(g4, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int occ; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, g4, WPB * 32, smem);
  for (int cps = occ; cps >= 1 && cps >= occ / 2; --cps) {
    std::vector<float> c, w;
    for (int cold = 1; cold >= 0; --cold) {
      std::vector<float>& v = cold ? c : w;
      for (int i = 0; i < 20; ++i) {
        if (cold) CK(cudaMemsetAsync(fl, i, 512 << 20));
        cudaEventRecord(a); g4<<<nsm * cps, WPB * 32, smem>>>(tm, di, M, out); cudaEventRecord(b); CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b); if (i > 2) v.push_back(ms * 1000);
      }
      std::sort(v.begin(), v.end());
    }
    printf("gather4 IL=%d NS=%d WPB=%d ctas/sm=%d (occ %d): cold %6.1f us warm %6.1f us (%.0f GB/s warm)\n", IL, NS, WPB, cps, occ, c[c.size()/2], w[w.size()/2], M * 128.0 / (w[w.size()/2] * 1e3));
  }
  CK(cudaGetLastError());
  return 0;
}
