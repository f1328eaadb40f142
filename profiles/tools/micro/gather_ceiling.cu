// Gather-ceiling microbenchmark for the TC-GNN SpMM on B200 (round 2).
//
// Question: how fast can an SM array pull U random neighbour rows (arxiv:
// U = 1.166M rows of 4*D bytes out of an N = 169,343-row X) into the SMs,
// by path, and what does the L2 state before the launch cost?
//   ldg    : 8 lanes per 128-B row, LDG.128, U rows in flight per warp
//   cpa    : cp.async.cg 16 B per lane into a per-warp smem ring (round-1 engine pattern)
//   g4     : TMA tile::gather4 (one elected lane per CTA) into an mbarrier ring
//   ldg96  : 96-B rows (a 24-bit TF32 packing of D = 32), 6 lanes per row
// L2 before each launch: "dirty" = 512 MB memset (the round-1 bench flush:
// leaves ~126 MB of dirty lines that the timed kernel must write back),
// "clean" = the memset then a 512 MB read, "warm" = back-to-back.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gc gather_ceiling.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__);             \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int UNR>
__global__ void __launch_bounds__(256) ldg_gather(const float4* __restrict__ x, const int* __restrict__ idx,
                                                  int m, float* out) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const int r = lane >> 3, q = lane & 7;
  float acc = 0.f;
  // rows [4*UNR*c, 4*UNR*(c+1)) per warp step
  for (int c = gw; c * 4 * UNR < m; c += nw) {
    int id[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int i = c * 4 * UNR + 4 * u + r;
      id[u] = i < m ? __ldg(idx + i) : 0;
    }
    float4 v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) v[u] = __ldg(x + (size_t)id[u] * 8 + q);
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 1234.5f) out[threadIdx.x] = acc;
}

// 64-B rows (D = 16): 4 lanes per row, 8 rows per warp instruction
template <int UNR>
__global__ void __launch_bounds__(256) ldg64_gather(const float4* __restrict__ x, const int* __restrict__ idx,
                                                    long m, float* out) {
  const int lane = threadIdx.x & 31;
  const long gw = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((long)gridDim.x * blockDim.x) >> 5;
  const int r = lane >> 2, q = lane & 3;
  float acc = 0.f;
  for (long c = gw; c * 8 * UNR < m; c += nw) {
    int id[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const long i = c * 8 * UNR + 8 * u + r;
      id[u] = i < m ? __ldg(idx + i) : 0;
    }
    float4 v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) v[u] = __ldg(x + (size_t)id[u] * 4 + q);
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 1234.5f) out[threadIdx.x] = acc;
}

// 96-B rows: lanes 0..29 -> 5 rows x 6 pieces of 16 B
template <int UNR>
__global__ void __launch_bounds__(256) ldg96_gather(const float4* __restrict__ x, const int* __restrict__ idx,
                                                    int m, float* out) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const int r = lane / 6, q = lane % 6;
  float acc = 0.f;
  for (int c = gw; c * 5 * UNR < m; c += nw) {
    int id[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int i = c * 5 * UNR + 5 * u + r;
      id[u] = (lane < 30 && i < m) ? __ldg(idx + i) : 0;
    }
    float4 v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) v[u] = lane < 30 ? __ldg(x + (size_t)id[u] * 6 + q) : make_float4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 1234.5f) out[threadIdx.x] = acc;
}

// cp.async ring: per warp NB stages of 4 rows (512 B) x 2 (two copies per lane: rows t, t+4)
template <int NB>
__global__ void __launch_bounds__(128) cpa_gather(const char* __restrict__ x, const int* __restrict__ idx, int m,
                                                  float* out) {
  __shared__ __align__(128) unsigned char sm[4][NB][1024];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const int r = lane >> 3, q = lane & 7;
  const int nblk = (m + 7) / 8;
  float acc = 0.f;
  auto issue = [&](int b, int s) {
    if (b < nblk) {
      const int i0 = min(b * 8 + r, m - 1), i1 = min(b * 8 + 4 + r, m - 1);
      const int a = __ldg(idx + i0), c = __ldg(idx + i1);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(&sm[wid][s][r * 128 + q * 16])),
                   "l"(x + (size_t)a * 128 + q * 16)
                   : "memory");
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(&sm[wid][s][512 + r * 128 + q * 16])),
                   "l"(x + (size_t)c * 128 + q * 16)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int k = 0;
  for (int s = 0; s < NB; ++s) issue(gw + s * nw, s);
  for (int b = gw; b < nblk; b += nw, ++k) {
    asm volatile("cp.async.wait_group %0;" ::"n"(NB - 1) : "memory");
    const int s = k % NB;
    const float4 v = *reinterpret_cast<const float4*>(&sm[wid][s][lane * 16]);
    acc += v.x + v.w;
    __syncwarp();
    issue(b + NB * nw, s);
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (acc == 1234.5f) out[threadIdx.x] = acc;
}

// TMA gather4: one producer lane per CTA, NS stages of 8 gather4 (32 rows, 4 KB);
// the CTA's consumer warps each touch their share of the stage and arrive on `empty`.
template <int NS, int NCW>
__global__ void __launch_bounds__((NCW + 1) * 32) g4_gather(const __grid_constant__ CUtensorMap tm,
                                                            const int* __restrict__ idx, int m, float* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  constexpr int STG = 4096;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NS * STG);
  uint64_t* empty = full + NS;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su(full + s)));
      asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(su(empty + s)), "r"(NCW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nst = (m + 31) / 32;  // stages of 32 rows
  float acc = 0.f;
  if (wid == NCW) {
    // producer warp: lane L issues gather4 (L % 8) of stage 4j + L/8; the ids of
    // iteration j + 1 are loaded while iteration j waits and issues
    const int sub = lane >> 3, gq = lane & 7;
    auto ids = [&](int j) {
      const int st = blockIdx.x + (4 * j + sub) * gridDim.x;
      const int i = st * 32 + gq * 4;
      int4 r;
      r.x = __ldg(idx + min(i, m - 1));
      r.y = __ldg(idx + min(i + 1, m - 1));
      r.z = __ldg(idx + min(i + 2, m - 1));
      r.w = __ldg(idx + min(i + 3, m - 1));
      return r;
    };
    int4 cur = ids(0);
    for (int j = 0;; ++j) {
      const int k = 4 * j + sub;
      const int st = blockIdx.x + k * gridDim.x;
      if (blockIdx.x + 4 * j * gridDim.x >= nst) break;
      const int4 nxt = ids(j + 1);
      if (st < nst) {
        const int s = k % NS;
        if (k >= NS) {
          const uint32_t ph = ((k / NS) - 1) & 1;
          asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W;}" ::"r"(
                           su(empty + s)),
                       "r"(ph)
                       : "memory");
        }
        if (gq == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su(full + s)), "r"(STG) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
            "%3, %4, %5, %6}], [%7];" ::"r"(su(sm + s * STG + gq * 512)),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(cur.x), "r"(cur.y), "r"(cur.z), "r"(cur.w), "r"(su(full + s))
            : "memory");
      }
      cur = nxt;
    }
  } else {
    int k = 0;
    for (int st = blockIdx.x; st < nst; st += gridDim.x, ++k) {
      const int s = k % NS;
      const uint32_t ph = (k / NS) & 1;
      asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W;}" ::"r"(
                       su(full + s)),
                   "r"(ph)
                   : "memory");
      const float4 v = *reinterpret_cast<const float4*>(sm + s * STG + ((wid * 32 + lane) * 16) % STG);
      acc += v.x + v.w;
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(su(empty + s)) : "memory");
    }
  }
  if (acc == 1234.5f) out[threadIdx.x] = acc;
}

__global__ void read_flush(const float4* __restrict__ p, size_t n, float* out) {
  float a = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float4 v = __ldcs(p + i);
    a += v.x;
  }
  if (a == 1234.5f) out[0] = a;
}

static char* g_fl;
static float* g_out;
static int g_nsm;
static void flush(int mode) {
  if (mode == 0) return;
  CK(cudaMemsetAsync(g_fl, 1, 512 << 20));
  if (mode == 2) read_flush<<<g_nsm * 8, 256>>>(reinterpret_cast<const float4*>(g_fl + (512 << 20)), (512 << 20) / 16, g_out);
}

template <class F>
static float timeit(F f, int mode, int reps = 30) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  std::vector<float> v;
  for (int i = 0; i < reps + 3; ++i) {
    flush(mode);
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (i >= 3) v.push_back(ms * 1000);
  }
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

int main() {
  if (getenv("GC_PRODUCTS")) {
    // products-scale D = 16: 61.86 M random 64-B rows out of a 2.45 M-row (157 MB) X
    const long N = 2449029, M = 61858832;
    std::mt19937 rng(1);
    std::vector<int> idx(M);
    for (auto& v : idx) v = rng() % N;
    float *x, *out;
    int* di;
    CK(cudaMalloc(&x, (size_t)N * 64));
    CK(cudaMalloc(&di, 4 * M));
    CK(cudaMalloc(&out, 1 << 24));
    CK(cudaMalloc(&g_fl, 1024ull << 20));
    g_out = out;
    CK(cudaMemset(x, 0, (size_t)N * 64));
    CK(cudaMemcpy(di, idx.data(), 4 * M, cudaMemcpyHostToDevice));
    cudaDeviceGetAttribute(&g_nsm, cudaDevAttrMultiProcessorCount, 0);
    const char* mn[3] = {"warm", "dirty", "clean"};
    for (int cps : {4, 8}) {
      for (int unr : {4, 8}) {
        printf("ldg64 U=%d ctas/sm=%d (rows %.2f GB + ids %.2f GB)", unr, cps, M * 64 / 1e9, M * 4 / 1e9);
        for (int mode = 0; mode < 3; ++mode) {
          auto f = [&] {
            if (unr == 4) ldg64_gather<4><<<g_nsm * cps, 256>>>((const float4*)x, di, M, out);
            else ldg64_gather<8><<<g_nsm * cps, 256>>>((const float4*)x, di, M, out);
          };
          const float us = timeit(f, mode);
          printf("  %s %7.1f us", mn[mode], us);
        }
        printf("\n");
        CK(cudaGetLastError());
      }
    }
    return 0;
  }
  const int N = 169343, M = 1165855;
  std::mt19937 rng(1);
  std::vector<int> idx(M);
  for (auto& v : idx) v = rng() % N;
  float *x, *x96, *out;
  int* di;
  CK(cudaMalloc(&x, (size_t)N * 128));
  CK(cudaMalloc(&x96, (size_t)N * 96));
  CK(cudaMalloc(&di, 4 * M));
  CK(cudaMalloc(&out, 1 << 24));
  CK(cudaMalloc(&g_fl, 1024ull << 20));
  g_out = out;
  CK(cudaMemset(x, 0, (size_t)N * 128));
  CK(cudaMemset(x96, 0, (size_t)N * 96));
  CK(cudaMemcpy(di, idx.data(), 4 * M, cudaMemcpyHostToDevice));
  cudaDeviceGetAttribute(&g_nsm, cudaDevAttrMultiProcessorCount, 0);
  const char* mn[3] = {"warm", "dirty", "clean"};
  auto report = [&](const char* name, double bytes, auto f) {
    printf("%-28s", name);
    for (int mode = 0; mode < 3; ++mode) {
      const float us = timeit(f, mode);
      printf("  %s %6.1f us (%5.0f GB/s)", mn[mode], us, bytes / (us * 1e3));
    }
    printf("\n");
    CK(cudaGetLastError());
  };
  const double B128 = (double)M * 128, B96 = (double)M * 96;
  const bool only_g4 = getenv("GC_G4") != nullptr;
  if (!only_g4) {
  for (int cps : {4, 8}) {
    char nm[64];
    snprintf(nm, 64, "ldg  U=4  ctas/sm=%d", cps);
    report(nm, B128, [&] { ldg_gather<4><<<g_nsm * cps, 256>>>((const float4*)x, di, M, out); });
    snprintf(nm, 64, "ldg  U=8  ctas/sm=%d", cps);
    report(nm, B128, [&] { ldg_gather<8><<<g_nsm * cps, 256>>>((const float4*)x, di, M, out); });
    snprintf(nm, 64, "ldg96 U=8 ctas/sm=%d", cps);
    report(nm, B96, [&] { ldg96_gather<8><<<g_nsm * cps, 256>>>((const float4*)x96, di, M, out); });
  }
  for (int cps : {2, 4}) {
    char nm[64];
    snprintf(nm, 64, "cp.async NB=4 ctas/sm=%d", cps);
    report(nm, B128, [&] { cpa_gather<4><<<g_nsm * cps * 2, 128>>>((const char*)x, di, M, out); });
    snprintf(nm, 64, "cp.async NB=8 ctas/sm=%d", cps);
    report(nm, B128, [&] { cpa_gather<8><<<g_nsm * cps * 2, 128>>>((const char*)x, di, M, out); });
  }
  }
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  CUtensorMap tm;
  cuuint64_t gd[2] = {32, (cuuint64_t)N};
  cuuint64_t gs[1] = {128};
  cuuint32_t box[2] = {32, 1}, es[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
#define G4(NS, NCW, CPS)                                                                                    \
  {                                                                                                         \
    const int smem = NS * 4096 + 16 * NS + 1024;                                                            \
    CK(cudaFuncSetAttribute(g4_gather<NS, NCW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));        \
    char nm[64];                                                                                            \
    snprintf(nm, 64, "g4 NS=%d (%dKB) ctas/sm=%d", NS, NS * 4, CPS);                                        \
    report(nm, B128, [&] { g4_gather<NS, NCW><<<g_nsm * CPS, (NCW + 1) * 32, smem>>>(tm, di, M, out); }); \
  }
  if (!only_g4) { G4(16, 2, 1) G4(16, 2, 2) G4(12, 2, 4) }
  G4(4, 1, 8) G4(6, 1, 8) G4(4, 2, 6) G4(6, 2, 6) G4(8, 1, 6) G4(4, 1, 12) G4(4, 1, 16)
  return 0;
}
