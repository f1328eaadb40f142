// Standalone design study: register-direct, warp-per-window-stream TF32 SpMM
// (arxiv-shaped uniform graph, D=32). Build: nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a -lineinfo spmm_rd.cu -o spmm_rd
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__device__ __forceinline__ uint32_t tf32_rn(float x) {
  uint32_t r;
  asm("cvt.rn.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

struct P {
  int64_t n, nwin;
  const int64_t* ptr;    // N+1
  const int64_t* boff;   // W+1 block offsets (exclusive cumsum of wp)
  const int* c2np;       // 8*TB padded col_to_node (-1 pad)
  const uint32_t* efl;   // per-edge local fragment slot lb*128 + lane*4 + slot
  const float* w;        // edge weights (nullable)
  const float* x;        // N x 32
  float* y;              // N x 32
  int nwarps;
  const int* wstart;  // nwarps+1 window starts
};

#ifndef WPC
#define WPC 4             // warps per CTA
#endif
#ifndef MINB
#define MINB 3
#endif
#ifndef NB
#define NB 8              // X ring depth (blocks)
#endif
#ifndef MAXB
#define MAXB 16           // A-frag blocks resident per warp
#endif
#ifndef EPL
#define EPL 5             // prefetched edges per lane
#endif
constexpr int NI = 2 * NB;  // idx ring (per-lane 8-B entries)
constexpr int WARP_SMEM = NB * 1024 + NI * 256 + MAXB * 512;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async16(uint32_t s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];\n" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint4 lds128u(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint2 lds64u(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];\n" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
  return v;
}

__global__ void __launch_bounds__(WPC * 32, MINB) spmm_rd(const P p) {
  extern __shared__ __align__(128) unsigned char smem_[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int gw = blockIdx.x * WPC + wid;
  unsigned char* wsm = smem_ + wid * WARP_SMEM;
  uint32_t* afr = reinterpret_cast<uint32_t*>(wsm + NB * 1024 + NI * 256);
  const int g = lane >> 2, t = lane & 3;
  const int nwin = (int)p.nwin;
  const int4 wm = __ldg(reinterpret_cast<const int4*>(p.wstart) + gw);  // ws, we, gb0, nblk
  const int ws = wm.x, we = wm.y;
  if (ws >= we) return;
  const int gb0 = wm.z;
  // per-lane constants
  const uint32_t xs = smem_u32(wsm) + t * 128 + ((g ^ (2 * t)) & 7) * 16;  // + slot*1024 (+512: row t+4)
  const uint32_t is = smem_u32(wsm) + NB * 1024 + lane * 8;                 // + slot*256
  const uint32_t as = smem_u32(afr) + lane * 16;                            // + lb*512
  const char* xb = reinterpret_cast<const char*>(p.x + 4 * g);
  const char* ib = reinterpret_cast<const char*>(p.c2np + 8 * (int64_t)gb0 + 2 * t);  // + s*32

  auto issue_idx = [&](int s, int slot) { cp_async8(is + slot * 256, ib + (int64_t)s * 32); };
  auto issue_x = [&](int islot, int xslot) {
    const uint2 id = lds64u(is + islot * 256);
    cp_async16(xs + xslot * 1024, xb + (uint64_t)id.x * 128u);
    cp_async16(xs + xslot * 1024 + 512, xb + (uint64_t)id.y * 128u);
  };
#pragma unroll
  for (int s = 0; s < NB; ++s) issue_idx(s, s);
  cp_commit();
  cp_wait<0>();
#pragma unroll
  for (int s = 0; s < NB; ++s) {
    issue_x(s, s);
    issue_idx(s + NB, s + NB);
    cp_commit();
  }
  auto ptr_of = [&](int w) { return (int)__ldg(p.ptr + min((int64_t)w * 16, p.n)); };
  auto blk_of = [&](int w) { return (int)(__ldg(p.boff + min(w, nwin))) - gb0; };
  int w = ws;
  int cb0 = 0, cb1 = blk_of(ws + 1), nb2 = blk_of(ws + 2), nb3 = blk_of(ws + 3);
  int e0 = ptr_of(ws), e1 = ptr_of(ws + 1), e2 = ptr_of(ws + 2), e3 = ptr_of(ws + 3);
  uint32_t pf[EPL], of[EPL];
  float pw[EPL];
  auto prefetch = [&](int a, int b) {
#pragma unroll
    for (int k = 0; k < EPL; ++k) {
      const int e = a + lane + 32 * k;
      const bool ok = e < b;
      pf[k] = ok ? __ldg(p.efl + e) : 0xffffffffu;
      pw[k] = ok && p.w ? __ldg(p.w + e) : 1.f;
    }
  };
  for (int q = 0; q < MAXB; ++q) reinterpret_cast<uint4*>(afr)[q * 32 + lane] = make_uint4(0, 0, 0, 0);
#pragma unroll
  for (int k = 0; k < EPL; ++k) of[k] = 0xffffffffu;
  prefetch(e0, e1);
  float acc[4][4];
  int lb = 0, lim = 0, nbw = 0;
  bool hub = false;
  // start window w: scatter prefetched edges, prefetch w+1 (windows with no blocks are
  // written as zero rows here)
  auto store = [&](int wv) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = wv * 16 + g + 8 * h;
      if (r < p.n) {
        float4* yr = reinterpret_cast<float4*>(p.y + (int64_t)r * 32 + 8 * t);
        yr[0] = make_float4(acc[0][2 * h] + 0.f, acc[1][2 * h] + 0.f, acc[2][2 * h] + 0.f, acc[3][2 * h] + 0.f);
        yr[1] = make_float4(acc[0][2 * h + 1] + 0.f, acc[1][2 * h + 1] + 0.f, acc[2][2 * h + 1] + 0.f, acc[3][2 * h + 1] + 0.f);
      }
    }
  };
  auto roll = [&]() {
    cb0 = cb1; cb1 = nb2; nb2 = nb3; nb3 = blk_of(w + 3);
    e0 = e1; e1 = e2; e2 = e3; e3 = ptr_of(w + 3);
  };
  auto hub_load = [&](int r0) {
    __syncwarp();
    for (int q = 0; q < MAXB; ++q) reinterpret_cast<uint4*>(afr)[q * 32 + lane] = make_uint4(0, 0, 0, 0);
    __syncwarp();
    for (int e = e0 + lane; e < e1; e += 32) {
      const uint32_t f = __ldg(p.efl + e) - r0 * 128;
      if (f < (uint32_t)(MAXB * 128)) afr[f] = tf32_rn(p.w ? __ldg(p.w + e) : 1.f);
    }
    __syncwarp();
  };
  // returns false when the warp's last window is done
  auto begin_window = [&]() -> bool {
    for (;;) {
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
      if (w >= we) return false;
      nbw = cb1 - cb0;
      hub = nbw > MAXB || e1 - e0 > 32 * EPL;
      __syncwarp();
      if (!hub) {
#pragma unroll
        for (int k = 0; k < EPL; ++k)
          if (pf[k] < (uint32_t)(MAXB * 128)) afr[pf[k]] = tf32_rn(pw[k]);
#pragma unroll
        for (int k = 0; k < EPL; ++k) of[k] = pf[k];
      } else {
        hub_load(0);
      }
      __syncwarp();
      prefetch(e1, e2);
      if (nbw > 0) break;
      store(w);  // empty window
      ++w;
      roll();
    }
    lb = 0;
    lim = min(nbw, MAXB);
#ifdef DBG
    if (gw == 0 && lane == 0) printf("w %d nbw %d e0 %d e1 %d hub %d cb0 %d cb1 %d\n", w, nbw, e0, e1, (int)hub, cb0, cb1);
#endif
    return true;
  };
  auto end_window = [&]() {
    store(w);
    __syncwarp();
    if (!hub) {
#pragma unroll
      for (int k = 0; k < EPL; ++k)
        if (of[k] < (uint32_t)(MAXB * 128)) afr[of[k]] = 0u;
    } else {
      for (int q = 0; q < MAXB; ++q) reinterpret_cast<uint4*>(afr)[q * 32 + lane] = make_uint4(0, 0, 0, 0);
    }
    ++w;
    roll();
  };
  if (!begin_window()) goto done;
  for (int s = 0;; ++s) {
    const uint32_t xo = (uint32_t)(s & (NB - 1)) * 1024u;
    cp_wait<NB - 1>();
    const float4 xa = lds128(xs + xo);
    const float4 xc = lds128(xs + xo + 512);
    const uint4 af = lds128u(as + (lb & (MAXB - 1)) * 512);
    mma_tf32(acc[0], af.x, af.y, af.z, af.w, tf32_rn(xa.x), tf32_rn(xc.x));
    mma_tf32(acc[1], af.x, af.y, af.z, af.w, tf32_rn(xa.y), tf32_rn(xc.y));
    mma_tf32(acc[2], af.x, af.y, af.z, af.w, tf32_rn(xa.z), tf32_rn(xc.z));
    mma_tf32(acc[3], af.x, af.y, af.z, af.w, tf32_rn(xa.w), tf32_rn(xc.w));
    {
      const uint2 id = lds64u(is + (uint32_t)((s + NB) & (NI - 1)) * 256u);
      cp_async16(xs + xo, xb + (uint64_t)id.x * 128u);
      cp_async16(xs + xo + 512, xb + (uint64_t)id.y * 128u);
    }
    cp_async8(is + (uint32_t)(s & (NI - 1)) * 256u, ib + (int64_t)(s + 2 * NB) * 32);
    cp_commit();
    if (++lb == lim) {
      if (lb == nbw) {
        end_window();
        if (!begin_window()) goto done;
      } else {
        hub_load(lb);
        lim = min(nbw, lb + MAXB);
      }
    }
  }
done:
  cp_wait<0>();
}

// ------------------------------------------------------------------ host
int main(int argc, char** argv) {
  const int64_t N = 169343;
  const double avg = 1166243.0 / N;
  std::mt19937_64 rng(1);
  const int64_t Mreq = (int64_t)(avg * N);
  std::vector<std::pair<uint32_t, uint32_t>> ed(Mreq);
  std::uniform_int_distribution<uint32_t> U(0, (uint32_t)N - 1);
  for (auto& e : ed) e = {U(rng), U(rng)};
  std::sort(ed.begin(), ed.end());
  ed.erase(std::unique(ed.begin(), ed.end()), ed.end());
  const int64_t M = ed.size();
  std::vector<int64_t> ptr(N + 1, 0);
  std::vector<uint32_t> col(M);
  for (int64_t i = 0; i < M; ++i) ptr[ed[i].first + 1]++, col[i] = ed[i].second;
  for (int64_t i = 0; i < N; ++i) ptr[i + 1] += ptr[i];
  const int64_t W = (N + 15) / 16;
  std::vector<int64_t> boff(W + 1, 0);
  std::vector<int> c2np;
  std::vector<uint32_t> efl(M);
  int maxb = 0;
  for (int64_t w = 0; w < W; ++w) {
    int64_t e0 = ptr[w * 16], e1 = ptr[std::min(w * 16 + 16, N)];
    std::vector<uint32_t> u(col.begin() + e0, col.begin() + e1);
    std::sort(u.begin(), u.end());
    u.erase(std::unique(u.begin(), u.end()), u.end());
    int nb = (int)((u.size() + 7) / 8);
    maxb = std::max(maxb, nb);
    boff[w + 1] = boff[w] + nb;
    for (int bb = 0; bb < nb; ++bb) for (int i = 0; i < 8; ++i) { int c = bb * 8 + ((i & 1) ? 4 + i / 2 : i / 2); c2np.push_back(c < (int)u.size() ? (int)u[c] : (int)u[0]); }
    for (int64_t r = w * 16; r < std::min(w * 16 + 16, N); ++r)
      for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e) {
        int c = (int)(std::lower_bound(u.begin(), u.end(), col[e]) - u.begin());
        int rl = (int)(r & 15), k = c & 7;
        efl[e] = (c >> 3) * 128 + ((((rl & 7) << 2) | (k & 3)) << 2) + (rl >> 3) + 2 * (k >> 2);
      }
  }
  const int64_t TB = boff[W];
  for (int i = 0; i < 8 * 64; ++i) c2np.push_back(c2np[i]);
  printf("N=%ld M=%ld W=%ld TB=%ld maxb=%d\n", N, M, W, TB, maxb);
  std::vector<float> x(N * 32), wv(M);
  std::normal_distribution<float> nd;
  for (auto& v : x) v = nd(rng);
  std::uniform_real_distribution<float> ud(0.f, 1.f);
  for (auto& v : wv) v = ud(rng);
  // reference (double)
  std::vector<double> yref(N * 32, 0.0);
  for (int64_t r = 0; r < N; ++r)
    for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e)
      for (int d = 0; d < 32; ++d) yref[r * 32 + d] += (double)wv[e] * x[col[e] * 32 + d];

  int64_t *dptr, *dboff;
  int* dc2np;
  uint32_t* defl;
  float *dw, *dx, *dy;
  CK(cudaMalloc(&dptr, 8 * (N + 1)));
  CK(cudaMalloc(&dboff, 8 * (W + 1)));
  CK(cudaMalloc(&dc2np, 4 * c2np.size()));
  CK(cudaMalloc(&defl, 4 * M));
  CK(cudaMalloc(&dw, 4 * M));
  CK(cudaMalloc(&dx, 4 * N * 32));
  CK(cudaMalloc(&dy, 4 * N * 32));
  CK(cudaMemcpy(dptr, ptr.data(), 8 * (N + 1), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dboff, boff.data(), 8 * (W + 1), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dc2np, c2np.data(), 4 * c2np.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(defl, efl.data(), 4 * M, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dw, wv.data(), 4 * M, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dx, x.data(), 4 * N * 32, cudaMemcpyHostToDevice));
  char* flush;
  const size_t FL = 512ull << 20;
  CK(cudaMalloc(&flush, FL));
  int nsm;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const int ctas_per_sm = argc > 1 ? atoi(argv[1]) : MINB;
  printf("WPC %d NB %d MAXB %d smem/cta %d\n", WPC, NB, MAXB, WPC * WARP_SMEM);
  const int blocks = nsm * ctas_per_sm;
  const int nwarps = blocks * WPC;
  std::vector<int> wst(nwarps + 1);
  for (int k = 0; k <= nwarps; ++k)
    wst[k] = (int)(std::lower_bound(boff.begin(), boff.begin() + W, (TB * k) / nwarps) - boff.begin());
  std::vector<int> wm(4 * nwarps);
  for (int k = 0; k < nwarps; ++k) { wm[4*k] = wst[k]; wm[4*k+1] = wst[k+1]; wm[4*k+2] = (int)boff[wst[k]]; wm[4*k+3] = (int)(boff[wst[k+1]] - boff[wst[k]]); }
  int* dwst;
  CK(cudaMalloc(&dwst, 16 * nwarps));
  CK(cudaMemcpy(dwst, wm.data(), 16 * nwarps, cudaMemcpyHostToDevice));
  P p{N, W, dptr, dboff, dc2np, defl, dw, dx, dy, 0, dwst};
  const int SMEM = WPC * WARP_SMEM;
  CK(cudaFuncSetAttribute(spmm_rd, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  p.nwarps = nwarps;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  std::vector<float> cold, warm;
  for (int it = 0; it < 30; ++it) {
#ifdef DBG
    if (it) break;
#endif
    CK(cudaMemsetAsync(flush, it & 255, FL));
    cudaEventRecord(a);
    spmm_rd<<<blocks, WPC * 32, SMEM>>>(p);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (it >= 3) cold.push_back(ms * 1000);
  }
  for (int it = 0; it < 30; ++it) {
    cudaEventRecord(a);
    spmm_rd<<<blocks, WPC * 32, SMEM>>>(p);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (it >= 3) warm.push_back(ms * 1000);
  }
  CK(cudaGetLastError());
  std::sort(cold.begin(), cold.end());
  std::sort(warm.begin(), warm.end());
  std::vector<float> y(N * 32);
  CK(cudaMemcpy(y.data(), dy, 4 * N * 32, cudaMemcpyDeviceToHost));
  double num = 0, den = 0;
  for (int64_t i = 0; i < N * 32; ++i) num += (y[i] - yref[i]) * (y[i] - yref[i]), den += yref[i] * yref[i];
  {
    int shown = 0; int64_t bad = 0;
    for (int64_t r = 0; r < N; ++r) {
      double nn = 0, dd = 0;
      for (int d = 0; d < 32; ++d) { double df = y[r*32+d] - yref[r*32+d]; nn += df*df; dd += yref[r*32+d]*yref[r*32+d]; }
      if (nn > 1e-6 * (dd + 1e-12)) { ++bad; if (shown < 6) { ++shown; printf("bad row %ld (win %ld, lw %ld): y[0..3]=%g %g %g %g ref %g %g %g %g\n", r, r/16, r%16, y[r*32], y[r*32+1], y[r*32+2], y[r*32+3], yref[r*32], yref[r*32+1], yref[r*32+2], yref[r*32+3]); } }
    }
    printf("bad rows %ld of %ld\n", bad, N);
  }
  const double U_ = (double)c2np.size();
  const double bytes = 8.0 * N * 32 + 8.0 * M + 4 * U_ + 8.0 * (N + 1) + 8.0 * (W + 1) + 4 * W;
  printf("ctas/sm=%d cold median %.2f us (min %.2f)  warm median %.2f us  relL2 %.3e  alg %.1f GB/s (frac %.3f)\n",
         ctas_per_sm, cold[cold.size() / 2], cold[0], warm[warm.size() / 2], std::sqrt(num / den),
         bytes / (cold[cold.size() / 2] * 1e3), bytes / (cold[cold.size() / 2] * 1e3) / 6549.8);
  return 0;
}
