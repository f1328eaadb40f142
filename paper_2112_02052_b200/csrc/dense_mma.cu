// 32 x 32 dense layers on the tensor cores with fp32-class accuracy (3xTF32):
// the AGNN convolution weights (Z = H W) and their backward
// dH = dZ W^T, dW = H^T dZ.
//
// The FFMA2 tile kernels (dense_rows.cuh) read W and the staged rows back from
// shared memory in 8-lane phases that all address the same 128 B, so at 32 x 32
// they spend four L1 wavefronts per LDS.128 and are bound by the L1 pipe
// (0.42 / 0.36 of HBM). Here each warp owns 16-row tiles:
//   * the rows arrive with cp.async in a 128-B-row XOR swizzle and are read as
//     mma A fragments with ldmatrix.x4 (a 32-bit element is a pair of b16, so
//     ldmatrix's (row i/4, column i%4) word is exactly the m16n8k8 TF32 A slot);
//   * W's B fragments (hi and lo, 64 registers) are loaded once per warp;
//   * each k chunk does D += Ahi.Bhi + Ahi.Blo + Alo.Bhi with the residuals
//     lo = x - tf32(x) (tf32 = cvt.rn: the reference quantizer's RNE);
//   * output feature 4n + j sits in column n of n-tile j, so a lane's eight
//     accumulators of a row are eight consecutive features: two 16-B stores.
// The backward runs the same product with W^T for dH and accumulates the
// per-warp partial dW = H^T dZ (A = H^T and B = dZ fragments from the staged
// tiles), reduced per CTA in a fixed order, then by sum_slabs (dense.cu).
#include <cstdlib>

#include "common.cuh"

namespace tcg {
namespace dm {

constexpr int WPC = 4;  // warps per CTA

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ float tf32f(float x) { return __uint_as_float(tf32_rn(x)); }

// staged tile: 16 rows x 32 floats, 16-B chunk c of row r at r * 128 + ((c ^ (r & 7)) * 16)
__device__ __forceinline__ uint32_t sw(int r, int c) { return r * 128 + ((c ^ (r & 7)) << 4); }

__device__ __forceinline__ void cp16z(uint32_t d, const void* s, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(s), "r"(ok ? 16 : 0) : "memory");
}

// rows [row0, row0 + 16) of a [n x 32] matrix into a staged tile (zero past n)
__device__ __forceinline__ void stage_rows(uint32_t tile, const float* __restrict__ x, int64_t ldx, int64_t n,
                                           int64_t row0, int lane) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = (lane >> 3) + 4 * i, c = lane & 7;
    const int64_t gr = row0 + r;
    const bool ok = gr < n;
    cp16z(tile + sw(r, c), x + (ok ? gr : 0) * ldx + 4 * c, ok);
  }
}

// A fragment (16 rows x 8 k) of k chunk kc from a staged tile
__device__ __forceinline__ void ldm_a(uint32_t (&a)[4], uint32_t tile, int kc, int lane) {
  const int m = lane >> 3, rr = lane & 7;
  const int r = rr + 8 * (m & 1), c = 2 * kc + (m >> 1);
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3])
               : "r"(tile + sw(r, c)));
}

__device__ __forceinline__ void mma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// split fp32 words into tf32 hi (RNE) and the tf32 of the residual
__device__ __forceinline__ void split(const uint32_t (&a)[4], uint32_t (&hi)[4], uint32_t (&lo)[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float v = __uint_as_float(a[i]);
    hi[i] = tf32_rn(v);
    lo[i] = tf32_rn(v - __uint_as_float(hi[i]));
  }
}

// B fragments of M (32 x 32, m(k, c) = trans ? w[c * 32 + k] : w[k * 32 + c]) in the
// permuted column order: n-tile j, column n <-> output 4n + j
__device__ __forceinline__ void load_b(uint32_t (&bh)[4][4][2], uint32_t (&bl)[4][4][2], const float* __restrict__ w,
                                       int trans, int lane) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int kc = 0; kc < 4; ++kc)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int k = 8 * kc + t + 4 * h, c = 4 * g + j;
        const float v = trans ? __ldg(w + c * 32 + k) : __ldg(w + k * 32 + c);
        bh[kc][j][h] = tf32_rn(v);
        bl[kc][j][h] = tf32_rn(v - __uint_as_float(bh[kc][j][h]));
      }
}

// acc[j][.] += A (16 x 32, staged) . M (3xTF32)
__device__ __forceinline__ void tile_times(float (&acc)[4][4], uint32_t tile, const uint32_t (&bh)[4][4][2],
                                           const uint32_t (&bl)[4][4][2], int lane) {
#pragma unroll
  for (int kc = 0; kc < 4; ++kc) {
    uint32_t a[4], ah[4], al[4];
    ldm_a(a, tile, kc, lane);
    split(a, ah, al);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      mma(acc[j], al, bh[kc][j][0], bh[kc][j][1]);
      mma(acc[j], ah, bl[kc][j][0], bl[kc][j][1]);
      mma(acc[j], ah, bh[kc][j][0], bh[kc][j][1]);
    }
  }
}

// rows g / g+8 of the tile: outputs 8t .. 8t+7 (acc[j][2h] = feature 8t + j, acc[j][2h+1] = 8t + 4 + j)
__device__ __forceinline__ void store_tile(const float (&acc)[4][4], float* __restrict__ y, int64_t ldy, int64_t n,
                                           int64_t row0, const float* __restrict__ bias, int relu, int lane) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t r = row0 + g + 8 * h;
    if (r >= n) continue;
    float o[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = acc[j][2 * h], o[4 + j] = acc[j][2 * h + 1];
    if (bias) {
#pragma unroll
      for (int q = 0; q < 8; ++q) o[q] += __ldg(bias + 8 * t + q);
    }
    if (relu) {
#pragma unroll
      for (int q = 0; q < 8; ++q) o[q] = fmaxf(o[q], 0.f);
    }
    float4* yr = reinterpret_cast<float4*>(y + r * ldy + 8 * t);
    yr[0] = make_float4(o[0], o[1], o[2], o[3]);
    yr[1] = make_float4(o[4], o[5], o[6], o[7]);
  }
}

// y = act(x M + b), M = W or W^T (32 x 32); persistent warps over 16-row tiles
__global__ void __launch_bounds__(WPC * 32) mma32_fwd(const float* __restrict__ x, int64_t ldx, int64_t n,
                                                       const float* __restrict__ w, int trans,
                                                       const float* __restrict__ bias, int relu,
                                                       float* __restrict__ y, int64_t ldy) {
  constexpr int RD = 4;  // tiles in flight per warp
  __shared__ __align__(128) unsigned char sm[WPC][RD][2048];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * WPC + wid, nw = (int64_t)gridDim.x * WPC;
  const int64_t tiles = (n + 15) / 16;
  uint32_t bh[4][4][2], bl[4][4][2];
  load_b(bh, bl, w, trans, lane);
  const uint32_t tb = su(&sm[wid][0][0]);
  int64_t tile = gw;
#pragma unroll
  for (int i = 0; i < RD - 1; ++i) {
    if (tile + i * nw < tiles) stage_rows(tb + 2048 * i, x, ldx, n, (tile + i * nw) * 16, lane);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  for (int it = 0; tile < tiles; tile += nw, ++it) {
    const uint32_t cur = tb + 2048 * (it % RD);
    const int64_t ahead = tile + (RD - 1) * nw;
    if (ahead < tiles) stage_rows(tb + 2048 * ((it + RD - 1) % RD), x, ldx, n, ahead * 16, lane);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group %0;\n" ::"n"(RD - 1) : "memory");
    __syncwarp();
    float acc[4][4] = {};
    tile_times(acc, cur, bh, bl, lane);
    store_tile(acc, y, ldy, n, tile * 16, bias, relu, lane);
    __syncwarp();  // the next stage_rows into this buffer comes after every lane's ldmatrix
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// dx = g W^T per tile; per-CTA partial dW = x^T g into part[blockIdx.x][32][32]
__global__ void __launch_bounds__(WPC * 32) mma32_bwd(const float* __restrict__ x, int64_t ldx,
                                                       const float* __restrict__ g, int64_t ldg, int64_t n,
                                                       const float* __restrict__ w, float* __restrict__ dx,
                                                       int64_t lddx, float* __restrict__ part) {
  constexpr int RD = 2;  // tiles in flight per warp
  __shared__ __align__(128) unsigned char sm[WPC][RD][2][2048];  // [warp][buffer][x | g]
  float (*red)[32][33] = reinterpret_cast<float (*)[32][33]>(&sm[0][0][0][0]);  // reused at the end
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int gq = lane >> 2, t = lane & 3;
  const int64_t gw = (int64_t)blockIdx.x * WPC + wid, nw = (int64_t)gridDim.x * WPC;
  const int64_t tiles = (n + 15) / 16;
  uint32_t bh[4][4][2], bl[4][4][2];
  load_b(bh, bl, w, 1, lane);  // W^T
  // dW partial: D[m][c] = sum_r x[r][m] g[r][c]; m-tile mt (features 16 mt ..), n-tile j
  // (columns in the permuted order 4n + j) -> 2 x 4 accumulators
  float dw[2][4][4] = {};
  // buffer b of this warp: x tile at wbase + 4096 b, g tile 2048 B after it
  const unsigned char* wbase = &sm[wid][0][0][0];
  const uint32_t wbase_s = su(wbase);
  auto word = [&](const unsigned char* tl, int r, int f) {  // staged element (row r, feature f)
    return *reinterpret_cast<const float*>(tl + sw(r, f >> 2) + 4 * (f & 3));
  };
  int64_t tile = gw;
#pragma unroll
  for (int i = 0; i < RD - 1; ++i) {
    if (tile + i * nw < tiles) {
      stage_rows(wbase_s + 4096 * i, x, ldx, n, (tile + i * nw) * 16, lane);
      stage_rows(wbase_s + 4096 * i + 2048, g, ldg, n, (tile + i * nw) * 16, lane);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  for (int it = 0; tile < tiles; tile += nw, ++it) {
    const int cb = it % RD, nb = (it + RD - 1) % RD;
    const uint32_t xcur = wbase_s + 4096 * cb, gcur = xcur + 2048;
    const unsigned char* xsc = wbase + 4096 * cb;
    const unsigned char* gsc = xsc + 2048;
    const int64_t ahead = tile + (RD - 1) * nw;
    if (ahead < tiles) {
      stage_rows(wbase_s + 4096 * nb, x, ldx, n, ahead * 16, lane);
      stage_rows(wbase_s + 4096 * nb + 2048, g, ldg, n, ahead * 16, lane);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group %0;\n" ::"n"(RD - 1) : "memory");
    __syncwarp();
    // dx tile = g tile . W^T
    float acc[4][4] = {};
    tile_times(acc, gcur, bh, bl, lane);
    store_tile(acc, dx, lddx, n, tile * 16, nullptr, 0, lane);
    // dW += x_tile^T . g_tile: A = x^T (m = feature, k = row), B = g (k = row, n = output)
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {  // rows 8 ks .. 8 ks + 7
      uint32_t bgh[4][2], bgl[4][2];
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float v = word(gsc, 8 * ks + t + 4 * h, 4 * gq + j);
          bgh[j][h] = tf32_rn(v);
          bgl[j][h] = tf32_rn(v - __uint_as_float(bgh[j][h]));
        }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        uint32_t a[4], ah[4], al[4];
        a[0] = __float_as_uint(word(xsc, 8 * ks + t, 16 * mt + gq));
        a[1] = __float_as_uint(word(xsc, 8 * ks + t, 16 * mt + gq + 8));
        a[2] = __float_as_uint(word(xsc, 8 * ks + t + 4, 16 * mt + gq));
        a[3] = __float_as_uint(word(xsc, 8 * ks + t + 4, 16 * mt + gq + 8));
        split(a, ah, al);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          mma(dw[mt][j], al, bgh[j][0], bgh[j][1]);
          mma(dw[mt][j], ah, bgl[j][0], bgl[j][1]);
          mma(dw[mt][j], ah, bgh[j][0], bgh[j][1]);
        }
      }
    }
    __syncwarp();
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();  // every warp is done with its staging buffers
  // dw[mt][j]: (m = 16 mt + gq (+8 for regs 2,3), output 4 (2t) + j / 4 (2t+1) + j)
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int m = 16 * mt + gq + 8 * (q >> 1);
        const int c = 4 * (2 * t + (q & 1)) + j;
        red[wid][m][c] = dw[mt][j][q];
      }
  __syncthreads();
  for (int i = threadIdx.x; i < 1024; i += WPC * 32) {
    const int m = i >> 5, c = i & 31;
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < WPC; ++q) s += red[q][m][c];
    part[(int64_t)blockIdx.x * 1024 + i] = s;
  }
}

}  // namespace dm

// 1 = not covered
int dense_mma32(const float* x, int64_t ldx, int64_t n, int ci, const float* w, int co, bool trans,
                const float* bias, int relu, const float* mask, float* y, int64_t ldy, cudaStream_t s) {
  static const bool off = std::getenv("TCG_NO_MMA32") != nullptr;  // A/B: FFMA2 tile kernels
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (off || ci != 32 || co != 32 || mask || n < 1 || !al(x) || !al(y) || ldx % 4 || ldy % 4) return 1;
  static int per_sm = 0;  // one resident wave of persistent warps
  if (per_sm == 0) {
    TCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dm::mma32_fwd, dm::WPC * 32, 0),
             "mma32_fwd occupancy");
    if (per_sm < 1) per_sm = 1;
  }
  const int64_t tiles = (n + 15) / 16;
  int64_t blocks = (tiles + dm::WPC - 1) / dm::WPC;
  const int64_t cap = (int64_t)num_sms() * per_sm;
  if (blocks > cap) blocks = cap;
  dm::mma32_fwd<<<(unsigned)blocks, dm::WPC * 32, 0, s>>>(x, ldx, n, w, trans ? 1 : 0, bias, relu, y, ldy);
  TCG_LAUNCHED("mma32_fwd");
  return TCG_OK;
}

int64_t dense_mma32_bwd_slabs() {  // one resident wave (<= 4 per SM: the workspace bound)
  static int per_sm = 0;
  if (per_sm == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dm::mma32_bwd, dm::WPC * 32, 0) != cudaSuccess ||
        per_sm < 1)
      per_sm = 1;
    if (per_sm > 4) per_sm = 4;
  }
  return (int64_t)num_sms() * per_sm;
}

// dx = g W^T and per-CTA partials of dW = x^T g (*slabs of them); 1 = not covered
int dense_mma32_bwd(const float* x, int64_t ldx, const float* g, int64_t ldg, int64_t n, const float* w,
                    float* dx, int64_t lddx, float* part, int64_t* slabs, cudaStream_t s) {
  static const bool off = std::getenv("TCG_NO_MMA32") != nullptr;
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (off || n < 1 || !al(x) || !al(g) || !al(dx) || ldx % 4 || ldg % 4 || lddx % 4) return 1;
  const int64_t tiles = (n + 15) / 16;
  int64_t blocks = (tiles + dm::WPC - 1) / dm::WPC;
  const int64_t cap = dense_mma32_bwd_slabs();
  if (blocks > cap) blocks = cap;
  dm::mma32_bwd<<<(unsigned)blocks, dm::WPC * 32, 0, s>>>(x, ldx, g, ldg, n, w, dx, lddx, part);
  TCG_LAUNCHED("mma32_bwd");
  *slabs = blocks;
  return TCG_OK;
}

}  // namespace tcg
