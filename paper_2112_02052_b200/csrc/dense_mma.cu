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
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];\n" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];\n" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ float tf32f(float x) { return __uint_as_float(tf32_rn(x)); }

// staged tile: 16 rows x 32 floats, 16-B chunk c of row r at r * 128 + ((c ^ (r & 7)) * 16)
__device__ __forceinline__ uint32_t sw(int r, int c) { return r * 128 + ((c ^ (r & 7)) << 4); }

__device__ __forceinline__ void cp16z(uint32_t d, const void* s, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(s), "r"(ok ? 16 : 0) : "memory");
}
// 16-B copy of the first `bytes` (0..16) bytes, zero-filling the rest
__device__ __forceinline__ void cp16n(uint32_t d, const void* s, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(s), "r"(bytes) : "memory");
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
    if (relu & 1) {
#pragma unroll
      for (int q = 0; q < 8; ++q) o[q] = fmaxf(o[q], 0.f);
    }
    if (relu & TCG_DENSE_OUT_TF32) {  // stored on the tf32 grid (RN) for tf32 consumers
#pragma unroll
      for (int q = 0; q < 8; ++q) o[q] = __uint_as_float(tf32_rn(o[q]));
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
  TCG_PDL_ENTRY();
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
  TCG_PDL_ENTRY();
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
  ::tcg::launch_pdl(dm::mma32_fwd, (unsigned)blocks, dm::WPC * 32, 0, s, x, ldx, n, w, trans ? 1 : 0, bias, relu, y, ldy);
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
  ::tcg::launch_pdl(dm::mma32_bwd, (unsigned)blocks, dm::WPC * 32, 0, s, x, ldx, g, ldg, n, w, dx, lddx, part);
  TCG_LAUNCHED("mma32_bwd");
  *slabs = blocks;
  return TCG_OK;
}

}  // namespace tcg

// ---- output layer fused with the softmax cross-entropy ----------------------
//
// logits = x W + b (x: [n x kin], kin <= 32; W: [kin x c], c <= 8 NTL) on mma.sync
// 3xTF32, and in the epilogue -- each quad of lanes holds a whole row -- the
// row's log-sum-exp, the NLL of its label and dlogits = (softmax - onehot) / div.
// The logits never reach memory; dlogits does (the backward reads it), and the
// per-warp loss partials are summed in row order (deterministic), then by
// final_loss. Classes >= c are masked to -inf.
namespace tcg {
namespace dm {

// rows [row0, row0 + 16) of a [n x kin] matrix (kin a multiple of 4, <= 8 KT) into a
// staged 16 x 32 tile (its first 2 KT 16-B chunks per row), zero past kin and past n
template <int KT>
__device__ __forceinline__ void stage_rows_k(uint32_t tile, const float* __restrict__ x, int64_t ldx, int64_t n,
                                             int kin, int64_t row0, int lane) {
  constexpr int CH = 2 * KT;
#pragma unroll
  for (int i = 0; i < KT; ++i) {
    const int q = lane + 32 * i, r = q / CH, c = q % CH;
    const int64_t gr = row0 + r;
    const bool ok = gr < n && 4 * c < kin;
    cp16z(tile + sw(r, c), x + (ok ? gr : 0) * ldx + (ok ? 4 * c : 0), ok);
  }
}

// The logits are carried in log2 units (W and the bias pre-scaled by log2 e),
// so the softmax runs on MUFU ex2 / lg2 directly.
constexpr float kLog2e = 1.4426950408889634f, kLn2 = 0.6931471805599453f;
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// W (kin x c) * log2 e as tf32 hi / lo in shared memory, [feature][class] with a
// pitch that keeps both fragment reads conflict-free (row stride = 8 or 24 banks)
constexpr int lx_pitch(int ntl) { return (ntl * 8) % 16 == 8 ? ntl * 8 : ntl * 8 + 8; }

template <int NTL, int KT>
struct LxW {
  float v[2][KT * 8][lx_pitch(NTL)];
};

template <int NTL, int KT>
__device__ __forceinline__ void lx_load_w(LxW<NTL, KT>& ws, const float* __restrict__ w, int kin, int c) {
  constexpr int WP = lx_pitch(NTL);
  for (int i = threadIdx.x; i < KT * 8 * WP; i += blockDim.x) {
    const int k = i / WP, cl = i % WP;
    const float v = (k < kin && cl < c) ? __ldg(w + (int64_t)k * c + cl) * kLog2e : 0.f;
    const float hi = tf32f(v);
    ws.v[0][k][cl] = hi;
    ws.v[1][k][cl] = tf32f(v - hi);
  }
}

// bias * log2 e per owned class (8 j + 2 t + e); -inf masks the padding classes
template <int NTL>
__device__ __forceinline__ void lx_bias(float (&bv)[NTL][2], const float* __restrict__ bias, int c, int t) {
#pragma unroll
  for (int j = 0; j < NTL; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int cl = 8 * j + 2 * t + e;
      bv[j][e] = cl < c ? (bias ? __ldg(bias + cl) * kLog2e : 0.f) : -INFINITY;
    }
}

// logits (log2 units) of the staged 16-row tile, 3xTF32: acc[j] = rows g / g + 8, classes 8 j + 2 t (+1)
template <int NTL, int KT>
__device__ __forceinline__ void lx_logits(float (&acc)[NTL][4], uint32_t cur, uint32_t wh, uint32_t wl, int lane) {
  constexpr int WP = lx_pitch(NTL);
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int j = 0; j < NTL; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
#pragma unroll
  for (int kc = 0; kc < KT; ++kc) {
    uint32_t a[4], ah[4], al[4];
    ldm_a(a, cur, kc, lane);
    split(a, ah, al);
#pragma unroll
    for (int j = 0; j < NTL; ++j) {
      const uint32_t o0 = ((8 * kc + t) * WP + 8 * j + g) * 4, o1 = o0 + 4 * WP * 4;
      const uint32_t h0 = lds32(wh + o0), h1 = lds32(wh + o1), l0 = lds32(wl + o0), l1 = lds32(wl + o1);
      mma(acc[j], al, h0, h1);
      mma(acc[j], ah, l0, l1);
      mma(acc[j], ah, h0, h1);
    }
  }
}

// adds the bias to row half h (rows g / g + 8) and returns its log2-sum-exp2 (quad-wide)
template <int NTL>
__device__ __forceinline__ float lx_lse(float (&v)[NTL][4], const float (&bv)[NTL][2], int h) {
  float mx = -INFINITY;
#pragma unroll
  for (int j = 0; j < NTL; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      v[j][2 * h + e] += bv[j][e];
      mx = fmaxf(mx, v[j][2 * h + e]);
    }
  mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
  mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
  float sm = 0.f;
#pragma unroll
  for (int j = 0; j < NTL; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) sm += ex2(v[j][2 * h + e] - mx);
  sm += __shfl_xor_sync(0xffffffffu, sm, 1);
  sm += __shfl_xor_sync(0xffffffffu, sm, 2);
  return mx + lg2(sm);
}

// labels of rows g, g + 8 of a tile (0 past n), loaded one tile ahead
__device__ __forceinline__ void lx_labels(int64_t (&lab)[2], const int64_t* __restrict__ labels, int64_t n,
                                          int64_t tile, int64_t tiles, int g) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t row = tile * 16 + g + 8 * h;
    lab[h] = (tile < tiles && row < n) ? __ldg(labels + row) : 0;
  }
}

template <int NTL, int KT>
__global__ void __launch_bounds__(WPC * 32, 4) linear_xent(const float* __restrict__ x, int64_t ldx, int64_t n,
                                                         int kin, const float* __restrict__ w, int c,
                                                         const float* __restrict__ bias,
                                                         const int64_t* __restrict__ labels, float inv_div,
                                                         float* __restrict__ dl, int64_t ldd,
                                                         float* __restrict__ lpart) {
  TCG_PDL_ENTRY();
  constexpr int RD = 3;
  __shared__ __align__(128) unsigned char sm[WPC][RD][2048];
  __shared__ LxW<NTL, KT> ws;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t gw = (int64_t)blockIdx.x * WPC + wid, nw = (int64_t)gridDim.x * WPC;
  const int64_t tiles = (n + 15) / 16;
  const uint32_t tb = su(&sm[wid][0][0]);
  int64_t tile = gw;
#pragma unroll
  for (int i = 0; i < RD - 1; ++i) {
    if (tile + i * nw < tiles) stage_rows_k<KT>(tb + 2048 * i, x, ldx, n, kin, (tile + i * nw) * 16, lane);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  lx_load_w(ws, w, kin, c);
  float bv[NTL][2];
  lx_bias(bv, bias, c, t);
  int64_t lab[2];
  lx_labels(lab, labels, n, tile, tiles, g);
  __syncthreads();
  const uint32_t wh = su(&ws.v[0][0][0]), wl = su(&ws.v[1][0][0]);
  float wsum = 0.f;  // this warp's loss, in row order
  const float bad = __int_as_float(0x7fc00000);
  for (int it = 0; tile < tiles; tile += nw, ++it) {
    const uint32_t cur = tb + 2048 * (it % RD);
    const int64_t ahead = tile + (RD - 1) * nw;
    if (ahead < tiles) stage_rows_k<KT>(tb + 2048 * ((it + RD - 1) % RD), x, ldx, n, kin, ahead * 16, lane);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    int64_t labn[2];
    lx_labels(labn, labels, n, tile + nw, tiles, g);
    asm volatile("cp.async.wait_group %0;\n" ::"n"(RD - 1) : "memory");
    __syncwarp();
    float v[NTL][4];
    lx_logits<NTL, KT>(v, cur, wh, wl, lane);
    __syncwarp();  // the staging slot is refilled after every lane's ldmatrix
    float tsum = 0.f;
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // rows g, g + 8 of the tile; the quad holds the row
      const int64_t row = tile * 16 + g + 8 * h;
      const float lse = lx_lse(v, bv, h);
      const bool ok = lab[h] >= 0 && lab[h] < c;
      // the label's logit, held by lane t = (lab >> 1) & 3 of the quad: a select
      // tree over the n-tiles (lab >> 3) instead of a compare per class
      const int lb = (int)lab[h];
      float cand[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) cand[j] = j < NTL ? ((lb & 1) ? v[j < NTL ? j : 0][2 * h + 1] : v[j < NTL ? j : 0][2 * h]) : 0.f;
#pragma unroll
      for (int lvl = 0; lvl < 3; ++lvl) {
        const bool bit = (lb >> (3 + lvl)) & 1;
#pragma unroll
        for (int i = 0; i < (4 >> lvl); ++i) cand[i] = bit ? cand[2 * i + 1] : cand[2 * i];
      }
      float ly = ((lb >> 1) & 3) == t ? cand[0] : 0.f;
      ly += __shfl_xor_sync(0xffffffffu, ly, 1);
      ly += __shfl_xor_sync(0xffffffffu, ly, 2);
      if (dl && row < n) {  // dl null: the loss only (the backward recomputes)
        float* dr = dl + row * ldd;
#pragma unroll
        for (int j = 0; j < NTL; ++j) {
          const int cl = 8 * j + 2 * t;
          float d[2];
#pragma unroll
          for (int e = 0; e < 2; ++e)
            d[e] = ok ? (ex2(v[j][2 * h + e] - lse) - (cl + e == lab[h] ? 1.f : 0.f)) * inv_div : bad;
          if (cl + 1 < c && (ldd % 2) == 0) *reinterpret_cast<float2*>(dr + cl) = make_float2(d[0], d[1]);
          else {
            if (cl < c) dr[cl] = d[0];
            if (cl + 1 < c) dr[cl + 1] = d[1];
          }
        }
      }
      const float lrow = row < n ? (ok ? (lse - ly) * kLn2 : bad) : 0.f;
      tsum += (t == 0) ? lrow : 0.f;  // rows g (h = 0) then g + 8 (h = 1)
    }
    // tile sum over g in a fixed tree order (lanes t = 0 hold the values)
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) tsum += __shfl_xor_sync(0xffffffffu, tsum, o);
    wsum += tsum;
    lab[0] = labn[0];
    lab[1] = labn[1];
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  if (lane == 0) lpart[gw] = wsum;
}

// The backward of linear_xent, recomputing instead of storing dlogits: per
// 16-row tile the logits again (3xTF32), d = (softmax - onehot) * g / div in
// registers, dx = d W^T (mma, the class index permuted so the accumulator
// layout is the A fragment: k-slot t <-> class 2t, t + 4 <-> 2t + 1), and the
// warp's running dW += x^T d (d through shared memory: its rows must move from
// the g to the t lane index) and db += colsum d. Per CTA partials
// [kin x c | c] in fixed warp order; sum_slabs finishes (deterministic).
template <int NTL, int KT>
__global__ void __launch_bounds__(WPC * 32, 3) linear_xent_bwd(
    const float* __restrict__ x, int64_t ldx, int64_t n, int kin, const float* __restrict__ w, int c,
    const float* __restrict__ bias, const int64_t* __restrict__ labels, const float* __restrict__ gscale,
    float inv_div, float* __restrict__ dx, int64_t lddx, float* __restrict__ part) {
  TCG_PDL_ENTRY();
  constexpr int RD = 2, WP = lx_pitch(NTL), MT = KT / 2, PW = KT * 8 * NTL * 8 + NTL * 8;
  constexpr int RING = WPC * RD * 2048, DSM = WPC * 16 * WP * 4, RED = WPC * PW * 4;
  constexpr int UNI = (RING + DSM) > RED ? (RING + DSM) : RED;
  __shared__ __align__(128) unsigned char smu[UNI];
  __shared__ LxW<NTL, KT> ws;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t gw = (int64_t)blockIdx.x * WPC + wid, nw = (int64_t)gridDim.x * WPC;
  const int64_t tiles = (n + 15) / 16;
  const uint32_t tb = su(smu + wid * RD * 2048);
  int64_t tile = gw;
#pragma unroll
  for (int i = 0; i < RD - 1; ++i) {
    if (tile + i * nw < tiles) stage_rows_k<KT>(tb + 2048 * i, x, ldx, n, kin, (tile + i * nw) * 16, lane);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  lx_load_w(ws, w, kin, c);
  float bv[NTL][2];
  lx_bias(bv, bias, c, t);
  int64_t lab[2];
  lx_labels(lab, labels, n, tile, tiles, g);
  const float gs = (gscale ? __ldg(gscale) : 1.f) * inv_div;
  __syncthreads();
  float* dsm = reinterpret_cast<float*>(smu + RING) + wid * 16 * WP;
  const uint32_t wh = su(&ws.v[0][0][0]), wl = su(&ws.v[1][0][0]);
  float aw[MT][NTL][4] = {}, ab[NTL][2] = {};
  const float bad = __int_as_float(0x7fc00000);
  for (int it = 0; tile < tiles; tile += nw, ++it) {
    const uint32_t cur = tb + 2048 * (it % RD);
    const int64_t ahead = tile + (RD - 1) * nw;
    if (ahead < tiles) stage_rows_k<KT>(tb + 2048 * ((it + RD - 1) % RD), x, ldx, n, kin, ahead * 16, lane);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    int64_t labn[2];
    lx_labels(labn, labels, n, tile + nw, tiles, g);
    asm volatile("cp.async.wait_group %0;\n" ::"n"(RD - 1) : "memory");
    __syncwarp();
    float d[NTL][4];
    lx_logits<NTL, KT>(d, cur, wh, wl, lane);
    // d = (softmax - onehot) * g / div; 0 on padding rows and classes
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t row = tile * 16 + g + 8 * h;
      const float lse = lx_lse(d, bv, h);
      const bool in = row < n;
      const bool ok = lab[h] >= 0 && lab[h] < c;
#pragma unroll
      for (int j = 0; j < NTL; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int cl = 8 * j + 2 * t + e;
          const float p = (ex2(d[j][2 * h + e] - lse) - (cl == lab[h] ? 1.f : 0.f)) * gs;
          d[j][2 * h + e] = !in || cl >= c ? 0.f : (ok ? p : bad);
        }
    }
    lab[0] = labn[0];
    lab[1] = labn[1];
    // dx = d W^T
    if (dx) {
      float ax[KT][4] = {};
#pragma unroll
      for (int j = 0; j < NTL; ++j) {
        const uint32_t a[4] = {__float_as_uint(d[j][0]), __float_as_uint(d[j][2]), __float_as_uint(d[j][1]),
                               __float_as_uint(d[j][3])};
        uint32_t ah[4], al[4];
        split(a, ah, al);
#pragma unroll
        for (int nf = 0; nf < KT; ++nf) {
          const uint32_t o = ((8 * nf + g) * WP + 8 * j + 2 * t) * 4;
          const uint2 h = lds64(wh + o), l = lds64(wl + o);
          mma(ax[nf], al, h.x, h.y);
          mma(ax[nf], ah, l.x, l.y);
          mma(ax[nf], ah, h.x, h.y);
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t row = tile * 16 + g + 8 * h;
        if (row >= n) continue;
#pragma unroll
        for (int nf = 0; nf < KT; ++nf) {
          const int f = 8 * nf + 2 * t;
          float* dr = dx + row * lddx + f;
          // the staged W carries log2 e
          const float v0 = ax[nf][2 * h] * kLn2, v1 = ax[nf][2 * h + 1] * kLn2;
          if (f + 1 < kin && (lddx % 2) == 0)
            *reinterpret_cast<float2*>(dr) = make_float2(v0, v1);
          else {
            if (f < kin) dr[0] = v0;
            if (f + 1 < kin) dr[1] = v1;
          }
        }
      }
    }
    // db += colsum d; d to shared memory, rows on the t index for dW += x^T d
#pragma unroll
    for (int j = 0; j < NTL; ++j) {
      ab[j][0] += d[j][0] + d[j][2];
      ab[j][1] += d[j][1] + d[j][3];
      *reinterpret_cast<float2*>(dsm + g * WP + 8 * j + 2 * t) = make_float2(d[j][0], d[j][1]);
      *reinterpret_cast<float2*>(dsm + (g + 8) * WP + 8 * j + 2 * t) = make_float2(d[j][2], d[j][3]);
    }
    __syncwarp();
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      const int r0 = 8 * kk + t, r1 = r0 + 4;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int f0 = 16 * mt + g, f1 = f0 + 8;
        const uint32_t a[4] = {lds32(cur + sw(r0, f0 >> 2) + (f0 & 3) * 4),
                               lds32(cur + sw(r0, f1 >> 2) + (f1 & 3) * 4),
                               lds32(cur + sw(r1, f0 >> 2) + (f0 & 3) * 4),
                               lds32(cur + sw(r1, f1 >> 2) + (f1 & 3) * 4)};
        uint32_t ah[4], al[4];
        split(a, ah, al);
#pragma unroll
        for (int j = 0; j < NTL; ++j) {
          const float b0 = dsm[r0 * WP + 8 * j + g], b1 = dsm[r1 * WP + 8 * j + g];
          const uint32_t bh0 = tf32_rn(b0), bh1 = tf32_rn(b1);
          const uint32_t bl0 = tf32_rn(b0 - __uint_as_float(bh0)), bl1 = tf32_rn(b1 - __uint_as_float(bh1));
          mma(aw[mt][j], al, bh0, bh1);
          mma(aw[mt][j], ah, bl0, bl1);
          mma(aw[mt][j], ah, bh0, bh1);
        }
      }
    }
    __syncwarp();  // the x slot and dsm are rewritten next tile
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  // db over the 8 row groups (fixed order)
#pragma unroll
  for (int j = 0; j < NTL; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) ab[j][e] += __shfl_xor_sync(0xffffffffu, ab[j][e], o);
  __syncthreads();  // the ring / dsm become the reduction area
  float* red = reinterpret_cast<float*>(smu) + wid * PW;
  const int kw = KT * 8, cw = NTL * 8;
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int j = 0; j < NTL; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) red[(16 * mt + g + 8 * (q >> 1)) * cw + 8 * j + 2 * t + (q & 1)] = aw[mt][j][q];
  if (g == 0)
#pragma unroll
    for (int j = 0; j < NTL; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) red[kw * cw + 8 * j + 2 * t + e] = ab[j][e];
  __syncthreads();
  // CTA partial [kin x c | c], warps summed in order
  const float* r = reinterpret_cast<const float*>(smu);
  float* out = part + (int64_t)blockIdx.x * (kin * c + c);
  for (int i = threadIdx.x; i < kin * c + c; i += WPC * 32) {
    const int src = i < kin * c ? (i / c) * cw + i % c : kw * cw + (i - kin * c);
    float v = 0.f;
#pragma unroll
    for (int q = 0; q < WPC; ++q) v += r[q * PW + src];
    out[i] = v;
  }
}


// ---- weight gradients of the wide input layers: dW = A^T (B .* [M > 0]) --------
//
// A [n x k] (k <= 128, a multiple of 4), B / M [n x CO] (CO 16 or 32): one CTA of
// 8 warps per 32-row chunk, warp w owning features 16 w .. 16 w + 15 (the M
// dimension of m16n8k8, with the chunk's rows as K), 3xTF32. A, B and M stream
// through a 3-stage cp.async ring shared by the CTA (A rows padded to 136
// floats: the t / t + 4 row reads land 8 banks apart). Per-CTA partials of dW
// and of the column sums of B .* [M > 0]; sum_slabs finishes (deterministic).
namespace gt {
constexpr int R = 32, S = 3, AP = 136;
template <int CO>
struct Smem {
  static constexpr int BP = CO + 8;
  float a[S][R][AP];
  float b[S][R][BP];
  float m[S][R][BP];
  float bh[R][BP], bl[R][BP];  // the chunk's B .* [M > 0], tf32 hi / lo (split once per CTA)
  float cs[256 / CO][CO];      // column-sum partials per row residue
};
}  // namespace gt

template <int CO>
__global__ void __launch_bounds__(256, 2) gemm_tn_mma(const float* __restrict__ a, int64_t lda,
                                                       const float* __restrict__ b, int64_t ldb,
                                                       const float* __restrict__ mk, int64_t ldm, int64_t n,
                                                       int k, float* __restrict__ part,
                                                       float* __restrict__ colpart) {
  TCG_PDL_ENTRY();
  using namespace gt;
  using Sm = Smem<CO>;
  constexpr int BP = Sm::BP, NJ = CO / 8;
  extern __shared__ __align__(128) unsigned char gsm[];
  Sm& sm = *reinterpret_cast<Sm*>(gsm);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t chunks = (n + R - 1) / R;
  // blockIdx.y: 128-feature panel of A (k > 128); the partial rows k0 .. k0 + kp
  const int k0 = 128 * blockIdx.y, kp = min(128, k - k0);
  a += k0;
  const int kc = (kp + 3) / 4;  // 16-B chunks per A row (a partial last one zero-filled)
  auto stage = [&](int slot, int64_t ch) {
    const int64_t r0 = ch * R;
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // A: 32 rows x 32 chunks
      const int q = tid + 256 * i, r = q >> 5, c = q & 31;
      const bool ok = r0 + r < n && c < kc;
      cp16n(su(&sm.a[slot][r][4 * c]), a + (ok ? (r0 + r) * lda + 4 * c : 0), ok ? 4 * min(4, kp - 4 * c) : 0);
    }
    if (tid < R * CO / 4) {  // B (and M): 32 rows x CO / 4 chunks
      const int r = tid / (CO / 4), c = tid % (CO / 4);
      const bool ok = r0 + r < n;
      cp16z(su(&sm.b[slot][r][4 * c]), b + (ok ? (r0 + r) * ldb + 4 * c : 0), ok);
      if (mk) cp16z(su(&sm.m[slot][r][4 * c]), mk + (ok ? (r0 + r) * ldm + 4 * c : 0), ok);
    }
  };
  int64_t ch = blockIdx.x;
#pragma unroll
  for (int i = 0; i < S - 1; ++i) {
    if (ch + i * (int64_t)gridDim.x < chunks) stage(i, ch + i * (int64_t)gridDim.x);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  float acc[NJ][4] = {};
  float csum[R * CO / 256] = {};  // this thread's column (tid % CO) over its rows, in order
  const bool active = 16 * w < kp;
  const int f0 = 16 * w + g, f1 = f0 + 8;
  for (int it = 0; ch < chunks; ch += gridDim.x, ++it) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(S - 2) : "memory");
    __syncthreads();
    const int slot = it % S;
    {  // the slot computed last iteration is free for the chunk S - 1 ahead
      const int64_t ahead = ch + (int64_t)(S - 1) * gridDim.x;
      if (ahead < chunks) stage((it + S - 1) % S, ahead);
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    // B .* [M > 0] split once for all warps, column sums on the way
#pragma unroll
    for (int i = 0; i < R * CO / 256; ++i) {
      const int e = tid + 256 * i, r = e / CO, c = e % CO;
      float v = sm.b[slot][r][c];
      if (mk) v = sm.m[slot][r][c] > 0.f ? v : 0.f;
      csum[i] += v;
      const float hi = tf32f(v);
      sm.bh[r][c] = hi;
      sm.bl[r][c] = tf32f(v - hi);
    }
    __syncthreads();
    if (!active) continue;
    // the chunk's products start from zero and are folded into acc with FADD
    // (RNE): the tensor-core accumulation chain stays 12 deep, not the whole slab
    float ca[NJ][4] = {};
#pragma unroll
    for (int ks = 0; ks < R / 8; ++ks) {
      const int r0 = 8 * ks + t, r1 = r0 + 4;
      const uint32_t av[4] = {__float_as_uint(sm.a[slot][r0][f0]), __float_as_uint(sm.a[slot][r0][f1]),
                              __float_as_uint(sm.a[slot][r1][f0]), __float_as_uint(sm.a[slot][r1][f1])};
      uint32_t ah[4], al[4];
      split(av, ah, al);
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const uint32_t bh0 = __float_as_uint(sm.bh[r0][8 * j + g]), bh1 = __float_as_uint(sm.bh[r1][8 * j + g]);
        const uint32_t bl0 = __float_as_uint(sm.bl[r0][8 * j + g]), bl1 = __float_as_uint(sm.bl[r1][8 * j + g]);
        mma(ca[j], al, bh0, bh1);
        mma(ca[j], ah, bl0, bl1);
        mma(ca[j], ah, bh0, bh1);
      }
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[j][q] += ca[j][q];
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  float* pp = part + (int64_t)blockIdx.x * k * CO + (int64_t)k0 * CO;
  if (active) {
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int c = 8 * j + 2 * t;
      if (f0 < kp) *reinterpret_cast<float2*>(pp + (int64_t)f0 * CO + c) = make_float2(acc[j][0], acc[j][1]);
      if (f1 < kp) *reinterpret_cast<float2*>(pp + (int64_t)f1 * CO + c) = make_float2(acc[j][2], acc[j][3]);
    }
  }
  if (colpart && blockIdx.y == 0) {  // rows r = tid / CO + (256 / CO) i: fold the row residues in order
    float v = 0.f;
#pragma unroll
    for (int i = 0; i < R * CO / 256; ++i) v += csum[i];
    __syncthreads();
    sm.cs[tid / CO][tid % CO] = v;
    __syncthreads();
    if (tid < CO) {
      float tot = 0.f;
#pragma unroll
      for (int q = 0; q < 256 / CO; ++q) tot += sm.cs[q][tid];
      colpart[(int64_t)blockIdx.x * CO + tid] = tot;
    }
  }
}

// ---- the wide input layers: Y = act(X W + b), X [n x ci] (ci <= 128), W [ci x CO] ----
//
// One CTA of 4 warps per 64-row chunk through a 2-stage cp.async ring (rows of
// 512 B, 16-B chunk c of row r at r * 512 + ((c ^ (r & 7)) << 4): ldmatrix
// conflict-free); warp w computes rows 16 w .. + 15 of the chunk for every
// n-tile (each A fragment is split into tf32 hi / lo once), 3xTF32 with W
// (tf32 hi / lo) in shared memory.
namespace di {
constexpr int R = 64, S = 2;
template <int CO>
struct Smem {
  static constexpr int WP = CO + 8;  // B fragment reads: rows t / t + 4 land 8 banks apart
  unsigned char x[S][R * 512];
  float wh[128][WP], wl[128][WP];
};
}  // namespace di

template <int CO>
__global__ void __launch_bounds__(128, 2) dense_in_mma(const float* __restrict__ x, int64_t ldx, int64_t n, int ci,
                                                        const float* __restrict__ w, const float* __restrict__ bias,
                                                        int relu, float* __restrict__ y, int64_t ldy) {
  TCG_PDL_ENTRY();
  using namespace di;
  using Sm = Smem<CO>;
  constexpr int WP = Sm::WP, NJ = CO / 8, NT = 128;
  extern __shared__ __align__(128) unsigned char dsm_[];
  Sm& sm = *reinterpret_cast<Sm*>(dsm_);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int rg = wid, j0 = 0;  // warp w: rows 16 w .. 16 w + 15 of the chunk, every n-tile
  const int64_t chunks = (n + R - 1) / R;
  const int kc8 = (ci + 7) / 8;
  auto stage = [&](int slot, int64_t ch) {
    const uint32_t base = su(&sm.x[slot][0]);
    const int64_t r0 = ch * R;
#pragma unroll
    for (int i = 0; i < 16; ++i) {  // 64 rows x 32 chunks
      const int q = tid + NT * i, r = q >> 5, c = q & 31;
      const bool ok = r0 + r < n && 4 * c < ci;  // a partial last chunk is zero-filled past ci
      cp16n(base + r * 512 + ((c ^ (r & 7)) << 4), x + (ok ? (r0 + r) * ldx + 4 * c : 0),
            ok ? 4 * min(4, ci - 4 * c) : 0);
    }
  };
  int64_t ch = blockIdx.x;
  if (ch < chunks) stage(0, ch);
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  for (int i = tid; i < 128 * CO; i += NT) {
    const int k = i / CO, c = i % CO;
    const float v = k < ci ? __ldg(w + (int64_t)k * CO + c) : 0.f;
    const float hi = tf32f(v);
    sm.wh[k][c] = hi;
    sm.wl[k][c] = tf32f(v - hi);
  }
  float bv[NJ][2];
#pragma unroll
  for (int j = 0; j < NJ; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) bv[j][e] = bias ? __ldg(bias + 8 * (j0 + j) + 2 * t + e) : 0.f;
  const uint32_t wh = su(&sm.wh[0][0]), wl = su(&sm.wl[0][0]);
  for (int it = 0; ch < chunks; ch += gridDim.x, ++it) {
    const int slot = it & 1;
    {
      const int64_t ahead = ch + gridDim.x;
      if (ahead < chunks) stage(slot ^ 1, ahead);
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    __syncthreads();
    const uint32_t tile = su(&sm.x[slot][0]);
    // two accumulator sets (k chunks even / odd), added at the end: the
    // tensor-core accumulation chains stay half as deep
    float acc[2][NJ][4] = {};
    const int m = lane >> 3, rr = lane & 7;
    const int ar = 16 * rg + rr + 8 * (m & 1);
    auto kstep = [&](int kc, float (&ac)[NJ][4]) {
      uint32_t a[4], ah[4], al[4];
      const int c = 2 * kc + (m >> 1);
      asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                   : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3])
                   : "r"(tile + ar * 512 + ((c ^ (ar & 7)) << 4)));
      split(a, ah, al);
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const uint32_t o0 = ((8 * kc + t) * WP + 8 * (j0 + j) + g) * 4, o1 = o0 + 4 * WP * 4;
        const uint32_t h0 = lds32(wh + o0), h1 = lds32(wh + o1), l0 = lds32(wl + o0), l1 = lds32(wl + o1);
        mma(ac[j], al, h0, h1);
        mma(ac[j], ah, l0, l1);
        mma(ac[j], ah, h0, h1);
      }
    };
    int kc = 0;
#pragma unroll 2
    for (; kc + 1 < kc8; kc += 2) {
      kstep(kc, acc[0]);
      kstep(kc + 1, acc[1]);
    }
    if (kc < kc8) kstep(kc, acc[0]);
    __syncthreads();  // the slot is restaged next iteration
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t row = ch * R + 16 * rg + g + 8 * h;
      if (row >= n) continue;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        float v0 = acc[0][j][2 * h] + acc[1][j][2 * h] + bv[j][0];
        float v1 = acc[0][j][2 * h + 1] + acc[1][j][2 * h + 1] + bv[j][1];
        if (relu) v0 = fmaxf(v0, 0.f), v1 = fmaxf(v1, 0.f);
        *reinterpret_cast<float2*>(y + row * ldy + 8 * (j0 + j) + 2 * t) = make_float2(v0, v1);
      }
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// ---- input layers wider than 128 features (Cora 1433, Pubmed 500): K panels ----
//
// dense_in_mma's layout with the K dimension walked in 128-feature panels: the
// ring stages (row chunk, panel) items, X rows and the raw W panel together,
// and W is split into tf32 hi / lo at the fragment load. The accumulators of a
// row chunk live across its panels (even / odd panels in separate sets).
namespace dw {
constexpr int R = 64, S = 2;
template <int CO>
struct Smem {
  static constexpr int WP = CO + 8;
  unsigned char x[S][R * 512];
  float w[S][128][WP];
};
}  // namespace dw

template <int CO>
__global__ void __launch_bounds__(128, 2) dense_wide_mma(const float* __restrict__ x, int64_t ldx, int64_t n,
                                                          int ci, const float* __restrict__ w,
                                                          const float* __restrict__ bias, int relu,
                                                          float* __restrict__ y, int64_t ldy) {
  TCG_PDL_ENTRY();
  using namespace dw;
  using Sm = Smem<CO>;
  constexpr int WP = Sm::WP, NJ = CO / 8, NT = 128;
  extern __shared__ __align__(128) unsigned char wsm_[];
  Sm& sm = *reinterpret_cast<Sm*>(wsm_);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t chunks = (n + R - 1) / R;
  const int panels = (ci + 127) / 128;
  const int64_t mine = chunks > blockIdx.x ? (chunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t items = mine * panels;
  auto stage = [&](int slot, int64_t item) {
    const int64_t ch = blockIdx.x + (item / panels) * gridDim.x;
    const int k0 = (int)(item % panels) * 128;
    const int kv = min(128, ci - k0);  // features of this panel
    const uint32_t base = su(&sm.x[slot][0]);
    const int64_t r0 = ch * R;
#pragma unroll
    for (int i = 0; i < 16; ++i) {  // 64 rows x 32 chunks
      const int q = tid + NT * i, r = q >> 5, c = q & 31;
      const bool ok = r0 + r < n && 4 * c < kv;  // a partial last chunk is zero-filled past kv
      cp16n(base + r * 512 + ((c ^ (r & 7)) << 4), x + (ok ? (r0 + r) * ldx + k0 + 4 * c : 0),
            ok ? 4 * min(4, kv - 4 * c) : 0);
    }
    // the W panel: 128 rows x CO (CO / 4 chunks per row)
    for (int q = tid; q < 128 * CO / 4; q += NT) {
      const int r = q / (CO / 4), c = q % (CO / 4);
      const bool ok = r < kv;
      cp16z(su(&sm.w[slot][r][4 * c]), w + (ok ? (int64_t)(k0 + r) * CO + 4 * c : 0), ok);
    }
  };
  float bv[NJ][2];
#pragma unroll
  for (int j = 0; j < NJ; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) bv[j][e] = bias ? __ldg(bias + 8 * j + 2 * t + e) : 0.f;
  if (items > 0) stage(0, 0);
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  float acc[NJ][4] = {};
  const int m = lane >> 3, rr = lane & 7;
  const int ar = 16 * wid + rr + 8 * (m & 1);
  for (int64_t it = 0; it < items; ++it) {
    const int slot = (int)(it & 1);
    if (it + 1 < items) stage(slot ^ 1, it + 1);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    __syncthreads();
    const uint32_t tile = su(&sm.x[slot][0]);
    const int p = (int)(it % panels);
    const int kc8 = (min(128, ci - 128 * p) + 7) / 8;
    // per panel: even / odd k chunks in fresh accumulators (24-deep tensor-core
    // chains), folded into acc with FADD (RNE) -- K = 1433 stays fp32-class
    float c0[NJ][4] = {}, c1[NJ][4] = {};
    auto kstep = [&](int kc, float (&ac)[NJ][4]) {
      uint32_t a[4], ah[4], al[4];
      const int c = 2 * kc + (m >> 1);
      asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                   : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3])
                   : "r"(tile + ar * 512 + ((c ^ (ar & 7)) << 4)));
      split(a, ah, al);
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const float w0 = sm.w[slot][8 * kc + t][8 * j + g], w1 = sm.w[slot][8 * kc + t + 4][8 * j + g];
        const uint32_t h0 = tf32_rn(w0), h1 = tf32_rn(w1);
        const uint32_t l0 = tf32_rn(w0 - __uint_as_float(h0)), l1 = tf32_rn(w1 - __uint_as_float(h1));
        mma(ac[j], al, h0, h1);
        mma(ac[j], ah, l0, l1);
        mma(ac[j], ah, h0, h1);
      }
    };
    int kc = 0;
    for (; kc + 1 < kc8; kc += 2) {
      kstep(kc, c0);
      kstep(kc + 1, c1);
    }
    if (kc < kc8) kstep(kc, c0);
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[j][q] += c0[j][q] + c1[j][q];
    __syncthreads();  // the slot is restaged next iteration
    if (p == panels - 1) {  // the row chunk is complete
      const int64_t ch = blockIdx.x + (it / panels) * gridDim.x;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t row = ch * R + 16 * wid + g + 8 * h;
        if (row < n) {
#pragma unroll
          for (int j = 0; j < NJ; ++j) {
            float v0 = acc[j][2 * h] + bv[j][0];
            float v1 = acc[j][2 * h + 1] + bv[j][1];
            if (relu) v0 = fmaxf(v0, 0.f), v1 = fmaxf(v1, 0.f);
            *reinterpret_cast<float2*>(y + row * ldy + 8 * j + 2 * t) = make_float2(v0, v1);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < NJ; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}
}  // namespace dm

// one resident wave of persistent warps per kernel instantiation
template <typename K>
int64_t lx_wave(K kern) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, dm::WPC * 32, 0) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  return (int64_t)num_sms() * std::min(per_sm, 8);
}

// the per-warp loss partials / per-CTA gradient slabs the workspaces hold (the
// grid never exceeds 8 CTAs per SM)
int64_t linear_xent_parts(int64_t n) {
  return std::min<int64_t>(((n + 15) / 16 + dm::WPC - 1) / dm::WPC, (int64_t)num_sms() * 8) * dm::WPC;
}
int64_t linear_xent_bwd_slabs(int64_t n) {
  return std::min<int64_t>(((n + 15) / 16 + dm::WPC - 1) / dm::WPC, (int64_t)num_sms() * 8);
}

static bool lx_covered(const float* x, int64_t ldx, int64_t n, int kin, int c) {
  static const bool off = std::getenv("TCG_NO_FUSED_XENT") != nullptr;
  return !off && n >= 1 && kin >= 4 && kin <= 32 && kin % 4 == 0 && c >= 1 && c <= 48 &&
         (reinterpret_cast<uintptr_t>(x) & 15) == 0 && ldx % 4 == 0;
}

// dispatch on (class tiles, kin <= 16); F(NV, KV) launches one instantiation
#define TCG_LX_DISPATCH(F)                  \
  switch ((c + 7) / 8) {                    \
    case 1: if (kin <= 16) F(1, 2) else F(1, 4) break; \
    case 2: if (kin <= 16) F(2, 2) else F(2, 4) break; \
    case 3: if (kin <= 16) F(3, 2) else F(3, 4) break; \
    case 4: if (kin <= 16) F(4, 2) else F(4, 4) break; \
    case 5: if (kin <= 16) F(5, 2) else F(5, 4) break; \
    case 6: if (kin <= 16) F(6, 2) else F(6, 4) break; \
  }

int linear_xent_bwd(const float* x, int64_t ldx, int64_t n, int kin, const float* w, int c, const float* bias,
                    const int64_t* labels, const float* gscale, float inv_div, float* dx, int64_t lddx, float* part,
                    int64_t* slabs, cudaStream_t s) {
  if (!lx_covered(x, ldx, n, kin, c)) return 1;
  int64_t blocks = linear_xent_bwd_slabs(n);
#define TCG_LXB(NV, KV)                                                                                  \
  {                                                                                                      \
    static const int64_t wave = lx_wave(dm::linear_xent_bwd<NV, KV>);                                    \
    blocks = std::min(blocks, wave);                                                                     \
    ::tcg::launch_pdl(dm::linear_xent_bwd<NV, KV>, (unsigned)blocks, dm::WPC * 32, 0, s, x, ldx, n, kin, w, c, bias,    \
                                                                         labels, gscale, inv_div, dx,   \
                                                                         lddx, part);                    \
  }
  TCG_LX_DISPATCH(TCG_LXB)
#undef TCG_LXB
  TCG_LAUNCHED("linear_xent_bwd");
  *slabs = blocks;
  return TCG_OK;
}

// loss = sum_rows NLL / div into lpart (one partial per warp of the grid, *nparts);
// dl = dlogits / div (dl may be null). 1 = shape not covered.
int linear_xent(const float* x, int64_t ldx, int64_t n, int kin, const float* w, int c, const float* bias,
                const int64_t* labels, float inv_div, float* dl, int64_t ldd, float* lpart, int64_t cap_parts,
                int64_t* nparts, cudaStream_t s) {
  if (!lx_covered(x, ldx, n, kin, c)) return 1;
  int64_t blocks = std::min(linear_xent_parts(n), cap_parts) / dm::WPC;
  if (blocks < 1) return 1;
#define TCG_LXF(NV, KV)                                                                                  \
  {                                                                                                      \
    static const int64_t wave = lx_wave(dm::linear_xent<NV, KV>);                                        \
    blocks = std::min(blocks, wave);                                                                     \
    ::tcg::launch_pdl(dm::linear_xent<NV, KV>, (unsigned)blocks, dm::WPC * 32, 0, s, x, ldx, n, kin, w, c, bias, labels, \
                                                                     inv_div, dl, ldd, lpart);          \
  }
  TCG_LX_DISPATCH(TCG_LXF)
#undef TCG_LXF
  TCG_LAUNCHED("linear_xent");
  *nparts = blocks * dm::WPC;
  return TCG_OK;
}
#undef TCG_LX_DISPATCH


// dW = A^T (B .* [M > 0]) partials (and column-sum partials) on the tensor cores;
// 1 = shape not covered. *used = CTAs (slabs) written, <= cap_slabs.
int gemm_tn_mma(const float* a, int64_t lda, const float* b, int64_t ldb, const float* mask, int64_t ldm,
                int64_t n, int k, int c, float* part, float* colpart, int64_t cap_slabs, int64_t* used,
                cudaStream_t s) {
  static const bool off = std::getenv("TCG_NO_GEMM_TN_MMA") != nullptr;
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (off || n < 1024 || k < 33 || (c != 16 && c != 32) || !al(a) || !al(b) || lda % 4 || ldb % 4 ||
      (mask && (!al(mask) || ldm % 4)))
    return 1;
  const unsigned panels = (unsigned)((k + 127) / 128);
  const int64_t chunks = (n + dm::gt::R - 1) / dm::gt::R;
#define TCG_GTM(CV)                                                                                    \
  {                                                                                                    \
    auto kern = dm::gemm_tn_mma<CV>;                                                                   \
    const int smem = (int)sizeof(dm::gt::Smem<CV>);                                                    \
    static int per_sm = 0;                                                                             \
    if (per_sm == 0) {                                                                                 \
      TCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),         \
               "gemm_tn_mma attr");                                                                    \
      TCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem),               \
               "gemm_tn_mma occupancy");                                                               \
      if (per_sm < 1) per_sm = 1;                                                                      \
    }                                                                                                  \
    const int64_t grid = std::min<int64_t>(std::min<int64_t>((int64_t)num_sms() * per_sm, chunks), cap_slabs); \
    ::tcg::launch_pdl(kern, dim3((unsigned)grid, panels), 256, smem, s, a, lda, b, ldb, mask, ldm, n, k, part, colpart); \
    *used = grid;                                                                                      \
  }
  if (c == 16) TCG_GTM(16) else TCG_GTM(32)
#undef TCG_GTM
  TCG_LAUNCHED("gemm_tn_mma");
  return TCG_OK;
}


// Y = act(X W + b) for the wide input layers (ci 33..128 -> 16 / 32, n >= 4096) on
// mma.sync 3xTF32; 1 = shape not covered.
int dense_in_mma(const float* x, int64_t ldx, int64_t n, int ci, const float* w, int co, bool trans,
                 const float* bias, int relu, const float* mask, float* y, int64_t ldy, cudaStream_t s) {
  static const bool off = std::getenv("TCG_NO_DENSE_IN_MMA") != nullptr;
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (off || trans || mask || n < 4096 || ci < 33 || ci > 128 || (co != 16 && co != 32) || !al(x) ||
      ldx % 4 || (reinterpret_cast<uintptr_t>(y) & 7) || ldy % 2)
    return 1;
  const int64_t chunks = (n + dm::di::R - 1) / dm::di::R;
#define TCG_DIM(CV)                                                                                     \
  {                                                                                                     \
    auto kern = dm::dense_in_mma<CV>;                                                                   \
    const int smem = (int)sizeof(dm::di::Smem<CV>);                                                     \
    static int per_sm = 0;                                                                              \
    if (per_sm == 0) {                                                                                  \
      TCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),          \
               "dense_in_mma attr");                                                                    \
      TCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, smem),                \
               "dense_in_mma occupancy");                                                               \
      if (per_sm < 1) per_sm = 1;                                                                       \
    }                                                                                                   \
    const int64_t grid = std::min<int64_t>((int64_t)num_sms() * per_sm, chunks);                        \
    ::tcg::launch_pdl(kern, (unsigned)grid, 128, smem, s, x, ldx, n, ci, w, bias, relu, y, ldy);         \
  }
  if (co == 16) TCG_DIM(16) else TCG_DIM(32)
#undef TCG_DIM
  TCG_LAUNCHED("dense_in_mma");
  return TCG_OK;
}


// Y = act(X W + b) for inputs wider than 128 features (-> 16 / 32) on mma.sync
// 3xTF32, K in 128-feature panels; 1 = shape not covered.
int dense_wide_mma(const float* x, int64_t ldx, int64_t n, int ci, const float* w, int co, bool trans,
                   const float* bias, int relu, const float* mask, float* y, int64_t ldy, cudaStream_t s) {
  static const bool off = std::getenv("TCG_NO_DENSE_IN_MMA") != nullptr;
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (off || trans || mask || n < 256 || ci <= 128 || (co != 16 && co != 32) || !al(x) || !al(w) ||
      ldx % 4 || (reinterpret_cast<uintptr_t>(y) & 7) || ldy % 2)
    return 1;
  const int64_t chunks = (n + dm::dw::R - 1) / dm::dw::R;
#define TCG_DWM(CV)                                                                                     \
  {                                                                                                     \
    auto kern = dm::dense_wide_mma<CV>;                                                                 \
    const int smem = (int)sizeof(dm::dw::Smem<CV>);                                                     \
    static int per_sm = 0;                                                                              \
    if (per_sm == 0) {                                                                                  \
      TCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),          \
               "dense_wide_mma attr");                                                                  \
      TCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, smem),                \
               "dense_wide_mma occupancy");                                                             \
      if (per_sm < 1) per_sm = 1;                                                                       \
    }                                                                                                   \
    const int64_t grid = std::min<int64_t>((int64_t)num_sms() * per_sm, chunks);                        \
    ::tcg::launch_pdl(kern, (unsigned)grid, 128, smem, s, x, ldx, n, ci, w, bias, relu, y, ldy);         \
  }
  if (co == 16) TCG_DWM(16) else TCG_DWM(32)
#undef TCG_DWM
  TCG_LAUNCHED("dense_wide_mma");
  return TCG_OK;
}

}  // namespace tcg
