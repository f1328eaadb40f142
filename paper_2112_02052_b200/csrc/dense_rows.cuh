// Pipelined row-tile dense kernels for the models' tall-skinny fp32 GEMMs
// (see dense.cu). Both stream 128-row tiles of the N-row operands through a
// cp.async multi-stage shared-memory ring (coalesced 16-B copies, several
// tiles in flight per SM) and are HBM-bound by design:
//
//  * dense_tile: Y = act((X .* [mask > 0]) . M + b). Thread (rg, q) owns
//    rows rg + 32 j (j < 4) x output columns 4q..4q+3; M is broadcast from
//    shared memory (one LDS.128 per 16 FMA), outputs leave as coalesced
//    float4 stores. CI > 64 is streamed in 32-wide k-chunks.
//  * gemm_tn_tile: per-CTA partial of A^T (B .* [mask > 0]) and colsum(B);
//    thread (og, rq) owns a 4 x 4 block of the product over a quarter of
//    every tile's rows; the row quarters are reduced in a fixed order at the
//    end (deterministic).
#pragma once

#include "common.cuh"

namespace tcg {
namespace dr {

__device__ __forceinline__ void cp16(void* dst, const void* src, bool valid) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  const int sz = valid ? 16 : 0;  // 0: zero-fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(sz)
               : "memory");
}
// 16-byte copy of the first `bytes` (0..16) bytes of src, the rest zero-filled
__device__ __forceinline__ void cp16n(void* dst, const void* src, int bytes) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// c.xyzw += a * w.xyzw as two packed fp32 FMAs (FFMA2 with a broadcast
// operand): each lane is an ordinary round-to-nearest fma, so the result is
// bitwise that of four fmaf, with half the FMA issue slots.
__device__ __forceinline__ void fma2x(float& c0, float& c1, float a, float w0, float w1) {
  unsigned long long cp, ap, wp, r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(cp) : "f"(c0), "f"(c1));
  asm("mov.b64 %0, {%1, %1};" : "=l"(ap) : "f"(a));
  asm("mov.b64 %0, {%1, %2};" : "=l"(wp) : "f"(w0), "f"(w1));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(ap), "l"(wp), "l"(cp));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(c0), "=f"(c1) : "l"(r));
}
__device__ __forceinline__ void fma4(float4& c, float a, const float4& w) {
  fma2x(c.x, c.y, a, w.x, w.y);
  fma2x(c.z, c.w, a, w.z, w.w);
}
__device__ __forceinline__ void fma4(float (&c)[4], float a, const float4& w) {
  fma2x(c[0], c[1], a, w.x, w.y);
  fma2x(c[2], c[3], a, w.z, w.w);
}

template <int CI, int CO, bool MASK>
struct DenseCfg {
  // k-chunk staged per pipeline item (a divisor of CI: 32 for 96 / 128, 20 for 100)
  static constexpr int KC = CI <= 64 ? CI : CI % 32 == 0 ? 32 : CI % 20 == 0 ? 20 : 4;
  static constexpr int NKC = CI / KC;
  static_assert(CI % KC == 0 && KC % 4 == 0, "dense_tile k-chunk");
  static constexpr int XS = KC + 4;  // padded row stride: conflict-free LDS.128
  static constexpr int Q = CO / 4;   // column quads
  static constexpr int NT = Q * 32;  // threads
  static constexpr int R = 4;        // rows per thread
  static constexpr int ROWS = 32 * R;
  static constexpr int STAGES = MASK ? 2 : 3;
  static constexpr int STAGE = ROWS * XS * (MASK ? 2 : 1);
  static constexpr size_t SMEM = (size_t)(CI * CO + STAGES * STAGE) * sizeof(float);
};

// y[n x co] = act((x .* [mask > 0]) . M + b); M [ci x co] (or [co x ci] when TRANS);
// CI = ci rounded up to a multiple of 4 (the columns past ci are zero-filled
// in shared memory, so padded-stride inputs need no clean padding), CO = co
// rounded up; ldx, ldm multiples of 4.
template <int CI, int CO, bool TRANS, bool MASK>
__global__ void __launch_bounds__(DenseCfg<CI, CO, MASK>::NT)
    dense_tile(const float* __restrict__ x, int64_t ldx, int64_t n, const float* __restrict__ m,
               int co, const float* __restrict__ bias, int relu, const float* __restrict__ mask,
               int64_t ldm, float* __restrict__ y, int64_t ldy, int vec_out, int ci) {
  using C = DenseCfg<CI, CO, MASK>;
  extern __shared__ __align__(16) float sh[];
  float* ws = sh;            // [CI][CO]
  float* ring = sh + CI * CO;  // STAGES x ([ROWS][XS] x, [ROWS][XS] mask)
  const int tid = threadIdx.x;
  const int q = tid % C::Q, rg = tid / C::Q;
  for (int i = tid; i < CI * CO; i += C::NT) {
    const int k = i / CO, c = i % CO;
    ws[i] = c < co && k < ci
                ? (TRANS ? __ldg(m + (int64_t)c * ci + k) : __ldg(m + (int64_t)k * co + c))
                : 0.f;
  }
  const int64_t ntiles = (n + C::ROWS - 1) / C::ROWS;
  const int64_t my_tiles =
      blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t items = my_tiles * C::NKC;

  auto issue = [&](int64_t it) {
    if (it < items) {
      const int64_t tile = blockIdx.x + (it / C::NKC) * gridDim.x;
      const int kc = (int)(it % C::NKC);
      float* st = ring + (it % C::STAGES) * C::STAGE;
      constexpr int F4 = C::KC / 4;
      for (int i = tid; i < C::ROWS * F4; i += C::NT) {
        const int r = i / F4, c4 = i % F4;
        const int64_t gr = tile * C::ROWS + r;
        const int col = kc * C::KC + c4 * 4;
        const int nb = gr < n ? min(16, max(0, 4 * (ci - col))) : 0;
        const int64_t grc = nb ? gr : 0;
        const int colc = nb ? col : 0;
        cp16n(st + r * C::XS + c4 * 4, x + grc * ldx + colc, nb);
        if (MASK) cp16n(st + C::ROWS * C::XS + r * C::XS + c4 * 4, mask + grc * ldm + colc, nb);
      }
    }
    cp_commit();
  };
#pragma unroll
  for (int s = 0; s < C::STAGES - 1; ++s) issue(s);

  float4 acc[C::R];
  const float4 b4 = (bias && 4 * q < co)
                        ? make_float4(__ldg(bias + 4 * q), 4 * q + 1 < co ? __ldg(bias + 4 * q + 1) : 0.f,
                                      4 * q + 2 < co ? __ldg(bias + 4 * q + 2) : 0.f,
                                      4 * q + 3 < co ? __ldg(bias + 4 * q + 3) : 0.f)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t it = 0; it < items; ++it) {
    issue(it + C::STAGES - 1);
    cp_wait<C::STAGES - 1>();
    __syncthreads();
    const int kc = (int)(it % C::NKC);
    if (kc == 0)
#pragma unroll
      for (int j = 0; j < C::R; ++j) acc[j] = b4;
    const float* st = ring + (it % C::STAGES) * C::STAGE;
    const float* wk = ws + kc * C::KC * CO + 4 * q;
#pragma unroll 2
    for (int k = 0; k < C::KC; k += 4) {
      float4 a[C::R];
#pragma unroll
      for (int j = 0; j < C::R; ++j) {
        a[j] = *reinterpret_cast<const float4*>(st + (rg + 32 * j) * C::XS + k);
        if (MASK) {
          const float4 mk =
              *reinterpret_cast<const float4*>(st + C::ROWS * C::XS + (rg + 32 * j) * C::XS + k);
          a[j].x = mk.x > 0.f ? a[j].x : 0.f, a[j].y = mk.y > 0.f ? a[j].y : 0.f;
          a[j].z = mk.z > 0.f ? a[j].z : 0.f, a[j].w = mk.w > 0.f ? a[j].w : 0.f;
        }
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const float4 w = *reinterpret_cast<const float4*>(wk + (k + kk) * CO);
#pragma unroll
        for (int j = 0; j < C::R; ++j) {
          const float av = kk == 0 ? a[j].x : kk == 1 ? a[j].y : kk == 2 ? a[j].z : a[j].w;
          fma4(acc[j], av, w);
        }
      }
    }
    if (kc == C::NKC - 1) {
      const int64_t tile = blockIdx.x + (it / C::NKC) * gridDim.x;
#pragma unroll
      for (int j = 0; j < C::R; ++j) {
        const int64_t row = tile * C::ROWS + rg + 32 * j;
        if (row >= n) continue;
        float4 v = acc[j];
        if (relu) v.x = fmaxf(v.x, 0.f), v.y = fmaxf(v.y, 0.f), v.z = fmaxf(v.z, 0.f), v.w = fmaxf(v.w, 0.f);
        float* yr = y + row * ldy + 4 * q;
        if (vec_out && 4 * q + 3 < co) {
          *reinterpret_cast<float4*>(yr) = v;
        } else {
          if (4 * q < co) yr[0] = v.x;
          if (4 * q + 1 < co) yr[1] = v.y;
          if (4 * q + 2 < co) yr[2] = v.z;
          if (4 * q + 3 < co) yr[3] = v.w;
        }
      }
    }
    __syncthreads();  // stage (it % STAGES) is refilled by the next iteration's issue
  }
  cp_wait<0>();
}

template <int CI, int CO, bool MASK>
struct GemmCfg {
  static constexpr int PB = CI % 8 == 0 && CI >= 64 ? 8 : 4;  // product rows per thread
  static constexpr int OG = (CI / PB) * (CO / 4);        // PB x 4 output blocks
  // row groups (a power of two dividing ROWS): ~256 threads per CTA
  static constexpr int RQ = OG >= 256 ? 1 : OG >= 128 ? 2 : OG >= 64 ? 4 : OG >= 32 ? 8 : 16;
  static constexpr int NT = OG * RQ;
  static constexpr int ROWS = CI <= 40 ? 128 : CI <= 64 ? 64 : 32;  // ring <= ~110 KB
  static constexpr int AS = CI + 4, BS = CO + 4;
  static constexpr int STAGES = 3;
  static constexpr int STAGE = ROWS * (AS + (MASK ? 2 : 1) * BS);
  static constexpr size_t SMEM_RING = (size_t)STAGES * STAGE * sizeof(float);
  static constexpr size_t SMEM_RED = (size_t)(RQ * CI * CO + RQ * CO) * sizeof(float);
  static constexpr size_t SMEM = SMEM_RING > SMEM_RED ? SMEM_RING : SMEM_RED;
};
static_assert(GemmCfg<128, 64, true>::SMEM <= 227 * 1024, "gemm_tn_tile smem");
static_assert(DenseCfg<128, 64, true>::SMEM <= 227 * 1024, "dense_tile smem");

// part[blockIdx] = A^T (B .* [mask > 0]) over this CTA's row tiles [CI x co];
// colpart[blockIdx] = colsum(B .* [mask > 0]). CI, CO multiples of 4 (CO = c
// rounded up; B's padding columns are read only when ldb allows, else zero).
template <int CI, int CO, bool MASK>
__global__ void __launch_bounds__(GemmCfg<CI, CO, MASK>::NT)
    gemm_tn_tile(const float* __restrict__ a, int64_t lda, const float* __restrict__ b,
                 int64_t ldb, const float* __restrict__ mask, int64_t ldm, int64_t n, int co,
                 float* __restrict__ part, float* __restrict__ colpart) {
  using C = GemmCfg<CI, CO, MASK>;
  extern __shared__ __align__(16) float sh[];
  const int tid = threadIdx.x;
  constexpr int PB = C::PB;
  const int og = tid % C::OG, rq = tid / C::OG;
  const int ib = og / (CO / 4), cb = og % (CO / 4);  // product rows PB ib.., cols 4cb..
  const int64_t ntiles = (n + C::ROWS - 1) / C::ROWS;
  const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int cq = (co + 3) / 4;  // B quads holding real columns

  auto issue = [&](int64_t it) {
    if (it < my_tiles) {
      const int64_t tile = blockIdx.x + it * gridDim.x;
      float* at = sh + (it % C::STAGES) * C::STAGE;
      float* bt = at + C::ROWS * C::AS;
      for (int i = tid; i < C::ROWS * (CI / 4); i += C::NT) {
        const int r = i / (CI / 4), c4 = i % (CI / 4);
        const int64_t gr = tile * C::ROWS + r;
        const bool ok = gr < n;
        cp16(at + r * C::AS + c4 * 4, a + (ok ? gr : 0) * lda + c4 * 4, ok);
      }
      for (int i = tid; i < C::ROWS * (CO / 4); i += C::NT) {
        const int r = i / (CO / 4), c4 = i % (CO / 4);
        const int64_t gr = tile * C::ROWS + r;
        const bool ok = gr < n && c4 < cq;
        cp16(bt + r * C::BS + c4 * 4, b + (ok ? gr : 0) * ldb + c4 * 4, ok);
        if (MASK)
          cp16(bt + C::ROWS * C::BS + r * C::BS + c4 * 4, mask + (ok ? gr : 0) * ldm + c4 * 4, ok);
      }
    }
    cp_commit();
  };
#pragma unroll
  for (int s = 0; s < C::STAGES - 1; ++s) issue(s);

  float acc[PB][4];
#pragma unroll
  for (int i = 0; i < PB; ++i)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[i][c] = 0.f;
  float4 cs = make_float4(0.f, 0.f, 0.f, 0.f);  // colsum of cols 4cb.. (ib == 0 threads)
  constexpr int RPG = C::ROWS / C::RQ;          // rows per group per tile
  for (int64_t it = 0; it < my_tiles; ++it) {
    issue(it + C::STAGES - 1);
    cp_wait<C::STAGES - 1>();
    __syncthreads();
    const float* at = sh + (it % C::STAGES) * C::STAGE;
    const float* bt = at + C::ROWS * C::AS;
#pragma unroll 4
    for (int rr = 0; rr < RPG; ++rr) {
      const int r = rq * RPG + rr;
      float ai[PB];
#pragma unroll
      for (int h = 0; h < PB / 4; ++h) {
        const float4 av = *reinterpret_cast<const float4*>(at + r * C::AS + PB * ib + 4 * h);
        ai[4 * h] = av.x, ai[4 * h + 1] = av.y, ai[4 * h + 2] = av.z, ai[4 * h + 3] = av.w;
      }
      float4 bv = *reinterpret_cast<const float4*>(bt + r * C::BS + 4 * cb);
      if (MASK) {
        const float4 mk = *reinterpret_cast<const float4*>(bt + C::ROWS * C::BS + r * C::BS + 4 * cb);
        bv.x = mk.x > 0.f ? bv.x : 0.f, bv.y = mk.y > 0.f ? bv.y : 0.f;
        bv.z = mk.z > 0.f ? bv.z : 0.f, bv.w = mk.w > 0.f ? bv.w : 0.f;
      }
#pragma unroll
      for (int i = 0; i < PB; ++i) {
        fma4(acc[i], ai[i], bv);
      }
      if (ib == 0) cs.x += bv.x, cs.y += bv.y, cs.z += bv.z, cs.w += bv.w;
    }
    __syncthreads();
  }
  cp_wait<0>();
  __syncthreads();
  // fixed-order reduction over the row groups through shared memory
  float* red = sh;  // [RQ][CI][CO] + [RQ][CO]
#pragma unroll
  for (int i = 0; i < PB; ++i)
#pragma unroll
    for (int c = 0; c < 4; ++c) red[(rq * CI + PB * ib + i) * CO + 4 * cb + c] = acc[i][c];
  if (ib == 0) {
    float* rc = red + C::RQ * CI * CO + rq * CO + 4 * cb;
    rc[0] = cs.x, rc[1] = cs.y, rc[2] = cs.z, rc[3] = cs.w;
  }
  __syncthreads();
  float* out = part + (int64_t)blockIdx.x * CI * co;
  for (int i = tid; i < CI * co; i += C::NT) {
    const int r = i / co, c = i % co;
    float s = 0.f;
    for (int g = 0; g < C::RQ; ++g) s += red[(g * CI + r) * CO + c];
    out[i] = s;
  }
  if (colpart)
    for (int c = tid; c < co; c += C::NT) {
      float s = 0.f;
      for (int g = 0; g < C::RQ; ++g) s += red[C::RQ * CI * CO + g * CO + c];
      colpart[(int64_t)blockIdx.x * co + c] = s;
    }
}

// Fused backward of y = x W (no activation), W [CI x CO]: one pass over the
// 128-row tiles of x [n x CI] and g [n x CO] computes
//   dx = g W^T  (thread (rg, q): rows rg + 32 j, columns 4q..4q+3, the
//               dense_tile<CO, CI, TRANS> dataflow and fold order), and
//   part[blockIdx] = x^T g over this CTA's tiles (thread (og, rq): a 4 x 4
//               block of dW over a quarter of each tile's rows; the row groups
//               are reduced in a fixed order, as gemm_tn_tile),
// so g is read once for both products. 256 threads: CI / 4 * 32 == 256.
template <int CI, int CO>
struct BwdCfg {
  static constexpr int ROWS = 128;
  static constexpr int XS = CI + 4, GS = CO + 4;
  static constexpr int STAGES = 2;  // 78 KB at 32 x 32: two CTAs per SM
  static constexpr int STAGE = ROWS * (XS + GS);
  static constexpr int NT = 256;
  static constexpr int Q = CI / 4;
  static constexpr int OG = (CI / 4) * (CO / 4);
  static constexpr int RQ = NT / OG;
  static_assert(Q * 32 == NT && OG * RQ == NT && ROWS % RQ == 0, "dense_bwd_tile shape");
  static constexpr size_t SMEM_RING = (size_t)(CO * CI + STAGES * STAGE) * sizeof(float);
  static constexpr size_t SMEM_RED = (size_t)RQ * CI * CO * sizeof(float);
  static constexpr size_t SMEM = SMEM_RING > SMEM_RED ? SMEM_RING : SMEM_RED;
};

template <int CI, int CO>
__global__ void __launch_bounds__(256)
    dense_bwd_tile(const float* __restrict__ x, int64_t ldx, const float* __restrict__ g,
                   int64_t ldg, int64_t n, const float* __restrict__ w, float* __restrict__ dx,
                   int64_t lddx, float* __restrict__ part) {
  using C = BwdCfg<CI, CO>;
  extern __shared__ __align__(16) float sh[];
  float* wt = sh;               // [CO][CI]: wt[k][c] = W[c][k]
  float* ring = sh + CO * CI;   // STAGES x ([ROWS][XS] x, [ROWS][GS] g)
  const int tid = threadIdx.x;
  for (int i = tid; i < CI * CO; i += C::NT) {
    const int k = i / CI, c = i % CI;
    wt[i] = __ldg(w + (int64_t)c * CO + k);
  }
  const int64_t ntiles = (n + C::ROWS - 1) / C::ROWS;
  const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto issue = [&](int64_t it) {
    if (it < my_tiles) {
      const int64_t tile = blockIdx.x + it * gridDim.x;
      float* xt = ring + (it % C::STAGES) * C::STAGE;
      float* gt = xt + C::ROWS * C::XS;
      for (int i = tid; i < C::ROWS * (CI / 4); i += C::NT) {
        const int r = i / (CI / 4), c4 = i % (CI / 4);
        const int64_t gr = tile * C::ROWS + r;
        const bool ok = gr < n;
        cp16(xt + r * C::XS + c4 * 4, x + (ok ? gr : 0) * ldx + c4 * 4, ok);
      }
      for (int i = tid; i < C::ROWS * (CO / 4); i += C::NT) {
        const int r = i / (CO / 4), c4 = i % (CO / 4);
        const int64_t gr = tile * C::ROWS + r;
        const bool ok = gr < n;
        cp16(gt + r * C::GS + c4 * 4, g + (ok ? gr : 0) * ldg + c4 * 4, ok);
      }
    }
    cp_commit();
  };
#pragma unroll
  for (int s = 0; s < C::STAGES - 1; ++s) issue(s);

  const int q = tid % C::Q, rg = tid / C::Q;                 // dx role
  const int og = tid % C::OG, rq = tid / C::OG;              // dW role
  const int ib = og / (CO / 4), cb = og % (CO / 4);
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[i][c] = 0.f;
  constexpr int RPG = C::ROWS / C::RQ;
  for (int64_t it = 0; it < my_tiles; ++it) {
    issue(it + C::STAGES - 1);
    cp_wait<C::STAGES - 1>();
    __syncthreads();
    const float* xt = ring + (it % C::STAGES) * C::STAGE;
    const float* gt = xt + C::ROWS * C::XS;
    // dx rows of this tile
    float4 d[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) d[j] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 2
    for (int k = 0; k < CO; k += 4) {
      float4 av[4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        av[j] = *reinterpret_cast<const float4*>(gt + (rg + 32 * j) * C::GS + k);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const float4 wv = *reinterpret_cast<const float4*>(wt + (k + kk) * CI + 4 * q);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float a = kk == 0 ? av[j].x : kk == 1 ? av[j].y : kk == 2 ? av[j].z : av[j].w;
          fma4(d[j], a, wv);
        }
      }
    }
    const int64_t tile = blockIdx.x + it * gridDim.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t row = tile * C::ROWS + rg + 32 * j;
      if (row < n) *reinterpret_cast<float4*>(dx + row * lddx + 4 * q) = d[j];
    }
    // dW partial over this thread's row group
#pragma unroll 4
    for (int rr = 0; rr < RPG; ++rr) {
      const int r = rq * RPG + rr;
      const float4 av = *reinterpret_cast<const float4*>(xt + r * C::XS + 4 * ib);
      const float4 bv = *reinterpret_cast<const float4*>(gt + r * C::GS + 4 * cb);
      const float ai[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        fma4(acc[i], ai[i], bv);
      }
    }
    __syncthreads();
  }
  cp_wait<0>();
  __syncthreads();
  float* red = sh;  // [RQ][CI][CO]
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int c = 0; c < 4; ++c) red[(rq * CI + 4 * ib + i) * CO + 4 * cb + c] = acc[i][c];
  __syncthreads();
  float* out = part + (int64_t)blockIdx.x * CI * CO;
  for (int i = tid; i < CI * CO; i += C::NT) {
    float s = 0.f;
    for (int gq = 0; gq < C::RQ; ++gq) s += red[gq * CI * CO + i];
    out[i] = s;
  }
}

}  // namespace dr
}  // namespace tcg
