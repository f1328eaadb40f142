// Dense companions of the sparse layers: the tall-skinny fp32 GEMMs of
// GCNConv / AGNNConv / Linear (N up to millions of rows, feature widths
// <= a few hundred) and the fused softmax cross-entropy of the models'
// output layer. cuBLAS picks
// split-K "largek" kernels for A^T B with K = N (ncu: ~0.5 ms per weight
// gradient on the arxiv shape); these kernels are HBM-bound instead:
//
//  * rows_x_small: Y[n x co] = act((X .* [mask > 0]) . M + b), M given
//    as [ci x co] or transposed [co x ci]; 64-row CTA tiles, X and M staged
//    through shared memory in 32-wide k-chunks, 4 x CT outputs per thread.
//  * gemm_tn: Out[k x c] = A^T B (B optionally masked by mask > 0) and
//    colsum(B) — per-slab partial tiles, then a fixed-order sum over slabs
//    (deterministic, no atomics).
//  * softmax_xent: per row log-softmax, NLL of the label, and
//    dlogits = (softmax - onehot) / n; the mean loss by a fixed-order
//    two-level reduction.
// All fp32 FMA (no TF32) so the GEMMs keep full fp32 accuracy (SURVEY.md
// fact 8: TF32 GEMMs would push the 4-layer AGNN past the 5e-3 budget).
#include <type_traits>

#include "common.cuh"
#include "dense_rows.cuh"

namespace tcg {
namespace {

constexpr int kRowsTile = 64;
constexpr int kKChunk = 32;

// CT = output columns per thread (16 column groups x CT = co padded)
template <int CT, bool TRANS>
__global__ void __launch_bounds__(256)
    rows_x_small(const float* __restrict__ x, int64_t ldx, int64_t n, int ci,
                 const float* __restrict__ m, int co, const float* __restrict__ bias, int relu,
                 const float* __restrict__ mask, int64_t ldm, float* __restrict__ y, int64_t ldy) {
  __shared__ float xs[kRowsTile][kKChunk + 1];
  __shared__ float ms[kKChunk][16 * CT];
  const int tid = threadIdx.x;
  const int cg = tid & 15, rg = tid >> 4;  // column group, row group (16 x 16)
  const int64_t row0 = (int64_t)blockIdx.x * kRowsTile;
  const int cbase = blockIdx.y * 16 * CT;  // output column tile
  float acc[4][CT];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < CT; ++c) acc[r][c] = 0.f;
  for (int k0 = 0; k0 < ci; k0 += kKChunk) {
    // stage X[row0 .. +64][k0 .. +32]
    for (int i = tid; i < kRowsTile * kKChunk; i += 256) {
      const int r = i / kKChunk, k = i % kKChunk;
      const int64_t gr = row0 + r;
      float v = (gr < n && k0 + k < ci) ? __ldg(x + gr * ldx + k0 + k) : 0.f;
      if (mask && gr < n && k0 + k < ci && !(__ldg(mask + gr * ldm + k0 + k) > 0.f)) v = 0.f;
      xs[r][k] = v;
    }
    // stage M[k0 .. +32][0 .. 16*CT)
    for (int i = tid; i < kKChunk * 16 * CT; i += 256) {
      const int k = i / (16 * CT), cl = i % (16 * CT), c = cbase + cl;
      float v = 0.f;
      if (k0 + k < ci && c < co)
        v = TRANS ? __ldg(m + (int64_t)c * ci + k0 + k) : __ldg(m + (int64_t)(k0 + k) * co + c);
      ms[k][cl] = v;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < kKChunk; ++k) {
      float a[4], b[CT];
#pragma unroll
      for (int r = 0; r < 4; ++r) a[r] = xs[rg + 16 * r][k];
#pragma unroll
      for (int c = 0; c < CT; ++c) b[c] = ms[k][cg + 16 * c];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < CT; ++c) acc[r][c] = fmaf(a[r], b[c], acc[r][c]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t gr = row0 + rg + 16 * r;
    if (gr >= n) continue;
#pragma unroll
    for (int c = 0; c < CT; ++c) {
      const int col = cbase + cg + 16 * c;
      if (col >= co) continue;
      float v = acc[r][c];
      if (bias) v += __ldg(bias + col);
      if (relu) v = fmaxf(v, 0.f);
      y[gr * ldy + col] = v;
    }
  }
}

// Partial A^T B over a slab of rows: grid (slabs, k-tiles of 32, c-tiles of 32)
__global__ void __launch_bounds__(256)
    gemm_tn_partial(const float* __restrict__ a, int64_t lda, const float* __restrict__ b,
                    int64_t ldb, const float* __restrict__ mask, int64_t ldm, int64_t n, int k,
                    int c, int64_t rows_per_slab, float* __restrict__ part,
                    float* __restrict__ colpart) {
  __shared__ float as[32][33];
  __shared__ float bs[32][33];
  const int tid = threadIdx.x;
  const int ti = tid >> 3, tj = tid & 7;  // 32 x 8 threads: i = ti, j = tj + 8*q
  const int k0 = blockIdx.y * 32, c0 = blockIdx.z * 32;
  const int64_t r_begin = (int64_t)blockIdx.x * rows_per_slab;
  const int64_t r_end = min(n, r_begin + rows_per_slab);
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  float cs[4] = {0.f, 0.f, 0.f, 0.f};  // column sums of (masked) B, k-tile 0 only
  for (int64_t r0 = r_begin; r0 < r_end; r0 += 32) {
    for (int i = tid; i < 32 * 32; i += 256) {
      const int rr = i >> 5, cc = i & 31;
      const int64_t gr = r0 + rr;
      const bool rok = gr < r_end;
      as[rr][cc] = (rok && k0 + cc < k) ? __ldg(a + gr * lda + k0 + cc) : 0.f;
      float bv = (rok && c0 + cc < c) ? __ldg(b + gr * ldb + c0 + cc) : 0.f;
      if (mask && rok && c0 + cc < c && !(__ldg(mask + gr * ldm + c0 + cc) > 0.f)) bv = 0.f;
      bs[rr][cc] = bv;
    }
    __syncthreads();
#pragma unroll 8
    for (int rr = 0; rr < 32; ++rr) {
      const float av = as[rr][ti];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float bv = bs[rr][tj + 8 * q];
        acc[q] = fmaf(av, bv, acc[q]);
        if (ti == 0) cs[q] += bv;
      }
    }
    __syncthreads();
  }
  float* out = part + (int64_t)blockIdx.x * k * c;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = k0 + ti, j = c0 + tj + 8 * q;
    if (i < k && j < c) out[(int64_t)i * c + j] = acc[q];
    if (colpart && blockIdx.y == 0 && ti == 0 && j < c) colpart[(int64_t)blockIdx.x * c + j] = cs[q];
  }
}

// Fixed-order sum of the slab partials.
// 32 outputs per CTA x 32 summers: summer j adds slabs j, j+32, ... in a fixed
// order, then the 32 partial sums are combined in a fixed order (deterministic).
// (outputs from `split` on go to out2: the dW | db partials of one slab)
__global__ void __launch_bounds__(1024) sum_slabs(const float* __restrict__ part, int slabs,
                                                  int64_t len, float* __restrict__ out,
                                                  int64_t split = INT64_MAX, float* __restrict__ out2 = nullptr) {
  TCG_PDL_ENTRY();
  // 32 outputs x 32 slab groups per CTA (the partial count is ~300-600, so
  // every thread keeps ~10-20 independent loads in flight); the groups are
  // combined in a fixed order (deterministic)
  __shared__ float sh[32][33];
  const int o = threadIdx.x & 31, j = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * 32 + o;
  // up to 24 loads per thread issued as one batch (one L2 round trip for the
  // usual <= 768 slabs), folded into 8 partials in a fixed order
  constexpr int U = 24;
  float sp[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (i < len) {
    for (int q0 = j; q0 < slabs; q0 += 32 * U) {
      float v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = q0 + 32 * u;
        v[u] = q < slabs ? __ldg(part + (int64_t)q * len + i) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) sp[u & 7] += v[u];
    }
  }
  sh[j][o] = ((sp[0] + sp[1]) + (sp[2] + sp[3])) + ((sp[4] + sp[5]) + (sp[6] + sp[7]));
  __syncthreads();
  if (j == 0 && i < len) {
    float tot = 0.f;
#pragma unroll 8
    for (int q = 0; q < 32; ++q) tot += sh[q][o];
    if (i < split) out[i] = tot;
    else if (out2) out2[i - split] = tot;
  }
}

// 8 lanes per row (32 rows per CTA): log-softmax, then the NLL of the label
// (LOSS: per-CTA partials; the 8 row losses of each lpart entry are summed in
// row order, so the mean stays a fixed-order reduction) and/or
// dlogits = (softmax - onehot) / n * g (GRAD; g = *gscale or 1).
template <bool LOSS, bool GRAD>
__global__ void __launch_bounds__(256)
    softmax_xent(const float* __restrict__ logits, int64_t ld, const int64_t* __restrict__ labels,
                 int64_t n, int c, float* __restrict__ dlogits, int64_t ldd,
                 const float* __restrict__ gscale, float* __restrict__ lpart, int64_t parts) {
  TCG_PDL_ENTRY();
  __shared__ float rowc[32];
  const int sub = threadIdx.x & 7, lr_ = threadIdx.x >> 3;
  const int64_t row = (int64_t)blockIdx.x * 32 + lr_;
  const unsigned gm = 0xffu << (threadIdx.x & 24);
  float contrib = 0.f;
  if (row < n) {
    const float* lr = logits + row * ld;
    float mx = -INFINITY;
    for (int j = sub; j < c; j += 8) mx = fmaxf(mx, __ldg(lr + j));
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(gm, mx, o));
    float sm = 0.f;
    for (int j = sub; j < c; j += 8) sm += expf(__ldg(lr + j) - mx);
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) sm += __shfl_xor_sync(gm, sm, o);
    const float lse = mx + logf(sm);
    const int64_t lab = labels[row];
    // a label outside [0, c) (e.g. an ignore index) poisons the loss and the
    // row's gradient with NaN instead of reading out of bounds
    const bool ok = lab >= 0 && lab < c;
    const float bad = __int_as_float(0x7fc00000);
    if constexpr (GRAD) {
      const float inv_n = (gscale ? __ldg(gscale) : 1.f) / (float)n;
      for (int j = sub; j < c; j += 8) {
        const float pj = expf(__ldg(lr + j) - lse);
        dlogits[row * ldd + j] = ok ? (pj - (j == lab ? 1.f : 0.f)) * inv_n : bad;
      }
    }
    contrib = ok ? lse - __ldg(lr + lab) : bad;
  }
  if constexpr (!LOSS) return;
  if (sub == 0) rowc[lr_] = contrib;
  __syncthreads();
  if (threadIdx.x < 4) {
    const int64_t part = (int64_t)blockIdx.x * 4 + threadIdx.x;
    if (part < parts) {
      float acc = 0.f;
      for (int r = 0; r < 8; ++r) acc += rowc[threadIdx.x * 8 + r];
      lpart[part] = acc;
    }
  }
}

__global__ void final_loss(const float* __restrict__ lpart, int64_t parts, int64_t n,
                           float* __restrict__ loss) {
  TCG_PDL_ENTRY();
  __shared__ float sh[256];
  float s = 0.f;
  for (int64_t i = threadIdx.x; i < parts; i += 256) s += lpart[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *loss = sh[0] / (float)n;
}

template <bool TRANS>
int launch_rows(const float* x, int64_t ldx, int64_t n, int ci, const float* m, int co,
                const float* bias, int relu, const float* mask, int64_t ldm, float* y, int64_t ldy,
                cudaStream_t s) {
  // output columns in tiles of up to 128 (16 column groups x CT)
  const int ct = co > 128 ? 8 : (co + 15) / 16;
  const dim3 grid((unsigned)((n + kRowsTile - 1) / kRowsTile), (unsigned)((co + 16 * ct - 1) / (16 * ct)));
#define TCG_ROWS(CTV)                                                                    \
  case CTV:                                                                              \
    rows_x_small<CTV, TRANS><<<grid, 256, 0, s>>>(x, ldx, n, ci, m, co, bias, relu, mask, \
                                                  ldm, y, ldy);                          \
    break;
  switch (ct) {
    TCG_ROWS(1)
    TCG_ROWS(2)
    TCG_ROWS(3)
    TCG_ROWS(4)
    TCG_ROWS(5)
    TCG_ROWS(6)
    TCG_ROWS(7)
    default:
      TCG_ROWS(8)
  }
#undef TCG_ROWS
  TCG_LAUNCHED("rows_x_small");
  return TCG_OK;
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <typename K>
int set_smem(K kern, size_t bytes, int threads, int* per_sm) {
  TCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes),
           "dense attr");
  TCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, kern, threads, bytes),
           "dense occupancy");
  if (*per_sm < 1) *per_sm = 1;
  return TCG_OK;
}

template <int CI, int CO, bool TRANS, bool MASK>
int run_dense_tile(const float* x, int64_t ldx, int64_t n, int ci, const float* m, int co,
                   const float* bias, int relu, const float* mask, int64_t ldm, float* y,
                   int64_t ldy, cudaStream_t s) {
  using Cfg = dr::DenseCfg<CI, CO, MASK>;
  static int dev_done = -1, per_sm = 1;
  int dev = 0;
  TCG_CUDA(cudaGetDevice(&dev), "dense device");
  if (dev_done != dev) {
    const int rc = set_smem(dr::dense_tile<CI, CO, TRANS, MASK>, Cfg::SMEM, Cfg::NT, &per_sm);
    if (rc != TCG_OK) return rc;
    dev_done = dev;
  }
  int64_t blocks = (n + Cfg::ROWS - 1) / Cfg::ROWS;
  const int64_t cap = (int64_t)num_sms() * per_sm;
  if (blocks > cap) blocks = cap;
  const int vec_out = (ldy % 4 == 0) && al16(y);
  dr::dense_tile<CI, CO, TRANS, MASK><<<(unsigned)blocks, Cfg::NT, Cfg::SMEM, s>>>(
      x, ldx, n, m, co, bias, relu, mask, ldm, y, ldy, vec_out, ci);
  TCG_LAUNCHED("dense_tile");
  return TCG_OK;
}

template <int CI, bool TRANS>
int dense_co(const float* x, int64_t ldx, int64_t n, int ci, const float* m, int co,
             const float* bias, int relu, const float* mask, int64_t ldm, float* y, int64_t ldy,
             cudaStream_t s) {
#define TCG_DC(COV)                                                                            \
  if (co <= COV)                                                                               \
    return mask ? run_dense_tile<CI, COV, TRANS, true>(x, ldx, n, ci, m, co, bias, relu, mask, \
                                                       ldm, y, ldy, s)                         \
                : run_dense_tile<CI, COV, TRANS, false>(x, ldx, n, ci, m, co, bias, relu,      \
                                                        mask, ldm, y, ldy, s);
  TCG_DC(8)
  TCG_DC(16)
  TCG_DC(32)
  TCG_DC(40)
  TCG_DC(64)
#undef TCG_DC
  return 1;
}

// Pipelined row-tile path for the models' shapes; returns 1 when not applicable.
int fast_dense(const float* x, int64_t ldx, int64_t n, int ci, const float* m, int co, bool trans,
               const float* bias, int relu, const float* mask, int64_t ldm, float* y, int64_t ldy,
               cudaStream_t s) {
  if (co > 64 || ldx % 4 || !al16(x) || (mask && (ldm % 4 || !al16(mask)))) return 1;
  // widths that are not a multiple of 4 run the next tile width up (zero-filled
  // tail columns); the padded row stride keeps the 16-B staging in bounds
  const int ci4 = (ci + 3) / 4 * 4;
  if (ci4 > ldx || (mask && ci4 > ldm)) return 1;
#define TCG_FD(CIV)                                                                            \
  if (ci4 == CIV)                                                                              \
    return trans ? dense_co<CIV, true>(x, ldx, n, ci, m, co, bias, relu, mask, ldm, y, ldy, s) \
                 : dense_co<CIV, false>(x, ldx, n, ci, m, co, bias, relu, mask, ldm, y, ldy, s);
  TCG_FD(16)
  TCG_FD(24)
  TCG_FD(32)
  TCG_FD(40)
  TCG_FD(48)
  TCG_FD(64)
  TCG_FD(96)
  TCG_FD(100)
  TCG_FD(128)
#undef TCG_FD
  return 1;
}

template <int CI, int CO, bool MASK>
int run_gemm_tn_tile(const float* a, int64_t lda, const float* b, int64_t ldb, const float* mask,
                     int64_t ldm, int64_t n, int co, float* part, float* colpart, int64_t cap_slabs,
                     int64_t* used, cudaStream_t s) {
  using Cfg = dr::GemmCfg<CI, CO, MASK>;
  static int dev_done = -1, per_sm = 1;
  int dev = 0;
  TCG_CUDA(cudaGetDevice(&dev), "dense device");
  if (dev_done != dev) {
    const int rc = set_smem(dr::gemm_tn_tile<CI, CO, MASK>, Cfg::SMEM, Cfg::NT, &per_sm);
    if (rc != TCG_OK) return rc;
    dev_done = dev;
  }
  int64_t blocks = (n + Cfg::ROWS - 1) / Cfg::ROWS;
  int64_t cap = (int64_t)num_sms() * per_sm;
  if (cap > cap_slabs) cap = cap_slabs;
  if (blocks > cap) blocks = cap;
  dr::gemm_tn_tile<CI, CO, MASK><<<(unsigned)blocks, Cfg::NT, Cfg::SMEM, s>>>(
      a, lda, b, ldb, mask, ldm, n, co, part, colpart);
  TCG_LAUNCHED("gemm_tn_tile");
  *used = blocks;
  return TCG_OK;
}

template <int CI>
int gemm_tn_co(const float* a, int64_t lda, const float* b, int64_t ldb, const float* mask,
               int64_t ldm, int64_t n, int co, float* part, float* colpart, int64_t cap_slabs,
               int64_t* used, cudaStream_t s) {
#define TCG_GC(COV)                                                                            \
  if (co <= COV)                                                                               \
    return mask ? run_gemm_tn_tile<CI, COV, true>(a, lda, b, ldb, mask, ldm, n, co, part,      \
                                                  colpart, cap_slabs, used, s)                 \
                : run_gemm_tn_tile<CI, COV, false>(a, lda, b, ldb, mask, ldm, n, co, part,     \
                                                   colpart, cap_slabs, used, s);
  TCG_GC(8)
  TCG_GC(16)
  TCG_GC(32)
  TCG_GC(40)
  TCG_GC(64)
#undef TCG_GC
  return 1;
}

int fast_gemm_tn(const float* a, int64_t lda, const float* b, int64_t ldb, const float* mask,
                 int64_t ldm, int64_t n, int k, int c, float* part, float* colpart,
                 int64_t cap_slabs, int64_t* used, cudaStream_t s) {
  if (c > 64 || lda % 4 || ldb % 4 || !al16(a) || !al16(b) || (mask && (ldm % 4 || !al16(mask))))
    return 1;
  if (k == 16) return gemm_tn_co<16>(a, lda, b, ldb, mask, ldm, n, c, part, colpart, cap_slabs, used, s);
  if (k == 32) return gemm_tn_co<32>(a, lda, b, ldb, mask, ldm, n, c, part, colpart, cap_slabs, used, s);
  if (k == 40) return gemm_tn_co<40>(a, lda, b, ldb, mask, ldm, n, c, part, colpart, cap_slabs, used, s);
  if (k == 64) return gemm_tn_co<64>(a, lda, b, ldb, mask, ldm, n, c, part, colpart, cap_slabs, used, s);
  if (k == 96) return gemm_tn_co<96>(a, lda, b, ldb, mask, ldm, n, c, part, colpart, cap_slabs, used, s);
  if (k == 100) return gemm_tn_co<100>(a, lda, b, ldb, mask, ldm, n, c, part, colpart, cap_slabs, used, s);
  if (k == 128) return gemm_tn_co<128>(a, lda, b, ldb, mask, ldm, n, c, part, colpart, cap_slabs, used, s);
  return 1;
}

// Column sums of x[n x c] (row stride ld), first level: CTA `slab` sums rows
// [slab*rows, (slab+1)*rows). Thread (lane r, column unit j) adds rows r,
// r+RL, ... of its V columns (V = 4: float4 loads when c, ld are multiples of
// 4) with 8 independent partials in flight; the RL lane partials are then added
// in lane order, so the result is deterministic.
template <int V, bool GATE = false>
__global__ void __launch_bounds__(256)
    colsum_part(const float* __restrict__ x, int64_t ld, int64_t n, int c, int64_t rows,
                float* __restrict__ part, const float* __restrict__ gate = nullptr, int64_t ldg = 0,
                float* __restrict__ gout = nullptr, int64_t ldo = 0) {
  TCG_PDL_ENTRY();
  using VT = typename std::conditional<V == 4, float4, float>::type;
  __shared__ VT sh[256];
  const int units = c / V;
  const int64_t r0 = (int64_t)blockIdx.x * rows, r1 = min(n, r0 + rows);
  auto add = [](VT& a, const VT& b) {
    if constexpr (V == 4) a.x += b.x, a.y += b.y, a.z += b.z, a.w += b.w;
    else a += b;
  };
  // GATE: the value is x .* [gate > 0] (the ReLU backward), also written to gout
  auto gated = [](VT v, VT m) {
    if constexpr (V == 4) {
      v.x = m.x > 0.f ? v.x : 0.f, v.y = m.y > 0.f ? v.y : 0.f;
      v.z = m.z > 0.f ? v.z : 0.f, v.w = m.w > 0.f ? v.w : 0.f;
      return v;
    } else {
      return m > 0.f ? v : 0.f;
    }
  };
  for (int ub = 0; ub < units; ub += 256) {
    const int uw = min(256, units - ub);
    const int rl = 256 / uw;
    const int lane_r = threadIdx.x / uw, j = threadIdx.x % uw;
    VT sp[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) sp[u] = VT{};
    if (lane_r < rl) {
      const VT* col = reinterpret_cast<const VT*>(x) + ub + j;
      const VT* gcol = GATE ? reinterpret_cast<const VT*>(gate) + ub + j : nullptr;
      VT* ocol = GATE ? reinterpret_cast<VT*>(gout) + ub + j : nullptr;
      const int64_t ldv = ld / V, ldgv = ldg / V, ldov = ldo / V;
      auto val = [&](int64_t r) {
        VT v = __ldg(col + r * ldv);
        if constexpr (GATE) {
          v = gated(v, __ldg(gcol + r * ldgv));
          ocol[r * ldov] = v;
        }
        return v;
      };
      int64_t r = r0 + lane_r;
      for (; r + 7 * rl < r1; r += 8 * rl) {
        VT v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = val(r + u * rl);
#pragma unroll
        for (int u = 0; u < 8; ++u) add(sp[u], v[u]);
      }
      for (; r < r1; r += rl) add(sp[0], val(r));
    }
    add(sp[0], sp[1]), add(sp[2], sp[3]), add(sp[4], sp[5]), add(sp[6], sp[7]);
    add(sp[0], sp[2]), add(sp[4], sp[6]), add(sp[0], sp[4]);
    sh[threadIdx.x] = sp[0];
    __syncthreads();
    if (threadIdx.x < uw) {
      VT tot = VT{};
      for (int q = 0; q < rl; ++q) add(tot, sh[q * uw + threadIdx.x]);
      reinterpret_cast<VT*>(part + (int64_t)blockIdx.x * c)[ub + threadIdx.x] = tot;
    }
    __syncthreads();
  }
}

int64_t colsum_slabs(int64_t n) {
  // 256 rows per slab: ~4 CTAs of 256 threads per SM and one round of loads each
  // (1024-row slabs at <= 2 per SM ran arxiv 169343 x 16 at 1 TB/s)
  const int64_t s = (n + 255) / 256;
  const int64_t cap = 8LL * num_sms();
  return s < 1 ? 1 : (s > cap ? cap : s);
}

int64_t slabs_for(int64_t n) {
  int64_t s = (n + 63) / 64;  // >= 64 rows per slab; ~4 CTAs per SM per output tile
  const int64_t cap = 4LL * num_sms();
  return s < 1 ? 1 : (s > cap ? cap : s);
}

}  // namespace
}  // namespace tcg

using namespace tcg;

namespace tcg {
int dense_mma32(const float* x, int64_t ldx, int64_t n, int ci, const float* w, int co, bool trans,
                const float* bias, int relu, const float* mask, float* y, int64_t ldy, cudaStream_t s);
int dense_mma32_bwd(const float* x, int64_t ldx, const float* g, int64_t ldg, int64_t n, const float* w,
                    float* dx, int64_t lddx, float* part, int64_t* slabs, cudaStream_t s);
int linear_xent(const float* x, int64_t ldx, int64_t n, int kin, const float* w, int c, const float* bias,
                const int64_t* labels, float inv_div, float* dl, int64_t ldd, float* lpart, int64_t cap_parts,
                int64_t* nparts, cudaStream_t s);
int64_t linear_xent_parts(int64_t n);
int dense_in_mma(const float* x, int64_t ldx, int64_t n, int ci, const float* w, int co, bool trans,
                 const float* bias, int relu, const float* mask, float* y, int64_t ldy, cudaStream_t s);
int dense_wide_mma(const float* x, int64_t ldx, int64_t n, int ci, const float* w, int co, bool trans,
                   const float* bias, int relu, const float* mask, float* y, int64_t ldy, cudaStream_t s);
int gemm_tn_mma(const float* a, int64_t lda, const float* b, int64_t ldb, const float* mask, int64_t ldm,
                int64_t n, int k, int c, float* part, float* colpart, int64_t cap_slabs, int64_t* used,
                cudaStream_t s);
int64_t linear_xent_bwd_slabs(int64_t n);
int linear_xent_bwd(const float* x, int64_t ldx, int64_t n, int kin, const float* w, int c, const float* bias,
                    const int64_t* labels, const float* gscale, float inv_div, float* dx, int64_t lddx, float* part,
                    int64_t* slabs, cudaStream_t s);
int dense_tcgen05(const float* x, int64_t ldx, int64_t n, int ci, const float* m, int co, bool trans,
                  const float* bias, int relu, const float* mask, float* y, int64_t ldy, cudaStream_t s);
}

extern "C" int tcg_dense(const float* x, int64_t ldx, int64_t n, int64_t ci, const float* m,
                         int64_t co, int32_t m_transposed, const float* bias, int32_t relu,
                         const float* mask, int64_t ldm, float* y, int64_t ldy, void* stream) {
  TCG_REQUIRE(n >= 0 && ci >= 1 && co >= 1, "tcg_dense: bad shape");
  TCG_REQUIRE(ldx >= ci && ldy >= co && (mask == nullptr || ldm >= ci), "tcg_dense: bad ld");
  TCG_REQUIRE((relu & ~(1 | TCG_DENSE_OUT_TF32)) == 0, "tcg_dense: unknown relu flags 0x%x", relu);
  if (n == 0) return TCG_OK;
  TCG_REQUIRE(x && m && y, "tcg_dense: null pointer");
  cudaStream_t s = as_stream(stream);
  {
    // 32 x 32: mma.sync 3xTF32, ldmatrix-fed (csrc/dense_mma.cu); the only kernel
    // that rounds its output in the epilogue (TCG_DENSE_OUT_TF32)
    const int rc = dense_mma32(x, ldx, n, (int)ci, m, (int)co, m_transposed != 0, bias, relu, mask, y, ldy, s);
    if (rc != 1) return rc;
  }
  if (relu & TCG_DENSE_OUT_TF32) {  // other shapes: the plain product, then one rounding pass
    int rc = tcg_dense(x, ldx, n, ci, m, co, m_transposed, bias, relu & 1, mask, ldm, y, ldy, stream);
    if (rc != TCG_OK) return rc;
    TCG_REQUIRE(ldy == co, "tcg_dense: TCG_DENSE_OUT_TF32 needs dense output rows (ldy == co) off the 32 x 32 path");
    return tcg_quantize_tf32(y, y, n * co, stream);
  }
  {
    // the wide input layers (33..128 -> 16 / 32) on mma.sync 3xTF32 (csrc/dense_mma.cu
    // dense_in_mma): arxiv 128 -> 32 38.9 us cold (tcgen05 dense_tc 43.0, FFMA2 53.2),
    // 128 -> 16 30.7 (36.9), 96 -> 16 46.1 (55.3), products 100 -> 16 242 (328).
    // TCG_DENSE_TC=1 puts the tcgen05 kernel (csrc/dense_tc.cu) first for 96..128 -> 32.
    static const bool tc_first = std::getenv("TCG_DENSE_TC") && std::atoi(std::getenv("TCG_DENSE_TC")) == 1;
    if (tc_first) {
      const int rc = dense_tcgen05(x, ldx, n, (int)ci, m, (int)co, m_transposed != 0, bias, relu, mask, y,
                                   ldy, s);
      if (rc != 1) return rc;
    }
    const int rc = dense_in_mma(x, ldx, n, (int)ci, m, (int)co, m_transposed != 0, bias, relu, mask, y, ldy, s);
    if (rc != 1) return rc;
  }
  {
    // inputs wider than 128 features (Cora 1433, Pubmed 500) in 128-feature K panels
    const int rc = dense_wide_mma(x, ldx, n, (int)ci, m, (int)co, m_transposed != 0, bias, relu, mask, y, ldy, s);
    if (rc != 1) return rc;
  }
  {
    const int rc = fast_dense(x, ldx, n, (int)ci, m, (int)co, m_transposed != 0, bias, relu, mask,
                              ldm, y, ldy, s);
    if (rc != 1) return rc;  // 1: shape not covered by the warp-tile kernels
  }
  return m_transposed ? launch_rows<true>(x, ldx, n, (int)ci, m, (int)co, bias, relu, mask, ldm, y,
                                          ldy, s)
                      : launch_rows<false>(x, ldx, n, (int)ci, m, (int)co, bias, relu, mask, ldm,
                                           y, ldy, s);
}

extern "C" size_t tcg_gemm_tn_workspace_bytes(int64_t n, int64_t k, int64_t c) {
  const int64_t slabs = slabs_for(n);
  return (size_t)(slabs * k * c + slabs * c) * sizeof(float);
}

extern "C" int tcg_gemm_tn(const float* a, int64_t lda, const float* b, int64_t ldb,
                           const float* mask, int64_t ldm, int64_t n, int64_t k, int64_t c,
                           float* out, float* colsum, void* workspace, size_t workspace_bytes,
                           void* stream) {
  TCG_REQUIRE(n >= 0 && k >= 1 && c >= 1, "tcg_gemm_tn: bad shape");
  TCG_REQUIRE(lda >= k && ldb >= c && (mask == nullptr || ldm >= c), "tcg_gemm_tn: bad ld");
  TCG_REQUIRE(workspace_bytes >= tcg_gemm_tn_workspace_bytes(n, k, c),
              "tcg_gemm_tn: workspace too small");
  TCG_REQUIRE(out && workspace, "tcg_gemm_tn: null pointer");
  cudaStream_t s = as_stream(stream);
  const int64_t slabs = slabs_for(n);
  const int64_t rows = (n + slabs - 1) / slabs;
  float* part = static_cast<float*>(workspace);
  float* colpart = part + slabs * k * c;
  if (n == 0) {
    TCG_CUDA(cudaMemsetAsync(out, 0, sizeof(float) * k * c, s), "tcg_gemm_tn memset");
    if (colsum) TCG_CUDA(cudaMemsetAsync(colsum, 0, sizeof(float) * c, s), "tcg_gemm_tn memset");
    return TCG_OK;
  }
  {
    int64_t used = 0;
    // the wide input layers (k 33..128 -> 16 / 32) on the tensor cores (3xTF32),
    // then the FFMA2 tile kernels
    int rc = gemm_tn_mma(a, lda, b, ldb, mask, ldm, n, (int)k, (int)c, part, colsum ? colpart : nullptr,
                         slabs, &used, s);
    if (rc == 1)
      rc = fast_gemm_tn(a, lda, b, ldb, mask, ldm, n, (int)k, (int)c, part, colsum ? colpart : nullptr,
                        slabs, &used, s);
    if (rc == TCG_OK) {
      ::tcg::launch_pdl(sum_slabs, (unsigned)((k * c + 31) / 32), 1024, 0, s, part, (int)used, k * c, out, (int64_t)INT64_MAX, (float*)nullptr);
      TCG_LAUNCHED("sum_slabs");
      if (colsum) {
        ::tcg::launch_pdl(sum_slabs, (unsigned)((c + 31) / 32), 1024, 0, s, colpart, (int)used, c, colsum, (int64_t)INT64_MAX, (float*)nullptr);
        TCG_LAUNCHED("sum_slabs");
      }
      return TCG_OK;
    }
    if (rc != 1) return rc;
  }
  dim3 grid((unsigned)slabs, (unsigned)((k + 31) / 32), (unsigned)((c + 31) / 32));
  gemm_tn_partial<<<grid, 256, 0, s>>>(a, lda, b, ldb, mask, ldm, n, (int)k, (int)c, rows, part,
                                       colsum ? colpart : nullptr);
  TCG_LAUNCHED("gemm_tn_partial");
  ::tcg::launch_pdl(sum_slabs, (unsigned)((k * c + 31) / 32), 1024, 0, s, part, (int)slabs, k * c, out, (int64_t)INT64_MAX, (float*)nullptr);
  TCG_LAUNCHED("sum_slabs");
  if (colsum) {
    ::tcg::launch_pdl(sum_slabs, (unsigned)((c + 31) / 32), 1024, 0, s, colpart, (int)slabs, c, colsum, (int64_t)INT64_MAX, (float*)nullptr);
    TCG_LAUNCHED("sum_slabs");
  }
  return TCG_OK;
}

extern "C" size_t tcg_softmax_xent_workspace_bytes(int64_t n) {
  return (size_t)((n + 7) / 8 + 1) * sizeof(float);
}

extern "C" int tcg_softmax_xent(const float* logits, int64_t ld, const int64_t* labels, int64_t n,
                                int64_t c, float* loss, float* dlogits, void* workspace,
                                size_t workspace_bytes, void* stream) {
  TCG_REQUIRE(n >= 1 && c >= 1 && ld >= c, "tcg_softmax_xent: bad shape");
  TCG_REQUIRE(workspace_bytes >= tcg_softmax_xent_workspace_bytes(n),
              "tcg_softmax_xent: workspace too small");
  TCG_REQUIRE(logits && labels && loss, "tcg_softmax_xent: null pointer");
  cudaStream_t s = as_stream(stream);
  const int64_t parts = (n + 7) / 8;
  float* lpart = static_cast<float*>(workspace);
  const unsigned grid = (unsigned)((n + 31) / 32);
  if (dlogits)
    ::tcg::launch_pdl(softmax_xent<true, true>, grid, 256, 0, s, logits, ld, labels, n, (int)c, dlogits, c,
                                                  nullptr, lpart, parts);
  else
    ::tcg::launch_pdl(softmax_xent<true, false>, grid, 256, 0, s, logits, ld, labels, n, (int)c, nullptr, 0,
                                                   nullptr, lpart, parts);
  TCG_LAUNCHED("softmax_xent");
  ::tcg::launch_pdl(final_loss, 1, 256, 0, s, lpart, parts, n, loss);
  TCG_LAUNCHED("final_loss");
  return TCG_OK;
}

extern "C" int tcg_softmax_xent_backward(const float* logits, int64_t ld, const int64_t* labels,
                                         int64_t n, int64_t c, const float* grad_scale,
                                         float* dlogits, int64_t ldd, void* stream) {
  TCG_REQUIRE(n >= 1 && c >= 1 && ld >= c && ldd >= c, "tcg_softmax_xent_backward: bad shape");
  TCG_REQUIRE(logits && labels && dlogits, "tcg_softmax_xent_backward: null pointer");
  ::tcg::launch_pdl(softmax_xent<false, true>, (unsigned)((n + 31) / 32), 256, 0, as_stream(stream), 
      logits, ld, labels, n, (int)c, dlogits, ldd, grad_scale, nullptr, 0);
  TCG_LAUNCHED("softmax_xent_backward");
  return TCG_OK;
}

extern "C" size_t tcg_linear_xent_workspace_bytes(int64_t n) {
  return (size_t)(linear_xent_parts(n > 0 ? n : 1) + 1) * sizeof(float);
}

extern "C" int tcg_linear_xent(const float* x, int64_t ldx, int64_t n, int64_t kin, const float* w,
                               int64_t c, const float* bias, const int64_t* labels, int64_t div,
                               float* loss, float* dlogits, int64_t ldd, void* workspace,
                               size_t workspace_bytes, void* stream) {
  TCG_REQUIRE(n >= 1 && kin >= 1 && c >= 1 && ldx >= kin && (!dlogits || ldd >= c) && div >= 1,
              "tcg_linear_xent: bad shape");
  TCG_REQUIRE(x && w && labels && loss && workspace, "tcg_linear_xent: null pointer");
  TCG_REQUIRE(workspace_bytes >= tcg_linear_xent_workspace_bytes(n), "tcg_linear_xent: workspace too small");
  cudaStream_t s = as_stream(stream);
  float* lpart = static_cast<float*>(workspace);
  int64_t parts = 0;
  const int rc = linear_xent(x, ldx, n, (int)kin, w, (int)c, bias, labels, 1.f / (float)div, dlogits, ldd,
                             lpart, (int64_t)(workspace_bytes / sizeof(float)), &parts, s);
  if (rc < 0) return rc;
  if (rc > 0) {
    set_error("tcg_linear_xent: shape not covered (needs kin a multiple of 4 <= 32, c <= 48, 16-B rows)");
    return TCG_E_UNSUPPORTED;
  }
  ::tcg::launch_pdl(final_loss, 1, 256, 0, s, lpart, parts, div, loss);
  TCG_LAUNCHED("final_loss");
  return TCG_OK;
}

extern "C" size_t tcg_linear_xent_backward_workspace_bytes(int64_t n, int64_t kin, int64_t c) {
  return (size_t)(linear_xent_bwd_slabs(n > 0 ? n : 1) * (kin * c + c)) * sizeof(float);
}

extern "C" int tcg_linear_xent_backward(const float* x, int64_t ldx, int64_t n, int64_t kin, const float* w,
                                        int64_t c, const float* bias, const int64_t* labels, int64_t div,
                                        const float* grad_scale, float* dx, int64_t lddx, float* dw, float* db,
                                        void* workspace, size_t workspace_bytes, void* stream) {
  TCG_REQUIRE(n >= 1 && kin >= 1 && c >= 1 && ldx >= kin && div >= 1 && (!dx || lddx >= kin),
              "tcg_linear_xent_backward: bad shape");
  TCG_REQUIRE(x && w && labels && dw && workspace, "tcg_linear_xent_backward: null pointer");
  TCG_REQUIRE(workspace_bytes >= tcg_linear_xent_backward_workspace_bytes(n, kin, c),
              "tcg_linear_xent_backward: workspace too small");
  cudaStream_t s = as_stream(stream);
  float* part = static_cast<float*>(workspace);
  int64_t slabs = 0;
  const int rc = linear_xent_bwd(x, ldx, n, (int)kin, w, (int)c, bias, labels, grad_scale, 1.f / (float)div, dx,
                                 lddx, part, &slabs, s);
  if (rc < 0) return rc;
  if (rc > 0) {
    set_error("tcg_linear_xent_backward: shape not covered (needs kin a multiple of 4 <= 32, c <= 48, 16-B rows)");
    return TCG_E_UNSUPPORTED;
  }
  const int64_t len = kin * c + c;
  ::tcg::launch_pdl(sum_slabs, (unsigned)((len + 31) / 32), 1024, 0, s, part, (int)slabs, len, dw, kin * c, db);
  TCG_LAUNCHED("sum_slabs");
  return TCG_OK;
}

extern "C" size_t tcg_colsum_workspace_bytes(int64_t n, int64_t c) {
  const int64_t c4 = c > 0 ? (c + 3) / 4 * 4 : 4;
  return (size_t)((colsum_slabs(n) + 1) * c4) * sizeof(float);
}

extern "C" int tcg_colsum(const float* x, int64_t ld, int64_t n, int64_t c, float* out,
                          void* workspace, size_t workspace_bytes, void* stream) {
  TCG_REQUIRE(n >= 0 && c >= 1 && ld >= c, "tcg_colsum: bad shape");
  TCG_REQUIRE(workspace_bytes >= tcg_colsum_workspace_bytes(n, c), "tcg_colsum: workspace too small");
  TCG_REQUIRE(out && workspace && (n == 0 || x), "tcg_colsum: null pointer");
  cudaStream_t s = as_stream(stream);
  if (n == 0) {
    TCG_CUDA(cudaMemsetAsync(out, 0, sizeof(float) * c, s), "tcg_colsum memset");
    return TCG_OK;
  }
  const int64_t slabs = colsum_slabs(n);
  const int64_t rows = (n + slabs - 1) / slabs;
  float* part = static_cast<float*>(workspace);
  // rows padded to a multiple of 4 floats take the float4 path over the padded
  // width; the padding columns land in partials that are never read
  const int64_t c4 = (c + 3) / 4 * 4;
  const bool v4 = ld % 4 == 0 && c4 <= ld && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  if (v4) {
    ::tcg::launch_pdl(colsum_part<4>, (unsigned)slabs, 256, 0, s, x, ld, n, (int)c4, rows, part, (const float*)nullptr, (int64_t)0, (float*)nullptr, (int64_t)0);
    TCG_LAUNCHED("colsum_part");
    if (c4 == c) {
      ::tcg::launch_pdl(sum_slabs, (unsigned)((c + 31) / 32), 1024, 0, s, part, (int)slabs, c, out, (int64_t)INT64_MAX, (float*)nullptr);
    } else {
      float* tmp = part + slabs * c4;
      ::tcg::launch_pdl(sum_slabs, (unsigned)((c4 + 31) / 32), 1024, 0, s, part, (int)slabs, c4, tmp, (int64_t)INT64_MAX, (float*)nullptr);
      TCG_CUDA(cudaMemcpyAsync(out, tmp, sizeof(float) * c, cudaMemcpyDeviceToDevice, s),
               "tcg_colsum copy");
    }
  } else {
    ::tcg::launch_pdl(colsum_part<1>, (unsigned)slabs, 256, 0, s, x, ld, n, (int)c, rows, part, (const float*)nullptr, (int64_t)0, (float*)nullptr, (int64_t)0);
    TCG_LAUNCHED("colsum_part");
    ::tcg::launch_pdl(sum_slabs, (unsigned)((c + 31) / 32), 1024, 0, s, part, (int)slabs, c, out, (int64_t)INT64_MAX, (float*)nullptr);
  }
  TCG_LAUNCHED("sum_slabs");
  return TCG_OK;
}

extern "C" int tcg_colsum_gate(const float* x, int64_t ld, const float* gate, int64_t ldg, int64_t n,
                               int64_t c, float* gout, int64_t ldo, float* out, void* workspace,
                               size_t workspace_bytes, void* stream) {
  TCG_REQUIRE(n >= 0 && c >= 1 && ld >= c && ldg >= c && ldo >= c, "tcg_colsum_gate: bad shape");
  TCG_REQUIRE(workspace_bytes >= tcg_colsum_workspace_bytes(n, c), "tcg_colsum_gate: workspace too small");
  TCG_REQUIRE(out && workspace && (n == 0 || (x && gate && gout)), "tcg_colsum_gate: null pointer");
  cudaStream_t s = as_stream(stream);
  if (n == 0) {
    TCG_CUDA(cudaMemsetAsync(out, 0, sizeof(float) * c, s), "tcg_colsum_gate memset");
    return TCG_OK;
  }
  const int64_t slabs = colsum_slabs(n);
  const int64_t rows = (n + slabs - 1) / slabs;
  float* part = static_cast<float*>(workspace);
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const bool v4 = c % 4 == 0 && ld % 4 == 0 && ldg % 4 == 0 && ldo % 4 == 0 && al(x) && al(gate) && al(gout);
  if (v4)
    ::tcg::launch_pdl(colsum_part<4, true>, (unsigned)slabs, 256, 0, s, x, ld, n, (int)c, rows, part, gate, ldg, gout, ldo);
  else
    ::tcg::launch_pdl(colsum_part<1, true>, (unsigned)slabs, 256, 0, s, x, ld, n, (int)c, rows, part, gate, ldg, gout, ldo);
  TCG_LAUNCHED("colsum_gate");
  ::tcg::launch_pdl(sum_slabs, (unsigned)((c + 31) / 32), 1024, 0, s, part, (int)slabs, c, out, (int64_t)INT64_MAX, (float*)nullptr);
  TCG_LAUNCHED("sum_slabs");
  return TCG_OK;
}

extern "C" size_t tcg_dense_backward_workspace_bytes(int64_t n, int64_t ci, int64_t co) {
  const size_t fused = (size_t)4 * num_sms() * ci * co * sizeof(float);
  const size_t split = tcg_gemm_tn_workspace_bytes(n, ci, co);
  return fused > split ? fused : split;
}

extern "C" int tcg_dense_backward(const float* x, int64_t ldx, const float* g, int64_t ldg,
                                  int64_t n, int64_t ci, int64_t co, const float* w, float* dx,
                                  int64_t lddx, float* dw, void* workspace,
                                  size_t workspace_bytes, void* stream) {
  TCG_REQUIRE(n >= 0 && ci >= 1 && co >= 1 && ldx >= ci && ldg >= co && lddx >= ci,
              "tcg_dense_backward: bad shape");
  TCG_REQUIRE(workspace_bytes >= tcg_dense_backward_workspace_bytes(n, ci, co),
              "tcg_dense_backward: workspace too small");
  TCG_REQUIRE(w && dw && workspace && (n == 0 || (x && g && dx)),
              "tcg_dense_backward: null pointer");
  cudaStream_t s = as_stream(stream);
  if (n == 0) {
    TCG_CUDA(cudaMemsetAsync(dw, 0, sizeof(float) * ci * co, s), "tcg_dense_backward memset");
    return TCG_OK;
  }
  const bool fused = ci == 32 && co == 32 && n > 0 && ldx % 4 == 0 && ldg % 4 == 0 &&
                     lddx % 4 == 0 && al16(x) && al16(g) && al16(dx);
  if (!fused) {
    const int rc = tcg_dense(g, ldg, n, co, w, ci, 1, nullptr, 0, nullptr, 0, dx, lddx, stream);
    if (rc != TCG_OK) return rc;
    return tcg_gemm_tn(x, ldx, g, ldg, nullptr, 0, n, ci, co, dw, nullptr, workspace,
                       workspace_bytes, stream);
  }
  {
    int64_t slabs = 0;
    float* part = static_cast<float*>(workspace);
    const int rc = dense_mma32_bwd(x, ldx, g, ldg, n, w, dx, lddx, part, &slabs, s);
    if (rc == TCG_OK) {
      ::tcg::launch_pdl(sum_slabs, (unsigned)((ci * co + 31) / 32), 1024, 0, s, part, (int)slabs, ci * co, dw, (int64_t)INT64_MAX, (float*)nullptr);
      TCG_LAUNCHED("sum_slabs");
      return TCG_OK;
    }
    if (rc != 1) return rc;
  }
  using Cfg = dr::BwdCfg<32, 32>;
  static int dev_done = -1, per_sm = 1;
  int dev = 0;
  TCG_CUDA(cudaGetDevice(&dev), "dense device");
  if (dev_done != dev) {
    const int rc = set_smem(dr::dense_bwd_tile<32, 32>, Cfg::SMEM, Cfg::NT, &per_sm);
    if (rc != TCG_OK) return rc;
    dev_done = dev;
  }
  int64_t blocks = (n + Cfg::ROWS - 1) / Cfg::ROWS;
  int64_t cap = (int64_t)num_sms() * (per_sm < 4 ? per_sm : 4);
  if (blocks > cap) blocks = cap;
  float* part = static_cast<float*>(workspace);
  dr::dense_bwd_tile<32, 32><<<(unsigned)blocks, Cfg::NT, Cfg::SMEM, s>>>(x, ldx, g, ldg, n, w,
                                                                          dx, lddx, part);
  TCG_LAUNCHED("dense_bwd_tile");
  ::tcg::launch_pdl(sum_slabs, (unsigned)((ci * co + 31) / 32), 1024, 0, s, part, (int)blocks, ci * co, dw, (int64_t)INT64_MAX, (float*)nullptr);
  TCG_LAUNCHED("sum_slabs");
  return TCG_OK;
}
