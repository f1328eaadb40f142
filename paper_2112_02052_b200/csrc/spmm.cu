// Neighbour aggregation Y = (F .* A) X over the SGT tiling — replaces the
// reference kernels.spmm (/root/reference/pkg/src/tcgraph/kernels.py:213-374,
// Alg. 2 of the paper).
//
// Two engines behind tcg_spmm:
//  * spmm_exact (TCG_PREC_F32): CUDA cores, one lane group per row, features
//    across lanes, edges folded in CSR order with one rounding per product
//    and per add (__fmul_rn/__fadd_rn). Bitwise equal to the reference f32
//    path, which is itself bitwise equal to oracle.ref_spmm
//    (test_acceptance.py:76-98).
//  * spmm_tc (TCG_PREC_TF32): tensor cores, one warp per (16-row window,
//    feature chunk). The window's condensed 16x8 A-tiles are scattered from
//    the edge list into shared memory directly in mma fragment order
//    (InitSparse, tiles.py:130-152); the 8 neighbour rows of each tile are
//    gathered straight into B fragments with vector loads (FetchDense,
//    tiles.py:155-181) using a feature permutation that makes every lane's
//    slice contiguous; mma.sync.m16n8k8 TF32 (RNE-rounded operands, fp32
//    accumulate) does the tile product; the epilogue (bias, accumulate)
//    stores contiguous 2*NT-float runs per lane (StoreDense, tiles.py:204-220)
//    into the caller's row slice (all-gather buffer in the sharded path).
#include "common.cuh"

namespace tcg {
namespace {

// ------------------------------------------------------------------------- //
// exact f32 engine
// ------------------------------------------------------------------------- //

struct SpmmArgs {
  const int64_t* ptr;
  const uint32_t* cols;
  const uint32_t* e2c;
  const int64_t* col_offsets;
  const uint32_t* c2n;
  const uint32_t* wp;
  int64_t n;
  const float* x;
  int64_t ldx;
  const float* w;
  const uint32_t* widx;
  const float* x2;
  int64_t ldx2;
  const float* w2;
  const uint32_t* widx2;
  const float* bias;
  float* y;
  int64_t ldy;
  int64_t y_row0;
  int64_t row_begin, row_end;
  int64_t win_begin;
  int64_t nwin;
  int dim;
  int accumulate;
};

__device__ __forceinline__ float edge_weight(const float* w, const uint32_t* widx, int64_t e) {
  if (w == nullptr) return 1.0f;
  return widx ? __ldg(w + __ldg(widx + e)) : __ldg(w + e);
}

// G lanes per row, each lane 4 consecutive features (float4 when VEC).
template <int G, bool VEC>
__global__ void __launch_bounds__(256) spmm_exact(SpmmArgs a) {
  const int lane = threadIdx.x & 31;
  const int sub = lane % G;
  const int64_t group = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t r = a.row_begin + group;
  if (r >= a.row_end) return;
  const int64_t e0 = __ldg(a.ptr + r), e1 = __ldg(a.ptr + r + 1);
  const bool wtd = a.w != nullptr, dual = a.x2 != nullptr, wtd2 = a.w2 != nullptr;
  for (int f0 = sub * 4; f0 < a.dim; f0 += G * 4) {
    const int nf = min(4, a.dim - f0);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int64_t e = e0; e < e1; ++e) {
      const uint32_t c = __ldg(a.cols + e);
      float v[4];
      const float* xr = a.x + (int64_t)c * a.ldx + f0;
      if (VEC && nf == 4) {
        float4 q = __ldg(reinterpret_cast<const float4*>(xr));
        v[0] = q.x, v[1] = q.y, v[2] = q.z, v[3] = q.w;
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = i < nf ? __ldg(xr + i) : 0.f;
      }
      if (wtd) {
        const float we = edge_weight(a.w, a.widx, e);
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i] = __fadd_rn(acc[i], __fmul_rn(we, v[i]));
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i] = __fadd_rn(acc[i], v[i]);
      }
      if (dual) {
        const float* xr2 = a.x2 + (int64_t)c * a.ldx2 + f0;
        const float we2 = wtd2 ? edge_weight(a.w2, a.widx2, e) : 1.0f;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (i < nf) acc[i] = __fadd_rn(acc[i], __fmul_rn(we2, __ldg(xr2 + i)));
      }
    }
    float* yr = a.y + (r - a.y_row0) * a.ldy + f0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (i < nf) {
        float o = acc[i];
        if (a.bias) o = __fadd_rn(o, __ldg(a.bias + f0 + i));
        if (a.accumulate) o = __fadd_rn(yr[i], o);
        yr[i] = o;
      }
    }
  }
}

// ------------------------------------------------------------------------- //
// tensor-core engine
// ------------------------------------------------------------------------- //

constexpr int kTcWarps = 4;
constexpr int kBlocksPerRound = 16;  // condensed 16x8 tiles staged per round

template <int NT, bool VEC>
__device__ __forceinline__ void load_slice(float (&v)[NT], const float* __restrict__ x,
                                           int64_t node, int64_t ld, int f0, int dim) {
  if (node < 0) {
#pragma unroll
    for (int j = 0; j < NT; ++j) v[j] = 0.f;
    return;
  }
  const float* p = x + node * ld + f0;
  if (VEC && f0 + NT <= dim) {
    if constexpr (NT % 4 == 0) {
#pragma unroll
      for (int j = 0; j < NT; j += 4) {
        float4 q = __ldg(reinterpret_cast<const float4*>(p + j));
        v[j] = q.x, v[j + 1] = q.y, v[j + 2] = q.z, v[j + 3] = q.w;
      }
      return;
    } else if constexpr (NT % 2 == 0) {
#pragma unroll
      for (int j = 0; j < NT; j += 2) {
        float2 q = __ldg(reinterpret_cast<const float2*>(p + j));
        v[j] = q.x, v[j + 1] = q.y;
      }
      return;
    }
  }
#pragma unroll
  for (int j = 0; j < NT; ++j) v[j] = (f0 + j < dim) ? __ldg(p + j) : 0.f;
}

template <int NT, bool VEC, bool DUAL>
__global__ void __launch_bounds__(kTcWarps * 32) spmm_tc(SpmmArgs a, int nchunks) {
  extern __shared__ __align__(16) uint32_t smem_u32[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  constexpr int kBufWords = kBlocksPerRound * 128;
  uint32_t* abuf = smem_u32 + warp * (kBufWords * (DUAL ? 2 : 1));
  uint32_t* abuf2 = abuf + kBufWords;
  __shared__ int64_t rps_all[kTcWarps][17];  // window row pointers
  int64_t* rps = rps_all[warp];

  const int64_t task = (int64_t)blockIdx.x * kTcWarps + warp;
  if (task >= a.nwin * nchunks) return;
  const int64_t w = a.win_begin + task / nchunks;
  const int chunk = (int)(task % nchunks);
  const int d0 = chunk * 8 * NT;
  const int64_t r0 = w * 16;
  const int64_t r1 = min(r0 + 16, a.n);
  if (lane <= 16) rps[lane] = __ldg(a.ptr + min(r0 + lane, r1));
  const int64_t c0 = __ldg(a.col_offsets + w);
  const int64_t cend = __ldg(a.col_offsets + w + 1);
  const int nb = (int)__ldg(a.wp + w);
  __syncwarp();
  const int64_t e0 = rps[0], e1 = rps[16];

  float acc[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;

  for (int bb = 0; bb < nb; bb += kBlocksPerRound) {
    const int nbr = min(kBlocksPerRound, nb - bb);
    // zero the staged A fragments of this round
    for (int i = lane; i < nbr * 32; i += 32) {
      reinterpret_cast<uint4*>(abuf)[i] = make_uint4(0, 0, 0, 0);
      if (DUAL) reinterpret_cast<uint4*>(abuf2)[i] = make_uint4(0, 0, 0, 0);
    }
    __syncwarp();
    // InitSparse: scatter edge values into fragment order
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const uint32_t c = __ldg(a.e2c + e);
      const int b = (int)(c >> 3) - bb;
      if (b < 0 || b >= nbr) continue;
      int row = 0;
#pragma unroll
      for (int s = 8; s > 0; s >>= 1)
        if (rps[row + s] <= e) row += s;
      const int k = c & 7;
      const int slot = (row >> 3) + 2 * (k >> 2);
      const int idx = b * 128 + (((row & 7) << 2) | (k & 3)) * 4 + slot;
      abuf[idx] = tf32_rn(edge_weight(a.w, a.widx, e));
      if (DUAL) abuf2[idx] = tf32_rn(a.w2 ? edge_weight(a.w2, a.widx2, e) : 1.0f);
    }
    __syncwarp();
    // FetchDense + MMA, one tile ahead in registers
    const int fl = d0 + g * NT;
    auto node_of = [&](int b, int k) -> int64_t {
      const int64_t ci = c0 + (int64_t)(bb + b) * 8 + k;
      return ci < cend ? (int64_t)__ldg(a.c2n + ci) : -1;
    };
    float xv0[NT], xv1[NT], nx0[NT], nx1[NT];
    float yv0[NT], yv1[NT], ny0[NT], ny1[NT];
    {
      const int64_t n0 = node_of(0, t), n1 = node_of(0, t + 4);
      load_slice<NT, VEC>(xv0, a.x, n0, a.ldx, fl, a.dim);
      load_slice<NT, VEC>(xv1, a.x, n1, a.ldx, fl, a.dim);
      if (DUAL) {
        load_slice<NT, VEC>(yv0, a.x2, n0, a.ldx2, fl, a.dim);
        load_slice<NT, VEC>(yv1, a.x2, n1, a.ldx2, fl, a.dim);
      }
    }
    for (int b = 0; b < nbr; ++b) {
      if (b + 1 < nbr) {
        const int64_t n0 = node_of(b + 1, t), n1 = node_of(b + 1, t + 4);
        load_slice<NT, VEC>(nx0, a.x, n0, a.ldx, fl, a.dim);
        load_slice<NT, VEC>(nx1, a.x, n1, a.ldx, fl, a.dim);
        if (DUAL) {
          load_slice<NT, VEC>(ny0, a.x2, n0, a.ldx2, fl, a.dim);
          load_slice<NT, VEC>(ny1, a.x2, n1, a.ldx2, fl, a.dim);
        }
      }
      const uint4 af = reinterpret_cast<const uint4*>(abuf)[b * 32 + lane];
#pragma unroll
      for (int j = 0; j < NT; ++j)
        mma_tf32(acc[j], af.x, af.y, af.z, af.w, tf32_rn(xv0[j]), tf32_rn(xv1[j]));
      if (DUAL) {
        const uint4 af2 = reinterpret_cast<const uint4*>(abuf2)[b * 32 + lane];
#pragma unroll
        for (int j = 0; j < NT; ++j)
          mma_tf32(acc[j], af2.x, af2.y, af2.z, af2.w, tf32_rn(yv0[j]), tf32_rn(yv1[j]));
      }
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        xv0[j] = nx0[j];
        xv1[j] = nx1[j];
        if (DUAL) {
          yv0[j] = ny0[j];
          yv1[j] = ny1[j];
        }
      }
    }
    __syncwarp();
  }

  // StoreDense: lane owns rows g, g+8 and features [d0 + 2t*NT, +2NT)
  const int fo = d0 + 2 * t * NT;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t r = r0 + g + 8 * h;
    if (r >= r1) continue;
    float o[2 * NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      o[j] = acc[j][2 * h];
      o[NT + j] = acc[j][2 * h + 1];
    }
    float* yr = a.y + (r - a.y_row0) * a.ldy + fo;
    if (VEC && fo + 2 * NT <= a.dim && ((2 * NT) % 4 == 0)) {
#pragma unroll
      for (int q = 0; q < 2 * NT; q += 4) {
        float4 v = make_float4(o[q], o[q + 1], o[q + 2], o[q + 3]);
        if (a.bias) {
          float4 bv = __ldg(reinterpret_cast<const float4*>(a.bias + fo + q));
          v.x += bv.x, v.y += bv.y, v.z += bv.z, v.w += bv.w;
        }
        if (a.accumulate) {
          float4 old = *reinterpret_cast<float4*>(yr + q);
          v.x += old.x, v.y += old.y, v.z += old.z, v.w += old.w;
        }
        *reinterpret_cast<float4*>(yr + q) = v;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 2 * NT; ++q) {
        if (fo + q < a.dim) {
          float v = o[q];
          if (a.bias) v += __ldg(a.bias + fo + q);
          if (a.accumulate) v += yr[q];
          yr[q] = v;
        }
      }
    }
  }
}

template <int NT, bool VEC, bool DUAL>
int launch_tc(const SpmmArgs& a, int nchunks, cudaStream_t s) {
  const int64_t tasks = a.nwin * nchunks;
  const int64_t blocks = (tasks + kTcWarps - 1) / kTcWarps;
  const size_t smem = (size_t)kTcWarps * (kBlocksPerRound * 128 * (DUAL ? 2 : 1)) * 4;
  auto kern = spmm_tc<NT, VEC, DUAL>;
  static bool attr_set = false;
  if (!attr_set) {
    TCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
             "spmm_tc attr");
    attr_set = true;
  }
  kern<<<(unsigned)blocks, kTcWarps * 32, smem, s>>>(a, nchunks);
  TCG_LAUNCHED("spmm_tc");
  return TCG_OK;
}

template <bool VEC, bool DUAL>
int dispatch_nt(int nt, const SpmmArgs& a, int nchunks, cudaStream_t s) {
  switch (nt) {
    case 1: return launch_tc<1, VEC, DUAL>(a, nchunks, s);
    case 2: return launch_tc<2, VEC, DUAL>(a, nchunks, s);
    case 3: return launch_tc<3, false, DUAL>(a, nchunks, s);
    case 4: return launch_tc<4, VEC, DUAL>(a, nchunks, s);
    case 5: return launch_tc<5, false, DUAL>(a, nchunks, s);
    case 6: return launch_tc<6, VEC, DUAL>(a, nchunks, s);
    case 7: return launch_tc<7, false, DUAL>(a, nchunks, s);
    default: return launch_tc<8, VEC, DUAL>(a, nchunks, s);
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace
}  // namespace tcg

using namespace tcg;

extern "C" int tcg_spmm(const tcg_tiling* t, const float* x, int64_t ldx, int64_t dim,
                        const float* weights, const uint32_t* weight_idx, const float* x2,
                        int64_t ldx2, const float* weights2, const uint32_t* weight_idx2,
                        const float* bias, float* y, int64_t ldy, int64_t y_row0,
                        int64_t win_begin, int64_t win_end, int32_t precision, int32_t accumulate,
                        void* stream) {
  TCG_REQUIRE(t != nullptr, "tcg_spmm: null tiling");
  TCG_REQUIRE(dim >= 1, "tcg_spmm: embedding dimension must be >= 1, got %lld", (long long)dim);
  TCG_REQUIRE(ldx >= dim && ldy >= dim, "tcg_spmm: leading dimension < dim");
  TCG_REQUIRE(x2 == nullptr || ldx2 >= dim, "tcg_spmm: ldx2 < dim");
  TCG_REQUIRE(0 <= win_begin && win_begin <= win_end && win_end <= t->num_windows,
              "tcg_spmm: window range [%lld, %lld) outside [0, %lld)", (long long)win_begin,
              (long long)win_end, (long long)t->num_windows);
  TCG_REQUIRE(precision == TCG_PREC_F32 || precision == TCG_PREC_TF32,
              "tcg_spmm: unknown precision %d", precision);
  if (win_begin == win_end || t->num_nodes == 0) return TCG_OK;
  TCG_REQUIRE(x && y && t->node_ptr, "tcg_spmm: null pointer");
  cudaStream_t s = as_stream(stream);
  SpmmArgs a{};
  a.ptr = t->node_ptr;
  a.cols = t->edge_list;
  a.e2c = t->edge_to_col;
  a.col_offsets = t->col_offsets;
  a.c2n = t->col_to_node;
  a.wp = t->win_partition;
  a.n = t->num_nodes;
  a.x = x, a.ldx = ldx, a.w = weights, a.widx = weight_idx;
  a.x2 = x2, a.ldx2 = ldx2, a.w2 = weights2, a.widx2 = weight_idx2;
  a.bias = bias, a.y = y, a.ldy = ldy, a.y_row0 = y_row0;
  a.row_begin = win_begin * t->blk_h;
  a.row_end = win_end * (int64_t)t->blk_h < t->num_nodes ? win_end * (int64_t)t->blk_h
                                                          : t->num_nodes;
  a.win_begin = win_begin;
  a.nwin = win_end - win_begin;
  a.dim = (int)dim;
  a.accumulate = accumulate;
  TCG_REQUIRE(a.row_begin <= a.y_row0 || a.row_begin >= a.row_end,
              "tcg_spmm: y_row0 beyond first output row");

  if (precision == TCG_PREC_F32) {
    TCG_REQUIRE(t->edge_list != nullptr || t->num_edges == 0, "tcg_spmm: null edge_list");
    const bool vec = dim % 4 == 0 && ldx % 4 == 0 && aligned16(x) &&
                     (x2 == nullptr || (ldx2 % 4 == 0 && aligned16(x2)));
    int quads = (int)((dim + 3) / 4);
    int G = 1;
    while (G < quads && G < 32) G <<= 1;
    const int64_t rows = a.row_end - a.row_begin;
    const int64_t threads = rows * G;
    const int tpb = 256;
    const unsigned blocks = (unsigned)((threads + tpb - 1) / tpb);
#define TCG_EXACT(GG)                                              \
  case GG:                                                         \
    if (vec)                                                       \
      spmm_exact<GG, true><<<blocks, tpb, 0, s>>>(a);              \
    else                                                           \
      spmm_exact<GG, false><<<blocks, tpb, 0, s>>>(a);             \
    break;
    switch (G) {
      TCG_EXACT(1)
      TCG_EXACT(2)
      TCG_EXACT(4)
      TCG_EXACT(8)
      TCG_EXACT(16)
      TCG_EXACT(32)
    }
#undef TCG_EXACT
    TCG_LAUNCHED("spmm_exact");
    return TCG_OK;
  }

  TCG_REQUIRE(t->blk_h == 16 && t->blk_w == 8,
              "tf32 mode requires the 16x8 tile shape, got %dx%d", t->blk_h, t->blk_w);
  TCG_REQUIRE(t->col_offsets && t->win_partition &&
                  (t->num_edges == 0 || (t->edge_to_col && t->col_to_node)),
              "tcg_spmm: tiling arrays missing");
  int nt, nchunks;
  if (dim <= 64) {
    nt = (int)((dim + 7) / 8);
    nchunks = 1;
  } else {
    nt = 8;
    nchunks = (int)((dim + 63) / 64);
  }
  const bool vec = ldx % 4 == 0 && ldy % 4 == 0 && aligned16(x) && aligned16(y) &&
                   (bias == nullptr || aligned16(bias)) &&
                   (x2 == nullptr || (ldx2 % 4 == 0 && aligned16(x2)));
  if (x2 != nullptr)
    return vec ? dispatch_nt<true, true>(nt, a, nchunks, s)
               : dispatch_nt<false, true>(nt, a, nchunks, s);
  return vec ? dispatch_nt<true, false>(nt, a, nchunks, s)
             : dispatch_nt<false, false>(nt, a, nchunks, s);
}
