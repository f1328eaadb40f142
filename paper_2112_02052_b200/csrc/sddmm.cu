// Edge attention scores F[e] = <Xa[row e], Xb[col e]> over the SGT tiling —
// replaces the reference kernels.sddmm (/root/reference/pkg/src/tcgraph/
// kernels.py:377-538, Alg. 3) and, fused into its epilogue, the row
// softmax kernels.segment_softmax (kernels.py:541-556) and its backward.
//
// One warp per 16-row window in both engines:
//  * sddmm_exact (TCG_PREC_F32): lanes over the window's edges, each folding
//    k ascending from +0.0 with one rounding per product and add — bitwise
//    equal to the reference f32 path (kernels.py:518-525).
//  * sddmm_tc (TCG_PREC_TF32, 16x8 only): the window's 16 rows are the A
//    operand (held in registers for D <= 64), each 16-column paired block of
//    condensed neighbours (paired_block_counts, sgt.py:190-198) is the B
//    operand, gathered with vector loads through a feature permutation; the
//    D dimension is the mma k dimension (m16n8k8 TF32, RNE operands, fp32
//    accumulate). 16x16 output tiles go to shared memory and are scattered
//    to edge order (StoreSparse, tiles.py:223-250).
// Epilogues run on the window's edges while they are hot in L1: row softmax
// (rows never straddle windows) or dS = P * (dP - rowsum(P dP)).
#include "common.cuh"

namespace tcg {
namespace {

constexpr int kWarps = 4;
constexpr int kPairsPerRound = 8;  // 16x16 output tiles staged per round

struct SddmmArgs {
  const int64_t* ptr;
  const uint32_t* cols;
  const uint32_t* e2c;
  const int64_t* col_offsets;
  const uint32_t* c2n;
  const uint32_t* wp;
  int64_t n;
  int bh;
  const float* xa;
  int64_t lda;
  const float* xb;
  int64_t ldb;
  const float* aux;
  float* out;
  int64_t e_base;
  int64_t win_begin, nwin;
  int dim;
  int epilogue;
};

// Row softmax / softmax-backward over the window's rows [r0, r1), values in
// out[e - e_base] already written by this warp.
__device__ __forceinline__ void window_epilogue(const SddmmArgs& a, int64_t r0, int64_t r1) {
  if (a.epilogue == TCG_EPI_NONE) return;
  __syncwarp();
  const int lane = threadIdx.x & 31;
  for (int64_t r = r0; r < r1; ++r) {
    const int64_t s = __ldg(a.ptr + r), e = __ldg(a.ptr + r + 1);
    if (s == e) continue;
    float* o = a.out - a.e_base;
    if (a.epilogue == TCG_EPI_SOFTMAX) {
      float m = -INFINITY;
      for (int64_t i = s + lane; i < e; i += 32) m = fmaxf(m, o[i]);
      m = warp_max(m);
      float sum = 0.f;
      for (int64_t i = s + lane; i < e; i += 32) sum += expf(o[i] - m);
      sum = warp_sum(sum);
      for (int64_t i = s + lane; i < e; i += 32) o[i] = expf(o[i] - m) / sum;
    } else {
      const float* p = a.aux - a.e_base;
      float dot = 0.f;
      for (int64_t i = s + lane; i < e; i += 32) dot += p[i] * o[i];
      dot = warp_sum(dot);
      for (int64_t i = s + lane; i < e; i += 32) o[i] = p[i] * (o[i] - dot);
    }
  }
}

__device__ __forceinline__ int64_t find_row(const int64_t* ptr, int64_t r0, int64_t r1,
                                             int64_t e) {
  // largest r in [r0, r1) with ptr[r] <= e
  int64_t lo = r0, hi = r1 - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (__ldg(ptr + mid) <= e) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(kWarps * 32) sddmm_exact(SddmmArgs a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t task = (int64_t)blockIdx.x * kWarps + warp;
  if (task >= a.nwin) return;
  const int64_t w = a.win_begin + task;
  const int64_t r0 = w * a.bh, r1 = min(r0 + a.bh, a.n);
  const int64_t e0 = __ldg(a.ptr + r0), e1 = __ldg(a.ptr + r1);
  const bool vec = (a.dim % 4 == 0) && (a.lda % 4 == 0) && (a.ldb % 4 == 0) &&
                   ((reinterpret_cast<uintptr_t>(a.xa) | reinterpret_cast<uintptr_t>(a.xb)) & 15) == 0;
  for (int64_t e = e0 + lane; e < e1; e += 32) {
    const int64_t r = find_row(a.ptr, r0, r1, e);
    const uint32_t c = __ldg(a.cols + e);
    const float* pa = a.xa + r * a.lda;
    const float* pb = a.xb + (int64_t)c * a.ldb;
    float acc = 0.f;
    if (vec) {
      for (int k = 0; k < a.dim; k += 4) {
        const float4 u = __ldg(reinterpret_cast<const float4*>(pa + k));
        const float4 v = __ldg(reinterpret_cast<const float4*>(pb + k));
        acc = __fadd_rn(acc, __fmul_rn(u.x, v.x));
        acc = __fadd_rn(acc, __fmul_rn(u.y, v.y));
        acc = __fadd_rn(acc, __fmul_rn(u.z, v.z));
        acc = __fadd_rn(acc, __fmul_rn(u.w, v.w));
      }
    } else {
      for (int k = 0; k < a.dim; ++k) acc = __fadd_rn(acc, __fmul_rn(__ldg(pa + k), __ldg(pb + k)));
    }
    a.out[e - a.e_base] = acc;
  }
  window_epilogue(a, r0, r1);
}

template <int KT, bool VEC>
__device__ __forceinline__ void load_k(float (&v)[KT], const float* __restrict__ x, int64_t row,
                                       int64_t ld, int f0, int dim) {
  if (row < 0) {
#pragma unroll
    for (int j = 0; j < KT; ++j) v[j] = 0.f;
    return;
  }
  const float* p = x + row * ld + f0;
  if (VEC && f0 + KT <= dim) {
    if constexpr (KT % 4 == 0) {
#pragma unroll
      for (int j = 0; j < KT; j += 4) {
        float4 q = __ldg(reinterpret_cast<const float4*>(p + j));
        v[j] = q.x, v[j + 1] = q.y, v[j + 2] = q.z, v[j + 3] = q.w;
      }
      return;
    } else if constexpr (KT % 2 == 0) {
#pragma unroll
      for (int j = 0; j < KT; j += 2) {
        float2 q = __ldg(reinterpret_cast<const float2*>(p + j));
        v[j] = q.x, v[j + 1] = q.y;
      }
      return;
    }
  }
#pragma unroll
  for (int j = 0; j < KT; ++j) v[j] = (f0 + j < dim) ? __ldg(p + j) : 0.f;
}

// KT = k-steps (of 8 features) per chunk; nkc chunks cover D.
template <int KT, bool VEC>
__global__ void __launch_bounds__(kWarps * 32) sddmm_tc(SddmmArgs a, int nkc) {
  __shared__ __align__(16) float tiles[kWarps][kPairsPerRound][16][17];
  __shared__ int64_t rps_all[kWarps][17];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int64_t task = (int64_t)blockIdx.x * kWarps + warp;
  if (task >= a.nwin) return;
  const int64_t w = a.win_begin + task;
  const int64_t r0 = w * 16, r1 = min(r0 + 16, a.n);
  int64_t* rps = rps_all[warp];
  if (lane <= 16) rps[lane] = __ldg(a.ptr + min(r0 + lane, r1));
  const int64_t c0 = __ldg(a.col_offsets + w);
  const int64_t cend = __ldg(a.col_offsets + w + 1);
  const int nsb = (int)((cend - c0 + 15) >> 4);
  __syncwarp();
  const int64_t e0 = rps[0], e1 = rps[16];
  if (e0 == e1) return;
  const int64_t ra = r0 + g < r1 ? r0 + g : -1;
  const int64_t rb = r0 + 8 + g < r1 ? r0 + 8 + g : -1;

  // A fragments (window rows), kept for all paired blocks when nkc == 1
  float A0[KT], A1[KT], A2[KT], A3[KT];
  if (nkc == 1) {
    load_k<KT, VEC>(A0, a.xa, ra, a.lda, t * KT, a.dim);
    load_k<KT, VEC>(A1, a.xa, rb, a.lda, t * KT, a.dim);
    load_k<KT, VEC>(A2, a.xa, ra, a.lda, (t + 4) * KT, a.dim);
    load_k<KT, VEC>(A3, a.xa, rb, a.lda, (t + 4) * KT, a.dim);
  }
  float (*tl)[16][17] = tiles[warp];
  for (int sbb = 0; sbb < nsb; sbb += kPairsPerRound) {
    const int nr = min(kPairsPerRound, nsb - sbb);
    for (int sb = 0; sb < nr; ++sb) {
      const int64_t ci0 = c0 + (int64_t)(sbb + sb) * 16 + g;
      const int64_t n0 = ci0 < cend ? (int64_t)__ldg(a.c2n + ci0) : -1;
      const int64_t n1 = ci0 + 8 < cend ? (int64_t)__ldg(a.c2n + ci0 + 8) : -1;
      float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
      for (int kc = 0; kc < nkc; ++kc) {
        const int f0 = kc * 8 * KT;
        if (nkc > 1) {
          load_k<KT, VEC>(A0, a.xa, ra, a.lda, f0 + t * KT, a.dim);
          load_k<KT, VEC>(A1, a.xa, rb, a.lda, f0 + t * KT, a.dim);
          load_k<KT, VEC>(A2, a.xa, ra, a.lda, f0 + (t + 4) * KT, a.dim);
          load_k<KT, VEC>(A3, a.xa, rb, a.lda, f0 + (t + 4) * KT, a.dim);
        }
        float B0[KT], B1[KT], B2[KT], B3[KT];
        load_k<KT, VEC>(B0, a.xb, n0, a.ldb, f0 + t * KT, a.dim);
        load_k<KT, VEC>(B1, a.xb, n0, a.ldb, f0 + (t + 4) * KT, a.dim);
        load_k<KT, VEC>(B2, a.xb, n1, a.ldb, f0 + t * KT, a.dim);
        load_k<KT, VEC>(B3, a.xb, n1, a.ldb, f0 + (t + 4) * KT, a.dim);
#pragma unroll
        for (int j = 0; j < KT; ++j) {
          const uint32_t a0 = tf32_rn(A0[j]), a1 = tf32_rn(A1[j]);
          const uint32_t a2 = tf32_rn(A2[j]), a3 = tf32_rn(A3[j]);
          mma_tf32(acc[0], a0, a1, a2, a3, tf32_rn(B0[j]), tf32_rn(B1[j]));
          mma_tf32(acc[1], a0, a1, a2, a3, tf32_rn(B2[j]), tf32_rn(B3[j]));
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        tl[sb][g][h * 8 + 2 * t] = acc[h][0];
        tl[sb][g][h * 8 + 2 * t + 1] = acc[h][1];
        tl[sb][g + 8][h * 8 + 2 * t] = acc[h][2];
        tl[sb][g + 8][h * 8 + 2 * t + 1] = acc[h][3];
      }
    }
    __syncwarp();
    // StoreSparse: edges whose condensed column falls in this round
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const uint32_t c = __ldg(a.e2c + e);
      const int sb = (int)(c >> 4) - sbb;
      if (sb < 0 || sb >= nr) continue;
      int row = 0;
#pragma unroll
      for (int s = 8; s > 0; s >>= 1)
        if (rps[row + s] <= e) row += s;
      a.out[e - a.e_base] = tl[sb][row][c & 15];
    }
    __syncwarp();
  }
  window_epilogue(a, r0, r1);
}

template <int KT, bool VEC>
int launch_tc(const SddmmArgs& a, int nkc, cudaStream_t s) {
  const unsigned blocks = (unsigned)((a.nwin + kWarps - 1) / kWarps);
  sddmm_tc<KT, VEC><<<blocks, kWarps * 32, 0, s>>>(a, nkc);
  TCG_LAUNCHED("sddmm_tc");
  return TCG_OK;
}

template <bool VEC>
int dispatch_kt(int kt, const SddmmArgs& a, int nkc, cudaStream_t s) {
  switch (kt) {
    case 1: return launch_tc<1, VEC>(a, nkc, s);
    case 2: return launch_tc<2, VEC>(a, nkc, s);
    case 3: return launch_tc<3, false>(a, nkc, s);
    case 4: return launch_tc<4, VEC>(a, nkc, s);
    case 5: return launch_tc<5, false>(a, nkc, s);
    case 6: return launch_tc<6, VEC>(a, nkc, s);
    case 7: return launch_tc<7, false>(a, nkc, s);
    default: return launch_tc<8, VEC>(a, nkc, s);
  }
}

}  // namespace
}  // namespace tcg

using namespace tcg;

extern "C" int tcg_sddmm(const tcg_tiling* t, const float* xa, int64_t lda, const float* xb,
                         int64_t ldb, int64_t dim, const float* aux, float* out,
                         int64_t win_begin, int64_t win_end, int32_t precision, int32_t epilogue,
                         void* stream) {
  TCG_REQUIRE(t != nullptr, "tcg_sddmm: null tiling");
  TCG_REQUIRE(dim >= 1, "tcg_sddmm: embedding dimension must be >= 1");
  TCG_REQUIRE(lda >= dim && ldb >= dim, "tcg_sddmm: leading dimension < dim");
  TCG_REQUIRE(0 <= win_begin && win_begin <= win_end && win_end <= t->num_windows,
              "tcg_sddmm: window range outside [0, %lld)", (long long)t->num_windows);
  TCG_REQUIRE(precision == TCG_PREC_F32 || precision == TCG_PREC_TF32,
              "tcg_sddmm: unknown precision %d", precision);
  TCG_REQUIRE(epilogue >= TCG_EPI_NONE && epilogue <= TCG_EPI_SOFTMAX_BWD,
              "tcg_sddmm: unknown epilogue %d", epilogue);
  TCG_REQUIRE(epilogue != TCG_EPI_SOFTMAX_BWD || aux != nullptr,
              "tcg_sddmm: softmax backward needs P");
  if (win_begin == win_end || t->num_edges == 0) return TCG_OK;
  if (xb == nullptr) {
    xb = xa;
    ldb = lda;
  }
  TCG_REQUIRE(xa && out && t->node_ptr && t->edge_list, "tcg_sddmm: null pointer");
  cudaStream_t s = as_stream(stream);
  SddmmArgs a{};
  a.ptr = t->node_ptr;
  a.cols = t->edge_list;
  a.e2c = t->edge_to_col;
  a.col_offsets = t->col_offsets;
  a.c2n = t->col_to_node;
  a.wp = t->win_partition;
  a.n = t->num_nodes;
  a.bh = t->blk_h;
  a.xa = xa, a.lda = lda, a.xb = xb, a.ldb = ldb;
  a.aux = aux, a.out = out;
  a.win_begin = win_begin;
  a.nwin = win_end - win_begin;
  a.dim = (int)dim;
  a.epilogue = epilogue;
  a.e_base = 0;  // edge arrays are indexed by absolute edge id
  if (precision == TCG_PREC_F32) {
    const unsigned blocks = (unsigned)((a.nwin + kWarps - 1) / kWarps);
    sddmm_exact<<<blocks, kWarps * 32, 0, s>>>(a);
    TCG_LAUNCHED("sddmm_exact");
    return TCG_OK;
  }
  TCG_REQUIRE(t->blk_h == 16 && t->blk_w == 8,
              "tf32 mode requires the 16x8 tile shape, got %dx%d", t->blk_h, t->blk_w);
  int kt, nkc;
  if (dim <= 64) {
    kt = (int)((dim + 7) / 8);
    nkc = 1;
  } else {
    kt = 8;
    nkc = (int)((dim + 63) / 64);
  }
  const bool vec = lda % 4 == 0 && ldb % 4 == 0 &&
                   ((reinterpret_cast<uintptr_t>(xa) | reinterpret_cast<uintptr_t>(xb)) & 15) == 0;
  return vec ? dispatch_kt<true>(kt, a, nkc, s) : dispatch_kt<false>(kt, a, nkc, s);
}
