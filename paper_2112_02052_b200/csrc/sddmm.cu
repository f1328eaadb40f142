#include <algorithm>
#include <cstdlib>
// Edge attention scores F[e] = <Xa[row e], Xb[col e]> over the SGT tiling —
// replaces the reference kernels.sddmm (/root/reference/pkg/src/tcgraph/
// kernels.py:377-538, Alg. 3) and, fused into its epilogue, the row softmax
// kernels.segment_softmax (kernels.py:541-556) and its backward; plus the
// fused AGNN layer entry points (kernels.agnn_layer, kernels.py:586-601).
//
//  * sddmm_exact (TCG_PREC_F32): one warp per window, lanes over its edges,
//    each folding k ascending from +0.0 with one rounding per product and
//    add — bitwise equal to the reference f32 path (kernels.py:518-525).
//  * TCG_PREC_TF32: the tensor-core row-window engine (window.cu, modes
//    SDDMM, AGNN_FWD, AGNN_BWD).
#include "common.cuh"
#include "window.cuh"

namespace tcg {
namespace {

constexpr int kWarps = 4;

struct ExactArgs {
  const int64_t* ptr;
  const uint32_t* cols;
  int64_t n;
  int bh;
  const float* xa;
  int64_t lda;
  const float* xb;
  int64_t ldb;
  const float* aux;
  float* out;
  int64_t win_begin, nwin;
  int dim;
  int epilogue;
  int vec;
};

__device__ __forceinline__ int64_t find_row(const int64_t* ptr, int64_t r0, int64_t r1,
                                             int64_t e) {
  int64_t lo = r0, hi = r1 - 1;  // largest r in [r0, r1) with ptr[r] <= e
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (__ldg(ptr + mid) <= e) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(kWarps * 32) sddmm_exact(ExactArgs a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t task = (int64_t)blockIdx.x * kWarps + warp;
  if (task >= a.nwin) return;
  const int64_t w = a.win_begin + task;
  const int64_t r0 = w * a.bh, r1 = min(r0 + a.bh, a.n);
  const int64_t e0 = __ldg(a.ptr + r0), e1 = __ldg(a.ptr + r1);
  for (int64_t e = e0 + lane; e < e1; e += 32) {
    const int64_t r = find_row(a.ptr, r0, r1, e);
    const uint32_t c = __ldg(a.cols + e);
    const float* pa = a.xa + r * a.lda;
    const float* pb = a.xb + (int64_t)c * a.ldb;
    float acc = 0.f;
    if (a.vec) {
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
    a.out[e] = acc;
  }
  if (a.epilogue == TCG_EPI_NONE) return;
  __syncwarp();
  for (int64_t r = r0; r < r1; ++r) {
    const int64_t s = __ldg(a.ptr + r), e = __ldg(a.ptr + r + 1);
    if (s == e) continue;
    if (a.epilogue == TCG_EPI_SOFTMAX) {
      float m = -INFINITY;
      for (int64_t i = s + lane; i < e; i += 32) m = fmaxf(m, a.out[i]);
      m = warp_max(m);
      float sum = 0.f;
      for (int64_t i = s + lane; i < e; i += 32) sum += expf(a.out[i] - m);
      sum = warp_sum(sum);
      for (int64_t i = s + lane; i < e; i += 32) a.out[i] = expf(a.out[i] - m) / sum;
    } else {
      float dot = 0.f;
      for (int64_t i = s + lane; i < e; i += 32) dot += __ldg(a.aux + i) * a.out[i];
      dot = warp_sum(dot);
      for (int64_t i = s + lane; i < e; i += 32) a.out[i] = __ldg(a.aux + i) * (a.out[i] - dot);
    }
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

win::Params base_params(const tcg_tiling* t, int64_t win_begin, int64_t win_end) {
  win::Params q{};
  q.ptr = t->node_ptr;
  q.e2c = t->edge_to_col;
  q.efrag = t->edge_frag;
  q.coff = t->col_offsets;
  q.c2n = t->col_to_node;
  q.n = t->num_nodes;
  q.win_begin = win_begin;
  q.nwin = win_end - win_begin;
  q.nchunks = 1;
  q.nkc = 1;
  return q;
}

// fused AGNN kernels keep the whole window in shared memory
bool fits_fused(const tcg_tiling* t, int nt) {
  return t->max_window_edges > 0 && t->max_window_edges <= win::kEdgesPerWindow &&
         t->max_window_unique <= win::cols_per_round(nt, win::MODE_AGNN_FWD);
}

// windows too wide for the fused stream kernels: the two-step form on the block
// stream (sddmm_wide + row epilogue, then the stream SpMM) beats the window
// engine's fused kernels there (products D=16: the SDDMM alone 7.1 -> 1.7 ms)
bool wide_two_step(const tcg_tiling* t, int64_t dim) {
  static const bool off = std::getenv("TCG_NO_STREAM") != nullptr || std::getenv("TCG_AGNN_WIN_FUSED") != nullptr;
  return !off && dim <= 32 && dim % 4 == 0 && stream_sddmm_wide(t);
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
  if (xb == nullptr) {
    xb = xa;
    ldb = lda;
  }
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
  TCG_REQUIRE(xa && out && t->node_ptr && t->edge_list, "tcg_sddmm: null pointer");
  cudaStream_t s = as_stream(stream);
  const bool vec = dim % 4 == 0 && lda % 4 == 0 && ldb % 4 == 0 && aligned16(xa) && aligned16(xb);
  if (precision == TCG_PREC_F32) {
    ExactArgs a{t->node_ptr, t->edge_list, t->num_nodes, t->blk_h, xa, lda, xb, ldb, aux, out,
                win_begin, win_end - win_begin, (int)dim, epilogue, vec ? 1 : 0};
    const unsigned blocks = (unsigned)((a.nwin + kWarps - 1) / kWarps);
    sddmm_exact<<<blocks, kWarps * 32, 0, s>>>(a);
    TCG_LAUNCHED("sddmm_exact");
    return TCG_OK;
  }
  TCG_REQUIRE(t->blk_h == 16 && t->blk_w == 8,
              "tf32 mode requires the 16x8 tile shape, got %dx%d", t->blk_h, t->blk_w);
  TCG_REQUIRE(t->edge_frag, "tcg_sddmm: tf32 needs edge_frag (tcg_edge_frag)");
  {
    static const bool no_stream = std::getenv("TCG_NO_STREAM") != nullptr;
    if (!no_stream && dim <= 32 && dim % 4 == 0) {
      const int rc = stream_sddmm(t, (int)dim, xa, lda, xb, ldb, aux, out, epilogue, win_begin, win_end, s);
      if (rc != TCG_E_UNSUPPORTED) return rc;
    }
  }
  win::Params q = base_params(t, win_begin, win_end);
  const int nt = win::nt_for(dim);
  const int kw = 8 * nt;  // features per launch (<= 64)
  const int nkc = (int)((dim + kw - 1) / kw);
  q.dim = (int)dim;
  q.vec16 = vec;
  q.x = xb, q.ldx = ldb, q.xa = xa, q.lda = lda;
  q.aux = aux, q.eout = out;
  // D > 64: partial dot products per 64-feature chunk, accumulated into out;
  // the row softmax (if any) then runs as its own pass
  q.epilogue = nkc == 1 ? epilogue : TCG_EPI_NONE;
  for (int kc = 0; kc < nkc; ++kc) {
    q.koff = kc * kw;
    q.accumulate = kc > 0;
    const int rc = win::launch(win::MODE_SDDMM, nt, q, s);
    if (rc != TCG_OK) return rc;
  }
  if (nkc > 1 && epilogue != TCG_EPI_NONE) {
    const int64_t rb = win_begin * 16;
    const int64_t re = win_end * 16 < t->num_nodes ? win_end * 16 : t->num_nodes;
    // rows [rb, re): the softmax kernels index node_ptr from the first row
    if (epilogue == TCG_EPI_SOFTMAX)
      return tcg_segment_softmax(t->node_ptr + rb, re - rb, out, out, stream);
    return tcg_segment_softmax_backward(t->node_ptr + rb, re - rb, aux, out, out, stream);
  }
  return TCG_OK;
}

// Output row r of a window-range call lands at y[r - y_row0]: valid when
// 0 <= y_row0 <= the range's first row (empty ranges write nothing).
static bool row0_ok(const tcg_tiling* t, int64_t win_begin, int64_t win_end, int64_t y_row0) {
  const int64_t rb = win_begin * t->blk_h;
  const int64_t re = std::min<int64_t>(win_end * (int64_t)t->blk_h, t->num_nodes);
  return rb >= re || (y_row0 >= 0 && y_row0 <= rb);
}

extern "C" int tcg_agnn_forward(const tcg_tiling* t, const float* z, int64_t ldz, int64_t dim,
                                float* p, float* y, int64_t ldy, int64_t y_row0,
                                int64_t win_begin, int64_t win_end, void* stream) {
  return tcg_agnn_forward_ex(t, z, ldz, dim, p, y, ldy, y_row0, win_begin, win_end, 0, stream);
}

extern "C" int tcg_agnn_forward_ex(const tcg_tiling* t, const float* z, int64_t ldz, int64_t dim,
                                   float* p, float* y, int64_t ldy, int64_t y_row0,
                                   int64_t win_begin, int64_t win_end, int32_t flags, void* stream) {
  TCG_REQUIRE((flags & ~TCG_AGNN_Z_TF32) == 0, "tcg_agnn_forward_ex: unknown flags 0x%x", flags);
  TCG_REQUIRE(t != nullptr && dim >= 1 && ldz >= dim && ldy >= dim,
              "tcg_agnn_forward: bad arguments");
  TCG_REQUIRE(t->blk_h == 16 && t->blk_w == 8,
              "tf32 mode requires the 16x8 tile shape, got %dx%d", t->blk_h, t->blk_w);
  TCG_REQUIRE(0 <= win_begin && win_begin <= win_end && win_end <= t->num_windows,
              "tcg_agnn_forward: window range outside [0, %lld)", (long long)t->num_windows);
  TCG_REQUIRE(row0_ok(t, win_begin, win_end, y_row0),
              "tcg_agnn_forward: y_row0 %lld beyond first output row", (long long)y_row0);
  const int nt = win::nt_for(dim);
  static const bool no_stream = std::getenv("TCG_NO_STREAM") != nullptr;
  if (!no_stream && dim <= 32 && dim % 4 == 0 && t->num_edges > 0 && win_begin < win_end && z && p &&
      y) {
    const int rc = stream_agnn(t, false, (int)dim, z, ldz, z, ldz, nullptr, 0, nullptr, p, y, ldy, y_row0,
                               win_begin, win_end, as_stream(stream), nullptr, nullptr, 0,
                               (flags & TCG_AGNN_Z_TF32) != 0);
    if (rc != TCG_E_UNSUPPORTED) return rc;
  }
  if (t->num_edges == 0 || dim > 64 || !fits_fused(t, nt) || wide_two_step(t, dim)) {
    if (t->num_edges) {
      int rc = tcg_sddmm(t, z, ldz, z, ldz, dim, nullptr, p, win_begin, win_end, TCG_PREC_TF32,
                         TCG_EPI_SOFTMAX, stream);
      if (rc != TCG_OK) return rc;
    }
    return tcg_spmm(t, z, ldz, dim, t->num_edges ? p : nullptr, nullptr, nullptr, 0, nullptr,
                    nullptr, nullptr, y, ldy, y_row0, win_begin, win_end, TCG_PREC_TF32, 0, stream);
  }
  if (win_begin == win_end) return TCG_OK;
  TCG_REQUIRE(z && p && y, "tcg_agnn_forward: null pointer");
  win::Params q = base_params(t, win_begin, win_end);
  q.dim = (int)dim;
  q.vec16 = dim % 4 == 0 && ldz % 4 == 0 && aligned16(z);
  q.vec_out = ldy % 4 == 0 && aligned16(y);
  q.x = z, q.ldx = ldz, q.xa = z, q.lda = ldz;
  q.eout = p, q.y = y, q.ldy = ldy, q.y_row0 = y_row0;
  return win::launch(win::MODE_AGNN_FWD, nt, q, as_stream(stream));
}

extern "C" int tcg_agnn_forward_next(const tcg_tiling* t, const float* z, int64_t ldz, int64_t dim, float* p,
                                     float* y, int64_t ldy, int64_t y_row0, int64_t win_begin, int64_t win_end,
                                     const float* w_next, int64_t co, float* z_next, int64_t ldzn, void* stream) {
  TCG_REQUIRE(t != nullptr && w_next && z_next && co >= 1 && ldzn >= co, "tcg_agnn_forward_next: bad arguments");
  static const bool no_stream = std::getenv("TCG_NO_STREAM") != nullptr;
  if (!no_stream && dim == 32 && co == 32 && t->num_edges > 0 && win_begin < win_end && z && p &&
      y && t->blk_h == 16 && t->blk_w == 8 && row0_ok(t, win_begin, win_end, y_row0)) {
    const int rc = stream_agnn(t, false, (int)dim, z, ldz, z, ldz, nullptr, 0, nullptr, p, y, ldy, y_row0,
                               win_begin, win_end, as_stream(stream), w_next, z_next, ldzn);
    if (rc != TCG_E_UNSUPPORTED) return rc;
  }
  // the two-step form: the aggregation, then the dense step on its rows
  const int rc = tcg_agnn_forward(t, z, ldz, dim, p, y, ldy, y_row0, win_begin, win_end, stream);
  if (rc != TCG_OK || win_begin == win_end) return rc;
  const int64_t r0 = win_begin * t->blk_h, r1 = std::min<int64_t>(win_end * (int64_t)t->blk_h, t->num_nodes);
  if (r1 <= r0) return TCG_OK;
  return tcg_dense(y + (r0 - y_row0) * ldy, ldy, r1 - r0, dim, w_next, co, 0, nullptr, 0, nullptr, 0,
                   z_next + (r0 - y_row0) * ldzn, ldzn, stream);
}

extern "C" int tcg_agnn_forward_t(const tcg_tiling* t, const float* z, int64_t ldz, int64_t dim,
                                  float* p, float* p_t, const uint32_t* inv_perm, float* y,
                                  int64_t ldy, int64_t y_row0, int64_t win_begin, int64_t win_end,
                                  void* stream) {
  const int rc = tcg_agnn_forward(t, z, ldz, dim, p, y, ldy, y_row0, win_begin, win_end, stream);
  if (rc != TCG_OK || !p_t || !inv_perm || !t || t->num_edges == 0) return rc;
  return tcg_scatter_f32(p, inv_perm, p_t, t->num_edges, stream);
}

extern "C" int tcg_agnn_backward_fused(const tcg_tiling* t, const float* z, int64_t ldz,
                                       const float* gy, int64_t ldg, const float* y_fwd,
                                       int64_t ld_yfwd, int64_t dim, const float* p, float* ds,
                                       float* ds_t, const uint32_t* inv_perm,
                                       float* dz, int64_t lddz, int64_t dz_row0,
                                       int64_t win_begin, int64_t win_end, void* stream) {
  return tcg_agnn_backward_fused_ex(t, z, ldz, gy, ldg, y_fwd, ld_yfwd, dim, p, ds, ds_t, inv_perm, dz, lddz,
                                    dz_row0, win_begin, win_end, 0, stream);
}

extern "C" int tcg_agnn_backward_fused_ex(const tcg_tiling* t, const float* z, int64_t ldz,
                                          const float* gy, int64_t ldg, const float* y_fwd,
                                          int64_t ld_yfwd, int64_t dim, const float* p, float* ds,
                                          float* ds_t, const uint32_t* inv_perm,
                                          float* dz, int64_t lddz, int64_t dz_row0,
                                          int64_t win_begin, int64_t win_end, int32_t flags, void* stream) {
  TCG_REQUIRE((flags & ~TCG_AGNN_Z_TF32) == 0, "tcg_agnn_backward_fused_ex: unknown flags 0x%x", flags);
  TCG_REQUIRE(t != nullptr && dim >= 1 && ldz >= dim && ldg >= dim && lddz >= dim &&
                  ld_yfwd >= dim,
              "tcg_agnn_backward_fused: bad arguments");
  TCG_REQUIRE(t->blk_h == 16 && t->blk_w == 8,
              "tf32 mode requires the 16x8 tile shape, got %dx%d", t->blk_h, t->blk_w);
  TCG_REQUIRE(0 <= win_begin && win_begin <= win_end && win_end <= t->num_windows,
              "tcg_agnn_backward_fused: window range outside [0, %lld)",
              (long long)t->num_windows);
  TCG_REQUIRE(row0_ok(t, win_begin, win_end, dz_row0),
              "tcg_agnn_backward_fused: dz_row0 %lld beyond first output row",
              (long long)dz_row0);
  static const bool no_stream = std::getenv("TCG_NO_STREAM") != nullptr;
  if (!no_stream && dim <= 32 && dim % 4 == 0 && t->num_edges > 0 && win_begin < win_end) {
    TCG_REQUIRE(z && gy && y_fwd && p && ds && dz, "tcg_agnn_backward_fused: null pointer");
    const int rc = stream_agnn(t, true, (int)dim, z, ldz, gy, ldg, y_fwd, ld_yfwd, p, ds, dz, lddz, dz_row0,
                               win_begin, win_end, as_stream(stream), nullptr, nullptr, 0,
                               (flags & TCG_AGNN_Z_TF32) != 0);
    if (rc != TCG_E_UNSUPPORTED) {
      if (rc != TCG_OK || !ds_t || !inv_perm) return rc;
      return tcg_scatter_f32(ds, inv_perm, ds_t, t->num_edges, stream);
    }
  }
  const int rc = tcg_agnn_backward(t, z, ldz, gy, ldg, dim, p, ds, dz, lddz, dz_row0, win_begin,
                                   win_end, stream);
  if (rc != TCG_OK || !ds_t || !inv_perm || t->num_edges == 0) return rc;
  return tcg_scatter_f32(ds, inv_perm, ds_t, t->num_edges, stream);
}

extern "C" int tcg_agnn_backward(const tcg_tiling* t, const float* z, int64_t ldz,
                                 const float* gy, int64_t ldg, int64_t dim, const float* p,
                                 float* ds, float* dz, int64_t lddz, int64_t dz_row0,
                                 int64_t win_begin, int64_t win_end, void* stream) {
  TCG_REQUIRE(t != nullptr && dim >= 1 && ldz >= dim && ldg >= dim && lddz >= dim,
              "tcg_agnn_backward: bad arguments");
  TCG_REQUIRE(t->blk_h == 16 && t->blk_w == 8,
              "tf32 mode requires the 16x8 tile shape, got %dx%d", t->blk_h, t->blk_w);
  TCG_REQUIRE(0 <= win_begin && win_begin <= win_end && win_end <= t->num_windows,
              "tcg_agnn_backward: window range outside [0, %lld)", (long long)t->num_windows);
  TCG_REQUIRE(row0_ok(t, win_begin, win_end, dz_row0),
              "tcg_agnn_backward: dz_row0 %lld beyond first output row", (long long)dz_row0);
  const int nt = win::nt_for(dim);
  if (t->num_edges == 0 || dim > 64 || !fits_fused(t, nt) || wide_two_step(t, dim)) {
    if (t->num_edges) {
      int rc = tcg_sddmm(t, gy, ldg, z, ldz, dim, p, ds, win_begin, win_end, TCG_PREC_TF32,
                         TCG_EPI_SOFTMAX_BWD, stream);
      if (rc != TCG_OK) return rc;
    }
    return tcg_spmm(t, z, ldz, dim, t->num_edges ? ds : nullptr, nullptr, nullptr, 0, nullptr,
                    nullptr, nullptr, dz, lddz, dz_row0, win_begin, win_end, TCG_PREC_TF32, 0,
                    stream);
  }
  if (win_begin == win_end) return TCG_OK;
  TCG_REQUIRE(z && gy && p && ds && dz, "tcg_agnn_backward: null pointer");
  win::Params q = base_params(t, win_begin, win_end);
  q.dim = (int)dim;
  q.vec16 = dim % 4 == 0 && ldz % 4 == 0 && ldg % 4 == 0 && aligned16(z) && aligned16(gy);
  q.vec_out = lddz % 4 == 0 && aligned16(dz);
  q.x = z, q.ldx = ldz, q.xa = gy, q.lda = ldg;
  q.aux = p, q.eout = ds, q.y = dz, q.ldy = lddz, q.y_row0 = dz_row0;
  return win::launch(win::MODE_AGNN_BWD, nt, q, as_stream(stream));
}

extern "C" int tcg_edge_frag(const tcg_tiling* t, uint32_t* edge_frag, void* stream) {
  TCG_REQUIRE(t != nullptr, "tcg_edge_frag: null tiling");
  TCG_REQUIRE(t->blk_h == 16 && t->blk_w == 8,
              "tf32 mode requires the 16x8 tile shape, got %dx%d", t->blk_h, t->blk_w);
  if (t->num_edges == 0) return TCG_OK;
  TCG_REQUIRE(t->node_ptr && t->edge_to_col && edge_frag, "tcg_edge_frag: null pointer");
  return win::edge_frag(t->node_ptr, t->edge_to_col, t->num_nodes, edge_frag, as_stream(stream));
}

// SURVEY.md Appendix D form of the fused AGNN forward: whole graph, dense Z.
extern "C" int tcg_agnn_fused_fwd(const tcg_tiling* t, const float* z, int64_t dim, float* p,
                                  float* y, int64_t ldy, void* stream) {
  TCG_REQUIRE(t != nullptr, "tcg_agnn_fused_fwd: null tiling");
  return tcg_agnn_forward(t, z, dim, dim, p, y, ldy, 0, 0, t->num_windows, stream);
}
