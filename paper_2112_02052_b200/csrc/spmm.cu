#include <cstdlib>
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
//  * TCG_PREC_TF32: the tensor-core row-window engine (window.cu, modes SPMM
//    and SPMM_DUAL).
#include <algorithm>

#include "common.cuh"
#include "window.cuh"

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

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace
}  // namespace tcg

using namespace tcg;

namespace tcg {
// ReLU over output rows [r0, r1) (absolute; stored at y[r - y_row0]), for the
// engines that do not fuse it
__global__ void spmm_relu_rows(float* __restrict__ y, int64_t ldy, int64_t r0, int64_t r1, int64_t y_row0, int dim) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t rows = r1 - r0;
  if (i >= rows * dim) return;
  const int64_t r = r0 + i / dim;
  float* p = y + (r - y_row0) * ldy + i % dim;
  *p = fmaxf(*p, 0.f);
}
}  // namespace tcg

static int spmm_run(const tcg_tiling* t, const float* x, int64_t ldx, int64_t dim, const float* weights,
                    const uint32_t* weight_idx, const float* x2, int64_t ldx2, const float* weights2,
                    const uint32_t* weight_idx2, const float* bias, float* y, int64_t ldy, int64_t y_row0,
                    int64_t win_begin, int64_t win_end, int32_t precision, int32_t accumulate, int relu,
                    bool* fused, void* stream);

extern "C" int tcg_spmm(const tcg_tiling* t, const float* x, int64_t ldx, int64_t dim,
                        const float* weights, const uint32_t* weight_idx, const float* x2,
                        int64_t ldx2, const float* weights2, const uint32_t* weight_idx2,
                        const float* bias, float* y, int64_t ldy, int64_t y_row0,
                        int64_t win_begin, int64_t win_end, int32_t precision, int32_t accumulate,
                        void* stream) {
  bool fused = false;
  return spmm_run(t, x, ldx, dim, weights, weight_idx, x2, ldx2, weights2, weight_idx2, bias, y, ldy, y_row0,
                  win_begin, win_end, precision, accumulate, 0, &fused, stream);
}

extern "C" int tcg_spmm_act(const tcg_tiling* t, const float* x, int64_t ldx, int64_t dim,
                            const float* weights, const uint32_t* weight_idx, const float* bias, float* y,
                            int64_t ldy, int64_t y_row0, int64_t win_begin, int64_t win_end,
                            int32_t precision, int32_t accumulate, int32_t act, void* stream) {
  TCG_REQUIRE(act == TCG_ACT_NONE || act == TCG_ACT_RELU, "tcg_spmm_act: unknown activation %d", act);
  bool fused = false;
  const int rc = spmm_run(t, x, ldx, dim, weights, weight_idx, nullptr, 0, nullptr, nullptr, bias, y, ldy,
                          y_row0, win_begin, win_end, precision, accumulate, act == TCG_ACT_RELU, &fused, stream);
  if (rc != TCG_OK || act != TCG_ACT_RELU || fused || win_begin == win_end || t->num_nodes == 0) return rc;
  const int64_t r0 = win_begin * t->blk_h, r1 = std::min<int64_t>(win_end * (int64_t)t->blk_h, t->num_nodes);
  if (r1 <= r0) return TCG_OK;
  const int64_t total = (r1 - r0) * dim;
  tcg::spmm_relu_rows<<<(unsigned)((total + 255) / 256), 256, 0, as_stream(stream)>>>(y, ldy, r0, r1, y_row0,
                                                                                   (int)dim);
  TCG_LAUNCHED("relu_rows");
  return TCG_OK;
}

static int spmm_run(const tcg_tiling* t, const float* x, int64_t ldx, int64_t dim, const float* weights,
                    const uint32_t* weight_idx, const float* x2, int64_t ldx2, const float* weights2,
                    const uint32_t* weight_idx2, const float* bias, float* y, int64_t ldy, int64_t y_row0,
                    int64_t win_begin, int64_t win_end, int32_t precision, int32_t accumulate, int relu,
                    bool* fused, void* stream) {
  TCG_REQUIRE(t != nullptr, "tcg_spmm: null tiling");
  TCG_REQUIRE(dim >= 1, "tcg_spmm: embedding dimension must be >= 1, got %lld", (long long)dim);
  TCG_REQUIRE(ldx >= dim && ldy >= dim, "tcg_spmm: leading dimension < dim");
  TCG_REQUIRE(x2 == nullptr || ldx2 >= dim, "tcg_spmm: ldx2 < dim");
  TCG_REQUIRE(0 <= win_begin && win_begin <= win_end && win_end <= t->num_windows,
              "tcg_spmm: window range [%lld, %lld) outside [0, %lld)", (long long)win_begin,
              (long long)win_end, (long long)t->num_windows);
  // TCG_PREC_X2_TF32 (tf32 only): x2 is already on the tf32 grid, its B-operand
  // rounding is skipped (same result)
  const int x2_tf32 = (precision & TCG_PREC_X2_TF32) != 0;
  precision &= ~TCG_PREC_X2_TF32;
  TCG_REQUIRE(precision == TCG_PREC_F32 || precision == TCG_PREC_TF32,
              "tcg_spmm: unknown precision %d", precision);
  TCG_REQUIRE(!x2_tf32 || precision == TCG_PREC_TF32, "tcg_spmm: TCG_PREC_X2_TF32 needs TCG_PREC_TF32");
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
  // output row r lands at y[r - y_row0]: valid when 0 <= y_row0 <= first row
  TCG_REQUIRE((a.y_row0 >= 0 && a.y_row0 <= a.row_begin) || a.row_begin >= a.row_end,
              "tcg_spmm: y_row0 %lld beyond first output row %lld", (long long)a.y_row0,
              (long long)a.row_begin);

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
  TCG_REQUIRE(t->num_edges == 0 || t->edge_frag, "tcg_spmm: tf32 needs edge_frag (tcg_edge_frag)");
  win::Params q{};
  q.ptr = t->node_ptr;
  q.e2c = t->edge_to_col;
  q.efrag = t->edge_frag;
  q.coff = t->col_offsets;
  q.c2n = t->col_to_node;
  q.n = t->num_nodes;
  q.win_begin = win_begin;
  q.nwin = win_end - win_begin;
  const int nt = win::nt_for(dim);
  q.nchunks = dim <= 64 ? 1 : (int)((dim + 63) / 64);
  q.nkc = 1;
  q.dim = (int)dim;
  q.vec16 = dim % 4 == 0 && ldx % 4 == 0 && aligned16(x) &&
            (x2 == nullptr || (ldx2 % 4 == 0 && aligned16(x2)));
  q.vec_out = ldy % 4 == 0 && aligned16(y) && (bias == nullptr || aligned16(bias));
  q.x = x, q.ldx = ldx, q.x2 = x2, q.ldx2 = ldx2;
  q.w = weights, q.widx = weight_idx, q.w2 = weights2, q.widx2 = weight_idx2;
  q.bias = bias, q.y = y, q.ldy = ldy, q.y_row0 = y_row0, q.accumulate = accumulate;
  q.relu = relu;
  q.x2_tf32 = x2 ? x2_tf32 : 0;
  static const bool no_stream = std::getenv("TCG_NO_STREAM") != nullptr;
  if (!no_stream) {
    const int rc = stream_spmm(t, q, s);
    if (rc != TCG_E_UNSUPPORTED) {
      *fused = relu != 0;
      return rc;
    }
  }
  q.relu = 0;
  return win::launch(x2 ? win::MODE_SPMM_DUAL : win::MODE_SPMM, nt, q, s);
}
