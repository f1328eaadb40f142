// Direct CSR evaluation without tiling: the reference's oracle API
// (tcgraph.oracle.ref_spmm / ref_sddmm, oracle.py:28-91) on the GPU.
//
//  * tcg_csr_spmm: out[i] = sum over the row's edges, in CSR order, of
//    f[e] * x[col e]. f32 mode rounds each product and each add (no FMA),
//    starting from +0.0 -- the reference fold (oracle.py:54-59); f64 mode
//    widens the term to double before the add (accumulate="f64").
//  * tcg_csr_sddmm: F[e] = <x[row e], x[col e]>, k ascending; f32 mode is the
//    cumsum left fold of oracle.py:86-90, f64 sums in double.
// One warp per row (SpMM, features across lanes) / one thread per edge
// (SDDMM); these are checkers and API parity, not the hot path.
#include "common.cuh"

namespace tcg {
namespace {

template <bool F64>
__global__ void __launch_bounds__(256) csr_spmm_kernel(const int64_t* __restrict__ ptr,
                                                       const uint32_t* __restrict__ cols,
                                                       const float* __restrict__ f, int64_t n,
                                                       const float* __restrict__ x, int64_t ldx,
                                                       int64_t dim, void* __restrict__ out,
                                                       int64_t ldo) {
  const int lane = threadIdx.x & 31;
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= n) return;
  const int64_t e0 = __ldg(ptr + row), e1 = __ldg(ptr + row + 1);
  for (int64_t k = lane; k < dim; k += 32) {
    if constexpr (F64) {
      double acc = 0.0;
      for (int64_t e = e0; e < e1; ++e) {
        const float v = __ldg(x + (int64_t)__ldg(cols + e) * ldx + k);
        acc += (double)(f ? __fmul_rn(__ldg(f + e), v) : v);
      }
      reinterpret_cast<double*>(out)[row * ldo + k] = acc;
    } else {
      float acc = 0.f;
      for (int64_t e = e0; e < e1; ++e) {
        const float v = __ldg(x + (int64_t)__ldg(cols + e) * ldx + k);
        acc = __fadd_rn(acc, f ? __fmul_rn(__ldg(f + e), v) : v);
      }
      reinterpret_cast<float*>(out)[row * ldo + k] = acc;
    }
  }
}

__global__ void edge_rows_kernel(const int64_t* __restrict__ ptr, int64_t n,
                                 uint32_t* __restrict__ rows) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e) rows[e] = (uint32_t)r;
}

template <bool F64>
__global__ void __launch_bounds__(256) csr_sddmm_kernel(const uint32_t* __restrict__ rows,
                                                        const uint32_t* __restrict__ cols,
                                                        int64_t m, const float* __restrict__ x,
                                                        int64_t ldx, int64_t dim,
                                                        void* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m) return;
  const float* a = x + (int64_t)__ldg(rows + e) * ldx;
  const float* b = x + (int64_t)__ldg(cols + e) * ldx;
  if constexpr (F64) {
    double acc = 0.0;
    for (int64_t k = 0; k < dim; ++k) acc += (double)__fmul_rn(__ldg(a + k), __ldg(b + k));
    reinterpret_cast<double*>(out)[e] = acc;
  } else {
    float acc = 0.f;
    for (int64_t k = 0; k < dim; ++k) acc = __fadd_rn(acc, __fmul_rn(__ldg(a + k), __ldg(b + k)));
    reinterpret_cast<float*>(out)[e] = acc;
  }
}

}  // namespace
}  // namespace tcg

using tcg::as_stream;

extern "C" int tcg_csr_spmm(const int64_t* node_ptr, const uint32_t* edge_list,
                            const float* values, int64_t num_nodes, const float* x, int64_t ldx,
                            int64_t dim, void* out, int64_t ldo, int32_t acc_f64, void* stream) {
  TCG_REQUIRE(num_nodes >= 0 && dim >= 1 && ldx >= dim && ldo >= dim,
              "tcg_csr_spmm: bad sizes (n=%lld, dim=%lld)", (long long)num_nodes,
              (long long)dim);
  if (num_nodes == 0) return TCG_OK;
  TCG_REQUIRE(node_ptr && x && out, "tcg_csr_spmm: null pointer");
  const unsigned blocks = (unsigned)((num_nodes * 32 + 255) / 256);
  if (acc_f64)
    tcg::csr_spmm_kernel<true><<<blocks, 256, 0, as_stream(stream)>>>(
        node_ptr, edge_list, values, num_nodes, x, ldx, dim, out, ldo);
  else
    tcg::csr_spmm_kernel<false><<<blocks, 256, 0, as_stream(stream)>>>(
        node_ptr, edge_list, values, num_nodes, x, ldx, dim, out, ldo);
  TCG_LAUNCHED("csr_spmm");
  return TCG_OK;
}

extern "C" int tcg_csr_sddmm(const int64_t* node_ptr, const uint32_t* edge_list,
                             int64_t num_nodes, int64_t num_edges, const float* x, int64_t ldx,
                             int64_t dim, uint32_t* row_ws, void* out, int32_t acc_f64,
                             void* stream) {
  TCG_REQUIRE(num_nodes >= 0 && num_edges >= 0 && dim >= 1 && ldx >= dim,
              "tcg_csr_sddmm: bad sizes");
  if (num_edges == 0) return TCG_OK;
  TCG_REQUIRE(node_ptr && edge_list && x && row_ws && out, "tcg_csr_sddmm: null pointer");
  tcg::edge_rows_kernel<<<(unsigned)((num_nodes + 255) / 256), 256, 0, as_stream(stream)>>>(
      node_ptr, num_nodes, row_ws);
  TCG_LAUNCHED("edge_rows");
  const unsigned blocks = (unsigned)((num_edges + 255) / 256);
  if (acc_f64)
    tcg::csr_sddmm_kernel<true><<<blocks, 256, 0, as_stream(stream)>>>(row_ws, edge_list,
                                                                        num_edges, x, ldx, dim, out);
  else
    tcg::csr_sddmm_kernel<false><<<blocks, 256, 0, as_stream(stream)>>>(row_ws, edge_list,
                                                                         num_edges, x, ldx, dim, out);
  TCG_LAUNCHED("csr_sddmm");
  return TCG_OK;
}
