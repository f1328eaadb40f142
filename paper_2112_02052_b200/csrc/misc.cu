// Library plumbing and small kernels of the C ABI:
//  * error text / launch counter / device info;
//  * segment softmax forward (reference kernels.segment_softmax,
//    kernels.py:541-556) and its backward (no reference counterpart);
//  * TF32 operand rounding (reference tiles.quantize_tf32, tiles.py:67-82);
//  * CSR transpose with the edge permutation (backward support);
#include <cstdlib>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <string>

#include "common.cuh"

namespace tcg {

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

std::atomic<int64_t>& launch_counter() {
  static std::atomic<int64_t> c{0};
  return c;
}

namespace {

// One warp per row (rows are short: avg degree 7 on the BASELINE shapes).
__global__ void softmax_fwd(const int64_t* __restrict__ ptr, int64_t n, const float* __restrict__ v,
                            float* __restrict__ out) {
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  const int64_t s = ptr[r], e = ptr[r + 1];
  if (s == e) return;
  float m = -INFINITY;
  for (int64_t i = s + lane; i < e; i += 32) m = fmaxf(m, v[i]);
  m = warp_max(m);
  float sum = 0.f;
  for (int64_t i = s + lane; i < e; i += 32) sum += expf(v[i] - m);
  sum = warp_sum(sum);
  for (int64_t i = s + lane; i < e; i += 32) out[i] = expf(v[i] - m) / sum;
}

__global__ void softmax_bwd(const int64_t* __restrict__ ptr, int64_t n, const float* __restrict__ p,
                            const float* __restrict__ dp, float* __restrict__ ds) {
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  const int64_t s = ptr[r], e = ptr[r + 1];
  float dot = 0.f;
  for (int64_t i = s + lane; i < e; i += 32) dot += p[i] * dp[i];
  dot = warp_sum(dot);
  for (int64_t i = s + lane; i < e; i += 32) ds[i] = p[i] * (dp[i] - dot);
}

// Same bits as the reference quantizer: cvt.rn.tf32.f32 (the instruction the
// tensor-core kernels use) for finite values, NaN payloads passed through.
__global__ void quantize(const float* __restrict__ in, float* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float x = in[i];
    const uint32_t u = __float_as_uint(x);
    out[i] = ((u & 0x7f800000u) == 0x7f800000u) ? x : __uint_as_float(tf32_rn(x));
  }
}

__global__ void csr_rows(const int64_t* __restrict__ ptr, int64_t n, uint32_t* __restrict__ row_of,
                         uint32_t* __restrict__ iota, unsigned long long* __restrict__ counts,
                         const uint32_t* __restrict__ cols) {
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  for (int64_t e = ptr[r] + lane; e < ptr[r + 1]; e += 32) {
    row_of[e] = (uint32_t)r;
    iota[e] = (uint32_t)e;
    atomicAdd(counts + cols[e], 1ull);
  }
}

__global__ void gather_rows(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ row_of,
                            uint32_t* __restrict__ cols_t, int64_t m) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m;
       k += (int64_t)gridDim.x * blockDim.x)
    cols_t[k] = row_of[perm[k]];
}

struct TrWs {
  size_t counts, row_of, iota, keys, cub_tmp, cub_bytes, total;
};

TrWs tr_layout(int64_t n, int64_t m) {
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  TrWs L{};
  size_t off = 0;
  L.counts = off;
  off += al(sizeof(int64_t) * (n + 1));
  L.row_of = off;
  off += al(sizeof(uint32_t) * (m + 1));
  L.iota = off;
  off += al(sizeof(uint32_t) * (m + 1));
  L.keys = off;
  off += al(sizeof(uint32_t) * (m + 1));
  size_t scan_b = 0, sort_b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_b, (int64_t*)nullptr, (int64_t*)nullptr,
                                (int)(n + 1));
  cub::DeviceRadixSort::SortPairs(nullptr, sort_b, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (uint32_t*)nullptr, (int)(m > 0 ? m : 1));
  L.cub_bytes = scan_b > sort_b ? scan_b : sort_b;
  L.cub_tmp = off;
  off += al(L.cub_bytes);
  L.total = off;
  return L;
}

}  // namespace

int num_sms() {
  int dev = 0, v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
  return v;
}

}  // namespace tcg

using namespace tcg;

extern "C" const char* tcg_last_error(void) { return g_last_error.c_str(); }

extern "C" const char* tcg_version(void) { return "tcg_b200 0.1.0 (sm_100a)"; }

extern "C" int64_t tcg_launch_count(void) { return launch_counter().load(); }

namespace tcg {
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TCG_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
}  // namespace tcg

extern "C" int tcg_device_info(int64_t* num_sms_out, int64_t* l2_bytes) {
  int dev = 0, sms = 0, l2 = 0;
  TCG_CUDA(cudaGetDevice(&dev), "tcg_device_info");
  TCG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "tcg_device_info");
  TCG_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev), "tcg_device_info");
  if (num_sms_out) *num_sms_out = sms;
  if (l2_bytes) *l2_bytes = l2;
  return TCG_OK;
}

extern "C" int tcg_segment_softmax(const int64_t* node_ptr, int64_t num_rows, const float* values,
                                   float* out, void* stream) {
  TCG_REQUIRE(num_rows >= 0, "tcg_segment_softmax: negative rows");
  if (num_rows == 0) return TCG_OK;
  TCG_REQUIRE(node_ptr && values && out, "tcg_segment_softmax: null pointer");
  const int tpb = 256;
  const unsigned blocks = (unsigned)((num_rows * 32 + tpb - 1) / tpb);
  softmax_fwd<<<blocks, tpb, 0, as_stream(stream)>>>(node_ptr, num_rows, values, out);
  TCG_LAUNCHED("softmax_fwd");
  return TCG_OK;
}

extern "C" int tcg_segment_softmax_backward(const int64_t* node_ptr, int64_t num_rows,
                                            const float* p, const float* dp, float* ds,
                                            void* stream) {
  TCG_REQUIRE(num_rows >= 0, "tcg_segment_softmax_backward: negative rows");
  if (num_rows == 0) return TCG_OK;
  TCG_REQUIRE(node_ptr && p && dp && ds, "tcg_segment_softmax_backward: null pointer");
  const int tpb = 256;
  const unsigned blocks = (unsigned)((num_rows * 32 + tpb - 1) / tpb);
  softmax_bwd<<<blocks, tpb, 0, as_stream(stream)>>>(node_ptr, num_rows, p, dp, ds);
  TCG_LAUNCHED("softmax_bwd");
  return TCG_OK;
}

extern "C" int tcg_quantize_tf32(const float* in, float* out, int64_t n, void* stream) {
  TCG_REQUIRE(n >= 0, "tcg_quantize_tf32: negative size");
  if (n == 0) return TCG_OK;
  TCG_REQUIRE(in && out, "tcg_quantize_tf32: null pointer");
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  quantize<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(in, out, n);
  TCG_LAUNCHED("quantize_tf32");
  return TCG_OK;
}

namespace tcg {
namespace {
__global__ void permute_f32(const float* __restrict__ src, const uint32_t* __restrict__ idx,
                            float* __restrict__ dst, int64_t n) {
  TCG_PDL_ENTRY();
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    dst[k] = __ldg(src + __ldg(idx + k));
}

// two arrays through the same permutation (P and dS of the AGNN backward):
// four indices per thread (one 16-B load) so eight random 4-B gathers are in
// flight per thread; the scalar tail handles n % 4 and unaligned bases
__global__ void permute2_f32(const float* __restrict__ a, const float* __restrict__ b,
                             const uint32_t* __restrict__ idx, float* __restrict__ da,
                             float* __restrict__ db, int64_t n) {
  TCG_PDL_ENTRY();
  const bool vec = ((reinterpret_cast<uintptr_t>(idx) | reinterpret_cast<uintptr_t>(da) |
                     reinterpret_cast<uintptr_t>(db)) & 15) == 0;
  const int64_t n4 = vec ? n / 4 : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += stride) {
    const uint4 j = __ldg(reinterpret_cast<const uint4*>(idx) + q);
    const float4 va = make_float4(__ldg(a + j.x), __ldg(a + j.y), __ldg(a + j.z), __ldg(a + j.w));
    const float4 vb = make_float4(__ldg(b + j.x), __ldg(b + j.y), __ldg(b + j.z), __ldg(b + j.w));
    reinterpret_cast<float4*>(da)[q] = va;
    reinterpret_cast<float4*>(db)[q] = vb;
  }
  for (int64_t k = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
    const uint32_t j = __ldg(idx + k);
    da[k] = __ldg(a + j);
    db[k] = __ldg(b + j);
  }
}
}  // namespace
}  // namespace tcg

namespace tcg {
namespace {
// edgeToRow: row of each edge inside its row window (one thread per row)
__global__ void edge_to_row_kernel(const int64_t* __restrict__ ptr, int64_t n, int blk_h,
                                   uint32_t* __restrict__ e2r) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const uint32_t rl = (uint32_t)(r % blk_h);
  for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e) e2r[e] = rl;
}
}  // namespace
}  // namespace tcg

extern "C" int tcg_edge_to_row(const int64_t* node_ptr, int64_t num_nodes, int32_t blk_h,
                               uint32_t* edge_to_row, void* stream) {
  TCG_REQUIRE(num_nodes >= 0 && blk_h >= 1, "tcg_edge_to_row: bad arguments");
  if (num_nodes == 0) return TCG_OK;
  TCG_REQUIRE(node_ptr && edge_to_row, "tcg_edge_to_row: null pointer");
  tcg::edge_to_row_kernel<<<(unsigned)((num_nodes + 255) / 256), 256, 0, as_stream(stream)>>>(
      node_ptr, num_nodes, blk_h, edge_to_row);
  TCG_LAUNCHED("edge_to_row");
  return TCG_OK;
}

extern "C" int tcg_permute2_f32(const float* src_a, const float* src_b, const uint32_t* idx,
                                float* dst_a, float* dst_b, int64_t n, void* stream) {
  TCG_REQUIRE(n >= 0, "tcg_permute2_f32: negative size");
  if (n == 0) return TCG_OK;
  TCG_REQUIRE(src_a && src_b && idx && dst_a && dst_b, "tcg_permute2_f32: null pointer");
  int64_t blocks = (n / 4 + 255) / 256 + 1;
  if (blocks > 148 * 16) blocks = 148 * 16;
  ::tcg::launch_pdl(permute2_f32, (unsigned)blocks, 256, 0, as_stream(stream), src_a, src_b, idx, dst_a, dst_b, n);
  TCG_LAUNCHED("permute2_f32");
  return TCG_OK;
}

extern "C" int tcg_permute_f32(const float* src, const uint32_t* idx, float* dst, int64_t n,
                               void* stream) {
  TCG_REQUIRE(n >= 0, "tcg_permute_f32: negative size");
  if (n == 0) return TCG_OK;
  TCG_REQUIRE(src && idx && dst, "tcg_permute_f32: null pointer");
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  ::tcg::launch_pdl(permute_f32, (unsigned)blocks, 256, 0, as_stream(stream), src, idx, dst, n);
  TCG_LAUNCHED("permute_f32");
  return TCG_OK;
}

namespace tcg {
namespace {
__global__ void scatter_f32(const float* __restrict__ src, const uint32_t* __restrict__ idx,
                            float* __restrict__ dst, int64_t n) {
  TCG_PDL_ENTRY();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[idx[i]] = src[i];
}
}  // namespace
}  // namespace tcg

extern "C" int tcg_scatter_f32(const float* src, const uint32_t* idx, float* dst, int64_t n,
                               void* stream) {
  TCG_REQUIRE(n >= 0, "tcg_scatter_f32: negative size");
  if (n == 0) return TCG_OK;
  TCG_REQUIRE(src && idx && dst, "tcg_scatter_f32: null pointer");
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  ::tcg::launch_pdl(tcg::scatter_f32, (unsigned)blocks, 256, 0, as_stream(stream), src, idx, dst, n);
  TCG_LAUNCHED("scatter_f32");
  return TCG_OK;
}

extern "C" size_t tcg_csr_transpose_workspace_bytes(int64_t num_nodes, int64_t num_edges) {
  if (num_nodes < 0 || num_edges < 0) return 0;
  return tr_layout(num_nodes, num_edges).total;
}

extern "C" int tcg_csr_transpose(const int64_t* node_ptr, const uint32_t* edge_list,
                                 int64_t num_nodes, int64_t num_edges, int64_t* ptr_t,
                                 uint32_t* cols_t, uint32_t* perm, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  TCG_REQUIRE(num_nodes >= 0 && num_edges >= 0, "tcg_csr_transpose: negative size");
  TCG_REQUIRE(num_edges <= 0xffffffffLL, "tcg_csr_transpose: edge ids must fit u32");
  const TrWs L = tr_layout(num_nodes, num_edges);
  TCG_REQUIRE(workspace_bytes >= L.total, "tcg_csr_transpose: workspace %zu < %zu",
              workspace_bytes, L.total);
  TCG_REQUIRE(ptr_t != nullptr, "tcg_csr_transpose: null ptr_t");
  cudaStream_t s = as_stream(stream);
  char* ws = static_cast<char*>(workspace);
  int64_t* counts = reinterpret_cast<int64_t*>(ws + L.counts);
  uint32_t* row_of = reinterpret_cast<uint32_t*>(ws + L.row_of);
  uint32_t* iota = reinterpret_cast<uint32_t*>(ws + L.iota);
  uint32_t* keys = reinterpret_cast<uint32_t*>(ws + L.keys);
  TCG_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * (num_nodes + 1), s), "transpose memset");
  if (num_edges > 0) {
    TCG_REQUIRE(node_ptr && edge_list && cols_t && perm, "tcg_csr_transpose: null pointer");
    const int tpb = 256;
    csr_rows<<<(unsigned)((num_nodes * 32 + tpb - 1) / tpb), tpb, 0, s>>>(
        node_ptr, num_nodes, row_of, iota, reinterpret_cast<unsigned long long*>(counts),
        edge_list);
    TCG_LAUNCHED("csr_rows");
    int end_bit = 1;
    while (end_bit < 32 && (1LL << end_bit) < num_nodes) ++end_bit;
    size_t b = L.cub_bytes;
    // LSD radix sort is stable: equal columns keep ascending edge (= row) order
    TCG_CUDA(cub::DeviceRadixSort::SortPairs(ws + L.cub_tmp, b, edge_list, keys, iota, perm,
                                             (int)num_edges, 0, end_bit, s),
             "transpose sort");
    launch_counter().fetch_add(1, std::memory_order_relaxed);
    gather_rows<<<(unsigned)std::min<int64_t>((num_edges + 255) / 256, 148 * 32), 256, 0, s>>>(
        perm, row_of, cols_t, num_edges);
    TCG_LAUNCHED("gather_rows");
  }
  size_t b = L.cub_bytes;
  TCG_CUDA(cub::DeviceScan::ExclusiveSum(ws + L.cub_tmp, b, counts, ptr_t, (int)(num_nodes + 1), s),
           "transpose scan");
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  return TCG_OK;
}

// SURVEY.md Appendix D names of the segment-softmax pair.
extern "C" int tcg_softmax_fwd(const int64_t* node_ptr, int64_t num_rows, const float* values,
                               float* out, void* stream) {
  return tcg_segment_softmax(node_ptr, num_rows, values, out, stream);
}

extern "C" int tcg_softmax_bwd(const int64_t* node_ptr, int64_t num_rows, const float* p,
                               const float* dp, float* ds, void* stream) {
  return tcg_segment_softmax_backward(node_ptr, num_rows, p, dp, ds, stream);
}
