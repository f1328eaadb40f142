// Graph normalisation, invariant checks and tile accounting on the device —
// the steps either side of the hot path:
//
//  * tcg_from_edges: reference CsrGraph.from_edges (graph.py:55-89): sort the
//    (src, dst) pairs by (row, column) — one stable LSD radix sort of the
//    packed key (src << 32 | dst), so equal pairs keep their input order as
//    np.lexsort does — collapse duplicates, sum duplicate values in input
//    order in float64 (np.add.at order) and build the row pointer.
//    Bit-exact with the reference for ids in [0, 2^32).
//  * tcg_validate: the counts and first offending positions behind the
//    reference validate() messages (graph.py:92-142); the host formats them.
//  * tcg_structure_blocks: reference structure_blocks_before (sgt.py:199-217)
//    = count_blocks_before (sgt.py:140-157) on the condensed columns: per
//    window, the number of distinct col_to_node // tile_width buckets (the
//    window's condensed columns are sorted, so a bucket starts wherever the
//    bucket id changes).
#include <algorithm>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace tcg {
namespace {

__global__ void pack_keys(const int64_t* __restrict__ src, const int64_t* __restrict__ dst,
                          int64_t m, int64_t n, uint64_t* __restrict__ keys,
                          int64_t* __restrict__ idx, unsigned long long* __restrict__ bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int64_t s = src[i], d = dst[i];
  if (s < 0 || s >= n || d < 0 || d > 0xffffffffLL) {
    atomicAdd(bad, 1ull);
    keys[i] = ~0ull;
  } else {
    keys[i] = ((uint64_t)s << 32) | (uint64_t)d;
  }
  idx[i] = i;
}

__global__ void mark_heads(const uint64_t* __restrict__ keys, int64_t m, int32_t* __restrict__ head) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// one thread per run head: the surviving edge and its (float64, in-order) value sum
__global__ void emit_edges(const uint64_t* __restrict__ keys, const int64_t* __restrict__ idx,
                           const int32_t* __restrict__ head, const int64_t* __restrict__ pos,
                           int64_t m, const float* __restrict__ values,
                           uint32_t* __restrict__ cols, float* __restrict__ vals_out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m || !head[i]) return;
  const int64_t k = pos[i];
  cols[k] = (uint32_t)(keys[i] & 0xffffffffull);
  if (values) {
    double acc = 0.0;
    int64_t j = i;
    do {
      acc += (double)values[idx[j]];
      ++j;
    } while (j < m && !head[j]);
    vals_out[k] = (float)acc;
  }
}

// node_ptr[r] = first surviving edge of a row >= r (rows without edges repeat)
__global__ void fill_ptr(const uint64_t* __restrict__ keys, const int32_t* __restrict__ head,
                         const int64_t* __restrict__ pos, int64_t m, int64_t n,
                         int64_t* __restrict__ ptr) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > m) return;
  if (i < m && !head[i]) return;
  // row of this head (or n at the end) and of the previous surviving edge
  const int64_t r = i < m ? (int64_t)(keys[i] >> 32) : n;
  int64_t rp = -1;
  if (i > 0) rp = (int64_t)(keys[i - 1] >> 32);
  const int64_t k = i < m ? pos[i] : (m ? pos[m - 1] + head[m - 1] : 0);
  for (int64_t q = rp + 1; q <= r && q <= n; ++q) ptr[q] = k;
  if (i == m && r == n) ptr[n] = k;
}

struct Report {
  unsigned long long first_nonmono, n_nonmono, first_oob, n_oob, first_unsorted, n_unsorted;
};

__global__ void validate_rows(const int64_t* __restrict__ ptr, const uint32_t* __restrict__ cols,
                              int64_t n, int64_t m, Report* __restrict__ rep) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int64_t s = ptr[r], e = ptr[r + 1];
  if (e < s) {
    atomicMin(&rep->first_nonmono, (unsigned long long)r);
    atomicAdd(&rep->n_nonmono, 1ull);
  }
}

__global__ void validate_edges(const int64_t* __restrict__ ptr, const uint32_t* __restrict__ cols,
                               int64_t n, int64_t m, Report* __restrict__ rep) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int64_t s = ptr[r], e = ptr[r + 1];
  unsigned long long uns = 0, f_uns = ~0ull;
  for (int64_t q = max(s, (int64_t)0) + 1; q < min(e, m); ++q) {
    if (cols[q] <= cols[q - 1]) {
      if (!uns) f_uns = (unsigned long long)q;
      ++uns;
    }
  }
  if (uns) {
    atomicMin(&rep->first_unsorted, f_uns);
    atomicAdd(&rep->n_unsorted, uns);
  }
}

// column ids out of range, over every stored edge (graph.py:117-123)
__global__ void validate_oob(const uint32_t* __restrict__ cols, int64_t n, int64_t m,
                             Report* __restrict__ rep) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= m) return;
  if ((int64_t)cols[q] >= n) {
    atomicMin(&rep->first_oob, (unsigned long long)q);
    atomicAdd(&rep->n_oob, 1ull);
  }
}

__global__ void init_report(Report* rep) {
  rep->first_nonmono = rep->first_oob = rep->first_unsorted = ~0ull;
  rep->n_nonmono = rep->n_oob = rep->n_unsorted = 0;
}

// one warp per window; per-window distinct buckets, total in fixed order later
__global__ void structure_blocks(const int64_t* __restrict__ coff, const uint32_t* __restrict__ c2n,
                                 int64_t W, int64_t tw, int64_t* __restrict__ per_window) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= W) return;
  const int64_t c0 = coff[w], c1 = coff[w + 1];
  int64_t cnt = 0;
  for (int64_t c = c0 + lane; c < c1; c += 32) {
    const uint64_t b = c2n[c] / (uint64_t)tw;
    cnt += (c == c0 || c2n[c - 1] / (uint64_t)tw != b) ? 1 : 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if (lane == 0) per_window[w] = cnt;
}

__global__ void sum_i64(const int64_t* __restrict__ v, int64_t n, int64_t* __restrict__ out) {
  __shared__ long long sh[256];
  long long s = 0;
  for (int64_t i = threadIdx.x; i < n; i += 256) s += v[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

size_t sort_temp_bytes(int64_t m) {
  size_t b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, b, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (const int64_t*)nullptr, (int64_t*)nullptr, (int)m);
  return b;
}
size_t scan_temp_bytes(int64_t m) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, (const int32_t*)nullptr, (int64_t*)nullptr, (int)m);
  return b;
}

}  // namespace
}  // namespace tcg

using namespace tcg;

extern "C" size_t tcg_from_edges_workspace_bytes(int64_t num_edges) {
  const int64_t m = num_edges > 0 ? num_edges : 1;
  return 5 * align256(m * 8) + align256(m * sizeof(int32_t)) + align256(8) +
         align256(std::max(sort_temp_bytes(m), scan_temp_bytes(m)));
}

extern "C" int tcg_from_edges(const int64_t* src, const int64_t* dst, const float* values,
                              int64_t num_edges, int64_t num_nodes, int64_t* node_ptr,
                              uint32_t* edge_list, float* edge_values, int64_t* bad_ids,
                              void* workspace, size_t workspace_bytes, void* stream) {
  TCG_REQUIRE(num_edges >= 0 && num_nodes >= 0, "tcg_from_edges: negative size");
  TCG_REQUIRE(num_nodes <= (1LL << 32), "tcg_from_edges: num_nodes exceeds the 32-bit id width");
  TCG_REQUIRE(num_edges < (1LL << 31), "tcg_from_edges: more than 2^31 - 1 edges");
  TCG_REQUIRE(node_ptr && bad_ids, "tcg_from_edges: null output");
  TCG_REQUIRE(values == nullptr || edge_values != nullptr,
              "tcg_from_edges: values given but no edge_values output");
  TCG_REQUIRE(workspace_bytes >= tcg_from_edges_workspace_bytes(num_edges),
              "tcg_from_edges: workspace too small");
  cudaStream_t s = as_stream(stream);
  const int64_t m = num_edges;
  if (m == 0) {
    TCG_CUDA(cudaMemsetAsync(node_ptr, 0, (num_nodes + 1) * sizeof(int64_t), s), "from_edges");
    TCG_CUDA(cudaMemsetAsync(bad_ids, 0, sizeof(int64_t), s), "from_edges");
    return TCG_OK;
  }
  TCG_REQUIRE(src && dst && edge_list, "tcg_from_edges: null pointer");
  char* w = static_cast<char*>(workspace);
  auto take = [&](size_t b) {
    char* p = w;
    w += align256(b);
    return p;
  };
  uint64_t* k_in = reinterpret_cast<uint64_t*>(take(m * 8));
  uint64_t* k_out = reinterpret_cast<uint64_t*>(take(m * 8));
  int64_t* i_in = reinterpret_cast<int64_t*>(take(m * 8));
  int64_t* i_out = reinterpret_cast<int64_t*>(take(m * 8));
  int32_t* head = reinterpret_cast<int32_t*>(take(m * 4));
  int64_t* pos = reinterpret_cast<int64_t*>(take(m * 8));
  unsigned long long* bad = reinterpret_cast<unsigned long long*>(take(8));
  void* tmp = take(0);
  size_t tmp_bytes = std::max(sort_temp_bytes(m), scan_temp_bytes(m));
  const unsigned blocks = (unsigned)((m + 255) / 256);
  TCG_CUDA(cudaMemsetAsync(bad, 0, 8, s), "from_edges");
  pack_keys<<<blocks, 256, 0, s>>>(src, dst, m, num_nodes, k_in, i_in, bad);
  TCG_LAUNCHED("pack_keys");
  // bits: 32 column bits + enough row bits (invalid keys are all-ones)
  int row_bits = 1;
  while (row_bits < 32 && (1LL << row_bits) < num_nodes) ++row_bits;
  TCG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k_in, k_out, i_in, i_out, (int)m, 0,
                                           32 + row_bits, s),
           "from_edges sort");
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  mark_heads<<<blocks, 256, 0, s>>>(k_out, m, head);
  TCG_LAUNCHED("mark_heads");
  TCG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, head, pos, (int)m, s), "from_edges scan");
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  emit_edges<<<blocks, 256, 0, s>>>(k_out, i_out, head, pos, m, values, edge_list, edge_values);
  TCG_LAUNCHED("emit_edges");
  fill_ptr<<<(unsigned)((m + 1 + 255) / 256), 256, 0, s>>>(k_out, head, pos, m, num_nodes,
                                                            node_ptr);
  TCG_LAUNCHED("fill_ptr");
  TCG_CUDA(cudaMemcpyAsync(bad_ids, bad, 8, cudaMemcpyDeviceToDevice, s), "from_edges");
  return TCG_OK;
}

extern "C" int tcg_validate(const int64_t* node_ptr, const uint32_t* edge_list, int64_t num_nodes,
                            int64_t num_edges, int64_t* report, void* workspace,
                            size_t workspace_bytes, void* stream) {
  TCG_REQUIRE(num_nodes >= 0 && num_edges >= 0, "tcg_validate: negative size");
  TCG_REQUIRE(node_ptr && report, "tcg_validate: null pointer");
  TCG_REQUIRE(workspace_bytes >= sizeof(Report), "tcg_validate: workspace too small");
  cudaStream_t s = as_stream(stream);
  Report* rep = static_cast<Report*>(workspace);
  init_report<<<1, 1, 0, s>>>(rep);
  TCG_LAUNCHED("validate_init");
  if (num_nodes > 0) {
    const unsigned blocks = (unsigned)((num_nodes + 255) / 256);
    validate_rows<<<blocks, 256, 0, s>>>(node_ptr, edge_list, num_nodes, num_edges, rep);
    TCG_LAUNCHED("validate_rows");
    if (num_edges > 0 && edge_list) {
      validate_edges<<<blocks, 256, 0, s>>>(node_ptr, edge_list, num_nodes, num_edges, rep);
      TCG_LAUNCHED("validate_edges");
    }
  }
  if (num_edges > 0 && edge_list) {
    validate_oob<<<(unsigned)((num_edges + 255) / 256), 256, 0, s>>>(edge_list, num_nodes,
                                                                      num_edges, rep);
    TCG_LAUNCHED("validate_oob");
  }
  TCG_CUDA(cudaMemcpyAsync(report, rep, sizeof(Report), cudaMemcpyDeviceToDevice, s),
           "tcg_validate");
  return TCG_OK;
}

extern "C" int tcg_structure_blocks(const tcg_tiling* t, int64_t tile_width, int64_t* per_window,
                                    int64_t* total, void* stream) {
  TCG_REQUIRE(t != nullptr, "tcg_structure_blocks: null tiling");
  TCG_REQUIRE(tile_width >= 1, "tile_width must be >= 1");
  TCG_REQUIRE(per_window && total, "tcg_structure_blocks: null output");
  cudaStream_t s = as_stream(stream);
  const int64_t W = t->num_windows;
  if (W == 0) {
    TCG_CUDA(cudaMemsetAsync(total, 0, sizeof(int64_t), s), "structure_blocks");
    return TCG_OK;
  }
  TCG_REQUIRE(t->col_offsets && (t->num_unique == 0 || t->col_to_node),
              "tcg_structure_blocks: tiling arrays missing");
  structure_blocks<<<(unsigned)((W * 32 + 255) / 256), 256, 0, s>>>(
      t->col_offsets, t->col_to_node, W, tile_width, per_window);
  TCG_LAUNCHED("structure_blocks");
  sum_i64<<<1, 256, 0, s>>>(per_window, W, total);
  TCG_LAUNCHED("sum_i64");
  return TCG_OK;
}
