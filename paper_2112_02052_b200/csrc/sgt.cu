// Sparse Graph Translation on the GPU — replaces reference sgt.translate
// (/root/reference/pkg/src/tcgraph/sgt.py:101-137, Alg. 1 of the paper).
//
// Per row window w (rows [w*blk_h, min((w+1)*blk_h, N))), the window's edge
// column ids are sorted and deduplicated; an edge's condensed column
// (edge_to_col) is the rank of its column in that sorted unique set, the set
// itself is col_to_node[col_offsets[w] : col_offsets[w+1]], and
// win_partition[w] = ceil(u_w / blk_w). Ranks are order-independent, so any
// correct sort yields bit-exact reference output.
//
// Kernels (tcg_sgt = tcg_sgt_count + tcg_sgt_fill, stream-ordered):
//   sgt_rank     one CTA per window: column ids -> smem bitonic sort -> head
//                flags -> block scan -> compacted unique set; edge_to_col by
//                binary search in it, u_w. Windows with more than kSmemCap
//                edges are queued.
//   sgt_rank_big the queued windows: bitmap over the node range in global
//                scratch, rank = prefix popcount (no sort).
//   cub ExclusiveSum of u_w -> col_offsets.
//   sgt_fill     per window: col_to_node[col_offsets[w] + edge_to_col[e]] =
//                edge_list[e] (duplicates store the same value) and
//                win_partition[w] = ceil(u_w / blk_w).
#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace tcg {
namespace {

constexpr int kRankThreads = 128;
#ifndef TCG_SGT_CAP
#define TCG_SGT_CAP 4096
#endif
constexpr int kSmemCap = TCG_SGT_CAP;  // keys per window on the shared-memory path
constexpr int kBigCtas = 32;    // concurrent big-window CTAs (bitmap scratch each)
constexpr int kBigThreads = 512;

__device__ __forceinline__ uint32_t pow2_ceil(uint32_t x) {
  return x <= 1 ? 1u : 1u << (32 - __clz(x - 1));
}

__global__ void __launch_bounds__(kRankThreads)
    sgt_rank(const int64_t* __restrict__ ptr, const uint32_t* __restrict__ cols, int64_t n,
             int64_t num_windows, int bh, uint32_t* __restrict__ e2c,
             int64_t* __restrict__ ucount, int* __restrict__ big_list, int* __restrict__ big_count) {
  // 32-bit column ids are sorted (half the shared-memory traffic of sorting
  // (col, edge) pairs), compacted to the window's unique set, and every edge
  // is ranked by a binary search in it -- the reference's unique +
  // searchsorted (sgt.py:116-120)
  __shared__ uint32_t keys[kSmemCap];
  __shared__ uint32_t uniq[kSmemCap];
  __shared__ int scan_scratch[33];
  const int tid = threadIdx.x;
  for (int64_t w = blockIdx.x; w < num_windows; w += gridDim.x) {
    const int64_t r0 = w * bh;
    const int64_t r1 = min(r0 + bh, n);
    const int64_t e0 = ptr[r0], e1 = ptr[r1];
    const int64_t E = e1 - e0;
    if (E == 0) {
      if (tid == 0) ucount[w] = 0;
      continue;
    }
    if (E > kSmemCap) {
      if (tid == 0) {
        big_list[atomicAdd(big_count, 1)] = (int)w;
        ucount[w] = 0;
      }
      continue;
    }
    const uint32_t P = pow2_ceil((uint32_t)E);
    for (uint32_t i = tid; i < P; i += kRankThreads) keys[i] = i < E ? cols[e0 + i] : ~0u;
    __syncthreads();
    // bitonic sort, ascending
    for (uint32_t k = 2; k <= P; k <<= 1) {
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        for (uint32_t i = tid; i < (P >> 1); i += kRankThreads) {
          const uint32_t lo = ((i & ~(j - 1)) << 1) | (i & (j - 1));
          const uint32_t hi = lo | j;
          const uint32_t a = keys[lo], b = keys[hi];
          const bool up = (lo & k) == 0;
          if ((a > b) == up) {
            keys[lo] = b;
            keys[hi] = a;
          }
        }
        __syncthreads();
      }
    }
    // head flags over contiguous per-thread chunks, block scan -> compacted set
    const uint32_t per = (uint32_t)((E + kRankThreads - 1) / kRankThreads);
    const uint32_t beg = min((uint32_t)E, tid * per), end = min((uint32_t)E, beg + per);
    int heads = 0;
    for (uint32_t i = beg; i < end; ++i) heads += (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
    int total;
    int rank = block_excl_scan<kRankThreads>(heads, scan_scratch, &total);
    for (uint32_t i = beg; i < end; ++i)
      if (i == 0 || keys[i] != keys[i - 1]) uniq[rank++] = keys[i];
    __syncthreads();
    // rank of every edge's column in the unique set (lower bound)
    for (int64_t i = tid; i < E; i += kRankThreads) {
      const uint32_t c = cols[e0 + i];
      int lo = 0, hi = total;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (uniq[mid] < c) lo = mid + 1;
        else hi = mid;
      }
      e2c[e0 + i] = (uint32_t)lo;
    }
    if (tid == 0) ucount[w] = total;
    __syncthreads();
  }
}

// Windows with more than kSmemCap edges: mark columns in a bitmap over
// [0, N) (per-CTA scratch), prefix-popcount it, rank = popcount below col.
__global__ void __launch_bounds__(kBigThreads)
    sgt_rank_big(const int64_t* __restrict__ ptr, const uint32_t* __restrict__ cols, int64_t n,
                 int bh, const int* __restrict__ big_list, const int* __restrict__ big_count,
                 uint32_t* __restrict__ e2c, int64_t* __restrict__ ucount,
                 uint32_t* __restrict__ bitmaps, uint32_t* __restrict__ prefixes) {
  __shared__ int scan_scratch[33];
  const int nbig = *big_count;
  if (nbig == 0) return;
  const int64_t nwords = (n + 31) / 32;
  uint32_t* bm = bitmaps + (int64_t)blockIdx.x * nwords;
  uint32_t* pre = prefixes + (int64_t)blockIdx.x * nwords;
  const int tid = threadIdx.x;
  for (int b = blockIdx.x; b < nbig; b += gridDim.x) {
    const int64_t w = big_list[b];
    const int64_t r0 = w * bh, r1 = min(r0 + bh, n);
    const int64_t e0 = ptr[r0], e1 = ptr[r1];
    for (int64_t i = tid; i < nwords; i += kBigThreads) bm[i] = 0;
    __syncthreads();
    for (int64_t e = e0 + tid; e < e1; e += kBigThreads) {
      const uint32_t c = cols[e];
      atomicOr(&bm[c >> 5], 1u << (c & 31));
    }
    __syncthreads();
    int64_t carry = 0;
    for (int64_t base = 0; base < nwords; base += kBigThreads) {
      const int64_t i = base + tid;
      const int v = i < nwords ? __popc(bm[i]) : 0;
      int tot;
      const int ex = block_excl_scan<kBigThreads>(v, scan_scratch, &tot);
      if (i < nwords) pre[i] = (uint32_t)(carry + ex);
      carry += tot;
    }
    __syncthreads();
    for (int64_t e = e0 + tid; e < e1; e += kBigThreads) {
      const uint32_t c = cols[e];
      e2c[e] = pre[c >> 5] + __popc(bm[c >> 5] & ((1u << (c & 31)) - 1u));
    }
    if (tid == 0) ucount[w] = carry;
    __syncthreads();
  }
}

__global__ void sgt_fill(const int64_t* __restrict__ ptr, const uint32_t* __restrict__ cols,
                         int64_t n, int64_t num_windows, int bh, int bw,
                         const uint32_t* __restrict__ e2c, const int64_t* __restrict__ col_offsets,
                         uint32_t* __restrict__ c2n, uint32_t* __restrict__ wp) {
  // one warp per window
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= num_windows) return;
  const int64_t r0 = w * bh, r1 = min(r0 + bh, n);
  const int64_t e0 = ptr[r0], e1 = ptr[r1];
  const int64_t base = col_offsets[w];
  for (int64_t e = e0 + lane; e < e1; e += 32) c2n[base + e2c[e]] = cols[e];
  if (lane == 0) {
    const int64_t u = col_offsets[w + 1] - base;
    wp[w] = (uint32_t)((u + bw - 1) / bw);
  }
}

struct SgtWs {
  size_t ucount, big_count, big_list, cub_tmp, cub_bytes, bitmaps, prefixes, total;
};

SgtWs sgt_layout(int64_t n, int64_t num_windows) {
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  SgtWs L{};
  size_t off = 0;
  L.ucount = off;
  off += al(sizeof(int64_t) * (num_windows + 1));
  L.big_count = off;
  off += al(sizeof(int));
  L.big_list = off;
  off += al(sizeof(int) * (num_windows + 1));
  size_t cub_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, (int64_t*)nullptr, (int64_t*)nullptr,
                                (int)(num_windows + 1));
  L.cub_tmp = off;
  L.cub_bytes = cub_bytes;
  off += al(cub_bytes);
  const size_t nwords = (size_t)((n + 31) / 32);
  L.bitmaps = off;
  off += al(sizeof(uint32_t) * nwords * kBigCtas);
  L.prefixes = off;
  off += al(sizeof(uint32_t) * nwords * kBigCtas);
  L.total = off;
  return L;
}

}  // namespace
}  // namespace tcg

using namespace tcg;

extern "C" size_t tcg_sgt_workspace_bytes(int64_t num_nodes, int64_t num_edges, int32_t blk_h) {
  (void)num_edges;
  if (num_nodes < 0 || blk_h < 1) return 0;
  const int64_t W = (num_nodes + blk_h - 1) / blk_h;
  return sgt_layout(num_nodes, W).total;
}

// Phase 1 of SGT: ranks (edge_to_col), per-window unique counts and their
// exclusive scan (col_offsets[W+1]; U = col_offsets[W]).
extern "C" int tcg_sgt_count(const int64_t* node_ptr, const uint32_t* edge_list,
                             int64_t num_nodes, int64_t num_edges, int32_t blk_h, int32_t blk_w,
                             uint32_t* edge_to_col, int64_t* col_offsets, void* workspace,
                             size_t workspace_bytes, void* stream) {
  TCG_REQUIRE(blk_h >= 1 && blk_w >= 1, "tcg_sgt: tile shape must be >= 1, got %dx%d", blk_h,
              blk_w);
  TCG_REQUIRE(num_nodes >= 0 && num_edges >= 0, "tcg_sgt: negative size");
  TCG_REQUIRE(num_nodes <= 0xffffffffLL, "tcg_sgt: node ids must fit u32");
  TCG_REQUIRE(num_edges < (1LL << 31) * 2, "tcg_sgt: too many edges");
  const int64_t W = (num_nodes + blk_h - 1) / blk_h;
  const SgtWs L = sgt_layout(num_nodes, W);
  TCG_REQUIRE(workspace_bytes >= L.total, "tcg_sgt: workspace %zu < %zu bytes", workspace_bytes,
              L.total);
  cudaStream_t s = as_stream(stream);
  char* ws = static_cast<char*>(workspace);
  int64_t* ucount = reinterpret_cast<int64_t*>(ws + L.ucount);
  int* big_count = reinterpret_cast<int*>(ws + L.big_count);
  int* big_list = reinterpret_cast<int*>(ws + L.big_list);
  if (W == 0) {  // zero-node graph: col_offsets = [0] (the reference's zeros(1))
    if (col_offsets) TCG_CUDA(cudaMemsetAsync(col_offsets, 0, sizeof(int64_t), s), "tcg_sgt memset");
    return TCG_OK;
  }
  TCG_REQUIRE(node_ptr && col_offsets, "tcg_sgt: null pointer");
  TCG_CUDA(cudaMemsetAsync(ws + L.ucount, 0, sizeof(int64_t) * (W + 1), s), "tcg_sgt memset");
  TCG_CUDA(cudaMemsetAsync(big_count, 0, sizeof(int), s), "tcg_sgt memset");
  if (num_edges > 0) {
    TCG_REQUIRE(edge_list && edge_to_col, "tcg_sgt: null pointer");
    const int64_t grid = W < 65535LL * 16 ? W : 65535LL * 16;
    sgt_rank<<<(unsigned)grid, kRankThreads, 0, s>>>(node_ptr, edge_list, num_nodes, W, blk_h,
                                                     edge_to_col, ucount, big_list, big_count);
    TCG_LAUNCHED("sgt_rank");
    sgt_rank_big<<<kBigCtas, kBigThreads, 0, s>>>(
        node_ptr, edge_list, num_nodes, blk_h, big_list, big_count, edge_to_col, ucount,
        reinterpret_cast<uint32_t*>(ws + L.bitmaps), reinterpret_cast<uint32_t*>(ws + L.prefixes));
    TCG_LAUNCHED("sgt_rank_big");
  }
  size_t cub_bytes = L.cub_bytes;
  TCG_CUDA(cub::DeviceScan::ExclusiveSum(ws + L.cub_tmp, cub_bytes, ucount, col_offsets,
                                         (int)(W + 1), s),
           "tcg_sgt scan");
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  return TCG_OK;
}

// Phase 2: col_to_node[U] (caller-sized from col_offsets[W]) and win_partition.
extern "C" int tcg_sgt_fill(const int64_t* node_ptr, const uint32_t* edge_list,
                            int64_t num_nodes, int64_t num_edges, int32_t blk_h, int32_t blk_w,
                            const uint32_t* edge_to_col, const int64_t* col_offsets,
                            uint32_t* win_partition, uint32_t* col_to_node, void* stream) {
  TCG_REQUIRE(blk_h >= 1 && blk_w >= 1, "tcg_sgt: tile shape must be >= 1, got %dx%d", blk_h,
              blk_w);
  TCG_REQUIRE(num_nodes >= 0 && num_edges >= 0, "tcg_sgt: negative size");
  const int64_t W = (num_nodes + blk_h - 1) / blk_h;
  if (W == 0) return TCG_OK;
  TCG_REQUIRE(node_ptr && col_offsets && win_partition, "tcg_sgt: null pointer");
  TCG_REQUIRE(num_edges == 0 || (edge_list && edge_to_col && col_to_node),
              "tcg_sgt: null pointer");
  const int threads = 256;
  const int64_t blocks = (W * 32 + threads - 1) / threads;
  sgt_fill<<<(unsigned)blocks, threads, 0, as_stream(stream)>>>(
      node_ptr, edge_list, num_nodes, W, blk_h, blk_w, edge_to_col, col_offsets, col_to_node,
      win_partition);
  TCG_LAUNCHED("sgt_fill");
  return TCG_OK;
}

extern "C" int tcg_sgt(const int64_t* node_ptr, const uint32_t* edge_list, int64_t num_nodes,
                       int64_t num_edges, int32_t blk_h, int32_t blk_w, uint32_t* win_partition,
                       uint32_t* edge_to_col, int64_t* col_offsets, uint32_t* col_to_node,
                       void* workspace, size_t workspace_bytes, void* stream) {
  const int rc = tcg_sgt_count(node_ptr, edge_list, num_nodes, num_edges, blk_h, blk_w,
                               edge_to_col, col_offsets, workspace, workspace_bytes, stream);
  if (rc != TCG_OK) return rc;
  return tcg_sgt_fill(node_ptr, edge_list, num_nodes, num_edges, blk_h, blk_w, edge_to_col,
                      col_offsets, win_partition, col_to_node, stream);
}
