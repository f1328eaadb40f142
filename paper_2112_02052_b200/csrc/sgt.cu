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

#include <cstdlib>

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

// wlist: when non-null, the windows to rank (the warp path's overflow list)
__global__ void __launch_bounds__(kRankThreads)
    sgt_rank(const int64_t* __restrict__ ptr, const uint32_t* __restrict__ cols, int64_t n,
             int64_t w0, int64_t num_windows, int bh, int bw, uint32_t* __restrict__ e2c,
             int64_t* __restrict__ ucount, uint32_t* __restrict__ wp, int* __restrict__ big_list,
             int* __restrict__ big_count, const int* __restrict__ wlist, const int* __restrict__ wcount) {
  // 32-bit column ids are sorted (half the shared-memory traffic of sorting
  // (col, edge) pairs), compacted to the window's unique set, and every edge
  // is ranked by a binary search in it -- the reference's unique +
  // searchsorted (sgt.py:116-120)
  __shared__ uint32_t keys[kSmemCap];
  __shared__ uint32_t uniq[kSmemCap];
  __shared__ int scan_scratch[33];
  const int tid = threadIdx.x;
  const int64_t nwin = wlist ? (int64_t)*wcount : num_windows;
  for (int64_t q = blockIdx.x; q < nwin; q += gridDim.x) {
    const int64_t w = wlist ? (int64_t)wlist[q] : w0 + q;
    const int64_t r0 = w * bh;
    const int64_t r1 = min(r0 + bh, n);
    const int64_t e0 = ptr[r0], e1 = ptr[r1];
    const int64_t E = e1 - e0;
    if (E == 0) {
      if (tid == 0) ucount[w - w0] = 0, wp[w] = 0;
      continue;
    }
    if (E > kSmemCap) {
      if (tid == 0) big_list[atomicAdd(big_count, 1)] = (int)w;
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
    if (tid == 0) ucount[w - w0] = total, wp[w] = (uint32_t)((total + bw - 1) / bw);
    __syncthreads();
  }
}

// ---- warp-level path: windows of up to kWarpCap edges, one warp each ----
//
// Each edge becomes a 32-bit key (col << kIdxBits | local edge index); the
// window's keys are bitonic-sorted in registers (K keys per lane, position
// p = lane * K + r: stages with j < K are register compare-swaps, the rest
// __shfl_xor exchanges), then a head flag marks the first key of every
// distinct column, a warp scan of the per-lane head counts (ballot-free: K
// flags per lane, __shfl_up scan) gives every key its column's rank, and the
// rank is scattered back to the key's own edge. No shared memory, no
// __syncthreads. Needs N < 2^23 (col and index share the 32-bit key).
constexpr int kIdxBits = 9;
constexpr int kWarpCap = 1 << kIdxBits;  // 512 edges: K = 16 keys per lane

// Keys are kept complemented wherever the current merge level's block runs
// descending, so every compare-exchange is a plain (min, max) pair -- intra-lane
// two VIMNMX, inter-lane one SHFL and one VIMNMX with the lower lane keeping the
// minimum -- and the direction bookkeeping is one XOR per key per level (the
// last level is ascending everywhere, so the keys leave uncomplemented).
template <int K>
__device__ __forceinline__ void warp_bitonic(uint32_t (&v)[K], int lane) {
  auto desc = [&](int r, int k) { return ((lane * K + r) & k) != 0; };
#pragma unroll
  for (int r = 0; r < K; ++r)
    if (desc(r, 2)) v[r] = ~v[r];
#pragma unroll
  for (int k = 2; k <= 32 * K; k <<= 1) {
    if (k > 2) {
#pragma unroll
      for (int r = 0; r < K; ++r)
        if (desc(r, k >> 1) != desc(r, k)) v[r] = ~v[r];
    }
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= K) {
        const int lj = j / K;
        const bool lower = (lane & lj) == 0;
#pragma unroll
        for (int r = 0; r < K; ++r) {
          const uint32_t o = __shfl_xor_sync(0xffffffffu, v[r], lj);
          v[r] = lower ? min(v[r], o) : max(v[r], o);
        }
      } else {
#pragma unroll
        for (int r = 0; r < K; ++r) {
          if ((r & j) == 0) {
            const uint32_t x = v[r], y = v[r | j];
            v[r] = min(x, y);
            v[r | j] = max(x, y);
          }
        }
      }
    }
  }
}

template <int K>
__device__ __forceinline__ int64_t warp_rank_window(const uint32_t* __restrict__ cols, int64_t e0, int E,
                                                    uint32_t* __restrict__ e2c, int lane) {
  uint32_t v[K];
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const int i = r * 32 + lane;  // coalesced load; the key carries its edge index
    v[r] = i < E ? (__ldg(cols + e0 + i) << kIdxBits) | (uint32_t)i : 0xffffffffu;
  }
  warp_bitonic<K>(v, lane);
  const uint32_t prev_last = __shfl_up_sync(0xffffffffu, v[K - 1], 1);
  int heads = 0;
  uint32_t hmask = 0;
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const int p = lane * K + r;
    const uint32_t prev = r ? v[r - 1] : prev_last;
    const bool h = p < E && (p == 0 || (v[r] >> kIdxBits) != (prev >> kIdxBits));
    hmask |= (uint32_t)h << r;
    heads += h;
  }
  int incl = heads;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += n;
  }
  int run = incl - heads;  // heads before this lane's first key
#pragma unroll
  for (int r = 0; r < K; ++r) {
    run += (hmask >> r) & 1;
    if (lane * K + r < E) e2c[e0 + (v[r] & (kWarpCap - 1))] = (uint32_t)(run - 1);
  }
  return __shfl_sync(0xffffffffu, incl, 31);
}

__global__ void __launch_bounds__(256, 2)
    sgt_rank_warp(const int64_t* __restrict__ ptr, const uint32_t* __restrict__ cols, int64_t n,
                  int64_t w0, int64_t num_windows, int bh, int bw, uint32_t* __restrict__ e2c,
                  int64_t* __restrict__ ucount, uint32_t* __restrict__ wp, int* __restrict__ mid_list,
                  int* __restrict__ mid_count, int* __restrict__ big_list, int* __restrict__ big_count) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  if (blockIdx.x == 0 && threadIdx.x == 0) ucount[num_windows] = 0;
  for (int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < num_windows; q += nw) {
    const int64_t w = w0 + q;
    const int64_t r0 = w * bh, r1 = min(r0 + bh, n);
    const int64_t e0 = __ldg(ptr + r0), e1 = __ldg(ptr + r1);
    const int64_t E = e1 - e0;
    int64_t u = 0;
    if (E > kWarpCap) {
      if (lane == 0) {
        if (E > kSmemCap) big_list[atomicAdd(big_count, 1)] = (int)w;
        else mid_list[atomicAdd(mid_count, 1)] = (int)w;
      }
      continue;  // ucount[w] is written by the CTA kernels
    }
    if (E > 256) u = warp_rank_window<16>(cols, e0, (int)E, e2c, lane);
    else if (E > 128) u = warp_rank_window<8>(cols, e0, (int)E, e2c, lane);
    else if (E > 64) u = warp_rank_window<4>(cols, e0, (int)E, e2c, lane);
    else if (E > 32) u = warp_rank_window<2>(cols, e0, (int)E, e2c, lane);
    else if (E > 0) u = warp_rank_window<1>(cols, e0, (int)E, e2c, lane);
    if (lane == 0) ucount[q] = u, wp[w] = (uint32_t)((u + bw - 1) / bw);
  }
}

// Windows with more than kSmemCap edges: mark columns in a bitmap over
// [0, N) (per-CTA scratch), prefix-popcount it, rank = popcount below col.
__global__ void __launch_bounds__(kBigThreads)
    sgt_rank_big(const int64_t* __restrict__ ptr, const uint32_t* __restrict__ cols, int64_t n,
                 int64_t w0, int bh, int bw, const int* __restrict__ big_list, const int* __restrict__ big_count,
                 uint32_t* __restrict__ e2c, int64_t* __restrict__ ucount, uint32_t* __restrict__ wp,
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
    if (tid == 0) ucount[w - w0] = carry, wp[w] = (uint32_t)((carry + bw - 1) / bw);
    __syncthreads();
  }
}

// one warp per window of [w0, w0 + num_windows): col_to_node at the window's
// offset + base. base != 0 (a shard's share of the global scan) also turns the
// window's local col_offsets entry into the global one, in place: each entry
// is read and rewritten by its own window's warp only (win_partition came
// from the count phase, so nothing else reads col_offsets here).
__global__ void sgt_fill(const int64_t* __restrict__ ptr, const uint32_t* __restrict__ cols,
                         int64_t n, int64_t w0, int64_t num_windows, int bh, int64_t base,
                         const uint32_t* __restrict__ e2c, int64_t* __restrict__ col_offsets,
                         uint32_t* __restrict__ c2n, uint32_t* __restrict__ wp_out, int bw) {
  const int lane = threadIdx.x & 31;
  const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (q >= num_windows) return;
  const int64_t w = w0 + q;
  const int64_t r0 = w * bh, r1 = min(r0 + bh, n);
  const int64_t e0 = ptr[r0], e1 = ptr[r1];
  const int64_t off = col_offsets[w] + base;
  for (int64_t e = e0 + lane; e < e1; e += 32) c2n[off + e2c[e]] = cols[e];
  if (wp_out && lane == 0)  // base == 0 only (offsets not rewritten)
    wp_out[w] = (uint32_t)((col_offsets[w + 1] - col_offsets[w] + bw - 1) / bw);
  if (base != 0) {
    __syncwarp();
    if (lane == 0) {
      col_offsets[w] = off;
      if (q == num_windows - 1) col_offsets[w + 1] += base;
    }
  }
}

struct SgtWs {
  size_t ucount, big_count, big_list, mid_count, mid_list, wp, cub_tmp, cub_bytes, bitmaps, prefixes, total;
};

SgtWs sgt_layout(int64_t n, int64_t num_windows) {
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  SgtWs L{};
  size_t off = 0;
  L.ucount = off;
  off += al(sizeof(int64_t) * (num_windows + 1));
  L.big_count = off;  // big_count and mid_count are adjacent: one 8-byte memset
  L.mid_count = off + sizeof(int);
  off += al(2 * sizeof(int));
  L.big_list = off;
  off += al(sizeof(int) * (num_windows + 1));
  L.mid_list = off;
  off += al(sizeof(int) * (num_windows + 1));
  L.wp = off;
  off += al(sizeof(uint32_t) * (num_windows + 1));
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

// Phase 1 of SGT over windows [w0, w1): ranks (edge_to_col), win_partition,
// and col_offsets[w0..w1] = exclusive scan of the windows' unique counts
// starting at 0 (the whole graph: w0 = 0, w1 = W, so U = col_offsets[W]).
extern "C" int tcg_sgt_count_range(const int64_t* node_ptr, const uint32_t* edge_list,
                                   int64_t num_nodes, int64_t num_edges, int32_t blk_h, int32_t blk_w,
                                   int64_t win_begin, int64_t win_end, uint32_t* edge_to_col,
                                   int64_t* col_offsets, uint32_t* win_partition, void* workspace,
                                   size_t workspace_bytes, void* stream) {
  TCG_REQUIRE(blk_h >= 1 && blk_w >= 1, "tcg_sgt: tile shape must be >= 1, got %dx%d", blk_h,
              blk_w);
  TCG_REQUIRE(num_nodes >= 0 && num_edges >= 0, "tcg_sgt: negative size");
  TCG_REQUIRE(num_nodes <= 0xffffffffLL, "tcg_sgt: node ids must fit u32");
  TCG_REQUIRE(num_edges < (1LL << 31) * 2, "tcg_sgt: too many edges");
  const int64_t W = (num_nodes + blk_h - 1) / blk_h;
  TCG_REQUIRE(0 <= win_begin && win_begin <= win_end && win_end <= W,
              "tcg_sgt: window range [%lld, %lld) outside [0, %lld)", (long long)win_begin,
              (long long)win_end, (long long)W);
  const SgtWs L = sgt_layout(num_nodes, W);
  TCG_REQUIRE(workspace_bytes >= L.total, "tcg_sgt: workspace %zu < %zu bytes", workspace_bytes,
              L.total);
  cudaStream_t s = as_stream(stream);
  char* ws = static_cast<char*>(workspace);
  int64_t* ucount = reinterpret_cast<int64_t*>(ws + L.ucount);
  int* big_count = reinterpret_cast<int*>(ws + L.big_count);
  int* big_list = reinterpret_cast<int*>(ws + L.big_list);
  int* mid_count = reinterpret_cast<int*>(ws + L.mid_count);
  int* mid_list = reinterpret_cast<int*>(ws + L.mid_list);
  const int64_t nwin = win_end - win_begin;
  if (nwin == 0) {  // empty range (a zero-node graph: col_offsets = [0], the reference's zeros(1))
    if (col_offsets) TCG_CUDA(cudaMemsetAsync(col_offsets + win_begin, 0, sizeof(int64_t), s), "tcg_sgt memset");
    return TCG_OK;
  }
  TCG_REQUIRE(node_ptr && col_offsets && win_partition, "tcg_sgt: null pointer");
  // every window's ucount / win_partition entry is written by exactly one of the
  // ranking kernels; ucount[nwin] (the scan's last input) by sgt_rank_warp
  TCG_CUDA(cudaMemsetAsync(big_count, 0, 2 * sizeof(int), s), "tcg_sgt memset");
  if (num_edges == 0) {
    TCG_CUDA(cudaMemsetAsync(ucount, 0, sizeof(int64_t) * (nwin + 1), s), "tcg_sgt memset");
    TCG_CUDA(cudaMemsetAsync(win_partition + win_begin, 0, sizeof(uint32_t) * nwin, s), "tcg_sgt memset");
  }
  static const bool cta_only = std::getenv("TCG_SGT_CTA") != nullptr;  // round-1 path (A/B)
  if (num_edges > 0 && (num_nodes >= (1LL << 23) - 1 || cta_only))
    TCG_CUDA(cudaMemsetAsync(ucount + nwin, 0, sizeof(int64_t), s), "tcg_sgt memset");
  if (num_edges > 0) {
    TCG_REQUIRE(edge_list && edge_to_col, "tcg_sgt: null pointer");
    if (num_nodes < (1LL << 23) - 1 && !cta_only) {
      // a warp per window; windows past kWarpCap edges go to the CTA kernels
      const int64_t wblocks = (nwin + 7) / 8;
      const int64_t grid = wblocks < (int64_t)num_sms() * 16 ? wblocks : (int64_t)num_sms() * 16;
      sgt_rank_warp<<<(unsigned)grid, 256, 0, s>>>(node_ptr, edge_list, num_nodes, win_begin, nwin, blk_h,
                                                   blk_w, edge_to_col, ucount, win_partition, mid_list,
                                                   mid_count, big_list, big_count);
      TCG_LAUNCHED("sgt_rank_warp");
      sgt_rank<<<(unsigned)(num_sms() * 4), kRankThreads, 0, s>>>(
          node_ptr, edge_list, num_nodes, win_begin, nwin, blk_h, blk_w, edge_to_col, ucount, win_partition,
          big_list, big_count, mid_list, mid_count);
      TCG_LAUNCHED("sgt_rank");
    } else {
      const int64_t grid = nwin < 65535LL * 16 ? nwin : 65535LL * 16;
      sgt_rank<<<(unsigned)grid, kRankThreads, 0, s>>>(node_ptr, edge_list, num_nodes, win_begin, nwin,
                                                       blk_h, blk_w, edge_to_col, ucount, win_partition,
                                                       big_list, big_count, nullptr, nullptr);
      TCG_LAUNCHED("sgt_rank");
    }
    sgt_rank_big<<<kBigCtas, kBigThreads, 0, s>>>(
        node_ptr, edge_list, num_nodes, win_begin, blk_h, blk_w, big_list, big_count, edge_to_col, ucount,
        win_partition, reinterpret_cast<uint32_t*>(ws + L.bitmaps), reinterpret_cast<uint32_t*>(ws + L.prefixes));
    TCG_LAUNCHED("sgt_rank_big");
  }
  size_t cub_bytes = L.cub_bytes;
  TCG_CUDA(cub::DeviceScan::ExclusiveSum(ws + L.cub_tmp, cub_bytes, ucount, col_offsets + win_begin,
                                         (int)(nwin + 1), s),
           "tcg_sgt scan");
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  return TCG_OK;
}

// Phase 2 over windows [w0, w1): col_to_node at col_offsets[w] + base
// (col_to_node is global; base = the shard's exclusive prefix of the other
// shards' unique totals, 0 for the whole graph), then col_offsets[w0..w1] += base.
extern "C" int tcg_sgt_fill_range(const int64_t* node_ptr, const uint32_t* edge_list, int64_t num_nodes,
                                  int64_t num_edges, int32_t blk_h, int64_t win_begin, int64_t win_end,
                                  int64_t base, const uint32_t* edge_to_col, int64_t* col_offsets,
                                  uint32_t* col_to_node, void* stream) {
  TCG_REQUIRE(blk_h >= 1, "tcg_sgt: tile shape must be >= 1, got %d", blk_h);
  TCG_REQUIRE(num_nodes >= 0 && num_edges >= 0 && base >= 0, "tcg_sgt: negative size");
  const int64_t W = (num_nodes + blk_h - 1) / blk_h;
  TCG_REQUIRE(0 <= win_begin && win_begin <= win_end && win_end <= W,
              "tcg_sgt: window range [%lld, %lld) outside [0, %lld)", (long long)win_begin,
              (long long)win_end, (long long)W);
  const int64_t nwin = win_end - win_begin;
  if (nwin == 0) return TCG_OK;
  TCG_REQUIRE(node_ptr && col_offsets, "tcg_sgt: null pointer");
  TCG_REQUIRE(num_edges == 0 || (edge_list && edge_to_col && col_to_node), "tcg_sgt: null pointer");
  const int threads = 256;
  const int64_t blocks = (nwin * 32 + threads - 1) / threads;
  sgt_fill<<<(unsigned)blocks, threads, 0, as_stream(stream)>>>(node_ptr, edge_list, num_nodes, win_begin,
                                                                nwin, blk_h, base, edge_to_col, col_offsets,
                                                                col_to_node, nullptr, 1);
  TCG_LAUNCHED("sgt_fill");
  return TCG_OK;
}

// Phase 1 over the whole graph (SURVEY.md Appendix D signature): ranks and
// col_offsets[W+1]; win_partition is written by tcg_sgt_fill.
extern "C" int tcg_sgt_count(const int64_t* node_ptr, const uint32_t* edge_list,
                             int64_t num_nodes, int64_t num_edges, int32_t blk_h, int32_t blk_w,
                             uint32_t* edge_to_col, int64_t* col_offsets, void* workspace,
                             size_t workspace_bytes, void* stream) {
  TCG_REQUIRE(blk_h >= 1 && blk_w >= 1, "tcg_sgt: tile shape must be >= 1, got %dx%d", blk_h,
              blk_w);
  TCG_REQUIRE(num_nodes >= 0, "tcg_sgt: negative size");
  const int64_t W = (num_nodes + blk_h - 1) / blk_h;
  const SgtWs L = sgt_layout(num_nodes, W);
  TCG_REQUIRE(workspace_bytes >= L.total, "tcg_sgt: workspace %zu < %zu bytes", workspace_bytes,
              L.total);
  uint32_t* wp_scratch = reinterpret_cast<uint32_t*>(static_cast<char*>(workspace) + L.wp);
  return tcg_sgt_count_range(node_ptr, edge_list, num_nodes, num_edges, blk_h, blk_w, 0, W, edge_to_col,
                             col_offsets, wp_scratch, workspace, workspace_bytes, stream);
}

// Phase 2 over the whole graph: col_to_node[U] and win_partition[W].
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
      node_ptr, edge_list, num_nodes, 0, W, blk_h, 0, edge_to_col, const_cast<int64_t*>(col_offsets),
      col_to_node, win_partition, blk_w);
  TCG_LAUNCHED("sgt_fill");
  return TCG_OK;
}

extern "C" int tcg_sgt(const int64_t* node_ptr, const uint32_t* edge_list, int64_t num_nodes,
                       int64_t num_edges, int32_t blk_h, int32_t blk_w, uint32_t* win_partition,
                       uint32_t* edge_to_col, int64_t* col_offsets, uint32_t* col_to_node,
                       void* workspace, size_t workspace_bytes, void* stream) {
  const int64_t W = num_nodes >= 0 && blk_h >= 1 ? (num_nodes + blk_h - 1) / blk_h : 0;
  const int rc = tcg_sgt_count_range(node_ptr, edge_list, num_nodes, num_edges, blk_h, blk_w, 0, W,
                                     edge_to_col, col_offsets, win_partition, workspace, workspace_bytes,
                                     stream);
  if (rc != TCG_OK) return rc;
  return tcg_sgt_fill_range(node_ptr, edge_list, num_nodes, num_edges, blk_h, 0, W, 0, edge_to_col,
                            col_offsets, col_to_node, stream);
}
