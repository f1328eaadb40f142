// The row-window engine: every TF32 tensor-core op of the hot path.
//
// One warp owns one 16-row window at a time (persistent grid, windows
// round-robin over warps) and runs the reference's tile dataflow
// (tiles.py:130-250, kernels.py:254-538, Alg. 2/3) out of shared
// memory:
//
//   1. FetchDense  — the window's condensed neighbour rows X[col_to_node[c]]
//      are gathered into shared memory by TMA (cp.async.bulk.tensor
//      tile::gather4: one instruction moves 4 rows; each lane of the warp
//      issues one, so a whole window is in flight after a single warp
//      instruction) completing on an mbarrier. The tensor map's 128B/64B/32B
//      swizzle places row s's 16-B chunk k at k ^ f(s); condensed column c is
//      written to smem row srow(c) = (c & ~7) | bitrev3(c & 7), so both
//      fragment read patterns (SpMM: rows t / chunks g; SDDMM: rows g /
//      chunks t) are bank-conflict free for 128-B rows. Padding columns of
//      the last 16-column group use an out-of-range row index: TMA fills
//      them with zeros. (Fallback when TMA is not legal: cp.async 16-B/4-B.)
//      While the gather is in flight the warp prefetches the NEXT window's
//      metadata and col_to_node slice and loads this window's edge data.
//   2. InitSparse  — edge weights are scattered into the 16x8 A tiles in
//      mma.m16n8k8 fragment order through the per-edge fragment slot
//      `efrag` (computed once per tiling, the analogue of the reference's
//      per-edge `_spmm_aux` cache, kernels.py:173-188).
//   3. mma.sync.m16n8k8 TF32 (operands RNE-rounded by cvt.rn.tf32.f32, fp32
//      accumulate) for SpMM (B = staged rows, features permuted so each
//      lane's slice is contiguous) and for SDDMM (A = the window's own 16
//      rows, B = staged rows, k = features). Fragment addresses are per-lane
//      constants plus a block stride.
//   4. Epilogues: StoreDense (bias / accumulate, vectorised row stores),
//      StoreSparse (score tile -> edge order), row softmax and its backward
//      (rows never straddle windows, 2 lanes per row).
//
// Modes:
//   SPMM       Y = A_w X (+bias) (+=)                 reference spmm
//   SPMM_DUAL  Y += A_w1 X1 + A_w2 X2 (A^T pass of the AGNN backward)
//   SDDMM      s_e = <XA_row, X_col> (+ softmax / softmax-bwd epilogue)
//   AGNN_FWD   P = softmax(<Z_i,Z_j>), Y = A_P Z     reference agnn_layer,
//              one gather of Z's neighbour rows serves both products
//   AGNN_BWD   dS = P (dP - rowsum(P dP)), dP = <G_i,Z_j>; Y = A_dS Z
#include <cudaTypedefs.h>

#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "window.cuh"

namespace tcg {
namespace win {

constexpr int kWarps = 4;

__host__ __device__ constexpr int brev3(int x) { return ((x & 1) << 2) | (x & 2) | ((x >> 2) & 1); }
__device__ __forceinline__ int srow(int c) { return (c & ~7) | brev3(c & 7); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(s)), "l"(g));
}
__device__ __forceinline__ void cp_async4(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(s)), "l"(g));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait_all() {
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* tm, int col, int r0,
                                            int r1, int r2, int r3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
      "r"(smem_u32(bar))
      : "memory");
}

// Staged-row geometry. Rows are stored exactly as the TMA swizzle writes
// them (region bases 1024-B aligned): 16-B chunk k of row s goes to
// k ^ ((s * rowbytes >> 7) & mask). NT=8 rows are split into two 128-B
// halves stored in two regions.
template <int NT>
struct Geo {
  static constexpr int BW = NT >= 4 ? 32 : 8 * NT;  // floats per TMA box row
  static constexpr int HALVES = NT == 8 ? 2 : 1;
  static constexpr int DS = 8 * NT;                  // features per staged row
  static constexpr int V = NT < 4 ? NT : 4;          // fragment read vector width
  __host__ __device__ static constexpr int swz(int s) {
    return BW == 32 ? (s & 7) : BW == 16 ? ((s >> 1) & 3) : ((s >> 2) & 1);
  }
  template <int CPR>
  __host__ __device__ static constexpr int off(int s, int f) {
    return (f / BW) * CPR * BW + s * BW + ((((f % BW) >> 2) ^ swz(s)) << 2) + (f & 3);
  }
};

template <int NT, int MODE>
struct Carve {
  static constexpr bool kDual = MODE == MODE_SPMM_DUAL;
  static constexpr bool kFused = MODE == MODE_AGNN_FWD || MODE == MODE_AGNN_BWD;
  static constexpr int CPR = cols_per_round(NT, MODE);
  static constexpr int tile_stride = CPR + 4;
  static constexpr int xs = 0;  // 1024-B aligned
  static constexpr int xs_bytes = CPR * 8 * NT * 4;
  static constexpr int frag = xs + xs_bytes * (kDual ? 2 : 1);
  static constexpr int frag_a = (CPR / 8) * 512 * (kDual ? 2 : 1);
  static constexpr int frag_t = (kFused || MODE == MODE_SDDMM) ? 16 * tile_stride * 4 : 0;
  static constexpr int frag_bytes = frag_a > frag_t ? frag_a : frag_t;
  static constexpr int edges = frag + frag_bytes;
  static constexpr int rps = edges + (kFused ? kEdgesPerWindow * 4 : 0);  // 2 x 17 int64
  static constexpr int nodes = rps + 288;                                  // CPR int
  static constexpr int bar = nodes + CPR * 4;                              // mbarrier
  static constexpr int total = (bar + 8 + 1023) & ~1023;
};

template <int VW>
__device__ __forceinline__ void lds_vec(float* dst, const float* src) {
  if constexpr (VW == 4) {
    const float4 v = *reinterpret_cast<const float4*>(src);
    dst[0] = v.x, dst[1] = v.y, dst[2] = v.z, dst[3] = v.w;
  } else if constexpr (VW == 2) {
    const float2 v = *reinterpret_cast<const float2*>(src);
    dst[0] = v.x, dst[1] = v.y;
  } else {
    dst[0] = *src;
  }
}

// efrag slot -> (row within window, column within the round)
__device__ __forceinline__ void decode_slot(int fi, int& row, int& col) {
  const int ln = (fi >> 2) & 31, sl = fi & 3;
  row = (ln >> 2) + 8 * (sl & 1);
  col = (fi >> 7) * 8 + (ln & 3) + 4 * (sl >> 1);
}

template <int NT, int MODE>
__global__ void __launch_bounds__(kWarps * 32)
    window_kernel(const Params p, const __grid_constant__ CUtensorMap tmx,
                  const __grid_constant__ CUtensorMap tmx2) {
  using G = Geo<NT>;
  using CV = Carve<NT, MODE>;
  constexpr int CPR = CV::CPR;
  constexpr int DS = G::DS;
  constexpr int V = G::V;
  constexpr int NQ = NT / V;
  constexpr int NPF = CPR / 32;  // prefetched col_to_node registers per lane
  constexpr bool kDual = CV::kDual;
  constexpr bool kFused = CV::kFused;
  constexpr bool kSpmmPhase = MODE != MODE_SDDMM;
  constexpr bool kSddmmPhase = MODE == MODE_SDDMM || kFused;
  constexpr int TS = CV::tile_stride;
  constexpr int XS2 = CPR * DS;  // floats between the two operands' regions (dual)
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  unsigned char* sm = smem_raw + warp * CV::total;
  if ((smem_u32(sm) & 1023) != 0) __trap();  // TMA swizzle needs 1024-B aligned rows
  float* xs = reinterpret_cast<float*>(sm + CV::xs);
  uint32_t* afrag = reinterpret_cast<uint32_t*>(sm + CV::frag);
  uint32_t* afrag2 = afrag + (CPR / 8) * 128;
  float* tile = reinterpret_cast<float*>(sm + CV::frag);
  float* escore = reinterpret_cast<float*>(sm + CV::edges);
  int64_t* rps2 = reinterpret_cast<int64_t*>(sm + CV::rps);  // [2][17]
  int* nodes = reinterpret_cast<int*>(sm + CV::nodes);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + CV::bar);

  // zero the staged rows once: feature padding [dim, DS) is never written
  for (int i = lane; i < CPR * DS * (kDual ? 2 : 1); i += 32) xs[i] = 0.f;
  if (lane == 0) mbar_init(bar);
  uint32_t phase = 0;
  __syncwarp();

  // per-lane fragment offsets (floats) within an 8-row (SpMM) / 16-row
  // (SDDMM) block of staged rows; blocks add a constant stride
  int spo0[NQ], spo1[NQ], sdo0[NQ], sdo1[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    spo0[q] = G::template off<CPR>(brev3(t), g * NT + q * V);
    spo1[q] = G::template off<CPR>(brev3(t + 4), g * NT + q * V);
    sdo0[q] = G::template off<CPR>(brev3(g), t * NT + q * V);
    sdo1[q] = G::template off<CPR>(brev3(g), (t + 4) * NT + q * V);
  }

  const int64_t nwarps = (int64_t)gridDim.x * kWarps;
  const int64_t tasks = p.nwin * p.nchunks;
  int64_t task = (int64_t)blockIdx.x * kWarps + warp;

  // ---- prefetch registers for the next task ----
  int64_t pf_rp = 0, pf_c0 = 0, pf_cend = 0;
  int pf_node[NPF];
  auto prefetch = [&](int64_t tk) {
    if (tk >= tasks) return;
    const int64_t w = p.win_begin + tk / p.nchunks;
    const int64_t r0 = w * 16;
    pf_rp = lane <= 16 ? __ldg(p.ptr + min(r0 + lane, p.n)) : 0;
    pf_c0 = __ldg(p.coff + w);
    pf_cend = __ldg(p.coff + w + 1);
    const int64_t u = pf_cend - pf_c0;
#pragma unroll
    for (int k = 0; k < NPF; ++k) {
      const int c = lane + 32 * k;
      pf_node[k] = c < u ? (int)__ldg(p.c2n + pf_c0 + c) : 0;
    }
  };
  prefetch(task);
  int buf = 0;

  for (; task < tasks; task += nwarps, buf ^= 1) {
    const int64_t w = p.win_begin + task / p.nchunks;
    const int chunk = (int)(task % p.nchunks);
    const int d0 = chunk * 8 * NT;
    const int64_t r0 = w * 16;
    const int64_t r1 = min(r0 + 16, p.n);
    int64_t* rps = rps2 + buf * 17;
    if (lane <= 16) rps[lane] = pf_rp;
    const int64_t c0 = pf_c0;
    const int u = (int)(pf_cend - pf_c0);
#pragma unroll
    for (int k = 0; k < NPF; ++k) nodes[lane + 32 * k] = pf_node[k];
    __syncwarp();
    const int64_t e0 = rps[0], e1 = rps[16];
    const int E = (int)(e1 - e0);
    const int nrounds = kFused ? 1 : (u + CPR - 1) / CPR;
    const int nkc = MODE == MODE_SDDMM ? p.nkc : 1;

    float acc[NT][4];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;

    for (int rd = 0; rd < max(nrounds, 1); ++rd) {
      const int cb = rd * CPR;             // first column of this round
      const int ncols = min(CPR, u - cb);  // <= 0 for empty windows
      const int pad = min(CPR, (max(ncols, 0) + 15) & ~15);
      if (rd > 0) {
        __syncwarp();
        for (int c = lane; c < ncols; c += 32) nodes[c] = (int)__ldg(p.c2n + c0 + cb + c);
        __syncwarp();
      }
      for (int kc = 0; kc < nkc; ++kc) {
        // SDDMM folds D in k-chunks of 8*NT features; SpMM modes use one chunk
        const int dk = MODE == MODE_SDDMM ? kc * 8 * NT : d0;
        const int dv = min(8 * NT, p.dim - dk);
        if (kc > 0) __syncwarp();
        // ---- 1. FetchDense: stage rows [0, ncols) ----
        const bool staged_tma = p.use_tma && pad > 0;
        if (staged_tma) {
          constexpr uint32_t kGroupBytes = 4u * G::BW * 4u * G::HALVES * (kDual ? 2 : 1);
          fence_proxy_async();  // previous generic reads of xs before async writes
          __syncwarp();
          if (lane == 0) mbar_expect(bar, (uint32_t)(pad / 4) * kGroupBytes);
          __syncwarp();
          if (lane < pad / 4) {
            int rr[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const int srw = 4 * lane + r;
              const int c = (srw & ~7) | brev3(srw & 7);
              rr[r] = c < ncols ? nodes[c] : (int)p.n;  // out of range -> zero fill
            }
            float* dst = xs + 4 * lane * G::BW;
#pragma unroll
            for (int hv = 0; hv < G::HALVES; ++hv) {
              tma_gather4(dst + hv * CPR * G::BW, &tmx, dk + hv * 32, rr[0], rr[1], rr[2], rr[3],
                          bar);
              if (kDual)
                tma_gather4(dst + XS2 + hv * CPR * G::BW, &tmx2, dk + hv * 32, rr[0], rr[1],
                            rr[2], rr[3], bar);
            }
          }
        } else if (pad > 0) {
          for (int q = lane; q < pad * DS; q += 32) {
            const int c = q / DS, f = q % DS;
            float* dst = xs + G::template off<CPR>(srow(c), f);
            if (c < ncols) {
              if (f < dv) {
                const int64_t node = nodes[c];
                cp_async4(dst, p.x + node * p.ldx + dk + f);
                if (kDual) cp_async4(dst + XS2, p.x2 + node * p.ldx2 + dk + f);
              }
            } else {
              *dst = 0.f;
              if (kDual) dst[XS2] = 0.f;
            }
          }
          cp_commit();
        }
        // ---- prefetch the next task (overlaps the gather) ----
        if ((rd == nrounds - 1 || nrounds == 0) && kc == nkc - 1) prefetch(task + nwarps);

        // ---- 2. per-edge work while rows land ----
        if constexpr (kSpmmPhase && !kFused) {
          const int nb = (pad + 7) >> 3;
          for (int i = lane; i < nb * 32; i += 32) {
            reinterpret_cast<uint4*>(afrag)[i] = make_uint4(0, 0, 0, 0);
            if (kDual) reinterpret_cast<uint4*>(afrag2)[i] = make_uint4(0, 0, 0, 0);
          }
          __syncwarp();
          const int fbase = cb * 16, flim = ((max(ncols, 0) + 7) >> 3) * 128;  // whole blocks
          for (int64_t eb = e0; eb < e1; eb += 128) {
            int fi[4];
            float wv[4], wv2[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const int64_t e = eb + lane + 32 * v;
              fi[v] = e < e1 ? (int)__ldg(p.efrag + e) - fbase : -1;
              wv[v] = 1.f;
              wv2[v] = 1.f;
              if (e < e1 && p.w) wv[v] = p.widx ? __ldg(p.w + __ldg(p.widx + e)) : __ldg(p.w + e);
              if (kDual && e < e1 && p.w2)
                wv2[v] = p.widx2 ? __ldg(p.w2 + __ldg(p.widx2 + e)) : __ldg(p.w2 + e);
            }
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              if (fi[v] >= 0 && fi[v] < flim) {
                afrag[fi[v]] = tf32_rn(wv[v]);
                if (kDual) afrag2[fi[v]] = tf32_rn(wv2[v]);
              }
            }
          }
        }
        uint32_t efr[kFused ? kEdgesPerWindow / 32 : 1];
        if constexpr (kFused) {
#pragma unroll
          for (int v = 0; v < kEdgesPerWindow / 32; ++v) {
            const int i = lane + 32 * v;
            efr[v] = i < E ? __ldg(p.efrag + e0 + i) : 0u;
          }
        }
        // A operand of the SDDMM phase: the window's own rows, to registers
        float ar[4][NT];
        if constexpr (kSddmmPhase) {
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int64_t r = r0 + g + ((h & 1) ? 8 : 0);
            const int f0 = ((h & 2) ? (t + 4) : t) * NT;
            const float* src = p.xa + r * p.lda + dk + f0;
            bool done = false;
            if constexpr (NT % 4 == 0) {
              if (p.vec16 && r < r1 && f0 + NT <= dv) {
#pragma unroll
                for (int j = 0; j < NT; j += 4) {
                  const float4 q4 = __ldg(reinterpret_cast<const float4*>(src + j));
                  ar[h][j] = q4.x, ar[h][j + 1] = q4.y, ar[h][j + 2] = q4.z, ar[h][j + 3] = q4.w;
                }
                done = true;
              }
            }
            if (!done) {
#pragma unroll
              for (int j = 0; j < NT; ++j) ar[h][j] = (r < r1 && f0 + j < dv) ? __ldg(src + j) : 0.f;
            }
          }
        }
        if (staged_tma) {
          mbar_wait(bar, phase);
          phase ^= 1;
        } else {
          cp_wait_all();
        }
        __syncwarp();

        // ---- 3a. SDDMM phase: scores for 16-column paired blocks ----
        if constexpr (kSddmmPhase) {
          const int npb = pad >> 4;
          uint32_t a[4][NT];
#pragma unroll
          for (int h = 0; h < 4; ++h)
#pragma unroll
            for (int j = 0; j < NT; ++j) a[h][j] = tf32_rn(ar[h][j]);
          float* trow0 = tile + g * TS + 2 * t;
          float* trow1 = tile + (g + 8) * TS + 2 * t;
          for (int sb = 0; sb < npb; ++sb) {
            float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const float* blk = xs + (sb * 16 + hh * 8) * G::BW;
              float b0[NT], b1[NT];
#pragma unroll
              for (int q = 0; q < NQ; ++q) {
                lds_vec<V>(b0 + q * V, blk + sdo0[q]);
                lds_vec<V>(b1 + q * V, blk + sdo1[q]);
              }
#pragma unroll
              for (int j = 0; j < NT; ++j)
                mma_tf32(sc[hh], a[0][j], a[1][j], a[2][j], a[3][j], tf32_rn(b0[j]),
                         tf32_rn(b1[j]));
            }
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              float2* p0 = reinterpret_cast<float2*>(trow0 + sb * 16 + hh * 8);
              float2* p1 = reinterpret_cast<float2*>(trow1 + sb * 16 + hh * 8);
              if (kc == 0) {
                *p0 = make_float2(sc[hh][0], sc[hh][1]);
                *p1 = make_float2(sc[hh][2], sc[hh][3]);
              } else {
                const float2 o0 = *p0, o1 = *p1;
                *p0 = make_float2(o0.x + sc[hh][0], o0.y + sc[hh][1]);
                *p1 = make_float2(o1.x + sc[hh][2], o1.y + sc[hh][3]);
              }
            }
          }
        }
        if constexpr (kFused) {
          // edge scores out of the tile
          __syncwarp();
#pragma unroll
          for (int v = 0; v < kEdgesPerWindow / 32; ++v) {
            const int i = lane + 32 * v;
            if (i < E) {
              int row, col;
              decode_slot((int)efr[v], row, col);
              escore[i] = tile[row * TS + col];
            }
          }
          __syncwarp();
          // row softmax (fwd) / softmax backward (bwd): 2 lanes per row
          const int row = lane >> 1, sub = lane & 1;
          const int rb = (int)(rps[row] - e0), re = (int)(rps[row + 1] - e0);
          if constexpr (MODE == MODE_AGNN_FWD) {
            float m = -INFINITY;
            for (int i = rb + sub; i < re; i += 2) m = fmaxf(m, escore[i]);
            m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
            float s = 0.f;
            for (int i = rb + sub; i < re; i += 2) s += expf(escore[i] - m);
            s += __shfl_xor_sync(0xffffffffu, s, 1);
            for (int i = rb + sub; i < re; i += 2) escore[i] = expf(escore[i] - m) / s;
          } else {
            float s = 0.f;
            for (int i = rb + sub; i < re; i += 2) s += __ldg(p.aux + e0 + i) * escore[i];
            s += __shfl_xor_sync(0xffffffffu, s, 1);
            for (int i = rb + sub; i < re; i += 2)
              escore[i] = __ldg(p.aux + e0 + i) * (escore[i] - s);
          }
          // weights -> edge order (P or dS) and -> fragment-ordered A tiles
          const int nb = (pad + 7) >> 3;
          for (int i = lane; i < nb * 32; i += 32)
            reinterpret_cast<uint4*>(afrag)[i] = make_uint4(0, 0, 0, 0);
          __syncwarp();
#pragma unroll
          for (int v = 0; v < kEdgesPerWindow / 32; ++v) {
            const int i = lane + 32 * v;
            if (i < E) {
              const float wgt = escore[i];
              p.eout[e0 + i] = wgt;
              afrag[efr[v]] = tf32_rn(wgt);
            }
          }
        }
      }  // k-chunks
      if constexpr (MODE == MODE_SDDMM) {
        // StoreSparse: raw scores of this round's columns to edge order
        __syncwarp();
        const int fbase = cb * 16, flim = ((max(ncols, 0) + 7) >> 3) * 128;  // whole blocks
        for (int64_t e = e0 + lane; e < e1; e += 32) {
          const int fi = (int)__ldg(p.efrag + e) - fbase;
          if (fi < 0 || fi >= flim) continue;
          int row, col;
          decode_slot(fi, row, col);
          p.eout[e] = tile[row * TS + col];
        }
      }
      __syncwarp();

      // ---- 3c. SpMM phase over the 16x8 blocks of this round ----
      if constexpr (kSpmmPhase) {
        const int nb = (max(ncols, 0) + 7) >> 3;
#pragma unroll 2
        for (int b = 0; b < nb; ++b) {
          const uint4 af = reinterpret_cast<const uint4*>(afrag)[b * 32 + lane];
          const float* blk = xs + b * 8 * G::BW;
          float x0[NT], x1[NT];
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            lds_vec<V>(x0 + q * V, blk + spo0[q]);
            lds_vec<V>(x1 + q * V, blk + spo1[q]);
          }
#pragma unroll
          for (int j = 0; j < NT; ++j)
            mma_tf32(acc[j], af.x, af.y, af.z, af.w, tf32_rn(x0[j]), tf32_rn(x1[j]));
          if constexpr (kDual) {
            const uint4 af2 = reinterpret_cast<const uint4*>(afrag2)[b * 32 + lane];
            const float* blk2 = blk + XS2;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
              lds_vec<V>(x0 + q * V, blk2 + spo0[q]);
              lds_vec<V>(x1 + q * V, blk2 + spo1[q]);
            }
#pragma unroll
            for (int j = 0; j < NT; ++j)
              mma_tf32(acc[j], af2.x, af2.y, af2.z, af2.w, tf32_rn(x0[j]), tf32_rn(x1[j]));
          }
        }
        __syncwarp();
      }
    }  // rounds

    // ---- 4. epilogues after all rounds ----
    if constexpr (MODE == MODE_SDDMM) {
      if (p.epilogue != 0) {
        __syncwarp();
        const int row = lane >> 1, sub = lane & 1;
        const int64_t rb = rps[row], re = rps[row + 1];
        if (p.epilogue == 1) {
          float m = -INFINITY;
          for (int64_t i = rb + sub; i < re; i += 2) m = fmaxf(m, p.eout[i]);
          m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
          float s = 0.f;
          for (int64_t i = rb + sub; i < re; i += 2) s += expf(p.eout[i] - m);
          s += __shfl_xor_sync(0xffffffffu, s, 1);
          for (int64_t i = rb + sub; i < re; i += 2) p.eout[i] = expf(p.eout[i] - m) / s;
        } else {
          float s = 0.f;
          for (int64_t i = rb + sub; i < re; i += 2) s += __ldg(p.aux + i) * p.eout[i];
          s += __shfl_xor_sync(0xffffffffu, s, 1);
          for (int64_t i = rb + sub; i < re; i += 2) p.eout[i] = __ldg(p.aux + i) * (p.eout[i] - s);
        }
      }
    }
    if constexpr (kSpmmPhase) {
      // StoreDense: lane owns rows g, g+8 and features [2t*NT, 2t*NT + 2NT) of the chunk
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
        float* yr = p.y + (r - p.y_row0) * p.ldy + fo;
        if (p.vec_out && fo + 2 * NT <= p.dim) {
          constexpr int VO = (2 * NT) >= 4 ? 4 : 2 * NT;
#pragma unroll
          for (int q = 0; q < 2 * NT; q += VO) {
            if constexpr (VO == 4) {
              float4 v = make_float4(o[q], o[q + 1], o[q + 2], o[q + 3]);
              if (p.bias) {
                const float4 bv = __ldg(reinterpret_cast<const float4*>(p.bias + fo + q));
                v.x += bv.x, v.y += bv.y, v.z += bv.z, v.w += bv.w;
              }
              if (p.accumulate) {
                const float4 ov = *reinterpret_cast<const float4*>(yr + q);
                v.x += ov.x, v.y += ov.y, v.z += ov.z, v.w += ov.w;
              }
              *reinterpret_cast<float4*>(yr + q) = v;
            } else {
#pragma unroll
              for (int v = 0; v < VO; ++v) {
                float x = o[q + v];
                if (p.bias) x += __ldg(p.bias + fo + q + v);
                if (p.accumulate) x += yr[q + v];
                yr[q + v] = x;
              }
            }
          }
        } else {
#pragma unroll
          for (int q = 0; q < 2 * NT; ++q) {
            if (fo + q < p.dim) {
              float x = o[q];
              if (p.bias) x += __ldg(p.bias + fo + q);
              if (p.accumulate) x += yr[q];
              yr[q] = x;
            }
          }
        }
      }
    }
    __syncwarp();
  }
}

// Per-edge fragment slot of the 16x8 tiling: one thread per row.
__global__ void edge_frag_kernel(const int64_t* __restrict__ ptr, const uint32_t* __restrict__ e2c,
                                 int64_t n, uint32_t* __restrict__ efrag) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int rl = (int)(r & 15);
  const int lane_hi = (rl & 7) << 2, slot_hi = rl >> 3;
  for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e) {
    const uint32_t c = e2c[e];
    const uint32_t k = c & 7;
    efrag[e] = (c >> 3) * 128 + ((lane_hi | (k & 3)) << 2) + slot_hi + 2 * (k >> 2);
  }
}

// ---- host: tensor maps for the gathered operands ----------------------------

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

struct TmKey {
  const void* x;
  int64_t n, dim, ld;
  int bw;
  bool operator==(const TmKey& o) const {
    return x == o.x && n == o.n && dim == o.dim && ld == o.ld && bw == o.bw;
  }
};
struct TmHash {
  size_t operator()(const TmKey& k) const {
    return std::hash<const void*>()(k.x) ^ (size_t)(k.n * 1315423911u) ^ (size_t)(k.ld << 7) ^
           (size_t)k.bw;
  }
};

// fp32 [n rows, dim cols] with row stride ld; box = (bw cols, 1 row) for gather4
bool make_tmap(const float* x, int64_t n, int64_t dim, int64_t ld, int bw, CUtensorMap* out) {
  static std::mutex mu;
  static std::unordered_map<TmKey, CUtensorMap, TmHash> cache;
  const TmKey key{x, n, dim, ld, bw};
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return true;
  }
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t gdim[2] = {(cuuint64_t)dim, (cuuint64_t)n};
  cuuint64_t gstride[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)bw, 1};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle swz = bw == 32   ? CU_TENSOR_MAP_SWIZZLE_128B
                                 : bw == 16 ? CU_TENSOR_MAP_SWIZZLE_64B
                                            : CU_TENSOR_MAP_SWIZZLE_32B;
  CUtensorMap tm;
  if (fn(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(x), gdim, gstride, box, estr,
         CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, tm);
  *out = tm;
  return true;
}

int edge_frag(const int64_t* ptr, const uint32_t* e2c, int64_t n, uint32_t* efrag,
              cudaStream_t s) {
  if (n == 0) return TCG_OK;
  edge_frag_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(ptr, e2c, n, efrag);
  TCG_LAUNCHED("edge_frag");
  return TCG_OK;
}

template <int NT, int MODE>
int launch_nt(Params& p, cudaStream_t s) {
  using CV = Carve<NT, MODE>;
  using G = Geo<NT>;
  const size_t smem = (size_t)CV::total * kWarps;
  auto kern = window_kernel<NT, MODE>;
  static int configured_dev = -1;
  static int per_sm = 1;
  int dev = 0;
  TCG_CUDA(cudaGetDevice(&dev), "window_kernel device");
  if (configured_dev != dev) {
    TCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
             "window_kernel attr");
    TCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarps * 32, smem),
             "window_kernel occupancy");
    if (per_sm < 1) per_sm = 1;
    configured_dev = dev;
  }
  // TMA gather legality: 16-B aligned base and row stride, int32 row ids
  CUtensorMap tm1{}, tm2{};
  const bool dual = MODE == MODE_SPMM_DUAL;
  const int64_t tcols = p.dim;
  bool tma = p.n < (1LL << 31) - 1 && p.ldx % 4 == 0 &&
             (reinterpret_cast<uintptr_t>(p.x) & 15) == 0 &&
             (!dual || (p.ldx2 % 4 == 0 && (reinterpret_cast<uintptr_t>(p.x2) & 15) == 0));
  if (tma) tma = make_tmap(p.x, p.n, tcols, p.ldx, G::BW, &tm1);
  if (tma && dual) tma = make_tmap(p.x2, p.n, tcols, p.ldx2, G::BW, &tm2);
  p.use_tma = tma ? 1 : 0;
  const int64_t tasks = p.nwin * p.nchunks;
  int64_t blocks = (tasks + kWarps - 1) / kWarps;
  const int64_t cap = (int64_t)num_sms() * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) return TCG_OK;
  kern<<<(unsigned)blocks, kWarps * 32, smem, s>>>(p, tm1, tm2);
  TCG_LAUNCHED("window_kernel");
  return TCG_OK;
}

template <int MODE>
int launch_mode(int nt, Params& p, cudaStream_t s) {
  switch (nt) {
    case 1: return launch_nt<1, MODE>(p, s);
    case 2: return launch_nt<2, MODE>(p, s);
    case 4: return launch_nt<4, MODE>(p, s);
    default: return launch_nt<8, MODE>(p, s);
  }
}

int launch(int mode, int nt, Params& p, cudaStream_t s) {
  switch (mode) {
    case MODE_SPMM: return launch_mode<MODE_SPMM>(nt, p, s);
    case MODE_SPMM_DUAL: return launch_mode<MODE_SPMM_DUAL>(nt, p, s);
    case MODE_SDDMM: return launch_mode<MODE_SDDMM>(nt, p, s);
    case MODE_AGNN_FWD: return launch_mode<MODE_AGNN_FWD>(nt, p, s);
    default: return launch_mode<MODE_AGNN_BWD>(nt, p, s);
  }
}

}  // namespace win
}  // namespace tcg
