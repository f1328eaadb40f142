// The row-window engine: every TF32 tensor-core op of the hot path.
//
// One warp owns one 16-row window at a time (persistent grid, windows
// round-robin over warps) and runs the reference's tile dataflow
// (tiles.py:130-250, kernels.py:254-538, Alg. 2/3) out of shared
// memory:
//
//   1. FetchDense  — the window's condensed neighbour rows X[col_to_node[c]]
//      are gathered into shared memory with cp.async (16-B chunks, coalesced
//      per row), all rows of the window in flight at once. Row c of the
//      window is stored at smem row srow(c) = (c & ~7) | bitrev3(c & 7) with
//      the 16-B chunks XOR-swizzled by (srow & 7): with that placement both
//      fragment read patterns below (SpMM: rows t / chunks g; SDDMM: rows g /
//      chunks t) hit 32 distinct banks per phase.
//      While the gather is in flight the warp prefetches the NEXT window's
//      metadata and col_to_node slice (cross-window software pipeline) and
//      loads this window's edge_to_col / weights.
//   2. InitSparse  — edge weights are scattered into the 16x8 A tiles
//      directly in mma.m16n8k8 fragment order.
//   3. mma.sync.m16n8k8 TF32 (operands RNE-rounded by cvt.rn.tf32.f32, fp32
//      accumulate) for SpMM (B = staged rows, features permuted so each
//      lane's slice is contiguous) and for SDDMM (A = the window's own 16
//      rows, B = staged rows, k = features).
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
#include "common.cuh"
#include "window.cuh"

namespace tcg {
namespace win {

constexpr int kWarps = 4;

__device__ __forceinline__ int brev3(int x) { return ((x & 1) << 2) | (x & 2) | ((x >> 2) & 1); }
__device__ __forceinline__ int srow(int c) { return (c & ~7) | brev3(c & 7); }

__device__ __forceinline__ void cp_async16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(s)),
               "l"(g));
}
__device__ __forceinline__ void cp_async4(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(s)),
               "l"(g));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait_all() {
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

template <int NT>
struct Geo {
  static constexpr int DS = 8 * NT;                // staged row stride (floats)
  static constexpr int CH = DS / 4;                // 16-B chunks per row
  static constexpr int CHM = (CH < 8 ? CH : 8) - 1;  // swizzle mask
  __device__ static __forceinline__ int off(int s, int f) {
    return s * DS + ((((f >> 2) ^ (s & CHM)) << 2) | (f & 3));
  }
};

// smem carve per warp (bytes), shared with the host launcher
template <int NT, int MODE>
struct Carve {
  static constexpr bool kDual = MODE == MODE_SPMM_DUAL;
  static constexpr bool kFused = MODE == MODE_AGNN_FWD || MODE == MODE_AGNN_BWD;
  static constexpr int CPR = cols_per_round(NT, MODE);
  static constexpr int rps = 0;                                   // 2 x 17 int64
  static constexpr int nodes = 288;                               // CPR int
  static constexpr int xs = nodes + CPR * 4;                      // CPR x DS f32 (x2 dual)
  static constexpr int xs_bytes = CPR * 8 * NT * 4;
  static constexpr int frag = xs + xs_bytes * (kDual ? 2 : 1);    // A frags / score tile
  static constexpr int frag_bytes_a = (CPR / 8) * 512 * (kDual ? 2 : 1);
  static constexpr int tile_stride = CPR + 4;
  static constexpr int frag_bytes_t = kFused || MODE == MODE_SDDMM ? 16 * tile_stride * 4 : 0;
  static constexpr int frag_bytes = frag_bytes_a > frag_bytes_t ? frag_bytes_a : frag_bytes_t;
  static constexpr int edges = frag + frag_bytes;                 // fused: EPR f32 + 2 x EPR u8
  static constexpr int total = edges + (kFused ? kEdgesPerWindow * 6 : 0);
};

struct WinState {
  int64_t w;      // window id (absolute)
  int64_t c0, cend;
};

template <int NT, int MODE>
__global__ void __launch_bounds__(kWarps * 32) window_kernel(Params p) {
  using G = Geo<NT>;
  using CV = Carve<NT, MODE>;
  constexpr int CPR = CV::CPR;
  constexpr bool kDual = CV::kDual;
  constexpr bool kFused = CV::kFused;
  constexpr bool kSpmmPhase = MODE != MODE_SDDMM;
  constexpr bool kSddmmPhase = MODE == MODE_SDDMM || kFused;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  unsigned char* sm = smem_raw + warp * CV::total;
  int64_t* rps2 = reinterpret_cast<int64_t*>(sm + CV::rps);  // [2][17]
  int* nodes = reinterpret_cast<int*>(sm + CV::nodes);
  float* xs = reinterpret_cast<float*>(sm + CV::xs);
  float* xs2 = xs + CPR * G::DS;
  uint32_t* afrag = reinterpret_cast<uint32_t*>(sm + CV::frag);
  uint32_t* afrag2 = afrag + (CPR / 8) * 128;
  float* tile = reinterpret_cast<float*>(sm + CV::frag);
  float* escore = reinterpret_cast<float*>(sm + CV::edges);
  unsigned char* ecol = sm + CV::edges + kEdgesPerWindow * 4;
  unsigned char* erow = ecol + kEdgesPerWindow;

  // zero the staged rows once: feature padding [dim, DS) is never written
  for (int i = lane; i < CPR * G::DS * (kDual ? 2 : 1); i += 32) xs[i] = 0.f;

  const int64_t nwarps = (int64_t)gridDim.x * kWarps;
  const int64_t tasks = p.nwin * p.nchunks;
  int64_t task = (int64_t)blockIdx.x * kWarps + warp;
  const bool vec16 = p.vec16;

  // ---- prefetch registers for the next task ----
  int64_t pf_rp = 0, pf_c0 = 0, pf_cend = 0;
  int pf_node[CPR / 32];
  auto prefetch = [&](int64_t tk) {
    if (tk >= tasks) return;
    const int64_t w = p.win_begin + tk / p.nchunks;
    const int64_t r0 = w * 16;
    pf_rp = __ldg(p.ptr + min(r0 + min(lane, 16), p.n));
    if (lane > 16) pf_rp = 0;
    pf_c0 = __ldg(p.coff + w);
    pf_cend = __ldg(p.coff + w + 1);
    const int64_t u = pf_cend - pf_c0;
#pragma unroll
    for (int k = 0; k < CPR / 32; ++k) {
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
    const int64_t c0 = pf_c0, cend = pf_cend;
    const int u = (int)(cend - c0);
#pragma unroll
    for (int k = 0; k < CPR / 32; ++k) nodes[lane + 32 * k] = pf_node[k];
    __syncwarp();
    const int64_t e0 = rps[0], e1 = rps[16];
    const int E = (int)(e1 - e0);
    const int nrounds = kFused ? 1 : (u + CPR - 1) / CPR;

    float acc[NT][4];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;

    const int nkc = MODE == MODE_SDDMM ? p.nkc : 1;
    for (int rd = 0; rd < max(nrounds, 1); ++rd) {
      const int cb = rd * CPR;                 // first column of this round
      const int ncols = min(CPR, u - cb);      // may be <= 0 for empty windows
      if (rd > 0) {  // columns beyond the prefetched slice
        __syncwarp();
        for (int c = lane; c < ncols; c += 32) nodes[c] = (int)__ldg(p.c2n + c0 + cb + c);
        __syncwarp();
      }
      for (int kc = 0; kc < nkc; ++kc) {
      // SDDMM folds D in k-chunks of 8*NT features; SpMM modes use one chunk
      const int dk = MODE == MODE_SDDMM ? kc * 8 * NT : d0;
      const int dv = min(8 * NT, p.dim - dk);
      if (kc > 0) __syncwarp();  // previous chunk's fragment reads are done
      // ---- 1. FetchDense: stage rows of this round ----
      if (ncols > 0) {
        if (vec16) {
          constexpr int RPI = 32 / (G::CH < 32 ? G::CH : 32);  // rows per iteration
          const int ch = lane % G::CH;
          const int nch = (dv + 3) >> 2;
          for (int c = lane / G::CH; c < ncols; c += RPI) {
            const int64_t node = nodes[c];
            const int s = srow(c);
            if (ch < nch) {
              cp_async16(xs + G::off(s, ch * 4), p.x + node * p.ldx + dk + ch * 4);
              if (kDual) cp_async16(xs2 + G::off(s, ch * 4), p.x2 + node * p.ldx2 + dk + ch * 4);
            }
          }
        } else {
          for (int q = lane; q < ncols * G::DS; q += 32) {
            const int c = q / G::DS, f = q % G::DS;
            if (f < dv) {
              const int64_t node = nodes[c];
              const int s = srow(c);
              cp_async4(xs + G::off(s, f), p.x + node * p.ldx + dk + f);
              if (kDual) cp_async4(xs2 + G::off(s, f), p.x2 + node * p.ldx2 + dk + f);
            }
          }
        }
        cp_commit();
        // zero rows [ncols, pad16) so padded columns read as 0 (no stale NaN)
        const int pad = min(CPR, (ncols + 15) & ~15);
        for (int q = lane; q < (pad - ncols) * G::DS; q += 32) {
          const int c = ncols + q / G::DS, f = q % G::DS;
          xs[G::off(srow(c), f)] = 0.f;
          if (kDual) xs2[G::off(srow(c), f)] = 0.f;
        }
      }
      // ---- prefetch the next task's metadata + col_to_node (overlaps gather) ----
      if ((rd == nrounds - 1 || nrounds == 0) && kc == nkc - 1) prefetch(task + nwarps);

      // ---- 2. per-edge work while rows land ----
      if constexpr (kSpmmPhase && !kFused) {
        // InitSparse: weights -> fragment-ordered A tiles for blocks of this round
        const int nb = (max(ncols, 0) + 7) >> 3;
        for (int i = lane; i < nb * 32; i += 32) {
          reinterpret_cast<uint4*>(afrag)[i] = make_uint4(0, 0, 0, 0);
          if (kDual) reinterpret_cast<uint4*>(afrag2)[i] = make_uint4(0, 0, 0, 0);
        }
        __syncwarp();
        for (int64_t e = e0 + lane; e < e1; e += 32) {
          const int c = (int)__ldg(p.e2c + e) - cb;
          if (c < 0 || c >= ncols) continue;
          int row = 0;
#pragma unroll
          for (int s = 8; s > 0; s >>= 1)
            if (rps[row + s] <= e) row += s;
          const int k = c & 7;
          const int idx = (c >> 3) * 128 + (((row & 7) << 2) | (k & 3)) * 4 + (row >> 3) +
                          2 * (k >> 2);
          float wv = 1.f;
          if (p.w) wv = p.widx ? __ldg(p.w + __ldg(p.widx + e)) : __ldg(p.w + e);
          afrag[idx] = tf32_rn(wv);
          if (kDual) {
            float wv2 = 1.f;
            if (p.w2) wv2 = p.widx2 ? __ldg(p.w2 + __ldg(p.widx2 + e)) : __ldg(p.w2 + e);
            afrag2[idx] = tf32_rn(wv2);
          }
        }
      }
      if constexpr (kFused) {
        // edge -> (row, condensed col) bytes for the score / softmax / scatter phases
        for (int i = lane; i < E; i += 32) {
          const int64_t e = e0 + i;
          int row = 0;
#pragma unroll
          for (int s = 8; s > 0; s >>= 1)
            if (rps[row + s] <= e) row += s;
          erow[i] = (unsigned char)row;
          ecol[i] = (unsigned char)__ldg(p.e2c + e);
        }
      }
      // A operand of the SDDMM phase: the window's own rows, straight to registers
      float ar[4][NT];
      if constexpr (kSddmmPhase) {
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int64_t r = r0 + g + ((h & 1) ? 8 : 0);
          const int f0 = ((h & 2) ? (t + 4) : t) * NT;
          const float* src = p.xa + r * p.lda + dk + f0;
          bool done = false;
          if constexpr (NT % 4 == 0) {
            if (vec16 && r < r1 && f0 + NT <= dv) {
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
      cp_wait_all();
      __syncwarp();

      // ---- 3a. SDDMM phase: scores for 16-column paired blocks ----
      if constexpr (kSddmmPhase) {
        const int npb = (max(ncols, 0) + 15) >> 4;
        uint32_t a[4][NT];
#pragma unroll
        for (int h = 0; h < 4; ++h)
#pragma unroll
          for (int j = 0; j < NT; ++j) a[h][j] = tf32_rn(ar[h][j]);
        for (int sb = 0; sb < npb; ++sb) {
          float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int s = srow(sb * 16 + hh * 8 + g);
            float b0[NT], b1[NT];
#pragma unroll
            for (int j = 0; j < NT; ++j) {
              b0[j] = xs[G::off(s, t * NT + j)];
              b1[j] = xs[G::off(s, (t + 4) * NT + j)];
            }
#pragma unroll
            for (int j = 0; j < NT; ++j)
              mma_tf32(sc[hh], a[0][j], a[1][j], a[2][j], a[3][j], tf32_rn(b0[j]), tf32_rn(b1[j]));
          }
          // scores -> tile[row][col] (accumulated over k-chunks)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int col = sb * 16 + hh * 8 + 2 * t;
            float* t0 = tile + g * CV::tile_stride + col;
            float* t1 = tile + (g + 8) * CV::tile_stride + col;
            if (kc == 0) {
              t0[0] = sc[hh][0], t0[1] = sc[hh][1], t1[0] = sc[hh][2], t1[1] = sc[hh][3];
            } else {
              t0[0] += sc[hh][0], t0[1] += sc[hh][1], t1[0] += sc[hh][2], t1[1] += sc[hh][3];
            }
          }
        }
      }
      }  // k-chunks
      if constexpr (kSddmmPhase) {
        __syncwarp();
        if constexpr (MODE == MODE_SDDMM) {
          // StoreSparse: raw scores of this round's columns to edge order
          for (int64_t e = e0 + lane; e < e1; e += 32) {
            const int c = (int)__ldg(p.e2c + e) - cb;
            if (c < 0 || c >= ncols) continue;
            int row = 0;
#pragma unroll
            for (int s = 8; s > 0; s >>= 1)
              if (rps[row + s] <= e) row += s;
            p.eout[e] = tile[row * CV::tile_stride + c];
          }
          __syncwarp();
        } else {
          for (int i = lane; i < E; i += 32) escore[i] = tile[erow[i] * CV::tile_stride + ecol[i]];
          __syncwarp();
        }
      }

      // ---- 3b. fused epilogue between the two products ----
      if constexpr (kFused) {
        // 2 lanes per row: row softmax (fwd) or softmax backward (bwd)
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
          for (int i = rb + sub; i < re; i += 2) {
            const float pe = __ldg(p.aux + e0 + i);
            escore[i] = pe * (escore[i] - s);
          }
        }
        __syncwarp();
        for (int i = lane; i < E; i += 32) p.eout[e0 + i] = escore[i];
        // InitSparse from the fresh weights (frag buffer reused after the tile)
        const int nb = (u + 7) >> 3;
        for (int i = lane; i < nb * 32; i += 32)
          reinterpret_cast<uint4*>(afrag)[i] = make_uint4(0, 0, 0, 0);
        __syncwarp();
        for (int i = lane; i < E; i += 32) {
          const int row_e = erow[i], c = ecol[i], k = c & 7;
          const int idx = (c >> 3) * 128 + (((row_e & 7) << 2) | (k & 3)) * 4 + (row_e >> 3) +
                          2 * (k >> 2);
          afrag[idx] = tf32_rn(escore[i]);
        }
        __syncwarp();
      } else if constexpr (kSpmmPhase) {
        __syncwarp();
      }

      // ---- 3c. SpMM phase over the 16x8 blocks of this round ----
      if constexpr (kSpmmPhase) {
        const int nb = (max(ncols, 0) + 7) >> 3;
        constexpr int V = NT < 4 ? NT : 4;
        for (int b = 0; b < nb; ++b) {
          const uint4 af = reinterpret_cast<const uint4*>(afrag)[b * 32 + lane];
          const int s0 = srow(b * 8 + t), s1 = srow(b * 8 + t + 4);
          float x0[NT], x1[NT];
#pragma unroll
          for (int q = 0; q < NT; q += V) {
            if constexpr (V == 4) {
              const float4 u0 = *reinterpret_cast<const float4*>(xs + G::off(s0, g * NT + q));
              const float4 u1 = *reinterpret_cast<const float4*>(xs + G::off(s1, g * NT + q));
              x0[q] = u0.x, x0[q + 1] = u0.y, x0[q + 2] = u0.z, x0[q + 3] = u0.w;
              x1[q] = u1.x, x1[q + 1] = u1.y, x1[q + 2] = u1.z, x1[q + 3] = u1.w;
            } else if constexpr (V == 2) {
              const float2 u0 = *reinterpret_cast<const float2*>(xs + G::off(s0, g * NT + q));
              const float2 u1 = *reinterpret_cast<const float2*>(xs + G::off(s1, g * NT + q));
              x0[q] = u0.x, x0[q + 1] = u0.y;
              x1[q] = u1.x, x1[q + 1] = u1.y;
            } else {
              x0[q] = xs[G::off(s0, g * NT + q)];
              x1[q] = xs[G::off(s1, g * NT + q)];
            }
          }
#pragma unroll
          for (int j = 0; j < NT; ++j)
            mma_tf32(acc[j], af.x, af.y, af.z, af.w, tf32_rn(x0[j]), tf32_rn(x1[j]));
          if constexpr (kDual) {
            const uint4 af2 = reinterpret_cast<const uint4*>(afrag2)[b * 32 + lane];
#pragma unroll
            for (int q = 0; q < NT; q += V) {
#pragma unroll
              for (int v = 0; v < V; ++v) {
                x0[q + v] = xs2[G::off(s0, g * NT + q + v)];
                x1[q + v] = xs2[G::off(s1, g * NT + q + v)];
              }
            }
#pragma unroll
            for (int j = 0; j < NT; ++j)
              mma_tf32(acc[j], af2.x, af2.y, af2.z, af2.w, tf32_rn(x0[j]), tf32_rn(x1[j]));
          }
        }
      }
      __syncwarp();
    }  // rounds

    // ---- 4. epilogues after all rounds ----
    if constexpr (MODE == MODE_SDDMM) {
      if (p.epilogue != 0) {
        // rows of this window: 2 lanes per row over the scores in eout
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

template <int NT, int MODE>
int launch_nt(const Params& p, cudaStream_t s) {
  using CV = Carve<NT, MODE>;
  const size_t smem = (size_t)CV::total * kWarps;
  auto kern = window_kernel<NT, MODE>;
  static int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    TCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
             "window_kernel attr");
    configured_dev = dev;
  }
  int per_sm = 0;
  TCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarps * 32, smem),
           "window_kernel occupancy");
  if (per_sm < 1) per_sm = 1;
  const int64_t tasks = p.nwin * p.nchunks;
  int64_t blocks = (tasks + kWarps - 1) / kWarps;
  const int64_t cap = (int64_t)num_sms() * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) return TCG_OK;
  kern<<<(unsigned)blocks, kWarps * 32, smem, s>>>(p);
  TCG_LAUNCHED("window_kernel");
  return TCG_OK;
}

template <int MODE>
int launch_mode(int nt, const Params& p, cudaStream_t s) {
  switch (nt) {
    case 1: return launch_nt<1, MODE>(p, s);
    case 2: return launch_nt<2, MODE>(p, s);
    case 4: return launch_nt<4, MODE>(p, s);
    default: return launch_nt<8, MODE>(p, s);
  }
}

int launch(int mode, int nt, const Params& p, cudaStream_t s) {
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
