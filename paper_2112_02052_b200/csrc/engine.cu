// The row-window engine: every TF32 tensor-core op of the hot path.
//
// One warp owns one 16-row window at a time (persistent grid of 16 warps per
// SM, windows round-robin over warps) and runs the reference's tile
// dataflow (tiles.py:130-250, kernels.py:254-538, Alg. 2/3):
//
//   * FetchDense — the window's condensed neighbour rows X[col_to_node[c]]
//     are read straight into mma B fragments with 16-B vector loads (8 lanes
//     cover one 128-B row, so every load instruction moves whole L2
//     sectors). The feature dimension is permuted per lane (SpMM: lane g
//     owns features [g*NT, g*NT+NT); SDDMM: k-step j of lane t reads feature
//     t*NT+j) so each lane's slice is contiguous; the output permutation is
//     undone in the epilogue. Loads run LOOK blocks ahead of the MMAs; the
//     col_to_node slice of the next window is prefetched while the current
//     one computes. No shared-memory staging: 16 warps per SM provide the
//     memory-level parallelism (ncu showed staged variants were bound by
//     per-window issue latency at 4-8 warps/SM).
//   * InitSparse — edge weights are scattered into the 16x8 A tiles in
//     mma.m16n8k8 fragment order through the per-edge fragment slot `efrag`
//     (computed once per tiling, the analogue of the reference's per-edge
//     `_spmm_aux` cache, kernels.py:173-188).
//   * mma.sync.m16n8k8 TF32 (operands RNE-rounded by cvt.rn.tf32.f32, fp32
//     accumulate).
//   * Epilogues: StoreDense (bias / accumulate, vector stores), StoreSparse
//     (score tile -> edge order), row softmax / softmax backward (rows never
//     straddle windows; 2 lanes per row).
//
// Modes:
//   SPMM       Y = A_w X (+bias) (+=)                 reference spmm
//   SPMM_DUAL  Y += A_w1 X1 + A_w2 X2 (A^T pass of the AGNN backward)
//   SDDMM      s_e = <XA_row, X_col> (+ softmax / softmax-bwd epilogue)
//   AGNN_FWD   P = softmax(<Z_i,Z_j>), Y = A_P Z     reference agnn_layer
//   AGNN_BWD   dS = P (dP - rowsum(P dP)), dP = <G_i,Z_j>; Y = A_dS Z
//   (the fused modes read the window's neighbour rows for the SDDMM and
//    again for the SpMM; the second read hits L1)
#include "common.cuh"
#include "window.cuh"

namespace tcg {
namespace win {

constexpr int kWarps = 4;

template <int NT, int MODE>
struct Carve {
  static constexpr bool kDual = MODE == MODE_SPMM_DUAL;
  static constexpr bool kFused = MODE == MODE_AGNN_FWD || MODE == MODE_AGNN_BWD;
  static constexpr int CPR = cols_per_round(NT, MODE);
  static constexpr int tile_stride = CPR + 4;
  static constexpr int frag = 0;
  static constexpr int frag_a = (CPR / 8) * 512 * (kDual ? 2 : 1);
  static constexpr int frag_t = (kFused || MODE == MODE_SDDMM) ? 16 * tile_stride * 4 : 0;
  static constexpr int frag_bytes = frag_a > frag_t ? frag_a : frag_t;
  static constexpr int edges = frag + frag_bytes;
  static constexpr int rps = edges + (kFused ? kEdgesPerWindow * 4 : 0);  // 17 int64
  static constexpr int total = (rps + 136 + 127) & ~127;
};

// efrag slot -> (row within window, column within the round)
__device__ __forceinline__ void decode_slot(int fi, int& row, int& col) {
  const int ln = (fi >> 2) & 31, sl = fi & 3;
  row = (ln >> 2) + 8 * (sl & 1);
  col = (fi >> 7) * 8 + (ln & 3) + 4 * (sl >> 1);
}

// NT consecutive floats of row `node` starting at feature f0 (0 if node < 0
// or past dim). FULL: dim is a multiple of the chunk width and rows are
// 16-B aligned, so the loads are unconditional vectors (no per-load
// branches); an absent node reads row 0 and is zeroed by a select.
template <int NT, bool FULL>
__device__ __forceinline__ void load_slice(float (&v)[NT], const float* __restrict__ x, int node,
                                           int64_t ld, int f0, int dim) {
  const bool ok = node >= 0;
  const float* src = x + (int64_t)(ok ? node : 0) * ld + f0;
  if constexpr (FULL && NT % 4 == 0) {
#pragma unroll
    for (int j = 0; j < NT; j += 4) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(src + j));
      v[j] = q.x, v[j + 1] = q.y, v[j + 2] = q.z, v[j + 3] = q.w;
    }
  } else if constexpr (FULL && NT == 2) {
    const float2 q = __ldg(reinterpret_cast<const float2*>(src));
    v[0] = q.x, v[1] = q.y;
  } else if constexpr (FULL) {
    v[0] = __ldg(src);
  } else {
#pragma unroll
    for (int j = 0; j < NT; ++j) v[j] = (ok && f0 + j < dim) ? __ldg(src + j) : 0.f;
  }
  if constexpr (FULL) {
#pragma unroll
    for (int j = 0; j < NT; ++j) v[j] = ok ? v[j] : 0.f;
  }
}

template <int NT, int MODE, bool FULL>
__global__ void __launch_bounds__(kWarps * 32, NT >= 8 ? 2
                                                : (NT == 4 && MODE != MODE_SPMM &&
                                                   MODE != MODE_SDDMM) ? 3 : 4)
    window_kernel(const Params p) {
  using CV = Carve<NT, MODE>;
  constexpr int CPR = CV::CPR;
  constexpr int NPF = CPR / 32;   // col_to_node registers per lane
  constexpr int NB = CPR / 8;     // 16x8 blocks per round
  constexpr int NPB = CPR / 16;   // paired 16x16 blocks per round
  constexpr int LOOK = 4;         // SpMM blocks in flight ahead of the MMAs
  constexpr bool kDual = CV::kDual;
  constexpr bool kFused = CV::kFused;
  constexpr bool kSpmmPhase = MODE != MODE_SDDMM;
  constexpr bool kSddmmPhase = MODE == MODE_SDDMM || kFused;
  constexpr int TS = CV::tile_stride;
  constexpr int EV = kFused ? kEdgesPerWindow / 32 : 4;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  unsigned char* sm = smem_raw + warp * CV::total;
  uint32_t* afrag = reinterpret_cast<uint32_t*>(sm + CV::frag);
  uint32_t* afrag2 = afrag + NB * 128;
  float* tile = reinterpret_cast<float*>(sm + CV::frag);
  float* escore = reinterpret_cast<float*>(sm + CV::edges);
  int64_t* rps = reinterpret_cast<int64_t*>(sm + CV::rps);

  const int64_t nwarps = (int64_t)gridDim.x * kWarps;
  const int64_t tasks = p.nwin * p.nchunks;

  // next-window prefetch (metadata, then its col_to_node slice)
  auto meta_of = [&](int64_t tk, int64_t& rp, int64_t& c0, int64_t& ce) {
    if (tk >= tasks) {
      rp = 0, c0 = 0, ce = 0;
      return;
    }
    const int64_t w = p.win_begin + tk / p.nchunks;
    rp = lane <= 16 ? __ldg(p.ptr + min(w * 16 + lane, p.n)) : 0;
    c0 = __ldg(p.coff + w);
    ce = __ldg(p.coff + w + 1);
  };
  auto nodes_of = [&](int64_t c0, int64_t ce, int cb, int (&nd)[NPF]) {
#pragma unroll
    for (int k = 0; k < NPF; ++k) {
      const int64_t c = c0 + cb + lane + 32 * k;
      nd[k] = c < ce ? (int)__ldg(p.c2n + c) : -1;
    }
  };

  int64_t task = (int64_t)blockIdx.x * kWarps + warp;
  int64_t rp_n, c0_n, ce_n;
  meta_of(task, rp_n, c0_n, ce_n);
  int nd_n[NPF];
  nodes_of(c0_n, ce_n, 0, nd_n);

  for (; task < tasks; task += nwarps) {
    const int64_t w = p.win_begin + task / p.nchunks;
    const int d0 = (int)(task % p.nchunks) * 8 * NT;
    const int64_t r0 = w * 16, r1 = min(r0 + 16, p.n);
    const int64_t c0 = c0_n;
    const int u = (int)(ce_n - c0_n);
    __syncwarp();
    if (lane <= 16) rps[lane] = rp_n;
    int nd[NPF];
#pragma unroll
    for (int k = 0; k < NPF; ++k) nd[k] = nd_n[k];
    __syncwarp();
    const int64_t e0 = rps[0], e1 = rps[16];
    const int E = (int)(e1 - e0);
    // prefetch the next window's metadata now; its nodes after this one's loads
    meta_of(task + nwarps, rp_n, c0_n, ce_n);
    const int nrounds = kFused ? 1 : (u + CPR - 1) / CPR;

    // edge data of the fused modes (E <= 256 guaranteed by the host)
    uint32_t efr[kFused ? EV : 1];
    float pa[MODE == MODE_AGNN_BWD ? EV : 1];
    if constexpr (kFused) {
#pragma unroll
      for (int v = 0; v < EV; ++v) {
        const int i = lane + 32 * v;
        efr[v] = i < E ? __ldg(p.efrag + e0 + i) : 0u;
        if constexpr (MODE == MODE_AGNN_BWD) pa[v] = i < E ? __ldg(p.aux + e0 + i) : 0.f;
      }
    }

    float acc[NT][4];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;

    for (int rd = 0; rd < max(nrounds, 1); ++rd) {
      const int cb = rd * CPR;
      const int ncols = max(0, min(CPR, u - cb));
      const int nb = (ncols + 7) >> 3, npb = (ncols + 15) >> 4;
      if (rd > 0) nodes_of(c0, c0 + u, cb, nd);
      const int fbase = cb * 16, flim = nb * 128;  // efrag slots of this round

      // ================= SDDMM phase =================
      if constexpr (kSddmmPhase) {
        const int nkc = MODE == MODE_SDDMM ? p.nkc : 1;
        for (int kc = 0; kc < nkc; ++kc) {
          const int dk = kc * 8 * NT;
          // A operand: the window's own rows (features permuted: k-step j of
          // lane t reads feature t*NT + j, the +4 half (t+4)*NT + j)
          uint32_t a[4][NT];
          {
            float ar[4][NT];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const int64_t r = r0 + g + ((h & 1) ? 8 : 0);
              const int f0 = dk + ((h & 2) ? (t + 4) : t) * NT;
              load_slice<NT, FULL>(ar[h], p.xa, r < r1 ? (int)r : -1, p.lda, f0, p.dim);
            }
#pragma unroll
            for (int h = 0; h < 4; ++h)
#pragma unroll
              for (int j = 0; j < NT; ++j) a[h][j] = tf32_rn(ar[h][j]);
          }
          float* trow0 = tile + g * TS + 2 * t;
          float* trow1 = tile + (g + 8) * TS + 2 * t;
          // paired blocks, one ahead
          float bq[2][4][NT];
          auto issue_pb = [&](int sb, int slot) {
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const int col = sb * 16 + hh * 8 + g;
              const int node = __shfl_sync(0xffffffffu, nd[(sb * 16) >> 5], col & 31);
              load_slice<NT, FULL>(bq[slot][2 * hh], p.x, node, p.ldx, dk + t * NT, p.dim);
              load_slice<NT, FULL>(bq[slot][2 * hh + 1], p.x, node, p.ldx, dk + (t + 4) * NT,
                                   p.dim);
            }
          };
#pragma unroll
          for (int sb = 0; sb < NPB; ++sb) {
            if (sb >= npb) break;
            if (sb == 0) issue_pb(0, 0);
            if (sb + 1 < npb) issue_pb(sb + 1, (sb + 1) & 1);
            float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
            for (int hh = 0; hh < 2; ++hh)
#pragma unroll
              for (int j = 0; j < NT; ++j)
                mma_tf32(sc[hh], a[0][j], a[1][j], a[2][j], a[3][j],
                         tf32_rn(bq[sb & 1][2 * hh][j]), tf32_rn(bq[sb & 1][2 * hh + 1][j]));
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              float2* q0 = reinterpret_cast<float2*>(trow0 + sb * 16 + hh * 8);
              float2* q1 = reinterpret_cast<float2*>(trow1 + sb * 16 + hh * 8);
              if (kc == 0) {
                *q0 = make_float2(sc[hh][0], sc[hh][1]);
                *q1 = make_float2(sc[hh][2], sc[hh][3]);
              } else {
                const float2 o0 = *q0, o1 = *q1;
                *q0 = make_float2(o0.x + sc[hh][0], o0.y + sc[hh][1]);
                *q1 = make_float2(o1.x + sc[hh][2], o1.y + sc[hh][3]);
              }
            }
          }
        }
        __syncwarp();
        if constexpr (MODE == MODE_SDDMM) {
          // StoreSparse: raw scores of this round's columns to edge order
          for (int64_t e = e0 + lane; e < e1; e += 32) {
            const int fi = (int)__ldg(p.efrag + e) - fbase;
            if (fi < 0 || fi >= flim) continue;
            int row, col;
            decode_slot(fi, row, col);
            p.eout[e] = tile[row * TS + col];
          }
          __syncwarp();
        } else {
          // scores -> edge order, row softmax (fwd) / softmax bwd, -> A tiles
#pragma unroll
          for (int v = 0; v < EV; ++v) {
            const int i = lane + 32 * v;
            if (i < E) {
              int row, col;
              decode_slot((int)efr[v], row, col);
              const float s = tile[row * TS + col];
              escore[i] = MODE == MODE_AGNN_BWD ? pa[v] * s : s;
            }
          }
          __syncwarp();
          const int row = lane >> 1, sub = lane & 1;
          const int rb = (int)(rps[row] - e0), re = (int)(rps[row + 1] - e0);
          if constexpr (MODE == MODE_AGNN_FWD) {
            float mx = -INFINITY;
            for (int i = rb + sub; i < re; i += 2) mx = fmaxf(mx, escore[i]);
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            float s = 0.f;
            for (int i = rb + sub; i < re; i += 2) s += expf(escore[i] - mx);
            s += __shfl_xor_sync(0xffffffffu, s, 1);
            for (int i = rb + sub; i < re; i += 2) escore[i] = expf(escore[i] - mx) / s;
          } else {
            float s = 0.f;  // rowsum(P dP); escore holds P*dP
            for (int i = rb + sub; i < re; i += 2) s += escore[i];
            s += __shfl_xor_sync(0xffffffffu, s, 1);
            __syncwarp();
            for (int i = rb + sub; i < re; i += 2) escore[i] = s;  // row sum per edge
          }
          __syncwarp();
          // A tiles from the fresh weights (tile region reused after the scores)
          float wv[EV];
#pragma unroll
          for (int v = 0; v < EV; ++v) {
            const int i = lane + 32 * v;
            wv[v] = 0.f;
            if (i < E) {
              if constexpr (MODE == MODE_AGNN_FWD) {
                wv[v] = escore[i];
              } else {
                int rw, cl;
                decode_slot((int)efr[v], rw, cl);
                wv[v] = pa[v] * (tile[rw * TS + cl] - escore[i]);  // dS = P (dP - rowsum)
              }
            }
          }
          __syncwarp();
          for (int i = lane; i < nb * 32; i += 32)
            reinterpret_cast<uint4*>(afrag)[i] = make_uint4(0, 0, 0, 0);
          __syncwarp();
#pragma unroll
          for (int v = 0; v < EV; ++v) {
            const int i = lane + 32 * v;
            if (i < E) {
              p.eout[e0 + i] = wv[v];
              afrag[efr[v]] = tf32_rn(wv[v]);
            }
          }
          __syncwarp();
        }
      }

      // ================= SpMM phase =================
      if constexpr (kSpmmPhase) {
        // B fragments LOOK blocks ahead: lane (g,t) reads neighbours t, t+4
        // of each 8-column block, features [d0 + g*NT, +NT)
        float xq[LOOK][kDual ? 4 : 2][NT];
        auto issue_b = [&](int b, int slot) {
          const int k = (b * 8) >> 5;
          const int n0 = __shfl_sync(0xffffffffu, nd[k], (b * 8 + t) & 31);
          const int n1 = __shfl_sync(0xffffffffu, nd[k], (b * 8 + t + 4) & 31);
          load_slice<NT, FULL>(xq[slot][0], p.x, n0, p.ldx, d0 + g * NT, p.dim);
          load_slice<NT, FULL>(xq[slot][1], p.x, n1, p.ldx, d0 + g * NT, p.dim);
          if constexpr (kDual) {
            load_slice<NT, FULL>(xq[slot][2], p.x2, n0, p.ldx2, d0 + g * NT, p.dim);
            load_slice<NT, FULL>(xq[slot][3], p.x2, n1, p.ldx2, d0 + g * NT, p.dim);
          }
        };
#pragma unroll
        for (int b = 0; b < LOOK; ++b)
          if (b < nb) issue_b(b, b);
        if constexpr (!kFused) {
          // InitSparse while the rows are in flight
          for (int i = lane; i < nb * 32; i += 32) {
            reinterpret_cast<uint4*>(afrag)[i] = make_uint4(0, 0, 0, 0);
            if (kDual) reinterpret_cast<uint4*>(afrag2)[i] = make_uint4(0, 0, 0, 0);
          }
          __syncwarp();
          for (int64_t eb = e0; eb < e1; eb += 128) {
            int fi[4];
            float wa[4], wb[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const int64_t e = eb + lane + 32 * v;
              const bool ok = e < e1;
              fi[v] = ok ? (int)__ldg(p.efrag + e) - fbase : -1;
              wa[v] = 1.f;
              wb[v] = 1.f;
              if (ok && p.w) wa[v] = p.widx ? __ldg(p.w + __ldg(p.widx + e)) : __ldg(p.w + e);
              if (kDual && ok && p.w2)
                wb[v] = p.widx2 ? __ldg(p.w2 + __ldg(p.widx2 + e)) : __ldg(p.w2 + e);
            }
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              if (fi[v] >= 0 && fi[v] < flim) {
                afrag[fi[v]] = tf32_rn(wa[v]);
                if (kDual) afrag2[fi[v]] = tf32_rn(wb[v]);
              }
            }
          }
          __syncwarp();
        }
        if (rd == nrounds - 1 || nrounds == 0) nodes_of(c0_n, ce_n, 0, nd_n);  // next window
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          if (b >= nb) break;
          const int slot = b % LOOK;
          const uint4 af = reinterpret_cast<const uint4*>(afrag)[b * 32 + lane];
#pragma unroll
          for (int j = 0; j < NT; ++j)
            mma_tf32(acc[j], af.x, af.y, af.z, af.w, tf32_rn(xq[slot][0][j]),
                     tf32_rn(xq[slot][1][j]));
          if constexpr (kDual) {
            const uint4 af2 = reinterpret_cast<const uint4*>(afrag2)[b * 32 + lane];
#pragma unroll
            for (int j = 0; j < NT; ++j)
              mma_tf32(acc[j], af2.x, af2.y, af2.z, af2.w, tf32_rn(xq[slot][2][j]),
                       tf32_rn(xq[slot][3][j]));
          }
          if (b + LOOK < nb) issue_b(b + LOOK, slot);
        }
      } else {
        if (rd == nrounds - 1 || nrounds == 0) nodes_of(c0_n, ce_n, 0, nd_n);
      }
      __syncwarp();
    }  // rounds

    // ================= epilogues =================
    if constexpr (MODE == MODE_SDDMM) {
      if (p.epilogue != 0) {
        const int row = lane >> 1, sub = lane & 1;
        const int64_t rb = rps[row], re = rps[row + 1];
        if (p.epilogue == 1) {
          float mx = -INFINITY;
          for (int64_t i = rb + sub; i < re; i += 2) mx = fmaxf(mx, p.eout[i]);
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
          float s = 0.f;
          for (int64_t i = rb + sub; i < re; i += 2) s += expf(p.eout[i] - mx);
          s += __shfl_xor_sync(0xffffffffu, s, 1);
          for (int64_t i = rb + sub; i < re; i += 2) p.eout[i] = expf(p.eout[i] - mx) / s;
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

int edge_frag(const int64_t* ptr, const uint32_t* e2c, int64_t n, uint32_t* efrag,
              cudaStream_t s) {
  if (n == 0) return TCG_OK;
  edge_frag_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(ptr, e2c, n, efrag);
  TCG_LAUNCHED("edge_frag");
  return TCG_OK;
}

template <int NT, int MODE, bool FULL>
int launch_full(Params& p, cudaStream_t s) {
  using CV = Carve<NT, MODE>;
  const size_t smem = (size_t)CV::total * kWarps;
  auto kern = window_kernel<NT, MODE, FULL>;
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
  p.use_tma = 0;
  const int64_t tasks = p.nwin * p.nchunks;
  int64_t blocks = (tasks + kWarps - 1) / kWarps;
  const int64_t cap = (int64_t)num_sms() * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) return TCG_OK;
  kern<<<(unsigned)blocks, kWarps * 32, smem, s>>>(p);
  TCG_LAUNCHED("window_kernel");
  return TCG_OK;
}

template <int NT, int MODE>
int launch_nt(Params& p, cudaStream_t s) {
  // FULL: every feature chunk is complete and rows are 16-B aligned (the
  // caller's vec16 covers x, x2 and xa) -> branch-free vector loads
  const bool full = p.vec16 && p.dim % (8 * NT) == 0;
  return full ? launch_full<NT, MODE, true>(p, s) : launch_full<NT, MODE, false>(p, s);
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
