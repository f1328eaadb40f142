// The row-window engine: every TF32 tensor-core op of the hot path.
//
// Warp-specialised, persistent: per CTA kStages (producer warp, consumer
// warp) pairs, pair s owning shared-memory stage s; one stage holds one
// 16-row window (reference tile dataflow: tiles.py:130-250,
// kernels.py:254-538, Alg. 2/3); task i of the CTA goes to pair
// i % kStages:
//
//   producer (FetchDense): for window w, its condensed neighbour rows
//     X[col_to_node[c]] (8 lanes per 128-B row, cp.async 16 B, so each warp
//     instruction moves whole L2 sectors), the window's own 16 rows (SDDMM A
//     operand), and the window's edge data (fragment slot `efrag`, weights /
//     P) are copied into the stage with cp.async; completion is tracked by
//     cp.async.mbarrier.arrive.noinc on the stage's `full` mbarrier, so the
//     producer never waits for data and runs up to kStages windows ahead —
//     ~100+ KB of gathers in flight per SM, which the L2-latency-bound
//     gather needs (ncu: register-direct / single-buffer variants stalled on
//     long scoreboard at 15-30% issue). Metadata and col_to_node slices are
//     prefetched one / two windows ahead in producer registers.
//   consumer: waits on `full`, scatters the weights into the 16x8 A tiles in
//     mma.m16n8k8 fragment order (InitSparse via `efrag`, the analogue of
//     the reference's per-edge `_spmm_aux` cache, kernels.py:173-188), runs
//     mma.sync.m16n8k8 TF32 (cvt.rn.tf32 operands, fp32 accumulate) out of
//     shared memory, releases the stage (`empty` mbarrier) and writes the
//     epilogue (StoreDense / StoreSparse / row softmax).
//
// Staged rows: condensed column c lives at smem row srow(c) = (c & ~7) |
// bitrev3(c & 7) with 16-B chunks XOR-swizzled by (srow & 7); with that
// placement both fragment read patterns (SpMM: rows t / chunks g; SDDMM:
// rows g / chunks t) are bank-conflict free for 128-B rows.
//
// Modes:
//   SPMM       Y = A_w X (+bias) (+=)                 reference spmm
//   SPMM_DUAL  Y += A_w1 X1 + A_w2 X2 (A^T pass of the AGNN backward)
//   SDDMM      s_e = <XA_row, X_col> (+ softmax / softmax-bwd epilogue)
//   AGNN_FWD   P = softmax(<Z_i,Z_j>), Y = A_P Z     reference agnn_layer:
//              one staged copy of Z's neighbour rows serves both products
//   AGNN_BWD   dS = P (dP - rowsum(P dP)), dP = <G_i,Z_j>; Y = A_dS Z
// Windows with more condensed columns than one stage holds (or more edges
// than the stage's edge slots) finish the excess with direct global loads.
#include "common.cuh"
#include "window.cuh"

namespace tcg {
namespace win {

// producer warps per CTA = stages per CTA (one stage each, as many as fit)

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
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cp_async(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar))
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

template <int NT>
struct Geo {
  static constexpr int DS = 8 * NT;                  // features per staged row
  static constexpr int CH = DS / 4;                  // 16-B chunks per row
  static constexpr int CHM = (CH < 8 ? CH : 8) - 1;  // swizzle mask
  static constexpr int V = NT < 4 ? NT : 4;          // fragment read vector width
  __host__ __device__ static constexpr int off(int s, int f) {
    return s * DS + ((((f >> 2) ^ (s & CHM)) << 2) | (f & 3));
  }
};

template <int NT, int MODE>
struct Layout {
  static constexpr bool kDual = MODE == MODE_SPMM_DUAL;
  static constexpr bool kFused = MODE == MODE_AGNN_FWD || MODE == MODE_AGNN_BWD;
  static constexpr bool kSddmm = MODE == MODE_SDDMM || kFused;
  static constexpr int CPR = cols_per_round(NT, MODE);
  static constexpr int DS = 8 * NT;
  static constexpr int EPR = kEdgesPerWindow;  // staged edges per window
  // ---- one stage ----
  static constexpr int s_xs = 0;
  static constexpr int s_xs_bytes = CPR * DS * 4 * (kDual ? 2 : 1);
  static constexpr int s_xa = s_xs + s_xs_bytes;
  static constexpr int s_xa_bytes = kSddmm ? 16 * DS * 4 : 0;
  static constexpr int s_ef = s_xa + s_xa_bytes;
  static constexpr int s_wa = s_ef + EPR * 4;
  static constexpr int s_wb = s_wa + EPR * 4;
  static constexpr int s_hdr = s_wb + (kDual ? EPR * 4 : 0);  // rps[17] i64, w i64, u, E
  static constexpr int stage = (s_hdr + 17 * 8 + 8 + 8 + 127) & ~127;
  // ---- per consumer ----
  static constexpr int tile_stride = CPR + 4;
  static constexpr int c_frag_a = (CPR / 8) * 512 * (kDual ? 2 : 1);
  static constexpr int c_frag_t = kSddmm ? 16 * tile_stride * 4 : 0;
  static constexpr int c_frag = c_frag_a > c_frag_t ? c_frag_a : c_frag_t;
  static constexpr int c_esc = c_frag;
  static constexpr int cons = (c_esc + (kFused ? EPR * 4 : 0) + 127) & ~127;
  // ---- pipeline pairs: stage s is filled only by producer warp s and drained
  // only by consumer warp kStages + s (so mbarrier phases never alias across
  // warps); as many pairs as fit (<= 8, >= 2) ----
  static constexpr int budget = 220 * 1024;
  static constexpr int fit = (budget - 256) / (stage + cons);
  static constexpr int kStages = fit > 8 ? 8 : fit;
  static_assert(fit >= 2, "stages do not fit in shared memory");
  static constexpr int kProd = kStages;
  static constexpr int kCons = kStages;
  static constexpr int kThreads = (kCons + kProd) * 32;
  static constexpr int bars = kStages * stage + kCons * cons;
  static constexpr int total = bars + 2 * kStages * 8;
};

__device__ __forceinline__ void decode_slot(int fi, int& row, int& col) {
  const int ln = (fi >> 2) & 31, sl = fi & 3;
  row = (ln >> 2) + 8 * (sl & 1);
  col = (fi >> 7) * 8 + (ln & 3) + 4 * (sl >> 1);
}

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

// NT floats of row `node` from feature f0 (0 if node < 0 or past dim)
template <int NT>
__device__ __forceinline__ void load_slice(float (&v)[NT], const float* __restrict__ x, int node,
                                           int64_t ld, int f0, int dim) {
#pragma unroll
  for (int j = 0; j < NT; ++j)
    v[j] = (node >= 0 && f0 + j < dim) ? __ldg(x + (int64_t)node * ld + f0 + j) : 0.f;
}

template <int NT, int MODE, bool FULL>
__global__ void __launch_bounds__(Layout<NT, MODE>::kThreads, 1) window_kernel(const Params p) {
  using G = Geo<NT>;
  using L = Layout<NT, MODE>;
  constexpr int CPR = L::CPR;
  constexpr int DS = G::DS;
  constexpr int V = G::V;
  constexpr int NQ = NT / V;
  constexpr int NPF = CPR / 32;
  constexpr int EPR = L::EPR;
  constexpr int S = L::kStages;
  constexpr bool kDual = L::kDual;
  constexpr bool kFused = L::kFused;
  constexpr bool kSddmmPhase = L::kSddmm;
  constexpr bool kSpmmPhase = MODE != MODE_SDDMM;
  constexpr int TS = L::tile_stride;
  constexpr int XS2 = CPR * DS;
  constexpr int kProd = L::kProd;
  constexpr int kCons = L::kCons;
  constexpr int kThreads = L::kThreads;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::bars);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // zero every stage once: padding features [dim, DS) are never copied
  for (int i = threadIdx.x; i < S * L::stage / 4; i += kThreads)
    reinterpret_cast<float*>(smem)[i] = 0.f;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 64);  // 32 cp.async arrivals + 32 producer arrivals
      mbar_init(empty + s, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  __syncthreads();

  const int64_t tasks = p.nwin * p.nchunks;
  const int64_t tstep = gridDim.x;

  if (warp < kProd) {
    // ============================ producer ============================
    constexpr int RPI = 32 / G::CH;  // rows per staging instruction (16-B path)
    constexpr int IPK = 32 / RPI;
    const int ch = lane % G::CH, rsub = lane / G::CH;
    int soff[IPK];  // smem offset of (row RPI*i + rsub, chunk ch) inside a 32-row group
#pragma unroll
    for (int i = 0; i < IPK; ++i) soff[i] = G::off(srow(RPI * i + rsub), ch * 4);
    auto meta_of = [&](int64_t tk, int64_t& rp, int64_t& c0, int64_t& ce) {
      if (tk >= tasks) {
        rp = c0 = ce = 0;
        return;
      }
      const int64_t w = p.win_begin + tk / p.nchunks;
      rp = lane <= 16 ? __ldg(p.ptr + min(w * 16 + lane, p.n)) : 0;
      c0 = __ldg(p.coff + w);
      ce = __ldg(p.coff + w + 1);
    };
    auto nodes_of = [&](int64_t c0, int64_t ce, int (&nd)[NPF]) {
#pragma unroll
      for (int k = 0; k < NPF; ++k) {
        const int64_t c = c0 + lane + 32 * k;
        nd[k] = c < ce ? (int)__ldg(p.c2n + c) : -1;
      }
    };
    // register rings: metadata PD tasks ahead, col_to_node slices NA ahead,
    // so the producer never waits on its own index loads
    constexpr int PD = 3, NA = 2;
    const int64_t pstep = kProd * tstep;
    int64_t tk = blockIdx.x + warp * tstep;
    int64_t m_rp[PD], m_c0[PD], m_ce[PD];
#pragma unroll
    for (int k = 0; k < PD; ++k) meta_of(tk + k * pstep, m_rp[k], m_c0[k], m_ce[k]);
    int nd[NA][NPF];
#pragma unroll
    for (int k = 0; k < NA; ++k) nodes_of(m_c0[k], m_ce[k], nd[k]);
    for (int64_t i = warp; tk < tasks; tk += pstep, i += kProd) {
      const int64_t rp0 = m_rp[0], c00 = m_c0[0], ce0 = m_ce[0];
      const int(&nd0)[NPF] = nd[0];
      const int s = (int)(i % S);
      if (i >= S) mbar_wait(empty + s, (uint32_t)(((i / S) - 1) & 1));
      unsigned char* st = smem + s * L::stage;
      float* xs = reinterpret_cast<float*>(st + L::s_xs);
      const int64_t w = p.win_begin + tk / p.nchunks;
      const int d0 = MODE == MODE_SDDMM ? p.koff : (int)(tk % p.nchunks) * 8 * NT;
      const int u = (int)(ce0 - c00);
      const int ncols = min(u, CPR);
      const int pad = min(CPR, (ncols + 15) & ~15);
      const int dv = min(8 * NT, p.dim - d0);
      const int64_t e0 = __shfl_sync(0xffffffffu, rp0, 0);
      const int64_t e1 = __shfl_sync(0xffffffffu, rp0, 16);
      const int E = (int)(e1 - e0);
      // header
      int64_t* hdr = reinterpret_cast<int64_t*>(st + L::s_hdr);
      if (lane <= 16) hdr[lane] = rp0;
      if (lane == 0) {
        hdr[17] = w;
        reinterpret_cast<int*>(hdr + 18)[0] = u;
        reinterpret_cast<int*>(hdr + 18)[1] = d0;
      }
      // neighbour rows
      if constexpr (FULL) {
        const float* xl = p.x + d0 + ch * 4;
        const float* xl2 = kDual ? p.x2 + d0 + ch * 4 : nullptr;
#pragma unroll
        for (int k = 0; k < NPF; ++k) {
          if (32 * k < pad) {
#pragma unroll
            for (int ii = 0; ii < IPK; ++ii) {
              const int c = 32 * k + RPI * ii + rsub;
              const int node = __shfl_sync(0xffffffffu, nd0[k], RPI * ii + rsub);
              float* dst = xs + 32 * k * DS + soff[ii];
              if (c < ncols) {
                cp_async16(dst, xl + (int64_t)node * p.ldx);
                if (kDual) cp_async16(dst + XS2, xl2 + (int64_t)node * p.ldx2);
              } else if (c < pad) {
                *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
                if (kDual) *reinterpret_cast<float4*>(dst + XS2) = make_float4(0.f, 0.f, 0.f, 0.f);
              }
            }
          }
        }
      } else {
        for (int q = lane; q < pad * DS; q += 32) {
          const int c = q / DS, f = q % DS;
          float* dst = xs + G::off(srow(c), f);
          const int node = c < ncols ? (int)__ldg(p.c2n + c00 + c) : -1;
          if (c < ncols && f < dv) {
            cp_async4(dst, p.x + (int64_t)node * p.ldx + d0 + f);
            if (kDual) cp_async4(dst + XS2, p.x2 + (int64_t)node * p.ldx2 + d0 + f);
          } else if (c >= ncols) {
            *dst = 0.f;
            if (kDual) dst[XS2] = 0.f;
          }
        }
      }
      // the window's own rows (SDDMM A operand), unswizzled [16][DS]
      if constexpr (kSddmmPhase) {
        float* xa = reinterpret_cast<float*>(st + L::s_xa);
        const int64_t r0 = w * 16;
        for (int q = lane; q < 16 * DS / 4; q += 32) {
          const int r = q / (DS / 4), c4 = q % (DS / 4);
          float* dst = xa + r * DS + c4 * 4;
          if (r0 + r < p.n && FULL) {
            cp_async16(dst, p.xa + (r0 + r) * p.lda + d0 + c4 * 4);
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int f = c4 * 4 + j;
              if (r0 + r < p.n && f < dv) cp_async4(dst + j, p.xa + (r0 + r) * p.lda + d0 + f);
              else dst[j] = 0.f;
            }
          }
        }
      }
      // edge data
      {
        uint32_t* ef = reinterpret_cast<uint32_t*>(st + L::s_ef);
        float* wa = reinterpret_cast<float*>(st + L::s_wa);
        float* wb = reinterpret_cast<float*>(st + L::s_wb);
        const int ne = min(E, EPR);
        for (int j = lane; j < ne; j += 32) {
          cp_async4(ef + j, p.efrag + e0 + j);
          if constexpr (MODE == MODE_AGNN_BWD) {
            cp_async4(wa + j, p.aux + e0 + j);
          } else if constexpr (MODE == MODE_SPMM || kDual) {
            if (p.w && !p.widx) cp_async4(wa + j, p.w + e0 + j);
            else wa[j] = p.w ? __ldg(p.w + __ldg(p.widx + e0 + j)) : 1.f;
            if constexpr (kDual) {
              if (p.w2 && !p.widx2) cp_async4(wb + j, p.w2 + e0 + j);
              else wb[j] = p.w2 ? __ldg(p.w2 + __ldg(p.widx2 + e0 + j)) : 1.f;
            }
          }
        }
      }
      mbar_arrive_cp_async(full + s);
      mbar_arrive(full + s);
      // rotate the rings
#pragma unroll
      for (int k = 0; k < PD - 1; ++k) m_rp[k] = m_rp[k + 1], m_c0[k] = m_c0[k + 1], m_ce[k] = m_ce[k + 1];
      meta_of(tk + PD * pstep, m_rp[PD - 1], m_c0[PD - 1], m_ce[PD - 1]);
#pragma unroll
      for (int k = 0; k < NA - 1; ++k)
#pragma unroll
        for (int q = 0; q < NPF; ++q) nd[k][q] = nd[k + 1][q];
      nodes_of(m_c0[NA - 1], m_ce[NA - 1], nd[NA - 1]);
    }
    return;
  }

  // ============================= consumer =============================
  const int cw = warp - kProd;
  const int g = lane >> 2, t = lane & 3;
  unsigned char* cs = smem + S * L::stage + cw * L::cons;
  uint32_t* afrag = reinterpret_cast<uint32_t*>(cs);
  uint32_t* afrag2 = afrag + (CPR / 8) * 128;
  float* tile = reinterpret_cast<float*>(cs);
  float* escore = reinterpret_cast<float*>(cs + L::c_esc);
  int spo0[NQ], spo1[NQ], sdo0[NQ], sdo1[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    spo0[q] = G::off(brev3(t), g * NT + q * V);
    spo1[q] = G::off(brev3(t + 4), g * NT + q * V);
    sdo0[q] = G::off(brev3(g), t * NT + q * V);
    sdo1[q] = G::off(brev3(g), (t + 4) * NT + q * V);
  }

  int64_t i = cw;
  for (int64_t tk = blockIdx.x + cw * tstep; tk < tasks; tk += kCons * tstep, i += kCons) {
    const int s = (int)(i % S);
    mbar_wait(full + s, (uint32_t)((i / S) & 1));
    const unsigned char* st = smem + s * L::stage;
    const float* xs = reinterpret_cast<const float*>(st + L::s_xs);
    const int64_t* hdr = reinterpret_cast<const int64_t*>(st + L::s_hdr);
    const uint32_t* ef = reinterpret_cast<const uint32_t*>(st + L::s_ef);
    const float* wa = reinterpret_cast<const float*>(st + L::s_wa);
    const float* wb = reinterpret_cast<const float*>(st + L::s_wb);
    const int64_t e0 = hdr[0], e1 = hdr[16];
    const int64_t w = hdr[17];
    const int u = reinterpret_cast<const int*>(hdr + 18)[0];
    const int d0 = reinterpret_cast<const int*>(hdr + 18)[1];
    const int E = (int)(e1 - e0);
    const int64_t r0 = w * 16, r1 = min(r0 + 16, p.n);
    const int ncols = min(u, CPR);
    const int nb = (ncols + 7) >> 3, npb = (ncols + 15) >> 4;
    const int ne = min(E, EPR);

    float acc[NT][4];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;

    // ---------------- SDDMM phase (stage-resident) ----------------
    if constexpr (kSddmmPhase) {
      const float* xa = reinterpret_cast<const float*>(st + L::s_xa);
      uint32_t a[4][NT];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int r = g + ((h & 1) ? 8 : 0);
        const int f0 = ((h & 2) ? (t + 4) : t) * NT;
#pragma unroll
        for (int j = 0; j < NT; ++j) a[h][j] = tf32_rn(xa[r * DS + f0 + j]);
      }
      float* trow0 = tile + g * TS + 2 * t;
      float* trow1 = tile + (g + 8) * TS + 2 * t;
      for (int sb = 0; sb < npb; ++sb) {
        float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const float* blk = xs + (sb * 16 + hh * 8) * DS;
          float b0[NT], b1[NT];
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            lds_vec<V>(b0 + q * V, blk + sdo0[q]);
            lds_vec<V>(b1 + q * V, blk + sdo1[q]);
          }
#pragma unroll
          for (int j = 0; j < NT; ++j)
            mma_tf32(sc[hh], a[0][j], a[1][j], a[2][j], a[3][j], tf32_rn(b0[j]), tf32_rn(b1[j]));
        }
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          *reinterpret_cast<float2*>(trow0 + sb * 16 + hh * 8) = make_float2(sc[hh][0], sc[hh][1]);
          *reinterpret_cast<float2*>(trow1 + sb * 16 + hh * 8) = make_float2(sc[hh][2], sc[hh][3]);
        }
      }
      __syncwarp();
      if constexpr (MODE == MODE_SDDMM) {
        // StoreSparse (columns of the staged round) — edges past the stage
        // edge slots read their slot from global
        for (int j = lane; j < E; j += 32) {
          const int fi = j < ne ? (int)ef[j] : (int)__ldg(p.efrag + e0 + j);
          if (fi >= nb * 128) continue;
          int row, col;
          decode_slot(fi, row, col);
          float v = tile[row * TS + col];
          if (p.accumulate) v += p.eout[e0 + j];
          p.eout[e0 + j] = v;
        }
      } else {
        const int row = lane >> 1, sub = lane & 1;
        const int rb = (int)(hdr[row] - e0), re = (int)(hdr[row + 1] - e0);
        for (int j = lane; j < E; j += 32) {
          int rw, cl;
          decode_slot((int)ef[j], rw, cl);
          const float sv = tile[rw * TS + cl];
          escore[j] = MODE == MODE_AGNN_BWD ? wa[j] * sv : sv;
        }
        __syncwarp();
        if constexpr (MODE == MODE_AGNN_FWD) {
          float mx = -INFINITY;
          for (int j = rb + sub; j < re; j += 2) mx = fmaxf(mx, escore[j]);
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
          float sm = 0.f;
          for (int j = rb + sub; j < re; j += 2) sm += expf(escore[j] - mx);
          sm += __shfl_xor_sync(0xffffffffu, sm, 1);
          for (int j = rb + sub; j < re; j += 2) escore[j] = expf(escore[j] - mx) / sm;
          __syncwarp();
        } else {
          float sm = 0.f;  // rowsum(P dP)
          for (int j = rb + sub; j < re; j += 2) sm += escore[j];
          sm += __shfl_xor_sync(0xffffffffu, sm, 1);
          __syncwarp();
          for (int j = rb + sub; j < re; j += 2) escore[j] = sm;
          __syncwarp();
          for (int j = lane; j < E; j += 32) {
            int rw, cl;
            decode_slot((int)ef[j], rw, cl);
            escore[j] = wa[j] * (tile[rw * TS + cl] - escore[j]);  // dS = P (dP - rowsum)
          }
          __syncwarp();
        }
        for (int j = lane; j < E; j += 32) p.eout[e0 + j] = escore[j];
        for (int q = lane; q < nb * 32; q += 32)
          reinterpret_cast<uint4*>(afrag)[q] = make_uint4(0, 0, 0, 0);
        __syncwarp();
        for (int j = lane; j < E; j += 32) afrag[ef[j]] = tf32_rn(escore[j]);
        __syncwarp();
      }
    }

    // ---------------- SpMM phase (stage-resident round) ----------------
    if constexpr (kSpmmPhase) {
      if constexpr (!kFused) {
        for (int q = lane; q < nb * 32; q += 32) {
          reinterpret_cast<uint4*>(afrag)[q] = make_uint4(0, 0, 0, 0);
          if (kDual) reinterpret_cast<uint4*>(afrag2)[q] = make_uint4(0, 0, 0, 0);
        }
        __syncwarp();
        for (int j = lane; j < E; j += 32) {
          int fi;
          float va, vb = 1.f;
          if (j < ne) {
            fi = (int)ef[j];
            va = wa[j];
            if (kDual) vb = wb[j];
          } else {
            const int64_t e = e0 + j;
            fi = (int)__ldg(p.efrag + e);
            va = p.w ? (p.widx ? __ldg(p.w + __ldg(p.widx + e)) : __ldg(p.w + e)) : 1.f;
            if (kDual) vb = p.w2 ? (p.widx2 ? __ldg(p.w2 + __ldg(p.widx2 + e)) : __ldg(p.w2 + e)) : 1.f;
          }
          if (fi < nb * 128) {
            afrag[fi] = tf32_rn(va);
            if (kDual) afrag2[fi] = tf32_rn(vb);
          }
        }
        __syncwarp();
      }
#pragma unroll 2
      for (int b = 0; b < nb; ++b) {
        const uint4 af = reinterpret_cast<const uint4*>(afrag)[b * 32 + lane];
        const float* blk = xs + b * 8 * DS;
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
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            lds_vec<V>(x0 + q * V, blk + XS2 + spo0[q]);
            lds_vec<V>(x1 + q * V, blk + XS2 + spo1[q]);
          }
#pragma unroll
          for (int j = 0; j < NT; ++j)
            mma_tf32(acc[j], af2.x, af2.y, af2.z, af2.w, tf32_rn(x0[j]), tf32_rn(x1[j]));
        }
      }
    }
    // rows of the epilogue need the stage header: copy before release
    const int64_t rp_lane = lane <= 16 ? hdr[lane] : 0;
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + s);

    // ------- rounds beyond the stage (u > CPR): direct global loads -------
    if constexpr (!kFused) {
      if (u > CPR) {
        for (int cb = CPR; cb < u; cb += CPR) {
          const int nc = min(CPR, u - cb);
          const int64_t c0 = __ldg(p.coff + w);
          if constexpr (MODE == MODE_SDDMM) {
            // scores for columns [cb, cb + nc): per edge, direct dot products
            for (int64_t e = e0 + lane; e < e1; e += 32) {
              const int fi = (int)__ldg(p.efrag + e);
              int row, col;
              decode_slot(fi, row, col);
              if (col < cb || col >= cb + nc) continue;
              const int64_t r = r0 + row;
              const int node = (int)__ldg(p.c2n + c0 + col);
              float sacc = 0.f;
              for (int f = 0; f < min(8 * NT, p.dim - d0); ++f)
                sacc += __uint_as_float(tf32_rn(__ldg(p.xa + r * p.lda + d0 + f))) *
                        __uint_as_float(tf32_rn(__ldg(p.x + (int64_t)node * p.ldx + d0 + f)));
              if (p.accumulate) sacc += p.eout[e];
              p.eout[e] = sacc;
            }
          } else {
            const int nbr = (nc + 7) >> 3;
            for (int q = lane; q < nbr * 32; q += 32) {
              reinterpret_cast<uint4*>(afrag)[q] = make_uint4(0, 0, 0, 0);
              if (kDual) reinterpret_cast<uint4*>(afrag2)[q] = make_uint4(0, 0, 0, 0);
            }
            __syncwarp();
            for (int64_t e = e0 + lane; e < e1; e += 32) {
              const int fi = (int)__ldg(p.efrag + e) - cb * 16;
              if (fi < 0 || fi >= nbr * 128) continue;
              const float va = p.w ? (p.widx ? __ldg(p.w + __ldg(p.widx + e)) : __ldg(p.w + e)) : 1.f;
              afrag[fi] = tf32_rn(va);
              if constexpr (kDual) {
                const float vb =
                    p.w2 ? (p.widx2 ? __ldg(p.w2 + __ldg(p.widx2 + e)) : __ldg(p.w2 + e)) : 1.f;
                afrag2[fi] = tf32_rn(vb);
              }
            }
            __syncwarp();
            for (int b = 0; b < nbr; ++b) {
              const int c_t = cb + b * 8 + t, c_t4 = c_t + 4;
              const int n0 = c_t < u ? (int)__ldg(p.c2n + c0 + c_t) : -1;
              const int n1 = c_t4 < u ? (int)__ldg(p.c2n + c0 + c_t4) : -1;
              float x0[NT], x1[NT];
              const uint4 af = reinterpret_cast<const uint4*>(afrag)[b * 32 + lane];
              load_slice<NT>(x0, p.x, n0, p.ldx, d0 + g * NT, p.dim);
              load_slice<NT>(x1, p.x, n1, p.ldx, d0 + g * NT, p.dim);
#pragma unroll
              for (int j = 0; j < NT; ++j)
                mma_tf32(acc[j], af.x, af.y, af.z, af.w, tf32_rn(x0[j]), tf32_rn(x1[j]));
              if constexpr (kDual) {
                const uint4 af2 = reinterpret_cast<const uint4*>(afrag2)[b * 32 + lane];
                load_slice<NT>(x0, p.x2, n0, p.ldx2, d0 + g * NT, p.dim);
                load_slice<NT>(x1, p.x2, n1, p.ldx2, d0 + g * NT, p.dim);
#pragma unroll
                for (int j = 0; j < NT; ++j)
                  mma_tf32(acc[j], af2.x, af2.y, af2.z, af2.w, tf32_rn(x0[j]), tf32_rn(x1[j]));
              }
            }
            __syncwarp();
          }
        }
      }
    }

    // ---------------- epilogues ----------------
    if constexpr (MODE == MODE_SDDMM) {
      if (p.epilogue != 0) {
        __syncwarp();
        const int row = lane >> 1, sub = lane & 1;
        const int64_t rb = __shfl_sync(0xffffffffu, rp_lane, row);
        const int64_t re = __shfl_sync(0xffffffffu, rp_lane, row + 1);
        if (p.epilogue == 1) {
          float mx = -INFINITY;
          for (int64_t j = rb + sub; j < re; j += 2) mx = fmaxf(mx, p.eout[j]);
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
          float sm = 0.f;
          for (int64_t j = rb + sub; j < re; j += 2) sm += expf(p.eout[j] - mx);
          sm += __shfl_xor_sync(0xffffffffu, sm, 1);
          for (int64_t j = rb + sub; j < re; j += 2) p.eout[j] = expf(p.eout[j] - mx) / sm;
        } else {
          float sm = 0.f;
          for (int64_t j = rb + sub; j < re; j += 2) sm += __ldg(p.aux + j) * p.eout[j];
          sm += __shfl_xor_sync(0xffffffffu, sm, 1);
          for (int64_t j = rb + sub; j < re; j += 2) p.eout[j] = __ldg(p.aux + j) * (p.eout[j] - sm);
        }
      }
    }
    if constexpr (kSpmmPhase) {
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
  using L = Layout<NT, MODE>;
  constexpr int kThreads = L::kThreads;
  const size_t smem = (size_t)L::total;
  auto kern = window_kernel<NT, MODE, FULL>;
  static int configured_dev = -1;
  static int per_sm = 1;
  int dev = 0;
  TCG_CUDA(cudaGetDevice(&dev), "window_kernel device");
  if (configured_dev != dev) {
    TCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
             "window_kernel attr");
    TCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem),
             "window_kernel occupancy");
    if (per_sm < 1) per_sm = 1;
    configured_dev = dev;
  }
  p.use_tma = 0;
  const int64_t tasks = p.nwin * p.nchunks;
  int64_t blocks = (tasks + L::kCons - 1) / L::kCons;
  const int64_t cap = (int64_t)num_sms() * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) return TCG_OK;
  kern<<<(unsigned)blocks, kThreads, smem, s>>>(p);
  TCG_LAUNCHED("window_kernel");
  return TCG_OK;
}

template <int NT, int MODE>
int launch_nt(Params& p, cudaStream_t s) {
  // FULL: feature chunks complete and rows 16-B aligned -> 16-B cp.async
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
