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
  static constexpr int xs_bytes = CPR * 8 * NT * 4 * (kDual ? 2 : 1);  // one stage
  static constexpr int xs = 0;                                          // 2 stages, 1024-B aligned
  static constexpr int frag = xs + 2 * xs_bytes;
  static constexpr int frag_a = (CPR / 8) * 512 * (kDual ? 2 : 1);
  static constexpr int frag_t = (kFused || MODE == MODE_SDDMM) ? 16 * tile_stride * 4 : 0;
  static constexpr int frag_bytes = frag_a > frag_t ? frag_a : frag_t;
  static constexpr int edges = frag + frag_bytes;
  static constexpr int rps = edges + (kFused ? kEdgesPerWindow * 4 : 0);  // 17 int64
  static constexpr int nodes = rps + 136;                                  // CPR int
  static constexpr int bar = (nodes + CPR * 4 + 7) & ~7;                   // 2 mbarriers
  static constexpr int total = (bar + 16 + 1023) & ~1023;
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

// Per-window metadata carried in registers through the software pipeline.
struct Meta {
  int64_t w;     // window id (-1: no task)
  int chunk;     // feature chunk (SpMM modes)
  int64_t rp;    // lane <= 16: node_ptr[min(16*w + lane, n)]
  int64_t c0, cend;
};

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
  constexpr int NPF = CPR / 32;  // col_to_node registers per lane
  constexpr bool kDual = CV::kDual;
  constexpr bool kFused = CV::kFused;
  constexpr bool kSpmmPhase = MODE != MODE_SDDMM;
  constexpr bool kSddmmPhase = MODE == MODE_SDDMM || kFused;
  constexpr int TS = CV::tile_stride;
  constexpr int XS2 = CPR * DS;                 // floats to the second operand (dual)
  constexpr int XSTAGE = CV::xs_bytes / 4;      // floats per pipeline stage
  constexpr int EV = kFused ? kEdgesPerWindow / 32 : 4;  // prefetched edges / 32
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  unsigned char* sm = smem_raw + warp * CV::total;
  if ((smem_u32(sm) & 1023) != 0) __trap();  // TMA swizzle needs 1024-B aligned rows
  float* xs_base = reinterpret_cast<float*>(sm + CV::xs);
  uint32_t* afrag = reinterpret_cast<uint32_t*>(sm + CV::frag);
  uint32_t* afrag2 = afrag + (CPR / 8) * 128;
  float* tile = reinterpret_cast<float*>(sm + CV::frag);
  float* escore = reinterpret_cast<float*>(sm + CV::edges);
  int64_t* rps = reinterpret_cast<int64_t*>(sm + CV::rps);
  int* nodes_s = reinterpret_cast<int*>(sm + CV::nodes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + CV::bar);

  // zero both stages once: feature padding [dim, DS) is never written
  for (int i = lane; i < 2 * XSTAGE; i += 32) xs_base[i] = 0.f;
  if (lane == 0) {
    mbar_init(bars);
    mbar_init(bars + 1);
  }
  uint32_t ph0 = 0, ph1 = 0;
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
  const int nkc = MODE == MODE_SDDMM ? p.nkc : 1;

  // ------------------------------------------------------------------ //
  // pipeline helpers
  // ------------------------------------------------------------------ //
  auto load_meta = [&](int64_t tk) {
    Meta m;
    if (tk >= tasks) {
      m.w = -1, m.chunk = 0, m.rp = 0, m.c0 = 0, m.cend = 0;
      return m;
    }
    m.w = p.win_begin + tk / p.nchunks;
    m.chunk = (int)(tk % p.nchunks);
    m.rp = lane <= 16 ? __ldg(p.ptr + min(m.w * 16 + lane, p.n)) : 0;
    m.c0 = __ldg(p.coff + m.w);
    m.cend = __ldg(p.coff + m.w + 1);
    return m;
  };
  // col_to_node of the first CPR columns (out-of-range row id beyond u)
  auto load_nodes = [&](const Meta& m, int cb, int (&nd)[NPF]) {
    const int u = m.w < 0 ? 0 : (int)(m.cend - m.c0);
#pragma unroll
    for (int k = 0; k < NPF; ++k) {
      const int c = cb + lane + 32 * k;
      nd[k] = c < u ? (int)__ldg(p.c2n + m.c0 + c) : (int)p.n;
    }
  };
  // edge data of the first 32*EV edges: fragment slot (+ weights / P)
  auto load_edges = [&](const Meta& m, uint32_t (&ef)[EV], float (&wa)[EV], float (&wb)[EV]) {
    const int64_t e0 = __shfl_sync(0xffffffffu, m.rp, 0);
    const int64_t e1 = __shfl_sync(0xffffffffu, m.rp, 16);
#pragma unroll
    for (int v = 0; v < EV; ++v) {
      const int64_t e = e0 + lane + 32 * v;
      const bool ok = m.w >= 0 && e < e1;
      ef[v] = ok ? __ldg(p.efrag + e) : 0xffffffffu;
      wa[v] = 1.f;
      wb[v] = 1.f;
      if constexpr (MODE == MODE_SPMM || kDual) {
        if (ok && p.w) wa[v] = p.widx ? __ldg(p.w + __ldg(p.widx + e)) : __ldg(p.w + e);
      }
      if constexpr (kDual) {
        if (ok && p.w2) wb[v] = p.widx2 ? __ldg(p.w2 + __ldg(p.widx2 + e)) : __ldg(p.w2 + e);
      }
      if constexpr (MODE == MODE_AGNN_BWD) {
        if (ok) wa[v] = __ldg(p.aux + e);
      }
    }
  };
  // the window's own 16 rows (SDDMM A operand), feature chunk at dk
  auto load_arows = [&](const Meta& m, int dk, float (&ar)[4][NT]) {
    const int64_t r0 = m.w * 16, r1 = min(r0 + 16, p.n);
    const int dv = min(8 * NT, p.dim - dk);
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int64_t r = r0 + g + ((h & 1) ? 8 : 0);
      const int f0 = ((h & 2) ? (t + 4) : t) * NT;
      const bool rok = m.w >= 0 && r < r1;
      const float* src = p.xa + r * p.lda + dk + f0;
      bool done = false;
      if constexpr (NT % 4 == 0) {
        if (p.vec16 && rok && f0 + NT <= dv) {
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
        for (int j = 0; j < NT; ++j) ar[h][j] = (rok && f0 + j < dv) ? __ldg(src + j) : 0.f;
      }
    }
  };
  // FetchDense into stage `st`: returns true if a TMA transaction was issued
  auto stage_rows = [&](const Meta& m, const int (&nd)[NPF], int cb, int dk, int st) -> bool {
    const int u = m.w < 0 ? 0 : (int)(m.cend - m.c0);
    const int ncols = min(CPR, u - cb);
    if (ncols <= 0) return false;
    const int pad = min(CPR, (ncols + 15) & ~15);
    float* xs = xs_base + st * XSTAGE;
    fence_proxy_async();  // earlier generic reads of this stage before async writes
#pragma unroll
    for (int k = 0; k < NPF; ++k) nodes_s[lane + 32 * k] = nd[k];
    __syncwarp();
    if (p.use_tma) {
      constexpr uint32_t kGroupBytes = 4u * G::BW * 4u * G::HALVES * (kDual ? 2 : 1);
      if (lane == 0) mbar_expect(bars + st, (uint32_t)(pad / 4) * kGroupBytes);
      __syncwarp();
      if (lane < pad / 4) {
        int rr[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int srw = 4 * lane + r;
          rr[r] = nodes_s[(srw & ~7) | brev3(srw & 7)];
        }
        float* dst = xs + 4 * lane * G::BW;
#pragma unroll
        for (int hv = 0; hv < G::HALVES; ++hv) {
          tma_gather4(dst + hv * CPR * G::BW, &tmx, dk + hv * 32, rr[0], rr[1], rr[2], rr[3],
                      bars + st);
          if (kDual)
            tma_gather4(dst + XS2 + hv * CPR * G::BW, &tmx2, dk + hv * 32, rr[0], rr[1], rr[2],
                        rr[3], bars + st);
        }
      }
      return true;
    }
    const int dv = min(8 * NT, p.dim - dk);
    for (int q = lane; q < pad * DS; q += 32) {
      const int c = q / DS, f = q % DS;
      float* dst = xs + G::template off<CPR>(srow(c), f);
      if (c < ncols) {
        if (f < dv) {
          const int64_t node = nodes_s[c];
          cp_async4(dst, p.x + node * p.ldx + dk + f);
          if (kDual) cp_async4(dst + XS2, p.x2 + node * p.ldx2 + dk + f);
        }
      } else {
        *dst = 0.f;
        if (kDual) dst[XS2] = 0.f;
      }
    }
    cp_commit();
    return false;
  };
  auto wait_stage = [&](bool tma, int st) {
    if (tma) {
      if (st == 0) {
        mbar_wait(bars, ph0);
        ph0 ^= 1;
      } else {
        mbar_wait(bars + 1, ph1);
        ph1 ^= 1;
      }
    } else {
      cp_wait_all();
    }
    __syncwarp();
  };

  // ------------------------------------------------------------------ //
  // prologue: metadata 3 tasks ahead, nodes 2 ahead, rows + edges 1 ahead
  // ------------------------------------------------------------------ //
  int64_t task = (int64_t)blockIdx.x * kWarps + warp;
  Meta m0 = load_meta(task), m1 = load_meta(task + nwarps), m2 = load_meta(task + 2 * nwarps);
  int n0[NPF], n1[NPF];
  load_nodes(m0, 0, n0);
  load_nodes(m1, 0, n1);
  uint32_t ef0[EV];
  float wa0[EV], wb0[EV];
  load_edges(m0, ef0, wa0, wb0);
  float ar0[kSddmmPhase ? 4 : 1][kSddmmPhase ? NT : 1];
  if constexpr (kSddmmPhase) load_arows(m0, m0.chunk * 0, ar0);
  bool tma0 = stage_rows(m0, n0, 0, MODE == MODE_SDDMM ? 0 : m0.chunk * 8 * NT, 0);
  int st = 0;

  for (; task < tasks; task += nwarps) {
    // ---- 1. issue the next window's gather, prefetch further ahead ----
    const bool tma1 = stage_rows(m1, n1, 0, MODE == MODE_SDDMM ? 0 : m1.chunk * 8 * NT, st ^ 1);
    uint32_t ef1[EV];
    float wa1[EV], wb1[EV];
    load_edges(m1, ef1, wa1, wb1);
    float ar1[kSddmmPhase ? 4 : 1][kSddmmPhase ? NT : 1];
    if constexpr (kSddmmPhase) load_arows(m1, 0, ar1);
    int n2[NPF];
    load_nodes(m2, 0, n2);
    const Meta m3 = load_meta(task + 3 * nwarps);

    // ---- 2. compute the current window ----
    const int64_t w = m0.w;
    const int d0 = m0.chunk * 8 * NT;
    const int64_t r0 = w * 16, r1 = min(r0 + 16, p.n);
    if (lane <= 16) rps[lane] = m0.rp;
    __syncwarp();
    const int64_t e0 = rps[0], e1 = rps[16];
    const int E = (int)(e1 - e0);
    const int u = (int)(m0.cend - m0.c0);
    const int nrounds = kFused ? 1 : (u + CPR - 1) / CPR;

    float acc[NT][4];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;

    for (int rd = 0; rd < max(nrounds, 1); ++rd) {
      const int cb = rd * CPR;
      const int ncols = min(CPR, u - cb);
      const int pad = min(CPR, (max(ncols, 0) + 15) & ~15);
      const float* xs = xs_base + st * XSTAGE;
      const int fbase = cb * 16, flim = ((max(ncols, 0) + 7) >> 3) * 128;  // whole blocks
      for (int kc = 0; kc < nkc; ++kc) {
        const int dk = MODE == MODE_SDDMM ? kc * 8 * NT : d0;
        bool tma_cur = tma0;
        if (rd > 0 || kc > 0) {  // rare: rounds / k-chunks beyond the pipelined one
          int nd[NPF];
          load_nodes(m0, cb, nd);
          tma_cur = stage_rows(m0, nd, cb, dk, st);
          if constexpr (kSddmmPhase) load_arows(m0, dk, ar0);
        }
        // ---- InitSparse (non-fused SpMM modes) while rows land ----
        if constexpr (kSpmmPhase && !kFused) {
          const int nb = (pad + 7) >> 3;
          for (int i = lane; i < nb * 32; i += 32) {
            reinterpret_cast<uint4*>(afrag)[i] = make_uint4(0, 0, 0, 0);
            if (kDual) reinterpret_cast<uint4*>(afrag2)[i] = make_uint4(0, 0, 0, 0);
          }
          __syncwarp();
          if (rd == 0) {
#pragma unroll
            for (int v = 0; v < EV; ++v) {
              const int fi = (int)ef0[v];
              if (ef0[v] != 0xffffffffu && fi < flim) {
                afrag[fi] = tf32_rn(wa0[v]);
                if (kDual) afrag2[fi] = tf32_rn(wb0[v]);
              }
            }
          }
          for (int64_t e = e0 + (rd == 0 ? 32 * EV : 0) + lane; e < e1; e += 32) {
            const int fi = (int)__ldg(p.efrag + e) - fbase;
            if (fi < 0 || fi >= flim) continue;
            float wv = 1.f;
            if (p.w) wv = p.widx ? __ldg(p.w + __ldg(p.widx + e)) : __ldg(p.w + e);
            afrag[fi] = tf32_rn(wv);
            if constexpr (kDual) {
              float wv2 = 1.f;
              if (p.w2) wv2 = p.widx2 ? __ldg(p.w2 + __ldg(p.widx2 + e)) : __ldg(p.w2 + e);
              afrag2[fi] = tf32_rn(wv2);
            }
          }
        }
        wait_stage(tma_cur, st);

        // ---- SDDMM phase: scores for 16-column paired blocks ----
        if constexpr (kSddmmPhase) {
          const int npb = pad >> 4;
          uint32_t a[4][NT];
#pragma unroll
          for (int h = 0; h < 4; ++h)
#pragma unroll
            for (int j = 0; j < NT; ++j) a[h][j] = tf32_rn(ar0[h][j]);
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
          __syncwarp();
        }
      }  // k-chunks

      if constexpr (MODE == MODE_SDDMM) {
        // StoreSparse: raw scores of this round's columns to edge order
        if (rd == 0) {
#pragma unroll
          for (int v = 0; v < EV; ++v) {
            const int fi = (int)ef0[v];
            if (ef0[v] != 0xffffffffu && fi < flim) {
              int row, col;
              decode_slot(fi, row, col);
              p.eout[e0 + lane + 32 * v] = tile[row * TS + col];
            }
          }
        }
        for (int64_t e = e0 + (rd == 0 ? 32 * EV : 0) + lane; e < e1; e += 32) {
          const int fi = (int)__ldg(p.efrag + e) - fbase;
          if (fi < 0 || fi >= flim) continue;
          int row, col;
          decode_slot(fi, row, col);
          p.eout[e] = tile[row * TS + col];
        }
        __syncwarp();
      }
      if constexpr (kFused) {
        // edge scores out of the tile
#pragma unroll
        for (int v = 0; v < EV; ++v) {
          const int i = lane + 32 * v;
          if (i < E) {
            int row, col;
            decode_slot((int)ef0[v], row, col);
            escore[i] = tile[row * TS + col];
          }
        }
        __syncwarp();
        // row softmax (fwd) / softmax backward (bwd): 2 lanes per row
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
          __syncwarp();
        } else {
          // P_e * dP_e per edge (P prefetched in wa0), then the row sums
#pragma unroll
          for (int v = 0; v < EV; ++v) {
            const int i = lane + 32 * v;
            if (i < E) escore[i] = wa0[v] * escore[i];
          }
          __syncwarp();
          float s = 0.f;
          for (int i = rb + sub; i < re; i += 2) s += escore[i];
          s += __shfl_xor_sync(0xffffffffu, s, 1);
          __syncwarp();
          // dS = P dP - P * rowsum  (= P (dP - rowsum))
          for (int i = rb + sub; i < re; i += 2) escore[i] = s;  // broadcast row sum
          __syncwarp();
#pragma unroll
          for (int v = 0; v < EV; ++v) {
            const int i = lane + 32 * v;
            if (i < E) {
              int rw, cl;
              decode_slot((int)ef0[v], rw, cl);
              const float dp = tile[rw * TS + cl];
              escore[i] = wa0[v] * (dp - escore[i]);
            }
          }
          __syncwarp();
        }
        // weights -> edge order (P or dS) and -> fragment-ordered A tiles
        const int nb = (pad + 7) >> 3;
        for (int i = lane; i < nb * 32; i += 32)
          reinterpret_cast<uint4*>(afrag)[i] = make_uint4(0, 0, 0, 0);
        __syncwarp();
#pragma unroll
        for (int v = 0; v < EV; ++v) {
          const int i = lane + 32 * v;
          if (i < E) {
            const float wgt = escore[i];
            p.eout[e0 + i] = wgt;
            afrag[ef0[v]] = tf32_rn(wgt);
          }
        }
        __syncwarp();
      }

      // ---- SpMM phase over the 16x8 blocks of this round ----
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
      }
      __syncwarp();
    }  // rounds

    // ---- epilogues ----
    if constexpr (MODE == MODE_SDDMM) {
      if (p.epilogue != 0 && w >= 0) {
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
    __syncwarp();

    // ---- 3. rotate the pipeline ----
    m0 = m1;
    m1 = m2;
    m2 = m3;
#pragma unroll
    for (int k = 0; k < NPF; ++k) n1[k] = n2[k];
#pragma unroll
    for (int v = 0; v < EV; ++v) ef0[v] = ef1[v], wa0[v] = wa1[v], wb0[v] = wb1[v];
    if constexpr (kSddmmPhase) {
#pragma unroll
      for (int h = 0; h < 4; ++h)
#pragma unroll
        for (int j = 0; j < NT; ++j) ar0[h][j] = ar1[h][j];
    }
    tma0 = tma1;
    st ^= 1;
  }
  // drain: nothing in flight is consumed after the last window (the extra
  // stage issued for a non-existent task never starts: stage_rows skips w < 0)
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
