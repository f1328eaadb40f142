// Block-stream SpMM engine: the TF32 tensor-core SpMM of the hot path
// (reference kernels.spmm, kernels.py:213-374; paper Alg. 2) for 16x8 tilings.
//
// Why a second engine: on B200 the aggregation is bound by the per-SM L1
// data pipe that every gathered 32-B sector crosses (ncu:
// l1tex__data_pipe_lsu_wavefronts ~85% busy; a bare 128-B row gather tops
// out near 9 TB/s), and by per-warp issue latency, not by HBM. This engine
// is shaped for that:
//
//  * Flat block stream. The SGT's condensed columns, padded per window to
//    whole 8-column TC blocks (win_partition[w] blocks), form one stream of
//    TB = sum(win_partition) blocks (`col_stream`, built once per tiling by
//    tcg_block_stream; within a block the columns are stored pair-interleaved
//    (c, c+4) so each mma lane reads its two B rows with one 8-B load; padding
//    repeats the window's first node, which the zero A entries cancel).
//  * One warp owns a contiguous slice of the stream, balanced by blocks
//    (block_offsets = exclusive cumsum of win_partition, the per-window
//    TC-block offsets; the slice bounds are found with a 32-ary warp search).
//  * Per warp, a private shared-memory ring of NB blocks: block s + NB's
//    neighbour rows are requested with cp.async as block s is consumed, and
//    block s + 2NB's column ids one step earlier (lanes 0-1), so two levels
//    of dependent loads stay in flight without cross-warp synchronisation.
//  * InitSparse per window: the window's edges (prefetched one window ahead
//    into registers) are scattered into the A fragments (per-edge fragment
//    slot `edge_frag`, the analogue of the reference's _spmm_aux cache,
//    kernels.py:173-188) and un-scattered after the window, so the fragment
//    area is never bulk-cleared.
//  * mma.sync.m16n8k8 TF32 (cvt.rn.tf32 operands = reference quantize_tf32,
//    fp32 accumulate); features are permuted so each lane's B slice and C
//    slice are contiguous (one vector load / store).
//
// Modes: Y = A_w X (+bias) (+= Y), and the dual form Y = A_w1 X1 + A_w2 X2
// used by the A^T pass of the AGNN backward. Feature chunks of 8*NT (NT = 1,
// 2, 4) run as gridDim.y slices.
#include "common.cuh"

#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include "window.cuh"

namespace tcg {
namespace stream {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
template <int BYTES>
__device__ __forceinline__ void cp_async(uint32_t s, const void* g) {
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(g) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(s), "l"(g), "n"(BYTES)
                 : "memory");
}
// copy `src_bytes` (<= BYTES) and zero-fill the rest of the BYTES-wide slot
template <int BYTES>
__device__ __forceinline__ void cp_async_n(uint32_t s, const void* g, int src_bytes) {
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(g), "r"(src_bytes)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(s), "l"(g), "n"(BYTES),
                 "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <int NT>
__device__ __forceinline__ void lds_slice(float (&v)[NT], uint32_t a) {
  if constexpr (NT == 4) {
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];\n"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3])
                 : "r"(a)
                 : "memory");
  } else if constexpr (NT == 2) {
    asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];\n" : "=f"(v[0]), "=f"(v[1]) : "r"(a) : "memory");
  } else {
    asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(v[0]) : "r"(a) : "memory");
  }
}
__device__ __forceinline__ uint4 lds_frag(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a)
               : "memory");
  return v;
}

// Byte offset of (staged row r, lane slice g) inside one ring slot: rows of
// 32*NT bytes, slices of 4*NT bytes, XOR-swizzled so the SpMM fragment reads
// (rows t / t+4, slices g) are bank-conflict free.
template <int NT>
__device__ __forceinline__ uint32_t slot_off(int r, int g) {
  if constexpr (NT == 4) return r * 128 + ((g ^ (2 * r)) & 7) * 16;
  else if constexpr (NT == 2) return r * 64 + (g ^ (4 * ((r >> 1) & 1))) * 8;
  else return r * 32 + g * 4;
}

struct Args {
  const int64_t* ptr;
  const uint32_t* efrag;
  const int32_t* boff;   // block offsets [W+1]
  const uint32_t* cs;    // column stream, pair-interleaved, padded past the end
  int64_t n;
  int win_begin, win_end;
  int nwarps;            // warps per feature chunk
  int d0, ldx, ldx2;     // first feature of chunk 0 (chunk y adds y * 8 * NT)
  int dv;                // valid features of the (single) chunk when masked, else 8 * NT
  const float* x;
  const float* x2;
  const float* w;
  const uint32_t* widx;
  const float* w2;
  const uint32_t* widx2;
  const float* bias;
  float* y;
  int64_t ldy, y_row0;
  int accumulate;
  int vec_out;           // 16-B aligned output rows
  int x16;               // NT = 2: operand rows 16-B aligned (one 16-B copy per lane)
  int relu;              // ReLU on the stored output (after bias / accumulate)
};

constexpr int kEPL = 5;    // edges per lane prefetched for the next window (160)

// Ring depth, fragment area and CTA shape. Round 2 measured the alternatives
// at arxiv D = 32 (cold, clean L2): NB 8 / MB 8 / 4 warps 35.7 us, NB 8 / MB 16
// / 4 warps 35.9 us, NB 4 / MB 8 / 4 warps 34.9 us, against 33.8 us for this
// shape: more bytes in flight do not help, the ring is not what bounds it.
// PAIR (16-wide chunks): every step consumes two consecutive 8-column blocks of
// the window-even-padded pair stream (tcg_block_stream_pairs), so the per-step
// costs (ring wait, id copies, cursor updates, loop) are paid once per 1 KB of
// staged rows, as at 32-wide chunks.
template <int NT, bool DUAL, bool BIG = false, bool PAIR = false, int DMB = 8, int OCC = 1>
struct Cfg {
  static constexpr int KB = PAIR ? 2 : 1;  // blocks per step
  // ring depth in steps: 4 blocks of 32-wide rows in flight either way
  static constexpr int NB = (PAIR && NT == 4) ? 2 : 4;
  // column-id ring: ids of block s + NI are requested at step s (NI >= 2 NB so
  // the ids of block s + NB have landed by then); power of two
  static constexpr int NI = 2 * NB;
  static_assert(NI >= 2 * NB && (NI & (NI - 1)) == 0, "column-id ring depth");
  static constexpr int SLOT = 8 * 32 * NT;         // bytes of one operand's block
  static constexpr int OPS = DUAL ? 2 : 1;
  // dual form: DMB-block fragment rounds; 4 keeps a warp at 12.5 KB, 4 CTAs (16 warps)
  // per SM instead of 3 at 8, which pays on short windows (see stream_spmm)
  // OCC 3 (16-wide pair steps on large graphs): 8-block rounds and <= 85 registers, three
  // 8-warp CTAs per SM instead of two (amazon0601 D=16 61.4-63.5 -> 59.4 us cold)
  static constexpr int MB = DUAL ? DMB : (BIG || OCC > 1) ? 8 : 16;  // A-fragment blocks resident (one round)
  static constexpr int STEP = SLOT * OPS * KB;     // staged bytes of one step
  static constexpr int RING = NB * STEP;
  static constexpr int IDX = NI * 32 * KB;         // column ids of NI steps
  static constexpr int AFR = MB * 512 * OPS;
  // BIG: windows with more edges than the register prefetch holds (products:
  // ~400) stage the next window's edge slots and weights in shared memory
  static constexpr int EMAX = BIG ? 512 : 0;
  static constexpr int EDGE = 2 * EMAX * 4 * (1 + OPS);
  static constexpr int WARP = RING + IDX + AFR + EDGE;
  static constexpr int WPC = (DUAL || BIG) ? 4 : 8;  // warps per CTA
  static constexpr int SMEM = WPC * WARP;
};

// first p in [lo, hi) with a[p] >= v (hi if none); whole warp, 32-ary
__device__ __forceinline__ int warp_lower_bound(const int32_t* __restrict__ a, int lo, int hi,
                                                int v) {
  const int lane = threadIdx.x & 31;
  while (hi - lo > 32) {
    const int step = (hi - lo + 31) >> 5;
    const int p = lo + lane * step;
    const bool pr = p < hi && __ldg(a + p) < v;
    const int c = __popc(__ballot_sync(0xffffffffu, pr));
    if (c == 0) return lo;
    const int nlo = lo + (c - 1) * step + 1;
    hi = min(hi, lo + c * step);
    lo = nlo;
  }
  const int p = lo + lane;
  const bool pr = p < hi && __ldg(a + p) < v;
  return lo + __popc(__ballot_sync(0xffffffffu, pr));
}

template <int NT, bool DUAL, bool BIG, bool MASK, bool PAIR = false, bool X2R = false, int DMB = 8, int OCC = 1>
__global__ void __launch_bounds__(Cfg<NT, DUAL, BIG, PAIR, DMB, OCC>::WPC * 32, OCC) spmm_stream(const Args a) {
  TCG_PDL_ENTRY();
  using C = Cfg<NT, DUAL, BIG, PAIR, DMB, OCC>;
  constexpr int NB = C::NB, NI = C::NI, SLOT = C::SLOT, MB = C::MB, KB = C::KB;
  static_assert(!PAIR || (NT >= 2 && (!DUAL || NT == 4) && MB % 2 == 0), "pair steps: 16/32-wide");
  constexpr uint32_t RS = MB * 128;  // fragment slots of one round
  constexpr int CP = 4 * NT;  // bytes per lane per staged row
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int gw = blockIdx.x * C::WPC + wid;
  const int g = lane >> 2, t = lane & 3;
  unsigned char* wsm = smem + wid * C::WARP;
  const uint32_t ring = smem_u32(wsm);
  const uint32_t iring = ring + C::RING;
  const unsigned char* iring_p = wsm + C::RING;
  uint32_t* afr = reinterpret_cast<uint32_t*>(wsm + C::RING + C::IDX);
  uint32_t* afr2 = afr + MB * 128;
  // BIG: edge staging, 2 slots x {frag u32[EMAX], w f32[EMAX] (, w2 f32[EMAX])}
  unsigned char* ebuf = wsm + C::RING + C::IDX + C::AFR;

  // ---- this warp's slice of the block stream ----
  const int B0 = __ldg(a.boff + a.win_begin), B1 = __ldg(a.boff + a.win_end);
  const int64_t TBr = B1 - B0;
  const int lo_b = B0 + (int)(TBr * gw / a.nwarps);
  const int hi_b = B0 + (int)(TBr * (gw + 1) / a.nwarps);
  const int ws = warp_lower_bound(a.boff, a.win_begin, a.win_end, lo_b);
  const int we = gw + 1 == a.nwarps ? a.win_end : warp_lower_bound(a.boff, ws, a.win_end, hi_b);
  if (ws >= we) return;
  const int gb0 = __ldg(a.boff + ws);

  const int d0 = a.d0 + blockIdx.y * 8 * NT;
  const char* xb = reinterpret_cast<const char*>(a.x + d0 + g * NT);
  const char* xb2 = DUAL ? reinterpret_cast<const char*>(a.x2 + d0 + g * NT) : nullptr;
  const uint32_t xrow = (uint32_t)a.ldx * 4u, xrow2 = (uint32_t)a.ldx2 * 4u;
  // per-lane ring addresses: X slot s at xs + (s % NB) * SLOT * OPS (rows t / t+4 at
  // +0 / +d1), this lane's column-id pair of block s at is + (s % NI) * 256
  const uint32_t xs = ring + slot_off<NT>(t, g);
  const uint32_t d1 = slot_off<NT>(t + 4, g) - slot_off<NT>(t, g);
  const uint32_t is = iring + lane * 16;  // lanes 0-1 copy a block's 32 B of ids
  // each lane copies its own (c_t, c_t+4) pair of every block: no cross-lane
  // visibility, so the stream loop needs no warp barrier
  const char* csl = reinterpret_cast<const char*>(a.cs + 8 * (int64_t)gb0 + 4 * lane);
  // masked tail chunk: this lane's slice holds min(NT, dv - g NT) real features
  const int vb = MASK ? max(0, min(CP, (a.dv - g * NT) * 4)) : CP;
  constexpr bool masked = MASK;
  // 16-wide chunks (64-B row slices): lane L copies 16 B -- quarter L%4 of row
  // L/4 -- so a block's 8 rows take one 16-B cp.async per lane instead of two
  // 8-B ones (the staged layout is the same: 16-B pieces land on swizzle-paired
  // 8-B granules, which stay adjacent because the swizzle only flips bit 2)
  const int qr = lane >> 2, qk = lane & 3;
  const uint32_t q_id = 4u * (qr < 4 ? 2 * qr : 2 * qr - 7);
  const uint32_t q_dst = qr * 64 + ((2 * qk) ^ (4 * ((qr >> 1) & 1))) * 8;
  const int q_vb = MASK ? max(0, min(16, (a.dv - 4 * qk) * 4)) : 16;
  const char* q_x = reinterpret_cast<const char*>(a.x + d0) + 16 * qk;
  const char* q_x2 = DUAL ? reinterpret_cast<const char*>(a.x2 + d0) + 16 * qk : nullptr;
  auto issue_block = [&](uint32_t xo, uint32_t io) {
    if constexpr (PAIR && NT == 2) {  // x16 layout, both blocks of the step
      const uint32_t id0 = *reinterpret_cast<const uint32_t*>(iring_p + io + q_id);
      const uint32_t id1 = *reinterpret_cast<const uint32_t*>(iring_p + io + 32 + q_id);
      const uint32_t d = ring + xo + q_dst;
      if constexpr (masked) {
        cp_async_n<16>(d, q_vb ? (const void*)(q_x + (uint64_t)id0 * xrow) : (const void*)a.x, q_vb);
        cp_async_n<16>(d + SLOT, q_vb ? (const void*)(q_x + (uint64_t)id1 * xrow) : (const void*)a.x,
                       q_vb);
      } else {
        cp_async<16>(d, q_x + (uint64_t)id0 * xrow);
        cp_async<16>(d + SLOT, q_x + (uint64_t)id1 * xrow);
      }
      return;
    }
    if (NT == 2 && a.x16) {
      const uint32_t id = *reinterpret_cast<const uint32_t*>(iring_p + io + q_id);
      const uint32_t d = ring + xo + q_dst;
      if constexpr (masked) {
        cp_async_n<16>(d, q_vb ? (const void*)(q_x + (uint64_t)id * xrow) : (const void*)a.x,
                       q_vb);
        if constexpr (DUAL)
          cp_async_n<16>(d + SLOT,
                         q_vb ? (const void*)(q_x2 + (uint64_t)id * xrow2) : (const void*)a.x,
                         q_vb);
      } else {
        cp_async<16>(d, q_x + (uint64_t)id * xrow);
        if constexpr (DUAL) cp_async<16>(d + SLOT, q_x2 + (uint64_t)id * xrow2);
      }
      return;
    }
    const uint2 id = *reinterpret_cast<const uint2*>(iring_p + 8 * t + io);
    if constexpr (masked) {
      const void* z1 = a.x;  // any valid address when nothing is copied
      cp_async_n<CP>(xs + xo, vb ? (const void*)(xb + (uint64_t)id.x * xrow) : z1, vb);
      cp_async_n<CP>(xs + xo + d1, vb ? (const void*)(xb + (uint64_t)id.y * xrow) : z1, vb);
      if constexpr (DUAL) {
        cp_async_n<CP>(xs + xo + SLOT, vb ? (const void*)(xb2 + (uint64_t)id.x * xrow2) : z1, vb);
        cp_async_n<CP>(xs + xo + SLOT + d1, vb ? (const void*)(xb2 + (uint64_t)id.y * xrow2) : z1,
                       vb);
      }
      return;
    }
    cp_async<CP>(xs + xo, xb + (uint64_t)id.x * xrow);
    cp_async<CP>(xs + xo + d1, xb + (uint64_t)id.y * xrow);
    if constexpr (DUAL) {
      cp_async<CP>(xs + xo + SLOT, xb2 + (uint64_t)id.x * xrow2);
      cp_async<CP>(xs + xo + SLOT + d1, xb2 + (uint64_t)id.y * xrow2);
    }
  };
  auto issue_x = [&](uint32_t xo, uint32_t io) {
    if constexpr (PAIR && NT == 4) {
      issue_block(xo, io);
      issue_block(xo + SLOT * C::OPS, io + 32);
    } else {
      issue_block(xo, io);
    }
  };
  constexpr int IS = 32 * KB;  // id bytes per step (lanes 0 .. 2KB-1 copy 16 B each)
  if (lane < 2 * KB)
    for (int s = 0; s < NI - NB; ++s) cp_async<16>(is + s * IS, csl + IS * s);
  cp_commit();
  cp_wait<0>();
  __syncwarp();
  for (int s = 0; s < NB; ++s) {
    issue_x(s * C::STEP, s * IS);
    if (lane < 2 * KB) cp_async<16>(is + (s + NI - NB) * IS, csl + IS * (s + NI - NB));
    cp_commit();
  }
  // ring cursors of the consumed step s: X slot, id slot of s + NB, id slot of s + NI
  uint32_t xo = 0, io = NB * IS, iw = 0;
  const char* cnext = csl + IS * NI;

  // ---- window metadata, rolled 3 windows ahead ----
  auto ptr_of = [&](int w) { return (int64_t)__ldg(a.ptr + min((int64_t)w * 16, a.n)); };
  auto blk_of = [&](int w) { return __ldg(a.boff + min(w, a.win_end)) - gb0; };
  int cb0 = 0, cb1 = blk_of(ws + 1), nb2 = blk_of(ws + 2), nb3 = blk_of(ws + 3);
  int64_t e0 = ptr_of(ws), e1 = ptr_of(ws + 1), e2 = ptr_of(ws + 2), e3 = ptr_of(ws + 3);
  // next window's edges (pf/pw) and the current window's (of/ow), in registers
  uint32_t pf[kEPL], of[kEPL];
  float pw[kEPL], pw2[kEPL], ow[kEPL], ow2[kEPL];
  auto weight = [&](const float* w, const uint32_t* widx, int64_t e) {
    return w ? (widx ? __ldg(w + __ldg(widx + e)) : __ldg(w + e)) : 1.f;
  };
  auto prefetch = [&](int64_t lo, int64_t hi) {
#pragma unroll
    for (int k = 0; k < kEPL; ++k) {
      const int64_t e = lo + lane + 32 * k;
      const bool ok = e < hi;
      pf[k] = ok ? __ldg(a.efrag + e) : 0xffffffffu;
      pw[k] = ok ? weight(a.w, a.widx, e) : 0.f;
      if constexpr (DUAL) pw2[k] = ok ? weight(a.w2, a.widx2, e) : 0.f;
    }
  };
  auto clear_frags = [&]() {
    __syncwarp();
#pragma unroll
    for (int q = 0; q < MB * C::OPS; ++q) reinterpret_cast<uint4*>(afr)[q * 32 + lane] = make_uint4(0, 0, 0, 0);
    __syncwarp();
  };
  // InitSparse for round [lo, lo + RS) of the current window's slots from registers
  auto put_round = [&](uint32_t lo, bool zero) {
#pragma unroll
    for (int k = 0; k < kEPL; ++k) {
      const uint32_t f = of[k] - lo;
      if (f < RS) {
        afr[f] = zero ? 0u : tf32_rn(ow[k]);
        if constexpr (DUAL) afr2[f] = zero ? 0u : tf32_rn(ow2[k]);
      }
    }
  };
  // BIG: copy the edges of [lo, hi) into staging slot `slot` (cp.async, own group);
  // returns false when they do not fit (the window then reads global memory)
  auto stage_edges = [&](int64_t lo, int64_t hi, int slot) -> bool {
    if constexpr (BIG) {
      const int64_t ne = hi - lo;
      if (ne > C::EMAX || a.widx || (DUAL && a.widx2)) return false;
      const uint32_t sb = smem_u32(ebuf) + slot * C::EMAX * 4 * (1 + C::OPS);
      for (int j = lane; j < ne; j += 32) {
        cp_async<4>(sb + 4 * j, a.efrag + lo + j);
        if (a.w) cp_async<4>(sb + 4 * (C::EMAX + j), a.w + lo + j);
        if constexpr (DUAL)
          if (a.w2) cp_async<4>(sb + 4 * (2 * C::EMAX + j), a.w2 + lo + j);
      }
      cp_commit();
      return true;
    }
    return false;
  };
  // Staged windows are consumed round by round (MB blocks each). Within a row the
  // edges are sorted by column, hence by block, so every row's edges of round k
  // follow its edges of round k-1: two lanes per row walk their row with a
  // cursor instead of rescanning the whole window each round.
  int rc_cur = 0, rc_end = 0;  // this lane's cursor into its row's staged edges
  auto rows_begin = [&](int64_t wbase_e, int w) {
    const int row = lane >> 1;
    const int64_t r = (int64_t)w * 16 + row;
    const int64_t rb = r < a.n ? __ldg(a.ptr + r) : wbase_e;
    const int64_t re = r < a.n ? __ldg(a.ptr + r + 1) : wbase_e;
    rc_cur = (int)(rb - wbase_e) + (lane & 1);
    rc_end = (int)(re - wbase_e);
  };
  auto round_from_stage = [&](int r0, int slot) {
    clear_frags();
    const uint32_t* ef = reinterpret_cast<const uint32_t*>(ebuf + slot * C::EMAX * 4 * (1 + C::OPS));
    const float* ew = reinterpret_cast<const float*>(ef + C::EMAX);
    const uint32_t lo = (uint32_t)(r0 * 128);
    while (rc_cur < rc_end) {
      const uint32_t f = ef[rc_cur] - lo;
      if (f >= RS) break;  // this row's next edges belong to a later round
      afr[f] = tf32_rn(a.w ? ew[rc_cur] : 1.f);
      if constexpr (DUAL) afr2[f] = tf32_rn(a.w2 ? ew[C::EMAX + rc_cur] : 1.f);
      rc_cur += 2;
    }
    __syncwarp();
  };
  auto hub_load = [&](int r0) {  // windows with more than 32*kEPL edges
    clear_frags();
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const uint32_t f = __ldg(a.efrag + e) - (uint32_t)(r0 * 128);
      if (f < RS) {
        afr[f] = tf32_rn(weight(a.w, a.widx, e));
        if constexpr (DUAL) afr2[f] = tf32_rn(weight(a.w2, a.widx2, e));
      }
    }
    __syncwarp();
  };
  clear_frags();
  prefetch(e0, e1);
  int eslot = 0;
  bool staged = BIG ? stage_edges(e0, e1, 0) : false;
  int stage_age = 0;  // block groups committed since the current staging group

  const uint32_t as = smem_u32(afr) + lane * 16;
  float acc[NT][4];
  auto store = [&](int wv) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t r = (int64_t)wv * 16 + g + 8 * h;
      if (r >= a.n) continue;
      float o[2 * NT];
#pragma unroll
      for (int j = 0; j < NT; ++j) o[j] = acc[j][2 * h] + 0.f, o[NT + j] = acc[j][2 * h + 1] + 0.f;
      const int fo = d0 + 2 * t * NT;
      float* yr = a.y + (r - a.y_row0) * a.ldy + fo;
      if (a.bias) {
#pragma unroll
        for (int q = 0; q < 2 * NT; ++q)
          if (!MASK || 2 * t * NT + q < a.dv) o[q] += __ldg(a.bias + fo + q);
      }
      if (a.accumulate) {
#pragma unroll
        for (int q = 0; q < 2 * NT; ++q)
          if (!MASK || 2 * t * NT + q < a.dv) o[q] += yr[q];
      }
      if (a.relu) {
#pragma unroll
        for (int q = 0; q < 2 * NT; ++q) o[q] = fmaxf(o[q], 0.f);
      }
      if (MASK || !a.vec_out) {
        // lane t holds chunk features 2t NT .. 2t NT + 2NT
#pragma unroll
        for (int q = 0; q < 2 * NT; ++q)
          if (!MASK || 2 * t * NT + q < a.dv) yr[q] = o[q];
      } else if constexpr (NT == 4) {
        reinterpret_cast<float4*>(yr)[0] = make_float4(o[0], o[1], o[2], o[3]);
        reinterpret_cast<float4*>(yr)[1] = make_float4(o[4], o[5], o[6], o[7]);
      } else if constexpr (NT == 2) {
        reinterpret_cast<float4*>(yr)[0] = make_float4(o[0], o[1], o[2], o[3]);
      } else {
        reinterpret_cast<float2*>(yr)[0] = make_float2(o[0], o[1]);
      }
    }
  };

  for (int w = ws; w < we; ++w) {
    const int nbw = cb1 - cb0;
    const bool hub = e1 - e0 > 32 * kEPL;
    const bool from_stage = BIG && hub && staged;
    const int cur_slot = eslot;
#pragma unroll
    for (int k = 0; k < kEPL; ++k) {
      of[k] = pf[k], ow[k] = pw[k];
      if constexpr (DUAL) ow2[k] = pw2[k];
    }
    __syncwarp();
    if (!hub) {
      put_round(0, false);
      __syncwarp();
    } else if (from_stage) {
      // the staging group was committed before the previous window's nbw block
      // groups; after >= NB of them the per-step wait has already retired it
      if (stage_age < NB) cp_wait<0>();
      __syncwarp();
      rows_begin(e0, w);
      round_from_stage(0, cur_slot);
    } else {
      hub_load(0);
    }
    prefetch(e1, e2);
    if constexpr (BIG) {
      eslot ^= 1;
      staged = (e2 - e1 > 32 * kEPL) ? stage_edges(e1, e2, eslot) : false;
      stage_age = nbw;  // this window's block steps follow the new staging group
    }
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
    for (int r0 = 0; r0 < nbw; r0 += MB) {
      if (r0 > 0) {  // next round of fragment blocks
        if (!hub) {
          __syncwarp();
          put_round((uint32_t)(r0 - MB) * 128, true);
          __syncwarp();
          put_round((uint32_t)r0 * 128, false);
          __syncwarp();
        } else if (from_stage) {
          round_from_stage(r0, cur_slot);
        } else {
          hub_load(r0);
        }
      }
      const int rend = min(nbw, r0 + MB);
      uint32_t fa = as;
      for (int lb = r0; lb < rend; lb += KB, fa += 512 * KB) {
        cp_wait<NB - 1>();
        __syncwarp();  // ids copied by lanes 0-1 visible to the warp
#pragma unroll
        for (int kb = 0; kb < KB; ++kb) {  // block kb of the step at kb * SLOT * OPS
          {
            float x0[NT], x1[NT];
            lds_slice<NT>(x0, xs + xo + kb * SLOT * C::OPS);
            lds_slice<NT>(x1, xs + xo + kb * SLOT * C::OPS + d1);
            const uint4 af = lds_frag(fa + kb * 512);
#pragma unroll
            for (int j = 0; j < NT; ++j) mma_tf32_rb(acc[j], af.x, af.y, af.z, af.w, x0[j], x1[j]);
          }
          if constexpr (DUAL) {
            float x0[NT], x1[NT];
            lds_slice<NT>(x0, xs + xo + kb * SLOT * C::OPS + SLOT);
            lds_slice<NT>(x1, xs + xo + kb * SLOT * C::OPS + SLOT + d1);
            const uint4 af = lds_frag(fa + kb * 512 + MB * 512);
#pragma unroll
            for (int j = 0; j < NT; ++j) mma_tf32_b<X2R>(acc[j], af.x, af.y, af.z, af.w, x0[j], x1[j]);
          }
        }
        // refill: X of block s + NB into this slot, ids of block s + 2NB. The
        // 16-wide path's lanes read slices copied by other lanes: all reads of
        // this slot must be done before any lane re-fills it (racecheck)
        if constexpr (NT == 2) {
          if (a.x16) __syncwarp();
        }
        issue_x(xo, io);
        if (lane < 2 * KB) cp_async<16>(is + iw, cnext);
        cp_commit();
        cnext += IS;
        xo = (xo + C::STEP) & (NB * C::STEP - 1);
        io = (io + IS) & (NI * IS - 1);
        iw = (iw + IS) & (NI * IS - 1);
      }
    }
    store(w);
    // un-scatter this window's last round
    __syncwarp();
    if (!hub) {
      put_round((uint32_t)(nbw > 0 ? ((nbw - 1) & ~(MB - 1)) : 0) * 128, true);
    } else {
      clear_frags();
    }
    cb0 = cb1, cb1 = nb2, nb2 = nb3, nb3 = blk_of(w + 4);
    e0 = e1, e1 = e2, e2 = e3, e3 = ptr_of(w + 4);
  }
  cp_wait<0>();
}

// ---- TMA-gather block stream (round 2) -----------------------------------------
//
// The neighbour rows of a block are fetched by two TMA tile::gather4 loads
// (UTMALDG.GATHER4: 4 rows of the 2-D tensor map each) straight into a per-warp
// shared-memory ring with an mbarrier per slot, so the gather bypasses the L1
// data pipe and the registers: the bytes in flight live in shared memory
// (NS KB per warp) and a block costs two single-lane TMA instructions. The
// column ids of block s + NI are copied (cp.async, 16 B by lanes 0-1) NS steps
// before the gathers that use them. The ring slot of a block holds its rows in
// the column stream's pair-interleaved order (c0 c4 c1 c5 | c2 c6 c3 c7), so
// mma lane (g, t) reads k-rows t / t+4 from slot rows 2t / 2t+1; with the
// 128-B TMA swizzle (chunk ^= row) these LDS.128 are conflict-free.
template <int MB_, int NS_>
struct TmaCfg {
  static constexpr int MB = MB_, NS = NS_, NI = 2 * NS_;
  static_assert((NI & (NI - 1)) == 0 && NI <= TCG_STREAM_PAD, "id ring depth");
  static constexpr int RING = NS * 1024;
  static constexpr int AFR = MB * 512;
  static constexpr int IDX = NI * 32;
  static constexpr int BAR = NS * 8;
  static constexpr int WARP = (RING + AFR + IDX + BAR + 1023) & ~1023;
  static constexpr int WPC = 4;
  static constexpr int SMEM = WPC * WARP + 1024;  // + alignment slack
};

__device__ __forceinline__ void mbar_init(uint32_t bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nTCG_MBW:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra TCG_MBW;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap* tm, int x, uint4 rows,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(rows.x), "r"(rows.y), "r"(rows.z), "r"(rows.w),
      "r"(bar)
      : "memory");
}

template <int MB_, int NS_>
__global__ void __launch_bounds__(TmaCfg<MB_, NS_>::WPC * 32)
    spmm_tma(const Args a, const __grid_constant__ CUtensorMap tmx) {
  using C = TmaCfg<MB_, NS_>;
  constexpr int MB = C::MB, NS = C::NS, NI = C::NI;
  constexpr uint32_t RS = MB * 128;
  extern __shared__ unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int gw = blockIdx.x * C::WPC + wid;
  const int g = lane >> 2, t = lane & 3;
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t ring = base + wid * C::WARP;
  const uint32_t afr_s = ring + C::RING;
  uint32_t* afr = reinterpret_cast<uint32_t*>(smem_raw + (afr_s - smem_u32(smem_raw)));
  const uint32_t iring = afr_s + C::AFR;
  const unsigned char* iring_p = smem_raw + (iring - smem_u32(smem_raw));
  const uint32_t bars = iring + C::IDX;

  const int B0 = __ldg(a.boff + a.win_begin), B1 = __ldg(a.boff + a.win_end);
  const int64_t TBr = B1 - B0;
  const int lo_b = B0 + (int)(TBr * gw / a.nwarps);
  const int hi_b = B0 + (int)(TBr * (gw + 1) / a.nwarps);
  const int ws = warp_lower_bound(a.boff, a.win_begin, a.win_end, lo_b);
  const int we = gw + 1 == a.nwarps ? a.win_end : warp_lower_bound(a.boff, ws, a.win_end, hi_b);
  if (ws >= we) return;
  const int gb0 = __ldg(a.boff + ws);
  const int nb = __ldg(a.boff + we) - gb0;
  const int xcol = a.d0 + blockIdx.y * 32;

  if (lane == 0) {
    for (int q = 0; q < NS; ++q) mbar_init(bars + 8 * q, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  // ids: lanes 0-1 copy 16 B (half a block) each; each lane only reads back its own
  const char* csl = reinterpret_cast<const char*>(a.cs + 8 * (int64_t)gb0) + 16 * lane;
  const uint32_t is = iring + 16 * lane;
  auto copy_ids = [&](int b) {
    if (lane < 2) cp_async<16>(is + (b & (NI - 1)) * 32, csl + 32 * (int64_t)b);
  };
  auto issue_rows = [&](int b) {  // after the ids of block b have landed
    if (lane < 2 && b < nb) {
      const uint4 r = *reinterpret_cast<const uint4*>(iring_p + (b & (NI - 1)) * 32 + 16 * lane);
      const uint32_t bar = bars + 8 * (b % NS);
      if (lane == 0) mbar_expect_tx(bar, 1024);
      tma_gather4(ring + (b % NS) * 1024 + 512 * lane, &tmx, xcol, r, bar);
    }
  };
  for (int b = 0; b < NS; ++b) copy_ids(b);
  cp_commit();
  cp_wait<0>();
  for (int b = 0; b < NS; ++b) issue_rows(b);
  for (int b = NS; b < NI; ++b) {
    copy_ids(b);
    cp_commit();
  }

  auto ptr_of = [&](int w) { return (int64_t)__ldg(a.ptr + min((int64_t)w * 16, a.n)); };
  auto blk_of = [&](int w) { return __ldg(a.boff + min(w, a.win_end)) - gb0; };
  int w = ws;
  int cb0 = 0, cb1 = blk_of(ws + 1), nb2 = blk_of(ws + 2), nb3 = blk_of(ws + 3);
  int64_t e0 = ptr_of(ws), e1 = ptr_of(ws + 1), e2 = ptr_of(ws + 2), e3 = ptr_of(ws + 3);
  uint32_t pf[kEPL], of[kEPL];
  float pw[kEPL], ow[kEPL];
  auto weight = [&](int64_t e) {
    return a.w ? (a.widx ? __ldg(a.w + __ldg(a.widx + e)) : __ldg(a.w + e)) : 1.f;
  };
  auto prefetch = [&](int64_t lo, int64_t hi) {
#pragma unroll
    for (int k = 0; k < kEPL; ++k) {
      const int64_t e = lo + lane + 32 * k;
      const bool ok = e < hi;
      pf[k] = ok ? __ldg(a.efrag + e) : 0xffffffffu;
      pw[k] = ok ? weight(e) : 0.f;
    }
  };
  auto clear_frags = [&]() {
    __syncwarp();
#pragma unroll
    for (int q = 0; q < MB; ++q) reinterpret_cast<uint4*>(afr)[q * 32 + lane] = make_uint4(0, 0, 0, 0);
    __syncwarp();
  };
  auto put_round = [&](uint32_t lo, bool zero) {
#pragma unroll
    for (int k = 0; k < kEPL; ++k) {
      const uint32_t f = of[k] - lo;
      if (f < RS) afr[f] = zero ? 0u : tf32_rn(ow[k]);
    }
  };
  auto hub_load = [&](int r0) {
    clear_frags();
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const uint32_t f = __ldg(a.efrag + e) - (uint32_t)(r0 * 128);
      if (f < RS) afr[f] = tf32_rn(weight(e));
    }
    __syncwarp();
  };
  float acc[4][4];
  auto store = [&]() {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t r = (int64_t)w * 16 + g + 8 * h;
      if (r >= a.n) continue;
      float o[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) o[j] = acc[j][2 * h] + 0.f, o[4 + j] = acc[j][2 * h + 1] + 0.f;
      const int fo = xcol + 8 * t;
      float* yr = a.y + (r - a.y_row0) * a.ldy + fo;
      if (a.bias) {
#pragma unroll
        for (int q = 0; q < 8; ++q) o[q] += __ldg(a.bias + fo + q);
      }
      if (a.accumulate) {
#pragma unroll
        for (int q = 0; q < 8; ++q) o[q] += yr[q];
      }
      if (!a.vec_out) {
#pragma unroll
        for (int q = 0; q < 8; ++q) yr[q] = o[q];
      } else {
        reinterpret_cast<float4*>(yr)[0] = make_float4(o[0], o[1], o[2], o[3]);
        reinterpret_cast<float4*>(yr)[1] = make_float4(o[4], o[5], o[6], o[7]);
      }
    }
  };
  bool hub = false;
  auto begin_window = [&]() {
#pragma unroll
    for (int k = 0; k < kEPL; ++k) of[k] = pf[k], ow[k] = pw[k];
    hub = e1 - e0 > 32 * kEPL;
    __syncwarp();
    if (!hub) {
      put_round(0, false);
      __syncwarp();
    } else {
      hub_load(0);
    }
    prefetch(e1, e2);
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
  };
  auto end_window = [&]() {
    store();
    const int nbw = cb1 - cb0;
    __syncwarp();
    if (!hub) {
      put_round((uint32_t)(nbw > 0 ? ((nbw - 1) & ~(MB - 1)) : 0) * 128, true);
    } else {
      clear_frags();
    }
    ++w;
    cb0 = cb1, cb1 = nb2, nb2 = nb3, nb3 = blk_of(w + 3);
    e0 = e1, e1 = e2, e2 = e3, e3 = ptr_of(w + 3);
  };

  // lane (g, t): k-row t is slot row 2t, k-row t+4 is slot row 2t+1 (128-B swizzle)
  const uint32_t b0o = (2 * t) * 128 + ((g ^ (2 * t)) & 7) * 16;
  const uint32_t b1o = (2 * t + 1) * 128 + ((g ^ (2 * t + 1)) & 7) * 16;
  const uint32_t as = afr_s + lane * 16;
  clear_frags();
  prefetch(e0, e1);
  begin_window();
  for (int s = 0; s < nb; ++s) {
    while (s == cb1) {
      end_window();
      begin_window();
    }
    const int lb = s - cb0;
    if (lb > 0 && (lb & (MB - 1)) == 0) {
      if (!hub) {
        __syncwarp();
        put_round((uint32_t)(lb - MB) * 128, true);
        __syncwarp();
        put_round((uint32_t)lb * 128, false);
        __syncwarp();
      } else {
        hub_load(lb);
      }
    }
    const uint32_t slot = ring + (s % NS) * 1024;
    mbar_wait(bars + 8 * (s % NS), (uint32_t)(s / NS) & 1u);
    {
      float x0[4], x1[4];
      lds_slice<4>(x0, slot + b0o);
      lds_slice<4>(x1, slot + b1o);
      const uint4 af = lds_frag(as + (uint32_t)(lb & (MB - 1)) * 512);
#pragma unroll
      for (int j = 0; j < 4; ++j) mma_tf32_rb(acc[j], af.x, af.y, af.z, af.w, x0[j], x1[j]);
    }
    __syncwarp();
    // refill this slot: ids of block s + NS (copied NS steps ago), then ids of s + NI
    cp_wait<NS - 1>();
    issue_rows(s + NS);
    copy_ids(s + NI);
    cp_commit();
  }
  for (;;) {
    end_window();
    if (w >= we) break;
    begin_window();
  }
  cp_wait<0>();
}

template <int MB, int NS>
int launch_tma(Args& a, const CUtensorMap& tm, int nchunks, cudaStream_t s) {
  using C = TmaCfg<MB, NS>;
  auto kern = spmm_tma<MB, NS>;
  static int configured = -1;
  int dev = 0;
  TCG_CUDA(cudaGetDevice(&dev), "spmm_tma device");
  if (configured != dev) {
    TCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM),
             "spmm_tma attr");
    configured = dev;
  }
  int per_sm = 1;
  TCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::WPC * 32, C::SMEM),
           "spmm_tma occupancy");
  if (per_sm < 1) per_sm = 1;
  const int64_t ctas = (int64_t)num_sms() * per_sm;
  a.nwarps = (int)(ctas * C::WPC);
  dim3 grid((unsigned)ctas, (unsigned)nchunks);
  kern<<<grid, C::WPC * 32, C::SMEM, s>>>(a, tm);
  TCG_LAUNCHED("spmm_tma");
  return TCG_OK;
}

// ---- warp-specialised TMA gather (round 2) --------------------------------------
//
// spmm_tma above makes every consumer warp issue its own gathers, so the TMA issue
// (a waterfall over the lanes holding row ids) and the id copies sit on the same
// serial chain as the mma. Here one producer warp per CTA issues the gathers of
// all NCW consumer warps: producer lane c walks consumer c's contiguous slice of
// the block stream, polls the slot's `empty` barrier (non-blocking), and issues
// the block's two tile::gather4 (8 rows, 1 KB) with complete_tx on `full`. The
// consumers only wait, read two LDS.128 + one fragment LDS.128 and run the 4 mma.
// Row layout in a slot and the 128-B swizzle are those of spmm_tma.
template <int NCW_, int NS_, int MB_>
struct WsCfg {
  static constexpr int NCW = NCW_, NS = NS_, MB = MB_;
  static constexpr int RING = NS * 1024;
  static constexpr int AFR = MB * 512;
  static constexpr int WARP = (RING + AFR + 1023) & ~1023;
  static constexpr int BARS = 2 * NCW * NS * 8;
  static constexpr int THREADS = (NCW + 1) * 32;
  static constexpr int SMEM = NCW * WARP + BARS + 1024;
};

__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

template <int NCW_, int NS_, int MB_, int MINB>
__global__ void __launch_bounds__(WsCfg<NCW_, NS_, MB_>::THREADS, MINB)
    spmm_ws(const Args a, const __grid_constant__ CUtensorMap tmx) {
  using C = WsCfg<NCW_, NS_, MB_>;
  constexpr int NCW = C::NCW, NS = C::NS, MB = C::MB;
  constexpr uint32_t RS = MB * 128;
  extern __shared__ unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t bars = base + NCW * C::WARP;  // full[c][s], then empty[c][s]
  auto full_bar = [&](int c, int s) { return bars + 8u * (uint32_t)(c * NS + s); };
  auto empty_bar = [&](int c, int s) { return bars + 8u * (uint32_t)(NCW * NS + c * NS + s); };
  if (threadIdx.x == 0) {
    for (int q = 0; q < 2 * NCW * NS; ++q) mbar_init(bars + 8 * q, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int B0 = __ldg(a.boff + a.win_begin), B1 = __ldg(a.boff + a.win_end);
  const int64_t TBr = B1 - B0;
  // window range of consumer gw (whole warp)
  auto range_of = [&](int gw, int& ws, int& we) {
    const int lo_b = B0 + (int)(TBr * gw / a.nwarps);
    const int hi_b = B0 + (int)(TBr * (gw + 1) / a.nwarps);
    ws = warp_lower_bound(a.boff, a.win_begin, a.win_end, lo_b);
    we = gw + 1 == a.nwarps ? a.win_end : warp_lower_bound(a.boff, ws, a.win_end, hi_b);
    if (we < ws) we = ws;
  };
  const int xcol = a.d0 + blockIdx.y * 32;

  if (wid == NCW) {
    // ---- producer: lane c serves consumer c ----
    int my_gb0 = 0, my_nb = 0;
    for (int c = 0; c < NCW; ++c) {
      int ws, we;
      range_of(blockIdx.x * NCW + c, ws, we);
      if (lane == c && ws < we) {
        my_gb0 = __ldg(a.boff + ws);
        my_nb = __ldg(a.boff + we) - my_gb0;
      }
    }
    const int c = lane < NCW ? lane : 0;
    const uint4* ids = reinterpret_cast<const uint4*>(a.cs + 8 * (int64_t)my_gb0);
    const uint32_t ring = base + c * C::WARP;
    int b = 0;
    uint4 r0 = make_uint4(0, 0, 0, 0), r1 = r0;
    if (my_nb > 0) r0 = __ldg(ids), r1 = __ldg(ids + 1);
    while (__any_sync(0xffffffffu, b < my_nb)) {
      if (b < my_nb) {
        const int s = b % NS;
        const bool ready = b < NS || mbar_test(empty_bar(c, s), (uint32_t)((b / NS) - 1) & 1u);
        if (ready) {
          const uint32_t fb = full_bar(c, s);
          mbar_expect_tx(fb, 1024);
          tma_gather4(ring + s * 1024, &tmx, xcol, r0, fb);
          tma_gather4(ring + s * 1024 + 512, &tmx, xcol, r1, fb);
          ++b;
          if (b < my_nb) r0 = __ldg(ids + 2 * b), r1 = __ldg(ids + 2 * b + 1);
        }
      }
    }
    return;
  }

  // ---- consumer warp `wid` ----
  int ws, we;
  range_of(blockIdx.x * NCW + wid, ws, we);
  if (ws >= we) return;
  const int g = lane >> 2, t = lane & 3;
  const uint32_t ring = base + wid * C::WARP;
  const uint32_t afr_s = ring + C::RING;
  uint32_t* afr = reinterpret_cast<uint32_t*>(smem_raw + (afr_s - smem_u32(smem_raw)));
  const int gb0 = __ldg(a.boff + ws);
  const int nb = __ldg(a.boff + we) - gb0;

  auto ptr_of = [&](int w) { return (int64_t)__ldg(a.ptr + min((int64_t)w * 16, a.n)); };
  auto blk_of = [&](int w) { return __ldg(a.boff + min(w, a.win_end)) - gb0; };
  int w = ws;
  int cb0 = 0, cb1 = blk_of(ws + 1), nb2 = blk_of(ws + 2), nb3 = blk_of(ws + 3);
  int64_t e0 = ptr_of(ws), e1 = ptr_of(ws + 1), e2 = ptr_of(ws + 2), e3 = ptr_of(ws + 3);
  uint32_t pf[kEPL], of[kEPL];
  float pw[kEPL], ow[kEPL];
  auto weight = [&](int64_t e) {
    return a.w ? (a.widx ? __ldg(a.w + __ldg(a.widx + e)) : __ldg(a.w + e)) : 1.f;
  };
  auto prefetch = [&](int64_t lo, int64_t hi) {
#pragma unroll
    for (int k = 0; k < kEPL; ++k) {
      const int64_t e = lo + lane + 32 * k;
      const bool ok = e < hi;
      pf[k] = ok ? __ldg(a.efrag + e) : 0xffffffffu;
      pw[k] = ok ? weight(e) : 0.f;
    }
  };
  auto clear_frags = [&]() {
    __syncwarp();
#pragma unroll
    for (int q = 0; q < MB; ++q) reinterpret_cast<uint4*>(afr)[q * 32 + lane] = make_uint4(0, 0, 0, 0);
    __syncwarp();
  };
  auto put_round = [&](uint32_t lo, bool zero) {
#pragma unroll
    for (int k = 0; k < kEPL; ++k) {
      const uint32_t f = of[k] - lo;
      if (f < RS) afr[f] = zero ? 0u : tf32_rn(ow[k]);
    }
  };
  auto hub_load = [&](int r0) {
    clear_frags();
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const uint32_t f = __ldg(a.efrag + e) - (uint32_t)(r0 * 128);
      if (f < RS) afr[f] = tf32_rn(weight(e));
    }
    __syncwarp();
  };
  float acc[4][4];
  auto store = [&]() {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t r = (int64_t)w * 16 + g + 8 * h;
      if (r >= a.n) continue;
      float o[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) o[j] = acc[j][2 * h] + 0.f, o[4 + j] = acc[j][2 * h + 1] + 0.f;
      const int fo = xcol + 8 * t;
      float* yr = a.y + (r - a.y_row0) * a.ldy + fo;
      if (a.bias) {
#pragma unroll
        for (int q = 0; q < 8; ++q) o[q] += __ldg(a.bias + fo + q);
      }
      if (a.accumulate) {
#pragma unroll
        for (int q = 0; q < 8; ++q) o[q] += yr[q];
      }
      if (a.relu) {
#pragma unroll
        for (int q = 0; q < 8; ++q) o[q] = fmaxf(o[q], 0.f);
      }
      if (!a.vec_out) {
#pragma unroll
        for (int q = 0; q < 8; ++q) yr[q] = o[q];
      } else {
        reinterpret_cast<float4*>(yr)[0] = make_float4(o[0], o[1], o[2], o[3]);
        reinterpret_cast<float4*>(yr)[1] = make_float4(o[4], o[5], o[6], o[7]);
      }
    }
  };
  bool hub = false;
  auto begin_window = [&]() {
#pragma unroll
    for (int k = 0; k < kEPL; ++k) of[k] = pf[k], ow[k] = pw[k];
    hub = e1 - e0 > 32 * kEPL;
    __syncwarp();
    if (!hub) {
      put_round(0, false);
      __syncwarp();
    } else {
      hub_load(0);
    }
    prefetch(e1, e2);
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
  };
  auto end_window = [&]() {
    store();
    const int nbw = cb1 - cb0;
    __syncwarp();
    if (!hub) {
      put_round((uint32_t)(nbw > 0 ? ((nbw - 1) & ~(MB - 1)) : 0) * 128, true);
    } else {
      clear_frags();
    }
    ++w;
    cb0 = cb1, cb1 = nb2, nb2 = nb3, nb3 = blk_of(w + 3);
    e0 = e1, e1 = e2, e2 = e3, e3 = ptr_of(w + 3);
  };

  const uint32_t b0o = (2 * t) * 128 + ((g ^ (2 * t)) & 7) * 16;
  const uint32_t b1o = (2 * t + 1) * 128 + ((g ^ (2 * t + 1)) & 7) * 16;
  const uint32_t as = afr_s + lane * 16;
  clear_frags();
  prefetch(e0, e1);
  begin_window();
  for (int s = 0; s < nb; ++s) {
    while (s == cb1) {
      end_window();
      begin_window();
    }
    const int lb = s - cb0;
    if (lb > 0 && (lb & (MB - 1)) == 0) {
      if (!hub) {
        __syncwarp();
        put_round((uint32_t)(lb - MB) * 128, true);
        __syncwarp();
        put_round((uint32_t)lb * 128, false);
        __syncwarp();
      } else {
        hub_load(lb);
      }
    }
    const int sl = s % NS;
    const uint32_t slot = ring + sl * 1024;
    mbar_wait(full_bar(wid, sl), (uint32_t)(s / NS) & 1u);
    {
      float x0[4], x1[4];
      lds_slice<4>(x0, slot + b0o);
      lds_slice<4>(x1, slot + b1o);
      const uint4 af = lds_frag(as + (uint32_t)(lb & (MB - 1)) * 512);
#pragma unroll
      for (int j = 0; j < 4; ++j) mma_tf32_rb(acc[j], af.x, af.y, af.z, af.w, x0[j], x1[j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty_bar(wid, sl));
  }
  for (;;) {
    end_window();
    if (w >= we) break;
    begin_window();
  }
}

template <int NCW, int NS, int MB, int MINB>
int launch_ws(Args& a, const CUtensorMap& tm, int nchunks, cudaStream_t s) {
  using C = WsCfg<NCW, NS, MB>;
  auto kern = spmm_ws<NCW, NS, MB, MINB>;
  static int configured = -1;
  int dev = 0;
  TCG_CUDA(cudaGetDevice(&dev), "spmm_ws device");
  if (configured != dev) {
    TCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM),
             "spmm_ws attr");
    configured = dev;
  }
  int per_sm = 1;
  TCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::THREADS, C::SMEM),
           "spmm_ws occupancy");
  if (per_sm < 1) per_sm = 1;
  const int64_t ctas = (int64_t)num_sms() * per_sm;
  a.nwarps = (int)(ctas * NCW);
  dim3 grid((unsigned)ctas, (unsigned)nchunks);
  kern<<<grid, C::THREADS, C::SMEM, s>>>(a, tm);
  TCG_LAUNCHED("spmm_ws");
  return TCG_OK;
}

// 2-D tensor map over X (rows = nodes, inner = features), 32-feature boxes of one
// row, 128-B swizzle: the operand of tile::gather4. false when it cannot be made.
bool make_row_map(CUtensorMap* tm, const float* x, int64_t rows, int64_t dim, int64_t ld) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  }();
  if (!enc || rows < 1 || rows >= (1LL << 31) || (reinterpret_cast<uintptr_t>(x) & 15) || (ld * 4) % 16)
    return false;
  cuuint64_t gd[2] = {(cuuint64_t)dim, (cuuint64_t)rows};
  cuuint64_t gs[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {32, 1}, es[2] = {1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(x), gd, gs, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ---- fused AGNN aggregation on the block stream (D = 32) -------------------
//
// Forward (reference kernels.agnn_layer, kernels.py:586-601):
//   S_e = <Z_i, Z_j> (TF32 mma; A = the window's own 16 rows in registers,
//   B = the staged neighbour rows), P = rowsoftmax(S), Y = A_P Z.
// One pass per window with an online (running-max) softmax: per block the
// scores are computed, the row maxima updated, the accumulator rescaled and
// the unnormalised probabilities fed straight into the SpMM mma. The SDDMM's
// 8 output columns are permuted (C column 2t <-> column t, 2t+1 <-> t+4) so
// its C fragment IS the SpMM's A fragment: no shuffles between the two mmas.
// Raw scores are kept per edge in shared memory; P_e = exp(S_e - m_i) / l_i
// is written at the window end.
//
// Backward, A-side half (no reference counterpart):
//   dP_e = <G_i, Z_j>, dS_e = P_e (dP_e - rs_i), dZ_i = sum_e dS_e Z_j with
//   rs_i = sum_j P_ij dP_ij = <G_i, Y_i> (Y = the forward output; the
//   FlashAttention D_i identity), so dS is exact per block and one pass does
//   both products.
struct AgnnArgs {
  const int64_t* ptr;
  const uint32_t* efrag;
  const int32_t* boff;
  const uint32_t* cs;
  int64_t n;
  int win_begin, win_end, nwarps;
  const float* z;    // gathered operand (neighbour rows)
  int64_t ldz;
  const float* za;   // own-row operand: Z (fwd) / G (bwd)
  int64_t lda;
  const float* yf;   // bwd: forward output Y (absolute rows)
  int64_t ldyf;
  const float* pin;  // bwd: P
  float* eout;       // fwd: P, bwd: dS
  float* y;          // fwd: Y, bwd: dZ (A-side)
  int64_t ldy, y_row0;
  int epi;           // SDDMM-only launches: TCG_EPI_*
  int dv;            // MASK launches: valid features (a multiple of 4, < 32); the rest read as 0
  const float* wn;   // NEXT (fwd): the next layer's W (32 x 32, row-major); zn = Y wn
  float* zn;
  int64_t ldzn;
};

constexpr float kTau = 8.f;  // lazy-rescale threshold of the online softmax (natural log)

// 2^x (MUFU.EX2, ~2 ulp; ftz). exp(-inf) = 0.
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

constexpr int kMapB = 24;   // blocks per window covered by the slot map (192 columns)
constexpr int kMaxE = 255;  // edges per window (u8 slot map)

template <int KIND>
struct AgnnCfg {
  static constexpr int NB = 4, NI = 8;
  static constexpr int RING = NB * 1024;
  static constexpr int IDX = NI * 32;
  static constexpr int MAP = kMapB * 128;      // u8 per fragment slot: local edge + 1
  static constexpr int ESC = 256 * 4;          // per-edge scores (fwd) / P (bwd)
  static constexpr int ROW = 64 * 4;           // row stats
  static constexpr int EROW = 256;             // fwd / SDDMM: window-local row of each edge (u8)
  static constexpr int WARP = RING + IDX + MAP + ESC + ROW + EROW;
  static constexpr int WPC = 8;
  static constexpr int SMEM = WPC * WARP;
};

// staged-row swizzle serving both fragment patterns: SpMM (rows t, t+4;
// chunk g) and the column-permuted SDDMM (row (g>>1) + 4(g&1); chunks t, t+4)
__device__ __forceinline__ uint32_t agnn_off(int r, int c) {
  const int h = ((2 * (r & 3)) ^ (4 * (r >> 2))) & 7;
  return r * 128 + ((c ^ h) & 7) * 16;
}

// MASK: D < 32 (a multiple of 4) run in the D = 32 layout with the missing
// features zero-filled by the copies (src-size 0) and never stored: the scores,
// softmax and products are those of the D-wide rows.
// NEXT (forward, D = 32): the epilogue also computes the next layer's dense step
// Zn = Y Wn (3xTF32 mma.sync; Y staged through the window's slot-map area, free
// at the window end; Wn as tf32 hi / lo after the warps' areas), so Y is not
// read back by a separate GEMM.
// ZR: the gathered operand z is already on the tf32 grid (no B-operand cvt)
template <int KIND, bool PAIR = false, bool MASK = false, bool NEXT = false, bool ZR = false>
__global__ void __launch_bounds__(AgnnCfg<KIND>::WPC * 32, 2) agnn_stream(const AgnnArgs a) {
  TCG_PDL_ENTRY();
  using C = AgnnCfg<KIND>;
  constexpr bool BWD = KIND == 1;   // 0: forward, 1: backward A-side, 2: SDDMM only
  constexpr int NB = C::NB, NI = C::NI;
  constexpr int KB = PAIR ? 2 : 1;  // blocks per step
  constexpr float kLog2e = 1.4426950408889634f;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int gw = blockIdx.x * C::WPC + wid;
  const int g = lane >> 2, t = lane & 3;
  unsigned char* wsm = smem + wid * C::WARP;
  const uint32_t ring = smem_u32(wsm);
  const uint32_t iring = ring + C::RING;
  const unsigned char* iring_p = wsm + C::RING;
  unsigned char* map = wsm + C::RING + C::IDX;
  float* esc = reinterpret_cast<float*>(map + C::MAP);
  float* rowm = esc + 256;   // [16] running max (fwd)
  float* rowl = rowm + 16;   // [16] 1 / row sum (fwd)
  float* rowrs = rowl + 16;  // [16] rs (bwd)
  unsigned char* erow = reinterpret_cast<unsigned char*>(esc + 256 + 64);  // [256] fwd
  // window-local row of fragment slot f: lane (g, t) = (f >> 2) & 31, register f & 3
  // holds rows g (even) / g + 8 (odd)
  auto slot_row = [](uint32_t f) { return (unsigned char)((((f >> 2) & 31u) >> 2) + 8u * (f & 1u)); };

  const int B0 = __ldg(a.boff + a.win_begin), B1 = __ldg(a.boff + a.win_end);
  const int64_t TBr = B1 - B0;
  const int lo_b = B0 + (int)(TBr * gw / a.nwarps);
  const int hi_b = B0 + (int)(TBr * (gw + 1) / a.nwarps);
  float* wnh = reinterpret_cast<float*>(smem + C::WPC * C::WARP);  // NEXT: [2][32][32]
  if constexpr (NEXT) {
    for (int i = threadIdx.x; i < 1024; i += C::WPC * 32) {
      const float v = __ldg(a.wn + i);
      const float hi = __uint_as_float(tf32_rn(v));
      wnh[i] = hi;
      wnh[1024 + i] = __uint_as_float(tf32_rn(v - hi));
    }
    __syncthreads();
  }
  const int ws = warp_lower_bound(a.boff, a.win_begin, a.win_end, lo_b);
  const int we = gw + 1 == a.nwarps ? a.win_end : warp_lower_bound(a.boff, ws, a.win_end, hi_b);
  if (ws >= we) return;
  const int gb0 = __ldg(a.boff + ws);

  const char* xb = reinterpret_cast<const char*>(a.z + g * 4);
  const uint32_t xrow = (uint32_t)a.ldz * 4u;  // 32 x 32 -> 64-bit IMAD.WIDE per address
  const uint32_t so0 = agnn_off(t, g), so1 = agnn_off(t + 4, g);             // SpMM reads/writes
  const int pr = (g >> 1) + 4 * (g & 1);                                      // SDDMM row
  const uint32_t sd0 = agnn_off(pr, t), sd1 = agnn_off(pr, t + 4);
  const uint32_t* csw = a.cs + 8 * (int64_t)gb0;
  auto issue_idx = [&](int s) {
    if (lane < 2) cp_async<16>(iring + (s & (NI - 1)) * 32 + lane * 16, csw + 8 * (int64_t)s + 4 * lane);
  };
  const int xvb = MASK ? (4 * g < a.dv ? 16 : 0) : 16;  // this lane's bytes of a row
  auto issue_x = [&](int s) {
    const uint2 id = *reinterpret_cast<const uint2*>(iring_p + (s & (NI - 1)) * 32 + 8 * t);
    const uint32_t sb = ring + (s & (NB - 1)) * 1024;
    if constexpr (MASK) {
      const void* z0 = a.z;  // any valid address when nothing is copied
      cp_async_n<16>(sb + so0, xvb ? (const void*)(xb + (uint64_t)id.x * xrow) : z0, xvb);
      cp_async_n<16>(sb + so1, xvb ? (const void*)(xb + (uint64_t)id.y * xrow) : z0, xvb);
    } else {
      cp_async<16>(sb + so0, xb + (uint64_t)id.x * xrow);
      cp_async<16>(sb + so1, xb + (uint64_t)id.y * xrow);
    }
  };
  for (int s = 0; s < NB; ++s) issue_idx(s);
  cp_commit();
  cp_wait<0>();
  __syncwarp();
  for (int s = 0; s < NB; ++s) {
    issue_x(s);
    issue_idx(s + NB);
    cp_commit();
  }

  auto ptr_of = [&](int w) { return (int64_t)__ldg(a.ptr + min((int64_t)w * 16, a.n)); };
  auto blk_of = [&](int w) { return __ldg(a.boff + min(w, a.win_end)) - gb0; };
  int cb0 = 0, cb1 = blk_of(ws + 1), nb2 = blk_of(ws + 2), nb3 = blk_of(ws + 3);
  int64_t e0 = ptr_of(ws), e1 = ptr_of(ws + 1), e2 = ptr_of(ws + 2), e3 = ptr_of(ws + 3);
  // own rows (A operand of the SDDMM) of the next window, prefetched raw:
  // lane (g,t): rows g, g+8; features 4t..4t+3 and 4(t+4)..4(t+4)+3
  float4 own[4], ownn[4], yfn[4];
  auto load_own = [&](int w, float4 (&o)[4], float4 (&yv)[4]) {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int64_t r = (int64_t)w * 16 + g + 8 * (h & 1);
      const int f = 4 * (t + 4 * (h >> 1));
      const bool ok = w < a.win_end && r < a.n && (!MASK || f < a.dv);
      o[h] = ok ? __ldg(reinterpret_cast<const float4*>(a.za + r * a.lda + f)) : make_float4(0.f, 0.f, 0.f, 0.f);
      if constexpr (BWD)
        yv[h] = ok ? __ldg(reinterpret_cast<const float4*>(a.yf + r * a.ldyf + f)) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  uint32_t pf[kEPL];
  float pp[kEPL];
  auto prefetch = [&](int64_t lo, int64_t hi) {
#pragma unroll
    for (int k = 0; k < kEPL; ++k) {
      const int64_t e = lo + lane + 32 * k;
      const bool ok = e < hi;
      pf[k] = ok ? __ldg(a.efrag + e) : 0xffffffffu;
      if constexpr (BWD) pp[k] = ok ? __ldg(a.pin + e) : 0.f;
    }
  };
  float4 yv[4];
  load_own(ws, ownn, yfn);
  prefetch(e0, e1);
  const uint32_t* map32 = reinterpret_cast<const uint32_t*>(map);

  int s = 0;
  for (int w = ws; w < we; ++w) {
    const int nbw = cb1 - cb0;
    const int ne = (int)(e1 - e0);
    // ---- InitSparse: slot map (local edge + 1), per-edge P (bwd) ----
    __syncwarp();
    for (int q = lane; q < kMapB * 8; q += 32) reinterpret_cast<uint4*>(map)[q] = make_uint4(0, 0, 0, 0);
    __syncwarp();
#pragma unroll
    for (int k = 0; k < kEPL; ++k) {
      if (pf[k] < (uint32_t)(kMapB * 128)) {
        map[pf[k]] = (unsigned char)(lane + 32 * k + 1);
        if constexpr (KIND != 1) erow[lane + 32 * k] = slot_row(pf[k]);
      }
      if constexpr (BWD)
        if (lane + 32 * k < ne) esc[lane + 32 * k] = pp[k];
    }
    for (int j = 32 * kEPL + lane; j < ne; j += 32) {
      const uint32_t f = __ldg(a.efrag + e0 + j);
      if (f < (uint32_t)(kMapB * 128)) {
        map[f] = (unsigned char)(j + 1);
        if constexpr (KIND != 1) erow[j] = slot_row(f);
      }
      if constexpr (BWD) esc[j] = __ldg(a.pin + e0 + j);
    }
#pragma unroll
    for (int h = 0; h < 4; ++h) own[h] = ownn[h];
    if constexpr (BWD) {
#pragma unroll
      for (int h = 0; h < 4; ++h) yv[h] = yfn[h];
    }
    load_own(w + 1, ownn, yfn);
    prefetch(e1, e2);
    __syncwarp();
    // SDDMM A operand (tf32) for this window: a[h][j]: h = (row g/g+8) x (k t/t+4)
    uint32_t ao[4][4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int hs = (h & 1) | ((h >> 1) << 1);  // own[] index: bit0 row-half, bit1 k-half
      ao[h][0] = tf32_rn(own[hs].x), ao[h][1] = tf32_rn(own[hs].y);
      ao[h][2] = tf32_rn(own[hs].z), ao[h][3] = tf32_rn(own[hs].w);
    }
    // per-row state: rows g (index 0) and g+8 (index 1)
    float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f}, rs[2] = {0.f, 0.f};
    float ml2[2] = {-INFINITY, -INFINITY};
    if constexpr (BWD) {
      // rs_i = <G_i, Y_i> over the lane's 8 features, then over the quad
#pragma unroll
      for (int rh = 0; rh < 2; ++rh) {
        float d = 0.f;
#pragma unroll
        for (int kh = 0; kh < 2; ++kh) {
          const float4 gv = own[rh | (kh << 1)], fv = yv[rh | (kh << 1)];
          d += gv.x * fv.x + gv.y * fv.y + gv.z * fv.z + gv.w * fv.w;
        }
        d += __shfl_xor_sync(0xffffffffu, d, 1);
        d += __shfl_xor_sync(0xffffffffu, d, 2);
        rs[rh] = d;
      }
    }
    float acc[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
    // KB blocks per step (PAIR: the window-even-padded pair stream): one ring
    // wait, one row-max exchange and rescale check, and two independent
    // SDDMM mma chains per step
    for (int lb = 0; lb < nbw; lb += KB, s += KB) {
      cp_wait<NB - KB>();
      __syncwarp();
      // SDDMM: scores in SpMM-A layout (slot order: (g,t), (g+8,t), (g,t+4), (g+8,t+4))
      float v[KB][4];
      uint32_t mw[KB];
#pragma unroll
      for (int kb = 0; kb < KB; ++kb) {
        const uint32_t sb = ring + ((s + kb) & (NB - 1)) * 1024;
        float sc[4] = {0.f, 0.f, 0.f, 0.f};
        float b0[4], b1[4];
        lds_slice<4>(b0, sb + sd0);
        lds_slice<4>(b1, sb + sd1);
#pragma unroll
        for (int j = 0; j < 4; ++j) mma_tf32_b<ZR>(sc, ao[0][j], ao[1][j], ao[2][j], ao[3][j], b0[j], b1[j]);
        // C (g, 2t) <-> A (g, t); C (g, 2t+1) <-> A (g, t+4): A slots are
        // (0: (g,t), 1: (g+8,t), 2: (g,t+4), 3: (g+8,t+4)); C regs are
        // (0: (g,2t), 1: (g,2t+1), 2: (g+8,2t), 3: (g+8,2t+1))
        v[kb][0] = sc[0], v[kb][1] = sc[2], v[kb][2] = sc[1], v[kb][3] = sc[3];
        mw[kb] = lb + kb < kMapB ? map32[(lb + kb) * 32 + lane] : 0u;
      }
      float av[KB][4];
      if constexpr (KIND == 2) {
#pragma unroll
        for (int kb = 0; kb < KB; ++kb)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t ej = (mw[kb] >> (8 * q)) & 0xffu;
            if (ej) esc[ej - 1] = v[kb][q];
          }
        (void)av;
      } else if constexpr (KIND == 0) {
        // step row maxima (rows g, g+8) over the quad and the step's blocks
        float bm[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int kb = 0; kb < KB; ++kb) {
          bm[0] = fmaxf(bm[0], fmaxf((mw[kb] & 0xffu) ? v[kb][0] : -INFINITY,
                                     (mw[kb] & 0xff0000u) ? v[kb][2] : -INFINITY));
          bm[1] = fmaxf(bm[1], fmaxf((mw[kb] & 0xff00u) ? v[kb][1] : -INFINITY,
                                     (mw[kb] & 0xff000000u) ? v[kb][3] : -INFINITY));
        }
#pragma unroll
        for (int rh = 0; rh < 2; ++rh) {
          bm[rh] = fmaxf(bm[rh], __shfl_xor_sync(0xffffffffu, bm[rh], 1));
          bm[rh] = fmaxf(bm[rh], __shfl_xor_sync(0xffffffffu, bm[rh], 2));
        }
        // first scores of a row just set its max (acc and l are still zero);
        // after that the running max only moves when a score exceeds it by kTau
        // (lazy rescale: exp(s - m) stays <= e^kTau, and P uses the same stale
        // max, so the result is unchanged)
#pragma unroll
        for (int rh = 0; rh < 2; ++rh) {
          if (mrow[rh] == -INFINITY) {
            mrow[rh] = bm[rh];
            ml2[rh] = bm[rh] * kLog2e;
          }
        }
        if (__any_sync(0xffffffffu, bm[0] > mrow[0] + kTau || bm[1] > mrow[1] + kTau)) {
#pragma unroll
          for (int rh = 0; rh < 2; ++rh) {
            const bool up = bm[rh] > mrow[rh] + kTau;
            const float mn = up ? bm[rh] : mrow[rh];
            const float sf = up ? ex2_approx((mrow[rh] - mn) * kLog2e) : 1.f;
            mrow[rh] = mn;
            ml2[rh] = mn * kLog2e;
            lrow[rh] *= sf;
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[j][2 * rh] *= sf, acc[j][2 * rh + 1] *= sf;
          }
        }
#pragma unroll
        for (int kb = 0; kb < KB; ++kb)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t ej = (mw[kb] >> (8 * q)) & 0xffu;
            av[kb][q] = ej ? ex2_approx(fmaf(v[kb][q], kLog2e, -ml2[q & 1])) : 0.f;
            lrow[q & 1] += av[kb][q];
            if (ej) esc[ej - 1] = v[kb][q];
          }
      } else {
#pragma unroll
        for (int kb = 0; kb < KB; ++kb)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t ej = (mw[kb] >> (8 * q)) & 0xffu;
            float d = 0.f;
            if (ej) {
              const float pv = esc[ej - 1];
              d = pv * (v[kb][q] - rs[q & 1]);
              esc[ej - 1] = d;  // every edge once per window: dS replaces its P
            }
            av[kb][q] = d;
          }
      }
      // SpMM: acc += A_av * Zc
      if constexpr (KIND != 2) {
#pragma unroll
        for (int kb = 0; kb < KB; ++kb) {
          const uint32_t sb = ring + ((s + kb) & (NB - 1)) * 1024;
          float x0[4], x1[4];
          lds_slice<4>(x0, sb + so0);
          lds_slice<4>(x1, sb + so1);
          const uint32_t a0 = tf32_rn(av[kb][0]), a1 = tf32_rn(av[kb][1]), a2 = tf32_rn(av[kb][2]),
                         a3 = tf32_rn(av[kb][3]);
#pragma unroll
          for (int j = 0; j < 4; ++j) mma_tf32_b<ZR>(acc[j], a0, a1, a2, a3, x0[j], x1[j]);
        }
      }
      __syncwarp();
#pragma unroll
      for (int kb = 0; kb < KB; ++kb) {
        issue_x(s + kb + NB);
        issue_idx(s + kb + 2 * NB);
        cp_commit();
      }
    }
    // ---- window epilogue ----
    float inv[2] = {1.f, 1.f};
    if constexpr (KIND == 2) {
      // StoreSparse + the fused row epilogue, two lanes per row (rows never
      // straddle windows): raw scores, row softmax, or softmax backward
      __syncwarp();
      const int r = lane >> 1, sub = lane & 1;
      const int64_t rg = (int64_t)w * 16 + r;
      const bool live = rg < a.n;  // every lane runs the same shuffles
      const int64_t rb = live ? __ldg(a.ptr + rg) - e0 : 0;
      const int64_t re = live ? __ldg(a.ptr + rg + 1) - e0 : 0;
      // row statistics with two lanes per row, then the outputs in edge order
      // (coalesced) through the per-edge row table
      if (a.epi == TCG_EPI_NONE) {
        for (int j = lane; j < ne; j += 32) a.eout[e0 + j] = esc[j];
      } else if (a.epi == TCG_EPI_SOFTMAX) {
        float mx = -INFINITY;
        for (int64_t j = rb + sub; j < re; j += 2) mx = fmaxf(mx, esc[j]);
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        float sm = 0.f;
        for (int64_t j = rb + sub; j < re; j += 2) sm += expf(esc[j] - mx);
        sm += __shfl_xor_sync(0xffffffffu, sm, 1);
        if (sub == 0) rowm[r] = mx, rowl[r] = sm;
        __syncwarp();
        for (int j = lane; j < ne; j += 32) {
          const int q = erow[j];
          a.eout[e0 + j] = expf(esc[j] - rowm[q]) / rowl[q];
        }
      } else {
        float rsum = 0.f;
        for (int64_t j = rb + sub; j < re; j += 2) rsum += __ldg(a.pin + e0 + j) * esc[j];
        rsum += __shfl_xor_sync(0xffffffffu, rsum, 1);
        if (sub == 0) rowrs[r] = rsum;
        __syncwarp();
        for (int j = lane; j < ne; j += 32)
          a.eout[e0 + j] = __ldg(a.pin + e0 + j) * (esc[j] - rowrs[erow[j]]);
      }
    } else if constexpr (KIND == 0) {
#pragma unroll
      for (int rh = 0; rh < 2; ++rh) {
        float l = lrow[rh];
        l += __shfl_xor_sync(0xffffffffu, l, 1);
        l += __shfl_xor_sync(0xffffffffu, l, 2);
        inv[rh] = l > 0.f ? 1.f / l : 0.f;
      }
      __syncwarp();
      if (t == 0) {
        rowm[g] = mrow[0], rowm[g + 8] = mrow[1];
        rowl[g] = inv[0], rowl[g + 8] = inv[1];
      }
      __syncwarp();
      // P_e = exp(S_e - m_i) / l_i over the window's edges in order (coalesced)
      for (int j = lane; j < ne; j += 32) {
        const int r = erow[j];
        a.eout[e0 + j] = ex2_approx((esc[j] - rowm[r]) * kLog2e) * rowl[r];
      }
    } else if constexpr (KIND == 1) {
      // dS of the window's edges, in order (coalesced)
      __syncwarp();
      for (int j = lane; j < ne; j += 32) a.eout[e0 + j] = esc[j];
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if constexpr (KIND == 2) break;
      const int64_t r = (int64_t)w * 16 + g + 8 * h;
      if (r >= a.n) continue;
      float4* yr = reinterpret_cast<float4*>(a.y + (r - a.y_row0) * a.ldy + 8 * t);
      if (!MASK || 8 * t < a.dv)
        yr[0] = make_float4(acc[0][2 * h] * inv[h], acc[1][2 * h] * inv[h], acc[2][2 * h] * inv[h],
                            acc[3][2 * h] * inv[h]);
      if (!MASK || 8 * t + 4 < a.dv)
        yr[1] = make_float4(acc[0][2 * h + 1] * inv[h], acc[1][2 * h + 1] * inv[h],
                            acc[2][2 * h + 1] * inv[h], acc[3][2 * h + 1] * inv[h]);
    }
    if constexpr (NEXT) {
      // Y tile (rows g / g + 8, features 8t .. 8t + 7 per lane) into the map area as a
      // 16 x 32 tile, 16-B chunk c of row r at r * 128 + ((c ^ (r & 7)) << 4)
      const uint32_t ts = smem_u32(map);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int rr = g + 8 * h;
        const float4 v0 = make_float4(acc[0][2 * h] * inv[h], acc[1][2 * h] * inv[h], acc[2][2 * h] * inv[h],
                                      acc[3][2 * h] * inv[h]);
        const float4 v1 = make_float4(acc[0][2 * h + 1] * inv[h], acc[1][2 * h + 1] * inv[h],
                                      acc[2][2 * h + 1] * inv[h], acc[3][2 * h + 1] * inv[h]);
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(ts + rr * 128 + (((2 * t) ^ (rr & 7)) << 4)),
                     "f"(v0.x), "f"(v0.y), "f"(v0.z), "f"(v0.w) : "memory");
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(ts + rr * 128 + (((2 * t + 1) ^ (rr & 7)) << 4)),
                     "f"(v1.x), "f"(v1.y), "f"(v1.z), "f"(v1.w) : "memory");
      }
      __syncwarp();
      // Zn = Y Wn, n-tile j column n <-> output 4n + j (each lane's outputs contiguous)
      float zc[4][4];
#pragma unroll
      for (int j = 0; j < 4; ++j) zc[j][0] = zc[j][1] = zc[j][2] = zc[j][3] = 0.f;
      const int mm = lane >> 3, r8 = (lane & 7) + 8 * (mm & 1);
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) {
        uint32_t av4[4], ah[4], al[4];
        const int c = 2 * kc + (mm >> 1);
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                     : "=r"(av4[0]), "=r"(av4[1]), "=r"(av4[2]), "=r"(av4[3])
                     : "r"(ts + r8 * 128 + ((c ^ (r8 & 7)) << 4)));
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          ah[i] = tf32_rn(__uint_as_float(av4[i]));
          al[i] = tf32_rn(__uint_as_float(av4[i]) - __uint_as_float(ah[i]));
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int k0 = 8 * kc + t, col = 4 * g + j;
          const uint32_t bh0 = __float_as_uint(wnh[k0 * 32 + col]), bh1 = __float_as_uint(wnh[(k0 + 4) * 32 + col]);
          const uint32_t bl0 = __float_as_uint(wnh[1024 + k0 * 32 + col]),
                         bl1 = __float_as_uint(wnh[1024 + (k0 + 4) * 32 + col]);
          mma_tf32(zc[j], al[0], al[1], al[2], al[3], bh0, bh1);
          mma_tf32(zc[j], ah[0], ah[1], ah[2], ah[3], bl0, bl1);
          mma_tf32(zc[j], ah[0], ah[1], ah[2], ah[3], bh0, bh1);
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t r = (int64_t)w * 16 + g + 8 * h;
        if (r >= a.n) continue;
        float4* zr = reinterpret_cast<float4*>(a.zn + (r - a.y_row0) * a.ldzn + 8 * t);
        zr[0] = make_float4(zc[0][2 * h], zc[1][2 * h], zc[2][2 * h], zc[3][2 * h]);
        zr[1] = make_float4(zc[0][2 * h + 1], zc[1][2 * h + 1], zc[2][2 * h + 1], zc[3][2 * h + 1]);
      }
      __syncwarp();  // the map area is cleared by the next window's InitSparse
    }
    cb0 = cb1, cb1 = nb2, nb2 = nb3, nb3 = blk_of(w + 4);
    e0 = e1, e1 = e2, e2 = e3, e3 = ptr_of(w + 4);
  }
  cp_wait<0>();
}

template <int KIND, bool PAIR = false, bool MASK = false, bool NEXT = false, bool ZR = false>
int launch_agnn(AgnnArgs& a, cudaStream_t s) {
  using C = AgnnCfg<KIND>;
  auto kern = agnn_stream<KIND, PAIR, MASK, NEXT, ZR>;
  constexpr int SMEM = C::SMEM + (NEXT ? 2 * 1024 * 4 : 0);
  static int configured = -1;
  int dev = 0;
  TCG_CUDA(cudaGetDevice(&dev), "agnn_stream device");
  if (configured != dev) {
    TCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM),
             "agnn_stream attr");
    configured = dev;
  }
  int per_sm = 1;
  TCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::WPC * 32, SMEM),
           "agnn_stream occupancy");
  if (per_sm < 1) per_sm = 1;
  const int64_t ctas = (int64_t)num_sms() * per_sm;
  a.nwarps = (int)(ctas * C::WPC);
  ::tcg::launch_pdl(kern, (unsigned)ctas, C::WPC * 32, SMEM, s, a);
  TCG_LAUNCHED(KIND == 1 ? "agnn_stream_bwd" : KIND == 0 ? "agnn_stream_fwd" : "sddmm_stream");
  return TCG_OK;
}

// ---- SDDMM for wide windows (round 2) ------------------------------------------
//
// agnn_stream<2> keeps a u8 slot map of the window's first 24 blocks and its
// scores in a 256-entry buffer, so products-like windows (~400 edges, ~50
// blocks) fell back to the window engine (7.1 ms at products D = 16). This
// variant takes windows of up to kWideE edges: the slot map is u16 and covers a
// round of kWideRB blocks, rebuilt per round by two lanes per row walking their
// row's edges (within a row the edges are sorted by column, hence by block, so
// each edge's fragment slot is read once per window); scores, the per-edge row
// and the row epilogue (raw / softmax / softmax backward) are those of
// agnn_stream<2> with kWideE-entry buffers. One block per step.
constexpr int kWideE = 1024;
constexpr int kWideRB = 16;
// W16: 8 blocks of 512 B in flight per warp (the ring's bytes, not its depth,
// bound the gather: 4 x 512 B measured 1.50 ms at products, 8 x 512 B below)
template <bool W16 = false>
struct WideCfg {
  static constexpr int NB = W16 ? 8 : 4, NI = 2 * NB;
  static_assert(NI <= TCG_STREAM_PAD, "id ring reads past the stream padding");
  static constexpr int RING = NB * (W16 ? 512 : 1024);
  static constexpr int IDX = NI * 32;
  static constexpr int MAP = kWideRB * 128 * 2;  // u16 per fragment slot: local edge + 1
  static constexpr int ESC = kWideE * 4;
  static constexpr int ROW = 64 * 4;
  static constexpr int EROW = kWideE;
  static constexpr int WARP = RING + IDX + MAP + ESC + ROW + EROW;
  static constexpr int WPC = 8;
  static constexpr int SMEM = WPC * WARP;
};

// W16 (D <= 16): 64-B staged rows, one 16-B copy per lane per block (row L/4,
// chunk L%4; row r at (r & 3) * 128 + (r >> 2) * 64 so the SDDMM's row pairs
// r / r + 4 read different bank halves) and two mma per block instead of four:
// mma j takes features 4t + 2j (k = t) and 4t + 2j + 1 (k = t + 4).
template <bool MASK, bool W16 = false>
__global__ void __launch_bounds__(WideCfg<W16>::WPC * 32, 2) sddmm_wide(const AgnnArgs a) {
  TCG_PDL_ENTRY();
  using C = WideCfg<W16>;
  constexpr int NB = C::NB, NI = C::NI;
  constexpr uint32_t SLOT = W16 ? 512 : 1024;
  constexpr uint32_t RS = kWideRB * 128;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int gw = blockIdx.x * C::WPC + wid;
  const int g = lane >> 2, t = lane & 3;
  unsigned char* wsm = smem + wid * C::WARP;
  const uint32_t ring = smem_u32(wsm);
  const uint32_t iring = ring + C::RING;
  const unsigned char* iring_p = wsm + C::RING;
  uint16_t* map = reinterpret_cast<uint16_t*>(wsm + C::RING + C::IDX);
  float* esc = reinterpret_cast<float*>(wsm + C::RING + C::IDX + C::MAP);
  float* rowm = esc + kWideE;
  float* rowl = rowm + 16;
  float* rowrs = rowl + 16;
  unsigned char* erow = reinterpret_cast<unsigned char*>(esc + kWideE + 64);

  const int B0 = __ldg(a.boff + a.win_begin), B1 = __ldg(a.boff + a.win_end);
  const int64_t TBr = B1 - B0;
  const int lo_b = B0 + (int)(TBr * gw / a.nwarps);
  const int hi_b = B0 + (int)(TBr * (gw + 1) / a.nwarps);
  const int ws = warp_lower_bound(a.boff, a.win_begin, a.win_end, lo_b);
  const int we = gw + 1 == a.nwarps ? a.win_end : warp_lower_bound(a.boff, ws, a.win_end, hi_b);
  if (ws >= we) return;
  const int gb0 = __ldg(a.boff + ws);

  const char* xb = reinterpret_cast<const char*>(a.z + g * 4);
  const uint32_t xrow = (uint32_t)a.ldz * 4u;
  const uint32_t so0 = agnn_off(t, g), so1 = agnn_off(t + 4, g);
  const int pr = (g >> 1) + 4 * (g & 1);
  const uint32_t sd0 = agnn_off(pr, t), sd1 = agnn_off(pr, t + 4);
  const uint32_t* csw = a.cs + 8 * (int64_t)gb0;
  auto issue_idx = [&](int s) {
    if (lane < 2) cp_async<16>(iring + (s & (NI - 1)) * 32 + lane * 16, csw + 8 * (int64_t)s + 4 * lane);
  };
  const int xvb = MASK ? (4 * g < a.dv ? 16 : 0) : 16;
  // W16: lane L copies chunk L%4 of staged row L/4 (the block's column k = L/4,
  // at position 2 (k & 3) + (k >> 2) of the pair-interleaved ids)
  const int qr = lane >> 2, qc = lane & 3;
  const uint32_t q_id = 4u * (uint32_t)(2 * (qr & 3) + (qr >> 2));
  const uint32_t q_dst = (uint32_t)((qr & 3) * 128 + (qr >> 2) * 64 + qc * 16);
  const int q_vb = MASK ? (4 * qc < a.dv ? 16 : 0) : 16;
  const char* q_x = reinterpret_cast<const char*>(a.z) + 16 * qc;
  auto issue_x = [&](int s) {
    const uint32_t sb = ring + (s & (NB - 1)) * SLOT;
    if constexpr (W16) {
      const uint32_t id = *reinterpret_cast<const uint32_t*>(iring_p + (s & (NI - 1)) * 32 + q_id);
      if constexpr (MASK)
        cp_async_n<16>(sb + q_dst, q_vb ? (const void*)(q_x + (uint64_t)id * xrow) : (const void*)a.z, q_vb);
      else
        cp_async<16>(sb + q_dst, q_x + (uint64_t)id * xrow);
      return;
    }
    const uint2 id = *reinterpret_cast<const uint2*>(iring_p + (s & (NI - 1)) * 32 + 8 * t);
    if constexpr (MASK) {
      const void* z0 = a.z;
      cp_async_n<16>(sb + so0, xvb ? (const void*)(xb + (uint64_t)id.x * xrow) : z0, xvb);
      cp_async_n<16>(sb + so1, xvb ? (const void*)(xb + (uint64_t)id.y * xrow) : z0, xvb);
    } else {
      cp_async<16>(sb + so0, xb + (uint64_t)id.x * xrow);
      cp_async<16>(sb + so1, xb + (uint64_t)id.y * xrow);
    }
  };
  // W16: this lane's SDDMM B chunk (staged row pr, chunk t)
  const uint32_t sdw = (uint32_t)((pr & 3) * 128 + (pr >> 2) * 64 + t * 16);
  for (int s = 0; s < NB; ++s) issue_idx(s);
  cp_commit();
  cp_wait<0>();
  __syncwarp();
  for (int s = 0; s < NB; ++s) {
    issue_x(s);
    issue_idx(s + NB);
    cp_commit();
  }

  auto ptr_of = [&](int w) { return (int64_t)__ldg(a.ptr + min((int64_t)w * 16, a.n)); };
  auto blk_of = [&](int w) { return __ldg(a.boff + min(w, a.win_end)) - gb0; };
  int cb0 = 0, cb1 = blk_of(ws + 1);
  int64_t e0 = ptr_of(ws), e1 = ptr_of(ws + 1);
  float4 own[4];
  const uint32_t* map32 = reinterpret_cast<const uint32_t*>(map);
  int s = 0;
  for (int w = ws; w < we; ++w) {
    const int nbw = cb1 - cb0;
    const int ne = (int)(e1 - e0);
    // own rows (SDDMM A operand): rows g, g+8; features 4t.. and 4(t+4).. (W16: 4t.. only)
#pragma unroll
    for (int h = 0; h < (W16 ? 2 : 4); ++h) {
      const int64_t r = (int64_t)w * 16 + g + 8 * (h & 1);
      const int f = 4 * (t + 4 * (h >> 1));
      const bool ok = r < a.n && (!MASK || f < a.dv);
      own[h] = ok ? __ldg(reinterpret_cast<const float4*>(a.za + r * a.lda + f)) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    // two lanes per row: the row's edges [rb, re) (window-local)
    const int r = lane >> 1, sub = lane & 1;
    const int64_t rg = (int64_t)w * 16 + r;
    const bool live = rg < a.n;
    const int rb = live ? (int)(__ldg(a.ptr + rg) - e0) : 0;
    const int re = live ? (int)(__ldg(a.ptr + rg + 1) - e0) : 0;
    __syncwarp();
    for (int j = rb + sub; j < re; j += 2) erow[j] = (unsigned char)r;
    // the window's fragment slots, staged once (independent coalesced loads) in the
    // score buffer: edge j's slot is read by its round's map rebuild before the
    // round's blocks write edge j's score over it
    uint32_t* efs = reinterpret_cast<uint32_t*>(esc);
#pragma unroll 4
    for (int j = lane; j < ne; j += 32) efs[j] = __ldg(a.efrag + e0 + j);
    __syncwarp();
    int rc = rb + sub;  // this lane's cursor into its row's edges
    uint32_t ao[4][4];
    if constexpr (W16) {
      // mma j: a0 (g, k=t) = feature 4t+2j, a1 row g+8, a2 (g, k=t+4) = 4t+2j+1, a3 row g+8
      ao[0][0] = tf32_rn(own[0].x), ao[1][0] = tf32_rn(own[1].x), ao[2][0] = tf32_rn(own[0].y), ao[3][0] = tf32_rn(own[1].y);
      ao[0][1] = tf32_rn(own[0].z), ao[1][1] = tf32_rn(own[1].z), ao[2][1] = tf32_rn(own[0].w), ao[3][1] = tf32_rn(own[1].w);
    } else {
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        ao[h][0] = tf32_rn(own[h].x), ao[h][1] = tf32_rn(own[h].y);
        ao[h][2] = tf32_rn(own[h].z), ao[h][3] = tf32_rn(own[h].w);
      }
    }
    for (int lb = 0; lb < nbw; ++lb, ++s) {
      if (lb % kWideRB == 0) {  // slot map of blocks [lb, lb + kWideRB)
        __syncwarp();
#pragma unroll
        for (int q = 0; q < (int)(RS * 2 / 16 / 32); ++q)
          reinterpret_cast<uint4*>(map)[q * 32 + lane] = make_uint4(0, 0, 0, 0);
        __syncwarp();
        const uint32_t lo = (uint32_t)lb * 128;
        while (rc < re) {
          const uint32_t f = efs[rc] - lo;
          if (f >= RS) break;  // this row's next edges belong to a later round
          map[f] = (uint16_t)(rc + 1);
          rc += 2;
        }
        __syncwarp();
      }
      cp_wait<NB - 1>();
      __syncwarp();
      const uint32_t sb = ring + (s & (NB - 1)) * SLOT;
      float sc[4] = {0.f, 0.f, 0.f, 0.f};
      if constexpr (W16) {
        float b[4];
        lds_slice<4>(b, sb + sdw);
#pragma unroll
        for (int j = 0; j < 2; ++j) mma_tf32_rb(sc, ao[0][j], ao[1][j], ao[2][j], ao[3][j], b[2 * j], b[2 * j + 1]);
      } else {
        float b0[4], b1[4];
        lds_slice<4>(b0, sb + sd0);
        lds_slice<4>(b1, sb + sd1);
#pragma unroll
        for (int j = 0; j < 4; ++j) mma_tf32_rb(sc, ao[0][j], ao[1][j], ao[2][j], ao[3][j], b0[j], b1[j]);
      }
      const float v[4] = {sc[0], sc[2], sc[1], sc[3]};
      const uint2 mw = reinterpret_cast<const uint2*>(map32)[(lb % kWideRB) * 32 + lane];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t ej = ((q < 2 ? mw.x : mw.y) >> (16 * (q & 1))) & 0xffffu;
        if (ej) esc[ej - 1] = v[q];
      }
      __syncwarp();
      issue_x(s + NB);
      issue_idx(s + 2 * NB);
      cp_commit();
    }
    // StoreSparse + the row epilogue (as agnn_stream<2>)
    __syncwarp();
    if (a.epi == TCG_EPI_NONE) {
      for (int j = lane; j < ne; j += 32) a.eout[e0 + j] = esc[j];
    } else if (a.epi == TCG_EPI_SOFTMAX) {
      float mx = -INFINITY;
      for (int j = rb + sub; j < re; j += 2) mx = fmaxf(mx, esc[j]);
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      float sm = 0.f;
      for (int j = rb + sub; j < re; j += 2) sm += expf(esc[j] - mx);
      sm += __shfl_xor_sync(0xffffffffu, sm, 1);
      if (sub == 0) rowm[r] = mx, rowl[r] = sm;
      __syncwarp();
      for (int j = lane; j < ne; j += 32) {
        const int q = erow[j];
        a.eout[e0 + j] = expf(esc[j] - rowm[q]) / rowl[q];
      }
    } else {
      float rsum = 0.f;
      for (int j = rb + sub; j < re; j += 2) rsum += __ldg(a.pin + e0 + j) * esc[j];
      rsum += __shfl_xor_sync(0xffffffffu, rsum, 1);
      if (sub == 0) rowrs[r] = rsum;
      __syncwarp();
      for (int j = lane; j < ne; j += 32) a.eout[e0 + j] = __ldg(a.pin + e0 + j) * (esc[j] - rowrs[erow[j]]);
    }
    __syncwarp();
    cb0 = cb1, cb1 = blk_of(w + 2);
    e0 = e1, e1 = ptr_of(w + 2);
  }
  cp_wait<0>();
}

template <bool MASK, bool W16 = false>
int launch_wide(AgnnArgs& a, cudaStream_t s) {
  using C = WideCfg<W16>;
  auto kern = sddmm_wide<MASK, W16>;
  static int configured = -1;
  int dev = 0;
  TCG_CUDA(cudaGetDevice(&dev), "sddmm_wide device");
  if (configured != dev) {
    TCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM), "sddmm_wide attr");
    configured = dev;
  }
  int per_sm = 1;
  TCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::WPC * 32, C::SMEM),
           "sddmm_wide occupancy");
  if (per_sm < 1) per_sm = 1;
  const int64_t ctas = (int64_t)num_sms() * per_sm;
  a.nwarps = (int)(ctas * C::WPC);
  ::tcg::launch_pdl(kern, (unsigned)ctas, C::WPC * 32, C::SMEM, s, a);
  TCG_LAUNCHED("sddmm_wide");
  return TCG_OK;
}

// ---- tiling preprocessing ---------------------------------------------------

// block_offsets[w] = sum of win_partition[0..w) (single CTA; once per tiling)
__global__ void block_offsets_kernel(const uint32_t* __restrict__ wp, int64_t W, int32_t* boff,
                                     int even) {
  __shared__ int scratch[33];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < W; base += 1024) {
    const int64_t i = base + threadIdx.x;
    const int v = i < W ? (even ? (int)((wp[i] + 1) & ~1u) : (int)wp[i]) : 0;
    int total;
    const int ex = block_excl_scan<1024>(v, scratch, &total);
    if (i < W) boff[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) boff[W] = carry;
}

// col_stream[8 b + 2 i + j] = col_to_node[col_offsets[w] + 8 (b - boff[w]) + i + 4 j]
// (pair-interleaved); columns past the window's last repeat its first node;
// the kStreamPad blocks past the end repeat the stream's first block.
__global__ void col_stream_kernel(const int64_t* __restrict__ coff, const uint32_t* __restrict__ c2n,
                                  const int32_t* __restrict__ boff, int64_t W, uint32_t* cs) {
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= W) return;
  const int64_t c0 = coff[w], u = coff[w + 1] - c0;
  const int64_t b0 = boff[w], nb = boff[w + 1] - b0;
  for (int64_t q = lane; q < nb * 8; q += 32) {
    const int64_t b = q >> 3, k = q & 7;
    const int64_t c = b * 8 + (k >> 1) + 4 * (k & 1);
    cs[8 * b0 + q] = c2n[c0 + (c < u ? c : 0)];
  }
}

__global__ void stream_pad_kernel(const int32_t* __restrict__ boff, int64_t W, uint32_t* cs,
                                  const uint32_t* __restrict__ c2n) {
  const int64_t tb = boff[W];
  const uint32_t fill = tb > 0 ? cs[0] : (c2n ? c2n[0] : 0u);
  for (int q = threadIdx.x; q < 8 * TCG_STREAM_PAD; q += blockDim.x) cs[8 * tb + q] = fill;
}

template <int NT, bool DUAL, bool BIG, bool MASK, bool PAIR = false, bool X2R = false, int DMB = 8, int OCC = 1>
int launch_t(Args& a, int nchunks, cudaStream_t s) {
  using C = Cfg<NT, DUAL, BIG, PAIR, DMB, OCC>;
  auto kern = spmm_stream<NT, DUAL, BIG, MASK, PAIR, X2R, DMB, OCC>;
  static int configured = -1;
  int dev = 0;
  TCG_CUDA(cudaGetDevice(&dev), "spmm_stream device");
  if (configured != dev) {
    TCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM),
             "spmm_stream attr");
    configured = dev;
  }
  int per_sm = 1;
  TCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::WPC * 32, C::SMEM),
           "spmm_stream occupancy");
  if (per_sm < 1) per_sm = 1;
  int64_t ctas = (int64_t)num_sms() * per_sm;
  // a handful of blocks per warp at least (tiny graphs)
  const int64_t tb = 0;  // unknown on the host; the kernel tolerates idle warps
  (void)tb;
  a.nwarps = (int)(ctas * C::WPC);
  dim3 grid((unsigned)ctas, (unsigned)nchunks);
  ::tcg::launch_pdl(kern, grid, C::WPC * 32, C::SMEM, s, a);
  TCG_LAUNCHED("spmm_stream");
  return TCG_OK;
}

}  // namespace stream

// Returns TCG_E_UNSUPPORTED (nothing launched) when the operands do not fit
// the engine's vector paths; the caller then uses the window engine.
int stream_spmm(const tcg_tiling* t, const win::Params& q, cudaStream_t s) {
  if (!t->block_offsets || !t->col_stream) return TCG_E_UNSUPPORTED;
  const int dim = q.dim;
  const bool dual = q.x2 != nullptr;
  if (q.nwin <= 0) return TCG_E_UNSUPPORTED;
  auto al = [](const void* p, int b) { return (reinterpret_cast<uintptr_t>(p) % b) == 0; };
  // a chunk of 8*nt features starting at feature d needs 4*nt-byte aligned slices
  auto ok_at = [&](int nt, int d) {
    const int b = 4 * nt;
    return al(q.x + d, b) && (q.ldx * 4) % b == 0 &&
           (!dual || (al(q.x2 + d, b) && (q.ldx2 * 4) % b == 0));
  };
  stream::Args a{};
  a.ptr = t->node_ptr;
  a.efrag = t->edge_frag;
  a.boff = t->block_offsets;
  a.cs = t->col_stream;
  a.n = t->num_nodes;
  a.win_begin = (int)q.win_begin;
  a.win_end = (int)(q.win_begin + q.nwin);
  a.ldx = (int)q.ldx, a.ldx2 = (int)q.ldx2;
  a.x = q.x, a.x2 = q.x2, a.w = q.w, a.widx = q.widx, a.w2 = q.w2, a.widx2 = q.widx2;
  a.bias = q.bias, a.y = q.y, a.ldy = q.ldy, a.y_row0 = q.y_row0, a.accumulate = q.accumulate;
  a.relu = q.relu;
  // big windows (products: ~400 edges each) stage their edges in shared memory
#ifndef TCG_BIG_EPW
#define TCG_BIG_EPW 256  // measured: amazon0601 (134 edges per window) is faster without staging
#endif
  const bool big = t->num_windows > 0 && t->num_edges > TCG_BIG_EPW * t->num_windows;
  auto launch = [&](int nt, int nchunks) -> int {
    a.vec_out = (a.dv == 8 * nt) && q.vec_out &&
                ((a.d0 % 4) == 0);  // float4 / float2 row stores need aligned slices
    const bool mk = a.dv < 8 * nt;
    a.x16 = nt == 2 && al(q.x + a.d0, 16) && (q.ldx * 4) % 16 == 0 &&
            (!dual || (al(q.x2 + a.d0, 16) && (q.ldx2 * 4) % 16 == 0));
    // TMA tile::gather4 engine: opt-in (TCG_SPMM_ENGINE=tma), measured slower
    // than the cp.async ring on B200 (profiles/r02)
    static const char* eng = std::getenv("TCG_SPMM_ENGINE");
    static const bool pair_off = std::getenv("TCG_NO_PAIRS") != nullptr;  // A/B: one block per step
    const bool use_tma = eng && std::strcmp(eng, "tma") == 0;
    const bool use_ws = eng && std::strcmp(eng, "ws") == 0;
    if (use_ws && !dual && !mk && nt == 4) {
      CUtensorMap tm;
      if (stream::make_row_map(&tm, q.x, q.n, q.dim, q.ldx)) {
        static const char* wc = std::getenv("TCG_WS_CFG");
        const int cfg = wc ? std::atoi(wc) : 0;
        switch (cfg) {
          case 1: return stream::launch_ws<8, 6, 8, 2>(a, tm, nchunks, s);
          case 2: return stream::launch_ws<4, 4, 8, 4>(a, tm, nchunks, s);
          case 3: return stream::launch_ws<8, 4, 8, 3>(a, tm, nchunks, s);
          case 4: return stream::launch_ws<12, 4, 8, 2>(a, tm, nchunks, s);
          case 5: return stream::launch_ws<8, 8, 8, 2>(a, tm, nchunks, s);
          case 6: return stream::launch_ws<6, 4, 8, 3>(a, tm, nchunks, s);
          default: return stream::launch_ws<8, 4, 8, 2>(a, tm, nchunks, s);
        }
      }
    }
    if (use_tma && !dual && !big && !mk && nt == 4 && !q.relu) {
      CUtensorMap tm;
      if (stream::make_row_map(&tm, q.x, q.n, q.dim, q.ldx)) {
        return stream::launch_tma<8, 8>(a, tm, nchunks, s);
      }
    }
    // 16-wide single-operand chunks: two blocks per step over the pair stream
    // 32-wide single-operand chunks too (measured 34.8 -> 32.8 us at arxiv D=32, cold)
    if (nt == 4 && !big && !mk && t->pair_offsets && t->pair_stream && !pair_off) {
      stream::Args ap = a;
      ap.boff = t->pair_offsets;
      ap.cs = t->pair_stream;
      if (dual) {
        // 4-block fragment rounds (16 warps / SM) on short windows: arxiv (~14 blocks per
        // window) AGNN-4 epoch 0.869 -> 0.861 ms; 8-block rounds on longer ones: amazon0601
        // (~17) 2.049 vs 2.066 ms with 4
        const bool short_w = t->num_unique <= 124 * t->num_windows;  // <= 15.5 blocks per window
        if (short_w)
          return q.x2_tf32 ? stream::launch_t<4, true, false, false, true, true, 4>(ap, nchunks, s)
                           : stream::launch_t<4, true, false, false, true, false, 4>(ap, nchunks, s);
        return q.x2_tf32 ? stream::launch_t<4, true, false, false, true, true>(ap, nchunks, s)
                         : stream::launch_t<4, true, false, false, true>(ap, nchunks, s);
      }
      return stream::launch_t<4, false, false, false, true>(ap, nchunks, s);
    }
    if (nt == 2 && !dual && a.x16 && t->pair_offsets && t->pair_stream && !pair_off) {
      stream::Args ap = a;
      ap.boff = t->pair_offsets;
      ap.cs = t->pair_stream;
      // large graphs (amazon0601-sized): three CTAs per SM; arxiv-sized ones measured
      // neutral to slightly slower that way (GCN-2 epoch 0.191-0.199 vs 0.196-0.203 ms)
      const bool occ3 = t->num_nodes >= 262144;
      if (!big && occ3)
        return mk ? stream::launch_t<2, false, false, true, true, false, 8, 3>(ap, nchunks, s)
                  : stream::launch_t<2, false, false, false, true, false, 8, 3>(ap, nchunks, s);
      return big ? (mk ? stream::launch_t<2, false, true, true, true>(ap, nchunks, s)
                       : stream::launch_t<2, false, true, false, true>(ap, nchunks, s))
                 : (mk ? stream::launch_t<2, false, false, true, true>(ap, nchunks, s)
                       : stream::launch_t<2, false, false, false, true>(ap, nchunks, s));
    }
#define TCG_SL(NTV, MK)                                                                   \
  if (nt == NTV && mk == MK)                                                              \
    return big ? (dual ? stream::launch_t<NTV, true, true, MK>(a, nchunks, s)             \
                       : stream::launch_t<NTV, false, true, MK>(a, nchunks, s))           \
               : (dual ? stream::launch_t<NTV, true, false, MK>(a, nchunks, s)            \
                       : stream::launch_t<NTV, false, false, MK>(a, nchunks, s));
    TCG_SL(4, false)
    TCG_SL(4, true)
    TCG_SL(2, false)
    TCG_SL(2, true)
    TCG_SL(1, false)
    TCG_SL(1, true)
#undef TCG_SL
    return TCG_E_UNSUPPORTED;
  };
  // plan: 32-wide chunks (one launch), then 16, then 8-wide, then one masked tail.
  // Rows whose stride breaks 16-B alignment would need one 8-wide pass per 8
  // features: past two such passes the single-pass window engine is faster.
  if (!ok_at(2, 0) && dim > 16) return TCG_E_UNSUPPORTED;
  int d = 0;
  const int full = dim / 32;
  if (full > 0 && ok_at(4, 0)) {
    a.d0 = 0, a.dv = 32;
    const int rc = launch(4, full);
    if (rc != TCG_OK) return rc;
    d = 32 * full;
  }
  while (d < dim) {
    const int rem = dim - d;
    // every pass costs about the same (it walks the whole block stream), so a
    // tail is one masked pass of the narrowest chunk that holds it (17..31
    // features: 32-wide, 9..15: 16-wide) rather than several narrow ones
    const int nt = (rem > 16 && ok_at(4, d)) ? 4 : (rem > 8 && ok_at(2, d)) ? 2 : 1;
    if (nt == 1 && !ok_at(1, d)) return d == 0 ? TCG_E_UNSUPPORTED : TCG_E_INVALID;
    a.d0 = d;
    a.dv = rem < 8 * nt ? rem : 8 * nt;
    const int rc = launch(nt, 1);
    if (rc != TCG_OK) return rc;
    d += a.dv;
  }
  return TCG_OK;
}

// Fused AGNN forward / backward on the block stream; TCG_E_UNSUPPORTED when
// the shape does not fit (D != 32, misaligned, windows wider than the slot map).
int stream_agnn(const tcg_tiling* t, bool bwd, int dim, const float* z, int64_t ldz, const float* za,
                int64_t lda, const float* yf, int64_t ldyf, const float* pin, float* eout,
                float* y, int64_t ldy, int64_t y_row0, int64_t win_begin, int64_t win_end,
                cudaStream_t s, const float* wn, float* zn, int64_t ldzn, bool z_tf32) {
  if (dim < 4 || dim > 32 || dim % 4) return TCG_E_UNSUPPORTED;
  if (!t->block_offsets || !t->col_stream || !t->edge_frag) return TCG_E_UNSUPPORTED;
  if (t->max_window_edges <= 0 || t->max_window_edges > stream::kMaxE ||
      t->max_window_unique > 8 * stream::kMapB)
    return TCG_E_UNSUPPORTED;
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!al(z) || !al(za) || !al(y) || ldz % 4 || lda % 4 || ldy % 4) return TCG_E_UNSUPPORTED;
  if (bwd && (!yf || !al(yf) || ldyf % 4 || !pin)) return TCG_E_UNSUPPORTED;
  stream::AgnnArgs a{};
  a.ptr = t->node_ptr, a.efrag = t->edge_frag, a.boff = t->block_offsets, a.cs = t->col_stream;
  a.n = t->num_nodes;
  a.win_begin = (int)win_begin, a.win_end = (int)win_end;
  a.z = z, a.ldz = ldz, a.za = za, a.lda = lda, a.yf = yf, a.ldyf = ldyf, a.pin = pin;
  a.eout = eout, a.y = y, a.ldy = ldy, a.y_row0 = y_row0;
  a.dv = dim;
  const bool mk = dim < 32;
  static const bool pair_off = std::getenv("TCG_NO_PAIRS") != nullptr;
  if (wn) {  // forward with the next layer's dense step in the epilogue (D = 32)
    if (bwd || mk || !zn || !al(zn) || ldzn % 4 || !t->pair_offsets || !t->pair_stream || pair_off)
      return TCG_E_UNSUPPORTED;
    a.wn = wn, a.zn = zn, a.ldzn = ldzn;
    a.boff = t->pair_offsets, a.cs = t->pair_stream;
    return stream::launch_agnn<0, true, false, true>(a, s);
  }
  // forward: two blocks per step (arxiv 59.4 -> 55.3 us cold); the backward
  // measured slower that way (55.3 -> 57.3 us with the coalesced dS writes,
  // 59.5 -> 63.5 us before) and keeps one block per step
  if (!bwd && t->pair_offsets && t->pair_stream && !pair_off) {
    a.boff = t->pair_offsets, a.cs = t->pair_stream;
    if (z_tf32 && !mk) return stream::launch_agnn<0, true, false, false, true>(a, s);
    return mk ? stream::launch_agnn<0, true, true>(a, s) : stream::launch_agnn<0, true>(a, s);
  }
  if (bwd && z_tf32 && !mk) return stream::launch_agnn<1, false, false, false, true>(a, s);
  if (bwd) return mk ? stream::launch_agnn<1, false, true>(a, s) : stream::launch_agnn<1>(a, s);
  return mk ? stream::launch_agnn<0, false, true>(a, s) : stream::launch_agnn<0>(a, s);
}

// true when the tiling's windows are past the fused stream kernels' slot map but
// within sddmm_wide's
bool stream_sddmm_wide(const tcg_tiling* t) {
  return t->block_offsets && t->col_stream && t->edge_frag && t->max_window_edges > 0 &&
         (t->max_window_edges > stream::kMaxE || t->max_window_unique > 8 * stream::kMapB) &&
         t->max_window_edges <= stream::kWideE;
}

// SDDMM (+ softmax / softmax-backward row epilogue) on the block stream, D <= 32
// (a multiple of 4; D < 32 runs masked)
int stream_sddmm(const tcg_tiling* t, int dim, const float* xa, int64_t lda, const float* xb, int64_t ldb,
                 const float* aux, float* out, int epi, int64_t win_begin, int64_t win_end,
                 cudaStream_t s) {
  if (dim < 4 || dim > 32 || dim % 4) return TCG_E_UNSUPPORTED;
  if (!t->block_offsets || !t->col_stream || !t->edge_frag) return TCG_E_UNSUPPORTED;
  // windows past the u8 slot map (products-like degree) take the wide variant
  const bool wide = t->max_window_edges > stream::kMaxE || t->max_window_unique > 8 * stream::kMapB;
  if (t->max_window_edges <= 0 || t->max_window_edges > (wide ? stream::kWideE : stream::kMaxE))
    return TCG_E_UNSUPPORTED;
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!al(xa) || !al(xb) || lda % 4 || ldb % 4) return TCG_E_UNSUPPORTED;
  if (epi == TCG_EPI_SOFTMAX_BWD && !aux) return TCG_E_UNSUPPORTED;
  stream::AgnnArgs a{};
  a.ptr = t->node_ptr, a.efrag = t->edge_frag, a.boff = t->block_offsets, a.cs = t->col_stream;
  a.n = t->num_nodes;
  a.win_begin = (int)win_begin, a.win_end = (int)win_end;
  a.z = xb, a.ldz = ldb, a.za = xa, a.lda = lda, a.pin = aux, a.eout = out, a.epi = epi;
  a.dv = dim;
  const bool mk = dim < 32;
  static const bool pair_off = std::getenv("TCG_NO_PAIRS") != nullptr;
  static const bool wide_all = std::getenv("TCG_SDDMM_WIDE") != nullptr;  // test hook: every window
  static const bool w16_off = std::getenv("TCG_SDDMM_W16_OFF") != nullptr;  // A/B: D <= 16 in the 32-wide layout
  if (wide || wide_all) {
    if (dim <= 16 && !w16_off) return dim < 16 ? stream::launch_wide<true, true>(a, s) : stream::launch_wide<false, true>(a, s);
    return mk ? stream::launch_wide<true>(a, s) : stream::launch_wide<false>(a, s);
  }
  if (t->pair_offsets && t->pair_stream && !pair_off) {
    a.boff = t->pair_offsets, a.cs = t->pair_stream;
    return mk ? stream::launch_agnn<2, true, true>(a, s) : stream::launch_agnn<2, true>(a, s);
  }
  return mk ? stream::launch_agnn<2, false, true>(a, s) : stream::launch_agnn<2>(a, s);
}

}  // namespace tcg

using namespace tcg;

namespace tcg {
namespace {
__global__ void invert_perm_kernel(const uint32_t* __restrict__ perm, int64_t m, uint32_t* inv) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < m) inv[perm[k]] = (uint32_t)k;
}
}  // namespace
}  // namespace tcg

extern "C" int tcg_invert_perm(const uint32_t* perm, int64_t n, uint32_t* inv, void* stream) {
  TCG_REQUIRE(n >= 0, "tcg_invert_perm: negative size");
  if (n == 0) return TCG_OK;
  TCG_REQUIRE(perm && inv, "tcg_invert_perm: null pointer");
  tcg::invert_perm_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(perm, n, inv);
  TCG_LAUNCHED("invert_perm");
  return TCG_OK;
}

static int block_stream(const tcg_tiling* t, int32_t* block_offsets, uint32_t* col_stream, int even,
                        void* stream) {
  TCG_REQUIRE(t != nullptr, "tcg_block_stream: null tiling");
  TCG_REQUIRE(t->blk_h == 16 && t->blk_w == 8,
              "tf32 mode requires the 16x8 tile shape, got %dx%d", t->blk_h, t->blk_w);
  TCG_REQUIRE(block_offsets != nullptr, "tcg_block_stream: null block_offsets");
  TCG_REQUIRE(t->num_windows < (1LL << 31) && t->num_unique < (1LL << 34),
              "tcg_block_stream: graph too large for 32-bit block offsets");
  cudaStream_t s = as_stream(stream);
  const int64_t W = t->num_windows;
  if (W == 0) {
    TCG_CUDA(cudaMemsetAsync(block_offsets, 0, sizeof(int32_t), s), "tcg_block_stream memset");
    return TCG_OK;
  }
  TCG_REQUIRE(t->win_partition && t->col_offsets, "tcg_block_stream: tiling arrays missing");
  stream::block_offsets_kernel<<<1, 1024, 0, s>>>(t->win_partition, W, block_offsets, even);
  TCG_LAUNCHED("block_offsets");
  if (col_stream == nullptr) return TCG_OK;  // offsets only (caller sizes the stream)
  if (t->num_unique > 0) {
    TCG_REQUIRE(t->col_to_node != nullptr, "tcg_block_stream: null col_to_node");
    stream::col_stream_kernel<<<(unsigned)((W + 7) / 8), 256, 0, s>>>(
        t->col_offsets, t->col_to_node, block_offsets, W, col_stream);
    TCG_LAUNCHED("col_stream");
  }
  stream::stream_pad_kernel<<<1, 256, 0, s>>>(block_offsets, W, col_stream, t->col_to_node);
  TCG_LAUNCHED("stream_pad");
  return TCG_OK;
}

extern "C" int tcg_block_stream(const tcg_tiling* t, int32_t* block_offsets, uint32_t* col_stream,
                                void* stream) {
  return block_stream(t, block_offsets, col_stream, 0, stream);
}

extern "C" int tcg_block_stream_pairs(const tcg_tiling* t, int32_t* pair_offsets, uint32_t* pair_stream,
                                      void* stream) {
  return block_stream(t, pair_offsets, pair_stream, 1, stream);
}
