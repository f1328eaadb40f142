// fp32-accurate tall-skinny GEMM on the 5th-generation tensor cores:
//   Y[n x co] = act(X[n x ci] . W[ci x co] + b),  ci <= 128, co in {16, 32}
// (the models' input layer: arxiv 128 -> 32 / 16, amazon0601 96, products 100;
// kernels.gcn_layer's update GEMM, kernels.py:577-582).
//
// In fp32 FMA this GEMM is issue-bound (0.69 GFMA for the arxiv 128 -> 32
// layer against 108 MB of HBM traffic; the FFMA2 kernel ran at 0.33 of HBM).
// Here it is one tcgen05.mma stream per 128-row tile (warp-specialised, below).
// Accuracy: rel-L2 ~1e-6 against float64 (3xTF32; the FFMA kernel ~2.5e-7).
// Measured: 44.0 vs 53.2 us at 128 -> 32; the TMA stream alone (no MMA) runs
// 29.7 us, so the X stream, not the tensor core, is what bounds it.
//   * TMA (cp.async.bulk.tensor, 128-B swizzle) brings 128 rows x 32 features
//     of X per pipeline stage into shared memory -- exactly the canonical
//     K-major SWIZZLE_128B operand layout (8-row atoms, SBO 1024 B);
//   * 3xTF32 keeps fp32 accuracy: the MMA reads fp32 bits as TF32 (the low 13
//     mantissa bits ignored), so X and W serve as their own "hi" parts and the
//     CTA writes the residuals lo = v - tf32(v) next to them; per 8-wide k step
//     D += Xhi.Whi + Xhi.Wlo + Xlo.Whi (the lo.lo term is below 2^-22);
//   * the accumulator lives in TMEM (M = 128 lanes x co columns), issued by one
//     thread, tracked by tcgen05.commit -> mbarrier; the epilogue reads it with
//     tcgen05.ld (one row per thread), adds the bias / ReLU and stores the row.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"

namespace tcg {
namespace tc {

constexpr int BM = 128;   // rows per tile (MMA M, one TMEM lane each)
constexpr int KC = 32;    // features per chunk: one 128-B swizzle row of fp32
constexpr int S = 6;      // X stages in flight (TMA)
constexpr int L = 4;      // residual (lo) buffers
constexpr int MAXKC = 4;  // ci <= 128
constexpr int NW = 10;    // warps: 0 TMA, 1 MMA, 2-5 residuals, 6-9 epilogue

template <int NO>
struct Cfg {
  static constexpr int ATILE = BM * KC * 4;   // 16 KB of X per stage
  static constexpr int BCH = NO * KC * 4;     // W^T bytes per chunk
  static constexpr int OFF_LO = S * ATILE;
  static constexpr int OFF_BHI = OFF_LO + L * ATILE;
  static constexpr int OFF_BLO = OFF_BHI + MAXKC * BCH;
  static constexpr int OFF_BAR = OFF_BLO + MAXKC * BCH;
  static constexpr int NBAR = 2 * S + 2 * L + 4;
  static constexpr int SMEM = OFF_BAR + 8 * NBAR + 16 + 1024;  // barriers, TMEM slot, 1 KB align slack
  static constexpr int TCOLS = 2 * (NO < 32 ? 32 : NO);  // two accumulators (>= 32 columns each)
  // instruction descriptor: D f32, A/B tf32, both K-major, N = NO, M = 128
  static constexpr uint32_t IDESC =
      (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NO >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
};

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major SWIZZLE_128B operand: 8-row x 128-B atoms, atoms 1024 B apart (SBO)
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void mbar_init(uint32_t b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred p;\nTCG_TCW:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra TCG_TCW;\n}\n" ::"r"(b),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
}
__device__ __forceinline__ void tma_load(uint32_t dst, const CUtensorMap* tm, int x, int y, uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(BM * KC * 4)
               : "memory");
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, int acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

// Warp-specialised, persistent: warp 0 streams X chunks with TMA into an
// S-deep ring; warps 2-5 write each chunk's residuals into one of L buffers;
// warp 1 (one lane) issues the 3xTF32 MMAs of a chunk once both are ready and
// commits them to the barriers that free the stage and the residual buffer;
// warps 6-9 drain a finished tile's accumulator (two TMEM accumulators, so the
// next tile's MMAs overlap the epilogue).
template <int NO>
__global__ void __launch_bounds__(NW * 32, 1) dense_tc(const __grid_constant__ CUtensorMap tmx, int64_t n, int ci,
                                                      const float* __restrict__ w, int co,
                                                      const float* __restrict__ bias, int relu,
                                                      float* __restrict__ y, int64_t ldy, int vec_out) {
  using C = Cfg<NO>;
  extern __shared__ unsigned char sraw[];
  const uint32_t s0 = su(sraw);
  const uint32_t sb = (s0 + 1023u) & ~1023u;
  unsigned char* sg = sraw + (sb - s0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nkc = (ci + KC - 1) / KC;
  const uint32_t bfull = sb + C::OFF_BAR, bempty = bfull + 8 * S, blofull = bempty + 8 * S,
                 bloempty = blofull + 8 * L, baccfull = bloempty + 8 * L, baccempty = baccfull + 16,
                 tslot = baccempty + 16;
  uint32_t* tslot_p = reinterpret_cast<uint32_t*>(sg + (tslot - sb));

  // W^T (hi = W itself, lo = W - tf32(W)) as the K-major B operand, zero-padded
  for (int i = tid; i < nkc * NO * KC; i += NW * 32) {
    const int kc = i / (NO * KC), rem = i % (NO * KC), nn = rem / KC, kk = rem % KC;
    const int k = kc * KC + kk;
    const float v = (k < ci && nn < co) ? __ldg(w + (int64_t)k * co + nn) : 0.f;
    const float hi = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
    const uint32_t off = kc * C::BCH + nn * 128 + ((((kk >> 2) ^ (nn & 7)) & 7) << 4) + (kk & 3) * 4;
    *reinterpret_cast<float*>(sg + C::OFF_BHI + off) = v;
    *reinterpret_cast<float*>(sg + C::OFF_BLO + off) = v - hi;
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tslot),
                 "r"(C::TCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    for (int i = 0; i < S; ++i) mbar_init(bfull + 8 * i, 1), mbar_init(bempty + 8 * i, 1);
    for (int i = 0; i < L; ++i) mbar_init(blofull + 8 * i, 4), mbar_init(bloempty + 8 * i, 1);
    for (int i = 0; i < 2; ++i) mbar_init(baccfull + 8 * i, 1), mbar_init(baccempty + 8 * i, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // B operand -> async proxy
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot_p;

  const int64_t ntiles = (n + BM - 1) / BM;
  const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t nchunks = my_tiles * nkc;

  if (warp == 0) {  // ---- TMA producer ----
    if (lane == 0) {
      for (int64_t q = 0; q < nchunks; ++q) {
        const int st = (int)(q % S);
        if (q >= S) mbar_wait(bempty + 8 * st, (uint32_t)((q / S) - 1) & 1u);
        const int64_t tile = blockIdx.x + (q / nkc) * gridDim.x;
        tma_load(sb + st * C::ATILE, &tmx, (int)(q % nkc) * KC, (int)(tile * BM), bfull + 8 * st);
      }
    }
  } else if (warp == 1) {  // ---- MMA issuer ----
    if (lane == 0) {
      for (int64_t q = 0; q < nchunks; ++q) {
        const int st = (int)(q % S), lb = (int)(q % L);
        const int kc = (int)(q % nkc);
        const int64_t t = q / nkc;
        const int ab = (int)(t & 1);
        if (kc == 0 && t >= 2) mbar_wait(baccempty + 8 * ab, (uint32_t)((t - 2) >> 1) & 1u);
        mbar_wait(bfull + 8 * st, (uint32_t)(q / S) & 1u);
        mbar_wait(blofull + 8 * lb, (uint32_t)(q / L) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + (uint32_t)(ab * (C::TCOLS / 2));
        const uint32_t a_hi = sb + st * C::ATILE, a_lo = sb + C::OFF_LO + lb * C::ATILE;
        const uint32_t b_hi = sb + C::OFF_BHI + kc * C::BCH, b_lo = sb + C::OFF_BLO + kc * C::BCH;
#pragma unroll
        for (int ks = 0; ks < KC / 8; ++ks) {  // 8 tf32 = 32 B per k step, inside the swizzle row
          const uint64_t ah = sw128_desc(a_hi + 32 * ks), al = sw128_desc(a_lo + 32 * ks);
          const uint64_t bh = sw128_desc(b_hi + 32 * ks), bl = sw128_desc(b_lo + 32 * ks);
          mma_tf32(d, ah, bh, C::IDESC, (kc | ks) != 0);
          mma_tf32(d, ah, bl, C::IDESC, 1);
          mma_tf32(d, al, bh, C::IDESC, 1);
        }
        mma_commit(bempty + 8 * st);
        mma_commit(bloempty + 8 * lb);
        if (kc == nkc - 1) mma_commit(baccfull + 8 * ab);
      }
    }
  } else if (warp < 6) {  // ---- residuals lo = x - tf32(x) ----
    const int ct = tid - 64;  // 0..127
    for (int64_t q = 0; q < nchunks; ++q) {
      const int st = (int)(q % S), lb = (int)(q % L);
      mbar_wait(bfull + 8 * st, (uint32_t)(q / S) & 1u);
      if (q >= L) mbar_wait(bloempty + 8 * lb, (uint32_t)((q / L) - 1) & 1u);
      const float4* src = reinterpret_cast<const float4*>(sg + st * C::ATILE);
      float4* dst = reinterpret_cast<float4*>(sg + C::OFF_LO + lb * C::ATILE);
#pragma unroll
      for (int i = 0; i < C::ATILE / 16 / 128; ++i) {
        const float4 v = src[i * 128 + ct];
        float4 l;
        l.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
        l.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
        l.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
        l.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
        dst[i * 128 + ct] = l;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(blofull + 8 * lb);
    }
  } else {  // ---- epilogue: TMEM lanes 32 (warp % 4) .. +31 = rows of the tile ----
    const int quarter = warp & 3;
    for (int64_t t = 0; t < my_tiles; ++t) {
      const int ab = (int)(t & 1);
      mbar_wait(baccfull + 8 * ab, (uint32_t)(t >> 1) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t r[NO];
      const uint32_t taddr = tmem + ((uint32_t)(32 * quarter) << 16) + (uint32_t)(ab * (C::TCOLS / 2));
      if constexpr (NO == 32) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
              "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
              "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
              "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(taddr)
            : "memory");
      } else {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15},"
            " [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
              "=r"(r[15])
            : "r"(taddr)
            : "memory");
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(baccempty + 8 * ab);  // accumulator free for tile t + 2
      const int64_t tile = blockIdx.x + t * gridDim.x;
      const int64_t row = tile * BM + quarter * 32 + lane;
      if (row < n) {
        float o[NO];
#pragma unroll
        for (int c = 0; c < NO; ++c) {
          float v = __uint_as_float(r[c]);
          if (bias && c < co) v += __ldg(bias + c);
          o[c] = relu ? fmaxf(v, 0.f) : v;
        }
        float* yr = y + row * ldy;
        if (vec_out && co == NO) {
#pragma unroll
          for (int c = 0; c < NO; c += 4)
            *reinterpret_cast<float4*>(yr + c) = make_float4(o[c], o[c + 1], o[c + 2], o[c + 3]);
        } else {
#pragma unroll
          for (int c = 0; c < NO; ++c)
            if (c < co) yr[c] = o[c];
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TCOLS)
                 : "memory");
  }
}

bool row_map(CUtensorMap* tm, const float* x, int64_t n, int64_t ci, int64_t ldx) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  }();
  if (!enc || n < 1 || n >= (1LL << 31)) return false;
  cuuint64_t gd[2] = {(cuuint64_t)ci, (cuuint64_t)n};
  cuuint64_t gs[1] = {(cuuint64_t)ldx * 4};
  cuuint32_t box[2] = {KC, BM}, es[2] = {1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(x), gd, gs, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int NO>
int launch(const CUtensorMap& tm, int64_t n, int ci, const float* w, int co, const float* bias, int relu,
           float* y, int64_t ldy, int vec_out, cudaStream_t s) {
  using C = Cfg<NO>;
  static int configured = -1;
  int dev = 0;
  TCG_CUDA(cudaGetDevice(&dev), "dense_tc device");
  if (configured != dev) {
    TCG_CUDA(cudaFuncSetAttribute(dense_tc<NO>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM),
             "dense_tc attr");
    configured = dev;
  }
  const int64_t tiles = (n + BM - 1) / BM;
  const int64_t grid = std::min<int64_t>(tiles, (int64_t)num_sms());  // persistent, one CTA per SM
  dense_tc<NO><<<(unsigned)grid, NW * 32, C::SMEM, s>>>(tm, n, ci, w, co, bias, relu, y, ldy, vec_out);
  TCG_LAUNCHED("dense_tc");
  return TCG_OK;
}

}  // namespace tc

// 1 = not covered (caller falls back to the FFMA kernels)
int dense_tcgen05(const float* x, int64_t ldx, int64_t n, int ci, const float* m, int co, bool trans,
                  const float* bias, int relu, const float* mask, float* y, int64_t ldy, cudaStream_t s) {
  static const bool off = std::getenv("TCG_DENSE_TC") && std::atoi(std::getenv("TCG_DENSE_TC")) == 0;
  // measured (profiles/r02/dense_tc.txt): faster than the FFMA2 tile kernel for
  // 96..128 -> 32 (arxiv 128 -> 32: 53.2 -> 44.0 us cold), slower at 16 outputs
  if (off || trans || mask || ci < 96 || ci > tc::MAXKC * tc::KC || co != 32 || n < 4096) return 1;
  if ((reinterpret_cast<uintptr_t>(x) & 15) || (ldx * 4) % 16) return 1;
  CUtensorMap tm;
  if (!tc::row_map(&tm, x, n, ci, ldx)) return 1;
  const int vec_out = (reinterpret_cast<uintptr_t>(y) % 16 == 0) && ldy % 4 == 0;
  return co == 32 ? tc::launch<32>(tm, n, ci, m, co, bias, relu, y, ldy, vec_out, s)
                  : tc::launch<16>(tm, n, ci, m, co, bias, relu, y, ldy, vec_out, s);
}

}  // namespace tcg
