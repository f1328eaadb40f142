// Shared helpers for the TC-GNN sm_100a kernels: error plumbing for the C ABI,
// launch accounting, TF32 rounding and small warp/block primitives.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>

#include "../../include/tcg.h"

namespace tcg {

// ---- ABI error plumbing ---------------------------------------------------
void set_error(const char* fmt, ...);
std::atomic<int64_t>& launch_counter();

#define TCG_REQUIRE(cond, ...)                 \
  do {                                         \
    if (!(cond)) {                             \
      ::tcg::set_error(__VA_ARGS__);           \
      return TCG_E_INVALID;                    \
    }                                          \
  } while (0)

// Call right after a kernel launch: counts it and converts a launch error
// into an ABI error code.
#define TCG_LAUNCHED(name)                                                   \
  do {                                                                       \
    ::tcg::launch_counter().fetch_add(1, std::memory_order_relaxed);         \
    cudaError_t _e = cudaGetLastError();                                     \
    if (_e != cudaSuccess) {                                                 \
      ::tcg::set_error("%s: launch failed: %s", name, cudaGetErrorString(_e)); \
      return TCG_E_CUDA;                                                     \
    }                                                                        \
  } while (0)

#define TCG_CUDA(call, name)                                                 \
  do {                                                                       \
    cudaError_t _e = (call);                                                 \
    if (_e != cudaSuccess) {                                                 \
      ::tcg::set_error("%s: %s", name, cudaGetErrorString(_e));              \
      return TCG_E_CUDA;                                                     \
    }                                                                        \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- programmatic dependent launch (PDL) -----------------------------------
// The epoch's kernels are launched with programmatic stream serialisation: a
// kernel's CTAs may be scheduled while its predecessor drains, and block in
// griddepcontrol.wait (TCG_PDL_ENTRY, the first statement of every such kernel)
// until the predecessor has completed and its writes are visible. Nothing is
// read or written before the wait, so the semantics are those of plain stream
// order; what overlaps is the launch and CTA rasterisation with the
// predecessor's tail. TCG_PDL=0 turns it off (A/B).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#ifndef TCG_PDL_TRIGGER
#define TCG_PDL_TRIGGER 0
#endif
#define TCG_PDL_ENTRY()                   \
  do {                                    \
    ::tcg::pdl_wait();                    \
    if (TCG_PDL_TRIGGER) ::tcg::pdl_trigger(); \
  } while (0)
bool pdl_enabled();
template <typename... P, typename... A>
inline void launch_pdl(void (*k)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, A&&... args) {
  if (!pdl_enabled()) {
    k<<<grid, block, smem, s>>>(static_cast<P>(args)...);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, static_cast<P>(args)...);
}

int num_sms();

// ---- numerics ---------------------------------------------------------------
// Round-to-nearest-even onto the 10-bit tf32 mantissa: the same rule as the
// reference quantize_tf32 (tiles.py:67-82). Lowers to F2FP.TF32.F32.PACK_B.
__device__ __forceinline__ uint32_t tf32_rn(float x) {
  uint32_t r;
  asm("cvt.rn.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// m16n8k8 TF32 MMA, fp32 accumulate (D = A*B + C), operands pre-rounded.
__device__ __forceinline__ void mma_tf32(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Same mma with the B operands rounded in the same asm block (cvt.rn.tf32 of
// two fp32 values straight into the HMMA register pair: no operand moves).
__device__ __forceinline__ void mma_tf32_rb(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                            uint32_t a3, float b0, float b1) {
  asm volatile(
      "{\n.reg .b32 tb0, tb1;\n"
      "cvt.rn.tf32.f32 tb0, %8;\n"
      "cvt.rn.tf32.f32 tb1, %9;\n"
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {tb0,tb1}, {%0,%1,%2,%3};\n}\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "f"(b0), "f"(b1));
}

// B operands already on the tf32 grid (RN-rounded by their producer): the mma
// reads the raw bits, which equals mma_tf32_rb on the same values
template <bool PRE>
__device__ __forceinline__ void mma_tf32_b(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                           float b0, float b1) {
  if constexpr (PRE) mma_tf32(d, a0, a1, a2, a3, __float_as_uint(b0), __float_as_uint(b1));
  else mma_tf32_rb(d, a0, a1, a2, a3, b0, b1);
}

template <typename T>
__device__ __forceinline__ T ldg_stream(const T* p) {
  return __ldg(p);
}

// ---- warp / block scans -------------------------------------------------------
__device__ __forceinline__ int warp_incl_scan(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide exclusive scan of one int per thread; returns the exclusive
// prefix and writes the block total. `scratch` holds >= 33 ints.
template <int THREADS>
__device__ __forceinline__ int block_excl_scan(int v, int* scratch, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = THREADS / 32;
  int incl = warp_incl_scan(v);
  if (lane == 31) scratch[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int s = lane < NW ? scratch[lane] : 0;
    int si = warp_incl_scan(s);
    if (lane < NW) scratch[lane] = si - s;
    if (lane == NW - 1) scratch[32] = si;
  }
  __syncthreads();
  int r = scratch[warp] + incl - v;
  *total = scratch[32];
  __syncthreads();
  return r;
}

}  // namespace tcg
