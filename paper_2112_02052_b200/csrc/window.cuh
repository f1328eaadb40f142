// Row-window engine interface (see window.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/tcg.h"

namespace tcg {
namespace win {

enum Mode { MODE_SPMM = 0, MODE_SPMM_DUAL = 1, MODE_SDDMM = 2, MODE_AGNN_FWD = 3, MODE_AGNN_BWD = 4 };

// edges per window the fused AGNN kernels keep in shared memory
constexpr int kEdgesPerWindow = 256;

// condensed columns staged per round (rows of X in shared memory)
// (the fused AGNN kernels need a whole window resident: 192 columns covers
//  the BASELINE shapes' largest windows — arxiv 153, amazon0601 ~190)
__host__ __device__ constexpr int cols_per_round(int nt, int mode) {
  return (mode == MODE_AGNN_FWD || mode == MODE_AGNN_BWD) ? (nt <= 4 ? 192 : 96)
         : (nt <= 4 ? 128 : 64) / (mode == MODE_SPMM_DUAL ? 2 : 1);
}

struct Params {
  // tiling (16x8)
  const int64_t* ptr;
  const uint32_t* e2c;
  const uint32_t* efrag;  // per-edge mma fragment slot: (c>>3)*128 + lane*4 + slot
  const int64_t* coff;
  const uint32_t* c2n;
  int64_t n;
  int64_t win_begin, nwin;
  int nchunks;  // feature chunks of 8*NT (SpMM modes); 1 otherwise
  int nkc;      // SDDMM k-chunks of 8*NT features
  int koff;     // SDDMM: first feature of this launch's k-chunk
  int dim;
  int vec16;    // 16-B staging legal (dim, ld, base aligned)
  int vec_out;  // 16-B output stores legal
  int use_tma;  // stage rows with TMA gather4 (tensor maps valid)
  // gathered operand(s)
  const float* x;
  int64_t ldx;
  const float* x2;
  int64_t ldx2;
  // SpMM weights (nullable; *_idx: indirection, A^T edge order)
  const float* w;
  const uint32_t* widx;
  const float* w2;
  const uint32_t* widx2;
  // SpMM output
  const float* bias;
  float* y;
  int64_t ldy;
  int64_t y_row0;
  int accumulate;
  int relu;  // ReLU on the stored output (stream engine epilogue only)
  int x2_tf32;  // dual form: x2 already on the tf32 grid (stream engine: no B-operand cvt)
  // SDDMM A operand (window rows) and edge outputs
  const float* xa;
  int64_t lda;
  const float* aux;
  float* eout;
  int epilogue;
};

int launch(int mode, int nt, Params& p, cudaStream_t s);

// per-edge fragment slots of a 16x8 tiling (InitSparse addresses)
int edge_frag(const int64_t* ptr, const uint32_t* e2c, int64_t n, uint32_t* efrag,
              cudaStream_t s);

inline int nt_for(int64_t dim) {
  if (dim <= 8) return 1;
  if (dim <= 16) return 2;
  if (dim <= 32) return 4;
  return 8;
}

}  // namespace win

// Block-stream engine (stream.cu); TCG_E_UNSUPPORTED => nothing launched.
int stream_sddmm(const tcg_tiling* t, int dim, const float* xa, int64_t lda, const float* xb, int64_t ldb,
                 const float* aux, float* out, int epi, int64_t win_begin, int64_t win_end,
                 cudaStream_t s);
int stream_spmm(const tcg_tiling* t, const win::Params& q, cudaStream_t s);
bool stream_sddmm_wide(const tcg_tiling* t);
int stream_agnn(const tcg_tiling* t, bool bwd, int dim, const float* z, int64_t ldz, const float* za,
                int64_t lda, const float* yf, int64_t ldyf, const float* pin, float* eout,
                float* y, int64_t ldy, int64_t y_row0, int64_t win_begin, int64_t win_end,
                cudaStream_t s, const float* wn = nullptr, float* zn = nullptr, int64_t ldzn = 0,
                bool z_tf32 = false);

}  // namespace tcg
