/*
 * tcg.h — C ABI of the B200-native TC-GNN hot path (libtcg_b200.so).
 *
 * Every entry point takes plain device pointers, int64 sizes and a
 * cudaStream_t (passed as void* so this header needs no CUDA include); it is
 * stream-ordered, never allocates or frees caller memory, never throws across
 * the ABI and returns 0 on success or a negative TCG_E* code; tcg_last_error()
 * gives the thread-local message of the last failure. Outputs are written
 * only; callers allocate them (the torch caching allocator in the Python
 * host layer). Nothing here falls back to the CPU.
 *
 * Each entry point replaces one function of the reference package `tcgraph`
 * (/root/reference/pkg/src/tcgraph, numpy emulation, no native code); the
 * reference interface it stands in for is cited per function. INTEGRATION.md
 * shows the ctypes binding the reference would add for each symbol.
 */
#ifndef TCG_B200_H
#define TCG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TCG_OK 0
#define TCG_E_INVALID (-1)   /* bad argument (shape, null pointer, mode)   */
#define TCG_E_CUDA (-2)      /* CUDA launch / runtime error                */
#define TCG_E_WORKSPACE (-3) /* workspace too small                        */
#define TCG_E_UNSUPPORTED (-4)

#define TCG_ACT_NONE 0
#define TCG_ACT_RELU 1 /* tcg_spmm_act: ReLU on the stored output */

#define TCG_PREC_F32 0  /* exact f32: CSR-order fold, bitwise = reference f32 */
#define TCG_PREC_TF32 1 /* tensor cores: RNE-to-tf32 operands, f32 accumulate */
/* flag bits (round 2): OR-ed into tcg_spmm's precision, tcg_dense's relu and the
 * flags of the *_ex AGNN entry points. The operand is already on the tf32 grid
 * (RN-rounded by its producer), so the kernels skip its rounding; the results are
 * those of the unflagged call on the same values. */
#define TCG_PREC_X2_TF32 0x10 /* tcg_spmm, tf32: x2 pre-rounded */
#define TCG_DENSE_OUT_TF32 0x2 /* tcg_dense: round the stored output RN to tf32 */
#define TCG_AGNN_Z_TF32 0x1    /* tcg_agnn_*_ex: z pre-rounded */

/* SDDMM epilogues (fused per row window; rows never straddle windows). */
#define TCG_EPI_NONE 0        /* out[e] = <xa[row e], xb[col e]>                 */
#define TCG_EPI_SOFTMAX 1     /* out[e] = row softmax of the scores               */
#define TCG_EPI_SOFTMAX_BWD 2 /* out[e] = P_e (s_e - sum_row P s), P = aux        */

/* Device-resident SGT result (reference TiledGraph, sgt.py:43-98) plus the
 * CSR it was built from. All pointers are device pointers. */
typedef struct tcg_tiling {
  int64_t num_nodes;            /* N                                         */
  int64_t num_edges;            /* M                                         */
  int64_t num_windows;          /* W = ceil(N / blk_h)                        */
  int64_t num_unique;           /* U = col_offsets[W]                         */
  int32_t blk_h, blk_w;         /* BlockConfig (sgt.py:21-40)                 */
  const int64_t* node_ptr;      /* i64[N+1]  CsrGraph.node_pointer            */
  const uint32_t* edge_list;    /* u32[M]    CsrGraph.edge_list               */
  const uint32_t* edge_to_col;  /* u32[M]    TiledGraph.edge_to_col           */
  const int64_t* col_offsets;   /* i64[W+1]  TiledGraph.col_offsets           */
  const uint32_t* col_to_node;  /* u32[U]    TiledGraph.col_to_node           */
  const uint32_t* win_partition;/* u32[W]    TiledGraph.win_partition         */
  const uint32_t* edge_frag;    /* u32[M]    mma fragment slot of each edge in
                                   its 16x8 A tile (tcg_edge_frag; TF32 only) */
  int64_t max_window_edges;     /* max edges of one window (0 = unknown)       */
  int64_t max_window_unique;    /* max condensed columns of one window         */
  /* Block stream (tcg_block_stream; optional, TF32 16x8 only; null => the
   * window engine runs): */
  const int32_t* block_offsets; /* i32[W+1] exclusive cumsum of win_partition:
                                   the per-window TC-block offsets            */
  const uint32_t* col_stream;   /* u32[8*(TB+TCG_STREAM_PAD)], TB = block_offsets[W]:
                                   col_to_node padded per window to whole
                                   8-column blocks, pair-interleaved          */
  /* Pair stream (tcg_block_stream_pairs; optional): the same with every
   * window padded to an even block count, for the 16-wide SpMM that consumes
   * two blocks per step. */
  const int32_t* pair_offsets;  /* i32[W+1] exclusive cumsum of win_partition rounded up to even */
  const uint32_t* pair_stream;  /* u32[8*(TP+TCG_STREAM_PAD)], TP = pair_offsets[W] */
} tcg_tiling;

/* Blocks of padding tcg_block_stream appends after the column stream. */
#define TCG_STREAM_PAD 16

/* ---- library ---------------------------------------------------------- */
const char* tcg_last_error(void);
const char* tcg_version(void);
/* Number of kernels this library has launched in this process (all entry
 * points; a CUDA-graph replay of captured launches is not re-counted). */
int64_t tcg_launch_count(void);
/* Multiprocessor count / L2 bytes of the current device (0 if unavailable). */
int tcg_device_info(int64_t* num_sms, int64_t* l2_bytes);

/* ---- graph normalisation / invariants ---------- */
/* Reference CsrGraph.from_edges (graph.py:55-89) on the device: sort the
 * (src, dst) pairs by (row, column) with one stable radix sort, collapse
 * duplicates, sum duplicate values (nullable) in input order in float64 and
 * build node_ptr[N+1]. edge_list / edge_values need capacity num_edges; the
 * surviving count is node_ptr[N]. Ids must lie in [0, N) for src and
 * [0, 2^32) for dst; bad_ids (device i64) receives the number of pairs that
 * do not (outputs are then unspecified). */
size_t tcg_from_edges_workspace_bytes(int64_t num_edges);
int tcg_from_edges(const int64_t* src, const int64_t* dst, const float* values,
                   int64_t num_edges, int64_t num_nodes, int64_t* node_ptr,
                   uint32_t* edge_list, float* edge_values, int64_t* bad_ids,
                   void* workspace, size_t workspace_bytes, void* stream);
/* Reference validate() (graph.py:92-142) counts on the device: report[6]
 * (device u64) = first non-monotone row, #such rows, first out-of-range
 * column, #such edges, first unsorted/duplicate column, #such edges (first =
 * 2^64-1 when none). The caller formats the reference messages. Workspace:
 * 48 bytes. */
int tcg_validate(const int64_t* node_ptr, const uint32_t* edge_list, int64_t num_nodes,
                 int64_t num_edges, int64_t* report, void* workspace, size_t workspace_bytes,
                 void* stream);

/* ---- tile accounting ---------------------------- */
/* Reference structure_blocks_before (sgt.py:199-217), equal to
 * count_blocks_before (sgt.py:140-157) on the same graph: per window the
 * distinct col_to_node // tile_width buckets (per_window i64[W]) and their
 * total (device i64). */
int tcg_structure_blocks(const tcg_tiling* t, int64_t tile_width, int64_t* per_window,
                         int64_t* total, void* stream);

/* ---- SGT: reference sgt.translate (sgt.py:101-137) ---------------------- */
/* Workspace bytes tcg_sgt needs for this graph size. */
size_t tcg_sgt_workspace_bytes(int64_t num_nodes, int64_t num_edges, int32_t blk_h);
/* Two-phase form. tcg_sgt_count writes edge_to_col[M]
 * and col_offsets[W+1] (exclusive scan of the per-window unique counts, so
 * U = col_offsets[W]); the caller allocates col_to_node (U entries, or its
 * upper bound M without reading U back) and calls tcg_sgt_fill, which writes
 * col_to_node and win_partition[W]. Windows of <= 512 edges are ranked by one
 * warp each (register bitonic sort of (column, edge) keys, warp-scan dedup);
 * larger ones by a CTA. Workspace as tcg_sgt_workspace_bytes (count only). */
int tcg_sgt_count(const int64_t* node_ptr, const uint32_t* edge_list, int64_t num_nodes,
                  int64_t num_edges, int32_t blk_h, int32_t blk_w, uint32_t* edge_to_col,
                  int64_t* col_offsets, void* workspace, size_t workspace_bytes, void* stream);
int tcg_sgt_fill(const int64_t* node_ptr, const uint32_t* edge_list, int64_t num_nodes,
                 int64_t num_edges, int32_t blk_h, int32_t blk_w, const uint32_t* edge_to_col,
                 const int64_t* col_offsets, uint32_t* win_partition, uint32_t* col_to_node,
                 void* stream);
/* Row-window shard of SGT (windows are independent; no
 * reference counterpart, sgt.py:101-137 restricted to windows
 * [win_begin, win_end)). Count: edge_to_col of the range's edges,
 * win_partition[win_begin..win_end) and col_offsets[win_begin..win_end] =
 * exclusive scan of the range's unique counts starting at 0 (arrays are
 * global-sized; nothing outside the range is touched). Fill: col_to_node at
 * col_offsets[w] + base for the range's windows, then
 * col_offsets[win_begin..win_end] += base -- with base = the exclusive scan of
 * the lower shards' totals the range matches the whole-graph SGT bit for bit.
 * tcg_sgt_count / tcg_sgt_fill / tcg_sgt are the whole-graph forms. */
int tcg_sgt_count_range(const int64_t* node_ptr, const uint32_t* edge_list, int64_t num_nodes,
                        int64_t num_edges, int32_t blk_h, int32_t blk_w, int64_t win_begin,
                        int64_t win_end, uint32_t* edge_to_col, int64_t* col_offsets,
                        uint32_t* win_partition, void* workspace, size_t workspace_bytes,
                        void* stream);
int tcg_sgt_fill_range(const int64_t* node_ptr, const uint32_t* edge_list, int64_t num_nodes,
                       int64_t num_edges, int32_t blk_h, int64_t win_begin, int64_t win_end,
                       int64_t base, const uint32_t* edge_to_col, int64_t* col_offsets,
                       uint32_t* col_to_node, void* stream);
/* One stream-ordered call (count + fill): per-window sort/dedup/rank on the GPU.
 * Writes win_partition[W], edge_to_col[M], col_offsets[W+1] and
 * col_to_node[0..U) where U = col_offsets[W] (col_to_node capacity must be
 * >= M). Bit-exact with the reference for any blk_h, blk_w >= 1. */
int tcg_sgt(const int64_t* node_ptr, const uint32_t* edge_list, int64_t num_nodes,
            int64_t num_edges, int32_t blk_h, int32_t blk_w, uint32_t* win_partition,
            uint32_t* edge_to_col, int64_t* col_offsets, uint32_t* col_to_node,
            void* workspace, size_t workspace_bytes, void* stream);

/* edgeToRow of the TC-GNN preprocessing: the row of each edge inside its
 * row window (reference TiledGraph.window_edge_rows, sgt.py:84-90, for all
 * windows at once); edge_to_row u32[M]. */
int tcg_edge_to_row(const int64_t* node_ptr, int64_t num_nodes, int32_t blk_h,
                    uint32_t* edge_to_row, void* stream);
/* Per-edge fragment slot for the TF32 kernels (16x8 tilings): edge e of row
 * r with condensed column c lands at (c/8)*128 + lane*4 + slot of its
 * window's A tiles, lane = (r%8)*4 + c%4, slot = r%16/8 + 2*(c%8/4). Derived
 * once per tiling, like the reference's per-edge _spmm_aux cache
 * (kernels.py:173-188: r_local, b_of_edge, c_local). */
int tcg_edge_frag(const tcg_tiling* t, uint32_t* edge_frag, void* stream);

/* Per-window TC-block offsets (block_offsets[w] = sum of win_partition[0..w),
 * W+1 entries; the "counts and offsets" the reference derives as
 * tile_base, kernels.py:461-462) and the block-padded column stream the SpMM
 * block-stream engine reads (col_stream may be null: offsets only, so the
 * caller can read TB = block_offsets[W] and size col_stream as
 * 8*(TB+TCG_STREAM_PAD) u32). Derived once per tiling. */
int tcg_block_stream(const tcg_tiling* t, int32_t* block_offsets, uint32_t* col_stream,
                     void* stream);
/* The pair stream of the 16-wide SpMM (tcg_tiling.pair_offsets / pair_stream):
 * as tcg_block_stream with win_partition rounded up to even per window (the
 * padding block repeats the window's first node; its A tile is zero). */
int tcg_block_stream_pairs(const tcg_tiling* t, int32_t* pair_offsets, uint32_t* pair_stream,
                           void* stream);
/* dst[k] = src[idx[k]] — carries A's edge weights (P, dS, edge values) into
 * A^T edge order once per backward, so the A^T SpMM reads them coalesced. */
int tcg_permute_f32(const float* src, const uint32_t* idx, float* dst, int64_t n, void* stream);

/* Both arrays through the same permutation in one pass (P and dS). */
int tcg_permute2_f32(const float* src_a, const float* src_b, const uint32_t* idx, float* dst_a,
                     float* dst_b, int64_t n, void* stream);
/* dst[idx[k]] = src[k] (the inverse move of tcg_permute_f32). */
int tcg_scatter_f32(const float* src, const uint32_t* idx, float* dst, int64_t n, void* stream);
/* inv[perm[k]] = k: for A^T's perm, inv[e] is the A^T position of A's edge e. */
int tcg_invert_perm(const uint32_t* perm, int64_t n, uint32_t* inv, void* stream);
/* ---- CSR transpose (backward support; no reference counterpart — the
 * reference has no backward. SURVEY.md Appendix B restates it as
 * CsrGraph.from_edges(dst, src), graph.py:55-89) ------------------------ */
size_t tcg_csr_transpose_workspace_bytes(int64_t num_nodes, int64_t num_edges);
/* ptr_t[N+1], cols_t[M] = A^T in CSR; perm[k] = edge of A that is edge k of
 * A^T (stable by row => equals np.lexsort((rows, cols))). */
int tcg_csr_transpose(const int64_t* node_ptr, const uint32_t* edge_list, int64_t num_nodes,
                      int64_t num_edges, int64_t* ptr_t, uint32_t* cols_t, uint32_t* perm,
                      void* workspace, size_t workspace_bytes, void* stream);

/* ---- SpMM: reference kernels.spmm (kernels.py:213-374, Alg. 2) ----------- */
/* Y[r - y_row0, :] (+)= sum_e w_e * X[col e, :] for rows r of windows
 * [win_begin, win_end), D columns, bias added if non-null.
 *  weights   : nullable f32[M] edge weights (null => 1.0);
 *  weight_idx: nullable u32[M] indirection (w_e = weights[weight_idx[e]]),
 *              used to read A's edge weights in A^T edge order;
 *  x2/weights2/weight_idx2: optional second term accumulated into the same
 *              tile (Y = A_w X + A_w2 X2), used by the AGNN backward;
 *  accumulate: 0 => overwrite Y rows, 1 => Y += result.
 * precision TCG_PREC_F32 is bitwise equal to the reference f32 path
 * (oracle.ref_spmm fold order); TCG_PREC_TF32 uses mma.sync m16n8k8 tf32. */
int tcg_spmm(const tcg_tiling* t, const float* x, int64_t ldx, int64_t dim,
             const float* weights, const uint32_t* weight_idx, const float* x2, int64_t ldx2,
             const float* weights2, const uint32_t* weight_idx2, const float* bias,
             float* y, int64_t ldy, int64_t y_row0, int64_t win_begin, int64_t win_end,
             int32_t precision, int32_t accumulate, void* stream);
/* tcg_spmm (single operand) with an activation on the stored rows: act =
 * TCG_ACT_RELU gives Y = relu(A_w X + bias (+ Y)), fused into the stream
 * engine's epilogue (a separate pass for the other engines). GCN's first
 * layer, relu(gcn_layer(...)). */
int tcg_spmm_act(const tcg_tiling* t, const float* x, int64_t ldx, int64_t dim,
                 const float* weights, const uint32_t* weight_idx, const float* bias, float* y,
                 int64_t ldy, int64_t y_row0, int64_t win_begin, int64_t win_end,
                 int32_t precision, int32_t accumulate, int32_t act, void* stream);

/* ---- SDDMM: reference kernels.sddmm (kernels.py:377-538, Alg. 3) --------- */
/* out[e] = <xa[row e], xb[col e]> for the edges e of windows
 * [win_begin, win_end); xb may equal xa (or be null => xa). Edge-indexed
 * arrays (out, aux, spmm weights) are addressed by absolute edge id: a shard
 * holding only edges [eb, ee) passes base - eb.
 * epilogue TCG_EPI_SOFTMAX fuses kernels.segment_softmax (kernels.py:541-556);
 * TCG_EPI_SOFTMAX_BWD reads aux = P (same indexing) and writes
 * P*(s - sum_row P*s). */
int tcg_sddmm(const tcg_tiling* t, const float* xa, int64_t lda, const float* xb, int64_t ldb,
              int64_t dim, const float* aux, float* out, int64_t win_begin, int64_t win_end,
              int32_t precision, int32_t epilogue, void* stream);

/* ---- segment softmax: reference kernels.segment_softmax (541-556) ------- */
int tcg_segment_softmax(const int64_t* node_ptr, int64_t num_rows, const float* values,
                        float* out, void* stream);
/* dS = P * (dP - rowsum(P * dP)) (backward; no reference counterpart). */
int tcg_segment_softmax_backward(const int64_t* node_ptr, int64_t num_rows, const float* p,
                                 const float* dp, float* ds, void* stream);
/* The same pair under the SURVEY.md Appendix D names. */
int tcg_softmax_fwd(const int64_t* node_ptr, int64_t num_rows, const float* values, float* out,
                    void* stream);
int tcg_softmax_bwd(const int64_t* node_ptr, int64_t num_rows, const float* p, const float* dp,
                    float* ds, void* stream);

/* ---- fused AGNN layer: reference kernels.agnn_layer (586-601) ----------- */
/* SDDMM -> row softmax -> SpMM with one gather of Z's neighbour rows per
 * 8-column block. With the block stream attached and dim == 32 this is
 * agnn_stream<fwd> (scores straight from the SDDMM C fragment into the SpMM
 * A fragment, online softmax); otherwise the window engine stages each
 * window's rows once in shared memory, and shapes neither fits run the two
 * products unfused. Writes P[e] (absolute edge ids; kept for the backward)
 * and Y rows [win_begin, win_end) at y - y_row0. TF32, 16x8 only. */
int tcg_agnn_forward(const tcg_tiling* t, const float* z, int64_t ldz, int64_t dim, float* p,
                     float* y, int64_t ldy, int64_t y_row0, int64_t win_begin, int64_t win_end,
                     void* stream);
/* SURVEY.md Appendix D form: the whole graph, Z dense with row stride dim. */
int tcg_agnn_fused_fwd(const tcg_tiling* t, const float* z, int64_t dim, float* p, float* y,
                       int64_t ldy, void* stream);
/* AGNN backward, A-side half (no reference counterpart):
 * dS = P * (dP - rowsum(P dP)) with dP_e = <G_row, Z_col> (written to ds),
 * and dZ rows = A_dS Z (overwritten). The A^T half (A^T_P G + A^T_dS Z) is
 * one dual tcg_spmm on the transposed tiling with weight_idx = perm. */
int tcg_agnn_backward(const tcg_tiling* t, const float* z, int64_t ldz, const float* gy,
                      int64_t ldg, int64_t dim, const float* p, float* ds, float* dz,
                      int64_t lddz, int64_t dz_row0, int64_t win_begin, int64_t win_end,
                      void* stream);

/* Same A-side half in one pass per window with the row term taken from the
 * forward output: rs_i = sum_j P_ij dP_ij = <G_i, Y_i> (y_fwd: the layer's
 * forward output, absolute rows), so dS_e = P_e (dP_e - rs_i) is exact per
 * 16x8 block and dS and A_dS Z come from a single gather of Z. Falls back to
 * tcg_agnn_backward where the block-stream engine does not apply. */
int tcg_agnn_backward_fused(const tcg_tiling* t, const float* z, int64_t ldz, const float* gy,
                            int64_t ldg, const float* y_fwd, int64_t ld_yfwd, int64_t dim,
                            const float* p, float* ds, float* ds_t, const uint32_t* inv_perm,
                            float* dz, int64_t lddz, int64_t dz_row0, int64_t win_begin,
                            int64_t win_end, void* stream);
/* tcg_agnn_forward / tcg_agnn_backward_fused with flags (TCG_AGNN_Z_TF32: z is
 * already on the tf32 grid, e.g. written by tcg_dense with TCG_DENSE_OUT_TF32). */
int tcg_agnn_forward_ex(const tcg_tiling* t, const float* z, int64_t ldz, int64_t dim, float* p,
                        float* y, int64_t ldy, int64_t y_row0, int64_t win_begin, int64_t win_end,
                        int32_t flags, void* stream);
int tcg_agnn_backward_fused_ex(const tcg_tiling* t, const float* z, int64_t ldz, const float* gy,
                               int64_t ldg, const float* y_fwd, int64_t ld_yfwd, int64_t dim,
                               const float* p, float* ds, float* ds_t, const uint32_t* inv_perm,
                               float* dz, int64_t lddz, int64_t dz_row0, int64_t win_begin,
                               int64_t win_end, int32_t flags, void* stream);
/* tcg_agnn_forward followed by P in A^T edge order (p_t[inv_perm[e]] = p[e];
 * inv_perm from tcg_invert_perm of the transpose's perm), for the backward's
 * A^T SpMM. tcg_agnn_backward_fused does the same for dS when ds_t is given.
 * (Writing the A^T copy from the kernel epilogue was measured slower than
 * this separate coalesced-read scatter.) */
/* tcg_agnn_forward plus the next AGNN layer's dense step in the same launch:
 * z_next = Y w_next (w_next [dim x co] row-major, 3xTF32, fp32-class), for the
 * stacked AGNNConv layers of the paper's model. D = co = 32
 * runs fused in the forward kernel's epilogue; other shapes run the two steps.
 * Rows of z_next follow y (y_row0). */
int tcg_agnn_forward_next(const tcg_tiling* t, const float* z, int64_t ldz, int64_t dim, float* p,
                          float* y, int64_t ldy, int64_t y_row0, int64_t win_begin, int64_t win_end,
                          const float* w_next, int64_t co, float* z_next, int64_t ldzn, void* stream);
int tcg_agnn_forward_t(const tcg_tiling* t, const float* z, int64_t ldz, int64_t dim, float* p,
                       float* p_t, const uint32_t* inv_perm, float* y, int64_t ldy,
                       int64_t y_row0, int64_t win_begin, int64_t win_end, void* stream);
/* ---- dense companions of the layers (fp32; no reference counterpart beyond
 * gcn_layer's `agg @ w + b`, kernels.py:577-582) ---------------------------- */
/* y[n x co] = act((x .* [mask > 0]) . M + bias) (mask: [n x ci]); M is [ci x co]
 * (m_transposed = 0) or [co x ci] (m_transposed = 1). co <= 128. */
int tcg_dense(const float* x, int64_t ldx, int64_t n, int64_t ci, const float* m, int64_t co,
              int32_t m_transposed, const float* bias, int32_t relu, const float* mask,
              int64_t ldm, float* y, int64_t ldy, void* stream);
size_t tcg_gemm_tn_workspace_bytes(int64_t n, int64_t k, int64_t c);
/* out[k x c] = a^T b (b .* [mask > 0] when mask != null), colsum[c] = column
 * sums of the (masked) b; deterministic fixed-order reduction. */
int tcg_gemm_tn(const float* a, int64_t lda, const float* b, int64_t ldb, const float* mask,
                int64_t ldm, int64_t n, int64_t k, int64_t c, float* out, float* colsum,
                void* workspace, size_t workspace_bytes, void* stream);
size_t tcg_dense_backward_workspace_bytes(int64_t n, int64_t ci, int64_t co);
/* Backward of y = x W (W [ci x co], no bias/activation): dx[n x ci] = g W^T and
 * dw[ci x co] = x^T g. For ci = co = 32 (the AGNN layers) one fused pass reads
 * g once for both products; other shapes run tcg_dense + tcg_gemm_tn.
 * Deterministic (fixed-order reductions). */
int tcg_dense_backward(const float* x, int64_t ldx, const float* g, int64_t ldg, int64_t n,
                       int64_t ci, int64_t co, const float* w, float* dx, int64_t lddx, float* dw,
                       void* workspace, size_t workspace_bytes, void* stream);
size_t tcg_colsum_workspace_bytes(int64_t n, int64_t c);
/* out[c] = column sums of x[n x c] (row stride ld); fixed-order two-level
 * reduction (deterministic). The bias gradient of gcn_layer's `+ b`. */
int tcg_colsum(const float* x, int64_t ld, int64_t n, int64_t c, float* out, void* workspace,
               size_t workspace_bytes, void* stream);
/* ReLU backward fused with the bias gradient: gout = x .* [gate > 0] (gate =
 * the layer's ReLU output) and out[c] = column sums of gout, fixed order
 * (deterministic); workspace as tcg_colsum. */
int tcg_colsum_gate(const float* x, int64_t ld, const float* gate, int64_t ldg, int64_t n, int64_t c,
                    float* gout, int64_t ldo, float* out, void* workspace, size_t workspace_bytes,
                    void* stream);
size_t tcg_softmax_xent_workspace_bytes(int64_t n);
/* loss = mean_i -log_softmax(logits_i)[labels_i]; dlogits = (softmax - onehot)/n
 * (dlogits may be null: loss only) */
int tcg_softmax_xent(const float* logits, int64_t ld, const int64_t* labels, int64_t n, int64_t c,
                     float* loss, float* dlogits, void* workspace, size_t workspace_bytes,
                     void* stream);
/* dlogits[n x c] (row stride ldd) = (softmax(logits) - onehot(labels)) / n * g,
 * g = *grad_scale (device scalar; null => 1): the backward recomputes the
 * softmax from the logits instead of keeping dlogits from the forward */
int tcg_softmax_xent_backward(const float* logits, int64_t ld, const int64_t* labels, int64_t n,
                              int64_t c, const float* grad_scale, float* dlogits, int64_t ldd,
                              void* stream);

size_t tcg_linear_xent_workspace_bytes(int64_t n);
/* The output layer fused with the loss: logits = x W + bias (x [n x kin], W
 * [kin x c] row-major, bias may be null) on mma.sync 3xTF32 (fp32-class), then
 * loss = sum_i -log_softmax(logits_i)[labels_i] / div and
 * dlogits[n x c] (row stride ldd) = (softmax - onehot) / div (dlogits may be
 * null: the loss only). The logits never reach memory. div = n for the mean;
 * the global row count for a row shard.
 * Covers kin a multiple of 4 up to 32, c <= 48, 16-B aligned x rows; other
 * shapes return TCG_E_UNSUPPORTED (callers run tcg_dense + tcg_softmax_xent).
 * The last layer and the training loss of the paper's GCN / AGNN models
 * (PAPER.md:684-689). Deterministic. */
int tcg_linear_xent(const float* x, int64_t ldx, int64_t n, int64_t kin, const float* w, int64_t c,
                    const float* bias, const int64_t* labels, int64_t div, float* loss,
                    float* dlogits, int64_t ldd, void* workspace, size_t workspace_bytes,
                    void* stream);

size_t tcg_linear_xent_backward_workspace_bytes(int64_t n, int64_t kin, int64_t c);
/* Backward of tcg_linear_xent for an incoming loss gradient g = *grad_scale
 * (device scalar; null => 1), recomputing the logits instead of reading a
 * stored dlogits: d = (softmax - onehot) * g / div, dx = d W^T (dx may be
 * null), dw = x^T d, db = colsum d (db may be null). Same coverage as
 * tcg_linear_xent (else TCG_E_UNSUPPORTED). Deterministic. */
int tcg_linear_xent_backward(const float* x, int64_t ldx, int64_t n, int64_t kin, const float* w,
                             int64_t c, const float* bias, const int64_t* labels, int64_t div,
                             const float* grad_scale, float* dx, int64_t lddx, float* dw, float* db,
                             void* workspace, size_t workspace_bytes, void* stream);

/* ---- TF32 operand rounding: reference tiles.quantize_tf32 (67-82) ------- */
int tcg_quantize_tf32(const float* in, float* out, int64_t n, void* stream);

/* ---- direct CSR evaluation (the reference oracle API) ------------------------
 * Replace tcgraph.oracle.ref_spmm / ref_sddmm (oracle.py:28-91): no tiling,
 * CSR order. acc_f64 = 0: f32 fold, product rounded then add rounded, from
 * +0.0 (oracle.py:54-59, 86-90), bitwise the reference; `out` is float.
 * acc_f64 = 1: the product (rounded in f32) is widened and summed in double;
 * `out` is double. values = NULL means all ones. tcg_csr_sddmm needs a
 * u32[num_edges] workspace for the edge rows. */
int tcg_csr_spmm(const int64_t* node_ptr, const uint32_t* edge_list, const float* values,
                 int64_t num_nodes, const float* x, int64_t ldx, int64_t dim, void* out,
                 int64_t ldo, int32_t acc_f64, void* stream);
int tcg_csr_sddmm(const int64_t* node_ptr, const uint32_t* edge_list, int64_t num_nodes,
                  int64_t num_edges, const float* x, int64_t ldx, int64_t dim, uint32_t* row_ws,
                  void* out, int32_t acc_f64, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TCG_B200_H */
