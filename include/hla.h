/*
 * hla.h -- C ABI of libhla.so: the B200 (sm_100a) hot path of Hilbert-guided
 * local attention (arXiv 2511.05832).
 *
 * Citation convention: P:Lnnn = line nnn of the paper text.
 *
 * The method (P:L7):
 *   1. image tokens of an H x W grid are reordered along a Hilbert curve
 *      (hla_hilbert_perm; "the path can be precomputed and cached");
 *   2. windows (HWA), slides (HSA) or neighborhoods (HNA) are formed on the
 *      reordered 1D sequence; the N x N attention matrix is tiled into
 *      b_q x b_k blocks that are full, partial or empty (hla_build_block_mask,
 *      P:L85);
 *   3. block-sparse attention skips empty blocks, runs full blocks unmasked and
 *      masks partial blocks element-wise (hla_attn_fwd / hla_attn_bwd, P:L85,
 *      P:L102 Eq. 1).
 * The same kernels run the row-major baselines (WSA / SA / NA2D)
 * and dense attention, selected by hla_pattern_desc.
 *
 * Conventions for every call:
 *   - Tensor pointers are DEVICE pointers owned by the caller.  The library
 *     allocates nothing and keeps no state between calls (thread-safe); the
 *     only host-side state is a thread-local error string (hla_last_error).
 *   - Calls are asynchronous on `stream` unless stated otherwise.
 *   - Every argument check is host-side and synchronous; on any non-OK status
 *     nothing has been launched.  No C++ exception crosses the ABI.
 *   - Q, K, V, O, dO, dQ, dK, dV are bf16 tensors of layout [batch, N, heads,
 *     head_dim] (head_dim contiguous), N = grid_h * grid_w, with token rows in
 *     the sequence order of the pattern (Hilbert order for Hilbert patterns,
 *     row-major grid order otherwise).  Base pointers must be 16-byte aligned.
 *   - LSE / D are fp32 [batch, heads, N].
 */
#ifndef HLA_H_
#define HLA_H_

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime_api.h>

#if defined(__GNUC__)
#define HLA_API __attribute__((visibility("default")))
#else
#define HLA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HLA_OK = 0,
  HLA_ERR_INVALID = 1,      /* malformed arguments (window does not divide grid, N mismatch, ...) */
  HLA_ERR_UNSUPPORTED = 2,  /* valid but outside the hot path's limits (head_dim, block, grid) */
  HLA_ERR_CAPACITY = 3,     /* caller's CSR arrays too small; *nnz_out holds the needed size */
  HLA_ERR_CUDA = 4          /* a CUDA runtime/driver call failed; see hla_last_error() */
} hla_status;

typedef enum {
  HLA_ORDER_ROW_MAJOR = 0,  /* token t = row*W + col */
  HLA_ORDER_HILBERT = 1,    /* token s = position on the Hilbert curve */
  HLA_ORDER_HILBERT_TILED = 2
  /* The Hilbert order with every aligned 64-token segment (an aligned 8 x 8 cell square of
   * a square 2^k grid, k >= 3) relabeled in raster order (hla_hilbert_tiled_index).  Not a
   * curve of the paper: an implementation order that is the SAME attention for the patterns
   * whose predicates only see whole 64-token segments -- HWA with n a multiple of 64 tokens
   * (the window of position s is s/n, unchanged by a relabeling inside a segment) and DENSE
   * (reading R23).  Any other pattern or grid: HLA_ERR_UNSUPPORTED.  With head_dim
   * 32 and the fused reorder the kernels load every aligned 64 positions (an aligned 8 x 8
   * cell square, raster order) with one 5-D TMA box instead of 16 .tile::gather4 ops. */
} hla_order;

/* Pattern families.  With order = HILBERT they are the paper's HWA / HSA / HNA /
 * HSWA, formed on the 1D Hilbert sequence with n = win_h*win_w tokens and
 * r = n/2.  With order = ROW_MAJOR they are the
 * conventional 2D baselines WSA / SA / NA2D.  Predicates (q, k
 * are sequence positions; (rho, gamma) = (t / W, t % W)):
 *   WINDOW        HWA : q/n == k/n                     WSA : rho_q/wh == rho_k/wh && gamma_q/ww == gamma_k/ww
 *   SLIDE         HSA : |q-k| <= r                     SA  : |rho_q-rho_k| <= wh/2 && |gamma_q-gamma_k| <= ww/2
 *   NEIGHBORHOOD  HNA : s <= k < s+2r+1,               NA2D: window of wh x ww cells whose start
 *                       s = clamp(q-r, 0, N-2r-1)            is clamped into the grid
 *   SHIFTED_WINDOW HSWA: floor((q-shift)/n) == floor((k-shift)/n)   (Hilbert order only)
 *   DENSE         every pair (FlashAttention baseline)                               */
typedef enum {
  HLA_WINDOW = 0,
  HLA_SLIDE = 1,
  HLA_NEIGHBORHOOD = 2,
  HLA_DENSE = 3,
  HLA_SHIFTED_WINDOW = 4
} hla_pattern;

typedef enum {
  HLA_TO_HILBERT = 0,       /* grid order  -> Hilbert order */
  HLA_FROM_HILBERT = 1      /* Hilbert order -> grid order  */
} hla_perm_dir;

/* The problem statement of the paper: H x W token grid, window / neighborhood
 * size, block size. */
typedef struct {
  int32_t grid_h, grid_w;   /* N = grid_h * grid_w */
  int32_t order;            /* hla_order: sequence order the tensors are in */
  int32_t pattern;          /* hla_pattern */
  int32_t win_h, win_w;     /* window / kernel in cells; Hilbert patterns use n = win_h*win_w tokens */
  int32_t shift;            /* HSWA 1D shift in tokens (0 < shift < n); must be 0 otherwise */
  int32_t block_q, block_k; /* tile shape b_q x b_k.  Mask builder: any >= 1.
                               Attention: block_q == block_k, 64 or 128. */
  /* Window / kernel sizes: WINDOW and SHIFTED_WINDOW need win_h | grid_h and win_w | grid_w
     (S:L98); SLIDE / NEIGHBORHOOD accept even kernels too, with radius floor(n/2) (DESIGN.md
     reading R5: BASELINE cfg3 uses a 16 x 16 = 256-token slide) -- an even 2D kernel then
     spans 2*floor(k/2)+1 rows / columns (SA) or k cells with an off-centre clamped start
     (NA2D, NATTEN's convention for the start). */
} hla_pattern_desc;

/* Block mask in CSR form (caller-allocated DEVICE arrays).  Entry kinds:
 * 1 = full (no element mask), 2 = partial (element-masked); empty tiles are not
 * listed.  Lists are ascending.  Immutable after the build and shared
 * read-only by every (batch, head) slice and every rank. */
typedef struct {
  int32_t n_qblocks, n_kblocks;  /* = ceil(N/block_q), ceil(N/block_k) */
  int64_t capacity;              /* entries available in col_idx/kind and t_col_idx/t_kind */
  int32_t* row_ptr;              /* [n_qblocks+1]  q-block -> kv-blocks (forward)  */
  int32_t* col_idx;              /* [capacity]                                     */
  uint8_t* kind;                 /* [capacity]                                     */
  int32_t* t_row_ptr;            /* [n_kblocks+1]  kv-block -> q-blocks (backward) */
  int32_t* t_col_idx;            /* [capacity]                                     */
  uint8_t* t_kind;               /* [capacity]                                     */
  int64_t* counts;               /* [4]: nnz, n_full, n_partial, n_empty           */
  /* Optional backward dQ plan (hla_build_bwd_plan).  In effect only when t_dq and
     q_dq_local are non-NULL and n_dq_nonlocal >= 0 (zero-initialised = no plan). */
  uint8_t* t_dq;                 /* [capacity] per transposed entry: HLA_DQ_* bits  */
  uint8_t* q_dq_local;           /* [n_qblocks] (block 64: per 128-row tile) 1 = dQ rows written by bwd_main */
  int32_t n_dq_nonlocal;         /* host: q-blocks with q_dq_local == 0 (-1: none)  */
  /* Host copy of counts (nnz, n_full, n_partial, n_empty), written by the fill call of
     hla_build_block_mask.  The backward picks its schedule from it: the full-tile
     schedule when n_full >= n_partial, the half-tile schedule otherwise (all zero,
     e.g. a mask not built by the library: half-tile).  The choice changes speed only. */
  int64_t host_counts[4];
  /* Attention tiling of a block-64 mask (hla_build_tile_lists; unused at block 128).  The
     kernels run 128 x 128 MMA tiles at 64-granular offsets: each 128-row tile (64-q-blocks
     2t, 2t+1) walks the union of the two blocks' kv lists cut into 128-key windows that
     start on any 64-block, so the columns it executes follow the block-64 sparsity (P:L85,
     tab:blocksize P:L172-190).  Forward lists per 128-q tile, transposed lists per 128-key
     tile; window kind 1 = all four 64 x 64 sub-tiles full (no element mask), 2 = otherwise. */
  int32_t* w_row_ptr;            /* [ceil(n_qblocks/2)+1]                             */
  int32_t* w_col;                /* [w_capacity] first kv 64-block of each window      */
  uint8_t* w_kind;               /* [w_capacity]                                       */
  int32_t* wt_row_ptr;           /* [ceil(n_kblocks/2)+1]                             */
  int32_t* wt_col;               /* [w_capacity] first q 64-block of each window       */
  uint8_t* wt_kind;              /* [w_capacity]                                       */
  int64_t w_capacity;
  int64_t w_counts[4];           /* host: windows, full windows (forward lists), same
                                    for the transposed lists                          */
} hla_block_mask;

/* Bits of hla_block_mask.t_dq.  The backward walks the transposed lists in work
 * units of two kv-blocks (2p, 2p+1) of one (batch, head); inside a unit the dQ_i
 * partial products of consecutive tiles with the same q-block i are chained in
 * one of two TMEM accumulators instead of being reduced into the fp32 workspace
 * one tile at a time.  A chain that covers q-block i's whole forward list is
 * the finished dQ_i and is written to dq directly (bf16). */
enum {
  HLA_DQ_BUF = 1,       /* TMEM dQ accumulator (0 / 1) of the tile's chain          */
  HLA_DQ_NEW = 2,       /* first tile of its chain (the dQ MMA overwrites)          */
  HLA_DQ_DRAIN = 4,     /* last tile of its chain (the accumulator is drained)      */
  HLA_DQ_LOCAL = 8      /* drained chain = complete dQ_i: written to dq as bf16     */
};

/* ---------------------------------------------------------------------------
 * hla_hilbert_index -- the cached Hilbert path: seq_to_cell[s] = cell
 * (row*W + col) of the s-th curve position, cell_to_seq = its inverse.  Either
 * output may be NULL.  Curve: classic Hilbert d2xy with x = column, y = row,
 * starting at (0,0) (reading R1).  Square 2^k grids: computed on the
 * device by a bit-loop kernel (asynchronous on `stream`).  Any other H x W
 * (1 <= H*W < 2^30; the paper's 56^2, 96^2, 160^2, 128x256 rows): the
 * generalized ("gilbert") curve, built on the host and copied -- this path
 * synchronises `stream` before returning (DESIGN.md f4, reading R2).
 * Invalid sizes: HLA_ERR_INVALID.
 */
HLA_API hla_status hla_hilbert_index(int32_t grid_h, int32_t grid_w,
                             int32_t* seq_to_cell, int32_t* cell_to_seq,
                             cudaStream_t stream);

/* ---------------------------------------------------------------------------
 * hla_hilbert_tiled_index -- seq_to_cell / cell_to_seq of HLA_ORDER_HILBERT_TILED:
 * position s of the Hilbert curve (hla_hilbert_index) with cell (row, col) moves to
 * (s & ~63) + 8 * (row & 7) + (col & 7).  Square 2^k grids with k >= 3 only (else
 * HLA_ERR_UNSUPPORTED); device kernel, asynchronous on `stream`; either output may be NULL.
 */
HLA_API hla_status hla_hilbert_tiled_index(int32_t grid_h, int32_t grid_w,
                                   int32_t* seq_to_cell, int32_t* cell_to_seq,
                                   cudaStream_t stream);

/* ---------------------------------------------------------------------------
 * hla_hilbert_perm -- reorder token rows between grid order and Hilbert order
 * ("image tokens are first reordered along a Hilbert curve", P:L7; the
 * "Reshape" step of P:L196).  Both directions are gathers:
 *   TO_HILBERT  : dst[b, s, :] = src[b, seq_to_cell[s], :]
 *   FROM_HILBERT: dst[b, t, :] = src[b, cell_to_seq[t], :]
 * src, dst: HOST arrays of n_tensors (1..4) DEVICE pointers, each a tensor of
 * [batch, N, row_bytes] bytes (bit-exact copy; any element type).  row_bytes
 * must be a multiple of 16 and pointers 16-byte aligned.  src[i] != dst[i].
 * seq_to_cell_out: optional device int32[N] export of the index table (NULL = skip).
 * Grid must be square 2^k (else HLA_ERR_UNSUPPORTED).
 */
HLA_API hla_status hla_hilbert_perm(int32_t grid_h, int32_t grid_w, int32_t dir,
                            int32_t batch, int32_t row_bytes, int32_t n_tensors,
                            const void* const* src, void* const* dst,
                            int32_t* seq_to_cell_out, cudaStream_t stream);

/* ---------------------------------------------------------------------------
 * hla_build_block_mask -- classify every b_q x b_k tile as full / partial /
 * empty and emit CSR lists, their transpose and counts.
 * Sizing call: if m->col_idx == NULL, only row_ptr, t_row_ptr and counts are
 * written; the call synchronises `stream` and writes nnz to *nnz_out.
 * Fill call: all arrays written; if nnz > m->capacity returns HLA_ERR_CAPACITY
 * with the needed nnz in *nnz_out (row_ptr/t_row_ptr/counts are then valid).
 * The fill call also synchronises (it reads nnz back).  Any block >= 1 and any
 * N are accepted (tiles with padding positions are never full).
 * Not on the per-step path: built once per (shape, pattern, block), like the
 * paper's cached path.
 */
HLA_API hla_status hla_build_block_mask(const hla_pattern_desc* d, hla_block_mask* m,
                                int64_t* nnz_out, cudaStream_t stream);

/* ---------------------------------------------------------------------------
 * hla_build_bwd_plan -- the backward's dQ chaining plan of a filled mask (fill
 * call of hla_build_block_mask done; block_q == block_k).  Writes m->t_dq
 * ([capacity] bytes, HLA_DQ_* bits per transposed entry) and m->q_dq_local
 * ([n_qblocks] bytes), both caller-allocated device arrays, and sets the host
 * field m->n_dq_nonlocal.  Synchronises `stream`.  Not on the per-step path
 * (built once per mask).  The plan changes only how dQ partial products are
 * summed (fewer fp32 reductions; P:L85 block-sparse structure), never which
 * products are summed.  Chains never cross a work unit; within a unit each
 * accumulator holds one chain at a time (a chain that would need a busy
 * accumulator is drained early through the fp32 workspace instead).
 * Block-64 masks (window lists built first, hla_build_tile_lists): the plan is over
 * the window lists -- t_dq per wt_col entry, q_dq_local per 128-row tile -- and is
 * built only when every window starts on a 128-row boundary (e.g. HWA with 64-token
 * windows); otherwise windows overlap in rows and the call leaves n_dq_nonlocal = -1
 * (no plan) and returns HLA_OK.
 */
HLA_API hla_status hla_build_bwd_plan(hla_block_mask* m, cudaStream_t stream);

/* ---------------------------------------------------------------------------
 * hla_build_tile_lists -- the window lists (w_*, wt_*) of a filled block-64 mask
 * (block_q == block_k == 64, fill call of hla_build_block_mask done), needed by the
 * attention calls at block 64.  Built on the host from the CSR lists (copied back),
 * once per mask; synchronises `stream`.  Sizing call: m->w_col == NULL -> writes
 * m->w_counts and the needed capacity to *n_out, nothing else.  Fill call: writes
 * all six arrays and m->w_counts; HLA_ERR_CAPACITY (with *n_out) if w_capacity is
 * too small.  Window formation (per 128-row tile, ascending): the first kv 64-block
 * of the two q-blocks' union not yet covered starts a window covering it and the
 * next 64-block; repeated until the union is covered (same for the transpose). */
HLA_API hla_status hla_build_tile_lists(hla_block_mask* m, int64_t* n_out, cudaStream_t stream);

/* Host helper: the two sparsity ratios of a built mask from its integer counts
 * (host copy of m->counts): empty_tile_ratio = n_empty / (Mq*Mk); sparsity =
 * 1 - nnz*b_q*b_k / N^2, the paper's "Sparsity" column (DESIGN.md
 * reading R7).  Either output may be NULL. */
HLA_API hla_status hla_mask_ratios(const hla_pattern_desc* d, const int64_t counts[4],
                           double* empty_tile_ratio, double* sparsity);

/* ---------------------------------------------------------------------------
 * Score modification (SPEC ScoreMod {none, global-RPB}).
 * HLA_SCORE_GLOBAL_RPB ("HWT enlarges the window to the full feature map,
 * enabling a global relative position bias"; reading R19):
 *   score(q, k) = scale * <q, k> + rpb[h][dr + grid_h - 1][dc + grid_w - 1],
 *   (dr, dc) = cell(q) - cell(k), the 2D grid offset of the pair,
 * added before the mask (masked pairs stay excluded).
 *   rpb         device fp32 [heads][2*grid_h-1][2*grid_w-1], read only.
 *   drpb        backward only: device fp32, same shape; the table gradient
 *               sum_{b, pairs with that offset} dL/dscore is ACCUMULATED into it
 *               (zero it first; fp32 atomics, summation order not deterministic).
 *   seq_to_cell device int32[N]: grid cell of every sequence position of d->order
 *               (hla_hilbert_index for Hilbert orders; NULL = identity, only
 *               valid for row-major patterns).  Independent of the fused-reorder
 *               seq_to_cell argument (which describes the TENSOR layout).
 * Passing NULL (or kind == HLA_SCORE_NONE) as the score_mod argument disables it.
 */
typedef enum { HLA_SCORE_NONE = 0, HLA_SCORE_GLOBAL_RPB = 1 } hla_score_kind;

typedef struct {
  int32_t kind;                 /* hla_score_kind */
  const float* rpb;
  float* drpb;
  const int32_t* seq_to_cell;
} hla_score_mod;

/* ---------------------------------------------------------------------------
 * hla_attn_fwd -- block-sparse attention forward:
 *   for every (b, h, q-block i) and every listed kv-block j (ascending):
 *     S = scale * Q_i K_j^T (tcgen05, fp32 in TMEM); mask only if kind == partial;
 *     online softmax (exp2); O_i += P V_j.
 *   O = O / l (bf16), LSE = m + ln(l) (fp32, natural log).
 * q, k, v, o: bf16 [batch, N, heads, head_dim] in d->order.  lse: fp32
 * [batch, heads, N].  scale <= 0 selects 1/sqrt(head_dim).
 * Limits: head_dim in {32, 64}; block_q == block_k in {64, 128}; N % 4 == 0 (a
 * ragged last tile is masked); mask built for the same descriptor
 * (n_qblocks == ceil(N / block)); block 64 also needs the mask's window lists
 * (hla_build_tile_lists).  tiles_visited counts executed 128 x 128 tiles (block
 * 64: windows).
 * tiles_visited: optional device int64 counter; when non-NULL the kernel adds
 * the number of tiles it executed (must equal batch*heads*nnz: empty tiles are
 * skipped).
 * seq_to_cell: NULL -> q, k, v, o are in the sequence order of d->order.
 * Non-NULL (Hilbert patterns only; 16-byte aligned device int32[N] from
 * hla_hilbert_index) -> FUSED REORDER: q, k, v, o are in GRID (row-major cell)
 * order; the kernel gathers each 128-token Hilbert tile with TMA .tile::gather4
 * row loads and writes O rows back to their grid cells, so the separate
 * "Reshape" passes of P:L196 disappear.  LSE stays in
 * sequence order.  For d->order == HLA_ORDER_HILBERT_TILED the table must come from
 * hla_hilbert_tiled_index (its aligned 8 positions are assumed to be 8 consecutive cells).
 */
HLA_API hla_status hla_attn_fwd(const hla_pattern_desc* d, const hla_block_mask* m,
                        int32_t batch, int32_t heads, int32_t head_dim, float scale,
                        const void* q, const void* k, const void* v,
                        void* o, float* lse, const int32_t* seq_to_cell,
                        const hla_score_mod* score_mod,
                        int64_t* tiles_visited, cudaStream_t stream);

/* ---------------------------------------------------------------------------
 * hla_attn_bwd -- backward of hla_attn_fwd over the transposed lists.
 *   P = exp(scale*S - LSE) (masked -> 0 on partial tiles), D = rowsum(dO o O),
 *   dV = P^T dO, dS = P o (dO V^T - D), dK = scale dS^T Q, dQ = scale dS K.
 * q, k, v, o, dout, dq, dk, dv: bf16 [batch, N, heads, head_dim]; lse from the
 * forward.  workspace: device memory of at least hla_attn_bwd_workspace(...)
 * bytes, 256-byte aligned (fp32 dQ accumulator + D); its contents need not be
 * initialised.  dQ accumulation uses fp32 TMA reduce-adds (summation order is
 * not deterministic; covered by the stated tolerance), except for the q-blocks
 * the mask's optional dQ plan (hla_build_bwd_plan) marks local, whose dQ is
 * summed in TMEM and written directly.  Same limits as the forward.
 * seq_to_cell: as in hla_attn_fwd (fused reorder: every bf16 tensor in grid order).
 * score_mod: as in hla_attn_fwd (same table); with global RPB, drpb receives the
 * table gradient (accumulated; hla_attn_bwd zeroes it first, hla_attn_bwd_main
 * does not).
 * Without a global RPB, when the mask's dQ plan makes every q-block local -- or the
 * mask is a block-64 one with non-local q-blocks (half-tile schedule) -- hla_attn_bwd
 * folds the preprocess into the main kernel (hla_attn_bwd_fuses_preprocess): it reads
 * the raw LSE and the O rows itself and forms D in the kernel; non-local dQ rows are
 * zeroed by a write-only pass and finalized as usual.  Same results up to the fp32
 * summation order of D.
 */
HLA_API hla_status hla_attn_bwd(const hla_pattern_desc* d, const hla_block_mask* m,
                        int32_t batch, int32_t heads, int32_t head_dim, float scale,
                        const void* q, const void* k, const void* v, const void* o,
                        const float* lse, const void* dout,
                        void* dq, void* dk, void* dv, const int32_t* seq_to_cell,
                        const hla_score_mod* score_mod,
                        void* workspace, size_t workspace_bytes,
                        int64_t* tiles_visited, cudaStream_t stream);

/* The three stages of hla_attn_bwd, callable separately (SURVEY 8(a) rows a6,
 * a7, a8) so they can be timed / overlapped individually.  Same arguments and
 * limits as hla_attn_bwd; the workspace carries D and the fp32 dQ accumulator
 * from one stage to the next and must not be touched in between.  All three
 * must see the same mask plan (plan_mask = the mask given to main; NULL or a
 * mask without plan = every q-block through the fp32 accumulator).
 *   preprocess: D = rowsum(dO o O) (fp32, stored x scale), LSE -> log2 domain,
 *               dQ accumulator := 0 for the q-blocks that are not local
 *   main      : the tcgen05 kernel over the transposed lists; writes dK, dV,
 *               writes dQ of local q-blocks (bf16) and accumulates the others
 *               (fp32, TMA reduce-add, sequence order)
 *   finalize  : dQ = bf16(accumulator) of the non-local q-blocks, written to
 *               grid cells when seq_to_cell is given (fused inverse reorder);
 *               launches nothing when the plan has no non-local q-block      */
HLA_API hla_status hla_attn_bwd_preprocess(int32_t batch, int32_t heads, int32_t n, int32_t head_dim,
                                   float scale, const void* o, const void* dout, const float* lse,
                                   const int32_t* seq_to_cell, const hla_block_mask* plan_mask,
                                   void* workspace, size_t workspace_bytes, cudaStream_t stream);
HLA_API hla_status hla_attn_bwd_main(const hla_pattern_desc* d, const hla_block_mask* m,
                             int32_t batch, int32_t heads, int32_t head_dim, float scale,
                             const void* q, const void* k, const void* v,
                             const void* dout, void* dq, void* dk, void* dv, const int32_t* seq_to_cell,
                             const hla_score_mod* score_mod,
                             void* workspace, size_t workspace_bytes,
                             int64_t* tiles_visited, cudaStream_t stream);
HLA_API hla_status hla_attn_bwd_finalize(int32_t batch, int32_t heads, int32_t n, int32_t head_dim,
                                 const void* workspace, size_t workspace_bytes, void* dq,
                                 const int32_t* seq_to_cell, const hla_block_mask* plan_mask,
                                 cudaStream_t stream);

HLA_API size_t hla_attn_bwd_workspace(int32_t batch, int32_t heads, int32_t n, int32_t head_dim);

/* 1 if hla_attn_bwd folds the preprocess into its main kernel for this pattern, mask
 * (with its dQ plan) and score_mod -- one launch instead of preprocess + main -- else 0
 * (also 0 for invalid arguments).  Host-only; launches nothing. */
HLA_API int32_t hla_attn_bwd_fuses_preprocess(const hla_pattern_desc* d, const hla_block_mask* m,
                                              const hla_score_mod* score_mod);

/* Thread-local message for the last non-OK status of this thread ("" if none). */
HLA_API const char* hla_last_error(void);

/* Library build identification (arch, version). */
HLA_API const char* hla_version(void);

#ifdef __cplusplus
}
#endif

#endif  /* HLA_H_ */
