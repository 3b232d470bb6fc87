/*
 * hla_debug.h -- bring-up entry points of libhla.so (not part of the hot path).
 *
 * hla_debug_umma: one CTA computes C[m][n] = sum_k A(m,k) * B(n,k) (fp32) with
 * tcgen05.mma (M = 128, kind::f16, bf16 inputs), staging the operands in shared
 * memory in the canonical SWIZZLE_128B layouts the attention kernels use, so the
 * descriptor / instruction-descriptor encodings can be checked against a plain
 * matmul.  A is stored [M][K] (a_major_mn = 0, K-major) or [K][M] (a_major_mn =
 * 1, MN-major); B is stored [N][K] (b_major_mn = 0) or [K][N] (b_major_mn = 1).
 * a_from_tmem = 1 stages A in tensor memory instead (then a_major_mn must be 0).
 * Limits: M == 128, N in {64,128,192,256}, K in {64, 128}.  All pointers device;
 * synchronous w.r.t. `stream` ordering only (asynchronous call).
 */
#ifndef HLA_DEBUG_H_
#define HLA_DEBUG_H_

#include "hla.h"

#ifdef __cplusplus
extern "C" {
#endif

HLA_API hla_status hla_debug_umma(const void* A, const void* B, float* C, int32_t M, int32_t N, int32_t K,
                          int32_t a_major_mn, int32_t b_major_mn, int32_t a_from_tmem, cudaStream_t stream);

/* hla_debug_gather4: 128 token rows idx[0..127] (row = batch*N + token) of head `head`
 * of a bf16 [rows, heads, head_dim] tensor, loaded with TMA .tile::gather4 into a
 * swizzled shared-memory tile and written back unswizzled to out[128][head_dim].
 * box_h: second box dimension of the 2-D tensor map (bring-up parameter). */
HLA_API hla_status hla_debug_gather4(const void* src, int64_t rows, int32_t heads, int32_t head_dim,
                                     const int32_t* idx, int32_t head, int32_t box_h, void* out,
                                     cudaStream_t stream);

/* hla_debug_mma_rate: `iters` back-to-back tcgen05.mma (M=128, N, K=16) from one CTA;
 * out_cycles (device int64[1]) = SM cycles from first issue to commit completion. */
HLA_API hla_status hla_debug_mma_rate(int32_t N, int32_t iters, int32_t a_major_mn, int32_t b_major_mn,
                                      int32_t a_from_tmem, long long* out_cycles, cudaStream_t stream);

/* hla_debug_tmem_rate: nwarps warps each issue `iters` tcgen05.ld (mode 0) / .st (mode 1)
 * 32x32b.x32 (4 KB per warp-instruction), waiting every `batch`; out_cycles = SM cycles. */
HLA_API hla_status hla_debug_tmem_rate(int32_t nwarps, int32_t iters, int32_t mode, int32_t batch,
                                       long long* out_cycles, cudaStream_t stream);

/* hla_debug_ex2_rate: one CTA of `threads` threads, each `iters` x 16 independent
 * ex2.approx.f32; out_cycles = SM cycles (MUFU throughput probe). */
HLA_API hla_status hla_debug_ex2_rate(int32_t threads, int32_t iters, long long* out_cycles, float* sink,
                                      cudaStream_t stream);

/* hla_debug_xu_rate: one CTA of `threads` threads, each `iters` x 16 independent instances of
 * one XU-pipe instruction form (mode 0 ex2.f32, 1 ex2.bf16x2, 2 ex2.f16x2, 3 cvt.rn.bf16x2.f32,
 * 4/5/6 softmax pair-loop variants, see debug_umma.cu); out_cycles[0] = SM cycles. */
HLA_API hla_status hla_debug_xu_rate(int32_t mode, int32_t threads, int32_t iters, long long* out_cycles,
                                     uint32_t* sink, cudaStream_t stream);

/* hla_debug_sync_latency: one CTA; out_cycles[0] = SM cycles per round trip of mode 0
 * tcgen05.commit -> mbarrier -> wait (no MMA), 1 one 128x128x16 MMA + commit -> wait, 2 warp <-> warp
 * mbarrier ping-pong (one arrive each way), 3 as 2 with 32 arriving threads on the way back. */
HLA_API hla_status hla_debug_sync_latency(int32_t mode, int32_t iters, long long* out_cycles, cudaStream_t stream);

/* hla_debug_softmax_tile: `blocks` CTAs x 128 threads run the forward softmax tile body
 * with its TMEM traffic (S ld, max, exp2, P st), `iters` times; out_cycles[cta]. */
HLA_API hla_status hla_debug_softmax_tile(int32_t blocks, int32_t iters, long long* out_cycles, uint32_t* sink,
                                          cudaStream_t stream);
/* hla_debug_load_rate: `ctas` CTAs (one per SM) each stream `tiles` 16 KB tiles (128
 * token rows x 64 bf16 of one head of a [rows, heads, 64] tensor) through a `stages`-deep
 * shared-memory ring; mode 0 = one 3-D TMA box, 1 = 32 TMA gather4, 2 = cp.async by 128
 * threads, 3 = one 16 KB contiguous bulk copy.  out_cycles[cta] = clock64 span. */
HLA_API hla_status hla_debug_load_rate(const void* src, int64_t rows, int32_t heads, int32_t mode, int32_t stages,
                                       int32_t ctas, int32_t tiles, long long* out_cycles, cudaStream_t stream);
/* hla_debug_softmax_rate: `blocks` CTAs x 128 threads run the forward softmax inner
 * loop (128 exps per thread) `iters` times; out_cycles[block] = SM cycles. */
HLA_API hla_status hla_debug_softmax_rate(int32_t blocks, int32_t iters, long long* out_cycles, uint32_t* sink,
                                          cudaStream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* HLA_DEBUG_H_ */
