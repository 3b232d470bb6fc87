// K8 (half-tile schedule): block-sparse attention backward on sm_100a for masks made
// mostly of PARTIAL tiles (slides, neighbourhoods, shifted / small windows: "partial
// blocks require element-wise masking").  Same operation, operands and outputs as the
// full-tile schedule in attn_bwd.cu (see its header for the gradient formulas); chosen by
// hla_attn_bwd_main when partial tiles outnumber full ones.
//
// Persistent, 1 CTA / SM, kv-major over the transposed CSR (work unit = a pair of
// consecutive kv-blocks of one (b, h)).  512 threads = 16 warps:
//    warps 0, 14, 15  TMA producers: K_j (+ LSE_i, D_i bulk copies) / V_j, Q_i / dO_i;
//    warp 1     TMEM allocator + single-thread tcgen05.mma issuer:
//                 S^T  = K_j Q_i^T     (SS, N = 64 per query half, TMEM cols [0,128))
//                 dP^T = V_j dO_i^T    (SS, N = 64 per query half, TMEM cols [128,256))
//                 dV  += P^T dO_i      (TS, P^T bf16 written over the first 16 columns of
//                                       each 32-column S^T chunk; acc [384,448))
//                 dK  += dS^T Q_i      (SS, dS^T bf16 in smem, K-major view; acc [448,512))
//                 dQ_i (+)= dS K_j     (SS, same dS smem, MN-major view; two accumulators
//                                       [256,320) / [320,384) chained by the mask's dQ plan)
//               half-tile software pipeline: the tensor core works on one 64-query half
//               while the compute warps turn the other into P^T / dS^T, so the element
//               masks of partial tiles overlap the MMAs;
//    warps 2-9  thread = key row (two warps per TMEM lane quarter, one 32-column chunk
//               each per half): P^T, dS^T (mask only on partial tiles);
//    warps 10-13 thread = query row: dQ_i drains (bf16 rows for complete chains, else
//               smem -> TMA reduce-add into the fp32 accumulator) and the dK / dV rows.
// Global-RPB score_mod (kBias): the bias joins the P recompute, and dL/dscore is
// accumulated per 2D offset in a shared-memory window (fixed point at the previous tile's
// scale, attn_bwd_common.cuh) flushed once per tile.
#ifdef HLA_BWD_PROF
#define HLA_PROF_ON
#endif
#include "attn_bwd_common.cuh"

namespace hla {
#ifdef HLA_BWD_PROF
__device__ unsigned long long g_bwd_split_prof[1024][24];
#define HLA_PROF_ARRAY g_bwd_split_prof
#endif
namespace bwd {
namespace {

constexpr int kThreads = 512;   // 16 warps: TMA, MMA, 8 x P/dS, 4 x dQ, 2 x TMA
constexpr uint32_t kColS = 0, kColDP = 128, kColDQ = 256, kColDV = 384, kColDK = 448;   // dQ: 2 x 64 columns
constexpr int kHalf = 64;       // q-columns per pipeline half
#ifndef HLA_BWD_VAR
#define HLA_BWD_VAR 0
#endif
constexpr int kVar = HLA_BWD_VAR;   // dev-only decomposition switches, see attn_bwd.cu

// Global RPB at d = 32 (the HWT stack): the compute warps hand each tile's dRPB window to the dQ
// warpgroup (win_full) instead of flushing it behind two 256-thread barriers; the window of tile g
// is reused by tile g + 2 after win_free, which also publishes the fixed-point scale of tile g + 2
// (from the maxima of tile g).  d = 64 keeps the synchronous flush (no shared memory for a second
// window).
template <int D, bool kBias>
constexpr bool async_flush() { return kBias && D == 32; }

template <int D, bool kBias>
struct SplitSmem {
  static constexpr uint32_t kTileBytes = kBlock * D * 2;
  alignas(1024) uint8_t k[2][kTileBytes];
  alignas(1024) uint8_t v[2][kTileBytes];
  alignas(1024) uint8_t q[2][kTileBytes];
  alignas(1024) uint8_t dO[2][kTileBytes];
  alignas(1024) uint8_t ds[2][2 * 128 * 128];   // dS^T bf16 x2 (tile parity): [q/64][kv 128][64 q], SWIZZLE_128B
  alignas(1024) float dq_stage[kBlock * 32];    // fp32 dQ half tile [128][32], SWIZZLE_128B
  alignas(16) float lse[2][kBlock];
  alignas(16) float dd[2][kBlock];
  alignas(16) int32_t qa[2][kBias ? kBlock : 4];   // kBias: A_q of the stage's query columns (RPB table index = A_q - B_k)
  alignas(16) float rpb_wmax[2][8];                // kBias: per compute warp max |dL/dscore| of a tile (tile parity)
  uint64_t kv_full[2], kv_empty[2], q_full[2], q_empty[2], s_full[2], ds_ready[2], dq_full[2], dq_free[2], dkv_full,
      epi_done;
  uint64_t o_full, o_empty;   // kFuse (preprocess folded in), as in attn_bwd.cu
  uint32_t tmem_base;
  // dRPB of a tile's offset box, fixed point: one window flushed by the compute warps after each
  // tile (d = 64), or two (tile parity) flushed asynchronously by the dQ warpgroup (d = 32, kAsyncFlush)
  int32_t rpb_win[async_flush<D, kBias>() ? 2 : 1][kBias ? rpb_win_cap<D>() : 1];
  struct RpbGeo { int32_t dr0, dc0, wrows, wcols, win, head; float fx; } rpb_geo[2];   // (async flush)
  float rpb_scale[2];                                                                // (async flush)
  uint64_t win_full[2], win_free[2];                                                 // (async flush)
  // per dQ warp: row-store transpose (store_rows_t); no room next to the dRPB window
  alignas(1024) uint8_t epi_stage[kBias ? 1 : 4][kBias ? 16 : 2048];   // (also a 64B-swizzled TMA source)
};

// kFuse: the preprocess folded into the kernel (every dQ chain local, no bias) exactly as in the
// full-tile schedule (attn_bwd.cu): warp 0 loads the raw LSE and the O tile into the dq_stage
// bytes, the compute threads form D * scale and LSE * log2(e) (form_d) when they first meet a
// q-block; tmO is the O map.  Non-local dQ chains still reduce into the fp32 accumulator (zeroed
// by dq_zero_kernel), staged in 16-column quarters through the epi_stage (tmDQ: 16-float boxes).
// kDiag: HWA with 64-token windows, N % 128 == 0 (the launcher checks): every tile pairs the two
// windows of its 128 key rows with the same two windows of queries, so key rows 0-63 (TMEM lane
// quarters 0, 1) meet only q-half A, unmasked, and rows 64-127 only q-half B.  The liveness of a
// warp's chunk is then known without the per-half interval reductions, and the dS^T quadrants no
// key row meets are zeroed once at the start (they are never written again).
template <int D, bool kTwoD, bool kGather, bool kBias, bool kFuse, bool kDiag = false>
__global__ void __launch_bounds__(kThreads, 1)
    attn_bwd_split_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                    const __grid_constant__ CUtensorMap tmDQ, const __grid_constant__ CUtensorMap tmO,
                    const BwdParams prm) {
  extern __shared__ uint8_t smem_raw[];
  using Smem = SplitSmem<D, kBias>;
  constexpr bool kAsyncFlush = async_flush<D, kBias>();
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  UnitGeom ug;
  ug.mk = (prm.N + kBlock - 1) / kBlock;   // last kv-block may be ragged
  ug.ppb = (ug.mk + 1) / 2;
  ug.pairs = ug.ppb * prm.heads * prm.batch;
    ug.mkd = prm.mk_div;
    ug.ppbd = prm.ppb_div;
  const int32_t mk = ug.mk;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < 2; ++s) {
      sm100::mbar_init(&sm.kv_full[s], 2);    // producer warps 0 (K), 14 (V)
      sm100::mbar_init(&sm.kv_empty[s], 1);
      sm100::mbar_init(&sm.q_full[s], 3);     // producer warps 0 (LSE, D), 14 (Q), 15 (dO)
      sm100::mbar_init(&sm.q_empty[s], 1);
    }
    for (int hh = 0; hh < 2; ++hh) {
      sm100::mbar_init(&sm.s_full[hh], 1);
      sm100::mbar_init(&sm.ds_ready[hh], 256);
    }
    for (int bb = 0; bb < 2; ++bb) {
      sm100::mbar_init(&sm.dq_full[bb], 1);
      sm100::mbar_init(&sm.dq_free[bb], 128);
    }
    sm100::mbar_init(&sm.dkv_full, 1);
    sm100::mbar_init(&sm.epi_done, 128);
    sm100::mbar_init(&sm.o_full, 1);
    sm100::mbar_init(&sm.o_empty, 1);
    for (int s = 0; s < 2; ++s) {
      sm100::mbar_init(&sm.win_full[s], 256);
      sm100::mbar_init(&sm.win_free[s], 128);
    }
        sm100::fence_mbar_init();
    sm100::tma_prefetch_desc(&tmQ);
    sm100::tma_prefetch_desc(&tmK);
    sm100::tma_prefetch_desc(&tmV);
    sm100::tma_prefetch_desc(&tmDO);
  }
  if (warp == 1) {
    sm100::tmem_alloc(&sm.tmem_base, kTmemCols);
    sm100::tmem_relinquish();
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  unsigned long long tiles_done = 0;

  if (warp == 0 || warp >= 14) {
    HLA_PDECL;
    // ----------------------------------------------------------- TMA producers
    // Three warps run the same schedule and split the loads (a CTA's TMA gather4
    // throughput grows with the number of issuing warps): warp 0 K + LSE / D,
    // warp 14 V + Q, warp 15 dO.  Every warp arrives (with its own byte count) on
    // the barriers it feeds, so no expect_tx has to precede another warp's copy.
    {
      const uint64_t pol_kv = sm100::policy_evict_first();
      const uint64_t pol_q = sm100::policy_evict_last();
      const int role = warp == 0 ? 0 : warp - 13;   // 0, 1, 2
      constexpr uint32_t kTile = Smem::kTileBytes;
      uint32_t n = 0, g = 0, n_o = 0;
      int64_t stage_tag0 = -1, stage_tag1 = -1;   // (b, h, q-block) held by stage 0 / 1
      for (int32_t kq = 0;; ++kq) {
        const int32_t u = unit_at(kq, ug);
        if (u == kUnitEnd) break;
        if (u < 0) continue;
        const int32_t bh_u = prm.mk_div.div(u), kb = u - bh_u * mk;
        const int32_t b = prm.heads_div.div(bh_u), h = bh_u - b * prm.heads;
        const int32_t rs = __ldg(prm.t_row_ptr + kb), nt = __ldg(prm.t_row_ptr + kb + 1) - rs;
        if (nt == 0) continue;
        const int64_t bh = (int64_t)b * prm.heads + h;
        const int kvs = n & 1;
        if (role < 2) {
          if (n >= 2) HLA_PW(13, sm100::mbar_wait(&sm.kv_empty[kvs], ((n >> 1) - 1) & 1));
          if (kVar & 4) {
            if (lane == 0) sm100::mbar_arrive(&sm.kv_full[kvs]);
          } else {
            if (lane == 0) sm100::mbar_arrive_expect_tx(&sm.kv_full[kvs], kTile);
            __syncwarp();
            load_rows<D, kGather>(role == 0 ? sm.k[kvs] : sm.v[kvs], role == 0 ? &tmK : &tmV, &sm.kv_full[kvs], h,
                                  b, prm.N, kb * kBlock, prm.s2c, pol_kv, lane, prm.box8);
          }
        }
        for (int t = 0; t < nt; ++t, ++g) {
          const int s = g & 1;
          if (g >= 2) HLA_PW(14, sm100::mbar_wait(&sm.q_empty[s], ((g >> 1) - 1) & 1));
          const int32_t qblk = __ldg(prm.t_col_idx + rs + t);
          const int64_t tag = bh * prm.N + qblk;     // (b, h, q-block) held by the stage
          if (tag == (s ? stage_tag1 : stage_tag0)) {
            // the stage already holds this q-block (consecutive kv-blocks share
            // q-blocks): no reload, just publish it again
            if (lane == 0) sm100::mbar_arrive(&sm.q_full[s]);
            continue;
          }
          if (s) stage_tag1 = tag; else stage_tag0 = tag;
          if (role == 0) {
            if (kBias) {
              // A_q = (qr + H - 1)(2W - 1) + qc + W - 1 of the q-block's 128 columns (phantom: cell 0),
              // read by the compute warps as warp-uniform 16-B loads next to LSE / D
              const int4 rc = make_int4(rpb_cell_rc(prm.cells, qblk * prm.col_mul + 4 * lane, prm.N, prm.pat.w_div),
                                        rpb_cell_rc(prm.cells, qblk * prm.col_mul + 4 * lane + 1, prm.N, prm.pat.w_div),
                                        rpb_cell_rc(prm.cells, qblk * prm.col_mul + 4 * lane + 2, prm.N, prm.pat.w_div),
                                        rpb_cell_rc(prm.cells, qblk * prm.col_mul + 4 * lane + 3, prm.N, prm.pat.w_div));
              const int32_t a0 = (prm.grid_h - 1) * prm.rpb_w + prm.grid_w - 1;
              auto a_of = [&](int32_t v) { return a0 + (v >> 16) * prm.rpb_w + (v & 0xffff); };
              sm100::sts_u4(sm100::smem_u32(sm.qa[s]) + 16u * lane, a_of(rc.x), a_of(rc.y), a_of(rc.z), a_of(rc.w));
              __syncwarp();   // every lane's A_q is written before lane 0 arrives on q_full
            }
            if (lane == 0 && (kVar & 4)) {
              sm100::mbar_arrive(&sm.q_full[s]);
            } else if (lane == 0) {
              // LSE / D of the real rows only (ragged last tile: N % 4 == 0, so 16-B multiples)
              const uint32_t vbytes = (uint32_t)min(kBlock, prm.N - qblk * prm.col_mul) * 4u;
              sm100::mbar_arrive_expect_tx(&sm.q_full[s], (kFuse ? 1 : 2) * vbytes);
              sm100::bulk_load(sm.lse[s], prm.lse2 + bh * prm.N + qblk * prm.col_mul, vbytes, &sm.q_full[s]);
              if (!kFuse)
                sm100::bulk_load(sm.dd[s], prm.dsum + bh * prm.N + qblk * prm.col_mul, vbytes, &sm.q_full[s]);
            }
            if (kFuse && !(kVar & 4)) {
              // the q-block's O rows into the single O stage (freed by the dQ warps after D)
              if (n_o > 0) sm100::mbar_wait(&sm.o_empty, (n_o - 1) & 1);
              ++n_o;
              if (lane == 0) sm100::mbar_arrive_expect_tx(&sm.o_full, kTile);
              __syncwarp();
              load_rows<D, kGather>(reinterpret_cast<uint8_t*>(sm.dq_stage), &tmO, &sm.o_full, h, b, prm.N,
                                    qblk * prm.col_mul, prm.s2c, pol_q, lane, prm.box8);
            }
          } else if (kVar & 4) {
            if (lane == 0) sm100::mbar_arrive(&sm.q_full[s]);
          } else {
            if (lane == 0) sm100::mbar_arrive_expect_tx(&sm.q_full[s], kTile);
            __syncwarp();
            load_rows<D, kGather>(role == 1 ? sm.q[s] : sm.dO[s], role == 1 ? &tmQ : &tmDO, &sm.q_full[s], h, b,
                                  prm.N, qblk * prm.col_mul, prm.s2c, pol_q, lane, prm.box8);
          }
        }
        ++n;
      }
    }
    HLA_PFLUSH(13, 15, warp == 0 && lane == 0);
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer
    // Half-tile software pipeline over the flattened (unit, q-block) sequence:
    //   S_A,dP_A(g) S_B,dP_B(g) | dV_A dK_A(g) S_A,dP_A(g+1) | dV_B dK_B dQ(g) S_B,dP_B(g+1) | ...
    // so the tensor core works on one q-half while the compute warps process the other.
    HLA_PDECL;
    if (lane == 0) {
      constexpr uint32_t idesc_h = sm100::make_idesc_bf16(kBlock, kHalf, false, false);  // S^T, dP^T halves
      constexpr uint32_t idesc_kv = sm100::make_idesc_bf16(kBlock, D, false, true);      // dV, dK
      constexpr uint32_t idesc_q = sm100::make_idesc_bf16(kBlock, D, true, true);        // dQ
      const uint32_t tDQ = tmem + kColDQ, tDV = tmem + kColDV, tDK = tmem + kColDK;
      TileIter cur;
      cur.init(prm.t_row_ptr, ug);
      uint32_t g = 0;
      uint32_t dq_started0 = 0, dq_started1 = 0;   // chains begun per dQ accumulator
      auto issue_sdp = [&](const TileIter& it, uint32_t gg, int half) {
        const int s = gg & 1;
        const uint8_t* sk = sm.k[it.n & 1];
        const uint8_t* sv = sm.v[it.n & 1];
        const uint32_t qoff = half * kHalf * D * 2;   // first row of this q half
#pragma unroll
        for (int kk = 0; kk < D / 16 && !(kVar & 1); ++kk)
          sm100::mma_ss(tmem + kColS + half * kHalf, kmajor_desc<D>(sk, kk), kmajor_desc<D>(sm.q[s] + qoff, kk),
                        idesc_h, kk > 0);
#pragma unroll
        for (int kk = 0; kk < D / 16 && !(kVar & 1); ++kk)
          sm100::mma_ss(tmem + kColDP + half * kHalf, kmajor_desc<D>(sv, kk), kmajor_desc<D>(sm.dO[s] + qoff, kk),
                        idesc_h, kk > 0);
        sm100::mma_commit(&sm.s_full[half]);
      };
      // kDiag: both halves' S^T / dP^T as one N = 128 product each (the two lane-quarter pairs
      // compute their halves concurrently anyway): half the instructions of the half-tile issue
      constexpr uint32_t idesc_f = sm100::make_idesc_bf16(kBlock, kBlock, false, false);
      auto issue_sdp_full = [&](const TileIter& it, uint32_t gg) {
        const int s = gg & 1;
        const uint8_t* sk = sm.k[it.n & 1];
        const uint8_t* sv = sm.v[it.n & 1];
#pragma unroll
        for (int kk = 0; kk < D / 16 && !(kVar & 1); ++kk)
          sm100::mma_ss(tmem + kColS, kmajor_desc<D>(sk, kk), kmajor_desc<D>(sm.q[s], kk), idesc_f, kk > 0);
#pragma unroll
        for (int kk = 0; kk < D / 16 && !(kVar & 1); ++kk)
          sm100::mma_ss(tmem + kColDP, kmajor_desc<D>(sv, kk), kmajor_desc<D>(sm.dO[s], kk), idesc_f, kk > 0);
        sm100::mma_commit(&sm.s_full[0]);
        sm100::mma_commit(&sm.s_full[1]);
      };
      auto issue_dvdk = [&](uint32_t gg, int half, bool first_tile) {
        const int s = gg & 1;
        const uint8_t* ds = sm.ds[gg & 1];
#pragma unroll
        for (int kk = half * 4; kk < half * 4 + 4 && !(kVar & 1); ++kk) {
          const uint32_t acc = (!first_tile || kk > 0) ? 1u : 0u;
          // P^T of q-columns [16kk, 16kk + 16): 8 packed columns at the start of S^T chunk kk/2
          sm100::mma_ts(tDV, tmem + kColS + (kk >> 1) * 32 + (kk & 1) * 8, mnmajor_desc<D>(sm.dO[s], kk), idesc_kv,
                        acc);
          sm100::mma_ss(tDK, ds_kmajor_desc(ds, kk), mnmajor_desc<D>(sm.q[s], kk), idesc_kv, acc);
        }
      };
      if (cur.valid) {
        sm100::mbar_wait(&sm.kv_full[cur.n & 1], (cur.n >> 1) & 1);
        sm100::mbar_wait(&sm.q_full[0], 0);
        sm100::tc_fence_after();
        if constexpr (kDiag) {
          issue_sdp_full(cur, 0);
        } else {
          issue_sdp(cur, 0, 0);
          issue_sdp(cur, 0, 1);
        }
      }
      HLA_PMARK(tl0);
      while (cur.valid) {
        TileIter nxt = cur;
        nxt.advance(prm.t_row_ptr, ug);
        const uint32_t fdq = dq_plan(prm.t_dq, cur.rs + cur.t, g);
        const int kvs = cur.n & 1;
        const bool last_of_unit = cur.t == cur.nt - 1;
        // half A of tile g
        HLA_PW(0, sm100::mbar_wait(&sm.ds_ready[0], g & 1));
        sm100::tc_fence_after();
        if (cur.t == 0 && cur.n > 0) {
          // the previous unit's dV / dK must have been drained from TMEM
          HLA_PW(1, sm100::mbar_wait(&sm.epi_done, (cur.n - 1) & 1));
          sm100::tc_fence_after();
        }
        issue_dvdk(g, 0, cur.t == 0);
        // S_A / dP_A of the next tile now if its operands already landed (never block
        // here: the B half of this tile must not wait behind the next tile's loads)
        bool next_a_issued = false;
        if (!kDiag && nxt.valid && (nxt.t != 0 || sm100::mbar_test_wait(&sm.kv_full[nxt.n & 1], (nxt.n >> 1) & 1)) &&
            sm100::mbar_test_wait(&sm.q_full[(g + 1) & 1], ((g + 1) >> 1) & 1)) {
          sm100::tc_fence_after();
          issue_sdp(nxt, g + 1, 0);
          next_a_issued = true;
        }
        // half B of tile g, then dQ (needs both halves of dS)
        HLA_PW(0, sm100::mbar_wait(&sm.ds_ready[1], g & 1));
        sm100::tc_fence_after();
        issue_dvdk(g, 1, false);
        sm100::mma_commit(&sm.q_empty[g & 1]);   // Q_g / dO_g no longer read (dQ needs only dS and K)
        if (last_of_unit) sm100::mma_commit(&sm.dkv_full);
        const int dqb = (int)(fdq & HLA_DQ_BUF);
        const bool dq_new = (fdq & HLA_DQ_NEW) != 0;
        if (dq_new) {
          // a new chain: the accumulator's previous chain must have been drained
          const uint32_t c = dqb ? dq_started1++ : dq_started0++;
          if (c > 0) {
            HLA_PW(3, sm100::mbar_wait(&sm.dq_free[dqb], (c - 1) & 1));
            sm100::tc_fence_after();
          }
        }
#pragma unroll
        for (int kk = 0; kk < kBlock / 16 && !(kVar & 1); ++kk)
          sm100::mma_ss(tDQ + dqb * 64, ds_mnmajor_desc(sm.ds[g & 1], kk), mnmajor_desc<D>(sm.k[kvs], kk), idesc_q,
                        (kk > 0 || !dq_new) ? 1u : 0u);
        if (fdq & HLA_DQ_DRAIN) sm100::mma_commit(&sm.dq_full[dqb]);
        if (last_of_unit) sm100::mma_commit(&sm.kv_empty[kvs]);
        if (nxt.valid) {
          if (!next_a_issued) {
            if (nxt.t == 0) HLA_PW(2, sm100::mbar_wait(&sm.kv_full[nxt.n & 1], (nxt.n >> 1) & 1));
            HLA_PW(2, sm100::mbar_wait(&sm.q_full[(g + 1) & 1], ((g + 1) >> 1) & 1));
            sm100::tc_fence_after();
            if (!kDiag) issue_sdp(nxt, g + 1, 0);
          }
          if (kDiag) issue_sdp_full(nxt, g + 1);
          else issue_sdp(nxt, g + 1, 1);
        }
        cur = nxt;
        ++g;
      }
      HLA_PADD(4, tl0);
#ifdef HLA_BWD_PROF
      prof[15] = g;
#endif
      HLA_PFLUSH(0, 5, true);
      HLA_PFLUSH(15, 16, true);
    }
  } else if (warp < 10) {
    HLA_PDECL;
    // --------------------------------------------- P^T / dS^T (thread = key row)
    // two warp sets (cset 0: warps 2-5, cset 1: warps 6-9) share every TMEM lane
    // quarter; within each q-half, cset c processes the 32-column chunk 2*half + c.
    const int quarter = warp & 3;
    const int cset = (warp - 2) >> 2;
    const int row = quarter * 32 + lane;
    const int cth = (warp - 2) * 32 + lane;   // compute thread 0 .. 255
    uint32_t n_od = 0;                          // kFuse: O tiles consumed
    int64_t dtag0 = -1, dtag1 = -1;             // kFuse: q-block held by stage 0 / 1
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const float sl2 = prm.scale_log2, scale = prm.scale;
    if (kBias) {   // the dRPB window starts (and is left after every flush) zeroed
      for (int i = (warp - 2) * 32 + lane; i < (kAsyncFlush ? 2 : 1) * rpb_win_cap<D>(); i += 256)
        (&sm.rpb_win[0][0])[i] = 0;
      sm100::named_bar_sync(3, 256);
    }
    if constexpr (kDiag) {   // both dS^T tiles start zeroed (the dead quadrants stay so)
      const uint32_t ds0 = sm100::smem_u32(sm.ds[0]);
      for (uint32_t i = (uint32_t)cth * 16u; i < 2u * sizeof(sm.ds[0]); i += 256u * 16u)
        sm100::sts_u4(ds0 + i, 0u, 0u, 0u, 0u);
      sm100::fence_proxy_async_smem();
      sm100::named_bar_sync(3, 256);
    }
    float rpb_fx = 0.f;   // fixed-point scale of the dRPB window, from the previous tile's maximum (0: none yet)
    uint32_t n = 0, g = 0;
    for (int32_t kq = 0;; ++kq) {
      const int32_t u = unit_at(kq, ug);
      if (u == kUnitEnd) break;
      if (u < 0) continue;
      const int32_t bh_u = prm.mk_div.div(u), kb = u - bh_u * mk;
      const int32_t b = prm.heads_div.div(bh_u), h = bh_u - b * prm.heads;
      const int32_t rs = __ldg(prm.t_row_ptr + kb), nt = __ldg(prm.t_row_ptr + kb + 1) - rs;
      const int32_t kidx = kb * kBlock + row;
      RowBox box = clip_box<kTwoD>(prm.pat, col_box(prm.pat, kidx));
      if (kidx >= prm.N) box.len = 0;   // phantom key row of a ragged tile: nothing allowed
      // RPB: this key row's cell, the key block's cell box, the head's table / gradient
      int32_t k_r = 0, k_c = 0, k_b = 0;
      CellBox kbox{0, 0, 0, 0};
      const float* rpbh = nullptr;
      float* drpbh = nullptr;
      if (kBias) {
        const int32_t rc = rpb_cell_rc(prm.cells, kidx, prm.N, prm.pat.w_div);
        k_r = rc >> 16;
        k_c = rc & 0xffff;
        k_b = k_r * prm.rpb_w + k_c;
        kbox = rpb_block_box(prm.cells, kb * kBlock, prm.N, prm.pat.w_div, lane);
        rpbh = prm.rpb + (int64_t)h * prm.rpb_hw;
        drpbh = prm.drpb + (int64_t)h * prm.rpb_hw;
      }
      for (int t = 0; t < nt; ++t, ++g) {
        const int s = g & 1;
        const uint8_t kd = __ldg(prm.t_kind + rs + t);
        const int32_t q0 = __ldg(prm.t_col_idx + rs + t) * prm.col_mul;
        // RPB: the tile's offset box (dr, dc) = q box - key box and whether its rows fit
        // the shared-memory dRPB window (query offsets A_q come staged with LSE / D)
        int32_t dr0 = 0, dc0 = 0, wc = 0, wrows = 0, wcols = 0, kwb = 0;
        bool win = false;
        if (kBias) {
          const CellBox qbox = rpb_block_box(prm.cells, q0, prm.N, prm.pat.w_div, lane);
          dr0 = qbox.r0 - kbox.r1;
          dc0 = qbox.c0 - kbox.c1;
          // window = the box's offset rows at the table's own row stride, so that the element
          // index (dr - dr0) * wc + (dc - dc0) = A_q - kwb (A_q staged per q-block)
          wc = prm.rpb_w;
          wrows = qbox.r1 - kbox.r0 - dr0 + 1;
          wcols = qbox.c1 - kbox.c0 - dc0 + 1;   // offset columns actually used (<= wc)
          win = wrows * wc <= rpb_win_cap<D>();
          kwb = (prm.grid_h - 1) * prm.rpb_w + prm.grid_w - 1 + k_b + dr0 * wc + dc0;
        }
        HLA_PW(5, sm100::mbar_wait(&sm.q_full[s], (g >> 1) & 1));
        HLA_PMARK(tc0);
        if (kAsyncFlush) {   // window g & 1 flushed (tile g - 2) and this tile's scale published
          if (g >= 2) {
            sm100::mbar_wait(&sm.win_free[g & 1], ((g >> 1) - 1) & 1);
            rpb_fx = sm.rpb_scale[g & 1];
          } else {
            rpb_fx = 0.f;   // (no scale yet: a CTA's first two tiles take the global path)
          }
        }
        if (kFuse) {   // a newly loaded q-block (the producer's stage tags, mirrored): form D and the
                       // log2-domain LSE in its stage from the O tile (form_d), then free the O tile
          const int64_t tag = ((int64_t)b * prm.heads + h) * prm.N + q0;
          if (tag != (s ? dtag1 : dtag0)) {
            if (s) dtag1 = tag; else dtag0 = tag;
            sm100::mbar_wait(&sm.o_full, n_od & 1);
            ++n_od;
            form_d<D>(sm100::smem_u32(sm.dq_stage), sm100::smem_u32(sm.dO[s]), sm.dd[s], sm.lse[s], cth, prm.N - q0,
                      prm.scale);
            sm100::fence_proxy_async_smem();   // O-stage reads before the next TMA write into it
            sm100::named_bar_sync(kBarFormD, 256);
            if (cth == 0) sm100::mbar_arrive(&sm.o_empty);
          }
        }
        const uint32_t lse2 = sm100::smem_u32(sm.lse[s]);
        const uint32_t dd = sm100::smem_u32(sm.dd[s]);
        const uint32_t qa = sm100::smem_u32(sm.qa[s]);
        const uint32_t dsbuf = sm100::smem_u32(sm.ds[g & 1]);
        float tmax = 0.f;   // kBias: largest |dL/dscore| of the tile (this thread)
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
          HLA_PW(6, sm100::mbar_wait(&sm.s_full[half], g & 1));
          sm100::tc_fence_after();
          const int c = 2 * half + cset;
          // [ulo, uhi): 8-column groups of this chunk that hold an allowed query of some key row
          // of this warp (partial tiles of 1D patterns: each key row's queries are one interval);
          // the other groups are all masked, their exponentials skipped (warp-uniform) and P = 0
          // there.  elem: some row of the warp has a masked query in the chunk (else no element
          // mask).  Full tiles / 2D patterns: all 4 groups, element mask on partial tiles.
          int ulo = 0, uhi = 4;
          bool elem = kd == 2;
          if constexpr (kDiag) {
            const bool live = (quarter >> 1) == half;
            ulo = live ? 0 : 4;
            uhi = live ? 4 : 0;
            elem = false;
          } else if (kd == 2 && !kTwoD) {
            const int32_t base = q0 + c * 32;
            const int32_t lo = min(max(box.lo - base, 0), 32), hi = min(max(box.lo + box.len - base, 0), 32);
            const bool any = hi > lo;
            ulo = __reduce_min_sync(0xffffffffu, any ? lo : 32) >> 3;
            uhi = (__reduce_max_sync(0xffffffffu, any ? hi : 0) + 7) >> 3;
            elem = !__all_sync(0xffffffffu, lo == 0 && hi == 32);
            // kBias: only the whole-chunk skip (the group-skipping loop around the RPB gather
            // measured slower: cfg5-hwt +6%)
            if (kBias && ulo < uhi) { ulo = 0; uhi = 4; }
          }
          if (!(kVar & 2) && ulo >= uhi) {
            // no key row of this warp meets a query of this chunk (e.g. the other window of an
            // HWA-64 tile): no TMEM loads or math -- P^T and dS^T are zero there
            uint32_t z[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) z[e] = 0u;
            sm100::tmem_st16(tmem + lane_off + kColS + c * 32, z);
#pragma unroll
            for (int u4 = 0; u4 < 4 && !kDiag; ++u4) {
              const int qc = c * 32 + u4 * 8;
              const uint32_t off =
                  (uint32_t)(qc >> 6) * 16384u + sm100::swz128((uint32_t)row * 128u + (uint32_t)(qc & 63) * 2u);
              sm100::sts_u4(dsbuf + off, 0u, 0u, 0u, 0u);
            }
          } else if (!(kVar & 2)) {
            uint32_t sr[32], dpr[32];
            sm100::tmem_ld32(tmem + lane_off + kColS + c * 32, sr);
            sm100::tmem_ld32(tmem + lane_off + kColDP + c * 32, dpr);
            sm100::tmem_wait_ld();
            // P first (so its TMEM store is in flight while dS is formed)
            float p[32];
#pragma unroll
            for (int u4 = 0; u4 < 4; ++u4) {
              if (u4 < ulo || u4 >= uhi) {
#pragma unroll
                for (int e = 0; e < 8; ++e) p[u4 * 8 + e] = 0.f;
                continue;
              }
              const int qc = c * 32 + u4 * 8;
              const float4 la = sm100::lds_f4(lse2 + qc * 4), lb = sm100::lds_f4(lse2 + qc * 4 + 16);
              const float lv[8] = {la.x, la.y, la.z, la.w, lb.x, lb.y, lb.z, lb.w};
              int32_t av[8] = {0, 0, 0, 0, 0, 0, 0, 0};
              if (kBias) {
                const float4 xa = sm100::lds_f4(qa + qc * 4), xb = sm100::lds_f4(qa + qc * 4 + 16);
                av[0] = __float_as_int(xa.x); av[1] = __float_as_int(xa.y); av[2] = __float_as_int(xa.z);
                av[3] = __float_as_int(xa.w); av[4] = __float_as_int(xb.x); av[5] = __float_as_int(xb.y);
                av[6] = __float_as_int(xb.z); av[7] = __float_as_int(xb.w);
              }
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                float x = fmaf(__uint_as_float(sr[u4 * 8 + e]), sl2, -lv[e]);
                if (kBias)   // + bias * log2(e), bias = table[h][dr + H - 1][dc + W - 1] = table[A_q - B_k]
                  x = fmaf(__ldg(rpbh + (av[e] - k_b)), 1.4426950408889634f, x);
                p[u4 * 8 + e] = sm100::ex2(x);
              }
            }
            uint32_t okbits = 0xffffffffu;   // element mask of this chunk (partial tiles only)
            if (elem) {
#pragma unroll
              for (int e = 0; e < 32; ++e) {
                const int32_t qq = q0 + c * 32 + e;
                bool ok;
                if (!kTwoD) {
                  ok = (uint32_t)(qq - box.lo) < (uint32_t)box.len;
                } else {
                  const int32_t rq = prm.pat.log2W >= 0 ? (qq >> prm.pat.log2W) : prm.pat.w_div.div(qq);
                  const int32_t cq = qq - rq * prm.pat.W;
                  ok = ((uint32_t)(rq - box.lo) < (uint32_t)box.len) && ((uint32_t)(cq - box.c0) < (uint32_t)box.cn);
                }
                if (!ok) {
                  p[e] = 0.f;
                  okbits &= ~(1u << e);
                }
              }
            }
            {
              uint32_t pk[16];
#pragma unroll
              for (int e = 0; e < 16; ++e) pk[e] = sm100::pack_bf16(p[2 * e], p[2 * e + 1]);
              // over the first 16 columns of this thread's own S^T chunk (already in registers)
              sm100::tmem_st16(tmem + lane_off + kColS + c * 32, pk);
            }
#pragma unroll
            for (int u4 = 0; u4 < 4; ++u4) {   // dS, 8 query columns (one 16B chunk) at a time
              const int qc = c * 32 + u4 * 8;
              const float4 da = sm100::lds_f4(dd + qc * 4), db = sm100::lds_f4(dd + qc * 4 + 16);
              const float dv[8] = {da.x, da.y, da.z, da.w, db.x, db.y, db.z, db.w};
              float ds[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                ds[e] = p[u4 * 8 + e] * fmaf(__uint_as_float(dpr[u4 * 8 + e]), scale, -dv[e]);
                // masked: exactly 0 (the D / LSE of phantom query columns may be stale, 0 * NaN = NaN)
                if (!((okbits >> (u4 * 8 + e)) & 1u)) ds[e] = 0.f;
              }
              if (kBias) {
                // dRPB[offset] += dL/dscore = dS / scale: into the tile's shared-memory
                // offset window (flushed once per tile), else straight to global
                const float4 xa = sm100::lds_f4(qa + qc * 4), xb = sm100::lds_f4(qa + qc * 4 + 16);
                const int32_t av[8] = {__float_as_int(xa.x), __float_as_int(xa.y), __float_as_int(xa.z),
                                       __float_as_int(xa.w), __float_as_int(xb.x), __float_as_int(xb.y),
                                       __float_as_int(xb.z), __float_as_int(xb.w)};
                const uint32_t wbase = sm100::smem_u32(sm.rpb_win[kAsyncFlush ? (g & 1) : 0]);
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                  if (!((okbits >> (u4 * 8 + e)) & 1u)) continue;
                  const float gv = ds[e] * prm.inv_scale;
                  tmax = fmaxf(tmax, fabsf(gv));
                  const float sv = gv * rpb_fx;
                  // window index (dr - dr0) * (2W - 1) + (dc - dc0) = A_q - kwb; a CTA's first tile
                  // (no scale yet: rpb_fx == 0) and out-of-range addends take the global path
                  if (win && rpb_fx > 0.f && fabsf(sv) < kRpbFixMax) {
                    asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(wbase + 4u * (uint32_t)(av[e] - kwb)),
                                 "r"(__float2int_rn(sv))
                                 : "memory");
                  } else {     // table index A_q - B_k (no window, or outside the fixed-point range)
                    atomicAdd(drpbh + (av[e] - k_b), gv);
                  }
                }
              }
              // dS^T row -> smem [q/64][kv][64] with the 128B swizzle (16B chunks)
              const uint32_t off =
                  (uint32_t)(qc >> 6) * 16384u + sm100::swz128((uint32_t)row * 128u + (uint32_t)(qc & 63) * 2u);
              sm100::sts_u4(dsbuf + off, sm100::pack_bf16(ds[0], ds[1]), sm100::pack_bf16(ds[2], ds[3]),
                            sm100::pack_bf16(ds[4], ds[5]), sm100::pack_bf16(ds[6], ds[7]));
            }
          }
          sm100::tmem_wait_st();
          sm100::fence_proxy_async_smem();
          sm100::tc_fence_before();
          sm100::mbar_arrive(&sm.ds_ready[half]);
        }
        HLA_PMARK(tf0);
        if (kAsyncFlush) {
          // hand the window to the dQ warpgroup: this warp's maximum, the tile's geometry, arrive
          const uint32_t wm = __reduce_max_sync(0xffffffffu, __float_as_uint(tmax));   // non-negative floats
          if (lane == 0) sm.rpb_wmax[g & 1][warp - 2] = __uint_as_float(wm);
          if (cth == 0) sm.rpb_geo[g & 1] = {dr0, dc0, wrows, wcols, win ? 1 : 0, h, rpb_fx};
          sm100::mbar_arrive(&sm.win_full[g & 1]);
        } else if (kBias && win) {
          // flush the tile's dRPB window to global (and re-zero it) -- all 256 compute threads;
          // the tile's largest |dL/dscore| sets the fixed-point scale of the NEXT tile (no
          // extra barrier; elements beyond that scale's range go to global fp32 atomics)
          const uint32_t wm = __reduce_max_sync(0xffffffffu, __float_as_uint(tmax));   // non-negative floats
          if (lane == 0) sm.rpb_wmax[g & 1][warp - 2] = __uint_as_float(wm);
          sm100::named_bar_sync(3, 256);
          const float inv_fx = rpb_fx > 0.f ? 1.f / rpb_fx : 0.f;   // (nothing accumulated without a scale)
          const int tid = (warp - 2) * 32 + lane;
          // only the box's used columns: entries i = tid, tid + 256, ... as (ir, ic), stepped
          // without a division per entry
          const int32_t wcs = wcols > 0 ? wcols : 1;
          const int32_t step_r = 256 / wcs, step_c = 256 - step_r * wcs;
          int32_t ir = wcols > 0 ? tid / wcs : wrows, ic = tid - (tid / wcs) * wcs;
          for (; ir < wrows; ir += step_r, ic += step_c) {
            if (ic >= wcols) { ic -= wcols; ++ir; if (ir >= wrows) break; }
            const int32_t v = sm.rpb_win[0][ir * wc + ic];
            if (v != 0) {
              atomicAdd(drpbh + (dr0 + ir + prm.grid_h - 1) * prm.rpb_w + (dc0 + ic + prm.grid_w - 1),
                        (float)v * inv_fx);
              sm.rpb_win[0][ir * wc + ic] = 0;
            }
          }
          rpb_fx = rpb_next_scale(sm.rpb_wmax[g & 1], rpb_fx);   // (stays 0 only for an all-zero tile)
          sm100::named_bar_sync(3, 256);
        }
        HLA_PADD(8, tf0);
        HLA_PADD(7, tc0);
      }
      tiles_done += nt;
    }
    HLA_PFLUSH(5, 9, warp == 2 && lane == 0);
  } else if (warp < 14) {
    HLA_PDECL;
    // ------------------------------------------ dQ partial -> fp32 accumulator
    // thread = query row: drain the dQ_i tile from TMEM (then release it), stage it
    // in shared memory (two 32-column halves, 128B swizzle) and let the TMA engine
    // add it into the fp32 accumulator (cp.reduce.async.bulk.tensor ... add) -- no
    // per-thread atomics, so the LSU stays free for the compute warps.
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const bool leader = warp == 10 && lane == 0;
    uint32_t g = 0, n = 0;
    uint32_t dq_drained0 = 0, dq_drained1 = 0;   // chains drained per dQ accumulator
    for (int32_t kq = 0;; ++kq) {
      const int32_t u = unit_at(kq, ug);
      if (u == kUnitEnd) break;
      if (u < 0) continue;
      const int32_t bh_u = prm.mk_div.div(u), kb = u - bh_u * mk;
      const int32_t b = prm.heads_div.div(bh_u), h = bh_u - b * prm.heads;
      const int32_t rs = __ldg(prm.t_row_ptr + kb), nt = __ldg(prm.t_row_ptr + kb + 1) - rs;
      for (int t = 0; t < nt; ++t, ++g) {
        if (kAsyncFlush) {
          // tile g's dRPB window: flush its box to the table (and re-zero it), publish the scale
          // of tile g + 2 from the tile's per-warp maxima, free the window
          sm100::mbar_wait(&sm.win_full[g & 1], (g >> 1) & 1);
          const auto geo = sm.rpb_geo[g & 1];
          if (geo.win && geo.fx > 0.f) {
            const float inv_fx = 1.f / geo.fx;
            float* drp = prm.drpb + (int64_t)geo.head * prm.rpb_hw;
            int32_t* w = sm.rpb_win[g & 1];
            const int tid = row;   // 0 .. 127
            const int32_t wcs = geo.wcols > 0 ? geo.wcols : 1;
            const int32_t step_r = 128 / wcs, step_c = 128 - step_r * wcs;
            int32_t ir = geo.wcols > 0 ? tid / wcs : geo.wrows, ic = tid - (tid / wcs) * wcs;
            for (; ir < geo.wrows; ir += step_r, ic += step_c) {
              if (ic >= geo.wcols) { ic -= geo.wcols; ++ir; if (ir >= geo.wrows) break; }
              const int32_t v = w[ir * prm.rpb_w + ic];
              if (v != 0) {
                atomicAdd(drp + (geo.dr0 + ir + prm.grid_h - 1) * prm.rpb_w + (geo.dc0 + ic + prm.grid_w - 1),
                          (float)v * inv_fx);
                w[ir * prm.rpb_w + ic] = 0;
              }
            }
          }
          if (row == 0) sm.rpb_scale[g & 1] = rpb_next_scale(sm.rpb_wmax[g & 1], geo.fx);
          sm100::mbar_arrive(&sm.win_free[g & 1]);
        }
        const uint32_t fdq = dq_plan(prm.t_dq, rs + t, g);
        if (!(fdq & HLA_DQ_DRAIN)) continue;   // the chain continues in TMEM
        const int dqb = (int)(fdq & HLA_DQ_BUF);
        HLA_PW(9, sm100::mbar_wait(&sm.dq_full[dqb], (dqb ? dq_drained1++ : dq_drained0++) & 1));
        HLA_PMARK(td0);
        sm100::tc_fence_after();
        if (kVar & 8) {
          sm100::mbar_arrive(&sm.dq_free[dqb]);
          continue;
        }
        const int32_t qblk = __ldg(prm.t_col_idx + rs + t);
        const int32_t qrow = b * prm.N + qblk * prm.col_mul;   // sequence order
        uint32_t r[D];
#pragma unroll
        for (int c = 0; c < D / 32; ++c)
          sm100::tmem_ld32(tmem + lane_off + kColDQ + dqb * 64 + c * 32, *reinterpret_cast<uint32_t(*)[32]>(r + c * 32));
        sm100::tmem_wait_ld();
        sm100::tc_fence_before();
        sm100::mbar_arrive(&sm.dq_free[dqb]);     // the TMEM dQ accumulator may now be overwritten
        if (fdq & HLA_DQ_LOCAL) {
          // complete dQ_i (dS carries the softmax scale): bf16 rows straight to dq, to the
          // grid cell under the fused reorder; phantom rows of a ragged tile write nothing
          const int32_t qs = qblk * prm.col_mul + row;
          if (!kBias) {
            uint4* dqp = nullptr;
            if (qs < prm.N) {
              const int32_t qcell = kGather ? __ldg(prm.s2c + qs) : qs;
              dqp = reinterpret_cast<uint4*>(prm.dq + (((int64_t)b * prm.N + qcell) * prm.heads + h) * D);
            }
            uint32_t w[D / 2];
#pragma unroll
            for (int e = 0; e < D / 2; ++e) w[e] = sm100::pack_bf16(__uint_as_float(r[2 * e]), __uint_as_float(r[2 * e + 1]));
            if (kFuse) {   // (the stage also carries the reduce-adds: the last one must have read it)
              if (leader) sm100::bulk_wait_group_read0();
              sm100::named_bar_sync(2, 128);
            }
            store_rows_t<D>(w, dqp, sm100::smem_u32(sm.epi_stage[kBias ? 0 : quarter]), lane);
          } else if (qs < prm.N) {
            const int32_t qcell = kGather ? __ldg(prm.s2c + qs) : qs;
            uint4* dqp = reinterpret_cast<uint4*>(prm.dq + (((int64_t)b * prm.N + qcell) * prm.heads + h) * D);
#pragma unroll
            for (int v4 = 0; v4 < D / 8; ++v4)
              dqp[v4] = make_uint4(sm100::pack_bf16(__uint_as_float(r[8 * v4 + 0]), __uint_as_float(r[8 * v4 + 1])),
                                   sm100::pack_bf16(__uint_as_float(r[8 * v4 + 2]), __uint_as_float(r[8 * v4 + 3])),
                                   sm100::pack_bf16(__uint_as_float(r[8 * v4 + 4]), __uint_as_float(r[8 * v4 + 5])),
                                   sm100::pack_bf16(__uint_as_float(r[8 * v4 + 6]), __uint_as_float(r[8 * v4 + 7])));
          }
          continue;
        }
        if constexpr (kFuse && !kBias) {
          // the dq_stage holds O tiles: 16-column quarters through the 8 KB epi_stage instead
          // (64-B rows, 64B swizzle; tmDQ has 16-float boxes in this mode)
#pragma unroll
          for (int hh = 0; hh < D / 16; ++hh) {
            if (leader) sm100::bulk_wait_group_read0();   // previous reduce finished reading the stage
            sm100::named_bar_sync(2, 128);
            const uint32_t st = sm100::smem_u32(sm.epi_stage[0]);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint32_t off = sm100::swz64((uint32_t)row * 64u + (uint32_t)j * 16u);
              sm100::sts_u4(st + off, r[hh * 16 + 4 * j], r[hh * 16 + 4 * j + 1], r[hh * 16 + 4 * j + 2],
                            r[hh * 16 + 4 * j + 3]);
            }
            sm100::fence_proxy_async_smem();
            sm100::named_bar_sync(2, 128);
            if (leader) {
              sm100::tma_reduce_add_3d(&tmDQ, sm.epi_stage[0], hh * 16, h, qrow);
              sm100::bulk_commit_group();
            }
          }
        } else {
#pragma unroll
          for (int hh = 0; hh < D / 32; ++hh) {
            if (leader) sm100::bulk_wait_group_read0();   // previous reduce finished reading the stage
            sm100::named_bar_sync(2, 128);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const uint32_t off = sm100::swz128((uint32_t)row * 128u + (uint32_t)j * 16u);
              sm100::sts_u4(sm100::smem_u32(sm.dq_stage) + off, r[hh * 32 + 4 * j], r[hh * 32 + 4 * j + 1],
                            r[hh * 32 + 4 * j + 2], r[hh * 32 + 4 * j + 3]);
            }
            sm100::fence_proxy_async_smem();
            sm100::named_bar_sync(2, 128);
            if (leader) {
              sm100::tma_reduce_add_3d(&tmDQ, sm.dq_stage, hh * 32, h, qrow);
              sm100::bulk_commit_group();
            }
          }
        }
      }
      // final dK, dV rows of this unit -> bf16 (thread = key row; dS already carries
      // the softmax scale).  Done here, off the compute warps' critical path; the
      // next unit's first dV/dK MMA waits for epi_done.
      const int32_t kidx = kb * kBlock + row;
      const bool real = kidx < prm.N;   // phantom key rows of a ragged tile write nothing
      const int32_t kcell = kGather ? (real ? __ldg(prm.s2c + kidx) : 0) : kidx;   // fused inverse reorder of dK, dV
      const int64_t grow = ((int64_t)b * prm.N + kcell) * prm.heads + h;
      uint4* dkp = reinterpret_cast<uint4*>(prm.dk + grow * D);
      uint4* dvp = reinterpret_cast<uint4*>(prm.dv + grow * D);
      if (nt > 0) {
        HLA_PW(11, sm100::mbar_wait(&sm.dkv_full, n & 1));
        HLA_PMARK(te0);
        sm100::tc_fence_after();
        if (kVar & 8) {
          sm100::mbar_arrive(&sm.epi_done);
          ++n;
          continue;
        }
        // dV then dK, each packed to bf16 right away (64 live registers, not 128)
        uint32_t pv[D / 2], pk[D / 2];
#pragma unroll
        for (int which = 0; which < 2; ++which) {
          uint32_t r[D];
#pragma unroll
          for (int c = 0; c < D / 32; ++c)
            sm100::tmem_ld32(tmem + lane_off + (which ? kColDK : kColDV) + c * 32,
                             *reinterpret_cast<uint32_t(*)[32]>(r + c * 32));
          sm100::tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < D / 2; ++e) {
            const uint32_t w = sm100::pack_bf16(__uint_as_float(r[2 * e]), __uint_as_float(r[2 * e + 1]));
            if (which) pk[e] = w; else pv[e] = w;
          }
        }
        sm100::tc_fence_before();
        sm100::mbar_arrive(&sm.epi_done);      // dV / dK accumulators may now be reset
        if (!kBias) {
          if (kFuse) {   // (the stage also carries the reduce-adds)
            if (leader) sm100::bulk_wait_group_read0();
            sm100::named_bar_sync(2, 128);
          }
          const uint32_t stg = sm100::smem_u32(sm.epi_stage[kBias ? 0 : quarter]);
          store_rows_t<D>(pv, real ? dvp : nullptr, stg, lane);
          store_rows_t<D>(pk, real ? dkp : nullptr, stg, lane);
        } else {
#pragma unroll
          for (int v4 = 0; v4 < D / 8 && real; ++v4) {
            dvp[v4] = make_uint4(pv[v4 * 4 + 0], pv[v4 * 4 + 1], pv[v4 * 4 + 2], pv[v4 * 4 + 3]);
            dkp[v4] = make_uint4(pk[v4 * 4 + 0], pk[v4 * 4 + 1], pk[v4 * 4 + 2], pk[v4 * 4 + 3]);
          }
        }
        HLA_PADD(12, te0);
        ++n;
      } else {
#pragma unroll
        for (int c = 0; c < D / 8 && real; ++c) {
          dvp[c] = make_uint4(0, 0, 0, 0);
          dkp[c] = make_uint4(0, 0, 0, 0);
        }
      }
    }
    if (leader) sm100::bulk_wait_group0();
    HLA_PFLUSH(9, 13, leader);
  }

  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (warp == 1) sm100::tmem_dealloc(tmem, kTmemCols);
  if (warp == 2 && lane == 0 && prm.visited != nullptr && tiles_done > 0) atomicAdd(prm.visited, tiles_done);
}


template <int D, bool kTwoD, bool kGather, bool kBias, bool kFuse = false, bool kDiag = false>
hla_status launch_split_t(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                          const CUtensorMap& mdo, const CUtensorMap& mdq, const BwdParams& prm, int32_t n_kblocks,
                          cudaStream_t stream, const CUtensorMap* mo = nullptr) {
  const size_t smem = sizeof(SplitSmem<D, kBias>) + 1024;
  auto* fn = attn_bwd_split_kernel<D, kTwoD, kGather, kBias, kFuse, kDiag>;
  HLA_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t pairs = (int64_t)((n_kblocks + 1) / 2) * prm.heads * prm.batch;   // work units (kv-block pairs)
  const int grid = (int)std::min<int64_t>(pairs, (int64_t)num_sms());
  fn<<<grid, kThreads, smem, stream>>>(mq, mk, mv, mdo, mdq, mo ? *mo : mdq, prm);
  HLA_CUDA_TRY(cudaGetLastError());
  return HLA_OK;
}

static_assert(sizeof(SplitSmem<64, true>) + 1024 <= 227 * 1024, "split bwd shared memory exceeds 227 KB");

template <bool kBias>
hla_status dispatch_split(int head_dim, bool gather, bool two_d, const CUtensorMap& mq, const CUtensorMap& mk,
                          const CUtensorMap& mv, const CUtensorMap& mdo, const CUtensorMap& mdq, const BwdParams& prm,
                          int32_t n_kblocks, cudaStream_t stream) {
  if (head_dim == 64) {
    if (gather) return launch_split_t<64, false, true, kBias>(mq, mk, mv, mdo, mdq, prm, n_kblocks, stream);
    return two_d ? launch_split_t<64, true, false, kBias>(mq, mk, mv, mdo, mdq, prm, n_kblocks, stream)
                 : launch_split_t<64, false, false, kBias>(mq, mk, mv, mdo, mdq, prm, n_kblocks, stream);
  }
  if (gather) return launch_split_t<32, false, true, kBias>(mq, mk, mv, mdo, mdq, prm, n_kblocks, stream);
  return two_d ? launch_split_t<32, true, false, kBias>(mq, mk, mv, mdo, mdq, prm, n_kblocks, stream)
               : launch_split_t<32, false, false, kBias>(mq, mk, mv, mdo, mdq, prm, n_kblocks, stream);
}

// HWA with 64-token windows and no ragged tile: the kDiag instantiation applies
inline bool diag64(const BwdParams& prm) { return prm.pat.kind == K_HWA && prm.pat.n == 64 && prm.N % 128 == 0; }

// preprocess folded in (no bias): every dQ chain local, mdq = the O map, lse2 = raw LSE
hla_status dispatch_split_fused(int head_dim, bool gather, bool two_d, const CUtensorMap& mq, const CUtensorMap& mk,
                                const CUtensorMap& mv, const CUtensorMap& mdo, const CUtensorMap& mdq,
                                const CUtensorMap& mo, const BwdParams& prm, int32_t n_kblocks, cudaStream_t stream) {
  if (head_dim == 64) {
    if (gather) return launch_split_t<64, false, true, false, true>(mq, mk, mv, mdo, mdq, prm, n_kblocks, stream, &mo);
    return two_d ? launch_split_t<64, true, false, false, true>(mq, mk, mv, mdo, mdq, prm, n_kblocks, stream, &mo)
                 : launch_split_t<64, false, false, false, true>(mq, mk, mv, mdo, mdq, prm, n_kblocks, stream, &mo);
  }
  if (gather && diag64(prm))
    return launch_split_t<32, false, true, false, true, true>(mq, mk, mv, mdo, mdq, prm, n_kblocks, stream, &mo);
  if (gather) return launch_split_t<32, false, true, false, true>(mq, mk, mv, mdo, mdq, prm, n_kblocks, stream, &mo);
  return two_d ? launch_split_t<32, true, false, false, true>(mq, mk, mv, mdo, mdq, prm, n_kblocks, stream, &mo)
               : launch_split_t<32, false, false, false, true>(mq, mk, mv, mdo, mdq, prm, n_kblocks, stream, &mo);
}

}  // namespace

hla_status launch_split(bool bias, int head_dim, bool gather, bool two_d, bool fuse, const CUtensorMap& mq,
                        const CUtensorMap& mk, const CUtensorMap& mv, const CUtensorMap& mdo, const CUtensorMap& mdq,
                        const CUtensorMap& mo, const BwdParams& prm, int32_t n_kblocks, cudaStream_t stream) {
  if (fuse && !bias)
    return dispatch_split_fused(head_dim, gather, two_d, mq, mk, mv, mdo, mdq, mo, prm, n_kblocks, stream);
  return bias ? dispatch_split<true>(head_dim, gather, two_d, mq, mk, mv, mdo, mdq, prm, n_kblocks, stream)
              : dispatch_split<false>(head_dim, gather, two_d, mq, mk, mv, mdo, mdq, prm, n_kblocks, stream);
}

}  // namespace bwd
}  // namespace hla

#ifdef HLA_BWD_PROF
// dev-only: per-CTA wait / work cycle sums of the last attn_bwd_split_kernel launch (HLA_BWD_PROF builds)
extern "C" __attribute__((visibility("default"))) int hla_debug_bwd_split_prof(unsigned long long* host, int ctas) {
  cudaDeviceSynchronize();
  const int n = ctas < 1024 ? ctas : 1024;
  cudaMemcpyFromSymbol(host, hla::g_bwd_split_prof, (size_t)n * 24 * sizeof(unsigned long long));
  return n;
}
#endif
