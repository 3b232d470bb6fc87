// K7-K9: block-sparse attention backward on sm_100a (tcgen05 + TMEM + TMA).
//
// Gradients of masked softmax attention (the paper times this pass in the
// "Backward" columns; skipping empty tiles is what makes it
// cheaper):
//   P = exp(scale S - LSE) (0 where masked),  D = rowsum(dO o O)
//   dV = P^T dO,  dS = scale P o (dO V^T - D),  dK = dS^T Q,  dQ = dS K.
//
// K7 bwd_preprocess : D = rowsum(dO o O) (fp32) and zero the fp32 dQ accumulator -- or folded
//    into K8 by hla_attn_bwd (kFuse: the compute warps form D and the log2 LSE from an O tile,
//    form_d; non-local accumulator rows are then zeroed by the write-only dq_zero_kernel).
// K8 attn_bwd_full_kernel (this file; attn_bwd_split.cu holds the half-tile schedule):
//    persistent, 1 CTA / SM, kv-major over the transposed CSR
//    (work unit = a pair of consecutive kv-blocks of one (b, h); per kv-block the
//    listed q-blocks i, ascending).  kThreads = 4 + kCmpWarps + 4 warps, registers
//    redistributed with setmaxnreg (kRegsCtl / kRegsCmp / kRegsDq):
//    warpgroup 0  warp 0 TMA K_j (+ LSE_i, D_i bulk copies), warp 2 TMA V_j, Q_i,
//                 warp 3 TMA dO_i (Q / dO in a 2-stage ring, K / V 2 stages);
//                 warp 1 TMEM allocator + single-thread tcgen05.mma issuer:
//                   S^T  = K_j Q_i^T   (SS, M = kv 128, N = q 128, TMEM cols [0,128))
//                   dP^T = V_j dO_i^T  (SS, N = 128, TMEM cols [128,256))
//                   dV  += P^T dO_i    (TS: P^T bf16 written over S^T; acc [384,448))
//                   dK  += dS^T Q_i    (SS: dS^T bf16 in smem, K-major view; acc [448,512))
//                   dQ_i (+)= dS K_j   (SS: same dS^T smem tile, MN-major view; two
//                                       accumulators [256,320) / [320,384) chained by
//                                       the mask's dQ plan)
//                 order per tile: dP^T(g+1) as soon as the compute warps hold S^T / dP^T(g)
//                 in registers | dV(g) S^T(g+1) | dK(g) dQ(g); dQ(g) overlaps the compute
//                 warps' start on tile g+1.
//    compute warps  thread = key row, kCmpWarps / 4 warps per TMEM lane quarter:
//                 P^T, dS^T from S^T, dP^T (element mask only on partial tiles: the
//                 full-tile code has none); P^T packed back into TMEM, dS^T to smem.
//    last warpgroup thread = query row: dQ_i drain at the end of a dQ
//                 chain (complete chains -> bf16 dq rows; others -> smem -> TMA
//                 reduce-add into the fp32 accumulator) and the dK / dV rows of
//                 each unit (row stores through a per-warp smem transpose, store_rows_t).
// K9 dq_finalize    : fp32 accumulator -> bf16 dQ.
#ifdef HLA_BWD_PROF
#define HLA_PROF_ON
#endif
#include <type_traits>

#include "attn_bwd_common.cuh"

namespace hla {
#ifdef HLA_BWD_PROF
__device__ unsigned long long g_bwd_prof[1024][24];
#define HLA_PROF_ARRAY g_bwd_prof
#endif
namespace bwd {
namespace {

// Warp roles: warpgroup 0 = TMA producers + MMA issuer, then kCmpWarps compute warps (P / dS;
// kCmpWarps / 4 per TMEM lane quarter, each over 128 / (kCmpWarps / 4) query columns), then
// one warpgroup for the dQ drains and the dK / dV epilogue.
#ifndef HLA_BWD_CMP_WARPS
#define HLA_BWD_CMP_WARPS 8
#endif
constexpr int kCmpWarps = HLA_BWD_CMP_WARPS;
static_assert(kCmpWarps == 8 || kCmpWarps == 16, "compute warps: 2 or 4 per TMEM lane quarter");
constexpr int kCmpThreads = kCmpWarps * 32;
constexpr int kChunks = 16 / kCmpWarps;              // 32-column chunks of S^T / dP^T per compute thread
constexpr int kDqWarp0 = 4 + kCmpWarps;              // first dQ / epilogue warp
constexpr int kThreads = (kDqWarp0 + 4) * 32;
// per-warpgroup register budgets (setmaxnreg; the launch allocates 65536 / kThreads, rounded to 8)
#ifndef HLA_BWD_REGS_CTL
#define HLA_BWD_REGS_CTL 64
#endif
constexpr int kRegsCtl = kCmpWarps == 16 ? 56 : HLA_BWD_REGS_CTL, kRegsCmp = kCmpWarps == 16 ? 88 : 168,
              kRegsDq = kCmpWarps == 16 ? 56 : 104;
// columns per TMEM load batch of the dQ drain / dK dV epilogue (a full D = 64 row needs ~96 registers)
template <int D>
constexpr int ep_cols() { return kRegsDq >= 96 ? D : 32; }
static_assert(128 * (kRegsCtl + kRegsDq) + kCmpThreads * kRegsCmp <= kThreads * ((65536 / kThreads) & ~7),
              "register budget");
constexpr uint32_t kColS = 0, kColDP = 128, kColDQ = 256, kColDV = 384, kColDK = 448;   // dQ: 2 x 64 columns
// Q / dO / LSE / D stages: tile g uses stage g & 1 (a stage that already holds the tile's
// q-block is re-published without a reload).  A third stage (reuse-aware ring, single dS^T
// tile) was measured slower: DESIGN.md 6f.
constexpr int kQStages = 2;

// Dev-only decomposition switches (`make VARIANT=name DEFS=-DHLA_BWD_VAR=<mask>`; results
// are garbage, the timing is the point -- DESIGN.md 6f): 1 no MMAs (commits still arrive),
// 2 no P / dS compute (the compute warps only wait and arrive), 4 no TMA loads (barriers
// still arrive), 8 no dQ drain / dK dV epilogue (waits and arrives only).
#ifndef HLA_BWD_VAR
#define HLA_BWD_VAR 0
#endif
constexpr int kVar = HLA_BWD_VAR;



template <int D>
struct FullSmem {
  static constexpr uint32_t kTileBytes = kBlock * D * 2;
  alignas(1024) uint8_t k[2][kTileBytes];
  alignas(1024) uint8_t v[2][kTileBytes];
  alignas(1024) uint8_t q[kQStages][kTileBytes];
  alignas(1024) uint8_t dO[kQStages][kTileBytes];
  alignas(1024) uint8_t ds[2][2 * 128 * 128];   // dS^T bf16 x2 (tile parity): [q/64][kv 128][64 q], SWIZZLE_128B
  alignas(1024) float dq_stage[kBlock * 32];    // fp32 dQ half tile [128][32], SWIZZLE_128B
  alignas(16) float lse[kQStages][kBlock];
  alignas(16) float dd[kQStages][kBlock];
  alignas(128) uint8_t epi_stage[4][2048];        // per dQ warp: row-store transpose (store_rows_t)
  uint64_t kv_full[2], kv_empty[2], q_full[kQStages], q_empty[kQStages], s_full, s_read, p_ready, ds_ready,
      dq_full[2], dq_free[2], dkv_full, epi_done;
  // kFuse (preprocess folded in): O tile of a newly loaded q-block (in the dq_stage bytes,
  // unused when every dQ chain is local) landed / consumed
  uint64_t o_full, o_empty;
  uint64_t dbg_bar;
  uint32_t tmem_base;
};

// Persistent: CTA c processes kv-block work units c, c + G, ... (pairs of kv-blocks of
// one (b, h)).  K/V are double-buffered across units, so the next unit's K/V (and first
// Q/dO) stream in while the current unit computes; the dK/dV epilogue of a unit
// overlaps the first MMAs of the next one.  Phase counters: n = units with tiles so
// far, g = (q-block) tiles so far.
// kFuse: the backward preprocess folded into the kernel (only when every q-block's dQ chain is
// local, so the dq_stage bytes are free): warp 0 loads the raw LSE and the O tile of each newly
// loaded q-block; the 256 compute warps' threads form D * scale = rowsum(dO o O) * scale and
// LSE * log2(e) in the stage (form_d) when they first meet the q-block, before its S^T lands.
// tmDQ is then the O map.  (D formed by the dQ warpgroup -- one tile ahead of its drains, or
// serviced inside its waits -- measured slower: that group is busy with drains and epilogues
// exactly when the next unit's q-blocks land, DESIGN 6g.)
template <int D, bool kTwoD, bool kGather, bool kFuse>
__global__ void __launch_bounds__(kThreads, 1)
    attn_bwd_full_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                    const __grid_constant__ CUtensorMap tmDQ, const BwdParams prm) {
  extern __shared__ uint8_t smem_raw[];
  using Smem = FullSmem<D>;
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < 2; ++s) {
      sm100::mbar_init(&sm.kv_full[s], 2);    // producer warps 0 (K), 2 (V)
      sm100::mbar_init(&sm.kv_empty[s], 1);
      sm100::mbar_init(&sm.dq_full[s], 1);
      sm100::mbar_init(&sm.dq_free[s], 128);
    }
    for (int s = 0; s < kQStages; ++s) {
      sm100::mbar_init(&sm.q_full[s], 3);     // producer warps 0 (LSE, D), 2 (Q), 3 (dO)
      sm100::mbar_init(&sm.q_empty[s], 1);
    }
    sm100::mbar_init(&sm.s_full, 1);
    sm100::mbar_init(&sm.s_read, kCmpThreads);
    sm100::mbar_init(&sm.p_ready, kCmpThreads);
    sm100::mbar_init(&sm.ds_ready, kCmpThreads);
    sm100::mbar_init(&sm.dkv_full, 1);
    sm100::mbar_init(&sm.epi_done, 128);
    sm100::mbar_init(&sm.dbg_bar, 1);
    sm100::mbar_init(&sm.o_full, 1);
    sm100::mbar_init(&sm.o_empty, 1);
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
  // LSE / D stages start zeroed: the bulk copies fill only real rows, and masked
  // (P = 0) phantom columns of a ragged tile must see finite values (0 * NaN = NaN)
  for (int i = threadIdx.x; i < kQStages * kBlock; i += kThreads) {
    (&sm.lse[0][0])[i] = 0.f;
    (&sm.dd[0][0])[i] = 0.f;
  }
  sm100::fence_proxy_async_smem();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  HLA_TR_DECL;

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsCtl) : "memory");
    const uint32_t tmem = sm.tmem_base;   // read after the register split (not spilled across it)
    HLA_PDECL;
    UnitGeom ug;
    ug.mk = (prm.N + kBlock - 1) / kBlock;   // last kv-block may be ragged
    ug.ppb = (ug.mk + 1) / 2;
    ug.pairs = ug.ppb * prm.heads * prm.batch;
    ug.mkd = prm.mk_div;
    ug.ppbd = prm.ppb_div;
    const int32_t mk = ug.mk;
    if (warp != 1) {
      // ----------------------------------------------------------- TMA producers
      // Three warps run the same schedule and split the loads (a CTA's TMA gather4
      // throughput grows with the number of issuing warps): warp 0 K + LSE / D,
      // warp 2 V + Q, warp 3 dO.  Every warp arrives (with its own byte count) on
      // the barriers it feeds, so no expect_tx has to precede another warp's copy.
      const uint64_t pol_kv = sm100::policy_evict_first();
      const uint64_t pol_q = sm100::policy_evict_last();
      const int role = warp == 0 ? 0 : warp - 1;   // 0, 1, 2
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
            if (lane == 0 && (kVar & 4)) {
              sm100::mbar_arrive(&sm.q_full[s]);
            } else if (lane == 0) {
              // LSE / D of the real rows only (ragged last tile: N % 4 == 0, so 16-B multiples);
              // kFuse: the raw LSE only (D is formed in the kernel from the O tile below)
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
              load_rows<D, kGather>(reinterpret_cast<uint8_t*>(sm.dq_stage), &tmDQ, &sm.o_full, h, b, prm.N,
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
      HLA_PFLUSH(13, 15, warp == 0 && lane == 0);
    } else if (lane == 0) {
      // ------------------------------------------------------------- MMA issuer
      // Per tile g of the flattened (unit, q-block) sequence, driven by the compute
      // warps' hand-offs for tile g:
      //   s_read(g)   S^T(g), dP^T(g) are in registers -> dP^T(g+1)         (SS, N = 128)
      //   p_ready(g)  P^T(g) is in TMEM over S^T(g)    -> dV(g) (TS), then S^T(g+1)
      //                                                   (SS, N = 128; after dV(g) in
      //                                                   the in-order pipe)
      //   ds_ready(g) dS^T(g) is in smem               -> dK(g), dQ(g)      (SS)
      // dQ(g) runs on the tensor pipe while the compute warps start tile g+1.  When tile
      // g+1's operands have not landed, its MMAs wait behind dK / dQ(g) instead of
      // blocking them.
      constexpr uint32_t idesc_s = sm100::make_idesc_bf16(kBlock, kBlock, false, false);   // S^T, dP^T
      constexpr uint32_t idesc_kv = sm100::make_idesc_bf16(kBlock, D, false, true);        // dV, dK
      constexpr uint32_t idesc_q = sm100::make_idesc_bf16(kBlock, D, true, true);          // dQ
      const uint32_t tDQ = tmem + kColDQ, tDV = tmem + kColDV, tDK = tmem + kColDK;
      TileIter cur;
      cur.init(prm.t_row_ptr, ug);
      uint32_t g = 0;
      uint32_t dq_started0 = 0, dq_started1 = 0;   // chains begun per dQ accumulator
      auto issue_dp = [&](const TileIter& it, uint32_t gg) {
#pragma unroll
        for (int kk = 0; kk < D / 16 && !(kVar & 1); ++kk)
          sm100::mma_ss(tmem + kColDP, kmajor_desc<D>(sm.v[it.n & 1], kk), kmajor_desc<D>(sm.dO[gg & 1], kk),
                        idesc_s, kk > 0);
      };
      auto issue_s = [&](const TileIter& it, uint32_t gg) {
#pragma unroll
        for (int kk = 0; kk < D / 16 && !(kVar & 1); ++kk)
          sm100::mma_ss(tmem + kColS, kmajor_desc<D>(sm.k[it.n & 1], kk), kmajor_desc<D>(sm.q[gg & 1], kk), idesc_s,
                        kk > 0);
        sm100::mma_commit(&sm.s_full);   // also covers the earlier dP^T(gg)
      };
      auto next_ready = [&](const TileIter& it, uint32_t gg) {
        return (it.t != 0 || sm100::mbar_test_wait(&sm.kv_full[it.n & 1], (it.n >> 1) & 1)) &&
               sm100::mbar_test_wait(&sm.q_full[gg & 1], (gg >> 1) & 1);
      };
      auto wait_next = [&](const TileIter& it, uint32_t gg) {
        HLA_PMARK(t0);
        if (it.t == 0) sm100::mbar_wait(&sm.kv_full[it.n & 1], (it.n >> 1) & 1);
        sm100::mbar_wait(&sm.q_full[gg & 1], (gg >> 1) & 1);
        HLA_PADD(2, t0);
        sm100::tc_fence_after();
      };
      if (cur.valid) {
        wait_next(cur, 0);
        issue_dp(cur, 0);
        issue_s(cur, 0);
      }
      HLA_PMARK(tl0);
      while (cur.valid) {
        TileIter nxt = cur;
        nxt.advance(prm.t_row_ptr, ug);
        const uint32_t fdq = dq_plan(prm.t_dq, cur.rs + cur.t, g);
        const int kvs = cur.n & 1;
        const int s = g & 1;
        const bool last_of_unit = cur.t == cur.nt - 1;
        bool dp_next = false, s_next = false;
        HLA_PW(0, sm100::mbar_wait(&sm.s_read, g & 1));
        if (nxt.valid && next_ready(nxt, g + 1)) {
          sm100::tc_fence_after();
          issue_dp(nxt, g + 1);
          dp_next = true;
        }
        HLA_PW(0, sm100::mbar_wait(&sm.p_ready, g & 1));
        sm100::tc_fence_after();
        if (cur.t == 0 && cur.n > 0) {
          // the previous unit's dV / dK must have been drained from TMEM
          HLA_PW(1, sm100::mbar_wait(&sm.epi_done, (cur.n - 1) & 1));
          sm100::tc_fence_after();
        }
#pragma unroll
        for (int kk = 0; kk < kBlock / 16 && !(kVar & 1); ++kk)
          sm100::mma_ts(tDV, tmem + kColS + packed_col(kk), mnmajor_desc<D>(sm.dO[s], kk), idesc_kv,
                        (cur.t > 0 || kk > 0) ? 1u : 0u);
        if (nxt.valid && (dp_next || next_ready(nxt, g + 1))) {
          sm100::tc_fence_after();
          if (!dp_next) issue_dp(nxt, g + 1);
          issue_s(nxt, g + 1);
          s_next = true;
        }
        HLA_PW(0, sm100::mbar_wait(&sm.ds_ready, g & 1));
        sm100::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < kBlock / 16 && !(kVar & 1); ++kk)
          sm100::mma_ss(tDK, ds_kmajor_desc(sm.ds[g & 1], kk), mnmajor_desc<D>(sm.q[s], kk), idesc_kv,
                        (cur.t > 0 || kk > 0) ? 1u : 0u);
        sm100::mma_commit(&sm.q_empty[s]);   // Q_g / dO_g no longer read (dQ needs only dS and K)
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
          sm100::mma_ss(tDQ + dqb * 64, ds_mnmajor_desc(sm.ds[g & 1], kk), mnmajor_desc<D>(sm.k[kvs], kk),
                        idesc_q, (kk > 0 || !dq_new) ? 1u : 0u);
        if (fdq & HLA_DQ_DRAIN) sm100::mma_commit(&sm.dq_full[dqb]);
        if (last_of_unit) sm100::mma_commit(&sm.kv_empty[kvs]);
        if (nxt.valid && !s_next) {
          wait_next(nxt, g + 1);
          if (!dp_next) issue_dp(nxt, g + 1);
          issue_s(nxt, g + 1);
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
  } else if (warp < kDqWarp0) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsCmp) : "memory");
    const uint32_t tmem = sm.tmem_base;   // read after the register split (not spilled across it)
    unsigned long long tiles_done = 0;
    HLA_PDECL;
    // --------------------------------------------- P^T / dS^T (thread = key row)
    // warp sets cset = 0 .. kCmpWarps / 4 - 1 (4 consecutive warps each) share every TMEM lane
    // quarter; cset c processes the kChunks 32-column chunks [c * kChunks, (c + 1) * kChunks).
    const int quarter = warp & 3;
    const int cset = (warp - 4) >> 2;
    const int row = quarter * 32 + lane;
    const int cth = (warp - 4) * 32 + lane;   // compute thread 0 .. 255
    uint32_t n_od = 0;                          // kFuse: O tiles consumed
    int64_t dtag0 = -1, dtag1 = -1;             // kFuse: q-block held by stage 0 / 1
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const float sl2 = prm.scale_log2, scale = prm.scale;
    UnitGeom ug;
    ug.mk = (prm.N + kBlock - 1) / kBlock;
    ug.ppb = (ug.mk + 1) / 2;
    ug.pairs = ug.ppb * prm.heads * prm.batch;
    ug.mkd = prm.mk_div;
    ug.ppbd = prm.ppb_div;
    const int32_t mk = ug.mk;
    uint32_t g = 0;
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
      for (int t = 0; t < nt; ++t, ++g) {
        const uint8_t kd = __ldg(prm.t_kind + rs + t);
        const int32_t q0 = __ldg(prm.t_col_idx + rs + t) * prm.col_mul;
        const int s = g & 1;
        HLA_PW(5, sm100::mbar_wait(&sm.q_full[s], (g >> 1) & 1));
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
            sm100::named_bar_sync(kBarFormD, kCmpThreads);
            if (cth == 0) sm100::mbar_arrive(&sm.o_empty);
          }
        }
        const uint32_t lse2 = sm100::smem_u32(sm.lse[s]);
        const uint32_t dd = sm100::smem_u32(sm.dd[s]);
        const uint32_t dsbuf = sm100::smem_u32(sm.ds[g & 1]);
        HLA_PW(6, sm100::mbar_wait(&sm.s_full, g & 1));
        HLA_PMARK(tc0);
        sm100::tc_fence_after();
        uint32_t sr[kChunks][32], dpr[kChunks][32];
        if (!(kVar & 2)) {
#pragma unroll
          for (int j = 0; j < kChunks; ++j) {
            sm100::tmem_ld32(tmem + lane_off + kColS + (cset * kChunks + j) * 32, sr[j]);
            sm100::tmem_ld32(tmem + lane_off + kColDP + (cset * kChunks + j) * 32, dpr[j]);
          }
          sm100::tmem_wait_ld();
        }
        sm100::tc_fence_before();
        sm100::mbar_arrive(&sm.s_read);      // dP^T(g+1) may overwrite the dP^T columns
        HLA_PADD(16, tc0);
        // P^T = exp2(S^T scale log2e - LSE log2e) (+ bias).  Partial tiles only: masked
        // elements get an exponent of -inf (P = 0, hence dS = 0: D and dP^T are finite --
        // the LSE / D stages start zeroed, phantom rows load finite data).
        auto p_math = [&](auto partial_tag) {
          constexpr bool kPart = decltype(partial_tag)::value;
#pragma unroll
          for (int j = 0; j < kChunks; ++j) {
            const int c = cset * kChunks + j;
            const int32_t base = q0 + c * 32;
            // [ulo, uhi): 8-column groups of this chunk that hold an allowed query of some
            // key row of this warp (partial tiles of 1D patterns: each key row's queries are
            // one interval); the other groups are all masked, their exponentials skipped
            // (warp-uniform) and P = 0 there.
            int ulo = 0, uhi = 4;
            bool elem_mask = kPart;   // false: every element of this warp's chunk is allowed
            if (kPart && !kTwoD) {
              const int32_t lo = min(max(box.lo - base, 0), 32), hi = min(max(box.lo + box.len - base, 0), 32);
              elem_mask = !__all_sync(0xffffffffu, lo == 0 && hi == 32);
              const bool any = hi > lo;
              ulo = __reduce_min_sync(0xffffffffu, any ? lo : 32) >> 3;
              uhi = (__reduce_max_sync(0xffffffffu, any ? hi : 0) + 7) >> 3;
            }
            float* p = reinterpret_cast<float*>(sr[j]);   // P overwrites S in place
#pragma unroll
            for (int u4 = 0; u4 < 4; ++u4) {
              if (kPart && (u4 < ulo || u4 >= uhi)) {
#pragma unroll
                for (int e = 0; e < 8; ++e) p[u4 * 8 + e] = 0.f;
                continue;
              }
              const int qc = c * 32 + u4 * 8;
              const float4 la = sm100::lds_f4(lse2 + qc * 4), lb = sm100::lds_f4(lse2 + qc * 4 + 16);
              const float lv[8] = {la.x, la.y, la.z, la.w, lb.x, lb.y, lb.z, lb.w};
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                float x = fmaf(__uint_as_float(sr[j][u4 * 8 + e]), sl2, -lv[e]);
                if (kPart && elem_mask) {
                  const int32_t qq = base + u4 * 8 + e;
                  bool ok;
                  if (!kTwoD) {
                    ok = (uint32_t)(qq - box.lo) < (uint32_t)box.len;
                  } else {
                    const int32_t rq = prm.pat.log2W >= 0 ? (qq >> prm.pat.log2W) : prm.pat.w_div.div(qq);
                    const int32_t cq = qq - rq * prm.pat.W;
                    ok = ((uint32_t)(rq - box.lo) < (uint32_t)box.len) && ((uint32_t)(cq - box.c0) < (uint32_t)box.cn);
                  }
                  x = ok ? x : -INFINITY;
                }
                p[u4 * 8 + e] = sm100::ex2(x);
              }
            }
          }
        };
        if (!(kVar & 2)) {
          if (kd == 2) p_math(std::true_type{}); else p_math(std::false_type{});
        }
        HLA_PADD(18, tc0);
        if (!(kVar & 2)) {
          // P^T packed to bf16 over the first 16 columns of each S^T chunk (in registers):
          // the A operand of dV += P^T dO
#pragma unroll
          for (int j = 0; j < kChunks; ++j) {
            const float* p = reinterpret_cast<const float*>(sr[j]);
            uint32_t pk[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) pk[e] = sm100::pack_bf16(p[2 * e], p[2 * e + 1]);
            sm100::tmem_st16(tmem + lane_off + kColS + (cset * kChunks + j) * 32, pk);
          }
        }
        sm100::tmem_wait_st();
        sm100::tc_fence_before();
        sm100::mbar_arrive(&sm.p_ready);     // P^T(g) in TMEM: dV(g), then S^T(g+1) over it
        HLA_PADD(19, tc0);
        // (dS^T buffer g & 1 was last read by dK / dQ(g - 2), issued before S^T(g): s_full(g)
        // already certified their completion)
        if (!(kVar & 2)) {
          // dS^T = P^T o (dP^T scale - D scale) in place of dP^T, then bf16 smem tile [q/64][kv][64]
          // with the 128B swizzle (A of dK += dS^T Q and, MN-major view, of dQ = dS K)
#pragma unroll
          for (int j = 0; j < kChunks; ++j) {
            const int c = cset * kChunks + j;
            const float* p = reinterpret_cast<const float*>(sr[j]);
            float* ds = reinterpret_cast<float*>(dpr[j]);
#pragma unroll
            for (int u4 = 0; u4 < 4; ++u4) {
              const int qc = c * 32 + u4 * 8;
              const float4 da = sm100::lds_f4(dd + qc * 4), db = sm100::lds_f4(dd + qc * 4 + 16);
              const float dv[8] = {da.x, da.y, da.z, da.w, db.x, db.y, db.z, db.w};
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const int i = u4 * 8 + e;
                ds[i] = p[i] * fmaf(__uint_as_float(dpr[j][i]), scale, -dv[e]);
              }
              const uint32_t off =
                  (uint32_t)(qc >> 6) * 16384u + sm100::swz128((uint32_t)row * 128u + (uint32_t)(qc & 63) * 2u);
              sm100::sts_u4(dsbuf + off, sm100::pack_bf16(ds[u4 * 8 + 0], ds[u4 * 8 + 1]),
                            sm100::pack_bf16(ds[u4 * 8 + 2], ds[u4 * 8 + 3]),
                            sm100::pack_bf16(ds[u4 * 8 + 4], ds[u4 * 8 + 5]),
                            sm100::pack_bf16(ds[u4 * 8 + 6], ds[u4 * 8 + 7]));
            }
          }
        }
        HLA_PADD(17, tc0);
        sm100::fence_proxy_async_smem();
        sm100::tc_fence_before();
        sm100::mbar_arrive(&sm.ds_ready);
        HLA_PADD(7, tc0);
      }
      tiles_done += nt;
    }
    if (warp == 4 && lane == 0 && prm.visited != nullptr && tiles_done > 0) atomicAdd(prm.visited, tiles_done);
    HLA_PFLUSH(5, 9, warp == 4 && lane == 0);
    HLA_PFLUSH(16, 20, warp == 4 && lane == 0);
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsDq) : "memory");
    const uint32_t tmem = sm.tmem_base;   // read after the register split (not spilled across it)
    HLA_PDECL;
    // ------------------------------------------ dQ partial -> fp32 accumulator
    // thread = query row: drain the dQ_i tile from TMEM (then release it), stage it
    // in shared memory (two 32-column halves, 128B swizzle) and let the TMA engine
    // add it into the fp32 accumulator (cp.reduce.async.bulk.tensor ... add) -- no
    // per-thread atomics, so the LSU stays free for the compute warps.
    UnitGeom ug;
    ug.mk = (prm.N + kBlock - 1) / kBlock;
    ug.ppb = (ug.mk + 1) / 2;
    ug.pairs = ug.ppb * prm.heads * prm.batch;
    ug.mkd = prm.mk_div;
    ug.ppbd = prm.ppb_div;
    const int32_t mk = ug.mk;
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const bool leader = warp == kDqWarp0 && lane == 0;
    constexpr int kEpCols = ep_cols<D>();
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
        const bool local = (fdq & HLA_DQ_LOCAL) != 0;
        // complete dQ_i (LOCAL; dS carries the softmax scale): bf16 rows straight to dq, to the
        // grid cell under the fused reorder; phantom rows of a ragged tile write nothing
        uint4* dqp = nullptr;
        if (local && qblk * prm.col_mul + row < prm.N) {
          const int32_t qs = qblk * prm.col_mul + row;
          const int32_t qcell = kGather ? __ldg(prm.s2c + qs) : qs;
          dqp = reinterpret_cast<uint4*>(prm.dq + (((int64_t)b * prm.N + qcell) * prm.heads + h) * D);
        }
        // the accumulator in kEpCols-column batches (all D columns when the register budget
        // allows: the dq_free hand-off then follows a single TMEM round trip)
#pragma unroll
        for (int hb = 0; hb < D / kEpCols; ++hb) {
          uint32_t r[kEpCols];
#pragma unroll
          for (int c = 0; c < kEpCols / 32; ++c)
            sm100::tmem_ld32(tmem + lane_off + kColDQ + dqb * 64 + hb * kEpCols + c * 32,
                             *reinterpret_cast<uint32_t(*)[32]>(r + c * 32));
          sm100::tmem_wait_ld();
          if (hb == D / kEpCols - 1) {
            sm100::tc_fence_before();
            sm100::mbar_arrive(&sm.dq_free[dqb]);     // the TMEM dQ accumulator may now be overwritten
          }
          if (local && kEpCols == D) {
            uint32_t w[D / 2];
#pragma unroll
            for (int e = 0; e < D / 2; ++e) w[e] = sm100::pack_bf16(__uint_as_float(r[2 * e]), __uint_as_float(r[2 * e + 1]));
            store_rows_t<D>(w, dqp, sm100::smem_u32(sm.epi_stage[quarter]), lane);
            continue;
          }
          if (local) {
#pragma unroll
            for (int v4 = 0; v4 < kEpCols / 8 && dqp; ++v4)
              dqp[hb * (kEpCols / 8) + v4] =
                  make_uint4(sm100::pack_bf16(__uint_as_float(r[8 * v4 + 0]), __uint_as_float(r[8 * v4 + 1])),
                             sm100::pack_bf16(__uint_as_float(r[8 * v4 + 2]), __uint_as_float(r[8 * v4 + 3])),
                             sm100::pack_bf16(__uint_as_float(r[8 * v4 + 4]), __uint_as_float(r[8 * v4 + 5])),
                             sm100::pack_bf16(__uint_as_float(r[8 * v4 + 6]), __uint_as_float(r[8 * v4 + 7])));
            continue;
          }
          // partial dQ_i -> smem stage (32 columns at a time, 128B swizzle) -> TMA reduce-add
          // into the fp32 accumulator
#pragma unroll
          for (int hh = 0; hh < kEpCols / 32; ++hh) {
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
              sm100::tma_reduce_add_3d(&tmDQ, sm.dq_stage, hb * kEpCols + hh * 32, h, qrow);
              sm100::bulk_commit_group();
            }
          }
        }
        HLA_PADD(10, td0);
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
        if constexpr (kEpCols == D) {
          // dV then dK: the dK load is in flight while the dV row is stored (<= 96 live registers)
          uint32_t r[D], pv[D / 2];
#pragma unroll
          for (int c = 0; c < D / 32; ++c)
            sm100::tmem_ld32(tmem + lane_off + kColDV + c * 32, *reinterpret_cast<uint32_t(*)[32]>(r + c * 32));
          sm100::tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < D / 2; ++e)
            pv[e] = sm100::pack_bf16(__uint_as_float(r[2 * e]), __uint_as_float(r[2 * e + 1]));
#pragma unroll
          for (int c = 0; c < D / 32; ++c)
            sm100::tmem_ld32(tmem + lane_off + kColDK + c * 32, *reinterpret_cast<uint32_t(*)[32]>(r + c * 32));
          const uint32_t stg = sm100::smem_u32(sm.epi_stage[quarter]);
          store_rows_t<D>(pv, real ? dvp : nullptr, stg, lane);
          sm100::tmem_wait_ld();
          sm100::tc_fence_before();
          sm100::mbar_arrive(&sm.epi_done);      // dV / dK accumulators may now be reset
#pragma unroll
          for (int e = 0; e < D / 2; ++e) pv[e] = sm100::pack_bf16(__uint_as_float(r[2 * e]), __uint_as_float(r[2 * e + 1]));
          store_rows_t<D>(pv, real ? dkp : nullptr, stg, lane);
        } else {
          // dV then dK in 32-column batches (register budget kRegsDq); epi_done after the last load
#pragma unroll
          for (int which = 0; which < 2; ++which) {
            uint4* dst = which ? dkp : dvp;
#pragma unroll
            for (int hh = 0; hh < D / 32; ++hh) {
              uint32_t r[32];
              sm100::tmem_ld32(tmem + lane_off + (which ? kColDK : kColDV) + hh * 32, r);
              sm100::tmem_wait_ld();
              if (which == 1 && hh == D / 32 - 1) {
                sm100::tc_fence_before();
                sm100::mbar_arrive(&sm.epi_done);      // dV / dK accumulators may now be reset
              }
#pragma unroll
              for (int v4 = 0; v4 < 4 && real; ++v4)
                dst[hh * 4 + v4] = make_uint4(sm100::pack_bf16(__uint_as_float(r[8 * v4 + 0]), __uint_as_float(r[8 * v4 + 1])),
                                              sm100::pack_bf16(__uint_as_float(r[8 * v4 + 2]), __uint_as_float(r[8 * v4 + 3])),
                                              sm100::pack_bf16(__uint_as_float(r[8 * v4 + 4]), __uint_as_float(r[8 * v4 + 5])),
                                              sm100::pack_bf16(__uint_as_float(r[8 * v4 + 6]), __uint_as_float(r[8 * v4 + 7])));
            }
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
  if (warp == 1) sm100::tmem_dealloc(sm.tmem_base, kTmemCols);
}

template <int D, bool kTwoD, bool kGather, bool kFuse>
hla_status launch_full_t(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv, const CUtensorMap& mdo,
                      const CUtensorMap& mdq, const BwdParams& prm, int32_t n_kblocks, cudaStream_t stream) {
  const size_t smem = sizeof(FullSmem<D>) + 1024;
  auto* fn = attn_bwd_full_kernel<D, kTwoD, kGather, kFuse>;
  HLA_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t pairs = (int64_t)((n_kblocks + 1) / 2) * prm.heads * prm.batch;   // work units (kv-block pairs)
  const int grid = (int)std::min<int64_t>(pairs, (int64_t)num_sms());
  fn<<<grid, kThreads, smem, stream>>>(mq, mk, mv, mdo, mdq, prm);
  HLA_CUDA_TRY(cudaGetLastError());
  return HLA_OK;
}

static_assert(sizeof(FullSmem<64>) + 1024 <= 227 * 1024, "bwd shared memory (d = 64) exceeds 227 KB");

}  // namespace

template <bool kFuse>
hla_status launch_full_f(int head_dim, bool gather, bool two_d, const CUtensorMap& mq, const CUtensorMap& mk,
                         const CUtensorMap& mv, const CUtensorMap& mdo, const CUtensorMap& mdq, const BwdParams& prm,
                         int32_t mkb, cudaStream_t stream) {
  if (head_dim == 64) {
    if (gather) return launch_full_t<64, false, true, kFuse>(mq, mk, mv, mdo, mdq, prm, mkb, stream);
    return two_d ? launch_full_t<64, true, false, kFuse>(mq, mk, mv, mdo, mdq, prm, mkb, stream)
                 : launch_full_t<64, false, false, kFuse>(mq, mk, mv, mdo, mdq, prm, mkb, stream);
  }
  if (gather) return launch_full_t<32, false, true, kFuse>(mq, mk, mv, mdo, mdq, prm, mkb, stream);
  return two_d ? launch_full_t<32, true, false, kFuse>(mq, mk, mv, mdo, mdq, prm, mkb, stream)
               : launch_full_t<32, false, false, kFuse>(mq, mk, mv, mdo, mdq, prm, mkb, stream);
}

hla_status launch_full(int head_dim, bool gather, bool two_d, bool fuse, const CUtensorMap& mq, const CUtensorMap& mk,
                       const CUtensorMap& mv, const CUtensorMap& mdo, const CUtensorMap& mdq, const BwdParams& prm,
                       int32_t mkb, cudaStream_t stream) {
  return fuse ? launch_full_f<true>(head_dim, gather, two_d, mq, mk, mv, mdo, mdq, prm, mkb, stream)
              : launch_full_f<false>(head_dim, gather, two_d, mq, mk, mv, mdo, mdq, prm, mkb, stream);
}

}  // namespace bwd

namespace {

using bwd::kBlock;
using bwd::kLog2e;

// K7: D = rowsum(dO o O) per (b, s, h) row of head_dim bf16, fp32, in sequence order s
// (rows read at grid cell s2c[s] under the fused reorder), stored pre-multiplied by
// the softmax scale; LSE converted to the log2 domain; dQ accumulator := 0 (rows of
// q-blocks whose dQ the main kernel writes directly -- q_local -- are skipped)
template <int D>
__global__ void __launch_bounds__(256) bwd_preprocess_kernel(const __nv_bfloat16* __restrict__ o,
                                                             const __nv_bfloat16* __restrict__ dout,
                                                             const float* __restrict__ lse, float scale,
                                                             float* __restrict__ dsum, float* __restrict__ lse2,
                                                             float* __restrict__ dq_acc,
                                                             const int32_t* __restrict__ s2c,
                                                             const uint8_t* __restrict__ q_local, FastDiv N,
                                                             FastDiv heads, int32_t rows) {
  // one thread per 8 elements (16 B of O and of dO); 32-bit index math (rows * D / 8 < 2^31).
  // Threads walk the OUTPUT order (b, h, s): D / LSE are written as contiguous runs (in
  // token order the 4-byte results of one warp land in `heads` different sectors).
  constexpr int kLanes = D / 8;   // lanes per row
  const int32_t gid = (int32_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int32_t i = gid / kLanes;             // (b * heads + h) * N + s
  const int part = gid - i * kLanes;
  if (i >= rows) return;
  const int32_t bh = N.div(i), s = i - bh * N.d;
  const int32_t bb = heads.div(bh), hq = bh - bb * heads.d;
  const int32_t r = (bb * N.d + s) * heads.d + hq;   // sequence-order row (b * N + s) * heads + h
  const int64_t src = s2c ? ((int64_t)(bb * N.d + __ldg(s2c + s)) * heads.d + hq) : (int64_t)r;
  const uint4 a = __ldg(reinterpret_cast<const uint4*>(o + src * D + part * 8));
  const uint4 g = __ldg(reinterpret_cast<const uint4*>(dout + src * D + part * 8));
  const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
  const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&g);
  float acc = 0.f;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 x = __bfloat1622float2(a2[e]), y = __bfloat1622float2(g2[e]);
    acc = fmaf(x.x, y.x, acc);
    acc = fmaf(x.y, y.y, acc);
  }
#pragma unroll
  for (int o2 = kLanes / 2; o2 > 0; o2 >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o2);
  if (!(q_local && __ldg(q_local + (s >> 7)))) {
    float4* z = reinterpret_cast<float4*>(dq_acc + (int64_t)r * D + part * 8);   // zeroing is layout-agnostic
    z[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (part == 0) {
    dsum[i] = acc * scale;                       // D * scale (dS = P o (dP * scale - D * scale))
    lse2[i] = __ldg(lse + i) * kLog2e;           // LSE in the log2 domain
  }
}

// Folded preprocess with non-local dQ chains: the accumulator rows of non-local q-blocks := 0
// (sequence order, 32 B per thread; rows of local q-blocks -- q_local -- are never read)
__global__ void __launch_bounds__(256) dq_zero_kernel(float4* __restrict__ acc, const uint8_t* __restrict__ q_local,
                                                      FastDiv N, FastDiv row_v, int32_t n_v) {
  const int32_t t = (int32_t)blockIdx.x * blockDim.x + threadIdx.x;   // (b * N + s) * row_v + part
  if (t >= n_v) return;
  if (q_local) {
    const int32_t bs = row_v.div(t);
    const int32_t s = bs - N.div(bs) * N.d;
    if (__ldg(q_local + (s >> 7))) return;
  }
  acc[2 * (int64_t)t] = make_float4(0.f, 0.f, 0.f, 0.f);
  acc[2 * (int64_t)t + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// K9: dQ = bf16(accumulator) -- the accumulator is in sequence order; under the
// fused reorder each row is written to its grid cell s2c[s] (SURVEY 8(a) a8:
// "dQ finalize + inverse permutation").  One thread per 8 elements (32 B in, 16 B out).
// Rows of local q-blocks (q_local: written by the main kernel) are left alone.
__global__ void __launch_bounds__(256) dq_finalize_kernel(const float4* __restrict__ acc, uint4* __restrict__ dq,
                                                          const int32_t* __restrict__ s2c,
                                                          const uint8_t* __restrict__ q_local, FastDiv N,
                                                          FastDiv row_v, int32_t n_v) {
  const int32_t t = (int32_t)blockIdx.x * blockDim.x + threadIdx.x;   // n_v = B * N * row_v < 2^31
  if (t >= n_v) return;
  int64_t o = t;
  if (s2c || q_local) {   // t = (b * N + s) * row_v + part, row_v = heads * D / 8
    const int32_t bs = row_v.div(t), part = t - bs * row_v.d;
    const int32_t b = N.div(bs), s = bs - b * N.d;
    if (q_local && __ldg(q_local + (s >> 7))) return;
    if (s2c) o = (int64_t)(b * N.d + __ldg(s2c + s)) * row_v.d + part;
  }
  const float4 v0 = __ldcs(acc + 2 * (int64_t)t), v1 = __ldcs(acc + 2 * (int64_t)t + 1);
  dq[o] = make_uint4(sm100::pack_bf16(v0.x, v0.y), sm100::pack_bf16(v0.z, v0.w), sm100::pack_bf16(v1.x, v1.y),
                     sm100::pack_bf16(v1.z, v1.w));
}

}  // namespace
}  // namespace hla

using namespace hla;

#ifdef HLA_BWD_PROF
// dev-only: per-CTA wait / work cycle sums of the last attn_bwd_kernel launch (HLA_BWD_PROF builds)
extern "C" __attribute__((visibility("default"))) int hla_debug_bwd_prof(unsigned long long* host, int ctas) {
  cudaDeviceSynchronize();
  const int n = ctas < 1024 ? ctas : 1024;
  cudaMemcpyFromSymbol(host, hla::g_bwd_prof, (size_t)n * 24 * sizeof(unsigned long long));
  return n;
}
#endif

extern "C" size_t hla_attn_bwd_workspace(int32_t batch, int32_t heads, int32_t n, int32_t head_dim) {
  const size_t acc = (size_t)batch * n * heads * head_dim * 4;
  const size_t row = (size_t)batch * heads * n * 4;
  return ((acc + 255) / 256) * 256 + 2 * ((row + 255) / 256) * 256;
}

namespace {

// q_dq_local of a mask with a complete dQ plan (else null: every q-block via the accumulator)
const uint8_t* plan_of(const hla_block_mask* m, int32_t n) {
  if (!m || !m->t_dq || !m->q_dq_local || m->n_dq_nonlocal < 0) return nullptr;
  const int32_t tiles = m->w_row_ptr ? (m->n_qblocks + 1) / 2 : m->n_qblocks;   // block 64: per 128-row tile
  return tiles == (n + kBlock - 1) / kBlock ? m->q_dq_local : nullptr;
}

// the backward schedule: full-tile (attn_bwd_full_kernel) when full tiles are at least half of the
// mask's tiles, half-tile (attn_bwd_split_kernel) otherwise and with the global RPB
#ifndef HLA_BWD_SCHED
#define HLA_BWD_SCHED 0   // dev A/B: 0 = by tile mix, 1 = full-tile whenever possible, 2 = half-tile always
#endif
bool full_schedule(bool rpb, const AttnLists& lists) {
  return !rpb && (HLA_BWD_SCHED == 1 ||
                  (HLA_BWD_SCHED == 0 && lists.t_n_full >= lists.t_n_partial && lists.t_n_full > 0));
}

// workspace carve-up: [fp32 dQ accumulator][fp32 D*scale][fp32 LSE*log2e], 256-aligned regions
hla_status carve_workspace(int32_t batch, int32_t heads, int32_t n, int32_t head_dim, void* workspace,
                           size_t workspace_bytes, float** dq_acc, float** dsum, float** lse2 = nullptr) {
  HLA_REQUIRE(workspace != nullptr, HLA_ERR_INVALID, "null workspace");
  HLA_REQUIRE((uintptr_t)workspace % 256 == 0, HLA_ERR_INVALID, "workspace must be 256-byte aligned");
  const size_t need = hla_attn_bwd_workspace(batch, heads, n, head_dim);
  HLA_REQUIRE(workspace_bytes >= need, HLA_ERR_INVALID, "workspace %zu < %zu bytes", workspace_bytes, need);
  const size_t acc = (size_t)batch * n * heads * head_dim * 4;
  *dq_acc = reinterpret_cast<float*>(workspace);
  const size_t row = (size_t)batch * heads * n * 4;
  *dsum = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(workspace) + ((acc + 255) / 256) * 256);
  if (lse2) *lse2 = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(*dsum) + ((row + 255) / 256) * 256);
  return HLA_OK;
}

}  // namespace

extern "C" hla_status hla_attn_bwd_preprocess(int32_t batch, int32_t heads, int32_t n, int32_t head_dim,
                                              float scale, const void* o, const void* dout, const float* lse,
                                              const int32_t* seq_to_cell, const hla_block_mask* plan_mask,
                                              void* workspace, size_t workspace_bytes, cudaStream_t stream) {
  clear_error();
  HLA_REQUIRE(head_dim == 32 || head_dim == 64, HLA_ERR_UNSUPPORTED, "head_dim %d not in {32, 64}", head_dim);
  HLA_REQUIRE(batch >= 1 && heads >= 1 && n >= 1, HLA_ERR_INVALID, "bad shape");
  const uint8_t* q_local = plan_of(plan_mask, n);
  HLA_REQUIRE(o && dout && ((uintptr_t)o | (uintptr_t)dout) % 16 == 0, HLA_ERR_INVALID, "o/dout null or unaligned");
  HLA_REQUIRE(lse != nullptr, HLA_ERR_INVALID, "null lse");
  float *dq_acc, *dsum, *lse2;
  hla_status st = carve_workspace(batch, heads, n, head_dim, workspace, workspace_bytes, &dq_acc, &dsum, &lse2);
  if (st != HLA_OK) return st;
  const float sc = scale > 0.f ? scale : 1.0f / sqrtf((float)head_dim);
  const int64_t rows = (int64_t)batch * n * heads;
  const int64_t threads = rows * (head_dim / 8);
  HLA_REQUIRE(threads < (1ll << 31), HLA_ERR_UNSUPPORTED, "B * N * heads * head_dim too large");
  const unsigned blocks = (unsigned)((threads + 255) / 256);
  if (head_dim == 64)
    bwd_preprocess_kernel<64><<<blocks, 256, 0, stream>>>(reinterpret_cast<const __nv_bfloat16*>(o),
                                                          reinterpret_cast<const __nv_bfloat16*>(dout), lse, sc,
                                                          dsum, lse2, dq_acc, seq_to_cell, q_local, make_fastdiv(n),
                                                          make_fastdiv(heads), (int32_t)rows);
  else
    bwd_preprocess_kernel<32><<<blocks, 256, 0, stream>>>(reinterpret_cast<const __nv_bfloat16*>(o),
                                                          reinterpret_cast<const __nv_bfloat16*>(dout), lse, sc,
                                                          dsum, lse2, dq_acc, seq_to_cell, q_local, make_fastdiv(n),
                                                          make_fastdiv(heads), (int32_t)rows);
  HLA_CUDA_TRY(cudaGetLastError());
  return HLA_OK;
}

namespace {

// Everything hla_attn_bwd_main launches with: validated arguments, kernel parameters, tensor
// maps and the schedule.  Built (and every argument checked) before anything is launched.
struct MainPlan {
  bwd::BwdParams prm;
  CUtensorMap mq, mk, mv, mdo, mdq, mo;
  int32_t head_dim, mkb;
  bool gather, two_d, full;
  bool fuse;       // preprocess folded into the main kernel (hla_attn_bwd only)
  bool zero_acc;   // fuse with non-local dQ chains: the accumulator rows still need zeroing
};

hla_status prepare_main(const hla_pattern_desc* d, const hla_block_mask* m, int32_t batch, int32_t heads,
                        int32_t head_dim, float scale, const void* q, const void* k, const void* v,
                        const void* dout, void* dq, void* dk, void* dv, const int32_t* seq_to_cell,
                        const hla_score_mod* score_mod, void* workspace, size_t workspace_bytes,
                        int64_t* tiles_visited, MainPlan* pl) {
  Pattern pat;
  AttnLists lists;
  hla_status st = check_attn_args(d, m, batch, heads, head_dim, &pat, &lists);
  if (st != HLA_OK) return st;
  HLA_REQUIRE(lists.t_row_ptr && lists.t_col && lists.t_kind, HLA_ERR_INVALID, "transposed mask arrays missing");
  HLA_REQUIRE(q && k && v && dout && dk && dv, HLA_ERR_INVALID, "null pointer");
  HLA_REQUIRE(dq || !plan_of(m, pat.N), HLA_ERR_INVALID, "dq required: the mask's dQ plan writes local q-blocks");
  HLA_REQUIRE(((uintptr_t)q | (uintptr_t)k | (uintptr_t)v | (uintptr_t)dout | (uintptr_t)dk | (uintptr_t)dv |
               (uintptr_t)dq) % 16 == 0,
              HLA_ERR_INVALID, "tensors must be 16-byte aligned");
  float *dq_acc, *dsum, *lse2;
  st = carve_workspace(batch, heads, pat.N, head_dim, workspace, workspace_bytes, &dq_acc, &dsum, &lse2);
  if (st != HLA_OK) return st;
  const float sc = scale > 0.f ? scale : 1.0f / sqrtf((float)head_dim);
  bwd::BwdParams& prm = pl->prm;
  prm.pat = pat;
  prm.N = pat.N;
  prm.heads = heads;
  prm.batch = batch;
  {
    const int32_t mkb = (pat.N + bwd::kBlock - 1) / bwd::kBlock;
    prm.mk_div = make_fastdiv(mkb);
    prm.ppb_div = make_fastdiv((mkb + 1) / 2);
    prm.heads_div = make_fastdiv(heads);
  }
  prm.scale = sc;
  prm.scale_log2 = sc * kLog2e;
  prm.t_row_ptr = lists.t_row_ptr;
  prm.t_col_idx = lists.t_col;
  prm.t_kind = lists.t_kind;
  prm.col_mul = lists.col_mul;
  prm.t_dq = plan_of(m, pat.N) ? m->t_dq : nullptr;
  prm.dq = reinterpret_cast<__nv_bfloat16*>(dq);
  prm.lse2 = lse2;
  prm.dsum = dsum;
  prm.dq_acc = dq_acc;
  prm.dk = reinterpret_cast<__nv_bfloat16*>(dk);
  prm.dv = reinterpret_cast<__nv_bfloat16*>(dv);
  prm.visited = reinterpret_cast<unsigned long long*>(tiles_visited);
  prm.s2c = seq_to_cell;
  if ((st = parse_score_mod(d, score_mod, true, &prm.rpb, &prm.drpb, &prm.cells)) != HLA_OK) return st;
  prm.grid_h = pat.H;
  prm.grid_w = pat.W;
  prm.rpb_w = 2 * pat.W - 1;
  prm.rpb_hw = (2 * pat.H - 1) * prm.rpb_w;
  prm.inv_scale = 1.f / sc;
  pl->gather = seq_to_cell != nullptr;
  HLA_REQUIRE(!pl->gather || d->order != HLA_ORDER_ROW_MAJOR, HLA_ERR_INVALID,
              "seq_to_cell (fused reorder) is only meaningful for Hilbert-order patterns");
  prm.box8 = (pl->gather && d->order == HLA_ORDER_HILBERT_TILED && head_dim == 32) ? ilog2(pat.W) + 1 : 0;
  HLA_REQUIRE(!pl->gather || ((uintptr_t)seq_to_cell & 15) == 0, HLA_ERR_INVALID,
              "seq_to_cell must be 16-byte aligned");
  const int64_t tok = (int64_t)batch * pat.N;
  auto mk_map = [&](CUtensorMap* mp, const void* base) {
    if (prm.box8) return make_square_map(mp, base, batch, pat.H, pat.W, heads, head_dim);
    return pl->gather ? make_gather_map(mp, base, tok, heads, head_dim)
                      : make_rows_map(mp, base, tok, heads, head_dim, kBlock);
  };
  if ((st = mk_map(&pl->mq, q)) != HLA_OK) return st;
  if ((st = mk_map(&pl->mk, k)) != HLA_OK) return st;
  if ((st = mk_map(&pl->mv, v)) != HLA_OK) return st;
  if ((st = mk_map(&pl->mdo, dout)) != HLA_OK) return st;
  // fp32 dQ accumulator, sequence order, 32-float (128 B) boxes for the TMA reduce-add
  if ((st = make_f32_rows_map(&pl->mdq, dq_acc, tok, heads, head_dim, 32, kBlock)) != HLA_OK) return st;
  pl->two_d = pat.kind == K_WSA || pat.kind == K_SA || pat.kind == K_NA2D;
  pl->mkb = (pat.N + kBlock - 1) / kBlock;
  pl->head_dim = head_dim;
  // schedule: full-tile (attn_bwd_full_kernel) when full tiles are at least half of the
  // mask's tiles; half-tile (attn_bwd_split_kernel) otherwise (the split
  // schedule overlaps the partial tiles' masked compute better) and with the global RPB (only
  // the half-tile schedule has the dRPB window: at the previous tile's scale, no extra barrier)
  pl->full = full_schedule(prm.rpb != nullptr, lists);
  pl->fuse = false;
  pl->zero_acc = false;
  return HLA_OK;
}

// hla_attn_bwd: fold the preprocess into the main kernel (no global RPB) when every q-block's
// dQ chain is local (either schedule: the kernel's dq_stage then holds O tiles instead of dQ
// partials, and the accumulator is never touched), or with the half-tile schedule for any plan
// (its dQ reduce-adds are then staged in 16-column quarters through the epi_stage; the
// accumulator rows of non-local q-blocks are zeroed by dq_zero_kernel, a pure write).  The main
// kernel reads the raw LSE and O; no preprocess launch.
// Non-local masks are folded only with the block-64 window lists: measured (DESIGN 6g) cfg4 @ b64
// 1.634 -> 1.549 ms, but cfg4 @ b128 1.913 -> 1.961 and cfg3 0.356 -> 0.361 ms (the folded kernel
// reloads O with every stage load, and q-blocks are reloaded by several units there).
bool fusable(bool full, bool rpb, const hla_block_mask* m, int32_t n, int32_t col_mul) {
  if (rpb) return false;
  const bool all_local = plan_of(m, n) && m->n_dq_nonlocal == 0;
  return all_local || (!full && col_mul == 64);
}

hla_status try_fuse(MainPlan* pl, const hla_block_mask* m, int32_t batch, int32_t heads, const void* o,
                    const float* lse) {
  if (!fusable(pl->full, pl->prm.rpb != nullptr, m, pl->prm.N, pl->prm.col_mul)) return HLA_OK;
  const bool all_local = plan_of(m, pl->prm.N) && m->n_dq_nonlocal == 0;
  const int64_t tok = (int64_t)batch * pl->prm.N;
  CUtensorMap* om = pl->full ? &pl->mdq : &pl->mo;   // (the full-tile kernel takes O in the dQ slot)
  hla_status st = pl->prm.box8 ? make_square_map(om, o, batch, pl->prm.pat.H, pl->prm.pat.W, heads, pl->head_dim)
                 : pl->gather ? make_gather_map(om, o, tok, heads, pl->head_dim)
                             : make_rows_map(om, o, tok, heads, pl->head_dim, kBlock);
  if (st != HLA_OK) return st;
  if (!pl->full && !all_local &&
      (st = make_f32_rows_map(&pl->mdq, pl->prm.dq_acc, tok, heads, pl->head_dim, 16, kBlock)) != HLA_OK)
    return st;
  pl->prm.lse2 = lse;
  pl->prm.dsum = nullptr;
  pl->fuse = true;
  pl->zero_acc = !all_local;
  return HLA_OK;
}

hla_status launch_main(const MainPlan& pl, cudaStream_t stream) {
  const bool bias = pl.prm.rpb != nullptr;
  if (pl.full)
    return bwd::launch_full(pl.head_dim, pl.gather, pl.two_d, pl.fuse, pl.mq, pl.mk, pl.mv, pl.mdo, pl.mdq, pl.prm,
                            pl.mkb, stream);
  return bwd::launch_split(bias, pl.head_dim, pl.gather, pl.two_d, pl.fuse, pl.mq, pl.mk, pl.mv, pl.mdo, pl.mdq,
                           pl.fuse ? pl.mo : pl.mdq, pl.prm, pl.mkb, stream);
}

}  // namespace

extern "C" hla_status hla_attn_bwd_main(const hla_pattern_desc* d, const hla_block_mask* m, int32_t batch,
                                        int32_t heads, int32_t head_dim, float scale, const void* q, const void* k,
                                        const void* v, const void* dout, void* dq, void* dk, void* dv,
                                        const int32_t* seq_to_cell, const hla_score_mod* score_mod,
                                        void* workspace, size_t workspace_bytes, int64_t* tiles_visited,
                                        cudaStream_t stream) {
  clear_error();
  MainPlan pl;
  const hla_status st = prepare_main(d, m, batch, heads, head_dim, scale, q, k, v, dout, dq, dk, dv, seq_to_cell,
                                     score_mod, workspace, workspace_bytes, tiles_visited, &pl);
  if (st != HLA_OK) return st;
  return launch_main(pl, stream);
}

extern "C" hla_status hla_attn_bwd_finalize(int32_t batch, int32_t heads, int32_t n, int32_t head_dim,
                                            const void* workspace, size_t workspace_bytes, void* dq,
                                            const int32_t* seq_to_cell, const hla_block_mask* plan_mask,
                                            cudaStream_t stream) {
  clear_error();
  HLA_REQUIRE(head_dim == 32 || head_dim == 64, HLA_ERR_UNSUPPORTED, "head_dim %d not in {32, 64}", head_dim);
  HLA_REQUIRE(dq && (uintptr_t)dq % 16 == 0, HLA_ERR_INVALID, "dq null or unaligned");
  float *dq_acc, *dsum;
  hla_status st = carve_workspace(batch, heads, n, head_dim, const_cast<void*>(workspace), workspace_bytes, &dq_acc,
                                  &dsum);
  if (st != HLA_OK) return st;
  const int64_t n_v = (int64_t)batch * n * heads * head_dim / 8;
  HLA_REQUIRE(n_v < (1ll << 31), HLA_ERR_UNSUPPORTED, "B * N * heads * head_dim too large");
  const uint8_t* q_local = plan_of(plan_mask, n);
  if (q_local && plan_mask->n_dq_nonlocal == 0) return HLA_OK;   // every dQ row written by the main kernel
  const unsigned blocks = (unsigned)((n_v + 255) / 256);
  dq_finalize_kernel<<<blocks, 256, 0, stream>>>(reinterpret_cast<const float4*>(dq_acc),
                                                 reinterpret_cast<uint4*>(dq), seq_to_cell, q_local, make_fastdiv(n),
                                                 make_fastdiv(heads * head_dim / 8), (int32_t)n_v);
  HLA_CUDA_TRY(cudaGetLastError());
  return HLA_OK;
}

extern "C" int32_t hla_attn_bwd_fuses_preprocess(const hla_pattern_desc* d, const hla_block_mask* m,
                                                 const hla_score_mod* score_mod) {
  Pattern pat;
  AttnLists lists;
  if (!d || !m || check_attn_args(d, m, 1, 1, 64, &pat, &lists) != HLA_OK) {
    clear_error();
    return 0;
  }
  const float* rpb = nullptr;
  float* drpb = nullptr;
  const int32_t* cells = nullptr;
  if (parse_score_mod(d, score_mod, true, &rpb, &drpb, &cells) != HLA_OK) {
    clear_error();
    return 0;
  }
  return fusable(full_schedule(rpb != nullptr, lists), rpb != nullptr, m, pat.N, lists.col_mul) ? 1 : 0;
}

extern "C" hla_status hla_attn_bwd(const hla_pattern_desc* d, const hla_block_mask* m, int32_t batch, int32_t heads,
                                   int32_t head_dim, float scale, const void* q, const void* k, const void* v,
                                   const void* o, const float* lse, const void* dout, void* dq, void* dk, void* dv,
                                   const int32_t* seq_to_cell, const hla_score_mod* score_mod, void* workspace,
                                   size_t workspace_bytes, int64_t* tiles_visited, cudaStream_t stream) {
  clear_error();
  // validate every stage's arguments (and build the main kernel's tensor maps) before
  // launching anything: a rejected call leaves drpb and the workspace untouched
  MainPlan pl;
  hla_status st = prepare_main(d, m, batch, heads, head_dim, scale, q, k, v, dout, dq, dk, dv, seq_to_cell,
                               score_mod, workspace, workspace_bytes, tiles_visited, &pl);
  if (st != HLA_OK) return st;
  HLA_REQUIRE(o && dq && lse, HLA_ERR_INVALID, "null pointer");
  HLA_REQUIRE(((uintptr_t)o | (uintptr_t)dq) % 16 == 0, HLA_ERR_INVALID, "tensors must be 16-byte aligned");
  HLA_REQUIRE((int64_t)batch * pl.prm.N * heads * head_dim / 8 < (1ll << 31), HLA_ERR_UNSUPPORTED,
              "B * N * heads * head_dim too large");
  if ((st = try_fuse(&pl, m, batch, heads, o, lse)) != HLA_OK) return st;
  if (pl.fuse) {   // D / LSE formed in the kernel
    if (pl.zero_acc) {   // non-local chains reduce into the accumulator: zero their rows first
      const int64_t n_v = (int64_t)batch * pl.prm.N * heads * head_dim / 8;
      dq_zero_kernel<<<(unsigned)((n_v + 255) / 256), 256, 0, stream>>>(
          reinterpret_cast<float4*>(pl.prm.dq_acc), plan_of(m, pl.prm.N), make_fastdiv(pl.prm.N),
          make_fastdiv(heads * head_dim / 8), (int32_t)n_v);
      HLA_CUDA_TRY(cudaGetLastError());
    }
    if ((st = launch_main(pl, stream)) != HLA_OK) return st;
    if (!pl.zero_acc) return HLA_OK;   // every dQ row written by the main kernel
    return hla_attn_bwd_finalize(batch, heads, pl.prm.N, head_dim, workspace, workspace_bytes, dq, seq_to_cell, m,
                                 stream);
  }
  if (pl.prm.drpb)   // the table gradient is accumulated: start from zero
    HLA_CUDA_TRY(cudaMemsetAsync(pl.prm.drpb, 0,
                                 sizeof(float) * heads * (2 * pl.prm.grid_h - 1) * (2 * pl.prm.grid_w - 1), stream));
  if ((st = hla_attn_bwd_preprocess(batch, heads, pl.prm.N, head_dim, scale, o, dout, lse, seq_to_cell, m, workspace,
                                    workspace_bytes, stream)) != HLA_OK)
    return st;
  if ((st = launch_main(pl, stream)) != HLA_OK) return st;
  return hla_attn_bwd_finalize(batch, heads, pl.prm.N, head_dim, workspace, workspace_bytes, dq, seq_to_cell, m,
                               stream);
}
