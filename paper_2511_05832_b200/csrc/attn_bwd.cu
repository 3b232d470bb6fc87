// K7-K9: block-sparse attention backward on sm_100a (tcgen05 + TMEM + TMA).
//
// Gradients of masked softmax attention (the paper times this pass in the
// "Backward" columns; skipping empty tiles is what makes it
// cheaper):
//   P = exp(scale S - LSE) (0 where masked),  D = rowsum(dO o O)
//   dV = P^T dO,  dS = scale P o (dO V^T - D),  dK = dS^T Q,  dQ = dS K.
//
// K7 bwd_preprocess : D = rowsum(dO o O) (fp32) and zero the fp32 dQ accumulator.
// K8 attn_bwd_kernel: one CTA per (kv-block j, head, batch), walking the
//    transposed CSR list of q-blocks i (ascending).  320 threads, 1 CTA / SM:
//    warp 0     TMA: K_j, V_j once; per q-block Q_i, dO_i (+ LSE_i, D_i via bulk
//               copy) into a 2-stage ring;
//    warp 1     TMEM allocator + single-thread tcgen05.mma issuer:
//                 S^T  = K_j Q_i^T     (SS, TMEM cols [0,128))
//                 dP^T = V_j dO_i^T    (SS, TMEM cols [128,256))
//                 dV  += P^T dO_i      (TS, P^T bf16 written over the first 16 columns of
//                                       each 32-column S^T chunk; acc [384,448))
//                 dK  += dS^T Q_i      (SS, dS^T bf16 in smem, K-major view; acc [448,512))
//                 dQ_i (+)= dS K_j     (SS, same dS smem, MN-major view; two accumulators
//                                       [256,320) / [320,384) chained by the mask's dQ plan)
//    warps 2-9  thread = key row (two warps per TMEM lane quarter, one 32-column
//               chunk each): P^T, dS^T from S^T, dP^T (mask only on partial
//               tiles); final dK (warps 6-9), dV (warps 2-5) -> bf16;
//    warps 10-13 thread = query row: at the end of a dQ chain, dQ_i -> bf16 dq rows
//               (complete chains) or -> smem -> TMA reduce-add into the fp32
//               accumulator (overlaps the next q-block's MMAs).
// K9 dq_finalize    : fp32 accumulator -> bf16 dQ.
#include "predicates.cuh"
#include "sm100.cuh"
#include "tensor_map.cuh"

namespace hla {
namespace {

constexpr int kBlock = 128;
constexpr int kThreads = 512;   // 16 warps: TMA, MMA, 8 x P/dS, 4 x dQ, 2 x TMA
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColS = 0, kColDP = 128, kColDQ = 256, kColDV = 384, kColDK = 448;   // dQ: 2 x 64 columns
constexpr float kLog2e = 1.4426950408889634f;
constexpr int kHalf = 64;   // q-columns per pipeline half

struct BwdParams {
  Pattern pat;
  int32_t N, heads, batch;
  float scale, scale_log2, inv_scale;
  const int32_t* t_row_ptr;
  const int32_t* t_col_idx;
  const uint8_t* t_kind;
  const uint8_t* t_dq;     // dQ chaining plan per transposed entry (HLA_DQ_*; null = one chain per tile)
  const float* lse2;       // LSE * log2(e), [B, H, N] (workspace, from the preprocess)
  const float* dsum;       // D * scale, [B, H, N] (workspace, from the preprocess)
  float* dq_acc;           // [B, N, H, Dh] fp32 (grid order when s2c != null)
  const int32_t* s2c;      // fused reorder: seq_to_cell table (tensors in grid order), else null
  const float* rpb;        // global RPB table [heads][2H-1][2W-1] (kBias)
  float* drpb;             // its gradient (accumulated)
  const int32_t* cells;    // grid cell of each sequence position (null: identity)
  int32_t grid_h, grid_w, rpb_w, rpb_hw;
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
  __nv_bfloat16* dq;       // dQ rows of LOCAL chains (bf16, same layout as dk)
  unsigned long long* visited;
};

// entries of the per-tile dRPB window (offset rows of the tile's box, full table row stride
// 2W - 1) in shared memory; more at D = 32, where the smaller tiles leave room
template <int D>
constexpr int rpb_win_cap() { return D == 32 ? 4096 : 2048; }
// The window accumulates in 32-bit fixed point: shared-memory fp32 atomics are
// compare-and-swap loops on sm_100 (ATOMS.CAST.SPIN, measured in SASS) while
// integer ATOMS.ADD is native.  Resolution 2^-16 (absolute; dS values are
// O(1e-2..1)), each addend saturated at +-2^14 so a tile's sum per offset (at most
// 128 pairs) cannot overflow; converted back to fp32 when the window is flushed.
constexpr float kRpbFix = 65536.f;

template <int D, bool kBias = false>
struct BwdSmem {
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
  uint64_t kv_full[2], kv_empty[2], q_full[2], q_empty[2], s_full[2], ds_ready[2], dq_full[2], dq_free[2], dkv_full,
      epi_done;
  uint64_t dbg_bar;
  uint32_t tmem_base;
  int32_t rpb_win[kBias ? rpb_win_cap<D>() : 1];   // dRPB of the current tile's offset box, fixed point (compute warps)
};

template <int D>
__device__ __forceinline__ uint64_t kmajor_desc(const uint8_t* tile, int kstep) {
  constexpr uint32_t layout = D == 64 ? sm100::kSwizzle128B : sm100::kSwizzle64B;
  return sm100::make_smem_desc(sm100::smem_u32(tile) + kstep * 32, 16, 8 * D * 2, layout);
}
template <int D>
__device__ __forceinline__ uint64_t mnmajor_desc(const uint8_t* tile, int kstep) {
  constexpr uint32_t layout = D == 64 ? sm100::kSwizzle128B : sm100::kSwizzle64B;
  return sm100::make_smem_desc(sm100::smem_u32(tile) + kstep * 16 * D * 2, kBlock * D * 2, 8 * D * 2, layout);
}
// dS^T smem tile viewed as K-major A (M = kv, K = q): K step = 16 q
__device__ __forceinline__ uint64_t ds_kmajor_desc(const uint8_t* ds, int kstep) {
  return sm100::make_smem_desc(sm100::smem_u32(ds) + (kstep >> 2) * 16384 + (kstep & 3) * 32, 16, 1024,
                               sm100::kSwizzle128B);
}
// dS^T smem tile viewed as MN-major A of dQ = dS K (M = q, K = kv): K step = 16 kv rows
__device__ __forceinline__ uint64_t ds_mnmajor_desc(const uint8_t* ds, int kstep) {
  return sm100::make_smem_desc(sm100::smem_u32(ds) + kstep * 2048, 16384, 1024, sm100::kSwizzle128B);
}

// Work units are pairs (2p, 2p+1) of kv-blocks of one (b, h) -- the unit of the dQ
// plan (hla_build_bwd_plan) -- strided over the grid.  Consecutive kv-blocks share
// q-blocks (the producer then skips reloading a Q/dO stage, and dQ partials chain in
// TMEM), while all CTAs stay on nearby units (L2 reuse).
constexpr int32_t kUnitEnd = 0x7fffffff, kUnitSkip = -1;
struct UnitGeom {
  int32_t mk, ppb, pairs;   // kv-blocks per (b, h), pairs per (b, h), pairs in total
};
// k-th kv-block of this CTA: flattened u = (b * heads + h) * mk + kb, kUnitSkip for
// the missing second block of a ragged last pair, kUnitEnd past the last pair
__device__ __forceinline__ int32_t unit_at(int32_t k, const UnitGeom& ug) {
  const int32_t P = (int32_t)blockIdx.x + (k >> 1) * (int32_t)gridDim.x;
  if (P >= ug.pairs) return kUnitEnd;
  const int32_t bh = P / ug.ppb;
  const int32_t kb = 2 * (P - bh * ug.ppb) + (k & 1);
  return kb < ug.mk ? bh * ug.mk + kb : kUnitSkip;
}

// Iterator over the flattened (work unit, q-block tile) sequence of this CTA,
// skipping units without tiles.  n = ordinal of the current non-empty unit.
struct TileIter {
  int32_t k, u, t, nt, rs;
  uint32_t n;
  bool valid;
  __device__ void seek(const int32_t* t_row_ptr, const UnitGeom& ug) {
    for (;; ++k) {
      u = unit_at(k, ug);
      if (u == kUnitEnd) break;
      if (u < 0) continue;
      const int32_t kb = u % ug.mk;
      rs = __ldg(t_row_ptr + kb);
      nt = __ldg(t_row_ptr + kb + 1) - rs;
      if (nt > 0) { valid = true; return; }
    }
    valid = false;
  }
  __device__ void init(const int32_t* t_row_ptr, const UnitGeom& ug) {
    k = 0; t = 0; n = 0;
    seek(t_row_ptr, ug);
  }
  __device__ void advance(const int32_t* t_row_ptr, const UnitGeom& ug) {
    if (++t < nt) return;
    t = 0; ++n; ++k;
    seek(t_row_ptr, ug);
  }
};

// dQ plan bits of the g-th tile (transposed entry e); without a plan every tile is
// its own chain, alternating between the two accumulators
__device__ __forceinline__ uint32_t dq_plan(const uint8_t* t_dq, int32_t e, uint32_t g) {
  return t_dq ? (uint32_t)__ldg(t_dq + e) : ((g & 1u) | HLA_DQ_NEW | HLA_DQ_DRAIN);
}

// Load the 128 token rows [seq0, seq0 + 128) (sequence order) of head h, batch b;
// see attn_fwd.cu load_rows (kGather = fused reorder through s2c with .tile::gather4).
template <int D, bool kGather>
__device__ __forceinline__ void load_rows(uint8_t* dst, const CUtensorMap* map, uint64_t* bar, int32_t h,
                                          int32_t b, int32_t N, int32_t seq0, const int32_t* s2c, uint64_t pol,
                                          int lane) {
  if (kGather) {
    // rows past N (ragged last tile) gather cell 0: their values are masked / discarded
    const int4 c = seq0 + 4 * lane < N ? __ldg(reinterpret_cast<const int4*>(s2c + seq0) + lane) : make_int4(0, 0, 0, 0);
    const int32_t base = b * N;
    sm100::tma_gather4(dst + lane * 4 * D * 2, map, bar, h * D, base + c.x, base + c.y, base + c.z, base + c.w, pol);
  } else if (lane == 0) {
    sm100::tma_load_3d(dst, map, bar, 0, h, b * N + seq0, pol);
  }
}

__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

// Persistent: CTA c processes kv-block work units c, c + G, ... (unit = kv-block,
// head, batch; kv-block fastest).  K/V are double-buffered across units, so the
// next unit's K/V (and first Q/dO) stream in while the current unit computes;
// the dK/dV epilogue of a unit overlaps the first S/dP MMAs of the next one.
// Phase counters: n = units with nt > 0 so far, g = (q-block) tiles so far.
// cell -> (row << 16) | col (RPB offsets; grid sides < 2^15)
__device__ __forceinline__ int32_t rpb_cell_rc(const int32_t* cells, int32_t seq, int32_t N, int32_t W) {
  const int32_t cell = seq < N ? (cells ? __ldg(cells + seq) : seq) : 0;
  const int32_t r = cell / W;
  return (r << 16) | (cell - r * W);
}
// min / max of the rows and columns of the cells of sequence block [s0, s0 + 128)
// (phantom positions >= N ignored); identical in every lane.
struct CellBox { int32_t r0, r1, c0, c1; };
__device__ __forceinline__ CellBox rpb_block_box(const int32_t* cells, int32_t s0, int32_t N, int32_t W, int lane) {
  CellBox bx{1 << 30, -(1 << 30), 1 << 30, -(1 << 30)};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int32_t sq = s0 + 32 * j + lane;
    if (sq < N) {
      const int32_t rc = rpb_cell_rc(cells, sq, N, W);
      const int32_t r = rc >> 16, c = rc & 0xffff;
      bx.r0 = min(bx.r0, r); bx.r1 = max(bx.r1, r); bx.c0 = min(bx.c0, c); bx.c1 = max(bx.c1, c);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    bx.r0 = min(bx.r0, __shfl_xor_sync(0xffffffffu, bx.r0, o));
    bx.r1 = max(bx.r1, __shfl_xor_sync(0xffffffffu, bx.r1, o));
    bx.c0 = min(bx.c0, __shfl_xor_sync(0xffffffffu, bx.c0, o));
    bx.c1 = max(bx.c1, __shfl_xor_sync(0xffffffffu, bx.c1, o));
  }
  return bx;
}

template <int D, bool kTwoD, bool kGather, bool kBias>
__global__ void __launch_bounds__(kThreads, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                    const __grid_constant__ CUtensorMap tmDQ, const BwdParams prm) {
  extern __shared__ uint8_t smem_raw[];
  using Smem = BwdSmem<D, kBias>;
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  UnitGeom ug;
  ug.mk = (prm.N + kBlock - 1) / kBlock;   // last kv-block may be ragged
  ug.ppb = (ug.mk + 1) / 2;
  ug.pairs = ug.ppb * prm.heads * prm.batch;
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
    sm100::mbar_init(&sm.dbg_bar, 1);
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
  HLA_TR_DECL;

  if (warp == 0 || warp >= 14) {
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
      uint32_t n = 0, g = 0;
      int64_t stage_tag0 = -1, stage_tag1 = -1;   // (b, h, q-block) held by stage 0 / 1
      for (int32_t kq = 0;; ++kq) {
        const int32_t u = unit_at(kq, ug);
        if (u == kUnitEnd) break;
        if (u < 0) continue;
        const int32_t kb = u % mk, h = (u / mk) % prm.heads, b = u / (mk * prm.heads);
        const int32_t rs = __ldg(prm.t_row_ptr + kb), nt = __ldg(prm.t_row_ptr + kb + 1) - rs;
        if (nt == 0) continue;
        const int64_t bh = (int64_t)b * prm.heads + h;
        const int kvs = n & 1;
        if (role < 2) {
          if (n >= 2) sm100::mbar_wait(&sm.kv_empty[kvs], ((n >> 1) - 1) & 1);
          if (lane == 0) HLA_TR((3 << 24) | ((1) << 16) | (n));
          if (lane == 0) sm100::mbar_arrive_expect_tx(&sm.kv_full[kvs], kTile);
          __syncwarp();
          load_rows<D, kGather>(role == 0 ? sm.k[kvs] : sm.v[kvs], role == 0 ? &tmK : &tmV, &sm.kv_full[kvs], h, b,
                                prm.N, kb * kBlock, prm.s2c, pol_kv, lane);
        }
        for (int t = 0; t < nt; ++t, ++g) {
          const int s = g & 1;
          if (g >= 2) sm100::mbar_wait(&sm.q_empty[s], ((g >> 1) - 1) & 1);
          if (lane == 0 && role == 1) HLA_TR((7 << 24) | ((2) << 16) | (g));
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
              const int4 rc = make_int4(rpb_cell_rc(prm.cells, qblk * kBlock + 4 * lane, prm.N, prm.grid_w),
                                        rpb_cell_rc(prm.cells, qblk * kBlock + 4 * lane + 1, prm.N, prm.grid_w),
                                        rpb_cell_rc(prm.cells, qblk * kBlock + 4 * lane + 2, prm.N, prm.grid_w),
                                        rpb_cell_rc(prm.cells, qblk * kBlock + 4 * lane + 3, prm.N, prm.grid_w));
              const int32_t a0 = (prm.grid_h - 1) * prm.rpb_w + prm.grid_w - 1;
              auto a_of = [&](int32_t v) { return a0 + (v >> 16) * prm.rpb_w + (v & 0xffff); };
              sm100::sts_u4(sm100::smem_u32(sm.qa[s]) + 16u * lane, a_of(rc.x), a_of(rc.y), a_of(rc.z), a_of(rc.w));
              __syncwarp();   // every lane's A_q is written before lane 0 arrives on q_full
            }
            if (lane == 0) {
              // LSE / D of the real rows only (ragged last tile: N % 4 == 0, so 16-B multiples)
              const uint32_t vbytes = (uint32_t)min(kBlock, prm.N - qblk * kBlock) * 4u;
              sm100::mbar_arrive_expect_tx(&sm.q_full[s], 2 * vbytes);
              sm100::bulk_load(sm.lse[s], prm.lse2 + bh * prm.N + qblk * kBlock, vbytes, &sm.q_full[s]);
              sm100::bulk_load(sm.dd[s], prm.dsum + bh * prm.N + qblk * kBlock, vbytes, &sm.q_full[s]);
            }
          } else {
            if (lane == 0) sm100::mbar_arrive_expect_tx(&sm.q_full[s], kTile);
            __syncwarp();
            load_rows<D, kGather>(role == 1 ? sm.q[s] : sm.dO[s], role == 1 ? &tmQ : &tmDO, &sm.q_full[s], h, b,
                                  prm.N, qblk * kBlock, prm.s2c, pol_q, lane);
          }
        }
        ++n;
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer
    // Half-tile software pipeline over the flattened (unit, q-block) sequence:
    //   S_A,dP_A(g) S_B,dP_B(g) | dV_A dK_A(g) S_A,dP_A(g+1) | dV_B dK_B dQ(g) S_B,dP_B(g+1) | ...
    // so the tensor core works on one q-half while the compute warps process the other.
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
        for (int kk = 0; kk < D / 16; ++kk)
          sm100::mma_ss(tmem + kColS + half * kHalf, kmajor_desc<D>(sk, kk), kmajor_desc<D>(sm.q[s] + qoff, kk),
                        idesc_h, kk > 0);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          sm100::mma_ss(tmem + kColDP + half * kHalf, kmajor_desc<D>(sv, kk), kmajor_desc<D>(sm.dO[s] + qoff, kk),
                        idesc_h, kk > 0);
        sm100::mma_commit(&sm.s_full[half]);
      };
      auto issue_dvdk = [&](uint32_t gg, int half, bool first_tile) {
        const int s = gg & 1;
        const uint8_t* ds = sm.ds[gg & 1];
#pragma unroll
        for (int kk = half * 4; kk < half * 4 + 4; ++kk) {
          const uint32_t acc = (!first_tile || kk > 0) ? 1u : 0u;
          // P^T of q-columns [16kk, 16kk + 16): 8 packed columns at the start of S^T chunk kk/2
          sm100::mma_ts(tDV, tmem + kColS + (kk >> 1) * 32 + (kk & 1) * 8, mnmajor_desc<D>(sm.dO[s], kk), idesc_kv,
                        acc);
          sm100::mma_ss(tDK, ds_kmajor_desc(ds, kk), mnmajor_desc<D>(sm.q[s], kk), idesc_kv, acc);
        }
      };
#if defined(HLA_TRACE) && defined(HLA_TRACE_MMA)
      uint32_t dbg_phase = 0;
      // trace builds: serialise after each MMA group and record its tensor-core time
      auto mma_probe = [&](int ev, uint32_t gg) {
        sm100::mma_commit(&sm.dbg_bar);
        sm100::mbar_wait(&sm.dbg_bar, dbg_phase);
        dbg_phase ^= 1;
        HLA_TR((5 << 24) | (ev << 16) | gg);
      };
#else
      auto mma_probe = [](int, uint32_t) {};
#endif
      if (cur.valid) {
        sm100::mbar_wait(&sm.kv_full[cur.n & 1], (cur.n >> 1) & 1);
        sm100::mbar_wait(&sm.q_full[0], 0);
        sm100::tc_fence_after();
        issue_sdp(cur, 0, 0);
        issue_sdp(cur, 0, 1);
      }
      while (cur.valid) {
        TileIter nxt = cur;
        nxt.advance(prm.t_row_ptr, ug);
        const uint32_t fdq = dq_plan(prm.t_dq, cur.rs + cur.t, g);
        const int kvs = cur.n & 1;
        const bool last_of_unit = cur.t == cur.nt - 1;
        // half A of tile g
        sm100::mbar_wait(&sm.ds_ready[0], g & 1);
        HLA_TR((1 << 24) | ((1) << 16) | (g));
        sm100::tc_fence_after();
        HLA_TR((5 << 24) | (0 << 16) | g);
        if (cur.t == 0 && cur.n > 0) {
          // the previous unit's dV / dK must have been drained from TMEM
          sm100::mbar_wait(&sm.epi_done, (cur.n - 1) & 1);
          sm100::tc_fence_after();
        }
        issue_dvdk(g, 0, cur.t == 0);
        mma_probe(1, g);
        // S_A / dP_A of the next tile now if its operands already landed (never block
        // here: the B half of this tile must not wait behind the next tile's loads)
        bool next_a_issued = false;
        if (nxt.valid && (nxt.t != 0 || sm100::mbar_test_wait(&sm.kv_full[nxt.n & 1], (nxt.n >> 1) & 1)) &&
            sm100::mbar_test_wait(&sm.q_full[(g + 1) & 1], ((g + 1) >> 1) & 1)) {
          HLA_TR((1 << 24) | ((4) << 16) | (g));
          sm100::tc_fence_after();
          issue_sdp(nxt, g + 1, 0);
          next_a_issued = true;
        }
        // half B of tile g, then dQ (needs both halves of dS)
        sm100::mbar_wait(&sm.ds_ready[1], g & 1);
        HLA_TR((1 << 24) | ((2) << 16) | (g));
        sm100::tc_fence_after();
        HLA_TR((5 << 24) | (0 << 16) | g);
        issue_dvdk(g, 1, false);
        mma_probe(3, g);
        sm100::mma_commit(&sm.q_empty[g & 1]);   // Q_g / dO_g no longer read (dQ needs only dS and K)
        if (last_of_unit) sm100::mma_commit(&sm.dkv_full);
        const int dqb = (int)(fdq & HLA_DQ_BUF);
        const bool dq_new = (fdq & HLA_DQ_NEW) != 0;
        if (dq_new) {
          // a new chain: the accumulator's previous chain must have been drained
          const uint32_t c = dqb ? dq_started1++ : dq_started0++;
          if (c > 0) {
            sm100::mbar_wait(&sm.dq_free[dqb], (c - 1) & 1);
            HLA_TR((1 << 24) | ((3) << 16) | (g));
            sm100::tc_fence_after();
          }
        }
#pragma unroll
        for (int kk = 0; kk < kBlock / 16; ++kk)
          sm100::mma_ss(tDQ + dqb * 64, ds_mnmajor_desc(sm.ds[g & 1], kk), mnmajor_desc<D>(sm.k[kvs], kk), idesc_q,
                        (kk > 0 || !dq_new) ? 1u : 0u);
        mma_probe(4, g);
        if (fdq & HLA_DQ_DRAIN) sm100::mma_commit(&sm.dq_full[dqb]);
        if (last_of_unit) sm100::mma_commit(&sm.kv_empty[kvs]);
        if (nxt.valid) {
          if (!next_a_issued) {
            if (nxt.t == 0) sm100::mbar_wait(&sm.kv_full[nxt.n & 1], (nxt.n >> 1) & 1);
            sm100::mbar_wait(&sm.q_full[(g + 1) & 1], ((g + 1) >> 1) & 1);
            HLA_TR((1 << 24) | ((4) << 16) | (g));
            sm100::tc_fence_after();
            issue_sdp(nxt, g + 1, 0);
          }
          HLA_TR((5 << 24) | (0 << 16) | g);
          issue_sdp(nxt, g + 1, 1);
          mma_probe(5, g);
        }
        cur = nxt;
        ++g;
      }
    }
  } else if (warp < 10) {
    // --------------------------------------------- P^T / dS^T (thread = key row)
    // two warp sets (cset 0: warps 2-5, cset 1: warps 6-9) share every TMEM lane
    // quarter; within each q-half, cset c processes the 32-column chunk 2*half + c.
    const int quarter = warp & 3;
    const int cset = (warp - 2) >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const float sl2 = prm.scale_log2, scale = prm.scale;
    if (kBias) {   // the dRPB window starts (and is left after every flush) zeroed
      for (int i = (warp - 2) * 32 + lane; i < rpb_win_cap<D>(); i += 256) sm.rpb_win[i] = 0;
      sm100::named_bar_sync(3, 256);
    }
    uint32_t n = 0, g = 0;
    for (int32_t kq = 0;; ++kq) {
      const int32_t u = unit_at(kq, ug);
      if (u == kUnitEnd) break;
      if (u < 0) continue;
      const int32_t kb = u % mk, h = (u / mk) % prm.heads, b = u / (mk * prm.heads);
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
        const int32_t rc = rpb_cell_rc(prm.cells, kidx, prm.N, prm.grid_w);
        k_r = rc >> 16;
        k_c = rc & 0xffff;
        k_b = k_r * prm.rpb_w + k_c;
        kbox = rpb_block_box(prm.cells, kb * kBlock, prm.N, prm.grid_w, lane);
        rpbh = prm.rpb + (int64_t)h * prm.rpb_hw;
        drpbh = prm.drpb + (int64_t)h * prm.rpb_hw;
      }
      for (int t = 0; t < nt; ++t, ++g) {
        const int s = g & 1;
        const uint8_t kd = __ldg(prm.t_kind + rs + t);
        const int32_t q0 = __ldg(prm.t_col_idx + rs + t) * kBlock;
        // RPB: the tile's offset box (dr, dc) = q box - key box and whether its rows fit
        // the shared-memory dRPB window (query offsets A_q come staged with LSE / D)
        int32_t dr0 = 0, dc0 = 0, wc = 0, wrows = 0, wcols = 0, kwb = 0;
        bool win = false;
        if (kBias) {
          const CellBox qbox = rpb_block_box(prm.cells, q0, prm.N, prm.grid_w, lane);
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
        sm100::mbar_wait(&sm.q_full[s], (g >> 1) & 1);
        if (row == 0 && cset == 0) HLA_TR((2 << 24) | ((1) << 16) | (g));
        const uint32_t lse2 = sm100::smem_u32(sm.lse[s]);
        const uint32_t dd = sm100::smem_u32(sm.dd[s]);
        const uint32_t qa = sm100::smem_u32(sm.qa[s]);
        const uint32_t dsbuf = sm100::smem_u32(sm.ds[g & 1]);
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
          sm100::mbar_wait(&sm.s_full[half], g & 1);
          if (row == 0 && cset == 0) HLA_TR((2 << 24) | ((2 + 2 * half) << 16) | (g));
          sm100::tc_fence_after();
          {
            const int c = 2 * half + cset;
            uint32_t sr[32], dpr[32];
            sm100::tmem_ld32(tmem + lane_off + kColS + c * 32, sr);
            sm100::tmem_ld32(tmem + lane_off + kColDP + c * 32, dpr);
            sm100::tmem_wait_ld();
            // [ulo, uhi): 8-column groups of this chunk that hold an allowed query of some
            // key row of this warp (partial tiles of 1D patterns: each key row's queries are
            // one interval); the other groups are all masked, their exponentials skipped
            // (warp-uniform) and P = 0 there.  Full tiles / 2D patterns: all 4 groups.
            int ulo = 0, uhi = 4;
            if (!kBias && kd == 2 && !kTwoD) {   // (with the RPB gather the branchy loop measured slower: cfg5 +6%)
              const int32_t base = q0 + c * 32;
              const int32_t lo = min(max(box.lo - base, 0), 32), hi = min(max(box.lo + box.len - base, 0), 32);
              const bool any = hi > lo;
              ulo = __reduce_min_sync(0xffffffffu, any ? lo : 32) >> 3;
              uhi = (__reduce_max_sync(0xffffffffu, any ? hi : 0) + 7) >> 3;
            }
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
            if (kd == 2) {
#pragma unroll
              for (int e = 0; e < 32; ++e) {
                const int32_t qq = q0 + c * 32 + e;
                bool ok;
                if (!kTwoD) {
                  ok = (uint32_t)(qq - box.lo) < (uint32_t)box.len;
                } else {
                  const int32_t rq = prm.pat.log2W >= 0 ? (qq >> prm.pat.log2W) : qq / prm.pat.W;
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
                const uint32_t wbase = sm100::smem_u32(sm.rpb_win);
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                  if (!((okbits >> (u4 * 8 + e)) & 1u)) continue;
                  const float gv = ds[e] * prm.inv_scale;
                  if (win) {   // window index (dr - dr0) * (2W - 1) + (dc - dc0) = A_q - kwb
                    const int32_t fx = __float2int_rn(fminf(fmaxf(gv, -16384.f), 16384.f) * kRpbFix);
                    asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(wbase + 4u * (uint32_t)(av[e] - kwb)), "r"(fx)
                                 : "memory");
                  } else {     // table index A_q - B_k
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
          if (row == 0 && cset == 0) HLA_TR((2 << 24) | ((3 + 2 * half) << 16) | (g));
        }
        if (kBias && win) {
          // flush the tile's dRPB window to global (and re-zero it) -- all 256 compute threads
          sm100::named_bar_sync(3, 256);
          const int tid = (warp - 2) * 32 + lane;
          for (int i = tid; i < wrows * wcols; i += 256) {   // only the box's used columns
            const int32_t ir = i / wcols, ic = i - ir * wcols;
            const int32_t v = sm.rpb_win[ir * wc + ic];
            if (v != 0) {
              atomicAdd(drpbh + (dr0 + ir + prm.grid_h - 1) * prm.rpb_w + (dc0 + ic + prm.grid_w - 1),
                        (float)v * (1.f / kRpbFix));
              sm.rpb_win[ir * wc + ic] = 0;
            }
          }
          sm100::named_bar_sync(3, 256);
        }
      }
      tiles_done += nt;
    }
  } else if (warp < 14) {
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
      const int32_t kb = u % mk, h = (u / mk) % prm.heads, b = u / (mk * prm.heads);
      const int32_t rs = __ldg(prm.t_row_ptr + kb), nt = __ldg(prm.t_row_ptr + kb + 1) - rs;
      for (int t = 0; t < nt; ++t, ++g) {
        const uint32_t fdq = dq_plan(prm.t_dq, rs + t, g);
        if (!(fdq & HLA_DQ_DRAIN)) continue;   // the chain continues in TMEM
        const int dqb = (int)(fdq & HLA_DQ_BUF);
        sm100::mbar_wait(&sm.dq_full[dqb], (dqb ? dq_drained1++ : dq_drained0++) & 1);
        if (leader) HLA_TR((4 << 24) | ((1) << 16) | (g));
        sm100::tc_fence_after();
        const int32_t qblk = __ldg(prm.t_col_idx + rs + t);
        const int32_t qrow = b * prm.N + qblk * kBlock;   // sequence order
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
          const int32_t qs = qblk * kBlock + row;
          if (qs < prm.N) {
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
        sm100::mbar_wait(&sm.dkv_full, n & 1);
        if (leader) HLA_TR((4 << 24) | ((6) << 16) | (n));
        sm100::tc_fence_after();
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
#pragma unroll
        for (int v4 = 0; v4 < D / 8 && real; ++v4) {
          dvp[v4] = make_uint4(pv[v4 * 4 + 0], pv[v4 * 4 + 1], pv[v4 * 4 + 2], pv[v4 * 4 + 3]);
          dkp[v4] = make_uint4(pk[v4 * 4 + 0], pk[v4 * 4 + 1], pk[v4 * 4 + 2], pk[v4 * 4 + 3]);
        }
        if (leader) HLA_TR((4 << 24) | ((7) << 16) | (n));
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
  }

  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (warp == 1) sm100::tmem_dealloc(tmem, kTmemCols);
  if (warp == 2 && lane == 0 && prm.visited != nullptr && tiles_done > 0) atomicAdd(prm.visited, tiles_done);
}

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
                                                             const uint8_t* __restrict__ q_local, int32_t N,
                                                             int32_t heads, int32_t rows) {
  // one thread per 8 elements (16 B of O and of dO); 32-bit index math (rows * D / 8 < 2^31).
  // Threads walk the OUTPUT order (b, h, s): D / LSE are written as contiguous runs (in
  // token order the 4-byte results of one warp land in `heads` different sectors).
  constexpr int kLanes = D / 8;   // lanes per row
  const int32_t gid = (int32_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int32_t i = gid / kLanes;             // (b * heads + h) * N + s
  const int part = gid - i * kLanes;
  if (i >= rows) return;
  const int32_t bh = i / N, s = i - bh * N;
  const int32_t bb = bh / heads, hq = bh - bb * heads;
  const int32_t r = (bb * N + s) * heads + hq;   // sequence-order row (b * N + s) * heads + h
  const int64_t src = s2c ? ((int64_t)(bb * N + __ldg(s2c + s)) * heads + hq) : (int64_t)r;
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

// K9: dQ = bf16(accumulator) -- the accumulator is in sequence order; under the
// fused reorder each row is written to its grid cell s2c[s] (SURVEY 8(a) a8:
// "dQ finalize + inverse permutation").  One thread per 8 elements (32 B in, 16 B out).
// Rows of local q-blocks (q_local: written by the main kernel) are left alone.
__global__ void __launch_bounds__(256) dq_finalize_kernel(const float4* __restrict__ acc, uint4* __restrict__ dq,
                                                          const int32_t* __restrict__ s2c,
                                                          const uint8_t* __restrict__ q_local, int32_t N,
                                                          int32_t row_v, int32_t n_v) {
  const int32_t t = (int32_t)blockIdx.x * blockDim.x + threadIdx.x;   // n_v = B * N * row_v < 2^31
  if (t >= n_v) return;
  int64_t o = t;
  if (s2c || q_local) {   // t = (b * N + s) * row_v + part, row_v = heads * D / 8
    const int32_t bs = t / row_v, part = t - bs * row_v;
    const int32_t b = bs / N, s = bs - b * N;
    if (q_local && __ldg(q_local + (s >> 7))) return;
    if (s2c) o = (int64_t)(b * N + __ldg(s2c + s)) * row_v + part;
  }
  const float4 v0 = __ldcs(acc + 2 * (int64_t)t), v1 = __ldcs(acc + 2 * (int64_t)t + 1);
  dq[o] = make_uint4(sm100::pack_bf16(v0.x, v0.y), sm100::pack_bf16(v0.z, v0.w), sm100::pack_bf16(v1.x, v1.y),
                     sm100::pack_bf16(v1.z, v1.w));
}

template <int D, bool kTwoD, bool kGather, bool kBias>
hla_status launch_bwd(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv, const CUtensorMap& mdo,
                      const CUtensorMap& mdq, const BwdParams& prm, int32_t n_kblocks, cudaStream_t stream) {
  const size_t smem = sizeof(BwdSmem<D, kBias>) + 1024;
  auto* fn = attn_bwd_kernel<D, kTwoD, kGather, kBias>;
  HLA_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t pairs = (int64_t)((n_kblocks + 1) / 2) * prm.heads * prm.batch;   // work units (kv-block pairs)
  const int grid = (int)std::min<int64_t>(pairs, (int64_t)num_sms());
  fn<<<grid, kThreads, smem, stream>>>(mq, mk, mv, mdo, mdq, prm);
  HLA_CUDA_TRY(cudaGetLastError());
  return HLA_OK;
}

static_assert(sizeof(BwdSmem<64, true>) + 1024 <= 227 * 1024, "bwd shared memory (d = 64, RPB) exceeds 227 KB");

template <bool kBias>
hla_status dispatch_bwd(int head_dim, bool gather, bool two_d, const CUtensorMap& mq, const CUtensorMap& mk,
                        const CUtensorMap& mv, const CUtensorMap& mdo, const CUtensorMap& mdq, const BwdParams& prm,
                        int32_t mkb, cudaStream_t stream) {
  if (head_dim == 64) {
    if (gather) return launch_bwd<64, false, true, kBias>(mq, mk, mv, mdo, mdq, prm, mkb, stream);
    return two_d ? launch_bwd<64, true, false, kBias>(mq, mk, mv, mdo, mdq, prm, mkb, stream)
                 : launch_bwd<64, false, false, kBias>(mq, mk, mv, mdo, mdq, prm, mkb, stream);
  }
  if (gather) return launch_bwd<32, false, true, kBias>(mq, mk, mv, mdo, mdq, prm, mkb, stream);
  return two_d ? launch_bwd<32, true, false, kBias>(mq, mk, mv, mdo, mdq, prm, mkb, stream)
               : launch_bwd<32, false, false, kBias>(mq, mk, mv, mdo, mdq, prm, mkb, stream);
}

}  // namespace
}  // namespace hla

using namespace hla;

extern "C" size_t hla_attn_bwd_workspace(int32_t batch, int32_t heads, int32_t n, int32_t head_dim) {
  const size_t acc = (size_t)batch * n * heads * head_dim * 4;
  const size_t row = (size_t)batch * heads * n * 4;
  return ((acc + 255) / 256) * 256 + 2 * ((row + 255) / 256) * 256;
}

namespace {

// q_dq_local of a mask with a complete dQ plan (else null: every q-block via the accumulator)
const uint8_t* plan_of(const hla_block_mask* m, int32_t n) {
  if (!m || !m->t_dq || !m->q_dq_local || m->n_dq_nonlocal < 0) return nullptr;
  return m->n_qblocks == (n + kBlock - 1) / kBlock ? m->q_dq_local : nullptr;
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
                                                          dsum, lse2, dq_acc, seq_to_cell, q_local, n, heads,
                                                          (int32_t)rows);
  else
    bwd_preprocess_kernel<32><<<blocks, 256, 0, stream>>>(reinterpret_cast<const __nv_bfloat16*>(o),
                                                          reinterpret_cast<const __nv_bfloat16*>(dout), lse, sc,
                                                          dsum, lse2, dq_acc, seq_to_cell, q_local, n, heads,
                                                          (int32_t)rows);
  HLA_CUDA_TRY(cudaGetLastError());
  return HLA_OK;
}

extern "C" hla_status hla_attn_bwd_main(const hla_pattern_desc* d, const hla_block_mask* m, int32_t batch,
                                        int32_t heads, int32_t head_dim, float scale, const void* q, const void* k,
                                        const void* v, const void* dout, void* dq, void* dk, void* dv,
                                        const int32_t* seq_to_cell, const hla_score_mod* score_mod,
                                        void* workspace, size_t workspace_bytes, int64_t* tiles_visited,
                                        cudaStream_t stream) {
  clear_error();
  Pattern pat;
  hla_status st = check_attn_args(d, m, batch, heads, head_dim, &pat);
  if (st != HLA_OK) return st;
  HLA_REQUIRE(m->t_row_ptr && m->t_col_idx && m->t_kind, HLA_ERR_INVALID, "transposed mask arrays missing");
  HLA_REQUIRE(q && k && v && dout && dk && dv, HLA_ERR_INVALID, "null pointer");
  HLA_REQUIRE(dq || !plan_of(m, pat.N), HLA_ERR_INVALID, "dq required: the mask's dQ plan writes local q-blocks");
  HLA_REQUIRE(((uintptr_t)q | (uintptr_t)k | (uintptr_t)v | (uintptr_t)dout | (uintptr_t)dk | (uintptr_t)dv |
               (uintptr_t)dq) % 16 == 0,
              HLA_ERR_INVALID, "tensors must be 16-byte aligned");
  float *dq_acc, *dsum, *lse2;
  st = carve_workspace(batch, heads, pat.N, head_dim, workspace, workspace_bytes, &dq_acc, &dsum, &lse2);
  if (st != HLA_OK) return st;
  const float sc = scale > 0.f ? scale : 1.0f / sqrtf((float)head_dim);
  BwdParams prm;
  prm.pat = pat;
  prm.N = pat.N;
  prm.heads = heads;
  prm.batch = batch;
  prm.scale = sc;
  prm.scale_log2 = sc * kLog2e;
  prm.t_row_ptr = m->t_row_ptr;
  prm.t_col_idx = m->t_col_idx;
  prm.t_kind = m->t_kind;
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
  const bool gather = seq_to_cell != nullptr;
  HLA_REQUIRE(!gather || d->order == HLA_ORDER_HILBERT, HLA_ERR_INVALID,
              "seq_to_cell (fused reorder) is only meaningful for Hilbert-order patterns");
  HLA_REQUIRE(!gather || ((uintptr_t)seq_to_cell & 15) == 0, HLA_ERR_INVALID, "seq_to_cell must be 16-byte aligned");
  const int64_t tok = (int64_t)batch * pat.N;
  CUtensorMap mq, mk, mv, mdo;
  auto mk_map = [&](CUtensorMap* mp, const void* base) {
    return gather ? make_gather_map(mp, base, tok, heads, head_dim) : make_rows_map(mp, base, tok, heads, head_dim, kBlock);
  };
  if ((st = mk_map(&mq, q)) != HLA_OK) return st;
  if ((st = mk_map(&mk, k)) != HLA_OK) return st;
  if ((st = mk_map(&mv, v)) != HLA_OK) return st;
  if ((st = mk_map(&mdo, dout)) != HLA_OK) return st;
  CUtensorMap mdq;   // fp32 dQ accumulator, sequence order, 32-float (128 B) boxes for the TMA reduce-add
  if ((st = make_f32_rows_map(&mdq, dq_acc, tok, heads, head_dim, 32, kBlock)) != HLA_OK) return st;
  const bool two_d = pat.kind == K_WSA || pat.kind == K_SA || pat.kind == K_NA2D;
  const int32_t mkb = (pat.N + kBlock - 1) / kBlock;
  return prm.rpb ? dispatch_bwd<true>(head_dim, gather, two_d, mq, mk, mv, mdo, mdq, prm, mkb, stream)
                 : dispatch_bwd<false>(head_dim, gather, two_d, mq, mk, mv, mdo, mdq, prm, mkb, stream);
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
                                                 reinterpret_cast<uint4*>(dq), seq_to_cell, q_local, n,
                                                 heads * head_dim / 8, (int32_t)n_v);
  HLA_CUDA_TRY(cudaGetLastError());
  return HLA_OK;
}

extern "C" hla_status hla_attn_bwd(const hla_pattern_desc* d, const hla_block_mask* m, int32_t batch, int32_t heads,
                                   int32_t head_dim, float scale, const void* q, const void* k, const void* v,
                                   const void* o, const float* lse, const void* dout, void* dq, void* dk, void* dv,
                                   const int32_t* seq_to_cell, const hla_score_mod* score_mod, void* workspace,
                                   size_t workspace_bytes, int64_t* tiles_visited, cudaStream_t stream) {
  clear_error();
  Pattern pat;
  hla_status st = check_attn_args(d, m, batch, heads, head_dim, &pat);
  if (st != HLA_OK) return st;
  HLA_REQUIRE(o && dq, HLA_ERR_INVALID, "null pointer");
  // validate everything before launching anything
  float *dq_acc, *dsum;
  st = carve_workspace(batch, heads, pat.N, head_dim, workspace, workspace_bytes, &dq_acc, &dsum);
  if (st != HLA_OK) return st;
  HLA_REQUIRE(((uintptr_t)o | (uintptr_t)dq) % 16 == 0, HLA_ERR_INVALID, "tensors must be 16-byte aligned");
  const float* rpb;
  float* drpb;
  const int32_t* cells;
  if ((st = parse_score_mod(d, score_mod, true, &rpb, &drpb, &cells)) != HLA_OK) return st;
  if (drpb)   // the table gradient is accumulated: start from zero
    HLA_CUDA_TRY(cudaMemsetAsync(drpb, 0, sizeof(float) * heads * (2 * pat.H - 1) * (2 * pat.W - 1), stream));
  if ((st = hla_attn_bwd_preprocess(batch, heads, pat.N, head_dim, scale, o, dout, lse, seq_to_cell, m, workspace,
                                    workspace_bytes, stream)) != HLA_OK)
    return st;
  if ((st = hla_attn_bwd_main(d, m, batch, heads, head_dim, scale, q, k, v, dout, dq, dk, dv, seq_to_cell,
                              score_mod, workspace, workspace_bytes, tiles_visited, stream)) != HLA_OK)
    return st;
  return hla_attn_bwd_finalize(batch, heads, pat.N, head_dim, workspace, workspace_bytes, dq, seq_to_cell, m,
                               stream);
}
