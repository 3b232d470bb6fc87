// K6: block-sparse attention forward on sm_100a (tcgen05 + TMEM + TMA).
//
// Paper: "Block-sparse attention tiles the N x N matrix into fixed-size blocks
// ... empty blocks are skipped, full blocks run unmasked, partial blocks require
// element-wise masking"; per CTA cost alpha + beta * r_i, where beta
// covers "loading q block and k/v block, computing qk^T within the block, ...,
// online softmax, and aggregation with value" (Eq. 1).
//
// Persistent CTAs (2 per SM), 256 threads:
//   warps 0,2,3 TMA producers (Q_i / K_j / V_j; several issuing warps because a
//               CTA's TMA gather4 rate grows with them): Q double-buffered per
//               unit, K / V of the listed kv-blocks in a 2-stage ring; warp 0
//               also stores each finished O tile (TMA store / scatter4) from
//               the unit's Q stage, where the softmax warps staged it.
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer:
//                 S_t  = Q_i K_j^T   (SS MMA, 128x128x D, fp32 in TMEM cols [0,128))
//                 O   += P_t V_j     (TS MMA, P bf16 in TMEM cols [128,192), O in [192,192+D))
//   warps 4..7  softmax: thread = query row (TMEM lane); reads its S row with
//               tcgen05.ld, applies the element mask only when the tile is
//               partial, keeps the online max / sum in registers (lazy rescale:
//               O is rescaled in TMEM only when the row max grows by > 2^8),
//               writes P (bf16) to TMEM; epilogue O / l -> bf16 rows staged in
//               shared memory (swizzled like a loaded tile), LSE.
// The S region is reused by S_{t+1} only after the softmax of tile t has
// released it (p_full); P has its own region, so S_{t+1} overlaps nothing the
// PV MMA still reads.  Every commit tracks all earlier MMAs, so s_full(t) also
// certifies that PV_{t-1} finished (O may then be rescaled safely).
#ifdef HLA_FWD_PROF
#define HLA_PROF_ON
#endif
#include "predicates.cuh"
#include "sm100.cuh"
#include "tensor_map.cuh"

namespace hla {
#ifdef HLA_FWD_PROF
__device__ unsigned long long g_fwd_prof[1024][24];
#define HLA_PROF_ARRAY g_fwd_prof
#endif
namespace {

constexpr int kBlock = 128;
constexpr int kThreads = 256;   // warpgroup 0: TMA (Q), MMA, TMA (K), TMA (V); warpgroup 1: softmax
constexpr uint32_t kTmemCols = 256;
constexpr uint32_t kColS = 0, kColP = 128, kColO = 192;
// per-warpgroup register budgets (setmaxnreg) at 2 CTAs / SM: 128 (kRegsCtl + kRegsSm) <= 32768
#ifndef HLA_FWD_REGS_CTL
#define HLA_FWD_REGS_CTL 56
#endif
constexpr int kRegsCtl = HLA_FWD_REGS_CTL, kRegsSm = 256 - HLA_FWD_REGS_CTL;
// O tile stores: the softmax warps read their staged rows back transposed and write them with
// coalesced STG.128 (each instruction 8 whole 64-B rows at d = 32), or warp 0 TMA-stores the
// staged tile (store / scatter4) before it reloads the Q stage.  Measured (DESIGN 6g): the warp
// stores win at d = 32 (cfg5 fwd -20 %), the TMA stores at d = 64 (cfg3 / cfg4 fwd -3 %).
// HLA_FWD_OSTORE: 0 = TMA always, 1 = warps always, 2 = warps at d = 32 only (default).
#ifndef HLA_FWD_OSTORE
#define HLA_FWD_OSTORE 2
#endif
template <int D>
constexpr bool warp_ostore() { return HLA_FWD_OSTORE == 1 || (HLA_FWD_OSTORE == 2 && D == 32); }
// d = 32: S 128 + P 64 + O 32 leave 32 TMEM columns, so O is double-buffered by unit parity
// (columns 192 / 224) and a unit's epilogue is deferred until the next unit's first P is in
// TMEM: it then overlaps that tile's PV / next S on the tensor pipe instead of waiting for
// the unit's last PV (cfg5 runs one tile per unit).  O is staged in its own shared-memory tile.
#ifndef HLA_FWD_ODB
#define HLA_FWD_ODB 1
#endif

template <int D>
constexpr bool o_double() { return HLA_FWD_ODB != 0 && D == 32 && warp_ostore<D>(); }

struct FwdParams {
  Pattern pat;
  FastDiv mq_div, heads_div;   // q-blocks per (b, h); heads
  int32_t N, heads, batch;
  float scale_log2;
  const int32_t* row_ptr;    // tile lists (AttnLists): per 128-row q tile
  const int32_t* col_idx;
  const uint8_t* kind;
  int32_t col_mul;           // start row of a list entry = column * col_mul (128, or 64: windows)
  const int32_t* s2c;        // fused reorder: seq_to_cell table (tensors in grid order), else null
  int32_t box8;              // d = 32, tiled Hilbert order: log2(W) + 1 (0 = off): Q / K / V as 8 x 8-cell square boxes
  const float* rpb;          // global RPB table [heads][2H-1][2W-1] (kBias), else null
  const int32_t* cells;      // grid cell of each sequence position for the RPB offsets (null: identity)
  int32_t grid_h, grid_w, rpb_w, rpb_hw;   // H, W, 2W-1, (2H-1)(2W-1)
  int32_t rpb_a0;                  // (H-1)(2W-1) + (W-1): index of the zero offset
  __nv_bfloat16* o;
  float* lse;
  unsigned long long* visited;
};

template <int D, bool kBias = false>
struct FwdSmem {
  static constexpr uint32_t kTileBytes = kBlock * D * 2;
  alignas(1024) uint8_t q[2][kTileBytes];
  alignas(1024) uint8_t k[2][kTileBytes];
  alignas(1024) uint8_t v[2][kTileBytes];
  // k_empty: the stage's K was read by its S MMA (K may reload while P / PV still run; with the
  // RPB bias the key offsets are read by the softmax, so K waits for v_empty there), v_empty: PV done
  uint64_t q_full[2], o_staged[2], k_full[2], v_full[2], k_empty[2], v_empty[2], s_full, s_free, p_full, pv_done,
      o_full;
  uint32_t tmem_base;
  // kBias: table offsets B_k of the keys of K/V stage s, written by the K producer
  // before it arms k_full[s] (read by the softmax after waiting on the same phase)
  alignas(16) int32_t key_b[2][kBias ? 128 : 4];
  alignas(1024) uint8_t ostage[o_double<D>() ? kBlock * D * 2 : 16];   // deferred O epilogue staging (d = 32)
};

template <int D>
__device__ __forceinline__ uint64_t kmajor_desc(const uint8_t* tile, int kstep) {
  // rows of D bf16 (= swizzle width), 8-row groups 8*2D bytes apart; K step = 16 elements = 32 B
  constexpr uint32_t layout = D == 64 ? sm100::kSwizzle128B : sm100::kSwizzle64B;
  return sm100::make_smem_desc(sm100::smem_u32(tile) + kstep * 32, 16, 8 * D * 2, layout);
}
template <int D>
__device__ __forceinline__ uint64_t mnmajor_desc(const uint8_t* tile, int kstep) {
  // V as the B operand of O = P V: N = D (one swizzle atom wide), K = kv rows;
  // 8-row K groups 8*2D bytes apart; K step = 16 rows
  constexpr uint32_t layout = D == 64 ? sm100::kSwizzle128B : sm100::kSwizzle64B;
  return sm100::make_smem_desc(sm100::smem_u32(tile) + kstep * 16 * D * 2, kBlock * D * 2, 8 * D * 2, layout);
}

// Load the 128 token rows [seq0, seq0 + 128) (sequence order) of head h, batch b.
// kGather (fused reorder): the tensor is in grid order; the warp gathers the rows of
// cells s2c[seq0 ..] with 32 TMA .tile::gather4 ops (4 rows each); otherwise one 3-D
// TMA box.  row_cells() looks the cells up (issued early: it is an L2 round trip),
// issue_rows() is called by all 32 lanes of the producer warp after lane 0 armed `bar`.
template <bool kGather>
__device__ __forceinline__ int4 row_cells(int32_t N, int32_t seq0, const int32_t* s2c, int lane) {
  // rows past N (ragged last tile) gather cell 0: their values are masked / discarded
  if (!kGather) return make_int4(0, 0, 0, 0);
  return seq0 + 4 * lane < N ? __ldg(reinterpret_cast<const int4*>(s2c + seq0) + lane) : make_int4(0, 0, 0, 0);
}
template <int D, bool kGather>
__device__ __forceinline__ void issue_rows(uint8_t* dst, const CUtensorMap* map, uint64_t* bar, int32_t h, int32_t b,
                                           int32_t N, int32_t seq0, int4 c, uint64_t pol, int lane, int sq) {
  if (kGather) {
    const int32_t base = b * N;
    if (D == 32 && sq) {   // see attn_bwd_common.cuh load_rows: lane 16l holds row 64l's cell
      const int32_t c64 = __shfl_sync(0xffffffffu, c.x, (16 * lane) & 31);
      const int lw = sq - 1;
      if (lane < 2)
        sm100::tma_load_5d(dst + lane * 64 * D * 2, map, bar, 0, h, c64 & ((1 << lw) - 1), c64 >> lw, b, pol);
    } else {
      sm100::tma_gather4(dst + lane * 4 * D * 2, map, bar, h * D, base + c.x, base + c.y, base + c.z, base + c.w,
                         pol);
    }
  } else if (lane == 0) {
    sm100::tma_load_3d(dst, map, bar, 0, h, b * N + seq0, pol);
  }
}

// Element mask of a partial tile for query row q (box = row_box(q)), keys k0 .. k0+127.
template <bool kTwoD>
__device__ __forceinline__ void apply_row_mask(float (&s)[kBlock], const Pattern& pat, const RowBox& box_in,
                                               int32_t k0) {
  const RowBox box = clip_box<kTwoD>(pat, box_in);   // phantom keys (k >= N) are never allowed
  if (!kTwoD) {
#pragma unroll
    for (int c = 0; c < kBlock; ++c)
      if ((uint32_t)(k0 + c - box.lo) >= (uint32_t)box.len) s[c] = -INFINITY;
  } else if (pat.log2W >= 0) {
    const int sh = pat.log2W;
    const int32_t wm = pat.W - 1;
#pragma unroll
    for (int c = 0; c < kBlock; ++c) {
      const int32_t k = k0 + c;
      const bool ok = ((uint32_t)((k >> sh) - box.lo) < (uint32_t)box.len) &&
                      ((uint32_t)((k & wm) - box.c0) < (uint32_t)box.cn);
      if (!ok) s[c] = -INFINITY;
    }
  } else {
    const int32_t W = pat.W;
#pragma unroll
    for (int c = 0; c < kBlock; ++c) {
      const int32_t k = k0 + c;
      const int32_t rk = pat.w_div.div(k), ck = k - rk * W;
      const bool ok = ((uint32_t)(rk - box.lo) < (uint32_t)box.len) &&
                      ((uint32_t)(ck - box.c0) < (uint32_t)box.cn);
      if (!ok) s[c] = -INFINITY;
    }
  }
}

// True when no key of the partial tile [k0, k0 + 128) is allowed for query row `box`:
// the 1D interval (clipped to [0, N)) or the 2D box's grid-row range misses the tile.
// A warp whose 32 rows all miss skips the tile's softmax (its P rows are zero).
template <bool kTwoD>
__device__ __forceinline__ bool row_misses_tile(const Pattern& pat, const RowBox& box_in, int32_t k0) {
  const RowBox box = clip_box<kTwoD>(pat, box_in);
  if (box.len <= 0) return true;
  if (!kTwoD) return box.lo + box.len <= k0 || box.lo >= k0 + kBlock;
  const int32_t r0 = pat.w_div.div(k0), r1 = pat.w_div.div(k0 + kBlock - 1);   // grid rows the tile's keys lie in
  return box.lo + box.len <= r0 || box.lo > r1;
}

// k-th work unit of this CTA: pairs of consecutive q-blocks (2p, 2p+1) of one
// (b, h), pairs strided over the grid.  Neighbouring q-blocks list the same
// kv-blocks (HWA: exactly), so the producer can skip reloading a K/V stage.
__device__ __forceinline__ int32_t fwd_unit_at(int32_t k) {
  return 2 * ((int32_t)blockIdx.x + (k >> 1) * (int32_t)gridDim.x) + (k & 1);
}

// Flattened (unit, kv-tile) iterator of this CTA, skipping units without tiles.
// The CSR row of the next unit is loaded one unit ahead (prefetch), so crossing a
// unit boundary does not put an L2 round trip on any role's critical path.
struct FwdIter {
  int32_t k, u, t, nt, rs;
  uint32_t n;   // ordinal of the current non-empty unit
  bool valid;
  bool from_pf;          // the current unit came from the prefetch (its per-lane metadata too)
  int32_t pu, prs, pre;  // prefetched unit k + 1 and its CSR row [prs, pre)
  __device__ void seek(const int32_t* row_ptr, const FastDiv& mq, int32_t units) {
    for (;; ++k) {
      u = fwd_unit_at(k);
      if (u >= units) break;
      const int32_t qb = u - mq.div(u) * mq.d;
      rs = __ldg(row_ptr + qb);
      nt = __ldg(row_ptr + qb + 1) - rs;
      if (nt > 0) { valid = true; return; }
    }
    valid = false;
  }
  __device__ void prefetch(const int32_t* row_ptr, const FastDiv& mq, int32_t units) {
    pu = fwd_unit_at(k + 1);
    prs = pre = 0;
    if (pu < units) {
      const int32_t qb = pu - mq.div(pu) * mq.d;
      prs = __ldg(row_ptr + qb);
      pre = __ldg(row_ptr + qb + 1);
    }
  }
  __device__ void init(const int32_t* row_ptr, const FastDiv& mq, int32_t units) {
    k = 0; t = 0; n = 0; from_pf = false;
    seek(row_ptr, mq, units);
    if (valid) prefetch(row_ptr, mq, units);
  }
  __device__ void advance(const int32_t* row_ptr, const FastDiv& mq, int32_t units) {
    if (++t < nt) return;
    t = 0; ++n; ++k;
    if (pu >= units) { valid = false; return; }
    if (pre > prs) {
      u = pu; rs = prs; nt = pre - prs; valid = true; from_pf = true;
    } else {
      ++k;
      seek(row_ptr, mq, units);
      from_pf = false;
      if (!valid) return;
    }
    prefetch(row_ptr, mq, units);
  }
};

// FwdIter with the CSR row pointers loaded two units ahead (the softmax warpgroup, which has
// the registers for it): at unit k those of unit k + 1 are already in registers, so the per-lane
// CSR entries of k + 1 can be requested without an L2 round trip first; those of k + 2 are in
// flight.  (The producer / MMA warps keep FwdIter: at 48 registers the extra state spills.)
struct FwdIter2 : FwdIter {
  int32_t qu, qrs, qre;  // unit k + 2
  __device__ static void load_rp(const int32_t* row_ptr, const FastDiv& mq, int32_t units, int32_t kk, int32_t& uu,
                                 int32_t& b0, int32_t& b1) {
    uu = fwd_unit_at(kk);
    b0 = b1 = 0;
    if (uu < units) {
      const int32_t qb = uu - mq.div(uu) * mq.d;
      b0 = __ldg(row_ptr + qb);
      b1 = __ldg(row_ptr + qb + 1);
    }
  }
  __device__ void init(const int32_t* row_ptr, const FastDiv& mq, int32_t units) {
    k = 0; t = 0; n = 0; from_pf = false;
    seek(row_ptr, mq, units);
    if (valid) {
      load_rp(row_ptr, mq, units, k + 1, pu, prs, pre);
      load_rp(row_ptr, mq, units, k + 2, qu, qrs, qre);
    }
  }
  __device__ void advance(const int32_t* row_ptr, const FastDiv& mq, int32_t units) {
    if (++t < nt) return;
    t = 0; ++n; ++k;
    if (pu >= units) { valid = false; return; }
    if (pre > prs) {
      u = pu; rs = prs; nt = pre - prs; valid = true; from_pf = true;
      pu = qu; prs = qrs; pre = qre;
      load_rp(row_ptr, mq, units, k + 2, qu, qrs, qre);
    } else {
      ++k;
      seek(row_ptr, mq, units);
      from_pf = false;
      if (!valid) return;
      load_rp(row_ptr, mq, units, k + 1, pu, prs, pre);
      load_rp(row_ptr, mq, units, k + 2, qu, qrs, qre);
    }
  }
};

// A unit's CSR entries as loaded (lane i: tile i), packed only when the unit starts, so the
// loads of the next unit's entries have no consumer (no scoreboard wait) before then.
struct MetaRaw {
  int32_t c, k;
};
__device__ __forceinline__ MetaRaw load_meta_raw(const int32_t* col, const uint8_t* kind, int32_t rs, int32_t nt,
                                                 int lane) {
  MetaRaw m{0, 0};
  if (lane < nt) {
    m.c = __ldg(col + rs + lane);
    m.k = (int32_t)__ldg(kind + rs + lane);
  }
  return m;
}

// Per-lane copy of a unit's CSR entries (lane i holds tile i), packed col * 4 + kind;
// tiles past 32 fall back to direct loads.
__device__ __forceinline__ int32_t load_meta(const int32_t* col, const uint8_t* kind, int32_t rs, int32_t nt,
                                             int lane) {
  return lane < nt ? (__ldg(col + rs + lane) << 2) | (int32_t)__ldg(kind + rs + lane) : 0;
}
__device__ __forceinline__ int32_t tile_meta(int32_t meta, const int32_t* col, const uint8_t* kind, int32_t rs,
                                             int32_t t) {
  const int32_t v = __shfl_sync(0xffffffffu, meta, t & 31);
  return t < 32 ? v : (__ldg(col + rs + t) << 2) | (int32_t)__ldg(kind + rs + t);
}

// Persistent CTAs (2 per SM).  Pipeline over the flattened tile sequence g:
//   TMA     : Q of unit n into stage n&1 (double-buffered); K/V of tile g into
//             stage g&1 (skipped when the stage already holds that kv-block)
//   MMA     : S(g+1) as soon as the softmax has pulled S(g) into registers
//             (s_free), then PV(g) after P(g) is in TMEM (p_full)
//   softmax : S(g) -> registers -> s_free -> mask / max / exp; before writing
//             P(g) (and before rescaling O) it waits pv_done(g-1)
// Global RPB (reading R19): the table index of the pair (q, k) is
// A_q - B_k with A_q = (qr + H - 1)(2W - 1) + qc + W - 1, B_k = kr (2W - 1) + kc.
__device__ __forceinline__ int32_t rpb_cell_off(const int32_t* cells, int32_t seq, int32_t N, const FastDiv& W,
                                                int32_t rw) {
  const int32_t cell = seq < N ? (cells ? __ldg(cells + seq) : seq) : 0;
  const int32_t r = W.div(cell);
  return r * rw + (cell - r * W.d);
}
// B_k of the 4 keys k0 + 4 lane .. + 3 of a kv tile (lane-distributed; 16-B loads)
__device__ __forceinline__ int4 rpb_key_offs(const int32_t* cells, int32_t k0, int32_t N, const FastDiv& W,
                                             int32_t rw, int lane) {
  const int32_t k = k0 + 4 * lane;
  int4 c = make_int4(0, 0, 0, 0);
  if (k < N) c = cells ? __ldg(reinterpret_cast<const int4*>(cells + k0) + lane) : make_int4(k, k + 1, k + 2, k + 3);
  auto off = [&](int32_t cell) { const int32_t r = W.div(cell); return r * rw + (cell - r * W.d); };
  return make_int4(off(c.x), off(c.y), off(c.z), off(c.w));
}

// kHalf: HWA with 64-token windows (launch_fwd checks it): every tile pairs the two windows of its
// 128 query rows with the same two windows of keys, so each softmax warp's 32 rows see exactly one
// unmasked 64-column half of S -- half the S loads, exponentials and P stores.
template <int D, bool kTwoD, bool kGather, bool kBias, bool kHalf = false>
__global__ void __launch_bounds__(kThreads, 2)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                    const FwdParams prm) {
  extern __shared__ uint8_t smem_raw[];
  FwdSmem<D, kBias>& sm = *reinterpret_cast<FwdSmem<D, kBias>*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < 2; ++s) {
      sm100::mbar_init(&sm.q_full[s], 1);
      sm100::mbar_init(&sm.o_staged[s], 128);   // softmax threads: O(n) staged in Q stage n&1
      sm100::mbar_init(&sm.k_full[s], 2);   // producer warps 2 and 3
      sm100::mbar_init(&sm.v_full[s], 2);
      sm100::mbar_init(&sm.k_empty[s], 1);
      sm100::mbar_init(&sm.v_empty[s], 1);
    }
    sm100::mbar_init(&sm.s_full, 1);
    sm100::mbar_init(&sm.s_free, 128);
    sm100::mbar_init(&sm.p_full, 128);
    sm100::mbar_init(&sm.pv_done, 1);
    sm100::mbar_init(&sm.o_full, 1);
    sm100::fence_mbar_init();
    sm100::tma_prefetch_desc(&tmQ);
    sm100::tma_prefetch_desc(&tmK);
    sm100::tma_prefetch_desc(&tmV);
  }
  if (warp == 1) {
    sm100::tmem_alloc(&sm.tmem_base, kTmemCols);
    sm100::tmem_relinquish();
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
#ifdef HLA_FWD_PROF
  const long long prof_c0 = clock64();
  unsigned long long prof_g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prof_g0));
#endif
  HLA_TR_DECL;

  // register split (setmaxnreg acts per warpgroup): the control warpgroup gives its
  // registers to the softmax warpgroup (one thread per row keeps a 128-wide S row)
  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsCtl) : "memory");
    const uint32_t tmem = sm.tmem_base;   // read after the register split (not spilled across it)
    HLA_PDECL;
    // (derived after the register split, so they are not spilled across it)
    const int32_t mq = (prm.N + kBlock - 1) / kBlock;   // last q-block may be ragged
    const int32_t units = mq * prm.heads * prm.batch;
    if (warp != 1) {
      // ---------------------------------------------------------- TMA producers
      // warp 0 loads Q, warp 2 K, warp 3 V: a CTA's TMA row / gather4 throughput grows
      // with the number of issuing warps (one warp alone caps gather4 at ~6 B/clk)
      const uint64_t pol_q = sm100::policy_evict_first();
      const uint64_t pol_kv = sm100::policy_evict_last();
      int64_t tag0 = -1, tag1 = -1;   // (b, h, kv-block) held by K/V stage 0 / 1
      uint32_t g = 0, n_units = 0;
      int32_t staged0 = 0, staged1 = 0;   // unit whose O is staged in Q stage 0 / 1
      // O tile of unit us (staged in Q stage qs, swizzled like a loaded tile) -> global;
      // ragged tiles were written row by row by the softmax warps
      auto store_o = [&](int qs, int32_t us) {
        const int32_t bh_s = prm.mq_div.div(us), sqb = us - bh_s * mq;
        const int32_t sb = prm.heads_div.div(bh_s), sh = bh_s - sb * prm.heads;
        if ((sqb + 1) * kBlock > prm.N) return;
        if (kGather) {
          const int4 c = row_cells<true>(prm.N, sqb * kBlock, prm.s2c, lane);
          const int32_t base = sb * prm.N;
          sm100::tma_scatter4(&tmO, sm.q[qs] + lane * 4 * D * 2, sh * D, base + c.x, base + c.y, base + c.z,
                              base + c.w);
        } else if (lane == 0) {
          sm100::tma_store_3d(&tmO, sm.q[qs], 0, sh, sb * prm.N + sqb * kBlock);
        }
        sm100::bulk_commit_group();
        sm100::bulk_wait_group_read0();   // the stage may be refilled once the engine has read it
        __syncwarp();
      };
      FwdIter it;
      it.init(prm.row_ptr, prm.mq_div, units);
      int32_t meta = 0, pmeta = 0;
      if (warp != 0 && it.valid) {
        meta = load_meta(prm.col_idx, prm.kind, it.rs, it.nt, lane);
        pmeta = load_meta(prm.col_idx, prm.kind, it.prs, it.pre - it.prs, lane);
      }
      while (it.valid) {
        const int32_t bh_u = prm.mq_div.div(it.u), qb = it.u - bh_u * mq;
        const int32_t b = prm.heads_div.div(bh_u), h = bh_u - b * prm.heads;
        const int64_t bh = (int64_t)b * prm.heads + h;
        if (warp == 0) {
          // Q(n) goes into stage n&1, which holds O(n-2) staged by the softmax warps:
          // store that tile first (TMA store / scatter4), then reuse the stage
          const int qs = it.n & 1;
          const int4 cells = row_cells<kGather>(prm.N, qb * kBlock, prm.s2c, lane);
          if (it.n >= 2) {
            HLA_PW(11, sm100::mbar_wait(&sm.o_staged[qs], ((it.n >> 1) - 1) & 1));
            if (!warp_ostore<D>()) HLA_PW(12, store_o(qs, qs ? staged1 : staged0));
          }
          if (qs) staged1 = it.u; else staged0 = it.u;
          if (lane == 0) HLA_TR((3 << 24) | (1 << 16) | it.n);
          if (lane == 0) sm100::mbar_arrive_expect_tx(&sm.q_full[qs], FwdSmem<D, kBias>::kTileBytes);
          __syncwarp();
          issue_rows<D, kGather>(sm.q[qs], &tmQ, &sm.q_full[qs], h, b, prm.N, qb * kBlock, cells, pol_q, lane,
                                 prm.box8);
          ++n_units;
        } else {
          // warps 2 and 3 both feed every K / V stage (k_full / v_full count 2).  Fused reorder:
          // warp 2 + hh gathers rows [64 hh, 64 hh + 64) of K (lanes 0-15) and of V (lanes 16-31),
          // so each tile's 32 gather4 ops are spread over two issuing warps (a warp's gather4 stream
          // is rate-limited) and K's go first.  Plain order: warp 2 loads K, warp 3 V (one box each)
          // and each arrives on the other barrier without bytes.
          const bool is_k = warp == 2;
          const int hh = warp - 2;
          constexpr uint32_t kTile = FwdSmem<D, kBias>::kTileBytes;
          for (int t = 0; t < it.nt; ++t, ++g) {
            const int s = g & 1;
            const int32_t kvb = tile_meta(meta, prm.col_idx, prm.kind, it.rs, t) >> 2;
            const int64_t tag = bh * prm.N + kvb;
            const bool reuse = tag == (s ? tag1 : tag0);   // stage already holds this K/V tile
            const int32_t r0 = kvb * prm.col_mul + hh * 64 + 4 * (lane & 15);   // this lane's 4 rows (gather)
            const int4 cells = (reuse || !kGather) ? make_int4(0, 0, 0, 0)
                               : (r0 < prm.N ? __ldg(reinterpret_cast<const int4*>(prm.s2c + r0)) : make_int4(0, 0, 0, 0));
            // every arrival on k_full / v_full follows the wait on the matching empty barrier,
            // so it always lands in this tile's phase
            uint64_t* kfree = kBias ? &sm.v_empty[s] : &sm.k_empty[s];
            const uint32_t par = ((g >> 1) - 1) & 1;
            if (reuse) {
              if (g >= 2) sm100::mbar_wait(kfree, par);
              if (lane == 0) sm100::mbar_arrive(&sm.k_full[s]);
              if (g >= 2) sm100::mbar_wait(&sm.v_empty[s], par);
              if (lane == 0) sm100::mbar_arrive(&sm.v_full[s]);
              continue;
            }
            if (s) tag1 = tag; else tag0 = tag;
            if (g >= 2) sm100::mbar_wait(kfree, par);
            if (kBias && is_k) {
              const int4 bk = rpb_key_offs(prm.cells, kvb * prm.col_mul, prm.N, prm.pat.w_div, prm.rpb_w, lane);
              sm100::sts_u4(sm100::smem_u32(sm.key_b[s]) + 16u * lane, bk.x, bk.y, bk.z, bk.w);
              __syncwarp();   // every lane's offsets are written before lane 0 arms k_full
            }
            const int32_t base = b * prm.N;
            const int row = hh * 64 + 4 * (lane & 15);
            if (kGather) {   // this warp's half of K (lanes 0-15), then, once PV freed the stage, of V
              if (lane == 0) sm100::mbar_arrive_expect_tx(&sm.k_full[s], kTile / 2);
              __syncwarp();
              // square boxes: this warp's 64 rows are one 8 x 8 cell square (its first cell: lane 0)
              const bool b8 = D == 32 && prm.box8;
              const int lw = prm.box8 - 1;
              const int32_t c8 = b8 ? __shfl_sync(0xffffffffu, cells.x, 0) : 0;
              if (b8) {
                if (lane == 0)
                  sm100::tma_load_5d(sm.k[s] + hh * 64 * D * 2, &tmK, &sm.k_full[s], 0, h, c8 & ((1 << lw) - 1),
                                     c8 >> lw, b, pol_kv);
              } else if (lane < 16) {
                sm100::tma_gather4(sm.k[s] + row * D * 2, &tmK, &sm.k_full[s], h * D, base + cells.x, base + cells.y,
                                   base + cells.z, base + cells.w, pol_kv);
              }
              if (g >= 2) sm100::mbar_wait(&sm.v_empty[s], par);
              if (lane == 0) sm100::mbar_arrive_expect_tx(&sm.v_full[s], kTile / 2);
              __syncwarp();
              if (b8) {
                if (lane == 0)
                  sm100::tma_load_5d(sm.v[s] + hh * 64 * D * 2, &tmV, &sm.v_full[s], 0, h, c8 & ((1 << lw) - 1),
                                     c8 >> lw, b, pol_kv);
              } else if (lane < 16) {
                sm100::tma_gather4(sm.v[s] + row * D * 2, &tmV, &sm.v_full[s], h * D, base + cells.x, base + cells.y,
                                   base + cells.z, base + cells.w, pol_kv);
              }
            } else {   // warp 2: K box, warp 3: V box; each arrives (no bytes) on the other barrier
              if (is_k) {
                if (lane == 0) {
                  sm100::mbar_arrive_expect_tx(&sm.k_full[s], kTile);
                  sm100::tma_load_3d(sm.k[s], &tmK, &sm.k_full[s], 0, h, b * prm.N + kvb * prm.col_mul, pol_kv);
                }
                if (g >= 2) sm100::mbar_wait(&sm.v_empty[s], par);
                if (lane == 0) sm100::mbar_arrive(&sm.v_full[s]);
              } else {
                if (lane == 0) sm100::mbar_arrive(&sm.k_full[s]);
                if (g >= 2) sm100::mbar_wait(&sm.v_empty[s], par);
                if (lane == 0) {
                  sm100::mbar_arrive_expect_tx(&sm.v_full[s], kTile);
                  sm100::tma_load_3d(sm.v[s], &tmV, &sm.v_full[s], 0, h, b * prm.N + kvb * prm.col_mul, pol_kv);
                }
              }
            }
          }
        }
        it.t = it.nt - 1;
        it.advance(prm.row_ptr, prm.mq_div, units);
        if (warp != 0 && it.valid) {
          meta = it.from_pf ? pmeta : load_meta(prm.col_idx, prm.kind, it.rs, it.nt, lane);
          pmeta = load_meta(prm.col_idx, prm.kind, it.prs, it.pre - it.prs, lane);
        }
      }
      if (warp == 0 && !warp_ostore<D>()) {
        // the last (up to) two units' O tiles are still staged
        for (uint32_t m = n_units >= 2 ? n_units - 2 : 0; m < n_units; ++m) {
          sm100::mbar_wait(&sm.o_staged[m & 1], (m >> 1) & 1);
          store_o(m & 1, (m & 1) ? staged1 : staged0);
        }
        sm100::bulk_wait_group0();
      }
      HLA_PFLUSH(11, 13, warp == 0 && lane == 0);
      HLA_PFLUSH(13, 14, warp == 2 && lane == 0);
    } else if (warp == 1 && lane == 0) {
      // ----------------------------------------------------------- MMA issuer
      constexpr uint32_t idesc_s = sm100::make_idesc_bf16(kBlock, kBlock, false, false);
      constexpr uint32_t idesc_o = sm100::make_idesc_bf16(kBlock, D, false, true);
      const uint32_t tS = tmem + kColS, tP = tmem + kColP, tO = tmem + kColO;
      auto issue_s = [&](uint32_t n, uint32_t gg) {
        const uint8_t* q = sm.q[n & 1];
        const uint8_t* k = sm.k[gg & 1];
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          sm100::mma_ss(tS, kmajor_desc<D>(q, kk), kmajor_desc<D>(k, kk), idesc_s, kk > 0);
        sm100::mma_commit(&sm.s_full);
        sm100::mma_commit(&sm.k_empty[gg & 1]);   // K(gg) read: the stage may reload its K
      };
      FwdIter it;   // always one tile ahead of the PV being issued
      it.init(prm.row_ptr, prm.mq_div, units);
      uint32_t g = 0;
      if (it.valid) {
        sm100::mbar_wait(&sm.q_full[0], 0);
        sm100::mbar_wait(&sm.k_full[0], 0);
        sm100::tc_fence_after();
        issue_s(0, 0);
      }
      HLA_PMARK(tl0);
      while (it.valid) {
        const int32_t ct = it.t, cnt = it.nt;
        const uint32_t tOb = tO + (o_double<D>() ? 32u * (it.n & 1u) : 0u);   // this unit's O buffer
        it.advance(prm.row_ptr, prm.mq_div, units);
        // Two independent issues: S(g+1) (needs the softmax to have pulled S(g) into
        // registers, and the next Q / K landed) and PV(g) (needs P(g)).  Whichever is
        // ready first goes first: waiting for one in a fixed order stalls the other
        // (S first stalls PV behind late K loads; PV first stalls S behind the softmax).
        bool s_pending = it.valid, pv_pending = true;
        if (s_pending) HLA_PW(0, sm100::mbar_wait(&sm.s_free, g & 1));
        HLA_PMARK(tp0);
        while (s_pending || pv_pending) {
          if (s_pending && (it.t != 0 || sm100::mbar_test_wait(&sm.q_full[it.n & 1], (it.n >> 1) & 1)) &&
              sm100::mbar_test_wait(&sm.k_full[(g + 1) & 1], ((g + 1) >> 1) & 1)) {
            sm100::tc_fence_after();
            issue_s(it.n, g + 1);
            s_pending = false;
            continue;
          }
          if (pv_pending && sm100::mbar_test_wait(&sm.p_full, g & 1)) {
            HLA_TR((1 << 24) | (2 << 16) | g);
            sm100::mbar_wait(&sm.v_full[g & 1], (g >> 1) & 1);
            sm100::tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < kBlock / 16; ++kk)
              sm100::mma_ts(tOb, tP + kk * 8, mnmajor_desc<D>(sm.v[g & 1], kk), idesc_o,
                            (ct > 0 || kk > 0) ? 1u : 0u);
            sm100::mma_commit(&sm.v_empty[g & 1]);
            sm100::mma_commit(&sm.pv_done);
            if (ct == cnt - 1) sm100::mma_commit(&sm.o_full);
            pv_pending = false;
            continue;
          }
          __nanosleep(32);
        }
        HLA_PADD(1, tp0);
        ++g;
      }
      HLA_PADD(2, tl0);
#ifdef HLA_FWD_PROF
      prof[15] = g;
      prof[16] = (unsigned long long)(clock64() - prof_c0);   // this CTA's cycles until its last PV issue
      prof[17] = prof_g0;                                       // globaltimer (ns) at start / end
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prof[18]));
      {
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        prof[23] = smid;
      }
#endif
      HLA_PFLUSH(0, 3, true);
      HLA_PFLUSH(15, 19, true);
      HLA_PFLUSH(20, 22, true);
      HLA_PFLUSH(23, 24, true);
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsSm) : "memory");
    const uint32_t tmem = sm.tmem_base;   // read after the register split (not spilled across it)
    unsigned long long tiles_done = 0;
    HLA_PDECL;
    const int32_t mq = (prm.N + kBlock - 1) / kBlock;
    const int32_t units = mq * prm.heads * prm.batch;
    // --------------------------------------------------- softmax + epilogue
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const float sl2 = prm.scale_log2;
    uint32_t g = 0;
    FwdIter2 it;
    it.init(prm.row_ptr, prm.mq_div, units);
    int32_t meta = 0;
    MetaRaw pm{0, 0};
    if (it.valid) {
      meta = load_meta(prm.col_idx, prm.kind, it.rs, it.nt, lane);
      pm = load_meta_raw(prm.col_idx, prm.kind, it.prs, it.pre - it.prs, lane);
    }
    // o_double<D>(): the deferred epilogue of the previous unit (its O buffer, normalisation and
    // destination row) runs right after the next unit's first P store (pv_done of its last tile
    // has been waited by then, so its O is complete)
    bool pend = false;
    uint32_t pend_ob = 0;
    float pend_inv_l = 0.f;
    unsigned long long pend_optr = 0;   // 0: phantom row
    bool pend_staged = false;
    // square mode (tiled order, prm.box8): this warp's 32 staged rows = 4 grid rows of 8 cells of one
    // square, stored with one TMA box (tmO: 8 x 4 cells) from the first row's cell
    int32_t pend_c = 0, pend_h = 0, pend_b = 0;
    const bool sq_store = prm.box8 != 0;
    auto run_pending = [&]() {
      if (sq_store && pend_staged) {   // the previous store has read its staging rows
        if (lane == 0) sm100::bulk_wait_group_read0();
        __syncwarp();
      }
      uint32_t o[D];
#pragma unroll
      for (int c = 0; c < D / 32; ++c)
        sm100::tmem_ld32(tmem + lane_off + kColO + pend_ob + c * 32, *reinterpret_cast<uint32_t(*)[32]>(o + c * 32));
      sm100::tmem_wait_ld();
      const uint32_t stage = sm100::smem_u32(sm.ostage);
#pragma unroll
      for (int v4 = 0; v4 < D / 8; ++v4) {
        uint4 w;
        w.x = sm100::pack_bf16(__uint_as_float(o[v4 * 8 + 0]) * pend_inv_l, __uint_as_float(o[v4 * 8 + 1]) * pend_inv_l);
        w.y = sm100::pack_bf16(__uint_as_float(o[v4 * 8 + 2]) * pend_inv_l, __uint_as_float(o[v4 * 8 + 3]) * pend_inv_l);
        w.z = sm100::pack_bf16(__uint_as_float(o[v4 * 8 + 4]) * pend_inv_l, __uint_as_float(o[v4 * 8 + 5]) * pend_inv_l);
        w.w = sm100::pack_bf16(__uint_as_float(o[v4 * 8 + 6]) * pend_inv_l, __uint_as_float(o[v4 * 8 + 7]) * pend_inv_l);
        if (pend_staged) {
          const uint32_t off = (uint32_t)row * (D * 2) + v4 * 16;
          sm100::sts_u4(stage + sm100::swz64(off), w.x, w.y, w.z, w.w);
        } else if (pend_optr) {
          reinterpret_cast<uint4*>(pend_optr)[v4] = w;
        }
      }
      if (pend_staged && sq_store) {
        sm100::fence_proxy_async_smem();   // the staged rows before the TMA engine reads them
        __syncwarp();
        if (lane == 0) {
          const int lw = prm.box8 - 1;
          sm100::tma_store_5d(&tmO, sm.ostage + quarter * 32 * D * 2, 0, pend_h, pend_c & ((1 << lw) - 1),
                              pend_c >> lw, pend_b);
          sm100::bulk_commit_group();
        }
      } else if (pend_staged) {   // this warp's rows back transposed: each STG.128 writes 8 whole 64-B rows
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int rl = lane / 4 + 8 * k, c = lane % 4;
          const uint32_t off = (uint32_t)(quarter * 32 + rl) * (D * 2) + (uint32_t)c * 16u;
          const float4 v = sm100::lds_f4(stage + sm100::swz64(off));
          const unsigned long long p = __shfl_sync(0xffffffffu, pend_optr, rl);
          if (p)
            reinterpret_cast<uint4*>(p)[c] =
                make_uint4(__float_as_uint(v.x), __float_as_uint(v.y), __float_as_uint(v.z), __float_as_uint(v.w));
        }
        __syncwarp();   // (the staging rows are rewritten by the next deferred epilogue)
      }
      pend = false;
    };
    // RPB: the row's table offset A_q (per unit); the keys' B_k come staged with K
    while (it.valid) {
      const int32_t bh_u = prm.mq_div.div(it.u), qb = it.u - bh_u * mq;
      const int32_t b = prm.heads_div.div(bh_u), h = bh_u - b * prm.heads;
      const int32_t q = qb * kBlock + row;
      float m_ref = -INFINITY, l = 0.f;
      const RowBox box = row_box(prm.pat, q);
      const bool real = q < prm.N;
      const int32_t ocell = kGather ? (real ? __ldg(prm.s2c + q) : 0) : q;   // fused inverse reorder of O (used at the end)
      const float* rpbh = kBias ? prm.rpb + (int64_t)h * prm.rpb_hw : nullptr;
      const int32_t a_q = kBias ? prm.rpb_a0 + rpb_cell_off(prm.cells, q, prm.N, prm.pat.w_div, prm.rpb_w) : 0;
      if (row == 0) HLA_TR((2 << 24) | (6 << 16) | it.n);
      const uint32_t obuf = o_double<D>() ? 32u * (it.n & 1u) : 0u;   // this unit's O columns
      for (int t = 0; t < it.nt; ++t, ++g) {
        HLA_PMARK(tw0);
        HLA_PW(3, sm100::mbar_wait(&sm.s_full, g & 1));
        HLA_PMARK(ts0);
        if (t == 0) HLA_PADD(19, tw0);
        if (row == 0) HLA_TR((2 << 24) | (1 << 16) | g);
        sm100::tc_fence_after();
        const int32_t tm = tile_meta(meta, prm.col_idx, prm.kind, it.rs, t);
        if constexpr (kHalf) {
          const uint32_t hc = (uint32_t)(row >> 6) * 64u;   // this warp's key columns [hc, hc + 64)
          uint32_t sr[64];
          sm100::tmem_ld32(tmem + lane_off + kColS + hc, *reinterpret_cast<uint32_t(*)[32]>(sr));
          sm100::tmem_ld32(tmem + lane_off + kColS + hc + 32, *reinterpret_cast<uint32_t(*)[32]>(sr + 32));
          sm100::tmem_wait_ld();
          sm100::tc_fence_before();
          sm100::mbar_arrive(&sm.s_free);
          HLA_PADD(4, ts0);
          const float* s = reinterpret_cast<const float*>(sr);
          float m8[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) m8[j] = s[j];
#pragma unroll
          for (int c = 8; c < 64; ++c) m8[c & 7] = fmaxf(m8[c & 7], s[c]);
#pragma unroll
          for (int j = 4; j > 0; j >>= 1)
#pragma unroll
            for (int i = 0; i < j; ++i) m8[i] = fmaxf(m8[i], m8[i + j]);
          const float m_tile = m8[0] * sl2;
          const float m_new = (m_tile > m_ref + 8.f) ? m_tile : m_ref;
          const float alpha = (m_new == m_ref) ? 1.f : sm100::ex2(m_ref - m_new);
          m_ref = m_new;
          l *= alpha;
          const float m_use = (m_ref == -INFINITY) ? 0.f : m_ref;
          float l4[4] = {0.f, 0.f, 0.f, 0.f};
          uint32_t pk[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const float p0 = sm100::ex2(fmaf(s[2 * e], sl2, -m_use));
            const float p1 = sm100::ex2(fmaf(s[2 * e + 1], sl2, -m_use));
            l4[e & 3] += p0 + p1;
            pk[e] = sm100::pack_bf16(p0, p1);
          }
          l += (l4[0] + l4[1]) + (l4[2] + l4[3]);
          HLA_PADD(5, ts0);
          if (g > 0) {
            HLA_PW(6, sm100::mbar_wait(&sm.pv_done, (g - 1) & 1));
            sm100::tc_fence_after();
          }
          HLA_PMARK(tst0);
          if (__any_sync(0xffffffffu, t > 0 && alpha != 1.f)) {
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
              uint32_t o[32];
              sm100::tmem_ld16(tmem + lane_off + kColO + obuf + c * 32, o);
              sm100::tmem_ld16(tmem + lane_off + kColO + obuf + c * 32 + 16, o + 16);
              sm100::tmem_wait_ld();
#pragma unroll
              for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
              sm100::tmem_st16(tmem + lane_off + kColO + obuf + c * 32, o);
              sm100::tmem_st16(tmem + lane_off + kColO + obuf + c * 32 + 16, o + 16);
            }
          }
          uint32_t z[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) z[e] = 0u;
          const uint32_t pl = kColP + hc / 2, pd = kColP + (64u - hc) / 2;   // live / dead P columns
          sm100::tmem_st16(tmem + lane_off + pl, pk);
          sm100::tmem_st16(tmem + lane_off + pl + 16, pk + 16);
          sm100::tmem_st16(tmem + lane_off + pd, z);
          sm100::tmem_st16(tmem + lane_off + pd + 16, z);
          sm100::tmem_wait_st();
          sm100::tc_fence_before();
          sm100::mbar_arrive(&sm.p_full);
          if (o_double<D>() && pend) run_pending();
          HLA_PADD(7, tst0);
          continue;
        }
        // partial tile that misses all 32 rows of this warp (1D windows: the warps away
        // from the window's edge): no S load, mask or exponentials -- P rows of zero
        if ((tm & 3) == 2 &&
            __all_sync(0xffffffffu, !real || row_misses_tile<kTwoD>(prm.pat, box, (tm >> 2) * prm.col_mul))) {
          sm100::tc_fence_before();
          sm100::mbar_arrive(&sm.s_free);   // after s_full(g): phases of the S handshake stay in step
          if (g > 0) {
            sm100::mbar_wait(&sm.pv_done, (g - 1) & 1);
            sm100::tc_fence_after();
          }
          uint32_t z[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) z[e] = 0u;
#pragma unroll
          for (int c = 0; c < 4; ++c) sm100::tmem_st16(tmem + lane_off + kColP + c * 16, z);
          sm100::tmem_wait_st();
          sm100::tc_fence_before();
          sm100::mbar_arrive(&sm.p_full);
          if (o_double<D>() && pend) run_pending();
          continue;
        }
        // the whole S row: four loads in flight, one wait (TMEM round trip ~200 cycles)
        uint32_t sr[kBlock];
#pragma unroll
        for (int c = 0; c < 4; ++c)
          sm100::tmem_ld32(tmem + lane_off + kColS + c * 32, *reinterpret_cast<uint32_t(*)[32]>(sr + c * 32));
        sm100::tmem_wait_ld();
        if (row == 0) HLA_TR((6 << 24) | (1 << 16) | g);
        sm100::tc_fence_before();
        sm100::mbar_arrive(&sm.s_free);          // the MMA may overwrite S with S(g+1)
        HLA_PADD(4, ts0);
        float (&s)[kBlock] = *reinterpret_cast<float(*)[kBlock]>(sr);
        // kBias: scores move to the log2 domain here (s = S * scale * log2e + bias * log2e)
        // so that the mask, the max and the exponentials see the biased score
        const float sl2e = kBias ? 1.f : sl2;
        if constexpr (kBias) {
          // key offsets B_k staged with K (warp-uniform 16-B loads); the k_full phase of this
          // tile is complete (S used it) -- the wait makes the producer's writes visible
          sm100::mbar_wait(&sm.k_full[g & 1], (g >> 1) & 1);
          const uint32_t kbo = sm100::smem_u32(sm.key_b[g & 1]);
#pragma unroll
          for (int c4 = 0; c4 < kBlock / 4; ++c4) {
            const float4 o = sm100::lds_f4(kbo + 16u * c4);
            const int32_t ov[4] = {__float_as_int(o.x), __float_as_int(o.y), __float_as_int(o.z), __float_as_int(o.w)};
#pragma unroll
            for (int j = 0; j < 4; ++j)
              s[4 * c4 + j] = fmaf(s[4 * c4 + j], sl2, __ldg(rpbh + (a_q - ov[j])) * 1.4426950408889634f);
          }
        }
        if ((tm & 3) == 2) apply_row_mask<kTwoD>(s, prm.pat, box, (tm >> 2) * prm.col_mul);
        // row max with 8 independent chains (a single dependent chain costs ~4 cycles x 128)
        float m8[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) m8[j] = s[j];
#pragma unroll
        for (int c = 8; c < kBlock; ++c) m8[c & 7] = fmaxf(m8[c & 7], s[c]);
#pragma unroll
        for (int j = 4; j > 0; j >>= 1)
#pragma unroll
          for (int i = 0; i < j; ++i) m8[i] = fmaxf(m8[i], m8[i + j]);
        const float m_tile = m8[0] * sl2e;
        if (row == 0) HLA_TR((6 << 24) | (2 << 16) | g);
        // lazy rescale (exact): keep the reference max unless it grew by > 8 (x256)
        const float m_new = (m_tile > m_ref + 8.f) ? m_tile : m_ref;
        const float alpha = (m_new == m_ref) ? 1.f : sm100::ex2(m_ref - m_new);
        m_ref = m_new;
        l *= alpha;
        const float m_use = (m_ref == -INFINITY) ? 0.f : m_ref;
        float l4[4] = {0.f, 0.f, 0.f, 0.f};
        uint32_t pk[64];
#pragma unroll
        for (int e = 0; e < 64; ++e) {
          // all exponentials on the MUFU pipe: a polynomial exp2 on the FMA pipe for part of
          // them (FA4's split) measured slower here
          const float p0 = sm100::ex2(fmaf(s[2 * e], sl2e, -m_use));
          const float p1 = sm100::ex2(fmaf(s[2 * e + 1], sl2e, -m_use));
          l4[e & 3] += p0 + p1;
          pk[e] = sm100::pack_bf16(p0, p1);
        }
        l += (l4[0] + l4[1]) + (l4[2] + l4[3]);
        if (row == 0) HLA_TR((6 << 24) | (3 << 16) | g);
        // P(g-1) / O are read by PV(g-1): wait for it before writing P(g) or rescaling O
        HLA_PADD(5, ts0);
        if (g > 0) {
          HLA_PW(6, sm100::mbar_wait(&sm.pv_done, (g - 1) & 1));
          sm100::tc_fence_after();
        }
        HLA_PMARK(tst0);
        if (row == 0) HLA_TR((6 << 24) | (4 << 16) | g);
        if (__any_sync(0xffffffffu, t > 0 && alpha != 1.f)) {
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            sm100::tmem_ld16(tmem + lane_off + kColO + obuf + c * 32, o);
            sm100::tmem_ld16(tmem + lane_off + kColO + obuf + c * 32 + 16, o + 16);
            sm100::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            sm100::tmem_st16(tmem + lane_off + kColO + obuf + c * 32, o);
            sm100::tmem_st16(tmem + lane_off + kColO + obuf + c * 32 + 16, o + 16);
          }
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) sm100::tmem_st16(tmem + lane_off + kColP + c * 16, pk + c * 16);
        sm100::tmem_wait_st();
        sm100::tc_fence_before();
        sm100::mbar_arrive(&sm.p_full);
        if (o_double<D>() && pend) run_pending();
        HLA_PADD(7, tst0);
        if (row == 0) HLA_TR((2 << 24) | (2 << 16) | g);
      }

      // epilogue: O / l -> bf16 row, LSE (natural log); phantom rows (q >= N) write nothing
      const int64_t orow = ((int64_t)b * prm.N + ocell) * prm.heads + h;
      uint4* optr = reinterpret_cast<uint4*>(prm.o + orow * D);
      const float inv_l = l > 0.f ? 1.f / l : 0.f;
      if constexpr (o_double<D>()) {
        // deferred (run_pending after the next unit's first P store); the Q stage is free now
        pend = true;
        pend_ob = obuf;
        pend_inv_l = inv_l;
        pend_optr = real ? reinterpret_cast<unsigned long long>(optr) : 0ull;
        pend_staged = (qb + 1) * kBlock <= prm.N;
        pend_c = __shfl_sync(0xffffffffu, ocell, 0);
        pend_h = h;
        pend_b = b;
        sm100::mbar_arrive(&sm.o_staged[it.n & 1]);
        const float m_use = (m_ref == -INFINITY) ? 0.f : m_ref;
        if (real)
          prm.lse[((int64_t)b * prm.heads + h) * prm.N + q] =
              l > 0.f ? (m_use + __log2f(l)) * 0.69314718055994530942f : -INFINITY;
        tiles_done += it.nt;
        it.t = it.nt - 1;
        it.advance(prm.row_ptr, prm.mq_div, units);
        if (it.valid) {
          meta = it.from_pf ? (pm.c << 2) | pm.k : load_meta(prm.col_idx, prm.kind, it.rs, it.nt, lane);
          pm = load_meta_raw(prm.col_idx, prm.kind, it.prs, it.pre - it.prs, lane);
        }
        continue;
      }
      HLA_PW(8, sm100::mbar_wait(&sm.o_full, it.n & 1));
      HLA_PMARK(te0);
      if (row == 0) HLA_TR((2 << 24) | (3 << 16) | it.n);
      sm100::tc_fence_after();
      uint32_t o[D];
#pragma unroll
      for (int c = 0; c < D / 32; ++c)
        sm100::tmem_ld32(tmem + lane_off + kColO + c * 32, *reinterpret_cast<uint32_t(*)[32]>(o + c * 32));
      sm100::tmem_wait_ld();
      // TMEM O may now be overwritten by the next unit's first PV (it waits p_full).
      // Full tiles: the bf16 row goes into this unit's Q stage (all S MMAs of the unit
      // are done), swizzled like a TMA-loaded tile; the producer stores the tile with one
      // TMA store / 32 scatter4 (full 128-B lines, no LSU store queue in this warp's way).
      // Ragged tiles: rows written directly.
      const bool staged = (qb + 1) * kBlock <= prm.N;
      const uint32_t stage = sm100::smem_u32(sm.q[it.n & 1]);
#pragma unroll
      for (int v4 = 0; v4 < D / 8; ++v4) {
        uint4 w;
        w.x = sm100::pack_bf16(__uint_as_float(o[v4 * 8 + 0]) * inv_l, __uint_as_float(o[v4 * 8 + 1]) * inv_l);
        w.y = sm100::pack_bf16(__uint_as_float(o[v4 * 8 + 2]) * inv_l, __uint_as_float(o[v4 * 8 + 3]) * inv_l);
        w.z = sm100::pack_bf16(__uint_as_float(o[v4 * 8 + 4]) * inv_l, __uint_as_float(o[v4 * 8 + 5]) * inv_l);
        w.w = sm100::pack_bf16(__uint_as_float(o[v4 * 8 + 6]) * inv_l, __uint_as_float(o[v4 * 8 + 7]) * inv_l);
        if (staged) {
          const uint32_t off = (uint32_t)row * (D * 2) + v4 * 16;
          sm100::sts_u4(stage + (D == 64 ? sm100::swz128(off) : sm100::swz64(off)), w.x, w.y, w.z, w.w);
        } else if (real) {
          optr[v4] = w;
        }
      }
      if (warp_ostore<D>() && staged) {
        // this warp's 32 staged rows back, transposed: lanes 8j .. 8j + 7 (d = 64; 4j .. 4j + 3 at
        // d = 32) hold one row's 16-B chunks, so each STG.128 writes whole 128-B (64-B) rows
        __syncwarp();
        constexpr int kCh = D / 8;                 // 16-B chunks per row
        constexpr int kRowsPer = 32 / kCh;         // rows per warp instruction
        const unsigned long long op = real ? reinterpret_cast<unsigned long long>(optr) : 0ull;
#pragma unroll
        for (int k = 0; k < 32 / kRowsPer; ++k) {
          const int rl = lane / kCh + kRowsPer * k, c = lane % kCh;
          const uint32_t off = (uint32_t)(quarter * 32 + rl) * (D * 2) + (uint32_t)c * 16u;
          const float4 v = sm100::lds_f4(stage + (D == 64 ? sm100::swz128(off) : sm100::swz64(off)));
          const unsigned long long p = __shfl_sync(0xffffffffu, op, rl);
          if (p)
            reinterpret_cast<uint4*>(p)[c] =
                make_uint4(__float_as_uint(v.x), __float_as_uint(v.y), __float_as_uint(v.z), __float_as_uint(v.w));
        }
      }
      sm100::fence_proxy_async_smem();
      sm100::mbar_arrive(&sm.o_staged[it.n & 1]);   // (warp_ostore<D>(): the Q stage is free again)
      if (row == 0) HLA_TR((2 << 24) | (4 << 16) | it.n);
      const float m_use = (m_ref == -INFINITY) ? 0.f : m_ref;
      if (real)
        prm.lse[((int64_t)b * prm.heads + h) * prm.N + q] =
            l > 0.f ? (m_use + __log2f(l)) * 0.69314718055994530942f : -INFINITY;
      HLA_PADD(9, te0);
      tiles_done += it.nt;
      it.t = it.nt - 1;
      it.advance(prm.row_ptr, prm.mq_div, units);
      if (it.valid) {
        meta = it.from_pf ? (pm.c << 2) | pm.k : load_meta(prm.col_idx, prm.kind, it.rs, it.nt, lane);
        pm = load_meta_raw(prm.col_idx, prm.kind, it.prs, it.pre - it.prs, lane);
      }
      HLA_PADD(10, te0);
      if (row == 0) HLA_TR((2 << 24) | (5 << 16) | it.n);
    }
    if (o_double<D>() && pend) {   // the last unit: its final PV (tile g - 1) must be complete
      sm100::mbar_wait(&sm.pv_done, (g - 1) & 1);
      sm100::tc_fence_after();
      run_pending();
    }
    if (o_double<D>() && sq_store && lane == 0) sm100::bulk_wait_group0();   // stores done before exit
    HLA_PFLUSH(3, 11, warp == 4 && lane == 0);
    HLA_PFLUSH(19, 20, warp == 4 && lane == 0);
    if (warp == 4 && lane == 0 && prm.visited != nullptr && tiles_done > 0) atomicAdd(prm.visited, tiles_done);
  }

  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (warp == 1) sm100::tmem_dealloc(sm.tmem_base, kTmemCols);
}

template <int D, bool kTwoD, bool kGather, bool kBias, bool kHalf = false>
hla_status launch_fwd(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv, const CUtensorMap& mo,
                      const FwdParams& prm, int32_t n_qblocks, cudaStream_t stream) {
  const size_t smem = sizeof(FwdSmem<D, kBias>) + 1024;
  auto* fn = attn_fwd_kernel<D, kTwoD, kGather, kBias, kHalf>;
  HLA_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t units = (int64_t)n_qblocks * prm.heads * prm.batch;
  const int grid = (int)std::min<int64_t>((units + 1) / 2, 2 * (int64_t)num_sms());   // pairs of units
  fn<<<grid, kThreads, smem, stream>>>(mq, mk, mv, mo, prm);
  HLA_CUDA_TRY(cudaGetLastError());
  return HLA_OK;
}

template <bool kBias>
hla_status dispatch_fwd(int head_dim, bool gather, bool two_d, const CUtensorMap& mq, const CUtensorMap& mk,
                        const CUtensorMap& mv, const CUtensorMap& mo, const FwdParams& prm, int32_t mqb,
                        cudaStream_t stream) {
  if (head_dim == 64) {
    if constexpr (!kBias) {
      if (gather && prm.pat.kind == K_HWA && prm.pat.n == 64)   // half-row softmax (see below)
        return launch_fwd<64, false, true, false, true>(mq, mk, mv, mo, prm, mqb, stream);
    }
    if (gather) return launch_fwd<64, false, true, kBias>(mq, mk, mv, mo, prm, mqb, stream);
    return two_d ? launch_fwd<64, true, false, kBias>(mq, mk, mv, mo, prm, mqb, stream)
                 : launch_fwd<64, false, false, kBias>(mq, mk, mv, mo, prm, mqb, stream);
  }
  if constexpr (!kBias) {
    // HWA with 64-token windows: the half-row softmax instantiation (attn_fwd_kernel kHalf); every
    // list entry is then the diagonal window pair of its 128-row tile (block 128: kv-block i of
    // q-block i; block 64: the window (2t, 2t + 1) of tile t)
    if (gather && prm.pat.kind == K_HWA && prm.pat.n == 64)
      return launch_fwd<32, false, true, false, true>(mq, mk, mv, mo, prm, mqb, stream);
  }
  if (gather) return launch_fwd<32, false, true, kBias>(mq, mk, mv, mo, prm, mqb, stream);
  return two_d ? launch_fwd<32, true, false, kBias>(mq, mk, mv, mo, prm, mqb, stream)
               : launch_fwd<32, false, false, kBias>(mq, mk, mv, mo, prm, mqb, stream);
}

}  // namespace

// shared argument validation of forward and backward (declared in attn_common.cuh)
hla_status check_attn_args(const hla_pattern_desc* d, const hla_block_mask* m, int32_t batch, int32_t heads,
                           int32_t head_dim, Pattern* pat, AttnLists* L) {
  hla_status st = make_pattern(d, pat);
  if (st != HLA_OK) return st;
  HLA_REQUIRE(m != nullptr && m->row_ptr && m->col_idx && m->kind, HLA_ERR_INVALID, "mask arrays missing");
  HLA_REQUIRE(head_dim == 32 || head_dim == 64, HLA_ERR_UNSUPPORTED, "head_dim %d not in {32, 64}", head_dim);
  HLA_REQUIRE(d->block_q == d->block_k && (d->block_q == 128 || d->block_q == 64), HLA_ERR_UNSUPPORTED,
              "attention needs block_q == block_k in {64, 128} (got %d, %d)", d->block_q, d->block_k);
  HLA_REQUIRE(pat->N % 4 == 0, HLA_ERR_UNSUPPORTED, "N=%d not a multiple of 4", pat->N);
  const int32_t b = d->block_q;
  const int32_t nb = (pat->N + b - 1) / b;   // ragged last block: phantom rows masked / not written
  HLA_REQUIRE(m->n_qblocks == nb && m->n_kblocks == nb, HLA_ERR_INVALID,
              "mask built for a different N / block");
  HLA_REQUIRE(batch >= 1 && batch <= 65535 && heads >= 1 && heads <= 65535, HLA_ERR_INVALID,
              "batch %d / heads %d out of range", batch, heads);
  if (b == 128) {
    *L = AttnLists{m->row_ptr, m->col_idx, m->kind, m->t_row_ptr, m->t_col_idx, m->t_kind, 128,
                   m->host_counts[1], m->host_counts[2], m->host_counts[1], m->host_counts[2]};
  } else {
    HLA_REQUIRE(m->w_row_ptr && m->w_col && m->w_kind && m->wt_row_ptr && m->wt_col && m->wt_kind, HLA_ERR_INVALID,
                "block 64 needs the mask's window lists (hla_build_tile_lists)");
    *L = AttnLists{m->w_row_ptr, m->w_col, m->w_kind, m->wt_row_ptr, m->wt_col, m->wt_kind, 64,
                   m->w_counts[1], m->w_counts[0] - m->w_counts[1], m->w_counts[3], m->w_counts[2] - m->w_counts[3]};
  }
  return HLA_OK;
}

hla_status parse_score_mod(const hla_pattern_desc* d, const hla_score_mod* mod, bool bwd, const float** rpb,
                           float** drpb, const int32_t** cells) {
  *rpb = nullptr;
  *cells = nullptr;
  if (drpb) *drpb = nullptr;
  if (mod == nullptr || mod->kind == HLA_SCORE_NONE) return HLA_OK;
  HLA_REQUIRE(mod->kind == HLA_SCORE_GLOBAL_RPB, HLA_ERR_UNSUPPORTED, "score_mod kind %d not supported", mod->kind);
  HLA_REQUIRE(mod->rpb != nullptr, HLA_ERR_INVALID, "score_mod: rpb table is null");
  HLA_REQUIRE(d->order == HLA_ORDER_ROW_MAJOR || mod->seq_to_cell != nullptr, HLA_ERR_INVALID,
              "score_mod: Hilbert order needs seq_to_cell for the 2D offsets");
  HLA_REQUIRE(((uintptr_t)mod->seq_to_cell & 15) == 0, HLA_ERR_INVALID, "score_mod: seq_to_cell must be 16-byte aligned");
  HLA_REQUIRE(!bwd || mod->drpb != nullptr, HLA_ERR_INVALID, "score_mod: drpb (table gradient) is null");
  *rpb = mod->rpb;
  *cells = mod->seq_to_cell;
  if (drpb) *drpb = mod->drpb;
  return HLA_OK;
}

}  // namespace hla

using namespace hla;

#ifdef HLA_FWD_PROF
// dev-only: per-CTA wait / work cycle sums of the last attn_fwd_kernel launch (HLA_FWD_PROF builds)
extern "C" __attribute__((visibility("default"))) int hla_debug_fwd_prof(unsigned long long* host, int ctas) {
  cudaDeviceSynchronize();
  const int n = ctas < 1024 ? ctas : 1024;
  cudaMemcpyFromSymbol(host, hla::g_fwd_prof, (size_t)n * 24 * sizeof(unsigned long long));
  return n;
}
#endif

extern "C" hla_status hla_attn_fwd(const hla_pattern_desc* d, const hla_block_mask* m, int32_t batch, int32_t heads,
                                   int32_t head_dim, float scale, const void* q, const void* k, const void* v,
                                   void* o, float* lse, const int32_t* seq_to_cell,
                                   const hla_score_mod* score_mod, int64_t* tiles_visited, cudaStream_t stream) {
  clear_error();
  Pattern pat;
  AttnLists lists;
  hla_status st = check_attn_args(d, m, batch, heads, head_dim, &pat, &lists);
  if (st != HLA_OK) return st;
  HLA_REQUIRE(q && k && v && o && lse, HLA_ERR_INVALID, "null tensor pointer");
  HLA_REQUIRE((((uintptr_t)q | (uintptr_t)k | (uintptr_t)v | (uintptr_t)o) & 15) == 0, HLA_ERR_INVALID,
              "tensors must be 16-byte aligned");
  const float sc = scale > 0.f ? scale : 1.0f / sqrtf((float)head_dim);
  FwdParams prm;
  prm.pat = pat;
  prm.N = pat.N;
  prm.heads = heads;
  prm.batch = batch;
  prm.mq_div = make_fastdiv((pat.N + kBlock - 1) / kBlock);
  prm.heads_div = make_fastdiv(heads);
  prm.scale_log2 = sc * 1.4426950408889634f;
  prm.row_ptr = lists.row_ptr;
  prm.col_idx = lists.col;
  prm.kind = lists.kind;
  prm.col_mul = lists.col_mul;
  prm.o = reinterpret_cast<__nv_bfloat16*>(o);
  prm.lse = lse;
  prm.s2c = seq_to_cell;
  if ((st = parse_score_mod(d, score_mod, false, &prm.rpb, nullptr, &prm.cells)) != HLA_OK) return st;
  prm.grid_h = pat.H;
  prm.grid_w = pat.W;
  prm.rpb_w = 2 * pat.W - 1;
  prm.rpb_hw = (2 * pat.H - 1) * prm.rpb_w;
  prm.rpb_a0 = (pat.H - 1) * prm.rpb_w + (pat.W - 1);
  prm.visited = reinterpret_cast<unsigned long long*>(tiles_visited);
  const bool two_d = pat.kind == K_WSA || pat.kind == K_SA || pat.kind == K_NA2D;
  const bool gather = seq_to_cell != nullptr;
  HLA_REQUIRE(!gather || d->order != HLA_ORDER_ROW_MAJOR, HLA_ERR_INVALID,
              "seq_to_cell (fused reorder) is only meaningful for Hilbert-order patterns");
  HLA_REQUIRE(!gather || ((uintptr_t)seq_to_cell & 15) == 0, HLA_ERR_INVALID, "seq_to_cell must be 16-byte aligned");
  prm.box8 = (gather && d->order == HLA_ORDER_HILBERT_TILED && head_dim == 32) ? ilog2(pat.W) + 1 : 0;
  const int64_t rows = (int64_t)batch * pat.N;
  CUtensorMap mq, mk, mv, mo;
  if (gather) {
    if ((st = prm.box8 ? make_square_map(&mo, o, batch, pat.H, pat.W, heads, head_dim, 4)
                       : make_gather_map(&mo, o, rows, heads, head_dim)) != HLA_OK)
      return st;
    auto mk_map = [&](CUtensorMap* mp, const void* base) {
      return prm.box8 ? make_square_map(mp, base, batch, pat.H, pat.W, heads, head_dim)
                      : make_gather_map(mp, base, rows, heads, head_dim);
    };
    if ((st = mk_map(&mq, q)) != HLA_OK) return st;
    if ((st = mk_map(&mk, k)) != HLA_OK) return st;
    if ((st = mk_map(&mv, v)) != HLA_OK) return st;
  } else {
    if ((st = make_rows_map(&mo, o, rows, heads, head_dim, kBlock)) != HLA_OK) return st;
    if ((st = make_rows_map(&mq, q, rows, heads, head_dim, kBlock)) != HLA_OK) return st;
    if ((st = make_rows_map(&mk, k, rows, heads, head_dim, kBlock)) != HLA_OK) return st;
    if ((st = make_rows_map(&mv, v, rows, heads, head_dim, kBlock)) != HLA_OK) return st;
  }
  const int32_t mqb = (pat.N + kBlock - 1) / kBlock;
  return prm.rpb ? dispatch_fwd<true>(head_dim, gather, two_d, mq, mk, mv, mo, prm, mqb, stream)
                 : dispatch_fwd<false>(head_dim, gather, two_d, mq, mk, mv, mo, prm, mqb, stream);
}
