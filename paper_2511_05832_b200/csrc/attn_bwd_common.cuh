// Shared pieces of the two backward schedules (attn_bwd.cu: full-tile schedule and the
// host API; attn_bwd_split.cu: half-tile schedule).  Internal header of libhla.
#pragma once

#include "predicates.cuh"
#include "sm100.cuh"
#include "tensor_map.cuh"

namespace hla {
namespace bwd {

constexpr int kBlock = 128;
constexpr uint32_t kTmemCols = 512;
constexpr float kLog2e = 1.4426950408889634f;

struct BwdParams {
  Pattern pat;
  int32_t N, heads, batch;
  FastDiv mk_div, ppb_div, heads_div;   // kv-blocks per (b, h), kv-block pairs per (b, h), heads
  float scale, scale_log2, inv_scale;
  const int32_t* t_row_ptr;   // tile lists (AttnLists): per 128-key tile
  const int32_t* t_col_idx;
  const uint8_t* t_kind;
  int32_t col_mul;            // start row of a list entry = column * col_mul (128, or 64: windows)
  const uint8_t* t_dq;     // dQ chaining plan per transposed entry (HLA_DQ_*; null = one chain per tile)
  const float* lse2;       // LSE * log2(e), [B, H, N] (workspace, from the preprocess)
  const float* dsum;       // D * scale, [B, H, N] (workspace, from the preprocess)
  float* dq_acc;           // [B, N, H, Dh] fp32 (grid order when s2c != null)
  const int32_t* s2c;      // fused reorder: seq_to_cell table (tensors in grid order), else null
  int32_t box8;            // d = 32, tiled Hilbert order: log2(W) + 1 (0 = off): square-box loads (load_rows)
  const float* rpb;        // global RPB table [heads][2H-1][2W-1] (kBias)
  float* drpb;             // its gradient (accumulated)
  const int32_t* cells;    // grid cell of each sequence position (null: identity)
  int32_t grid_h, grid_w, rpb_w, rpb_hw;
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
  __nv_bfloat16* dq;       // dQ rows of LOCAL chains (bf16, same layout as dk)
  unsigned long long* visited;
};

// Global-RPB table gradient (reading R19/R20).  Each tile's pairs are accumulated per 2D
// offset in a shared-memory window (the offset rows of the tile's cell box at the table's
// row stride 2W - 1) and flushed to the table with fp32 global reductions.  Entries of
// the window.  More at D = 32, where the smaller tiles leave room.
template <int D>
constexpr int rpb_win_cap() { return D == 32 ? 4096 : 2048; }
// The window accumulates in 32-bit fixed point (shared-memory fp32 / 64-bit atomics are
// compare-and-swap loops on sm_100, ATOMS.CAST.SPIN in SASS; 32-bit integer ATOMS.ADD is
// native) at a power-of-two scale relative to the largest |dL/dscore| of a tile: every
// addend below 2^22 and at most 128 pairs of a 128 x 128 tile per offset (one per key) keep
// an entry below 2^29; the resolution is 2^-22 of that largest addend, independent of the
// gradient's absolute magnitude.
constexpr int kRpbFixBits = 22;
constexpr float kRpbFixMax = 4194304.f;   // 2^kRpbFixBits: larger scaled addends go to global fp32 atomics
// scale whose largest addend (for the maximum tmx) lies in [2^(kRpbFixBits-1), 2^kRpbFixBits)
__device__ __forceinline__ float rpb_scale_for(float tmx, float fallback) {
  return tmx > 0.f ? ldexpf(1.f, kRpbFixBits - 1 - ilogbf(tmx)) : fallback;
}
// the next tile's scale from the eight compute warps' maxima of a tile (half-tile schedule)
__device__ __forceinline__ float rpb_next_scale(const float* wmax8, float cur) {
  float m = 0.f;
#pragma unroll
  for (int w = 0; w < 8; ++w) m = fmaxf(m, wmax8[w]);
  return rpb_scale_for(m, cur);
}

// Kernel launch of one schedule for the head_dim / reorder / 2D-pattern variant; the maps
// view Q, K, V, dO as bf16 rows and the fp32 dQ accumulator (see hla_attn_bwd_main).
// (the full-tile schedule has no global-RPB path: RPB layers take the half-tile schedule;
// fuse: preprocess folded into the kernel, every dQ chain local, mdq = the O map, lse2 = raw LSE)
hla_status launch_full(int head_dim, bool gather, bool two_d, bool fuse, const CUtensorMap& mq, const CUtensorMap& mk,
                       const CUtensorMap& mv, const CUtensorMap& mdo, const CUtensorMap& mdq, const BwdParams& prm,
                       int32_t n_kblocks, cudaStream_t stream);
hla_status launch_split(bool bias, int head_dim, bool gather, bool two_d, bool fuse, const CUtensorMap& mq,
                        const CUtensorMap& mk, const CUtensorMap& mv, const CUtensorMap& mdo, const CUtensorMap& mdq,
                        const CUtensorMap& mo, const BwdParams& prm, int32_t n_kblocks, cudaStream_t stream);

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
// TMEM column of the packed bf16 P^T (A of dV += P^T dO) for K step kk (16 q): the compute
// thread of 32-column chunk c writes its 32 values over the chunk's first 16 S^T columns
__device__ __forceinline__ uint32_t packed_col(int kk) { return (uint32_t)((kk >> 1) * 32 + (kk & 1) * 8); }
// dS^T smem tile viewed as K-major A of dK += dS^T Q (M = kv, K = q): K step = 16 q
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
  FastDiv mkd, ppbd;        // division by mk / ppb (multiply-shift)
};
// k-th kv-block of this CTA: flattened u = (b * heads + h) * mk + kb, kUnitSkip for
// the missing second block of a ragged last pair, kUnitEnd past the last pair
__device__ __forceinline__ int32_t unit_at(int32_t k, const UnitGeom& ug) {
  const int32_t P = (int32_t)blockIdx.x + (k >> 1) * (int32_t)gridDim.x;
  if (P >= ug.pairs) return kUnitEnd;
  const int32_t bh = ug.ppbd.div(P);
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
      const int32_t kb = u - ug.mkd.div(u) * ug.mk;
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
// sq (d = 32, HLA_ORDER_HILBERT_TILED; log2(grid_w) + 1, 0 = off): every aligned 64 sequence
// positions are an aligned 8 x 8 cell square in raster order, so 2 lanes each move one square with
// a 5-D box (`map` from make_square_map) instead of 32 gather4 ops of 4 x 64-B rows -- at d = 32
// the per-op cost of the TMA unit, not the bytes, bounds the loads.  A square past N (ragged
// last tile) loads the square at cell 0.
template <int D, bool kGather>
__device__ __forceinline__ void load_rows(uint8_t* dst, const CUtensorMap* map, uint64_t* bar, int32_t h,
                                          int32_t b, int32_t N, int32_t seq0, const int32_t* s2c, uint64_t pol,
                                          int lane, int sq) {
  if (kGather) {
    if (D == 32 && sq) {
      if (lane < 2) {
        const int32_t c = seq0 + 64 * lane < N ? __ldg(s2c + seq0 + 64 * lane) : 0;
        const int32_t lw = sq - 1;
        sm100::tma_load_5d(dst + lane * 64 * D * 2, map, bar, 0, h, c & ((1 << lw) - 1), c >> lw, b, pol);
      }
      return;
    }
    // rows past N (ragged last tile) gather cell 0: their values are masked / discarded
    const int4 c = seq0 + 4 * lane < N ? __ldg(reinterpret_cast<const int4*>(s2c + seq0) + lane) : make_int4(0, 0, 0, 0);
    const int32_t base = b * N;
    sm100::tma_gather4(dst + lane * 4 * D * 2, map, bar, h * D, base + c.x, base + c.y, base + c.z, base + c.w, pol);
  } else if (lane == 0) {
    sm100::tma_load_3d(dst, map, bar, 0, h, b * N + seq0, pol);
  }
}

// Rows held by one warp (thread = row: D / 2 packed bf16x2 words, one 2D-byte row at `rowp`, null
// = phantom row) stored through a per-warp shared-memory transpose, so that every STG.128 of the
// warp writes 8 rows x 64 contiguous bytes instead of 32 rows x 16 bytes (the row stores were
// bound by 16-byte segments, ~1 per cycle).  stage: this warp's 2 KB (shared address).
template <int D>
__device__ __forceinline__ void store_rows_t(const uint32_t* w, uint4* rowp, uint32_t stage, int lane) {
  const unsigned long long pr = reinterpret_cast<unsigned long long>(rowp);
#pragma unroll
  for (int seg = 0; seg < D / 32; ++seg) {
    // this lane's 64-byte segment -> stage row `lane`, 16-byte slots rotated by lane / 2 (the 8
    // lanes of each STS.128 / LDS.128 phase hit 8 distinct slots of 128 bytes: no bank conflict)
#pragma unroll
    for (int c = 0; c < 4; ++c)
      sm100::sts_u4(stage + lane * 64 + 16 * ((c + (lane >> 1)) & 3), w[seg * 16 + 4 * c], w[seg * 16 + 4 * c + 1],
                    w[seg * 16 + 4 * c + 2], w[seg * 16 + 4 * c + 3]);
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = (lane >> 2) + 8 * k, c = lane & 3;
      const float4 v = sm100::lds_f4(stage + r * 64 + 16 * ((c + (r >> 1)) & 3));
      const unsigned long long p = __shfl_sync(0xffffffffu, pr, r);
      if (p)
        reinterpret_cast<uint4*>(p)[seg * 4 + c] =
            make_uint4(__float_as_uint(v.x), __float_as_uint(v.y), __float_as_uint(v.z), __float_as_uint(v.w));
    }
    __syncwarp();
  }
}

// Preprocess folded into the kernel (kFuse): D * scale = rowsum(dO o O) * scale and the log2-domain
// LSE of a newly loaded q-block, formed in place in its stage by the 256 compute threads (two per
// query row, half a row each; t = 0 .. 255) from the O tile and the stage's dO tile (swizzled rows
// as loaded by TMA).  The caller synchronises the 256 threads afterwards.
template <int D>
__device__ __forceinline__ void form_d(uint32_t ostage, uint32_t dostage, float* dd, float* lse, int t,
                                       int32_t real_rows, float scale) {
  const int r = t >> 1, hf = t & 1;
  float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
  for (int j = 0; j < D / 16; ++j) {
    const uint32_t off = (uint32_t)r * (D * 2) + (uint32_t)(hf * (D / 16) + j) * 16u;
    const uint32_t so = D == 64 ? sm100::swz128(off) : sm100::swz64(off);
    const float4 a = sm100::lds_f4(ostage + so), c = sm100::lds_f4(dostage + so);
    const float av[4] = {a.x, a.y, a.z, a.w}, cv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t aw = __float_as_uint(av[e]), cw = __float_as_uint(cv[e]);
      acc0 = fmaf(__uint_as_float(aw << 16), __uint_as_float(cw << 16), acc0);
      acc1 = fmaf(__uint_as_float(aw & 0xffff0000u), __uint_as_float(cw & 0xffff0000u), acc1);
    }
  }
  float acc = acc0 + acc1;
  acc += __shfl_xor_sync(0xffffffffu, acc, 1);
  if (hf == 0) {
    dd[r] = acc * scale;
    if (r < real_rows) lse[r] *= kLog2e;   // raw LSE -> log2 domain (phantom rows: never loaded)
  }
}
constexpr uint32_t kBarFormD = 4;   // named barrier of the 256 compute threads after form_d

// cell -> (row << 16) | col (RPB offsets; grid sides < 2^15)
__device__ __forceinline__ int32_t rpb_cell_rc(const int32_t* cells, int32_t seq, int32_t N, const FastDiv& W) {
  const int32_t cell = seq < N ? (cells ? __ldg(cells + seq) : seq) : 0;
  const int32_t r = W.div(cell);
  return (r << 16) | (cell - r * W.d);
}
// min / max of the rows and columns of the cells of sequence block [s0, s0 + 128)
// (phantom positions >= N ignored); identical in every lane.
struct CellBox { int32_t r0, r1, c0, c1; };
__device__ __forceinline__ CellBox rpb_block_box(const int32_t* cells, int32_t s0, int32_t N, const FastDiv& W,
                                                 int lane) {
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

}  // namespace bwd
}  // namespace hla
