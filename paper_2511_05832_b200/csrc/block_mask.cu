// K3-K5: block-mask builder.  Classifies every b_q x b_k tile of the N x N
// attention matrix as full / partial / empty and emits CSR lists per
// q-block (forward) and their transpose per kv-block (backward), plus counts.
//
// Method: brute-force predicate evaluation with warp ballots and early exit
// (a tile is proven partial as soon as one allowed and one denied pair are
// seen).  This is deliberately a different algorithm from the oracle's
// interval counter.  One CTA per "line" (a q-block row or a kv-block column):
// the line's tile kinds are staged in shared memory, then counted (sizing pass)
// or compacted in ascending order (fill pass).  The library owns no scratch
// memory, so lines are re-classified in each pass (not on the per-step path;
// built once per shape like the cached Hilbert path).
#include <algorithm>
#include <vector>

#include "predicates.cuh"

namespace hla {

constexpr int kLineThreads = 256;

// Kind of tile (i, j): 0 empty, 1 full, 2 partial.  Warp-collective.
__device__ uint8_t classify_tile(const Pattern& p, int32_t i, int32_t j, int32_t bq, int32_t bk) {
  const int lane = threadIdx.x & 31;
  const int32_t q0 = i * bq, k0 = j * bk;
  const int32_t nq = min(bq, p.N - q0), nk = min(bk, p.N - k0);
  const int64_t total = (int64_t)nq * nk;
  // lane's (qq, kk) in the flattened tile, advanced by 32 per step
  int32_t qq = lane / nk, kk = lane - qq * nk;
  bool seen_allowed = false, seen_denied = false;
  for (int64_t e0 = 0; e0 < total; e0 += 32) {
    const bool valid = e0 + lane < total;
    const bool a = valid && allowed(p, q0 + qq, k0 + kk);
    const unsigned valid_mask = __ballot_sync(0xffffffffu, valid);
    const unsigned allow_mask = __ballot_sync(0xffffffffu, a);
    seen_allowed |= allow_mask != 0u;
    seen_denied |= allow_mask != valid_mask;
    if (seen_allowed && seen_denied) return 2;
    kk += 32;
    while (kk >= nk) { kk -= nk; ++qq; }
  }
  if (!seen_allowed) return 0;
  return (nq == bq && nk == bk) ? 1 : 2;   // tiles with padding positions are never full
}

// MODE 0: count (sizing).  MODE 1: fill (ascending compaction).
// Lines [0, Mq) are q-block rows, lines [Mq, Mq+Mk) are kv-block columns.
template <int MODE>
__global__ void __launch_bounds__(kLineThreads) classify_lines_kernel(
    Pattern p, int32_t bq, int32_t bk, int32_t Mq, int32_t Mk,
    int32_t* __restrict__ row_ptr, int32_t* __restrict__ col_idx, uint8_t* __restrict__ kind,
    int32_t* __restrict__ t_row_ptr, int32_t* __restrict__ t_col_idx, uint8_t* __restrict__ t_kind,
    unsigned long long* __restrict__ counts) {
  extern __shared__ uint8_t s_kind[];
  __shared__ int32_t s_warp[kLineThreads / 32];
  __shared__ int32_t s_total[3];
  const bool is_row = blockIdx.x < (unsigned)Mq;
  const int32_t line = is_row ? blockIdx.x : blockIdx.x - Mq;
  const int32_t len = is_row ? Mk : Mq;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kWarps = kLineThreads / 32;

  for (int32_t t = warp; t < len; t += kWarps) {
    const uint8_t kd = is_row ? classify_tile(p, line, t, bq, bk) : classify_tile(p, t, line, bq, bk);
    if (lane == 0) s_kind[t] = kd;
  }
  if (threadIdx.x < 3) s_total[threadIdx.x] = 0;
  __syncthreads();

  if (MODE == 0) {
    int32_t nnz = 0, nfull = 0;
    for (int32_t t = threadIdx.x; t < len; t += kLineThreads) {
      nnz += s_kind[t] != 0;
      nfull += s_kind[t] == 1;
    }
    atomicAdd(&s_total[0], nnz);
    atomicAdd(&s_total[1], nfull);
    __syncthreads();
    if (threadIdx.x == 0) {
      if (is_row) {
        row_ptr[line + 1] = s_total[0];
        atomicAdd(&counts[0], (unsigned long long)s_total[0]);
        atomicAdd(&counts[1], (unsigned long long)s_total[1]);
        atomicAdd(&counts[2], (unsigned long long)(s_total[0] - s_total[1]));
      } else {
        t_row_ptr[line + 1] = s_total[0];
      }
    }
    return;
  }

  // MODE 1: ordered compaction of the non-empty tiles of this line
  int32_t* out_idx = is_row ? col_idx : t_col_idx;
  uint8_t* out_kind = is_row ? kind : t_kind;
  int32_t base = is_row ? row_ptr[line] : t_row_ptr[line];
  for (int32_t t0 = 0; t0 < len; t0 += kLineThreads) {
    const int32_t t = t0 + threadIdx.x;
    const uint8_t kd = t < len ? s_kind[t] : 0;
    const unsigned ball = __ballot_sync(0xffffffffu, kd != 0);
    if (lane == 0) s_warp[warp] = __popc(ball);
    __syncthreads();
    int32_t before = 0, chunk_total = 0;
    for (int w = 0; w < kWarps; ++w) {
      if (w < warp) before += s_warp[w];
      chunk_total += s_warp[w];
    }
    if (kd != 0) {
      const int32_t pos = base + before + __popc(ball & ((1u << lane) - 1u));
      out_idx[pos] = t;
      out_kind[pos] = kd;
    }
    base += chunk_total;
    __syncthreads();
  }
}

// row_ptr[0] = 0 and inclusive prefix sum of the counts in row_ptr[1..n]
__global__ void __launch_bounds__(1024) scan_lines_kernel(int32_t* row_ptr, int32_t Mq, int32_t* t_row_ptr,
                                                          int32_t Mk, unsigned long long* counts) {
  int32_t* a = blockIdx.x == 0 ? row_ptr : t_row_ptr;
  const int32_t n = blockIdx.x == 0 ? Mq : Mk;
  __shared__ int32_t s_warp[32];
  __shared__ int32_t s_carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { s_carry = 0; a[0] = 0; }
  __syncthreads();
  for (int32_t c0 = 1; c0 <= n; c0 += 1024) {
    const int32_t idx = c0 + threadIdx.x;
    int32_t v = idx <= n ? a[idx] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    if (lane == 31) s_warp[warp] = v;
    __syncthreads();
    if (warp == 0) {
      int32_t w = s_warp[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t u = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += u;
      }
      s_warp[lane] = w;
    }
    __syncthreads();
    const int32_t incl = v + (warp > 0 ? s_warp[warp - 1] : 0) + s_carry;
    if (idx <= n) a[idx] = incl;
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = incl;
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) counts[3] = (unsigned long long)Mq * (unsigned long long)Mk - counts[0];
}

// Backward dQ plan (hla_build_bwd_plan): one thread per work unit = kv-block pair
// (2p, 2p+1).  Walks the unit's tiles in the order the backward kernel executes them
// (list(2p) ascending, then list(2p+1) ascending) and assigns dQ chains to the two
// TMEM accumulators: a q-block listed by both kv-blocks is held across the pair;
// a new chain takes a free accumulator (alternating), and if both are held the
// older hold is cut (its first tile drains through the fp32 workspace instead).
// (Block-64 masks: the plan runs over the attention kernels' window lists when every window
// starts on a 128-row boundary -- list entries are then 64-unit columns, col >> col_shift
// the 128-tile; see hla_build_bwd_plan.)
__global__ void bwd_plan_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ t_row_ptr,
                                const int32_t* __restrict__ t_col_idx, int32_t Mk, uint8_t* __restrict__ t_dq,
                                int col_shift) {
  const int32_t p = (int32_t)(blockIdx.x * blockDim.x + threadIdx.x);
  const int32_t j0 = 2 * p, j1 = 2 * p + 1;
  if (j0 >= Mk) return;
  const int32_t a0 = t_row_ptr[j0], a1 = t_row_ptr[j0 + 1];
  const int32_t b0 = j1 < Mk ? t_row_ptr[j1] : 0, b1 = j1 < Mk ? t_row_ptr[j1 + 1] : 0;
  auto row_len = [&](int32_t i) { return row_ptr[(i >> col_shift) + 1] - row_ptr[i >> col_shift]; };
  int32_t held_q[2] = {-1, -1}, held_e[2] = {-1, -1};
  int nb = 0;
  // a new chain's accumulator: prefer the alternate one, take the other if only it is
  // free, cut the hold of the alternate one if both are held
  auto take = [&]() {
    int b = nb;
    if (held_q[b] >= 0 && held_q[b ^ 1] < 0) b ^= 1;
    if (held_q[b] >= 0) {
      t_dq[held_e[b]] |= HLA_DQ_DRAIN;   // cut: drained (partial) at its first tile
      held_q[b] = -1;
    }
    nb = b ^ 1;
    return b;
  };
  int32_t e1 = b0;
  for (int32_t e = a0; e < a1; ++e) {
    const int32_t i = t_col_idx[e];
    while (e1 < b1 && t_col_idx[e1] < i) ++e1;
    const bool in1 = e1 < b1 && t_col_idx[e1] == i;
    const int b = take();
    uint8_t f = (uint8_t)(b | HLA_DQ_NEW);
    if (in1) {
      held_q[b] = i;
      held_e[b] = e;
    } else {
      f |= HLA_DQ_DRAIN | (row_len(i) == 1 ? HLA_DQ_LOCAL : 0);
    }
    t_dq[e] = f;
  }
  for (int32_t e = b0; e < b1; ++e) {
    const int32_t i = t_col_idx[e];
    int b = held_q[0] == i ? 0 : (held_q[1] == i ? 1 : -1);
    if (b >= 0) {   // continues the chain held since kv-block 2p: complete iff row i = {2p, 2p+1}
      t_dq[e] = (uint8_t)(b | HLA_DQ_DRAIN | (row_len(i) == 2 ? HLA_DQ_LOCAL : 0));
      held_q[b] = -1;
    } else {
      b = take();
      t_dq[e] = (uint8_t)(b | HLA_DQ_NEW | HLA_DQ_DRAIN | (row_len(i) == 1 ? HLA_DQ_LOCAL : 0));
    }
  }
}

// q_dq_local[i] = 1 iff q-block i's dQ is completed inside one work unit, read off
// the plan: the entry of i in the list of its last kv-block carries LOCAL (a chain
// is LOCAL only if it covers i's whole forward list)
__global__ void bwd_plan_local_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                                      const int32_t* __restrict__ t_row_ptr, const int32_t* __restrict__ t_col_idx,
                                      const uint8_t* __restrict__ t_dq, int32_t Mq, uint8_t* __restrict__ q_local,
                                      int col_shift) {
  const int32_t i = (int32_t)(blockIdx.x * blockDim.x + threadIdx.x);
  if (i >= Mq) return;
  uint8_t loc = 0;
  const int32_t r0 = row_ptr[i], r1 = row_ptr[i + 1];
  if (r1 > r0) {
    const int32_t jl = col_idx[r1 - 1] >> col_shift;
    for (int32_t e = t_row_ptr[jl]; e < t_row_ptr[jl + 1]; ++e)
      if (t_col_idx[e] == (i << col_shift)) { loc = (t_dq[e] & HLA_DQ_LOCAL) ? 1 : 0; break; }
  }
  q_local[i] = loc;
}

}  // namespace hla

using namespace hla;

extern "C" hla_status hla_build_bwd_plan(hla_block_mask* m, cudaStream_t stream) {
  clear_error();
  HLA_REQUIRE(m != nullptr, HLA_ERR_INVALID, "null mask");
  HLA_REQUIRE(m->row_ptr && m->col_idx && m->t_row_ptr && m->t_col_idx, HLA_ERR_INVALID,
              "the mask must be filled (hla_build_block_mask fill call) before its plan");
  HLA_REQUIRE(m->t_dq && m->q_dq_local, HLA_ERR_INVALID, "t_dq / q_dq_local arrays required");
  HLA_REQUIRE(m->n_qblocks == m->n_kblocks, HLA_ERR_UNSUPPORTED, "dQ plan needs block_q == block_k");
  HLA_REQUIRE(m->n_qblocks >= 1 && m->n_qblocks <= 65536, HLA_ERR_INVALID, "bad n_qblocks");
  // block 64 (window lists present): the plan is over the attention kernels' window lists and
  // exists only when every window starts on a 128-row boundary (windows = 128-row tiles, e.g.
  // HWA with 64-token windows); otherwise windows overlap in rows and there is no plan
  // (n_dq_nonlocal = -1: every dQ through the fp32 accumulator)
  const bool win = m->w_row_ptr != nullptr;
  const int32_t* rp = win ? m->w_row_ptr : m->row_ptr;
  const int32_t* ci = win ? m->w_col : m->col_idx;
  const int32_t* trp = win ? m->wt_row_ptr : m->t_row_ptr;
  const int32_t* tci = win ? m->wt_col : m->t_col_idx;
  const int32_t Mq = win ? (m->n_qblocks + 1) / 2 : m->n_qblocks, Mk = win ? (m->n_kblocks + 1) / 2 : m->n_kblocks;
  if (win) {
    HLA_REQUIRE(ci && trp && tci, HLA_ERR_INVALID, "block-64 mask without its window lists");
    std::vector<int32_t> hc((size_t)std::max<int64_t>(m->w_counts[0], 0)), htc((size_t)std::max<int64_t>(m->w_counts[2], 0));
    if (!hc.empty())
      HLA_CUDA_TRY(cudaMemcpyAsync(hc.data(), ci, sizeof(int32_t) * hc.size(), cudaMemcpyDeviceToHost, stream));
    if (!htc.empty())
      HLA_CUDA_TRY(cudaMemcpyAsync(htc.data(), tci, sizeof(int32_t) * htc.size(), cudaMemcpyDeviceToHost, stream));
    HLA_CUDA_TRY(cudaStreamSynchronize(stream));
    for (int32_t c : hc)
      if (c & 1) { m->n_dq_nonlocal = -1; return HLA_OK; }
    for (int32_t c : htc)
      if (c & 1) { m->n_dq_nonlocal = -1; return HLA_OK; }
  }
  const int col_shift = win ? 1 : 0;
  const int32_t pairs = (Mk + 1) / 2;
  bwd_plan_kernel<<<(pairs + 127) / 128, 128, 0, stream>>>(rp, trp, tci, Mk, m->t_dq, col_shift);
  bwd_plan_local_kernel<<<(Mq + 127) / 128, 128, 0, stream>>>(rp, ci, trp, tci, m->t_dq, Mq, m->q_dq_local, col_shift);
  HLA_CUDA_TRY(cudaGetLastError());
  std::vector<uint8_t> loc((size_t)Mq);
  HLA_CUDA_TRY(cudaMemcpyAsync(loc.data(), m->q_dq_local, (size_t)Mq, cudaMemcpyDeviceToHost, stream));
  HLA_CUDA_TRY(cudaStreamSynchronize(stream));
  int32_t n = 0;
  for (uint8_t x : loc) n += x ? 0 : 1;
  m->n_dq_nonlocal = n;
  return HLA_OK;
}

namespace {

// Windows of one 128-row tile from the CSR rows r0 (and r1 if it exists) of a block-64
// mask: `cols` / `kinds` per row; the union is cut into windows (u, u + 1) from its
// smallest uncovered element upward.  Kind 1 iff all four 64 x 64 sub-tiles are listed full.
void tile_windows(const std::vector<int32_t>& rp, const std::vector<int32_t>& ci, const std::vector<uint8_t>& kd,
                  int32_t r0, int32_t nrows, std::vector<int32_t>* wcol, std::vector<uint8_t>* wkind) {
  auto kind_of = [&](int32_t r, int32_t c) -> int {
    if (r >= nrows) return 0;
    for (int32_t e = rp[r]; e < rp[r + 1]; ++e)
      if (ci[e] == c) return kd[e];
    return 0;
  };
  std::vector<int32_t> u;
  for (int32_t r = r0; r < std::min(r0 + 2, nrows); ++r)
    for (int32_t e = rp[r]; e < rp[r + 1]; ++e) u.push_back(ci[e]);
  std::sort(u.begin(), u.end());
  u.erase(std::unique(u.begin(), u.end()), u.end());
  int32_t covered = -1;   // last 64-block covered by a window
  for (int32_t c : u) {
    if (c <= covered) continue;
    const bool full = kind_of(r0, c) == 1 && kind_of(r0, c + 1) == 1 && kind_of(r0 + 1, c) == 1 &&
                      kind_of(r0 + 1, c + 1) == 1;
    wcol->push_back(c);
    wkind->push_back(full ? 1 : 2);
    covered = c + 1;
  }
}

}  // namespace

extern "C" hla_status hla_build_tile_lists(hla_block_mask* m, int64_t* n_out, cudaStream_t stream) {
  clear_error();
  HLA_REQUIRE(m != nullptr && n_out != nullptr, HLA_ERR_INVALID, "null mask or n_out");
  HLA_REQUIRE(m->row_ptr && m->col_idx && m->kind && m->t_row_ptr && m->t_col_idx && m->t_kind, HLA_ERR_INVALID,
              "the mask must be filled (hla_build_block_mask fill call) before its window lists");
  HLA_REQUIRE(m->n_qblocks >= 1 && m->n_kblocks >= 1 && m->n_qblocks <= (1 << 20) && m->n_kblocks <= (1 << 20),
              HLA_ERR_INVALID, "bad block counts");
  const int32_t Mq = m->n_qblocks, Mk = m->n_kblocks;
  std::vector<int32_t> rp(Mq + 1), trp(Mk + 1);
  HLA_CUDA_TRY(cudaMemcpyAsync(rp.data(), m->row_ptr, sizeof(int32_t) * (Mq + 1), cudaMemcpyDeviceToHost, stream));
  HLA_CUDA_TRY(cudaMemcpyAsync(trp.data(), m->t_row_ptr, sizeof(int32_t) * (Mk + 1), cudaMemcpyDeviceToHost, stream));
  HLA_CUDA_TRY(cudaStreamSynchronize(stream));
  const int64_t nnz = rp[Mq];
  HLA_REQUIRE(nnz == trp[Mk], HLA_ERR_INVALID, "row / transposed lists disagree");
  std::vector<int32_t> ci(nnz), tci(nnz);
  std::vector<uint8_t> kd(nnz), tkd(nnz);
  if (nnz > 0) {
    HLA_CUDA_TRY(cudaMemcpyAsync(ci.data(), m->col_idx, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost, stream));
    HLA_CUDA_TRY(cudaMemcpyAsync(kd.data(), m->kind, nnz, cudaMemcpyDeviceToHost, stream));
    HLA_CUDA_TRY(cudaMemcpyAsync(tci.data(), m->t_col_idx, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost, stream));
    HLA_CUDA_TRY(cudaMemcpyAsync(tkd.data(), m->t_kind, nnz, cudaMemcpyDeviceToHost, stream));
    HLA_CUDA_TRY(cudaStreamSynchronize(stream));
  }
  const int32_t Tq = (Mq + 1) / 2, Tk = (Mk + 1) / 2;
  std::vector<int32_t> wrp(Tq + 1, 0), wtrp(Tk + 1, 0), wcol, wtcol;
  std::vector<uint8_t> wkind, wtkind;
  for (int32_t t = 0; t < Tq; ++t) {
    tile_windows(rp, ci, kd, 2 * t, Mq, &wcol, &wkind);
    wrp[t + 1] = (int32_t)wcol.size();
  }
  for (int32_t t = 0; t < Tk; ++t) {
    tile_windows(trp, tci, tkd, 2 * t, Mk, &wtcol, &wtkind);
    wtrp[t + 1] = (int32_t)wtcol.size();
  }
  auto nfull = [](const std::vector<uint8_t>& k) { return (int64_t)std::count(k.begin(), k.end(), (uint8_t)1); };
  m->w_counts[0] = (int64_t)wcol.size();
  m->w_counts[1] = nfull(wkind);
  m->w_counts[2] = (int64_t)wtcol.size();
  m->w_counts[3] = nfull(wtkind);
  const int64_t need = std::max<int64_t>(1, std::max(m->w_counts[0], m->w_counts[2]));
  *n_out = need;
  if (m->w_col == nullptr) return HLA_OK;
  HLA_REQUIRE(m->w_row_ptr && m->w_kind && m->wt_row_ptr && m->wt_col && m->wt_kind, HLA_ERR_INVALID,
              "fill call needs all window arrays");
  HLA_REQUIRE(need <= m->w_capacity, HLA_ERR_CAPACITY, "window capacity %lld < %lld", (long long)m->w_capacity,
              (long long)need);
  HLA_CUDA_TRY(cudaMemcpyAsync(m->w_row_ptr, wrp.data(), sizeof(int32_t) * (Tq + 1), cudaMemcpyHostToDevice, stream));
  HLA_CUDA_TRY(cudaMemcpyAsync(m->wt_row_ptr, wtrp.data(), sizeof(int32_t) * (Tk + 1), cudaMemcpyHostToDevice, stream));
  if (!wcol.empty()) {
    HLA_CUDA_TRY(cudaMemcpyAsync(m->w_col, wcol.data(), sizeof(int32_t) * wcol.size(), cudaMemcpyHostToDevice, stream));
    HLA_CUDA_TRY(cudaMemcpyAsync(m->w_kind, wkind.data(), wkind.size(), cudaMemcpyHostToDevice, stream));
  }
  if (!wtcol.empty()) {
    HLA_CUDA_TRY(cudaMemcpyAsync(m->wt_col, wtcol.data(), sizeof(int32_t) * wtcol.size(), cudaMemcpyHostToDevice,
                                 stream));
    HLA_CUDA_TRY(cudaMemcpyAsync(m->wt_kind, wtkind.data(), wtkind.size(), cudaMemcpyHostToDevice, stream));
  }
  HLA_CUDA_TRY(cudaStreamSynchronize(stream));
  return HLA_OK;
}

extern "C" hla_status hla_build_block_mask(const hla_pattern_desc* d, hla_block_mask* m, int64_t* nnz_out,
                                           cudaStream_t stream) {
  clear_error();
  Pattern p;
  hla_status st = make_pattern(d, &p);
  if (st != HLA_OK) return st;
  HLA_REQUIRE(m != nullptr && nnz_out != nullptr, HLA_ERR_INVALID, "null mask or nnz_out");
  const int32_t bq = d->block_q, bk = d->block_k;
  const int64_t Mq = (p.N + (int64_t)bq - 1) / bq, Mk = (p.N + (int64_t)bk - 1) / bk;
  HLA_REQUIRE(m->n_qblocks == Mq && m->n_kblocks == Mk, HLA_ERR_INVALID,
              "mask n_qblocks/n_kblocks (%d,%d) != (%lld,%lld) for this descriptor", m->n_qblocks,
              m->n_kblocks, (long long)Mq, (long long)Mk);
  HLA_REQUIRE(Mq <= 65536 && Mk <= 65536, HLA_ERR_UNSUPPORTED, "more than 65536 blocks per line");
  HLA_REQUIRE(m->row_ptr && m->t_row_ptr && m->counts, HLA_ERR_INVALID, "row_ptr/t_row_ptr/counts required");
  const bool fill = m->col_idx != nullptr;
  if (fill)
    HLA_REQUIRE(m->kind && m->t_col_idx && m->t_kind, HLA_ERR_INVALID, "fill call needs all CSR arrays");

  const size_t smem = (size_t)std::max(Mq, Mk);
  auto* counts = reinterpret_cast<unsigned long long*>(m->counts);
  HLA_CUDA_TRY(cudaMemsetAsync(m->counts, 0, 4 * sizeof(int64_t), stream));
  HLA_CUDA_TRY(cudaFuncSetAttribute(classify_lines_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  HLA_CUDA_TRY(cudaFuncSetAttribute(classify_lines_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  const unsigned lines = (unsigned)(Mq + Mk);
  classify_lines_kernel<0><<<lines, kLineThreads, smem, stream>>>(p, bq, bk, (int32_t)Mq, (int32_t)Mk, m->row_ptr,
                                                                  nullptr, nullptr, m->t_row_ptr, nullptr, nullptr,
                                                                  counts);
  HLA_CUDA_TRY(cudaGetLastError());
  scan_lines_kernel<<<2, 1024, 0, stream>>>(m->row_ptr, (int32_t)Mq, m->t_row_ptr, (int32_t)Mk, counts);
  HLA_CUDA_TRY(cudaGetLastError());
  int64_t nnz = 0;
  HLA_CUDA_TRY(cudaMemcpyAsync(&nnz, m->counts, sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
  HLA_CUDA_TRY(cudaStreamSynchronize(stream));
  *nnz_out = nnz;
  if (!fill) return HLA_OK;
  HLA_REQUIRE(nnz <= m->capacity, HLA_ERR_CAPACITY, "capacity %lld < nnz %lld", (long long)m->capacity,
              (long long)nnz);
  classify_lines_kernel<1><<<lines, kLineThreads, smem, stream>>>(p, bq, bk, (int32_t)Mq, (int32_t)Mk, m->row_ptr,
                                                                  m->col_idx, m->kind, m->t_row_ptr, m->t_col_idx,
                                                                  m->t_kind, counts);
  HLA_CUDA_TRY(cudaGetLastError());
  HLA_CUDA_TRY(cudaMemcpyAsync(m->host_counts, m->counts, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
  HLA_CUDA_TRY(cudaStreamSynchronize(stream));
  return HLA_OK;
}
