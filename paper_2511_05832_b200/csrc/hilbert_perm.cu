// K1/K2: Hilbert index and token permutation (grid order <-> Hilbert order).
//
// Paper: "Image tokens are first reordered along a Hilbert curve" (P:L7); "the
// path can be precomputed and cached"; the reorder is the "Reshape"
// step timed in P:L196 / P:L446-467.
//
// The curve is computed with the classic bit loops (d2xy / xy2d, x = column,
// y = row), independently of the oracle's gilbert2d recursion (R1).
// The permutation is a bit-exact row gather: one warp per token row, 16-byte
// vector loads/stores, up to 4 chunks per lane in flight, several tensors per
// launch.  HBM-bound: 2 * row_bytes of traffic per row.
#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace hla {

// s-th cell of the Hilbert curve on an n x n grid (n = 2^log2n) -> row*n + col
__device__ __forceinline__ int32_t hilbert_d2cell(uint32_t d, int log2n) {
  uint32_t t = d, x = 0, y = 0;
  for (int i = 0; i < log2n; ++i) {
    const uint32_t s = 1u << i;
    const uint32_t rx = 1u & (t >> 1);
    const uint32_t ry = 1u & (t ^ rx);
    if (ry == 0) {
      if (rx == 1) { x = s - 1 - x; y = s - 1 - y; }
      const uint32_t tmp = x; x = y; y = tmp;
    }
    x += s * rx;
    y += s * ry;
    t >>= 2;
  }
  return (int32_t)((y << log2n) | x);
}

// position on the curve of cell (row, col) = cell id row*n + col
__device__ __forceinline__ int32_t hilbert_cell2d(uint32_t cell, int log2n) {
  const uint32_t n = 1u << log2n;
  uint32_t x = cell & (n - 1), y = cell >> log2n, d = 0;
  for (uint32_t s = n >> 1; s > 0; s >>= 1) {
    const uint32_t rx = (x & s) ? 1u : 0u;
    const uint32_t ry = (y & s) ? 1u : 0u;
    d += s * s * ((3u * rx) ^ ry);
    if (ry == 0) {
      if (rx == 1) { x = n - 1 - x; y = n - 1 - y; }
      const uint32_t tmp = x; x = y; y = tmp;
    }
  }
  return (int32_t)d;
}

__global__ void hilbert_index_kernel(int32_t N, int log2n, int32_t* __restrict__ seq_to_cell,
                                     int32_t* __restrict__ cell_to_seq) {
  for (int32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < N; s += gridDim.x * blockDim.x) {
    const int32_t cell = hilbert_d2cell((uint32_t)s, log2n);
    if (seq_to_cell) seq_to_cell[s] = cell;
    if (cell_to_seq) cell_to_seq[cell] = s;
  }
}

// HLA_ORDER_HILBERT_TILED (reading R23): on a 2^k grid (k >= 3) every aligned 64-token
// segment of the curve is an aligned 8 x 8 cell square (the curve finishes each aligned 2^j
// square before it leaves it); inside each segment the cells are renumbered in raster order,
// s' = (s & ~63) + 8 * (row & 7) + (col & 7), so that every aligned 8 positions are 8
// consecutive cells of one grid row and every aligned 64 one aligned square in raster order (one
// 5-D TMA box per square instead of 16 gather4 ops, attn_bwd_common.cuh load_rows).
__global__ void hilbert_tiled_index_kernel(int32_t N, int log2n, int32_t* __restrict__ seq_to_cell,
                                           int32_t* __restrict__ cell_to_seq) {
  for (int32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < N; s += gridDim.x * blockDim.x) {
    const int32_t cell = hilbert_d2cell((uint32_t)s, log2n);
    const int32_t t = (s & ~63) | (((cell >> log2n) & 7) << 3) | (cell & 7);
    if (seq_to_cell) seq_to_cell[t] = cell;
    if (cell_to_seq) cell_to_seq[cell] = t;
  }
}

struct PermPtrs {
  const uint4* src[4];
  uint4* dst[4];
};

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// grid: x = token-row groups (8 rows per 256-thread block), y = batch, z = tensor.
// TO (DIR 0):   dst[b, s] = src[b, d2cell(s)]
// FROM (DIR 1): dst[b, t] = src[b, cell2d(t)]
template <int DIR>
__global__ void __launch_bounds__(256) hilbert_perm_kernel(PermPtrs ptrs, int32_t N, int log2n,
                                                           int32_t chunks_per_row) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t t = blockIdx.x * 8 + warp;
  if (t >= N) return;
  const int64_t b = blockIdx.y;
  const int32_t srow = DIR == 0 ? hilbert_d2cell((uint32_t)t, log2n) : hilbert_cell2d((uint32_t)t, log2n);
  const int z = blockIdx.z;  // select without dynamic indexing of the parameter array
  const uint4* sbase = z == 0 ? ptrs.src[0] : z == 1 ? ptrs.src[1] : z == 2 ? ptrs.src[2] : ptrs.src[3];
  uint4* dbase = z == 0 ? ptrs.dst[0] : z == 1 ? ptrs.dst[1] : z == 2 ? ptrs.dst[2] : ptrs.dst[3];
  const uint4* __restrict__ src = sbase + (b * N + srow) * (int64_t)chunks_per_row;
  uint4* __restrict__ dst = dbase + (b * N + t) * (int64_t)chunks_per_row;
  for (int32_t c0 = 0; c0 < chunks_per_row; c0 += 128) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int32_t c = c0 + u * 32 + lane;
      if (c < chunks_per_row) v[u] = ld_stream(src + c);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int32_t c = c0 + u * 32 + lane;
      if (c < chunks_per_row) dst[c] = v[u];
    }
  }
}

static hla_status check_grid(int32_t grid_h, int32_t grid_w, int* log2n) {
  HLA_REQUIRE(grid_h >= 1 && grid_w >= 1, HLA_ERR_INVALID, "grid %dx%d invalid", grid_h, grid_w);
  HLA_REQUIRE(grid_h == grid_w && is_pow2(grid_h) && grid_h <= 32768, HLA_ERR_UNSUPPORTED,
              "the explicit permutation kernel needs a square 2^k grid (got %dx%d); other grids: "
              "hla_hilbert_index + the fused reorder of the attention kernels", grid_h, grid_w);
  *log2n = ilog2(grid_h);
  return HLA_OK;
}

// Generalized Hilbert curve for any W x H grid (the "gilbert" construction the
// paper's shapes need: 56x56, 28x28, 14x14, 7x7, 96x96, ... ).
// Recursive split of the rectangle spanned by the major axis (ax, ay) and the
// minor axis (bx, by): a long rectangle is cut in two along its major axis, a
// squarish one in three (first and last parts turned), keeping every part's
// major side even when possible so the path stays adjacent-step connected.
// Host code, once per grid shape; on 2^k squares it yields the same path as the
// device bit loops above (tested: both against the oracle, bit-exact).
namespace {
inline int sgn(int v) { return (v > 0) - (v < 0); }
inline int floor_half(int v) { return v >= 0 ? v / 2 : -((1 - v) / 2); }   // floor(v / 2)

void gilbert_rect(int x, int y, int ax, int ay, int bx, int by, int W, int32_t* out, int& pos) {
  const int w = std::abs(ax + ay), h = std::abs(bx + by);
  const int dax = sgn(ax), day = sgn(ay), dbx = sgn(bx), dby = sgn(by);
  if (h == 1) {   // a single row along the major axis
    for (int i = 0; i < w; ++i, x += dax, y += day) out[pos++] = y * W + x;
    return;
  }
  if (w == 1) {   // a single column along the minor axis
    for (int i = 0; i < h; ++i, x += dbx, y += dby) out[pos++] = y * W + x;
    return;
  }
  int ax2 = floor_half(ax), ay2 = floor_half(ay), bx2 = floor_half(bx), by2 = floor_half(by);
  const int w2 = std::abs(ax2 + ay2), h2 = std::abs(bx2 + by2);
  if (2 * w > 3 * h) {   // long: two halves along the major axis
    if ((w2 & 1) && w > 2) { ax2 += dax; ay2 += day; }
    gilbert_rect(x, y, ax2, ay2, bx, by, W, out, pos);
    gilbert_rect(x + ax2, y + ay2, ax - ax2, ay - ay2, bx, by, W, out, pos);
  } else {               // squarish: up the minor half, across, back down
    if ((h2 & 1) && h > 2) { bx2 += dbx; by2 += dby; }
    gilbert_rect(x, y, bx2, by2, ax2, ay2, W, out, pos);
    gilbert_rect(x + bx2, y + by2, ax, ay, bx - bx2, by - by2, W, out, pos);
    gilbert_rect(x + (ax - dax) + (bx2 - dbx), y + (ay - day) + (by2 - dby), -bx2, -by2, -(ax - ax2),
                 -(ay - ay2), W, out, pos);
  }
}
}  // namespace

// seq_to_cell of the generalized curve (x = column along the wider side first)
void gilbert_path(int32_t grid_h, int32_t grid_w, int32_t* seq_to_cell) {
  int pos = 0;
  if (grid_w >= grid_h)
    gilbert_rect(0, 0, grid_w, 0, 0, grid_h, grid_w, seq_to_cell, pos);
  else
    gilbert_rect(0, 0, 0, grid_h, grid_w, 0, grid_w, seq_to_cell, pos);
}

}  // namespace hla

using namespace hla;

extern "C" hla_status hla_hilbert_index(int32_t grid_h, int32_t grid_w, int32_t* seq_to_cell,
                                        int32_t* cell_to_seq, cudaStream_t stream) {
  clear_error();
  HLA_REQUIRE(grid_h >= 1 && grid_w >= 1 && (int64_t)grid_h * grid_w < (1ll << 30), HLA_ERR_INVALID,
              "grid %dx%d invalid", grid_h, grid_w);
  const int32_t N = grid_h * grid_w;
  if (!(grid_h == grid_w && is_pow2(grid_h))) {
    // generalized curve: built on the host once per shape, copied (synchronises `stream`)
    if (!seq_to_cell && !cell_to_seq) return HLA_OK;
    std::vector<int32_t> s2c(N), c2s(N);
    gilbert_path(grid_h, grid_w, s2c.data());
    for (int32_t s = 0; s < N; ++s) c2s[s2c[s]] = s;
    if (seq_to_cell)
      HLA_CUDA_TRY(cudaMemcpyAsync(seq_to_cell, s2c.data(), sizeof(int32_t) * N, cudaMemcpyHostToDevice, stream));
    if (cell_to_seq)
      HLA_CUDA_TRY(cudaMemcpyAsync(cell_to_seq, c2s.data(), sizeof(int32_t) * N, cudaMemcpyHostToDevice, stream));
    HLA_CUDA_TRY(cudaStreamSynchronize(stream));
    return HLA_OK;
  }
  int log2n = 0;
  hla_status st = check_grid(grid_h, grid_w, &log2n);
  if (st != HLA_OK) return st;
  if (!seq_to_cell && !cell_to_seq) return HLA_OK;
  const int blocks = (N + 255) / 256;
  hilbert_index_kernel<<<blocks, 256, 0, stream>>>(N, log2n, seq_to_cell, cell_to_seq);
  HLA_CUDA_TRY(cudaGetLastError());
  return HLA_OK;
}

extern "C" hla_status hla_hilbert_tiled_index(int32_t grid_h, int32_t grid_w, int32_t* seq_to_cell,
                                              int32_t* cell_to_seq, cudaStream_t stream) {
  clear_error();
  HLA_REQUIRE(grid_h >= 1 && grid_w >= 1 && (int64_t)grid_h * grid_w < (1ll << 30), HLA_ERR_INVALID,
              "grid %dx%d invalid", grid_h, grid_w);
  HLA_REQUIRE(grid_h == grid_w && is_pow2(grid_h) && grid_h >= 8, HLA_ERR_UNSUPPORTED,
              "tiled Hilbert order needs a square 2^k grid, k >= 3 (got %dx%d)", grid_h, grid_w);
  int log2n = 0;
  hla_status st = check_grid(grid_h, grid_w, &log2n);
  if (st != HLA_OK) return st;
  if (!seq_to_cell && !cell_to_seq) return HLA_OK;
  const int32_t N = grid_h * grid_w;
  hilbert_tiled_index_kernel<<<(N + 255) / 256, 256, 0, stream>>>(N, log2n, seq_to_cell, cell_to_seq);
  HLA_CUDA_TRY(cudaGetLastError());
  return HLA_OK;
}

extern "C" hla_status hla_hilbert_perm(int32_t grid_h, int32_t grid_w, int32_t dir, int32_t batch,
                                       int32_t row_bytes, int32_t n_tensors, const void* const* src,
                                       void* const* dst, int32_t* seq_to_cell_out, cudaStream_t stream) {
  clear_error();
  int log2n = 0;
  hla_status st = check_grid(grid_h, grid_w, &log2n);
  if (st != HLA_OK) return st;
  HLA_REQUIRE(dir == HLA_TO_HILBERT || dir == HLA_FROM_HILBERT, HLA_ERR_INVALID, "dir %d invalid", dir);
  HLA_REQUIRE(batch >= 1 && batch <= 65535, HLA_ERR_INVALID, "batch %d invalid", batch);
  HLA_REQUIRE(row_bytes >= 16 && row_bytes % 16 == 0, HLA_ERR_UNSUPPORTED,
              "row_bytes %d must be a positive multiple of 16", row_bytes);
  HLA_REQUIRE(n_tensors >= 1 && n_tensors <= 4, HLA_ERR_INVALID, "n_tensors %d not in [1,4]", n_tensors);
  HLA_REQUIRE(src != nullptr && dst != nullptr, HLA_ERR_INVALID, "null pointer arrays");
  PermPtrs p{};
  for (int i = 0; i < n_tensors; ++i) {
    HLA_REQUIRE(src[i] && dst[i], HLA_ERR_INVALID, "tensor %d: null pointer", i);
    HLA_REQUIRE(src[i] != dst[i], HLA_ERR_INVALID, "tensor %d: in-place permutation is not supported", i);
    HLA_REQUIRE(((uintptr_t)src[i] & 15) == 0 && ((uintptr_t)dst[i] & 15) == 0, HLA_ERR_INVALID,
                "tensor %d: pointers must be 16-byte aligned", i);
    p.src[i] = reinterpret_cast<const uint4*>(src[i]);
    p.dst[i] = reinterpret_cast<uint4*>(dst[i]);
  }
  const int32_t N = grid_h * grid_w;
  dim3 grid((N + 7) / 8, batch, n_tensors);
  if (dir == HLA_TO_HILBERT)
    hilbert_perm_kernel<0><<<grid, 256, 0, stream>>>(p, N, log2n, row_bytes / 16);
  else
    hilbert_perm_kernel<1><<<grid, 256, 0, stream>>>(p, N, log2n, row_bytes / 16);
  HLA_CUDA_TRY(cudaGetLastError());
  if (seq_to_cell_out) {
    hilbert_index_kernel<<<(N + 255) / 256, 256, 0, stream>>>(N, log2n, seq_to_cell_out, nullptr);
    HLA_CUDA_TRY(cudaGetLastError());
  }
  return HLA_OK;
}
