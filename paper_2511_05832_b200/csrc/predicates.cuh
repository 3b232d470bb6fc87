// allowed(q, k) of the local-attention patterns, device side (see include/hla.h
// for the definitions and their paper passages).
#pragma once

#include "common.cuh"

namespace hla {

__host__ __device__ __forceinline__ int32_t floordiv(int32_t a, int32_t b) {
  int32_t q = a / b;
  return (q * b > a) ? q - 1 : q;
}
__host__ __device__ __forceinline__ int32_t clampi(int32_t x, int32_t lo, int32_t hi) {
  return x < lo ? lo : (x > hi ? hi : x);
}

// Generic scalar predicate (used by the tile classifier; every element).
__device__ __forceinline__ bool allowed(const Pattern& p, int32_t q, int32_t k) {
  switch (p.kind) {
    case K_HWA: return (q / p.n) == (k / p.n);
    case K_HSA: { int32_t dlt = q - k; return (dlt <= p.r) && (-dlt <= p.r); }
    case K_HNA: { int32_t s = clampi(q - p.r, 0, p.N - p.L); return k >= s && k < s + p.L; }
    case K_HSWA: return floordiv(q - p.shift, p.n) == floordiv(k - p.shift, p.n);
    case K_DENSE: return true;
    default: break;
  }
  int32_t rq = q / p.W, cq = q - rq * p.W;
  int32_t rk = k / p.W, ck = k - rk * p.W;
  switch (p.kind) {
    case K_WSA: return (rq / p.kh == rk / p.kh) && (cq / p.kw == ck / p.kw);
    case K_SA: {
      int32_t dr = rq - rk, dc = cq - ck;
      return (dr <= p.kh / 2) && (-dr <= p.kh / 2) && (dc <= p.kw / 2) && (-dc <= p.kw / 2);
    }
    case K_NA2D: {
      int32_t sr = clampi(rq - p.kh / 2, 0, p.H - p.kh);
      int32_t sc = clampi(cq - p.kw / 2, 0, p.W - p.kw);
      return rk >= sr && rk < sr + p.kh && ck >= sc && ck < sc + p.kw;
    }
    default: return false;
  }
}

// Per-query-row form used inside the attention kernels on partial tiles:
//   1D patterns: allowed(k) <=> (unsigned)(k - lo) < len
//   2D patterns: allowed(k) <=> (unsigned)(row(k) - r0) < rn && (unsigned)(col(k) - c0) < cn
struct RowBox {
  int32_t lo, len;      // 1D interval, or row range for 2D
  int32_t c0, cn;       // 2D column range
};

__device__ __forceinline__ RowBox row_box(const Pattern& p, int32_t q) {
  RowBox b;
  switch (p.kind) {
    case K_HWA: b.lo = p.n_div.div(q) * p.n; b.len = p.n; b.c0 = 0; b.cn = 0; return b;
    case K_HSA: b.lo = q - p.r; b.len = 2 * p.r + 1; b.c0 = 0; b.cn = 0; return b;
    case K_HNA: b.lo = clampi(q - p.r, 0, p.N - p.L); b.len = p.L; b.c0 = 0; b.cn = 0; return b;
    case K_HSWA:   // floor((q - shift) / n) with q - shift + n > 0 (0 < shift < n)
      b.lo = (p.n_div.div(q - p.shift + p.n) - 1) * p.n + p.shift; b.len = p.n; b.c0 = 0; b.cn = 0; return b;
    case K_DENSE: b.lo = 0; b.len = p.N; b.c0 = 0; b.cn = 0; return b;
    default: break;
  }
  int32_t rq = p.w_div.div(q), cq = q - rq * p.W;
  switch (p.kind) {
    case K_WSA:
      b.lo = p.kh_div.div(rq) * p.kh; b.len = p.kh; b.c0 = p.kw_div.div(cq) * p.kw; b.cn = p.kw; return b;
    case K_SA:
      b.lo = rq - p.kh / 2; b.len = 2 * (p.kh / 2) + 1; b.c0 = cq - p.kw / 2; b.cn = 2 * (p.kw / 2) + 1; return b;
    default:  // K_NA2D
      b.lo = clampi(rq - p.kh / 2, 0, p.H - p.kh); b.len = p.kh;
      b.c0 = clampi(cq - p.kw / 2, 0, p.W - p.kw); b.cn = p.kw; return b;
  }
}

// Transposed form for the backward pass (thread = key k, columns = queries q):
// the set {q : allowed(q, k)} as a box of the same shape.  For the symmetric
// patterns it equals row_box(k); HNA / NA2D clamp their windows, so the query
// range of a key is derived from the monotone window start s(q) = clamp(q - a, 0, n - L):
//   s(q) <= k        <=>  q <= k + a            (or every q if k >= n - L)
//   s(q) >= k - L + 1 <=> q >= k - L + 1 + a    (or every q if k - L + 1 <= 0)
__device__ __forceinline__ void clamped_col_range(int32_t k, int32_t a, int32_t L, int32_t n, int32_t* lo,
                                                  int32_t* len) {
  const int32_t q0 = (k - L + 1 <= 0) ? 0 : k - L + 1 + a;
  const int32_t q1 = (k >= n - L) ? n - 1 : k + a;
  *lo = q0;
  *len = q1 - q0 + 1;
}

__device__ __forceinline__ RowBox col_box(const Pattern& p, int32_t k) {
  if (p.kind == K_HNA) {
    RowBox b;
    clamped_col_range(k, p.r, p.L, p.N, &b.lo, &b.len);
    b.c0 = 0;
    b.cn = 0;
    return b;
  }
  if (p.kind == K_NA2D) {
    RowBox b;
    const int32_t rk = p.w_div.div(k), ck = k - rk * p.W;
    clamped_col_range(rk, p.kh / 2, p.kh, p.H, &b.lo, &b.len);
    clamped_col_range(ck, p.kw / 2, p.kw, p.W, &b.c0, &b.cn);
    return b;
  }
  return row_box(p, k);  // symmetric patterns
}

// Intersect a row / column box with the real sequence (ragged last tile): 1D
// intervals with [0, N), 2D row ranges with [0, H) (columns are inside [0, W) by
// construction of the 2D boxes, and rows < H imply k < N).
template <bool kTwoD>
__device__ __forceinline__ RowBox clip_box(const Pattern& p, RowBox b) {
  const int32_t lim = kTwoD ? p.H : p.N;
  const int32_t lo = b.lo < 0 ? 0 : b.lo;
  const int32_t hi = min(b.lo + b.len, lim);
  b.lo = lo;
  b.len = hi > lo ? hi - lo : 0;
  return b;
}

}  // namespace hla
