// Shared host/device helpers of libhla (not exported).
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>

#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "../../include/hla.h"

namespace hla {

// thread-local last error message (hla_last_error)
void set_error(const char* fmt, ...);
void clear_error();

#define HLA_REQUIRE(cond, status, ...)      \
  do {                                      \
    if (!(cond)) {                          \
      ::hla::set_error(__VA_ARGS__);        \
      return (status);                      \
    }                                       \
  } while (0)

#define HLA_CUDA_TRY(expr)                                                         \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess) {                                                       \
      ::hla::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),     \
                       __FILE__, __LINE__);                                        \
      return HLA_ERR_CUDA;                                                         \
    }                                                                              \
  } while (0)

// Internal pattern kinds (order x family), see include/hla.h.
enum Kind : int32_t {
  K_HWA = 0, K_HSA = 1, K_HNA = 2, K_HSWA = 3,
  K_WSA = 4, K_SA = 5, K_NA2D = 6, K_DENSE = 7
};

// Device-side description of the allowed(q, k) predicate.
// floor(n / d) for 0 <= n < 2^31 as one wide multiply and a shift (Granlund-Montgomery:
// m = ceil(2^(31+l) / d), l = ceil(log2 d)); the unit decode at every unit boundary of
// every role otherwise runs three integer divisions on its critical path (fwd + bwd)
struct FastDiv {
  uint32_t m, s;
  int32_t d;
  __device__ __forceinline__ int32_t div(int32_t n) const {
    return (int32_t)(((uint64_t)(uint32_t)n * m) >> s);
  }
};
inline FastDiv make_fastdiv(int32_t d) {
  uint32_t l = 0;
  while ((1ll << l) < d) ++l;
  const uint64_t p = 1ull << (31 + l);
  return FastDiv{(uint32_t)((p + (uint64_t)d - 1) / (uint64_t)d), 31 + l, d};
}

struct Pattern {
  int32_t kind;
  int32_t N, H, W;
  int32_t n, r, L, shift;   // 1D (Hilbert) parameters: window n, radius r, HNA length L
  int32_t kh, kw;           // 2D (row-major) window / kernel
  int32_t log2W;            // log2(W) if W is a power of two, else -1
  FastDiv n_div, w_div, kh_div, kw_div;   // division by n, W, kh, kw (multiply-shift)
};

hla_status make_pattern(const hla_pattern_desc* d, Pattern* p);

// The tile lists an attention call walks (tiles are 128 x 128 either way): the mask's CSR
// lists at block 128; its window lists (hla_build_tile_lists) at block 64, whose columns
// are 64-block starts.  Start row of a list entry = column * col_mul.
struct AttnLists {
  const int32_t* row_ptr;     // per 128-row q tile
  const int32_t* col;
  const uint8_t* kind;        // 1 full, 2 element-masked
  const int32_t* t_row_ptr;   // per 128-key tile (backward)
  const int32_t* t_col;
  const uint8_t* t_kind;
  int32_t col_mul;
  int64_t n_full, n_partial, t_n_full, t_n_partial;
};

// Argument checks shared by hla_attn_fwd / hla_attn_bwd (attn_fwd.cu); fills the lists.
hla_status check_attn_args(const hla_pattern_desc* d, const hla_block_mask* m, int32_t batch, int32_t heads,
                           int32_t head_dim, Pattern* pat, AttnLists* lists);

// Validates an optional hla_score_mod (attn_fwd.cu): outputs stay null when the
// score modification is off; drpb may be null for the forward.
hla_status parse_score_mod(const hla_pattern_desc* d, const hla_score_mod* mod, bool bwd, const float** rpb,
                           float** drpb, const int32_t** cells);

// number of SMs of the current device (cached per process; B200: 148)
inline int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

inline bool is_pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }
inline int ilog2(int64_t x) { int l = 0; while ((1ll << l) < x) ++l; return l; }

// ---- optional device-side event trace (dev builds only: make TRACE=1) ----------
// CTA 0 only; every tracing thread keeps its own counter (HLA_TR_DECL) and writes
// (tag, clock) pairs into the region of its role (tag >> 24), no atomics.
#ifdef HLA_TRACE
extern __device__ unsigned long long g_hla_trace[8 * 1024 * 2];
#define HLA_TR_DECL unsigned int _hla_tr = 0
#define HLA_TR(tag)                                                                       \
  do {                                                                                    \
    if (blockIdx.x == 0 && _hla_tr < 1024) {                                              \
      const unsigned int _s = (((unsigned int)(tag) >> 24) & 7u) * 1024u + _hla_tr++;     \
      ::hla::g_hla_trace[2 * _s] = (unsigned long long)(tag);                             \
      ::hla::g_hla_trace[2 * _s + 1] = clock64();                                         \
    }                                                                                     \
  } while (0)
#else
#define HLA_TR_DECL \
  do {              \
  } while (0)
#define HLA_TR(tag) \
  do {              \
  } while (0)
#endif

// ---- dev-only wait-time accounting (variant builds) --------------------
// Build with the kernel's switch (HLA_BWD_PROF / HLA_FWD_PROF; its .cu file then defines
// HLA_PROF_ON before its includes and HLA_PROF_ARRAY after them): one thread per role sums
// the cycles it spends in each wait / work phase into prof[slot]; HLA_PFLUSH writes the
// sums to HLA_PROF_ARRAY[blockIdx.x].
#ifdef HLA_PROF_ON
#define HLA_PW(slot, ...)                                \
  do {                                                   \
    const long long _t0 = clock64();                     \
    __VA_ARGS__;                                         \
    prof[slot] += (unsigned long long)(clock64() - _t0); \
  } while (0)
#define HLA_PDECL unsigned long long prof[24] = {0}
#define HLA_PMARK(v) const long long v = clock64()
#define HLA_PADD(slot, since) prof[slot] += (unsigned long long)(clock64() - (since))
#define HLA_PFLUSH(lo, hi, cond)                                                   \
  do {                                                                             \
    if (cond)                                                                      \
      for (int _i = (lo); _i < (hi); ++_i) HLA_PROF_ARRAY[blockIdx.x][_i] = prof[_i]; \
  } while (0)
#else
#define HLA_PW(slot, ...) __VA_ARGS__
#define HLA_PDECL do {} while (0)
#define HLA_PMARK(v) do {} while (0)
#define HLA_PADD(slot, since) do {} while (0)
#define HLA_PFLUSH(lo, hi, cond) do {} while (0)
#endif

}  // namespace hla
