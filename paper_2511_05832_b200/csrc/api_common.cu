// Host-side helpers of the C ABI: error string, pattern validation, ratios.
#include <cstdarg>
#include <cstring>

#include "common.cuh"

namespace hla {

static thread_local char g_err[1024] = {0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

void clear_error() { g_err[0] = 0; }

// Validate a pattern descriptor (S:L98-100 argument rules) and lower it to the
// device predicate parameters.
namespace {
hla_status make_pattern_fields(const hla_pattern_desc* d, Pattern* p) {
  HLA_REQUIRE(d != nullptr && p != nullptr, HLA_ERR_INVALID, "null descriptor");
  HLA_REQUIRE(d->grid_h >= 1 && d->grid_w >= 1, HLA_ERR_INVALID, "grid %dx%d invalid", d->grid_h, d->grid_w);
  int64_t N = (int64_t)d->grid_h * d->grid_w;
  HLA_REQUIRE(N <= (1 << 24), HLA_ERR_UNSUPPORTED, "N=%lld too large", (long long)N);
  HLA_REQUIRE(d->block_q >= 1 && d->block_k >= 1, HLA_ERR_INVALID, "block must be >= 1");
  HLA_REQUIRE(d->order == HLA_ORDER_ROW_MAJOR || d->order == HLA_ORDER_HILBERT || d->order == HLA_ORDER_HILBERT_TILED,
              HLA_ERR_INVALID, "order %d invalid", d->order);
  // the tiled order relabels positions inside aligned 64-token segments only: the patterns whose
  // predicates see a 64-segment as a unit (windows of a multiple of 64 tokens, dense) are the same
  // attention under it (reading R23)
  HLA_REQUIRE(d->order != HLA_ORDER_HILBERT_TILED || d->pattern == HLA_DENSE ||
                  (d->pattern == HLA_WINDOW && ((int64_t)d->win_h * d->win_w) % 64 == 0),
              HLA_ERR_UNSUPPORTED, "HLA_ORDER_HILBERT_TILED needs HLA_WINDOW with a multiple of 64 tokens, or HLA_DENSE");
  HLA_REQUIRE(d->order != HLA_ORDER_HILBERT_TILED || (d->grid_h == d->grid_w && is_pow2(d->grid_h) && d->grid_h >= 8),
              HLA_ERR_UNSUPPORTED, "HLA_ORDER_HILBERT_TILED needs a square 2^k grid, k >= 3");
  std::memset(p, 0, sizeof(*p));
  p->N = (int32_t)N;
  p->H = d->grid_h;
  p->W = d->grid_w;
  p->log2W = is_pow2(d->grid_w) ? ilog2(d->grid_w) : -1;
  const bool hil = d->order != HLA_ORDER_ROW_MAJOR;
  if (d->pattern == HLA_DENSE) {
    p->kind = K_DENSE;
    return HLA_OK;
  }
  HLA_REQUIRE(d->win_h >= 1 && d->win_w >= 1, HLA_ERR_INVALID, "window %dx%d invalid", d->win_h, d->win_w);
  HLA_REQUIRE(d->pattern == HLA_SHIFTED_WINDOW || d->shift == 0, HLA_ERR_INVALID,
              "shift is only meaningful for HLA_SHIFTED_WINDOW");
  if (hil) {
    int64_t n = (int64_t)d->win_h * d->win_w;
    HLA_REQUIRE(n <= N, HLA_ERR_INVALID, "window of %lld tokens exceeds N=%lld", (long long)n, (long long)N);
    p->n = (int32_t)n;
    p->r = (int32_t)(n / 2);
    p->L = 2 * p->r + 1;
    switch (d->pattern) {
      case HLA_WINDOW:
        HLA_REQUIRE(d->grid_h % d->win_h == 0 && d->grid_w % d->win_w == 0, HLA_ERR_INVALID,
                    "window %dx%d does not divide grid %dx%d", d->win_h, d->win_w, d->grid_h, d->grid_w);
        p->kind = K_HWA;
        return HLA_OK;
      case HLA_SLIDE: p->kind = K_HSA; return HLA_OK;
      case HLA_NEIGHBORHOOD:
        HLA_REQUIRE(p->L <= N, HLA_ERR_INVALID, "neighborhood length %d exceeds N", p->L);
        p->kind = K_HNA;
        return HLA_OK;
      case HLA_SHIFTED_WINDOW:
        // windows of n tokens on a grid the 2D window divides (as HWA); the shift moves them
        // by 0 < shift < n tokens (shift 0 would be HWA itself)
        HLA_REQUIRE(d->grid_h % d->win_h == 0 && d->grid_w % d->win_w == 0, HLA_ERR_INVALID,
                    "window %dx%d does not divide grid %dx%d", d->win_h, d->win_w, d->grid_h, d->grid_w);
        HLA_REQUIRE(d->shift > 0 && d->shift < n, HLA_ERR_INVALID, "shift %d outside (0, n)", d->shift);
        p->shift = d->shift;
        p->kind = K_HSWA;
        return HLA_OK;
      default: break;
    }
    HLA_REQUIRE(false, HLA_ERR_INVALID, "pattern %d invalid", d->pattern);
  }
  p->kh = d->win_h;
  p->kw = d->win_w;
  switch (d->pattern) {
    case HLA_WINDOW:
      HLA_REQUIRE(d->grid_h % d->win_h == 0 && d->grid_w % d->win_w == 0, HLA_ERR_INVALID,
                  "window %dx%d does not divide grid %dx%d", d->win_h, d->win_w, d->grid_h, d->grid_w);
      p->kind = K_WSA;
      return HLA_OK;
    case HLA_SLIDE:
      HLA_REQUIRE(d->win_h <= d->grid_h && d->win_w <= d->grid_w, HLA_ERR_INVALID, "kernel larger than grid");
      p->kind = K_SA;
      return HLA_OK;
    case HLA_NEIGHBORHOOD:
      HLA_REQUIRE(d->win_h <= d->grid_h && d->win_w <= d->grid_w, HLA_ERR_INVALID, "kernel larger than grid");
      p->kind = K_NA2D;
      return HLA_OK;
    case HLA_SHIFTED_WINDOW:
      HLA_REQUIRE(false, HLA_ERR_INVALID, "shifted window requires Hilbert order");
    default: break;
  }
  HLA_REQUIRE(false, HLA_ERR_INVALID, "pattern %d invalid", d->pattern);
}
}  // namespace

hla_status make_pattern(const hla_pattern_desc* d, Pattern* p) {
  const hla_status st = make_pattern_fields(d, p);
  if (st != HLA_OK) return st;
  p->n_div = make_fastdiv(p->n > 0 ? p->n : 1);
  p->w_div = make_fastdiv(p->W);
  p->kh_div = make_fastdiv(p->kh > 0 ? p->kh : 1);
  p->kw_div = make_fastdiv(p->kw > 0 ? p->kw : 1);
  return HLA_OK;
}

}  // namespace hla

#ifdef HLA_TRACE
namespace hla {
__device__ unsigned long long g_hla_trace[8 * 1024 * 2];
}  // namespace hla
// dev-only: copy the whole trace area (8 roles x 1024 (tag, clock) pairs) to host and clear it
extern "C" __attribute__((visibility("default"))) int hla_debug_trace_dump(unsigned long long* host, int max_events) {
  cudaDeviceSynchronize();
  const int n = max_events < 8 * 1024 ? max_events : 8 * 1024;
  cudaMemcpyFromSymbol(host, hla::g_hla_trace, (size_t)n * 2 * sizeof(unsigned long long));
  static unsigned long long zeros[8 * 1024 * 2];
  cudaMemcpyToSymbol(hla::g_hla_trace, zeros, sizeof(zeros));
  return n;
}
#endif

extern "C" const char* hla_last_error(void) { return hla::g_err; }

extern "C" const char* hla_version(void) { return "libhla 0.1 (sm_100a, tcgen05/TMEM/TMA)"; }

extern "C" hla_status hla_mask_ratios(const hla_pattern_desc* d, const int64_t counts[4],
                                      double* empty_tile_ratio, double* sparsity) {
  hla::clear_error();
  hla::Pattern p;
  hla_status st = hla::make_pattern(d, &p);
  if (st != HLA_OK) return st;
  HLA_REQUIRE(counts != nullptr, HLA_ERR_INVALID, "null counts");
  const int64_t N = p.N;
  const int64_t Mq = (N + d->block_q - 1) / d->block_q;
  const int64_t Mk = (N + d->block_k - 1) / d->block_k;
  const int64_t nnz = counts[0];
  const int64_t n_empty = counts[3];
  // Exactly the expressions of the paper's Sparsity column (reading R7) and
  // the plain empty-tile fraction, evaluated in IEEE double.
  if (empty_tile_ratio) *empty_tile_ratio = (double)n_empty / (double)(Mq * Mk);
  if (sparsity) *sparsity = 1.0 - (double)(nnz * (int64_t)d->block_q * (int64_t)d->block_k) / ((double)N * (double)N);
  return HLA_OK;
}
