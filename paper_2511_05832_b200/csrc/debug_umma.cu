// Bring-up microtest of the tcgen05 operand encodings (include/hla_debug.h).
// Operands are written to shared memory by plain threads in the canonical
// SWIZZLE_128B layouts (K-major: [K/64][rows][128 B]; MN-major: [MN/64][K][128 B]),
// exactly the layouts TMA produces for the attention tiles, then one thread
// issues the MMAs.
#include "../../include/hla_debug.h"
#include "common.cuh"
#include "sm100.cuh"
#include "tensor_map.cuh"

namespace hla {
namespace {

__global__ void __launch_bounds__(128) debug_umma_kernel(const __nv_bfloat16* __restrict__ A,
                                                         const __nv_bfloat16* __restrict__ B, float* __restrict__ C,
                                                         int N, int K, int a_mn, int b_mn, int a_tmem) {
  extern __shared__ uint8_t raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  constexpr int M = 128;
  uint8_t* sA = base;                       // M*K*2 bytes
  uint8_t* sB = base + M * K * 2;           // N*K*2 bytes
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;

  auto kmajor_off = [](int r, int k, int R) -> uint32_t {
    return (uint32_t)((k / 64) * R * 128) + sm100::swz128((uint32_t)(r * 128 + (k % 64) * 2));
  };
  auto mnmajor_off = [](int r, int k, int Kt) -> uint32_t {
    return (uint32_t)((r / 64) * Kt * 128) + sm100::swz128((uint32_t)(k * 128 + (r % 64) * 2));
  };
  for (int idx = tid; idx < M * K; idx += 128) {
    const int m = idx / K, k = idx % K;
    const __nv_bfloat16 v = a_mn ? A[k * M + m] : A[m * K + k];
    *reinterpret_cast<__nv_bfloat16*>(sA + (a_mn ? mnmajor_off(m, k, K) : kmajor_off(m, k, M))) = v;
  }
  for (int idx = tid; idx < N * K; idx += 128) {
    const int n = idx / K, k = idx % K;
    const __nv_bfloat16 v = b_mn ? B[k * N + n] : B[n * K + k];
    *reinterpret_cast<__nv_bfloat16*>(sB + (b_mn ? mnmajor_off(n, k, K) : kmajor_off(n, k, N))) = v;
  }
  if (warp == 0) {
    sm100::tmem_alloc(&tmem_base, 512);
    sm100::tmem_relinquish();
  }
  if (tid == 0) {
    sm100::mbar_init(&bar, 1);
    sm100::fence_mbar_init();
  }
  sm100::fence_proxy_async_smem();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t tD = tmem, tA = tmem + 256;
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
  if (a_tmem) {
    // thread m writes row m of A (bf16 pairs) into TMEM columns [256, 256 + K/2)
    for (int c0 = 0; c0 < K / 2; c0 += 16) {
      uint32_t r[16];
      for (int e = 0; e < 16; ++e) {
        const int k = 2 * (c0 + e);
        const float lo = __bfloat162float(A[tid * K + k]), hi = __bfloat162float(A[tid * K + k + 1]);
        r[e] = sm100::pack_bf16(lo, hi);
      }
      sm100::tmem_st16(tA + lane_off + c0, r);
    }
    sm100::tmem_wait_st();
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (tid == 0) {
    const uint32_t idesc = sm100::make_idesc_bf16(M, N, a_mn != 0, b_mn != 0);
    const uint32_t a_base = sm100::smem_u32(sA), b_base = sm100::smem_u32(sB);
    for (int s = 0; s < K / 16; ++s) {
      const uint32_t a_addr = a_mn ? a_base + s * 16 * 128 : a_base + (s / 4) * M * 128 + (s % 4) * 32;
      const uint32_t b_addr = b_mn ? b_base + s * 16 * 128 : b_base + (s / 4) * N * 128 + (s % 4) * 32;
      const uint64_t bdesc = sm100::make_smem_desc(b_addr, b_mn ? K * 128 : 16, 1024, sm100::kSwizzle128B);
      if (a_tmem) {
        sm100::mma_ts(tD, tA + s * 8, bdesc, idesc, s > 0);
      } else {
        const uint64_t adesc = sm100::make_smem_desc(a_addr, a_mn ? K * 128 : 16, 1024, sm100::kSwizzle128B);
        sm100::mma_ss(tD, adesc, bdesc, idesc, s > 0);
      }
    }
    sm100::mma_commit(&bar);
  }
  __syncwarp();
  sm100::mbar_wait(&bar, 0);
  sm100::tc_fence_after();
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t r[32];
    sm100::tmem_ld32(tD + lane_off + c0, r);
    sm100::tmem_wait_ld();
    for (int e = 0; e < 32; ++e) C[tid * N + c0 + e] = __uint_as_float(r[e]);
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (warp == 0) sm100::tmem_dealloc(tmem, 512);
}

// Tensor-core rate probe: `iters` back-to-back tcgen05.mma (M=128, N, K=16 each) on
// operands already in shared memory / TMEM (contents irrelevant), one commit at the
// end; returns elapsed SM cycles in out[0].
__global__ void __launch_bounds__(128) debug_mma_rate_kernel(int N, int iters, int a_mn, int b_mn, int a_tmem,
                                                             long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    sm100::tmem_alloc(&tmem_base, 512);
    sm100::tmem_relinquish();
  }
  if (tid == 0) {
    sm100::mbar_init(&bar, 1);
    sm100::fence_mbar_init();
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = sm100::make_idesc_bf16(128, N, a_mn != 0, b_mn != 0);
    const uint32_t a_base = sm100::smem_u32(base), b_base = sm100::smem_u32(base + 128 * 128 * 2);
    const uint64_t adesc0 = sm100::make_smem_desc(a_base, a_mn ? 128 * 128 : 16, 1024, sm100::kSwizzle128B);
    const uint64_t bdesc0 = sm100::make_smem_desc(b_base, b_mn ? 128 * 128 : 16, 1024, sm100::kSwizzle128B);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int s = i & 3;   // cycle over 4 k-steps of a 64-wide K atom
      const uint64_t ad = adesc0 + (uint64_t)((a_mn ? s * 2048 : s * 32) >> 4);
      const uint64_t bd = bdesc0 + (uint64_t)((b_mn ? s * 2048 : s * 32) >> 4);
      // a_tmem bit 1 (value 2/3): alternate between two independent accumulators
      const uint32_t dcol = (a_tmem & 2) ? (uint32_t)((i & 1) * (N <= 128 ? 128 : 0)) : 0u;
      if (a_tmem & 1)
        sm100::mma_ts(tmem + dcol, tmem + 256 + s * 8, bd, idesc, 1);
      else
        sm100::mma_ss(tmem + dcol, ad, bd, idesc, 1);
    }
    sm100::mma_commit(&bar);
    sm100::mbar_wait(&bar, 0);
    out[0] = clock64() - t0;
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (warp == 0) sm100::tmem_dealloc(tmem, 512);
}

// TMEM read/write rate probe: nwarps (multiple of 4) warps each issue `iters`
// tcgen05.ld (mode 0) or tcgen05.st (mode 1) of 32 lanes x 32 columns, waiting
// after every `batch` of them; returns SM cycles of warp 0 in out[0].
__global__ void debug_tmem_rate_kernel(int iters, int mode, int batch, long long* out) {
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    sm100::tmem_alloc(&tmem_base, 512);
    sm100::tmem_relinquish();
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tmem_base + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) & 3) * 128;
  uint32_t r[32];
  for (int e = 0; e < 32; ++e) r[e] = e;
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; i += batch) {
    for (int j = 0; j < batch; ++j) {
      const uint32_t col = (uint32_t)(((i + j) & 3) * 32);
      if (mode == 0) {
        sm100::tmem_ld32(tmem + col, r);
      } else {
        sm100::tmem_st32(tmem + col, r);
      }
    }
    if (mode == 0) {
      sm100::tmem_wait_ld();
      acc += r[0] + r[31];
    } else {
      sm100::tmem_wait_st();
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0 + (acc == 0xFFFFFFFF ? 1 : 0);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (warp == 0) sm100::tmem_dealloc(tmem_base, 512);
}

// MUFU.EX2 throughput probe: every thread runs `iters` x 16 independent ex2.approx;
// out[0] = SM cycles of the block.
__global__ void debug_ex2_rate_kernel(int iters, float seed, long long* out, float* sink) {
  float x[16];
  for (int i = 0; i < 16; ++i) x[i] = seed * (float)(threadIdx.x + i) * 1e-6f;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = sm100::ex2(x[i]) - 1.0f;
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.f) sink[0] = s;
  if (threadIdx.x == 0) out[0] = t1 - t0;
}

// XU / MUFU instruction-mix probe: `threads` threads of one CTA run `iters` x 16
// independent instances of one instruction form (mode):
//   0 ex2.approx.ftz.f32      1 ex2.approx.ftz.bf16x2   2 ex2.approx.f16x2
//   3 cvt.rn.bf16x2.f32       4 softmax pair loop as in attn_fwd (2 FFMA, 2 ex2.f32, FADD, cvt)
//   5 softmax pair loop with one ex2.bf16x2 per pair (FFMA x2 in fp32, ALU round + PRMT pack,
//     ex2.bf16x2, unpack + FADD for the row sum)
//   6 = 5 with the pack by cvt.rn.bf16x2.f32 instead of the ALU rounding
__device__ __forceinline__ uint32_t xu_ex2_bf16x2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t xu_ex2_f16x2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t xu_pack_round(float lo, float hi) {
  // round-half-up of the fp32 bits to bf16, both halves packed by one PRMT
  const uint32_t a = __float_as_uint(lo) + 0x8000u, b = __float_as_uint(hi) + 0x8000u;
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__global__ void debug_xu_rate_kernel(int mode, int iters, long long* out, uint32_t* sink) {
  uint32_t r[16];
  float f[16];
  for (int i = 0; i < 16; ++i) {
    f[i] = -(float)((threadIdx.x * 7 + i * 13) % 97) * 0.01f;
    r[i] = 0xBF00BF00u ^ (i << 3);
  }
  float l = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode == 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) f[i] = sm100::ex2(f[i]) - 1.0f;
    } else if (mode == 1) {
#pragma unroll
      for (int i = 0; i < 16; ++i) r[i] = xu_ex2_bf16x2(r[i]) ^ 0x80008000u;
    } else if (mode == 2) {
#pragma unroll
      for (int i = 0; i < 16; ++i) r[i] = xu_ex2_f16x2(r[i]) ^ 0x80008000u;
    } else if (mode == 3) {
#pragma unroll
      for (int i = 0; i < 16; ++i) r[i] = sm100::pack_bf16(f[i], __uint_as_float(r[i]));
    } else if (mode == 4) {
      float l4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float p0 = sm100::ex2(fmaf(f[2 * e], 0.18f, -l));
        const float p1 = sm100::ex2(fmaf(f[2 * e + 1], 0.18f, -l));
        l4[e & 3] += p0 + p1;
        r[e] ^= sm100::pack_bf16(p0, p1);
      }
      l += 1e-7f * ((l4[0] + l4[1]) + (l4[2] + l4[3]));
    } else {
      float l4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float x0 = fmaf(f[2 * e], 0.18f, -l), x1 = fmaf(f[2 * e + 1], 0.18f, -l);
        const uint32_t xp = mode == 5 ? xu_pack_round(x0, x1) : sm100::pack_bf16(x0, x1);
        const uint32_t p = xu_ex2_bf16x2(xp);
        l4[e & 3] += __uint_as_float(p << 16) + __uint_as_float(p & 0xFFFF0000u);
        r[e] ^= p;
      }
      l += 1e-7f * ((l4[0] + l4[1]) + (l4[2] + l4[3]));
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  uint32_t acc = __float_as_uint(l);
  for (int i = 0; i < 16; ++i) acc ^= r[i] ^ __float_as_uint(f[i]);
  if (acc == 0x12345678u) sink[0] = acc;
  if (threadIdx.x == 0) out[0] = t1 - t0;
}

// Synchronisation latency probe (one CTA, 64 threads; out[0] = cycles per round trip):
//   mode 0: one thread: tcgen05.commit (no MMA in flight) -> mbarrier -> wait, repeated
//   mode 1: one thread: one 128x128x16 SS MMA + commit -> wait, repeated
//   mode 2: ping-pong between warp 0 and warp 1 through two mbarriers (one arrive each way)
//   mode 3: as 2, warp 1 = 32 threads arriving (count 32) -- the softmax-style handoff
__global__ void __launch_bounds__(64) debug_sync_latency_kernel(int mode, int iters, long long* out) {
  __shared__ alignas(8) uint64_t bars[2];
  __shared__ uint32_t tmem_base;
  __shared__ alignas(1024) uint8_t tile[2][128 * 64 * 2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    sm100::mbar_init(&bars[0], 1);
    sm100::mbar_init(&bars[1], mode == 3 ? 32 : 1);
    sm100::fence_mbar_init();
  }
  if (warp == 0) {
    sm100::tmem_alloc(&tmem_base, 128);
    sm100::tmem_relinquish();
  }
  for (int i = threadIdx.x; i < 2 * 128 * 64 * 2 / 4; i += 64) reinterpret_cast<uint32_t*>(tile)[i] = 0;
  sm100::fence_proxy_async_smem();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tmem_base;
  long long t0 = 0, t1 = 0;
  if (mode <= 1) {
    if (threadIdx.x == 0) {
      const uint32_t idesc = sm100::make_idesc_bf16(128, 128, false, false);
      const uint64_t da = sm100::make_smem_desc(sm100::smem_u32(tile[0]), 16, 1024, sm100::kSwizzle128B);
      const uint64_t db = sm100::make_smem_desc(sm100::smem_u32(tile[1]), 16, 1024, sm100::kSwizzle128B);
      t0 = clock64();
      for (int it = 0; it < iters; ++it) {
        if (mode == 1) sm100::mma_ss(tmem, da, db, idesc, 0u);
        sm100::mma_commit(&bars[0]);
        sm100::mbar_wait(&bars[0], it & 1);
      }
      t1 = clock64();
    }
  } else {
    if (warp == 0 && lane == 0) {
      t0 = clock64();
      for (int it = 0; it < iters; ++it) {
        sm100::mbar_arrive(&bars[0]);
        sm100::mbar_wait(&bars[1], it & 1);
      }
      t1 = clock64();
    } else if (warp == 1 && (mode == 3 || lane == 0)) {
      for (int it = 0; it < iters; ++it) {
        sm100::mbar_wait(&bars[0], it & 1);
        sm100::mbar_arrive(&bars[1]);
      }
    }
  }
  if (threadIdx.x == 0) out[0] = (t1 - t0) / (iters > 0 ? iters : 1);
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc(tmem, 128);
}

// Softmax inner-loop probe: each thread exponentiates a 128-wide row `iters` times
// exactly like attn_fwd_kernel (FFMA + ex2 + row sum + bf16 pack); out[blockIdx] = cycles.
__global__ void __launch_bounds__(128) debug_softmax_rate_kernel(int iters, float sl2, long long* out, uint32_t* sink) {
  uint32_t sr[128];
  for (int i = 0; i < 128; ++i) sr[i] = __float_as_uint((float)((threadIdx.x * 7 + i * 13) % 97) * 0.01f);
  float l = 0.f, m_use = 0.5f;
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float l4[4] = {0.f, 0.f, 0.f, 0.f};
    uint32_t pk[64];
#pragma unroll
    for (int e = 0; e < 64; ++e) {
      const float p0 = sm100::ex2(fmaf(__uint_as_float(sr[2 * e]), sl2, -m_use));
      const float p1 = sm100::ex2(fmaf(__uint_as_float(sr[2 * e + 1]), sl2, -m_use));
      l4[e & 3] += p0 + p1;
      pk[e] = sm100::pack_bf16(p0, p1);
    }
    l += (l4[0] + l4[1]) + (l4[2] + l4[3]);
#pragma unroll
    for (int e = 0; e < 64; ++e) acc ^= pk[e];
    m_use += 1e-7f;
  }
  __syncthreads();
  const long long t1 = clock64();
  if (acc == 0x12345678u && l == 1.f) sink[0] = acc;
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

// The forward softmax tile body with its TMEM traffic, no MMA / TMA: per iteration
// S (128 fp32 per row) from TMEM -> row max -> 128 exponentials -> P (bf16) to TMEM.
// iters bit 20: a 5th warp keeps the tensor core busy meanwhile (SS MMAs N = 64 into
// TMEM cols [192, 256)), to see whether tcgen05 traffic slows the softmax warps.
__global__ void __launch_bounds__(160) debug_softmax_tile_kernel(int iters_flags, float sl2, long long* out,
                                                                   uint32_t* sink) {
  __shared__ uint32_t tmem_base;
  __shared__ alignas(1024) uint8_t ops[2 * 16384];
  __shared__ uint64_t bar;
  __shared__ volatile int done;
  const int iters = iters_flags & 0xFFFFF;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    sm100::tmem_alloc(&tmem_base, 256);
    sm100::tmem_relinquish();
  }
  if (threadIdx.x == 0) {
    sm100::mbar_init(&bar, 1);
    sm100::fence_mbar_init();
    done = 0;
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (warp == 4) {
    if (lane == 0 && (iters_flags >> 20)) {
      const uint32_t idesc = sm100::make_idesc_bf16(128, 64, false, false);
      const uint64_t ad = sm100::make_smem_desc(sm100::smem_u32(ops), 16, 1024, sm100::kSwizzle128B);
      const uint64_t bd = sm100::make_smem_desc(sm100::smem_u32(ops + 16384), 16, 1024, sm100::kSwizzle128B);
      uint32_t ph = 0;
      while (!done) {
        for (int i = 0; i < 64; ++i) sm100::mma_ss(tmem_base + 192, ad, bd, idesc, 1);
        sm100::mma_commit(&bar);
        sm100::mbar_wait(&bar, ph);
        ph ^= 1;
      }
    }
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    return;
  }
  const uint32_t tm = tmem_base + ((uint32_t)(warp * 32) << 16);
  {
    uint32_t init[32];
    for (int i = 0; i < 32; ++i) init[i] = __float_as_uint((float)((threadIdx.x * 7 + i * 13) % 97) * 0.01f);
    for (int c = 0; c < 4; ++c) sm100::tmem_st32(tm + c * 32, init);
    sm100::tmem_wait_st();
  }
  float l = 0.f, m_ref = -INFINITY;
  asm volatile("bar.sync 1, 128;" ::: "memory");
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t sr[128];
#pragma unroll
    for (int c = 0; c < 4; ++c) sm100::tmem_ld32(tm + c * 32, *reinterpret_cast<uint32_t(*)[32]>(sr + c * 32));
    sm100::tmem_wait_ld();
    float (&sv)[128] = *reinterpret_cast<float(*)[128]>(sr);
    float m8[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) m8[j] = sv[j];
#pragma unroll
    for (int c = 8; c < 128; ++c) m8[c & 7] = fmaxf(m8[c & 7], sv[c]);
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
    uint32_t pk[64];
#pragma unroll
    for (int e = 0; e < 64; ++e) {
      const float p0 = sm100::ex2(fmaf(sv[2 * e], sl2, -m_use));
      const float p1 = sm100::ex2(fmaf(sv[2 * e + 1], sl2, -m_use));
      l4[e & 3] += p0 + p1;
      pk[e] = sm100::pack_bf16(p0, p1);
    }
    l += (l4[0] + l4[1]) + (l4[2] + l4[3]);
#pragma unroll
    for (int c = 0; c < 4; ++c) sm100::tmem_st16(tm + 128 + c * 16, pk + c * 16);
    sm100::tmem_wait_st();
  }
  const long long t1 = clock64();
  if (l == 1.2345f) sink[0] = 1;
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  asm volatile("bar.sync 1, 128;" ::: "memory");
  if (threadIdx.x == 0) done = 1;
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (warp == 0) sm100::tmem_dealloc(tmem_base, 256);
}

// 128 token rows (indices idx[0..127]) of head h gathered with .tile::gather4 into a
// SWIZZLE_<2d> tile, then read back through the swizzle into out[128][d].
template <int D>
__global__ void __launch_bounds__(128) debug_gather_kernel(const __grid_constant__ CUtensorMap map,
                                                           const int32_t* __restrict__ idx, int h,
                                                           __nv_bfloat16* __restrict__ out) {
  __shared__ alignas(1024) uint8_t tile[128 * D * 2];
  __shared__ uint64_t bar;
  const int tid = threadIdx.x;
  if (tid == 0) {
    sm100::mbar_init(&bar, 1);
    sm100::fence_mbar_init();
  }
  __syncthreads();
  if (tid < 32) {
    if (tid == 0) sm100::mbar_arrive_expect_tx(&bar, 128 * D * 2);
    __syncwarp();
    const int4 r = *reinterpret_cast<const int4*>(idx + 4 * tid);
    sm100::tma_gather4(tile + 4 * tid * D * 2, &map, &bar, h * D, r.x, r.y, r.z, r.w, sm100::policy_evict_normal());
  }
  sm100::mbar_wait(&bar, 0);
  for (int e = 0; e < D; ++e) {
    const uint32_t off = (uint32_t)(tid * D * 2 + e * 2);
    const uint32_t phys = D == 64 ? sm100::swz128(off) : sm100::swz64(off);
    out[tid * D + e] = *reinterpret_cast<const __nv_bfloat16*>(tile + phys);
  }
}

}  // namespace
}  // namespace hla

using namespace hla;

extern "C" hla_status hla_debug_mma_rate(int32_t N, int32_t iters, int32_t a_major_mn, int32_t b_major_mn,
                                         int32_t a_from_tmem, long long* out_cycles, cudaStream_t stream) {
  clear_error();
  HLA_REQUIRE(N % 16 == 0 && N >= 16 && N <= 256 && iters > 0, HLA_ERR_INVALID, "bad N/iters");
  const size_t smem = 1024 + 2 * 128 * 256 * 2;
  HLA_CUDA_TRY(cudaFuncSetAttribute(debug_mma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  debug_mma_rate_kernel<<<1, 128, smem, stream>>>(N, iters, a_major_mn, b_major_mn, a_from_tmem, out_cycles);
  HLA_CUDA_TRY(cudaGetLastError());
  return HLA_OK;
}

extern "C" hla_status hla_debug_tmem_rate(int32_t nwarps, int32_t iters, int32_t mode, int32_t batch,
                                          long long* out_cycles, cudaStream_t stream) {
  clear_error();
  HLA_REQUIRE(nwarps % 4 == 0 && nwarps >= 4 && nwarps <= 16 && iters > 0 && batch >= 1, HLA_ERR_INVALID, "bad args");
  debug_tmem_rate_kernel<<<1, nwarps * 32, 0, stream>>>(iters, mode, batch, out_cycles);
  HLA_CUDA_TRY(cudaGetLastError());
  return HLA_OK;
}

extern "C" hla_status hla_debug_ex2_rate(int32_t threads, int32_t iters, long long* out_cycles, float* sink,
                                         cudaStream_t stream) {
  clear_error();
  debug_ex2_rate_kernel<<<1, threads, 0, stream>>>(iters, 1.0f, out_cycles, sink);
  HLA_CUDA_TRY(cudaGetLastError());
  return HLA_OK;
}

extern "C" hla_status hla_debug_xu_rate(int32_t mode, int32_t threads, int32_t iters, long long* out_cycles,
                                        uint32_t* sink, cudaStream_t stream) {
  clear_error();
  debug_xu_rate_kernel<<<1, threads, 0, stream>>>(mode, iters, out_cycles, sink);
  HLA_CUDA_TRY(cudaGetLastError());
  return HLA_OK;
}

extern "C" hla_status hla_debug_sync_latency(int32_t mode, int32_t iters, long long* out_cycles, cudaStream_t stream) {
  clear_error();
  debug_sync_latency_kernel<<<1, 64, 0, stream>>>(mode, iters, out_cycles);
  HLA_CUDA_TRY(cudaGetLastError());
  return HLA_OK;
}

extern "C" hla_status hla_debug_softmax_tile(int32_t blocks, int32_t iters, long long* out_cycles, uint32_t* sink,
                                             cudaStream_t stream) {
  clear_error();
  debug_softmax_tile_kernel<<<blocks, 160, 0, stream>>>(iters, 0.18f, out_cycles, sink);
  HLA_CUDA_TRY(cudaGetLastError());
  return HLA_OK;
}

extern "C" hla_status hla_debug_softmax_rate(int32_t blocks, int32_t iters, long long* out_cycles, uint32_t* sink,
                                             cudaStream_t stream) {
  clear_error();
  debug_softmax_rate_kernel<<<blocks, 128, 0, stream>>>(iters, 0.18f, out_cycles, sink);
  HLA_CUDA_TRY(cudaGetLastError());
  return HLA_OK;
}

// ---- load-rate probe: how fast can a CTA stream 16 KB K/V-like tiles (128 token
// rows x 64 bf16 of one head, rows heads*128 B apart) into shared memory?
// mode = base | (issuing warps W << 4) | (one barrier per issuing warp << 8);
// base 0 = 3-D TMA box (128 / W rows per warp), 1 = gather4 (32 / W per warp),
// 2 = cp.async by 128 threads (W = 4), 3 = 16 KB contiguous bulk copy (W = 1).
constexpr int kLoadStagesMax = 8;

__global__ void debug_load_kernel(const __grid_constant__ CUtensorMap m3, const __grid_constant__ CUtensorMap mg,
                                  const __grid_constant__ CUtensorMap m3b, const __grid_constant__ CUtensorMap mgb,
                                  const __nv_bfloat16* src, int64_t rows, int32_t heads, int32_t mode,
                                  int32_t stages, int32_t tiles, long long* out_cycles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t (*tile)[16384] = reinterpret_cast<uint8_t(*)[16384]>(base);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + stages * 16384);   // [stage][8]
  uint64_t* empty = full + kLoadStagesMax * 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kind = mode & 15, W = (mode >> 4) & 15, nb = (mode >> 8) & 1 ? W : 1;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      for (int j = 0; j < nb; ++j) sm100::mbar_init(&full[i * 8 + j], kind == 2 ? 128 / nb : 1);
      sm100::mbar_init(&empty[i * 8], 1);
    }
    sm100::fence_mbar_init();
  }
  __syncthreads();
  const long long t0 = clock64();
  const int64_t nrb = rows / 128;
  if (warp < W) {
    const int my_bar = nb > 1 ? warp : 0;
    const uint32_t part = 16384 / nb;
    for (int i = 0; i < tiles; ++i) {
      const int s = i % stages;
      if (i >= stages) sm100::mbar_wait(&empty[s * 8], ((i / stages) - 1) & 1);
      const int64_t t = (int64_t)blockIdx.x * tiles + i;
      const int32_t head = (int32_t)(t % heads);
      const int64_t r0 = ((t / heads) % nrb) * 128;
      uint8_t* dst = tile[s];
      uint64_t* bar = &full[s * 8 + my_bar];
      if ((mode >> 10) & 1) {   // L2 prefetch of tile i + 8
        const int64_t tp = (int64_t)blockIdx.x * tiles + i + 8;
        const int32_t hp = (int32_t)(tp % heads);
        const int64_t rp = ((tp / heads) % nrb) * 128;
        if (kind == 0) {
          if (lane == 0 && warp == 0) sm100::tma_prefetch_3d(&m3, 0, hp, (int32_t)rp);
        } else if (kind == 1) {
          const int per = 32 / W;
          if (lane < per) {
            const int32_t y = (int32_t)rp + 4 * (warp * per + lane);
            sm100::tma_prefetch_gather4(&mg, hp * 64, y, y + 1, y + 2, y + 3);
          }
        }
      }
      if (kind == 0) {
        if (lane == 0) {
          if (nb > 1 || warp == 0) sm100::mbar_arrive_expect_tx(bar, nb > 1 ? part : 16384);
        }
        if (W > 1) asm volatile("bar.sync 1, %0;" ::"r"(W * 32) : "memory");
        if (lane == 0) {
          const int rw = 128 / W;
          sm100::tma_load_3d(dst + warp * rw * 128, ((mode >> 9) & 1) && (warp & 1) ? &m3b : &m3, bar, 0, head, (int32_t)r0 + warp * rw,
                             sm100::policy_evict_first());
        }
      } else if (kind == 1) {
        if (lane == 0 && (nb > 1 || warp == 0)) sm100::mbar_arrive_expect_tx(bar, nb > 1 ? part : 16384);
        if (W > 1) asm volatile("bar.sync 1, %0;" ::"r"(W * 32) : "memory");
        const int per = 32 / W;
        if (lane < per) {
          const int gi = warp * per + lane;
          const int32_t y = (int32_t)r0 + 4 * gi;
          sm100::tma_gather4(dst + gi * 512, ((mode >> 9) & 1) && (warp & 1) ? &mgb : &mg, bar, head * 64, y, y + 1, y + 2, y + 3,
                             sm100::policy_evict_first());
        }
      } else if (kind == 2) {
        const int j = threadIdx.x;   // row
        const char* g = reinterpret_cast<const char*>(src + ((r0 + j) * heads + head) * 64);
        const uint32_t d = sm100::smem_u32(dst + j * 128);
#pragma unroll
        for (int c = 0; c < 8; ++c)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + c * 16), "l"(g + c * 16) : "memory");
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(sm100::smem_u32(bar)) : "memory");
      } else if (lane == 0) {
        const int64_t nt = rows * heads * 128 / 16384;
        sm100::mbar_arrive_expect_tx(bar, 16384);
        sm100::bulk_load(dst, reinterpret_cast<const char*>(src) + (t % nt) * 16384, 16384, bar);
      }
    }
  } else if (warp == W && lane == 0) {
    for (int i = 0; i < tiles; ++i) {
      const int s = i % stages;
      for (int j = 0; j < nb; ++j) sm100::mbar_wait(&full[s * 8 + j], (i / stages) & 1);
      sm100::mbar_arrive(&empty[s * 8]);
    }
    out_cycles[blockIdx.x] = clock64() - t0;
  }
}

extern "C" hla_status hla_debug_load_rate(const void* src, int64_t rows, int32_t heads, int32_t mode,
                                          int32_t stages, int32_t ctas, int32_t tiles, long long* out_cycles,
                                          cudaStream_t stream) {
  clear_error();
  const int kind = mode & 15, W = (mode >> 4) & 15;
  HLA_REQUIRE(src && out_cycles && kind <= 3 && W >= 1 && W <= 8 && 32 % W == 0 && (kind != 2 || W == 4) &&
                  stages >= 1 && stages <= kLoadStagesMax && rows % 128 == 0,
              HLA_ERR_INVALID, "bad load-rate probe arguments");
  CUtensorMap m3, mg, m3b, mgb;
  hla_status st = make_rows_map(&m3, src, rows, heads, 64, kind == 0 ? 128 / W : 128);
  if (st != HLA_OK) return st;
  st = make_gather_map(&mg, src, rows, heads, 64, 1);
  if (st != HLA_OK) return st;
  // mode bit 9: odd warps use a second (identical) tensor map
  if ((st = make_rows_map(&m3b, src, rows, heads, 64, kind == 0 ? 128 / W : 128)) != HLA_OK) return st;
  if ((st = make_gather_map(&mgb, src, rows, heads, 64, 1)) != HLA_OK) return st;
  const size_t smem = (size_t)stages * 16384 + 2 * kLoadStagesMax * 8 * 8 + 1024;
  HLA_CUDA_TRY(cudaFuncSetAttribute(debug_load_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  debug_load_kernel<<<ctas, 32 * (W + 1), smem, stream>>>(m3, mg, m3b, mgb, reinterpret_cast<const __nv_bfloat16*>(src),
                                                          rows, heads, mode, stages, tiles, out_cycles);
  HLA_CUDA_TRY(cudaGetLastError());
  return HLA_OK;
}

extern "C" hla_status hla_debug_gather4(const void* src, int64_t rows, int32_t heads, int32_t head_dim,
                                        const int32_t* idx, int32_t head, int32_t box_h, void* out,
                                        cudaStream_t stream) {
  clear_error();
  HLA_REQUIRE(head_dim == 32 || head_dim == 64, HLA_ERR_UNSUPPORTED, "head_dim");
  CUtensorMap map;
  hla_status st = make_gather_map(&map, src, rows, heads, head_dim, box_h);
  if (st != HLA_OK) return st;
  if (head_dim == 64)
    debug_gather_kernel<64><<<1, 128, 0, stream>>>(map, idx, head, reinterpret_cast<__nv_bfloat16*>(out));
  else
    debug_gather_kernel<32><<<1, 128, 0, stream>>>(map, idx, head, reinterpret_cast<__nv_bfloat16*>(out));
  HLA_CUDA_TRY(cudaGetLastError());
  return HLA_OK;
}

extern "C" hla_status hla_debug_umma(const void* A, const void* B, float* C, int32_t M, int32_t N, int32_t K,
                                     int32_t a_major_mn, int32_t b_major_mn, int32_t a_from_tmem,
                                     cudaStream_t stream) {
  clear_error();
  HLA_REQUIRE(A && B && C, HLA_ERR_INVALID, "null pointer");
  HLA_REQUIRE(M == 128, HLA_ERR_UNSUPPORTED, "M must be 128");
  HLA_REQUIRE(N % 64 == 0 && N >= 64 && N <= 256, HLA_ERR_UNSUPPORTED, "N must be 64..256 step 64");
  HLA_REQUIRE(K == 64 || K == 128, HLA_ERR_UNSUPPORTED, "K must be 64 or 128");
  HLA_REQUIRE(!(a_from_tmem && a_major_mn), HLA_ERR_INVALID, "A in TMEM is K-major");
  const size_t smem = 1024 + (size_t)(M + N) * K * 2;
  HLA_CUDA_TRY(cudaFuncSetAttribute(debug_umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  debug_umma_kernel<<<1, 128, smem, stream>>>(reinterpret_cast<const __nv_bfloat16*>(A),
                                              reinterpret_cast<const __nv_bfloat16*>(B), C, N, K, a_major_mn,
                                              b_major_mn, a_from_tmem);
  HLA_CUDA_TRY(cudaGetLastError());
  return HLA_OK;
}
