// common.cuh -- shared device helpers for the B200 hdll encoder.
//
// Every floating-point expression that restates a reference expression is
// compiled with -fmad=false (no contraction), so `a * b + c` rounds twice
// exactly like numpy / numba / CPython floats.  The only
// fused multiply-adds are explicit __fma_rn calls that model OpenBLAS's ddot.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace hdll {

constexpr int kRiceMaxK = 15;    // _kernels.py:13
constexpr int kRiceEscapeQ = 24; // _kernels.py:14
constexpr int kStateReset = 64;  // _kernels.py:15
constexpr int kEOB = 64;         // _kernels.py:19
constexpr int kRunCtx = 4;       // _kernels.py:17

// Error bits written to the per-launch device status word.
enum : uint32_t {
  kErrNonFinite = 1u << 0,   // float32 regression parameter overflow (estimator.py:66-67)
  kErrLookback = 1u << 1,    // decoupled look-back gave up (would otherwise hang)
  kErrCapacity = 1u << 2,    // a staging buffer bound was exceeded
  kErrInternal = 1u << 3,
};

// round_half_away, _util.py:8-11: trunc(x + copysign(0.5, x))
__device__ __forceinline__ double rha(double x) { return trunc(x + copysign(0.5, x)); }
// round_half_away(x) as an int: the truncating conversion does the trunc (one
// conversion instead of a rounding and a conversion; saturates out of range)
__device__ __forceinline__ int rha_int(double x) { return (int)(x + copysign(0.5, x)); }

__device__ __forceinline__ double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

// ---------------------------------------------------------------------------
// Warp helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

template <typename T>
__device__ __forceinline__ T warp_excl_sum(T v, T* total) {
  unsigned lane = lane_id();
  T x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= (unsigned)d) x += y;
  }
  if (total) *total = __shfl_sync(0xffffffffu, x, 31);
  return x - v;
}

// ---------------------------------------------------------------------------
// Adaptive Rice state algebra (the parallel form of _kernels.py:114-128).
//
// Per context the state A evolves symbol by symbol as A <- (A + u) >> h where
// h = 1 exactly when the context's running count N reaches 64 (N depends only
// on the symbol's index in the context, so h is known once counts are scanned).
// Maps f(A) = floor((A + c) / 2^s) compose exactly:
//   g(f(A)) = floor((A + c1 + (c2 << s1)) / 2^(s1+s2)).
// The state never exceeds 16194 < 2^14 (SURVEY.md hard part 2), so once
// s >= 14 the map takes at most two values on the domain [0, 2^14): it is
// kept as a step map f(A) = q + (A >= t).  Maps are then O(1) in size.
// ---------------------------------------------------------------------------
constexpr int kADomainBits = 14;
constexpr int kADomain = 1 << kADomainBits;  // 16384

struct AMap {
  long long c;  // exact: additive constant; step: q
  int s;        // exact: shift (< 14); step: -1
  int t;        // step: threshold in [0, kADomain]
};

__device__ __forceinline__ AMap amap_identity() { return AMap{0, 0, 0}; }
__device__ __forceinline__ bool amap_is_step(const AMap& m) { return m.s < 0; }

__device__ __forceinline__ long long amap_apply(const AMap& m, long long a) {
  if (m.s >= 0) return (a + m.c) >> m.s;
  return m.c + (a >= m.t ? 1 : 0);
}

__device__ __forceinline__ AMap amap_make_step_from_exact(long long c, int s) {
  // f(A) = (A + c) >> s for A in [0, 2^14), s >= 14: q or q+1, q+1 iff A >= ((q+1) << s) - c
  long long q = c >> s;
  long long t = ((q + 1) << s) - c;
  if (t > kADomain) t = kADomain;
  if (t < 0) t = 0;
  AMap r;
  r.c = q;
  r.s = -1;
  r.t = (int)t;
  return r;
}

// then(f, g) = g o f  (apply f first)
__device__ __forceinline__ AMap amap_then(const AMap& f, const AMap& g) {
  if (f.s < 0) {  // f is a step map with values q, q+1
    long long v0 = amap_apply(g, f.c);
    long long v1 = amap_apply(g, f.c + 1);
    AMap r;
    r.c = v0;
    r.s = -1;
    r.t = (v1 == v0) ? kADomain : f.t;
    return r;
  }
  if (g.s < 0) {  // exact then step: q2 + [((A + c1) >> s1) >= t2]
    long long t = ((long long)g.t << f.s) - f.c;
    if (g.t >= kADomain) t = kADomain;  // g never steps
    if (t > kADomain) t = kADomain;
    if (t < 0) t = 0;
    AMap r;
    r.c = g.c;
    r.s = -1;
    r.t = (int)t;
    return r;
  }
  long long c = f.c + (g.c << f.s);
  int s = f.s + g.s;
  if (s >= kADomainBits) return amap_make_step_from_exact(c, s);
  AMap r;
  r.c = c;
  r.s = s;
  r.t = 0;
  return r;
}

// One symbol u with halving flag h appended after map m.
__device__ __forceinline__ AMap amap_push(const AMap& m, int u, int h) {
  if (m.s < 0) {
    long long v0 = (m.c + u) >> h, v1 = (m.c + 1 + u) >> h;
    AMap r;
    r.c = v0;
    r.s = -1;
    r.t = (v1 == v0) ? kADomain : m.t;
    return r;
  }
  long long c = m.c + ((long long)u << m.s);
  int s = m.s + h;
  if (s >= kADomainBits) return amap_make_step_from_exact(c, s);
  AMap r;
  r.c = c;
  r.s = s;
  r.t = 0;
  return r;
}

__device__ __forceinline__ AMap shfl_amap(const AMap& m, int src, unsigned mask = 0xffffffffu) {
  AMap r;
  r.c = __shfl_sync(mask, m.c, src);
  r.s = __shfl_sync(mask, m.s, src);
  r.t = __shfl_sync(mask, m.t, src);
  return r;
}

__device__ __forceinline__ AMap shfl_up_amap(const AMap& m, int d) {
  AMap r;
  r.c = __shfl_up_sync(0xffffffffu, m.c, d);
  r.s = __shfl_up_sync(0xffffffffu, m.s, d);
  r.t = __shfl_up_sync(0xffffffffu, m.t, d);
  return r;
}

// Exclusive composition scan across the warp (lane 0 gets identity);
// *total = composition of all 32 lanes in lane order.
__device__ __forceinline__ AMap warp_excl_amap(const AMap& m, AMap* total) {
  unsigned lane = lane_id();
  AMap x = m;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    AMap y = shfl_up_amap(x, d);
    if (lane >= (unsigned)d) x = amap_then(y, x);
  }
  if (total) *total = shfl_amap(x, 31);
  AMap ex = shfl_up_amap(x, 1);
  if (lane == 0) ex = amap_identity();
  return ex;
}

// Halving happens after the symbol with 0-based context index j when
// N reaches 64: j = 62, 94, 126, ... (N runs 1..63, then 32..63).
__device__ __forceinline__ int halves_after(long long j) { return (j >= 62 && ((j - 62) & 31) == 0) ? 1 : 0; }

// N before the symbol with context index j.
__device__ __forceinline__ int n_before(long long j) { return j < 63 ? (int)(j + 1) : 32 + (int)((j - 63) & 31); }

// _select_k, _kernels.py:114-119
__device__ __forceinline__ int select_k(long long a, int n) {
  int k = 0;
  while (((long long)n << k) < a && k < kRiceMaxK) k++;
  return k;
}

// Code length of a Rice symbol (_rice_put, _kernels.py:65-79)
__device__ __forceinline__ int rice_len(int u, int k) {
  int q = u >> k;
  return q < kRiceEscapeQ ? q + 1 + k : kRiceEscapeQ + 8;
}

// The Rice code as a right-aligned bit pattern of rice_len bits (<= 32).
__device__ __forceinline__ uint32_t rice_bits(int u, int k) {
  int q = u >> k;
  if (q < kRiceEscapeQ) {
    // q ones, a zero, k remainder bits
    const uint32_t ones = ((1u << q) - 1u) << (k + 1);  // q + 1 + k <= 32 for u <= 255
    return ones | ((uint32_t)u & ((1u << k) - 1u));
  }
  return (((1u << kRiceEscapeQ) - 1u) << 8) | ((uint32_t)u & 0xFFu);
}

// ---------------------------------------------------------------------------
// Release/acquire flag helpers for decoupled look-back.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ---------------------------------------------------------------------------
// CRC-32 (zlib.crc32, codec_core.py:252-253): reflected 0xEDB88320.
// ---------------------------------------------------------------------------
constexpr uint32_t kCrcPoly = 0xEDB88320u;

// a * b mod P in the reflected representation (zlib multmodp)
__device__ __host__ __forceinline__ uint32_t crc_multmodp(uint32_t a, uint32_t b) {
  uint32_t p = 0;  // branch-free: bit 31 - i of a selects b * x^i
#pragma unroll
  for (int i = 0; i < 32; i++) {
    p ^= b & (0u - ((a >> (31 - i)) & 1u));
    b = (b >> 1) ^ (kCrcPoly & (0u - (b & 1u)));
  }
  return p;
}

// ---------------------------------------------------------------------------
// Bulk async copies (cp.async.bulk, the non-tensor TMA path) with mbarriers.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// Ampere-style per-thread async copies (LDGSTS), 8 bytes
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

}  // namespace hdll
