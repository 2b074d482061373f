// Device helpers shared by the ahead-of-time kernels (kernels.cu) and the
// NVRTC-specialised kernels (codegen.cpp embeds this file verbatim).
//
// Exactness rules:
//   * floor division is sign-correct like kernelcost::floor_div
//     (numeric.hpp:24-28);
//   * int -> double is round-to-nearest-even, also for 128-bit counts;
//   * predict accumulates part = alpha*count; s += part with two separate
//     roundings (__dmul_rn / __dadd_rn, never contracted to FMA), in schema
//     order, skipping zero counts (model.cpp:106-111) or, for the simulator,
//     zero weights (simdevice.cpp:84-88).
#pragma once

#ifndef KCG_DEVICE_HELPERS
#define KCG_DEVICE_HELPERS

typedef long long kcg_i64;
typedef unsigned long long kcg_u64;
typedef __int128 kcg_i128;
typedef unsigned __int128 kcg_u128;

#define KCG_PT_OK 0
#define KCG_PT_ASSUMPTION_VIOLATED 1
#define KCG_PT_NONINTEGRAL 2
#define KCG_PT_OVERFLOW 3
#define KCG_PT_COUNT_WIDE 4

template <class T>
__device__ __forceinline__ T kcg_const(kcg_i64 lo, kcg_i64 hi);
template <>
__device__ __forceinline__ kcg_i64 kcg_const<kcg_i64>(kcg_i64 lo, kcg_i64) {
  return lo;
}
template <>
__device__ __forceinline__ kcg_i128 kcg_const<kcg_i128>(kcg_i64 lo, kcg_i64 hi) {
  return (kcg_i128)(((kcg_u128)(kcg_u64)hi << 64) | (kcg_u128)(kcg_u64)lo);
}

// Stage hand-back of the TMA rings: each consumer warp's lane 0 (after
// __syncwarp, its shared-memory reads of the stage done) publishes them with
// a release fence and a counter increment; the last to arrive acquires
// every warp's reads with a second fence before it issues the async-proxy
// refill (fence-fence synchronisation through the counter). An `empty`
// mbarrier per stage instead cost 6-25% at one CTA per SM (F = 48: 8.70 ->
// 9.9 ms, F = 56: 11.0 -> 13.9), and compute-sanitizer racecheck models
// neither (profiles/racecheck_mbarrier_probe.cu: an mbarrier-ordered store is
// reported like an unsynchronised one), so racecheck runs at sizes where the
// rings do not refill.
#ifdef __CUDACC__  // not in the host build of the evaluator (source kind 4)
__device__ __forceinline__ bool kcg_ring_release(unsigned* count, unsigned consumers) {
  __threadfence_block();
  if (atomicAdd(count, 1u) != consumers - 1) return false;
  __threadfence_block();
  *count = 0;
  return true;
}
#endif

// floor(a / b) for b > 0

template <class T>
__device__ __forceinline__ T kcg_floordiv(T a, T b) {
  T q = a / b;
  if ((a % b != 0) && (a < 0)) q -= 1;
  return q;
}

// ((v % m) + m) % m  (LinCmp::evaluate, linexpr.cpp:128-133)
template <class T>
__device__ __forceinline__ T kcg_posmod(T v, T m) {
  T r = v % m;
  if (r < 0) r += m;
  return r;
}

__device__ __forceinline__ double kcg_to_double(kcg_i64 v) {
  return __ll2double_rn(v);
}

// correctly rounded (nearest-even) int128 -> double
__device__ __forceinline__ double kcg_to_double(kcg_i128 v) {
  const kcg_i64 lo = (kcg_i64)v;
  if ((kcg_i128)lo == v) return __ll2double_rn(lo);
  const bool neg = v < 0;
  const kcg_u128 u = neg ? (kcg_u128)0 - (kcg_u128)v : (kcg_u128)v;
  const kcg_u64 hi = (kcg_u64)(u >> 64);
  double d;
  if (hi == 0) {
    d = __ull2double_rn((kcg_u64)u);
  } else {
    const int shift = 64 - __clzll((long long)hi);  // bits beyond 64, 1..64
    const kcg_u128 mask = (((kcg_u128)1) << shift) - 1;
    kcg_u64 top = (kcg_u64)(u >> shift);
    if ((u & mask) != 0) top |= 1ull;  // sticky bit below the rounding point
    d = __ull2double_rn(top);
    d = scalbn(d, shift);  // exact power-of-two scaling
  }
  return neg ? -d : d;
}

__device__ __forceinline__ bool kcg_fits_i64(kcg_i64) { return true; }
__device__ __forceinline__ bool kcg_fits_i64(kcg_i128 v) {
  return (kcg_i128)(kcg_i64)v == v;
}
__device__ __forceinline__ kcg_i64 kcg_hi64(kcg_i64 v) { return v < 0 ? -1 : 0; }
__device__ __forceinline__ kcg_i64 kcg_hi64(kcg_i128 v) { return (kcg_i64)(v >> 64); }

// s += alpha * count, two roundings, skip per predict/simulate rule
template <class T>
__device__ __forceinline__ double kcg_accum(double s, double alpha, T count, int simulate) {
  const bool take = simulate ? (alpha != 0.0) : (count != 0);
  if (take) s = __dadd_rn(s, __dmul_rn(alpha, kcg_to_double(count)));
  return s;
}

// same rule when the count is already RN(double(count)) (count == 0 <=> 0.0)
__device__ __forceinline__ double kcg_accum(double s, double alpha, double count, int simulate) {
  const bool take = simulate ? (alpha != 0.0) : (count != 0.0);
  if (take) s = __dadd_rn(s, __dmul_rn(alpha, count));
  return s;
}

__device__ __forceinline__ double kcg_nan() { return __longlong_as_double(0x7ff8000000000000ll); }
__device__ __forceinline__ unsigned long long kcg_abs_bits(double x) {
  // |x| as a bit pattern with the sign cleared on the integer pipe (a plain
  // mask compiles to DADD |x| on the FP64 pipe, which the DMMAs share)
  unsigned lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "d"(x));
  asm volatile("and.b32 %0, %0, 0x7fffffff;" : "+r"(hi));
  return ((unsigned long long)hi << 32) | lo;
}

#endif  // KCG_DEVICE_HELPERS
