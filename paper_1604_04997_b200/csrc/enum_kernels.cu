// GPU enumeration oracle: brute-force walk of one statement domain at one
// binding (the reference's enumerate_points / FastDomain::run,
// enumerate.cpp:247-293 and 371-405), one thread per point of the
// rectangular prefix of the domain.
//
//   * Levels whose bounds depend on parameters only (group / local axes and
//     loops with parameter bounds -- every kernel of the bundled suite) form
//     a box that is flattened over the grid: thread t decodes its digits,
//     innermost level fastest.
//   * Deeper (triangular) levels are walked depth-first per thread exactly
//     like FastDomain::descend: bounds ceil(raw/den), guards at the depth of
//     their deepest variable, a guard failure is one visited dead end.
//   * A guard failing at box depth d is a dead end of the prefix
//     (x_0..x_d); it is charged once, by the thread whose deeper box digits
//     are all zero.
//   * Every leaf marks the cells of the statement's global accesses in the
//     array's bitmaps (distinct cells, the projection on the non-fastest
//     axes, and the fastest-axis coordinates); lanes hitting the same word
//     combine their bits (__match_any_sync / __reduce_or_sync) and the word
//     is read before the atomic, so repeated cells cost a load, not an L2
//     atomic.
// Leaves and visited points are reduced per warp into out[0..1].
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "kcg_enum_dev.h"
#include "kcg_kernels.hpp"

namespace {

typedef long long i64;
typedef unsigned long long u64;

__device__ __forceinline__ i64 ke_lin(const KeRow& r, const i64* x, int nv) {
  i64 v = r.c0;
#pragma unroll
  for (int s = 0; s < KE_MAXV; ++s)
    if (s < nv) v += r.c[s] * x[s];
  return v;
}

// floor(a / d), d > 0 (numeric.hpp:24-28)
__device__ __forceinline__ i64 ke_floor_div(i64 a, i64 d) {
  i64 q = a / d;
  if (a % d != 0 && a < 0) q -= 1;
  return q;
}

// the row's raw value, floor divisions over domain variables included
__device__ __forceinline__ i64 ke_raw(const KeRow& r, const i64* x, int nv, const KeStmt& S) {
  i64 v = ke_lin(r, x, nv);
  for (int f = 0; f < S.nf; ++f)
    if (r.cf[f] != 0) v += r.cf[f] * ke_floor_div(ke_lin(S.f[f].r, x, nv), S.f[f].div);
  return v;
}

// ceil(a / d) for d > 0 (enumerate.cpp:18-20)
__device__ __forceinline__ i64 ke_ceil_div(i64 a, i64 d) {
  i64 q = a / d;
  if (a % d != 0 && a > 0) q += 1;
  return q;
}

__device__ __forceinline__ bool ke_guard(const KeGuard& g, const i64* x, int nv, const KeStmt& S) {
  const i64 v = ke_raw(g.r, x, nv, S);
  if (g.divis) {
    i64 m = v % g.mod;
    if (m < 0) m += g.mod;
    return m == g.rem;
  }
  switch (g.op) {  // den > 0 keeps the orientation (enumerate.cpp:175-181)
    case 0: return v < 0;
    case 1: return v <= 0;
    case 2: return v > 0;
    case 3: return v >= 0;
    default: return v == 0;
  }
}

// set a bit; lanes of a warp that hit the same 32-bit word combine their
// bits first (one load and at most one atomic per distinct word)
__device__ __forceinline__ void ke_set(u64* bm64, u64 bit) {
  unsigned* w = reinterpret_cast<unsigned*>(bm64) + (bit >> 5);  // little endian: same bit numbering
  const unsigned m = 1u << (bit & 31);
  const unsigned act = __activemask();
  const unsigned grp = __match_any_sync(act, reinterpret_cast<unsigned long long>(w));
  const unsigned bits = __reduce_or_sync(grp, m);
  if ((threadIdx.x & 31) == (unsigned)(__ffs(grp) - 1) && (__ldcg(w) & bits) != bits) atomicOr(w, bits);
}

__device__ __forceinline__ void ke_mark(const KeStmt& S, const i64* x) {
  for (int a = 0; a < S.na; ++a) {
    const KeAccess& A = S.a[a];
    const KeMark& M = A.m;
    u64 lin = 0, lino = 0, fast = 0;
    for (int k = 0; k < M.nd; ++k) {
      const u64 v = (u64)(ke_raw(A.idx[k], x, S.nv, S) - M.lo[k]);
      lin = lin * (u64)M.ext[k] + v;
      if (k == M.fast)
        fast = v;
      else
        lino = lino * (u64)M.ext[k] + v;
    }
    ke_set(M.cells, lin);
    ke_set(M.others, lino);
    ke_set(M.fastp, fast);
  }
}

__global__ void __launch_bounds__(256) kcg_enum_walk(const KeStmt* __restrict__ sp) {
  const KeStmt& S = *sp;
  const int nv = S.nv, nbox = S.nbox, nbe = S.nbe;
  u64 leaves = 0, visited = 0;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < S.box_total; t += stride) {
    i64 x[KE_MAXV];
    int lowest_nonzero = -1;  // deepest box level with a nonzero digit
    {
      u64 r = t;
      for (int l = nbe - 1; l >= 0; --l) {
        const u64 e = (u64)S.box_ext[l];
        const u64 d = r % e;
        r /= e;
        x[l] = S.box_lo[l] + (i64)d;
        if (d != 0 && lowest_nonzero < 0) lowest_nonzero = l;
      }
    }
    for (int l = nbe; l < KE_MAXV; ++l) x[l] = 0;
    // guards of the box levels, shallowest first
    int dead = -1;
    for (int l = 0; l < nbe && dead < 0; ++l)
      for (int k = 0; k < S.ng; ++k)
        if (S.g[k].depth == l && !ke_guard(S.g[k], x, nv, S)) {
          dead = l;
          break;
        }
    if (dead >= 0) {
      if (lowest_nonzero <= dead) ++visited;  // one dead end per failing prefix
      continue;
    }
    if (!S.inner) continue;  // an empty box level: no leaves below
    if (nbox == nv) {
      ++visited;
      ++leaves;
      ke_mark(S, x);
      continue;
    }
    // depth-first over the triangular levels nbox..nv-1
    i64 hi[KE_MAXV];
    int l = nbox;
    x[l] = ke_ceil_div(ke_raw(S.lo[l], x, nv, S), S.lo[l].den);
    hi[l] = ke_ceil_div(ke_raw(S.hi[l], x, nv, S), S.hi[l].den);
    while (true) {
      if (x[l] >= hi[l]) {
        if (l == nbox) break;
        x[l] = 0;
        --l;
        ++x[l];
        continue;
      }
      bool pass = true;
      for (int k = 0; k < S.ng; ++k)
        if (S.g[k].depth == l && !ke_guard(S.g[k], x, nv, S)) {
          pass = false;
          break;
        }
      if (!pass) {
        ++visited;
        ++x[l];
        continue;
      }
      if (l == nv - 1) {
        ++visited;
        ++leaves;
        ke_mark(S, x);
        ++x[l];
        continue;
      }
      ++l;
      x[l] = ke_ceil_div(ke_raw(S.lo[l], x, nv, S), S.lo[l].den);
      hi[l] = ke_ceil_div(ke_raw(S.hi[l], x, nv, S), S.hi[l].den);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    leaves += __shfl_down_sync(0xffffffffu, leaves, o);
    visited += __shfl_down_sync(0xffffffffu, visited, o);
  }
  if ((threadIdx.x & 31) == 0 && (leaves | visited)) {
    atomicAdd(S.out, leaves);
    atomicAdd(S.out + 1, visited);
  }
}

// out[0] += popcount, out[1] = min set bit, out[2] = max set bit
__global__ void __launch_bounds__(256) kcg_enum_bits(const u64* __restrict__ bm, u64 words, u64* out) {
  u64 pop = 0, mn = ~0ull, mx = 0;
  bool any = false;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 w = (u64)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += stride) {
    const u64 v = bm[w];
    if (!v) continue;
    pop += (u64)__popcll(v);
    const u64 lo = w * 64 + (u64)(__ffsll((long long)v) - 1);
    const u64 hi = w * 64 + 63 - (u64)__clzll((long long)v);
    mn = lo < mn ? lo : mn;
    mx = hi > mx ? hi : mx;
    any = true;
  }
  for (int o = 16; o > 0; o >>= 1) {
    pop += __shfl_down_sync(0xffffffffu, pop, o);
    const u64 a = __shfl_down_sync(0xffffffffu, mn, o), b = __shfl_down_sync(0xffffffffu, mx, o);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
    any = __any_sync(0xffffffffu, any);
  }
  if ((threadIdx.x & 31) == 0 && any) {
    atomicAdd(out, pop);
    atomicMin(out + 1, mn);
    atomicMax(out + 2, mx);
  }
}

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

namespace kcg {

void launch_enum_walk(const KeStmt* dev_stmt, unsigned long long box_total, cudaStream_t stream) {
  if (box_total == 0) return;
  const unsigned long long need = (box_total + 255) / 256;
  const unsigned long long cap = static_cast<unsigned long long>(num_sms()) * 8;
  const unsigned grid = static_cast<unsigned>(need < cap ? need : cap);
  kcg_enum_walk<<<grid, 256, 0, stream>>>(dev_stmt);
  check(cudaGetLastError(), "kcg_enum_walk launch");
}

void launch_enum_bits(const unsigned long long* bm, unsigned long long words, unsigned long long* out,
                      cudaStream_t stream) {
  if (words == 0) return;
  const unsigned long long need = (words + 255) / 256;
  const unsigned long long cap = static_cast<unsigned long long>(num_sms()) * 8;
  const unsigned grid = static_cast<unsigned>(need < cap ? need : cap);
  kcg_enum_bits<<<grid, 256, 0, stream>>>(bm, words, out);
  check(cudaGetLastError(), "kcg_enum_bits launch");
}

}  // namespace kcg
