// Ahead-of-time sm_100a kernels:
//   * kcg_interp_eval   -- table interpreter for evaluate_properties + predict
//                          (generic engine; the JIT engine specialises the same
//                          semantics into straight-line code, codegen.cpp)
//   * kcg_gram_x        -- G += X^T X, X^T 1, column max|x| over a materialised
//                          fp64 design (the reduction fit_weights needs,
//                          model.cpp:62-80), register-tiled 4x4 over the upper
//                          triangle, rows staged through shared memory
//   * kcg_resid_x / kcg_resid_grad_x -- sum (1 - X a)^2 and X^T (1 - X a)
#include <mutex>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <utility>

#include "kcg_device.cuh"
#include "kcg_kernels.hpp"

namespace kcg {

namespace {

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class T>
__device__ __forceinline__ T wide(const KcgWide& w) {
  return kcg_const<T>(w.lo, w.hi);
}

// ---------------------------------------------------------------------------
// interpreter

template <class T>
__device__ __noinline__ int interp_body(const KcgDevProg* __restrict__ P,
                                        const kcg_i64* p, T* cnt) {
  T atom[KCG_MAX_ATOMS];
  T mono[KCG_MAX_MONOS];
  T expr[KCG_MAX_EXPRS];
  const int nops = P->n_ops;
  for (int k = 0; k < nops; ++k) {
    const KcgDevOp op = P->ops[k];
    switch (op.code) {
      case 0:
        atom[op.dst] = (T)p[op.a];
        break;
      case 1: {
        T m = (T)1;
        for (int i = op.a; i < op.b; ++i) {
          const T v = atom[P->fac_atom[i]];
          for (int e = 0; e < P->fac_exp[i]; ++e) m *= v;
        }
        mono[op.dst] = m;
        break;
      }
      case 2: {
        T s = (T)0;
        for (int i = op.a; i < op.b; ++i) {
          const T c = wide<T>(P->term_coef[i]);
          const int mi = P->term_mono[i];
          s += mi < 0 ? c : c * mono[mi];
        }
        expr[op.dst] = s;
        break;
      }
      case 3:
        atom[op.dst] = kcg_floordiv<T>(expr[op.a], wide<T>(P->fd_den[op.c]));
        break;
      case 6:
        atom[op.dst] = kcg_floordiv<T>((T)p[op.a] - wide<T>(P->quot_rem[op.c]),
                                       wide<T>(P->quot_mod[op.c]));
        break;
      default: {
        T best = expr[P->arg_expr[op.a]] * wide<T>(P->arg_scale[op.a]);
        for (int i = op.a + 1; i < op.b; ++i) {
          const T v = expr[P->arg_expr[i]] * wide<T>(P->arg_scale[i]);
          if (op.code == 4 ? v < best : v > best) best = v;
        }
        atom[op.dst] = best;
        break;
      }
    }
  }
  for (int c = 0; c < P->n_cons; ++c) {
    if (P->cons_div[c] == 2) {  // p == M * quot + R
      const T q = atom[P->cons_expr[c]];
      if ((T)p[P->cons_op[c]] - wide<T>(P->cons_rem[c]) != wide<T>(P->cons_mod[c]) * q)
        return KCG_PT_ASSUMPTION_VIOLATED;
      continue;
    }
    const T e = expr[P->cons_expr[c]];
    if (!P->cons_div[c]) {
      bool ok;
      switch (P->cons_op[c]) {
        case 0: ok = e < (T)0; break;
        case 1: ok = e <= (T)0; break;
        case 2: ok = e > (T)0; break;
        case 3: ok = e >= (T)0; break;
        default: ok = e == (T)0; break;
      }
      if (!ok) return KCG_PT_ASSUMPTION_VIOLATED;
    } else {
      const T D = wide<T>(P->expr_den[P->cons_expr[c]]);
      if (e % D != (T)0) return KCG_PT_NONINTEGRAL;
      const T v = e / D;
      if (kcg_posmod<T>(v, wide<T>(P->cons_mod[c])) != wide<T>(P->cons_rem[c]))
        return KCG_PT_ASSUMPTION_VIOLATED;
    }
  }
  for (int j = 0; j < P->n_keys; ++j) {
    const T e = expr[P->key_expr[j]];
    const T D = wide<T>(P->expr_den[P->key_expr[j]]);
    if (e % D != (T)0) return KCG_PT_NONINTEGRAL;
    cnt[j] = e / D;
  }
  return KCG_PT_OK;
}

template <class T>
__device__ __forceinline__ int interp_point(const KcgDevProg* __restrict__ P,
                                            const kcg_i64* p,
                                            const InterpEvalArgs& a, kcg_i64 i,
                                            double& s) {
  T c[KCG_MAX_KEYS];
  int st = interp_body<T>(P, p, c);
  if (st != KCG_PT_OK) return st;
  for (int j = 0; j < P->n_keys; ++j) s = kcg_accum(s, a.alpha[j], c[j], a.simulate);
  if (a.clo) {
    for (int j = 0; j < P->n_keys; ++j) {
      a.clo[(kcg_i64)j * a.n + i] = (kcg_i64)c[j];
      if (a.chi)
        a.chi[(kcg_i64)j * a.n + i] = kcg_hi64(c[j]);
      else if (!kcg_fits_i64(c[j]))
        st = KCG_PT_COUNT_WIDE;
    }
  }
  return st;
}

__global__ void __launch_bounds__(128)
    kcg_interp_eval(const KcgDevProg* __restrict__ P, const KcgDevProg* __restrict__ A,
                    const __grid_constant__ InterpEvalArgs a) {
  const kcg_i64 stride = (kcg_i64)gridDim.x * blockDim.x;
  const int np = P->n_params;
  for (kcg_i64 i = (kcg_i64)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {
    kcg_i64 p[KCG_MAX_PARAMS];
    bool neg = false, fast = P->b64 >= 0, wide_ok = P->b128 >= 0;
    for (int j = 0; j < np; ++j) {
      p[j] = a.p[j][i];
      neg |= p[j] < 0;
      fast &= p[j] <= P->b64;
      wide_ok &= p[j] <= P->b128;
    }
    double s = 0.0;
    int st;
    if (neg)
      st = KCG_PT_ASSUMPTION_VIOLATED;
    else if (fast)
      st = interp_point<kcg_i64>(P, p, a, i, s);
    else if (wide_ok)
      st = interp_point<kcg_i128>(P, p, a, i, s);
    else {
      // counts beyond 128 bits: admissibility still decides first
      st = KCG_PT_OVERFLOW;
      if (A) {
        bool ok = A->b128 >= 0;
        for (int j = 0; j < np; ++j) ok &= p[j] <= A->b128;
        kcg_i128 none[1];
        if (ok) {
          const int a0 = interp_body<kcg_i128>(A, p, none);
          if (a0 != KCG_PT_OK) st = a0;
        }
      }
    }
    if (a.pred) a.pred[i] = (st == KCG_PT_OK || st == KCG_PT_COUNT_WIDE) ? s : kcg_nan();
    if (a.status) a.status[i] = (uint8_t)st;
  }
}

// ---------------------------------------------------------------------------
// materialised Gram

constexpr int kGramRows = 32;
constexpr int kGramMaxF = 160;  // the 149-key schema fits (5 x 32 residual lanes, <= 820 tiles)

struct GramGeom {
  int FP, nb, ntiles, slice_threads, S;
};

// one 4x4 tile of the upper triangle per thread; S row-slices of the tile
// set when the triangle is small (256 threads, F <= 64), one slice of up to
// 1,024 threads for wide designs (F <= 176)
__host__ __device__ inline GramGeom gram_geom(int F, int threads) {
  GramGeom g;
  g.FP = (F + 3) & ~3;
  g.nb = g.FP / 4;
  g.ntiles = g.nb * (g.nb + 1) / 2;
  g.slice_threads = ((g.ntiles + 31) / 32) * 32;
  g.S = threads / g.slice_threads;
  if (g.S < 1) g.S = 1;
  return g;
}

// CUDA-core Gram for strided / unaligned X and for wide designs (F > 48):
// the upper triangle in 4x4 register tiles, rows staged through shared
// memory; column sums and maxima by the first FP threads from the staged rows
template <int MAXT>
__global__ void __launch_bounds__(MAXT)
    kcg_gram_x(const double* __restrict__ X, kcg_i64 n, int F, kcg_i64 ld,
               kcg_i64 rows_per_cta, double* __restrict__ G,
               double* __restrict__ xt1, double* __restrict__ cmax) {
  extern __shared__ double sm[];
  const GramGeom g = gram_geom(F, blockDim.x);
  double* tile = sm;                           // [kGramRows][FP]
  double* red = sm + kGramRows * g.FP;         // [ntiles][16]

  const int tid = threadIdx.x;
  const int slice = tid / g.slice_threads;
  const int t = tid % g.slice_threads;
  const bool active = slice < g.S && t < g.ntiles;
  int bi = 0, bj = 0;
  {
    int rem = active ? t : 0;
    while (bi < g.nb && rem >= g.nb - bi) {
      rem -= g.nb - bi;
      ++bi;
    }
    bj = bi + rem;
  }
  for (int k = tid; k < g.ntiles * 16; k += blockDim.x) red[k] = 0.0;

  double acc[4][4] = {};
  double cs = 0.0, cm = 0.0;  // column tid (< F): sum and max |x|
  const kcg_i64 r0 = (kcg_i64)blockIdx.x * rows_per_cta;
  kcg_i64 r1 = r0 + rows_per_cta;
  if (r1 > n) r1 = n;
  const int warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
  for (kcg_i64 base = r0; base < r1; base += kGramRows) {
    const int rows = (int)((r1 - base) < kGramRows ? (r1 - base) : kGramRows);
    __syncthreads();
    for (int r = warp; r < kGramRows; r += nwarps) {
      const double* src = X + (base + r) * ld;
      for (int c = lane; c < g.FP; c += 32)
        tile[r * g.FP + c] = (r < rows && c < F) ? __ldcs(src + c) : 0.0;
    }
    __syncthreads();
    if (tid < F)
      for (int r = 0; r < rows; ++r) {
        const double v = tile[r * g.FP + tid];
        cs += v;
        cm = fmax(cm, fabs(v));
      }
    if (active) {
      for (int r = slice; r < rows; r += g.S) {
        const double* row = tile + r * g.FP;
        const double2 a01 = *reinterpret_cast<const double2*>(row + 4 * bi);
        const double2 a23 = *reinterpret_cast<const double2*>(row + 4 * bi + 2);
        const double2 b01 = *reinterpret_cast<const double2*>(row + 4 * bj);
        const double2 b23 = *reinterpret_cast<const double2*>(row + 4 * bj + 2);
        const double av[4] = {a01.x, a01.y, a23.x, a23.y};
        const double bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) acc[x][y] = fma(av[x], bv[y], acc[x][y]);
      }
    }
  }
  __syncthreads();
  if (active)
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) atomicAdd(red + t * 16 + x * 4 + y, acc[x][y]);
  if (tid < F) {
    atomicAdd(xt1 + tid, cs);
    atomicMax(reinterpret_cast<unsigned long long*>(cmax + tid), (unsigned long long)__double_as_longlong(cm));
  }
  __syncthreads();
  if (slice == 0 && t < g.ntiles) {
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        const int r = 4 * bi + x, c = 4 * bj + y;
        if (r >= F || c >= F) continue;
        const double v = red[t * 16 + x * 4 + y];
        atomicAdd(G + r * F + c, v);
        if (bi != bj) atomicAdd(G + c * F + r, v);
      }
  }
}

// ---------------------------------------------------------------------------
// Gram on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64) fed by a TMA ring
//
// G = X^T X is a GEMM with M = N = F (<= 48 here) and K = rows. For a 4-row
// k-step, lane (gid = lane/4, tig = lane%4) loads v_b = X[k0+tig][8b+gid]
// for every 8-column block b; that one register is simultaneously the A
// fragment (row-major 8x4, A[i][k] = X[k][8I+i]) and the B fragment
// (col-major 4x8, B[k][j] = X[k][8J+j]) of the m8n8k4 DMMA, so each k-step
// costs NB shared loads and NB(NB+1)/2 tensor instructions for the upper
// block triangle. Rows stream through a 4-stage cp.async.bulk ring.

constexpr int kDmmaRows = 64;

// |x| as its bit pattern with the sign cleared on the integer pipe (a plain
// `& 0x7fff...` is turned into DADD |x|, which occupies the FP64 pipe the
// DMMAs run on)
__device__ __forceinline__ unsigned long long abs_bits(double x) {
  unsigned lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "d"(x));
  asm volatile("and.b32 %0, %0, 0x7fffffff;" : "+r"(hi));
  return ((unsigned long long)hi << 32) | lo;
}

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// stage hand-back: kcg_ring_release (kcg_device.cuh)
// R: rows per tile (64 * m): narrow designs take taller tiles so every
// stage is still a multi-KB bulk copy
template <int NB, int R, int CT>
__global__ void __launch_bounds__(256, CT)
    kcg_gram_dmma(const double* __restrict__ X, kcg_i64 n, int F, int stages,
                  double* __restrict__ G, double* __restrict__ xt1, double* __restrict__ cmax) {
  constexpr int NT = NB * (NB + 1) / 2;
  constexpr int FP = NB * 8;
  extern __shared__ __align__(128) unsigned char kcg_smem[];
  double* buf = reinterpret_cast<double*>(kcg_smem);
  constexpr int RW = R / 8;  // rows per warp per tile
  const int stage_d = R * F;
  double* red = buf + stages * stage_d;  // [FP][FP] + s1[FP] + mx[FP]
  double* red_s1 = red + FP * FP;
  double* red_mx = red_s1 + FP;
  __shared__ __align__(8) unsigned long long full[8];
  __shared__ unsigned reads[8];  // warps done with stage s (the last one refills it)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  for (int k = tid; k < FP * FP + 2 * FP; k += blockDim.x) red[k] = 0.0;
  if (tid < 8) reads[tid] = 0;
  const unsigned fb = (unsigned)__cvta_generic_to_shared(full);
  const unsigned bb = (unsigned)__cvta_generic_to_shared(buf);
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(fb + 8 * s));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const kcg_i64 ntiles = n / R;
  const unsigned bytes = (unsigned)(stage_d * 8);
  auto issue = [&](int s, kcg_i64 tile) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb + 8 * s), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     bb + (unsigned)(s * stage_d * 8)),
                 "l"(X + tile * stage_d), "r"(bytes), "r"(fb + 8 * s)
                 : "memory");
  };
  if (tid == 0)
    for (int s = 0; s < stages; ++s) {
      const kcg_i64 t = blockIdx.x + (kcg_i64)s * gridDim.x;
      if (t < ntiles) issue(s, t);
    }
  double acc[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
  // column maxima on the integer pipe: |x| compared as its bit pattern
  // (monotone for non-negative doubles), keeping the FP64/DMMA pipe -- which
  // ncu shows shared by DSETP and DMMA -- for the tensor work
  double s1[NB];
  unsigned long long mx[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    s1[b] = 0.0;
    mx[b] = 0ull;
  }

  auto kstep_regs = [&](const double* v) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      s1[b] += v[b];
      {
        const unsigned long long bits = abs_bits(v[b]);
        mx[b] = bits > mx[b] ? bits : mx[b];
      }
    }
    int t = 0;
#pragma unroll
    for (int I = 0; I < NB; ++I)
#pragma unroll
      for (int J = I; J < NB; ++J, ++t) dmma_8x8x4(acc[t][0], acc[t][1], v[I], v[J]);
  };
  auto kstep = [&](const double* rowp, bool valid) {
    double v[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int col = 8 * b + gid;
      v[b] = (valid && col < F) ? rowp[col] : 0.0;
      s1[b] += v[b];
      {
        const unsigned long long bits = abs_bits(v[b]);
        mx[b] = bits > mx[b] ? bits : mx[b];
      }
    }
    int t = 0;
#pragma unroll
    for (int I = 0; I < NB; ++I)
#pragma unroll
      for (int J = I; J < NB; ++J, ++t) dmma_8x8x4(acc[t][0], acc[t][1], v[I], v[J]);
  };

  for (kcg_i64 k = 0;; ++k) {
    const kcg_i64 tile = blockIdx.x + k * gridDim.x;
    if (tile >= ntiles) break;
    const int s = (int)(k % stages);
    const unsigned parity = (unsigned)((k / stages) & 1);
    unsigned done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(fb + 8 * s), "r"(parity)
                   : "memory");
    const double* st = buf + s * stage_d;
    // 8 warps x RW/4 k-steps x 4 rows = R rows; the last k-step's fragments
    // are loaded to registers, then the stage is released: the last warp to
    // finish reading it issues the refill, so warps drift freely
    double v[NB];
#pragma unroll
    for (int ks = 0; ks < RW / 4 - 1; ++ks) {
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int col = 8 * b + gid;
        v[b] = col < F ? st[(warp * RW + 4 * ks + tig) * F + col] : 0.0;
      }
      kstep_regs(v);
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int col = 8 * b + gid;
      v[b] = col < F ? st[(warp * RW + RW - 4 + tig) * F + col] : 0.0;
    }
    __syncwarp();
    if (lane == 0 && kcg_ring_release(&reads[s], blockDim.x / 32)) {
      const kcg_i64 nt = blockIdx.x + (k + stages) * gridDim.x;
      if (nt < ntiles) issue(s, nt);
    }
    kstep_regs(v);
  }
  // tail rows straight from global (block 0 only)
  if (blockIdx.x == 0)
    for (kcg_i64 r0 = ntiles * R + warp * 4; r0 < n; r0 += 32) {
      const kcg_i64 r = r0 + tig;
      kstep(X + (r < n ? r : 0) * F, r < n);
    }
  // reduce warps through shared memory, then one atomic per entry
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    double a = s1[b];
    unsigned long long m = mx[b];
    a += __shfl_xor_sync(0xffffffffu, a, 1);
    a += __shfl_xor_sync(0xffffffffu, a, 2);
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      const unsigned long long y = __shfl_xor_sync(0xffffffffu, m, o);
      m = y > m ? y : m;
    }
    if (tig == 0) {
      atomicAdd(red_s1 + 8 * b + gid, a);
      atomicMax(reinterpret_cast<unsigned long long*>(red_mx + 8 * b + gid), m);
    }
  }
  {
    int t = 0;
#pragma unroll
    for (int I = 0; I < NB; ++I)
#pragma unroll
      for (int J = I; J < NB; ++J, ++t) {
        atomicAdd(red + (8 * I + gid) * FP + 8 * J + 2 * tig, acc[t][0]);
        atomicAdd(red + (8 * I + gid) * FP + 8 * J + 2 * tig + 1, acc[t][1]);
      }
  }
  __syncthreads();
  for (int e = tid; e < FP * FP; e += blockDim.x) {
    const int r = e / FP, c = e % FP;
    if (r >= F || c >= F || (c / 8) < (r / 8)) continue;  // upper block triangle holds the data
    const double v = red[e];
    atomicAdd(G + r * F + c, v);
    if (c / 8 != r / 8) atomicAdd(G + c * F + r, v);
  }
  for (int c = tid; c < F; c += blockDim.x) {
    atomicAdd(xt1 + c, red_s1[c]);
    atomicMax(reinterpret_cast<unsigned long long*>(cmax + c),
              (unsigned long long)__double_as_longlong(red_mx[c]));
  }
}

template <int NB, int CT, int R = (NB <= 2 ? 256 : (NB == 3 ? 128 : 64))>
void launch_gram_dmma(const double* X, size_t n, int F, double* G, double* xt1, double* colmax,
                      cudaStream_t stream) {
  const size_t red_b = (size_t)(NB * 8 * NB * 8 + 2 * NB * 8) * sizeof(double);
  int stages;
  if (CT == 1) {
    // one CTA per SM (the 8 x 8 block triangle of NB >= 7 needs > 128
    // registers per thread): a deep ring within ~200 KB
    stages = (int)((200 * 1024 - red_b) / ((size_t)R * F * 8));
    stages = stages < 2 ? 2 : (stages > 8 ? 8 : stages);
  } else {
    // ring: up to 4 stages within ~100 KB so that two CTAs share an SM
    stages = (int)((100 * 1024) / ((size_t)R * F * 8));
    stages = stages < 2 ? 2 : (stages > 4 ? 4 : stages);
    if (NB >= 5 && R == 64) stages = F <= 40 ? 4 : 3;
  }
  const size_t smem = (size_t)stages * R * F * sizeof(double) + red_b;
  // the opt-in size grows with F within one NB (per device, process-wide)
  static std::mutex mu;
  static size_t attr_smem[64] = {};  // per device, this <NB, CT> instantiation
  int dev = 0;
  check(cudaGetDevice(&dev), "cudaGetDevice");
  {
    std::lock_guard<std::mutex> lk(mu);
    size_t& cur = attr_smem[dev & 63];
    if (smem + 4096 > cur) {
      check(cudaFuncSetAttribute(kcg_gram_dmma<NB, R, CT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem + 4096),
            "cudaFuncSetAttribute");
      cur = smem + 4096;
    }
  }
  const kcg_i64 tiles = (kcg_i64)n / R;
  kcg_i64 grid = (kcg_i64)num_sms() * CT;
  if (grid > tiles) grid = tiles > 0 ? tiles : 1;
  kcg_gram_dmma<NB, R, CT><<<(unsigned)grid, 256, smem, stream>>>(X, (kcg_i64)n, F, stages, G, xt1, colmax);
  check(cudaGetLastError(), "kcg_gram_dmma launch");
}

// ---------------------------------------------------------------------------
// Hybrid DMMA + DFMA Gram for NB = 4, 5 (even F in (8 (NB - 1), 8 NB])
//
// On B200 the FP64 tensor instruction (DMMA m8n8k4) and DFMA share one FP64
// datapath at the same flop rate: a warp mix of both runs in the sum of their
// separate times (profiles/dmma_dfma_probe.cu, r02_dmma_dfma.json: 37.1 and
// 37.0 TFLOP/s alone, mixed / sum = 1.05). So the block-diagonal 8 x 8 tiles,
// where a DMMA spends 64 products on 36 distinct entries, are cheaper as
// DFMAs of their upper triangles: at F = 40 a row costs 10 x 64 + 5 x 36 =
// 820 FP64 multiply-adds instead of 15 x 64 = 960.
//
// Every warp issues both kinds, in the proportion of the work: a first
// version with DFMA-only warps (one per SM sub-partition) ran at 8.1 ms
// instead of 6.2 -- the scheduler hands the shared pipe out per instruction,
// so the DFMA warp got one 2-cycle DFMA per 16-cycle DMMA and starved
// (ncu: DMMA active 42%, the DMMA warps spinning on the stage barrier).
// Measured at 1e8 x 40: 5.95 ms against 6.19 for kcg_gram_dmma
// (interleaved runs) with 96-row warp-group tiles (48 rows: 6.15 ms) --
// most of the 15% fewer FP64 operations are given back because 36 DFMA
// accumulators hold a warp at 250 registers, so only two warps share a
// sub-partition and tile-boundary latency (barrier wait, shared loads, the
// stage release) is exposed. Default for NB = 5 (at F = 32 it is slower:
// 4.72 vs 4.53 ms).
//
// 256 threads, one CTA per SM (up to 255 registers: 20 DMMA accumulators,
// 36 DFMA accumulators), two groups of 4 warps taking alternate R-row tiles.
// Each warp owns RW = R / 4 rows of its group's tile: the DMMA k-steps of the
// NB (NB - 1) / 2 off-diagonal tiles plus X^T 1 and the column maxima over
// those rows (kcg_gram_dmma's k-step without the diagonal tiles), and the
// diagonal blocks of the same rows on DFMA: lane l < NB J (J = 32 / NB) owns
// block l % NB for rows j + J u (j = l / NB), loads the block's 8 values of a
// row as four 16-byte shared loads and accumulates its 36 products. The
// 16-byte loads are staggered per lane pair (pair s of the block is loaded
// at step (s - c) mod 4, c = (l / 2) % 4) so the 8 lanes of a quarter-warp
// hit 8 distinct bank groups at F = 40.
template <int NB, int R, bool FULL>
__global__ void __launch_bounds__(256, 1)
    kcg_gram_hybrid(const double* __restrict__ X, kcg_i64 n, int F_, int stages,
                    double* __restrict__ G, double* __restrict__ xt1, double* __restrict__ cmax) {
  constexpr int NW = 8;
  // FULL: F == 8 NB, a compile-time row pitch and no column predicates
  const int F = FULL ? NB * 8 : F_;
  constexpr int J = 32 / NB;
  constexpr int NOFF = NB * (NB - 1) / 2;
  constexpr int FP = NB * 8;
  constexpr int RW = R / 4;  // rows per warp per tile (a tile belongs to one group of 4 warps)
  constexpr int TD = RW / J;  // rows per DFMA lane per tile
  static_assert(RW % 4 == 0 && RW % J == 0, "tile shape");
  extern __shared__ __align__(128) unsigned char kcg_smem[];
  double* buf = reinterpret_cast<double*>(kcg_smem);
  const int stage_d = R * F;
  double* red = buf + stages * stage_d;  // [FP][FP] + s1[FP] + mx[FP]
  double* red_s1 = red + FP * FP;
  double* red_mx = red_s1 + FP;
  __shared__ __align__(8) unsigned long long full[16];
  __shared__ unsigned reads[16];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  for (int k = tid; k < FP * FP + 2 * FP; k += blockDim.x) red[k] = 0.0;
  if (tid < 16) reads[tid] = 0;
  const unsigned fb = (unsigned)__cvta_generic_to_shared(full);
  const unsigned bb = (unsigned)__cvta_generic_to_shared(buf);
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(fb + 8 * s));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const kcg_i64 ntiles = n / R;
  const unsigned bytes = (unsigned)(stage_d * 8);
  auto issue = [&](int s, kcg_i64 tile) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb + 8 * s), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     bb + (unsigned)(s * stage_d * 8)),
                 "l"(X + tile * stage_d), "r"(bytes), "r"(fb + 8 * s)
                 : "memory");
  };
  if (tid == 0)
    for (int s = 0; s < stages; ++s) {
      const kcg_i64 t = blockIdx.x + (kcg_i64)s * gridDim.x;
      if (t < ntiles) issue(s, t);
    }

  // DMMA part: off-diagonal tiles, X^T 1, column maxima
  double acc[NOFF][2];
#pragma unroll
  for (int t = 0; t < NOFF; ++t) acc[t][0] = acc[t][1] = 0.0;
  double s1[NB];
  unsigned long long mx[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    s1[b] = 0.0;
    mx[b] = 0ull;
  }
  auto kstep = [&](const double* v) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      s1[b] += v[b];
      const unsigned long long bits = abs_bits(v[b]);
      mx[b] = bits > mx[b] ? bits : mx[b];
    }
    int t = 0;
#pragma unroll
    for (int I = 0; I < NB; ++I)
#pragma unroll
      for (int Jb = I + 1; Jb < NB; ++Jb, ++t) dmma_8x8x4(acc[t][0], acc[t][1], v[I], v[Jb]);
  };
  // DFMA part: one diagonal block per lane, 36 accumulators
  const bool act = lane < NB * J;
  const int db = lane % NB, dj = act ? lane / NB : 0;  // idle lanes re-read row 0: no predicate
  const int dc = (lane >> 1) & 3;
  int off[4];
  bool ok[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    off[s] = 8 * db + 2 * ((s + dc) & 3);
    ok[s] = FULL || off[s] < F;
  }
  double a[36];
#pragma unroll
  for (int k = 0; k < 36; ++k) a[k] = 0.0;
  auto diag = [&](const double* row) {
    double w[8];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      // lanes >= NB J read real rows too; their accumulators are never
      // written out
      const double2 x = ok[s] ? *reinterpret_cast<const double2*>(row + off[s]) : make_double2(0.0, 0.0);
      w[2 * s] = x.x;
      w[2 * s + 1] = x.y;
    }
    int k = 0;
#pragma unroll
    for (int p = 0; p < 8; ++p)
#pragma unroll
      for (int q = p; q < 8; ++q, ++k) a[k] = fma(w[p], w[q], a[k]);
  };

  // warp group g = warp / 4 (one warp per SM sub-partition) takes the tiles
  // k = g (mod 2): the two warps sharing a sub-partition work on different
  // tiles, so one's barrier wait / load / release phase overlaps the
  // other's FP64 work. `stages` is even, so stage s = k mod stages always
  // belongs to the same group; s and the parity advance incrementally.
  const int grp = warp >> 2, wg = warp & 3;
  int s = grp;
  unsigned parity = 0;
  for (kcg_i64 k = grp;; k += 2) {
    const kcg_i64 tile = blockIdx.x + k * gridDim.x;
    if (tile >= ntiles) break;
    unsigned done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(fb + 8 * s), "r"(parity)
                   : "memory");
    const double* st = buf + s * stage_d + wg * RW * F;
#pragma unroll
    for (int u = 0; u < TD; ++u) diag(st + (dj + J * u) * F);
#pragma unroll
    for (int ks = 0; ks < RW / 4; ++ks) {
      double v[NB];
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int col = 8 * b + gid;
        v[b] = (FULL || col < F) ? st[(4 * ks + tig) * F + col] : 0.0;
      }
      kstep(v);
    }
    // the last of the group's 4 warps to finish reading stage s refills it
    // with tile k + stages (same group)
    __syncwarp();
    if (lane == 0 && kcg_ring_release(&reads[s], 4)) {
      const kcg_i64 nt = blockIdx.x + (k + stages) * gridDim.x;
      if (nt < ntiles) issue(s, nt);
    }
    s += 2;
    if (s >= stages) {
      s -= stages;
      parity ^= 1u;
    }
  }
  // tail rows straight from global (block 0 only)
  if (blockIdx.x == 0) {
    for (kcg_i64 r0 = ntiles * R + warp * 4; r0 < n; r0 += 4 * NW) {
      const kcg_i64 r = r0 + tig;
      double v[NB];
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int col = 8 * b + gid;
        v[b] = (r < n && col < F) ? X[r * F + col] : 0.0;
      }
      kstep(v);
    }
    for (kcg_i64 r = ntiles * R + warp * J + dj; r < n; r += NW * J) diag(X + r * F);
  }
  // reduce through shared memory, then one atomic per entry
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    double x = s1[b];
    unsigned long long m = mx[b];
    x += __shfl_xor_sync(0xffffffffu, x, 1);
    x += __shfl_xor_sync(0xffffffffu, x, 2);
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      const unsigned long long y = __shfl_xor_sync(0xffffffffu, m, o);
      m = y > m ? y : m;
    }
    if (tig == 0) {
      atomicAdd(red_s1 + 8 * b + gid, x);
      atomicMax(reinterpret_cast<unsigned long long*>(red_mx + 8 * b + gid), m);
    }
  }
  {
    int t = 0;
#pragma unroll
    for (int I = 0; I < NB; ++I)
#pragma unroll
      for (int Jb = I + 1; Jb < NB; ++Jb, ++t) {
        atomicAdd(red + (8 * I + gid) * FP + 8 * Jb + 2 * tig, acc[t][0]);
        atomicAdd(red + (8 * I + gid) * FP + 8 * Jb + 2 * tig + 1, acc[t][1]);
      }
  }
  if (act) {
    int k = 0;
#pragma unroll
    for (int p = 0; p < 8; ++p)
#pragma unroll
      for (int q = p; q < 8; ++q, ++k) {
        const int fp = 2 * (((p >> 1) + dc) & 3) + (p & 1), fq = 2 * (((q >> 1) + dc) & 3) + (q & 1);
        const int lo = fp < fq ? fp : fq, hi = fp < fq ? fq : fp;
        atomicAdd(red + (8 * db + lo) * FP + 8 * db + hi, a[k]);
      }
  }
  __syncthreads();
  for (int e = tid; e < FP * FP; e += blockDim.x) {
    const int r = e / FP, c = e % FP;
    if (r >= F || c >= F || (c / 8) < (r / 8) || ((c / 8) == (r / 8) && c < r)) continue;
    const double v = red[e];
    atomicAdd(G + r * F + c, v);
    if (c != r) atomicAdd(G + c * F + r, v);
  }
  for (int c = tid; c < F; c += blockDim.x) {
    atomicAdd(xt1 + c, red_s1[c]);
    atomicMax(reinterpret_cast<unsigned long long*>(cmax + c), (unsigned long long)__double_as_longlong(red_mx[c]));
  }
}

template <int NB, int R>
void launch_gram_hybrid(const double* X, size_t n, int F, double* G, double* xt1, double* colmax,
                        cudaStream_t stream) {
  const size_t red_b = (size_t)(NB * 8 * NB * 8 + 2 * NB * 8) * sizeof(double);
  static const int ring_kb = std::getenv("KCG_GRAM_HYBRID_RING_KB") ? std::atoi(std::getenv("KCG_GRAM_HYBRID_RING_KB")) : 200;
  int stages = (int)(((size_t)ring_kb * 1024 - red_b) / ((size_t)R * F * 8));
  stages = stages < 2 ? 2 : (stages > 16 ? 16 : stages);
  stages &= ~1;  // even: a stage always holds the tiles of one warp group
  const size_t smem = (size_t)stages * R * F * sizeof(double) + red_b;
  static std::mutex mu;
  static size_t attr_smem[64] = {};
  int dev = 0;
  check(cudaGetDevice(&dev), "cudaGetDevice");
  {
    std::lock_guard<std::mutex> lk(mu);
    size_t& cur = attr_smem[dev & 63];
    if (smem + 4096 > cur) {
      check(cudaFuncSetAttribute(kcg_gram_hybrid<NB, R, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem + 4096),
            "cudaFuncSetAttribute");
      check(cudaFuncSetAttribute(kcg_gram_hybrid<NB, R, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem + 4096),
            "cudaFuncSetAttribute");
      cur = smem + 4096;
    }
  }
  const kcg_i64 tiles = (kcg_i64)n / R;
  kcg_i64 grid = (kcg_i64)num_sms();
  if (grid > tiles) grid = tiles > 0 ? tiles : 1;
  if (F == NB * 8)
    kcg_gram_hybrid<NB, R, true><<<(unsigned)grid, 256, smem, stream>>>(X, (kcg_i64)n, F, stages, G, xt1, colmax);
  else
    kcg_gram_hybrid<NB, R, false><<<(unsigned)grid, 256, smem, stream>>>(X, (kcg_i64)n, F, stages, G, xt1, colmax);
  check(cudaGetLastError(), "kcg_gram_hybrid launch");
}

// ---------------------------------------------------------------------------
// Row-per-lane DFMA Gram for narrow designs (F <= 13, 17..22)
//
// The DMMA kernels pad F to 8-column blocks: F = 9..12 pays the 3 DMMAs of
// F = 16 per 4 rows and F = 17..20 the 6 of F = 24, so both plateau on the
// FP64 pipe (1.49 and 2.7 ms for 1e8 rows) where HBM allows 1.0-1.3 and
// 1.9-2.2 ms. With DMMA and DFMA at the same rate, DFMAs over exactly the
// F(F+1)/2 distinct entries cost F(F+3)/2 FP64 lane operations per row with
// Xt1 (54 at F = 9), well under the 8 F bytes' HBM time. Each lane walks
// whole rows: it loads a row's F values from the TMA-staged tile and
// accumulates its share of the upper triangle in registers. G warps split
// the triangle of the same rows (part = warp % G, a warp-uniform switch to
// straight-line code per part): the entries [part C, part C + C) in
// row-major triangle order, C = ceil(E / G), and the Xt1 / column-maximum
// work of the columns c = part (mod G). Warp sums go through shuffles to
// shared memory, one global atomic per entry per CTA.
__host__ __device__ constexpr int tri_row(int e, int F) {
  int p = 0;
  while (e >= F - p) {
    e -= F - p;
    ++p;
  }
  return p;
}
__host__ __device__ constexpr int tri_col(int e, int F) {
  int p = 0;
  while (e >= F - p) {
    e -= F - p;
    ++p;
  }
  return p + e;
}

// Row pitches of F = 2 (mod 4) doubles put lanes 8 apart on the same banks
// (F = 4 (mod 8): lanes 4 apart, 4-way): such a lane reads its row rotated
// by rot = 0..1 (0..3) columns, register slot c holding column
// (c + rot) mod F -- the slot pairs still cover every column pair once, and
// the flush maps them back.
template <int F>
struct DfmaRot {
  static constexpr int RB = (F % 8 == 4) ? 2 : ((F % 4 == 2) ? 3 : -1);  // lane bit(s) selecting rot
  static constexpr int MAXR = RB == 2 ? 3 : (RB == 3 ? 1 : 0);
  // lanes sharing a rotation: xor masks over the other lane bits
  static constexpr unsigned KEEP = RB == 2 ? 0xcu : (RB == 3 ? 0x8u : 0x0u);
  __device__ static int rot(int lane) { return RB < 0 ? 0 : (lane >> RB) & MAXR; }
};

template <int F, int G, int PART>
struct DfmaPart {
  static constexpr int E = F * (F + 1) / 2;
  static constexpr int C = (E + G - 1) / G;
  static constexpr int E0 = PART * C;
  static constexpr int NE = (E - E0) < C ? (E - E0) : C;  // entries of this part
  static constexpr int NC = (F - PART + G - 1) / G;        // slots c = PART (mod G)
  using Rot = DfmaRot<F>;
  double acc[C];
  double s1[NC];
  unsigned long long mx[NC];
  int rot;
  __device__ __forceinline__ void zero(int lane) {
    rot = Rot::rot(lane);
#pragma unroll
    for (int k = 0; k < C; ++k) acc[k] = 0.0;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      s1[k] = 0.0;
      mx[k] = 0ull;
    }
  }
  // entry K of this part: the slot indices are constant expressions, so
  // v[] stays in registers
  template <int K>
  __device__ __forceinline__ void entry(const double* v) {
    constexpr int p = tri_row(E0 + K, F), q = tri_col(E0 + K, F);
    acc[K] = fma(v[p], v[q], acc[K]);
  }
  template <int... K>
  __device__ __forceinline__ void entries(const double* v, std::integer_sequence<int, K...>) {
    (entry<K>(v), ...);
  }
  __device__ __forceinline__ void row(const double* __restrict__ r) {
    double v[F];
#pragma unroll
    for (int c = 0; c < F; ++c) {  // unused slots are dead code
      int col = c + rot;
      if (c + Rot::MAXR >= F && col >= F) col -= F;
      v[c] = r[col];
    }
    entries(v, std::make_integer_sequence<int, NE>{});
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const double x = v[PART + G * k];
      s1[k] += x;
      const unsigned long long bits = abs_bits(x);
      mx[k] = bits > mx[k] ? bits : mx[k];
    }
  }
  __device__ __forceinline__ int col_of(int slot) const { return slot + rot >= F ? slot + rot - F : slot + rot; }
  __device__ static double lanes_sum(double x) {
#pragma unroll
    for (int o = 1; o <= 16; o <<= 1)
      if (!(o & Rot::KEEP)) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
  }
  template <int K>
  __device__ __forceinline__ void flush_entry(double* red, bool writer) {
    constexpr int p = tri_row(E0 + K, F), q = tri_col(E0 + K, F);
    const double x = lanes_sum(acc[K]);
    if (writer) {
      const int a = col_of(p), b = col_of(q);
      const int lo = a < b ? a : b, hi = a < b ? b : a;
      atomicAdd(red + lo * F - lo * (lo - 1) / 2 + (hi - lo), x);
    }
  }
  template <int... K>
  __device__ __forceinline__ void flush_entries(double* red, bool writer, std::integer_sequence<int, K...>) {
    (flush_entry<K>(red, writer), ...);
  }
  // totals of the lanes sharing a rotation into shared memory: red[E]
  // (row-major upper triangle), red_s1[F], red_mx[F]
  __device__ __forceinline__ void flush(double* red, double* red_s1, double* red_mx, int lane) {
    const bool writer = (lane & ~Rot::KEEP & 31u) == 0;
    flush_entries(red, writer, std::make_integer_sequence<int, NE>{});
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const double x = lanes_sum(s1[k]);
      unsigned long long m = mx[k];
#pragma unroll
      for (int o = 1; o <= 16; o <<= 1)
        if (!(o & Rot::KEEP)) {
          const unsigned long long y = __shfl_xor_sync(0xffffffffu, m, o);
          m = y > m ? y : m;
        }
      if (writer) {
        const int c = col_of(PART + G * k);
        atomicAdd(red_s1 + c, x);
        atomicMax(reinterpret_cast<unsigned long long*>(red_mx + c), m);
      }
    }
  }
};

// 256 threads = 8 warps = (8 / G) row sets x G parts; a stage holds
// R = 32 (8 / G) M rows, row set w / G takes rows 32 (w / G) + lane + 256 / G m
template <int F, int G, int M, int PART>
__device__ __forceinline__ void gram_dfma_part(const double* __restrict__ X, kcg_i64 n, int stages,
                                               double* __restrict__ buf, unsigned fb, unsigned bb,
                                               unsigned* reads, double* red, double* red_s1, double* red_mx) {
  constexpr int RS = 8 / G;          // row sets
  constexpr int R = 32 * RS * M;     // rows per stage
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int set = warp / G;
  const int stage_d = R * F;
  const unsigned bytes = (unsigned)(stage_d * 8);
  const kcg_i64 ntiles = n / R;
  DfmaPart<F, G, PART> P;
  P.zero(lane);
  int s = 0;
  unsigned parity = 0;
  for (kcg_i64 k = 0;; ++k) {
    const kcg_i64 tile = blockIdx.x + k * gridDim.x;
    if (tile >= ntiles) break;
    unsigned done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(fb + 8 * s), "r"(parity)
                   : "memory");
    const double* st = buf + s * stage_d;
#pragma unroll
    for (int m = 0; m < M; ++m) P.row(st + (32 * set + lane + 32 * RS * m) * F);
    __syncwarp();
    if (lane == 0 && kcg_ring_release(&reads[s], 8)) {
      {
        const kcg_i64 nt = blockIdx.x + (k + stages) * gridDim.x;
        if (nt < ntiles) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb + 8 * s), "r"(bytes)
                       : "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  bb + (unsigned)(s * stage_d * 8)),
              "l"(X + nt * stage_d), "r"(bytes), "r"(fb + 8 * s)
              : "memory");
        }
      }
    }
    if (++s == stages) {
      s = 0;
      parity ^= 1u;
    }
  }
  // tail rows straight from global (block 0 only)
  if (blockIdx.x == 0)
    for (kcg_i64 r = ntiles * R + 32 * set + lane; r < n; r += 32 * RS) P.row(X + r * F);
  P.flush(red, red_s1, red_mx, lane);
}

template <int F, int G, int M>
__global__ void __launch_bounds__(256, 1)
    kcg_gram_dfma(const double* __restrict__ X, kcg_i64 n, int stages, double* __restrict__ Gm,
                  double* __restrict__ xt1, double* __restrict__ cmax) {
  constexpr int E = F * (F + 1) / 2;
  constexpr int R = 32 * (8 / G) * M;
  extern __shared__ __align__(128) unsigned char kcg_smem[];
  double* buf = reinterpret_cast<double*>(kcg_smem);
  const int stage_d = R * F;
  double* red = buf + stages * stage_d;  // [E] + s1[F] + mx[F]
  double* red_s1 = red + E;
  double* red_mx = red_s1 + F;
  __shared__ __align__(8) unsigned long long full[16];
  __shared__ unsigned reads[16];
  const int tid = threadIdx.x;
  for (int k = tid; k < E + 2 * F; k += blockDim.x) red[k] = 0.0;
  if (tid < 16) reads[tid] = 0;
  const unsigned fb = (unsigned)__cvta_generic_to_shared(full);
  const unsigned bb = (unsigned)__cvta_generic_to_shared(buf);
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(fb + 8 * s));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const kcg_i64 ntiles = n / R;
  if (tid == 0)
    for (int s = 0; s < stages; ++s) {
      const kcg_i64 t = blockIdx.x + (kcg_i64)s * gridDim.x;
      if (t >= ntiles) break;
      const unsigned bytes = (unsigned)(stage_d * 8);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb + 8 * s), "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       bb + (unsigned)(s * stage_d * 8)),
                   "l"(X + t * stage_d), "r"(bytes), "r"(fb + 8 * s)
                   : "memory");
    }
  switch ((tid >> 5) % G) {  // warp-uniform
    case 0: gram_dfma_part<F, G, M, 0>(X, n, stages, buf, fb, bb, reads, red, red_s1, red_mx); break;
    case 1:
      if constexpr (G > 1) gram_dfma_part<F, G, M, 1>(X, n, stages, buf, fb, bb, reads, red, red_s1, red_mx);
      break;
    case 2:
      if constexpr (G > 2) gram_dfma_part<F, G, M, 2>(X, n, stages, buf, fb, bb, reads, red, red_s1, red_mx);
      break;
    default:
      if constexpr (G > 3) gram_dfma_part<F, G, M, 3>(X, n, stages, buf, fb, bb, reads, red, red_s1, red_mx);
      break;
  }
  __syncthreads();
  for (int e = tid; e < E; e += blockDim.x) {
    const int p = tri_row(e, F), q = tri_col(e, F);
    atomicAdd(Gm + p * F + q, red[e]);
    if (p != q) atomicAdd(Gm + q * F + p, red[e]);
  }
  for (int c = tid; c < F; c += blockDim.x) {
    atomicAdd(xt1 + c, red_s1[c]);
    atomicMax(reinterpret_cast<unsigned long long*>(cmax + c), (unsigned long long)__double_as_longlong(red_mx[c]));
  }
}

template <int F, int G, int M>
void launch_gram_dfma(const double* X, size_t n, double* Gm, double* xt1, double* colmax, cudaStream_t stream) {
  constexpr int R = 32 * (8 / G) * M;
  constexpr int E = F * (F + 1) / 2;
  const size_t red_b = (size_t)(E + 2 * F) * sizeof(double);
  const size_t stage_b = (size_t)R * F * sizeof(double);
  int stages = (int)((200 * 1024 - red_b) / stage_b);
  stages = stages < 2 ? 2 : (stages > 16 ? 16 : stages);
  const size_t smem = (size_t)stages * stage_b + red_b;
  static std::mutex mu;
  static bool attr[64] = {};
  int dev = 0;
  check(cudaGetDevice(&dev), "cudaGetDevice");
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!attr[dev & 63]) {
      check(cudaFuncSetAttribute(kcg_gram_dfma<F, G, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem + 1024),
            "cudaFuncSetAttribute");
      attr[dev & 63] = true;
    }
  }
  const kcg_i64 tiles = (kcg_i64)n / R;
  kcg_i64 grid = (kcg_i64)num_sms();
  if (grid > tiles) grid = tiles > 0 ? tiles : 1;
  kcg_gram_dfma<F, G, M><<<(unsigned)grid, 256, smem, stream>>>(X, (kcg_i64)n, stages, Gm, xt1, colmax);
  check(cudaGetLastError(), "kcg_gram_dfma launch");
}

// F -> the DFMA kernel (true) or the DMMA path (false). all: also the
// widths where it measured no faster than DMMA (7, 12, 13, 20-22; 1e8 rows,
// profiles/gpu_r02_dfma.sh: F = 7 0.86 vs 0.81, 12 1.52 vs 1.49, 13 1.54
// vs 1.59, 20 2.66 vs 2.66, 21 2.98 vs 2.70, 22 3.97 vs 2.73 ms)
bool launch_gram_dfma_for(const double* X, size_t n, int F, double* Gm, double* xt1, double* colmax,
                          cudaStream_t st, bool all) {
  switch (F) {
    case 1: launch_gram_dfma<1, 1, 8>(X, n, Gm, xt1, colmax, st); return true;
    case 2: launch_gram_dfma<2, 1, 8>(X, n, Gm, xt1, colmax, st); return true;
    case 3: launch_gram_dfma<3, 1, 4>(X, n, Gm, xt1, colmax, st); return true;
    case 4: launch_gram_dfma<4, 1, 4>(X, n, Gm, xt1, colmax, st); return true;
    case 5: launch_gram_dfma<5, 1, 2>(X, n, Gm, xt1, colmax, st); return true;
    case 6: launch_gram_dfma<6, 1, 2>(X, n, Gm, xt1, colmax, st); return true;
    case 7: if (!all) return false; launch_gram_dfma<7, 1, 2>(X, n, Gm, xt1, colmax, st); return true;
    case 9: launch_gram_dfma<9, 1, 2>(X, n, Gm, xt1, colmax, st); return true;
    case 10: launch_gram_dfma<10, 1, 2>(X, n, Gm, xt1, colmax, st); return true;
    case 11: launch_gram_dfma<11, 1, 2>(X, n, Gm, xt1, colmax, st); return true;
    case 12: if (!all) return false; launch_gram_dfma<12, 2, 2>(X, n, Gm, xt1, colmax, st); return true;
    case 13: if (!all) return false; launch_gram_dfma<13, 2, 2>(X, n, Gm, xt1, colmax, st); return true;
    case 17: launch_gram_dfma<17, 4, 4>(X, n, Gm, xt1, colmax, st); return true;
    case 18: launch_gram_dfma<18, 4, 4>(X, n, Gm, xt1, colmax, st); return true;
    case 19: launch_gram_dfma<19, 4, 4>(X, n, Gm, xt1, colmax, st); return true;
    case 20: if (!all) return false; launch_gram_dfma<20, 4, 4>(X, n, Gm, xt1, colmax, st); return true;
    case 21: if (!all) return false; launch_gram_dfma<21, 4, 4>(X, n, Gm, xt1, colmax, st); return true;
    case 22: if (!all) return false; launch_gram_dfma<22, 4, 4>(X, n, Gm, xt1, colmax, st); return true;
    default: return false;
  }
}

// double-double helpers: (hi, lo) with |lo| <= ulp(hi) / 2
__device__ __forceinline__ void kcg_two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}
__device__ __forceinline__ void kcg_dd_add(double& hi, double& lo, double bh, double bl) {
  double s, e;
  kcg_two_sum(hi, bh, s, e);
  e = __dadd_rn(e, __dadd_rn(lo, bl));
  hi = __dadd_rn(s, e);
  lo = __dsub_rn(e, __dsub_rn(hi, s));
}

// warp per row: lane owns columns lane + 32 c, c < NC (F <= 32 NC).
// GRAD: g += X^T r with the residual r = 1 - x . alpha formed in
// double-double (exact products by FMA, compensated sums, a compensated
// warp reduction) and rounded once: the refinement step of fit_weights
// then converges to the exact least-squares solution of the double data
// (a plain double residual of a near-consistent fit is all rounding noise).
template <bool GRAD, int NC>
__global__ void __launch_bounds__(256)
    kcg_resid_x(const double* __restrict__ X, kcg_i64 n, int F, kcg_i64 ld,
                const double* __restrict__ alpha, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const kcg_i64 warp = ((kcg_i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const kcg_i64 nwarps = ((kcg_i64)gridDim.x * blockDim.x) >> 5;
  double a[NC], g[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    a[c] = lane + 32 * c < F ? alpha[lane + 32 * c] : 0.0;
    g[c] = 0.0;
  }
  double acc = 0.0;
  for (kcg_i64 r = warp; r < n; r += nwarps) {
    const double* row = X + r * ld;
    double x[NC];
    double d = 0.0;
    if (GRAD) {
      double lo = 0.0;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        x[c] = lane + 32 * c < F ? __ldcs(row + lane + 32 * c) : 0.0;
        const double p = __dmul_rn(x[c], a[c]);
        kcg_dd_add(d, lo, p, fma(x[c], a[c], -p));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
        kcg_dd_add(d, lo, __shfl_xor_sync(0xffffffffu, d, o), __shfl_xor_sync(0xffffffffu, lo, o));
      d = -d;
      lo = -lo;
      kcg_dd_add(d, lo, 1.0, 0.0);  // 1 - x . alpha
      d = __dadd_rn(d, lo);
    } else {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        x[c] = lane + 32 * c < F ? __ldcs(row + lane + 32 * c) : 0.0;
        d = fma(x[c], a[c], d);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    }
    const double res = GRAD ? d : 1.0 - d;
    if (GRAD) {
#pragma unroll
      for (int c = 0; c < NC; ++c) g[c] = fma(x[c], res, g[c]);
    } else {
      acc = fma(res, res, acc);
    }
  }
  if (GRAD) {
#pragma unroll
    for (int c = 0; c < NC; ++c)
      if (lane + 32 * c < F) atomicAdd(out + lane + 32 * c, g[c]);
  } else if (lane == 0) {
    atomicAdd(out, acc);
  }
}

template <bool GRAD>
void launch_resid_nc(const double* X, size_t n, int F, size_t ld, const double* alpha, double* out,
                     cudaStream_t st) {
  const unsigned grid = num_sms() * 8;
  switch ((F + 31) / 32) {
    case 1: kcg_resid_x<GRAD, 1><<<grid, 256, 0, st>>>(X, (kcg_i64)n, F, (kcg_i64)ld, alpha, out); break;
    case 2: kcg_resid_x<GRAD, 2><<<grid, 256, 0, st>>>(X, (kcg_i64)n, F, (kcg_i64)ld, alpha, out); break;
    case 3: kcg_resid_x<GRAD, 3><<<grid, 256, 0, st>>>(X, (kcg_i64)n, F, (kcg_i64)ld, alpha, out); break;
    case 4: kcg_resid_x<GRAD, 4><<<grid, 256, 0, st>>>(X, (kcg_i64)n, F, (kcg_i64)ld, alpha, out); break;
    default: kcg_resid_x<GRAD, 5><<<grid, 256, 0, st>>>(X, (kcg_i64)n, F, (kcg_i64)ld, alpha, out); break;
  }
  check(cudaGetLastError(), "kcg_resid_x launch");
}

// ---------------------------------------------------------------------------
// simulate_time noise and geometric_mean_error

__device__ __forceinline__ kcg_u64 fnv_byte(kcg_u64 h, unsigned char c) {
  return (h ^ c) * 1099511628211ull;
}

__device__ __forceinline__ kcg_u64 splitmix64(kcg_u64& x) {
  x += 0x9e3779b97f4a7c15ull;
  kcg_u64 z = x;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__global__ void __launch_bounds__(256) kcg_noise(const __grid_constant__ NoiseArgs a) {
  const kcg_i64 stride = (kcg_i64)gridDim.x * blockDim.x;
  for (kcg_i64 i = (kcg_i64)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {
    const double t0 = a.t[i];
    if (t0 != t0) continue;  // inadmissible point (NaN) stays NaN
    // key = kernel + "|" + binding_str(b): "p=v;q=w" in std::map (name) order
    kcg_u64 h = a.prefix_hash;
    for (int j = 0; j < a.n_params; ++j) {
      for (int c = 0; c < a.seg_len[j]; ++c) h = fnv_byte(h, a.seg[j][c]);
      const kcg_i64 v = a.cols[j][i];
      kcg_u64 u = v < 0 ? (kcg_u64)0 - (kcg_u64)v : (kcg_u64)v;
      if (v < 0) h = fnv_byte(h, '-');
      unsigned char d[20];
      int nd = 0;
      do {
        d[nd++] = (unsigned char)('0' + u % 10);
        u /= 10;
      } while (u);
      while (nd) h = fnv_byte(h, d[--nd]);
    }
    kcg_u64 st = h ^ (a.seed * 0x9e3779b97f4a7c15ull) ^ (a.counter * 0xd1342543de82ef95ull);
    double u1 = (double)(splitmix64(st) >> 11) * 0x1.0p-53;
    const double u2 = (double)(splitmix64(st) >> 11) * 0x1.0p-53;
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    const double g = sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
    a.t[i] = t0 * exp(a.sigma * g);
  }
}

__global__ void __launch_bounds__(256)
    kcg_geomean(const double* __restrict__ pred, const double* __restrict__ actual, kcg_i64 n,
                double* log_sum, unsigned long long* count, unsigned long long* bad) {
  double acc = 0.0;
  unsigned long long c = 0, b = 0;
  const kcg_i64 stride = (kcg_i64)gridDim.x * blockDim.x;
  for (kcg_i64 i = (kcg_i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double p = pred[i], y = actual[i];
    if (!(y > 0.0)) {
      ++b;
      continue;
    }
    double rel = fabs(p - y) / y;
    if (rel < 1e-12) rel = 1e-12;
    acc += log(rel);
    ++c;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc += __shfl_down_sync(0xffffffffu, acc, o);
    c += __shfl_down_sync(0xffffffffu, c, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(log_sum, acc);
    atomicAdd(count, c);
    if (b) atomicAdd(bad, b);
  }
}

int g_sms = 0;

}  // namespace

int num_sms() {
  if (g_sms) return g_sms;
  int dev = 0;
  check(cudaGetDevice(&dev), "cudaGetDevice");
  check(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev),
        "cudaDeviceGetAttribute");
  return g_sms;
}

void launch_interp_eval(const KcgDevProg* dprog, const KcgDevProg* dadmit, const InterpEvalArgs& a,
                        void* stream) {
  if (a.n == 0) return;
  const int threads = 128;
  kcg_i64 blocks = (a.n + threads - 1) / threads;
  const kcg_i64 cap = (kcg_i64)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  kcg_interp_eval<<<(unsigned)blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(dprog, dadmit, a);
  check(cudaGetLastError(), "kcg_interp_eval launch");
}

void launch_gram(const double* X, size_t n, int F, size_t ld, double* G, double* xt1,
                 double* colmax, void* stream) {
  if (n == 0) return;
  if (F < 1 || F > kGramMaxF) throw std::invalid_argument("gram: n_cols must be in [1, 160]");
  static const bool no_dmma = std::getenv("KCG_NO_DMMA") != nullptr;
  if (!no_dmma && ld == (size_t)F && F <= 72 &&
      reinterpret_cast<uintptr_t>(X) % 16 == 0) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // one CTA per SM from NB = KCG_DMMA_ONE_CTA_NB (default 6): measured
    // F = 48: 4.84 -> 4.35 ms; NB = 7, 8 need it (> 128 registers)
    static const int one_from = std::getenv("KCG_DMMA_ONE_CTA_NB") ? std::atoi(std::getenv("KCG_DMMA_ONE_CTA_NB")) : 6;
    const int nb = (F + 7) / 8;
    const bool one = nb >= one_from;
    // 128-row tiles for NB = 4, 5 at two CTAs/SM (F = 40: 6.49 -> 6.17 ms);
    // KCG_DMMA_TALL=0 restores 64
    static const bool tall = !(std::getenv("KCG_DMMA_TALL") && std::atoi(std::getenv("KCG_DMMA_TALL")) == 0);
    // 256-row tiles for NB = 3 too (F = 24: 2.81 -> 2.74 ms, 7.0 TB/s); KCG_DMMA_TALL3=0 restores 128
    static const bool tall3 = !(std::getenv("KCG_DMMA_TALL3") && std::atoi(std::getenv("KCG_DMMA_TALL3")) == 0);
    // DMMA off-diagonal + DFMA diagonal blocks (kcg_gram_hybrid): the
    // default for even F in 34..40 (1e8 rows, interleaved runs,
    // profiles/ab_gram_hybrid_r.sh: F = 40 5.95 vs 6.19 ms, F = 36 6.18 vs
    // 6.23); KCG_GRAM_HYBRID=1 takes it for even F in 26..32 too (F = 32:
    // 4.72 vs 4.53 ms, slower), =0 never
    // narrow designs the DMMA blocks pad (F <= 6, 9..11, 17..19): row-per-lane
    // DFMA over the distinct entries (F = 2: 0.59 -> 0.26 ms, 9: 1.49 ->
    // 1.08, 18: 2.67 -> 2.44 for 1e8 rows); KCG_GRAM_DFMA=0 keeps them on
    // DMMA, =2 also takes 7, 12, 13, 20..22
    // integer-sliced Gram on the int8 tensor pipe (gram_sliced.cu), F in 17..40
    static const int sliced = std::getenv("KCG_GRAM_SLICED") ? std::atoi(std::getenv("KCG_GRAM_SLICED")) : 0;
    if (sliced && launch_gram_sliced(X, n, F, G, xt1, colmax, st)) return;
    static const int dfma = std::getenv("KCG_GRAM_DFMA") ? std::atoi(std::getenv("KCG_GRAM_DFMA")) : 1;
    if (dfma && launch_gram_dfma_for(X, n, F, G, xt1, colmax, st, dfma == 2)) return;
    static const int hybrid_mode = std::getenv("KCG_GRAM_HYBRID") ? std::atoi(std::getenv("KCG_GRAM_HYBRID")) : -1;
    const bool hybrid = hybrid_mode == 1 || (hybrid_mode == -1 && nb == 5);
    if (hybrid && F % 2 == 0 && (nb == 4 || nb == 5))
    {
      static const int hr = std::getenv("KCG_GRAM_HYBRID_R") ? std::atoi(std::getenv("KCG_GRAM_HYBRID_R")) : 96;
      // rows per warp-group tile: 96 at NB = 5 (48: 6.15 ms, 144: 6.10 ms at
      // F = 40), 128 at NB = 4 (64: 5.12 ms at F = 32)
      static const int hr4 = std::getenv("KCG_GRAM_HYBRID_R4") ? std::atoi(std::getenv("KCG_GRAM_HYBRID_R4")) : 128;
      if (nb == 4) return hr4 == 128 ? launch_gram_hybrid<4, 128>(X, n, F, G, xt1, colmax, st)
                                     : launch_gram_hybrid<4, 64>(X, n, F, G, xt1, colmax, st);
      if (hr == 48) return launch_gram_hybrid<5, 48>(X, n, F, G, xt1, colmax, st);
      if (hr == 144) return launch_gram_hybrid<5, 144>(X, n, F, G, xt1, colmax, st);
      return launch_gram_hybrid<5, 96>(X, n, F, G, xt1, colmax, st);
    }
    switch (nb) {
      case 1:
        // very narrow rows: taller tiles keep every bulk copy >= 16 KB
        if (!one && tall && F <= 2) return launch_gram_dmma<1, 2, 1024>(X, n, F, G, xt1, colmax, st);
        if (!one && tall && F <= 4) return launch_gram_dmma<1, 2, 512>(X, n, F, G, xt1, colmax, st);
        return one ? launch_gram_dmma<1, 1>(X, n, F, G, xt1, colmax, st) : launch_gram_dmma<1, 2>(X, n, F, G, xt1, colmax, st);
      case 2: return one ? launch_gram_dmma<2, 1>(X, n, F, G, xt1, colmax, st) : launch_gram_dmma<2, 2>(X, n, F, G, xt1, colmax, st);
      case 3:
        if (tall3 && !one) return launch_gram_dmma<3, 2, 256>(X, n, F, G, xt1, colmax, st);
        return one ? launch_gram_dmma<3, 1>(X, n, F, G, xt1, colmax, st) : launch_gram_dmma<3, 2>(X, n, F, G, xt1, colmax, st);
      case 4:
        if (tall && !one) return launch_gram_dmma<4, 2, 128>(X, n, F, G, xt1, colmax, st);
        return one ? launch_gram_dmma<4, 1>(X, n, F, G, xt1, colmax, st) : launch_gram_dmma<4, 2>(X, n, F, G, xt1, colmax, st);
      case 5:
        if (tall && !one) return launch_gram_dmma<5, 2, 128>(X, n, F, G, xt1, colmax, st);
        return one ? launch_gram_dmma<5, 1>(X, n, F, G, xt1, colmax, st) : launch_gram_dmma<5, 2>(X, n, F, G, xt1, colmax, st);
      case 6: return one ? launch_gram_dmma<6, 1>(X, n, F, G, xt1, colmax, st) : launch_gram_dmma<6, 2>(X, n, F, G, xt1, colmax, st);
      case 7: return launch_gram_dmma<7, 1>(X, n, F, G, xt1, colmax, st);
      case 8: return launch_gram_dmma<8, 1>(X, n, F, G, xt1, colmax, st);
      default: return launch_gram_dmma<9, 1>(X, n, F, G, xt1, colmax, st);
    }
  }
  const bool wide = F > 64;
  const GramGeom g0 = gram_geom(F, 256);
  const int threads = wide ? g0.slice_threads : 256;  // wide: one thread per tile, <= 1024
  const GramGeom g = gram_geom(F, threads);
  const size_t smem = (size_t)(kGramRows * g.FP + g.ntiles * 16) * sizeof(double);
  {
    static std::mutex mu;
    static int attr[64][2] = {};
    int dev = 0;
    check(cudaGetDevice(&dev), "cudaGetDevice");
    std::lock_guard<std::mutex> lk(mu);
    if (!attr[dev & 63][wide]) {
      check(wide ? cudaFuncSetAttribute(kcg_gram_x<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)
                 : cudaFuncSetAttribute(kcg_gram_x<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024),
            "cudaFuncSetAttribute");
      attr[dev & 63][wide] = 1;
    }
  }
  const kcg_i64 chunks = ((kcg_i64)n + kGramRows - 1) / kGramRows;
  kcg_i64 ctas = (kcg_i64)num_sms() * (wide ? 1 : 4);
  if (ctas > chunks) ctas = chunks;
  const kcg_i64 chunks_per_cta = (chunks + ctas - 1) / ctas;
  ctas = (chunks + chunks_per_cta - 1) / chunks_per_cta;
  if (wide)
    kcg_gram_x<1024><<<(unsigned)ctas, threads, smem, static_cast<cudaStream_t>(stream)>>>(
        X, (kcg_i64)n, F, (kcg_i64)ld, chunks_per_cta * kGramRows, G, xt1, colmax);
  else
    kcg_gram_x<256><<<(unsigned)ctas, threads, smem, static_cast<cudaStream_t>(stream)>>>(
        X, (kcg_i64)n, F, (kcg_i64)ld, chunks_per_cta * kGramRows, G, xt1, colmax);
  check(cudaGetLastError(), "kcg_gram_x launch");
}

void launch_noise(const NoiseArgs& a, void* stream) {
  if (a.n == 0) return;
  kcg_noise<<<num_sms() * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(a);
  check(cudaGetLastError(), "kcg_noise launch");
}

void launch_geomean(const double* pred, const double* actual, size_t n, double* log_sum,
                    unsigned long long* count, unsigned long long* bad, void* stream) {
  if (n == 0) return;
  kcg_geomean<<<num_sms() * 4, 256, 0, static_cast<cudaStream_t>(stream)>>>(pred, actual, (kcg_i64)n,
                                                                           log_sum, count, bad);
  check(cudaGetLastError(), "kcg_geomean launch");
}

void launch_residual(const double* X, size_t n, int F, size_t ld, const double* alpha,
                     double* obj, void* stream) {
  if (n == 0) return;
  if (F < 1 || F > kGramMaxF) throw std::invalid_argument("residual: n_cols must be in [1, 160]");
  launch_resid_nc<false>(X, n, F, ld, alpha, obj, static_cast<cudaStream_t>(stream));
}

void launch_residual_grad(const double* X, size_t n, int F, size_t ld, const double* alpha,
                          double* g, void* stream) {
  if (n == 0) return;
  if (F < 1 || F > kGramMaxF) throw std::invalid_argument("residual grad: n_cols must be in [1, 160]");
  launch_resid_nc<true>(X, n, F, ld, alpha, g, static_cast<cudaStream_t>(stream));
}

}  // namespace kcg

// ---- grid descriptor -> SoA bindings (kcg_grid_bindings) -------------------
namespace {
struct GridArgsDev {
  int np;
  long long start[8], step[8];
  unsigned long long count[8];
  unsigned long long first;
  long long n;
  long long* cols[8];
};

__global__ void __launch_bounds__(256) kcg_grid_fill(const __grid_constant__ GridArgsDev g) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += stride) {
    unsigned long long r = g.first + (unsigned long long)i;
    for (int j = g.np - 1; j >= 0; --j) {
      const unsigned long long d = r % g.count[j];
      r /= g.count[j];
      __stcs(g.cols[j] + i, g.start[j] + g.step[j] * (long long)d);
    }
  }
}
}  // namespace

namespace kcg {
void launch_grid_fill(int np, const int64_t* start, const int64_t* step, const uint64_t* count, uint64_t first,
                      size_t n, int64_t* const* cols, void* stream) {
  GridArgsDev g{};
  g.np = np;
  for (int j = 0; j < np; ++j) {
    g.start[j] = start[j];
    g.step[j] = step[j];
    g.count[j] = count[j];
    g.cols[j] = reinterpret_cast<long long*>(cols[j]);
  }
  g.first = first;
  g.n = static_cast<long long>(n);
  const size_t need = (n + 255) / 256, cap = static_cast<size_t>(num_sms()) * 8;
  kcg_grid_fill<<<static_cast<unsigned>(need < cap ? need : cap), 256, 0, static_cast<cudaStream_t>(stream)>>>(g);
  check(cudaGetLastError(), "kcg_grid_fill launch");
}
}  // namespace kcg

// ---- design rows from exact counts (wide fused Gram / residual) -----------
namespace {
__global__ void __launch_bounds__(256)
    kcg_form_rows(const long long* __restrict__ lo, const long long* __restrict__ hi,
                  const unsigned char* __restrict__ st, const double* __restrict__ T, long long n, int F,
                  double* __restrict__ X, unsigned long long* bad) {
  unsigned long long nb = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double t = T[i];
    const bool ok = st[i] == KCG_PT_OK && t > 0.0;
    nb += !ok;
    for (int j = 0; j < F; ++j) {
      double x = 0.0;
      if (ok) {
        const kcg_i128 c = (kcg_i128)(((kcg_u128)(kcg_u64)hi[(long long)j * n + i] << 64) |
                                      (kcg_u128)(kcg_u64)lo[(long long)j * n + i]);
        if (c != 0) x = __ddiv_rn(kcg_to_double(c), t);  // model.cpp:29
      }
      X[i * F + j] = x;
    }
  }
  for (int o = 16; o > 0; o >>= 1) nb += __shfl_down_sync(0xffffffffu, nb, o);
  if ((threadIdx.x & 31) == 0 && nb && bad) atomicAdd(bad, nb);
}
}  // namespace

namespace kcg {
void launch_form_rows(const int64_t* lo, const int64_t* hi, const uint8_t* status, const double* T, size_t n,
                      int F, double* X, unsigned long long* bad, void* stream) {
  if (n == 0) return;
  const size_t need = (n + 255) / 256, cap = static_cast<size_t>(num_sms()) * 8;
  kcg_form_rows<<<static_cast<unsigned>(need < cap ? need : cap), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const long long*>(lo), reinterpret_cast<const long long*>(hi), status, T,
      static_cast<long long>(n), F, X, bad);
  check(cudaGetLastError(), "kcg_form_rows launch");
}
}  // namespace kcg
