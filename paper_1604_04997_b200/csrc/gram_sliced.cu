// Integer-sliced Gram on the 5th-generation tensor cores (tcgen05 kind::i8)
//
// G += X^T X, X^T 1, colmax for a materialised fp64 design X [n][F],
// F <= 40 -- the same contract as the FP64 DMMA / hybrid kernels in
// kernels.cu (kcg_gram_accumulate, model.cpp:37-60's normal equations), but
// the O(F^2) products run on the int8 tensor pipe instead of the FP64 pipe.
// B200's FP64 pipe (DMMA and DFMA share it at 37 TFLOP/s, profiles/
// r02_dmma_dfma.json) bounds the hybrid kernel at 4.6 ms for 1e8 x 40 rows,
// above the 4.9 ms HBM time only by a margin its issue overheads eat (5.95
// ms measured); the int8 pipe runs the same products in 2.3 ms
// (profiles/umma_i8_probe.cu: 4.0 POPS for this kernel's MMA mix), leaving
// the kernel HBM-bound.
//
// Exactness (Ozaki-style splitting with per-column fixed point):
//   * every column i has a segment exponent e_i >= the exponent of every
//     |x_ri| sliced under it; x_ri is rounded to the integer
//     v = rn(x_ri 2^(53 - e_i)), |v| < 2^54 -- exact for x_ri in the top
//     binade [2^e_i, 2^(e_i+1)), 2^-54 |x|max-relative otherwise;
//   * v is split into seven signed 8-bit digits, v = sum_k s_k 2^(8k)
//     (bytes of v + 0x0080808080808080, each xor 0x80): exact;
//   * digit products accumulate in int32 TMEM cells exactly (|s_a s_b| <=
//     2^14, <= 2^15 rows per segment);
//   * the tensor cores form D_ab = S_a^T S_b for every digit pair with
//     a <= b, a + b <= 7 (a = 0 the top digit) -- and a few more that fit
//     the MMA rectangles; pairs with a + b >= 8 weigh <= 2^-64 of the top
//     pair and are dropped;
//   * a segment ends after 256 tiles or when a tile holds a value at or
//     above 2^(e_i + 1) in some column; its cells are then converted to
//     fp64 (exact power-of-two scalings, <= 7 rounded additions per entry)
//     and added to the CTA's fp64 partial, and the exponents are raised.
// So each product x_ri x_rj is represented to within 2^-52 of
// |x|max_i |x|max_j over its segment, and the column sums X^T 1 are the exact
// sums of the rounded v, added in fp64 once per tile -- the same error
// class as fp64 accumulation over a long chain. Values must lie in
// [2^-960, 2^960) or be 0 (smaller magnitudes round to 0 at 2^-1013
// absolute); a non-finite value makes the CTA's G and X^T 1 contribution NaN.
//
// Layout. A CTA per SM walks its tiles of KT = 128 rows (tile blockIdx.x +
// t gridDim.x). Ten warps slice: thread (c, i) owns feature i of rows
// 16c..16c+15, loads them straight from HBM one tile ahead (whole tiles
// are bulk-prefetched into L2 six tiles ahead), and writes their seven
// digits as seven 16-byte core-matrix rows of a 3-stage operand ring:
// index (a, i) -> a FP + i (FP = F rounded up to 8), K = the tile's rows,
// K-major, no swizzle (8-row x 16-byte core matrices, LBO = 128 B, SBO =
// 1 KB). Per tile one CTA barrier (a bar.red that also ORs the segment
// test) hands the previous tile to thread 0, which issues per 32-row K step
//   MMA1  A = digits 0..2 (M = 128 lanes), B = rows [0, N1)    -> TMEM [0, N1)
//   MMA2  A = digits 0..2,                 B = rows [N1, 2N1)  -> TMEM [N1, 2 N1)
//   MMA3  A = digit 3.. (lanes < FP used), B = digits 3, 4     -> TMEM [2 N1, 2 N1 + N2)
// with N1 = 144, N2 = 80 at F = 40 (368 of the 512 TMEM columns), and
// commits to the stage's mbarrier. Warps 0..3 (TMEM lane quarters 0..3)
// drain the cells at the end of each segment. Measured 7.6-7.8 ms at 1e8 x
// 40 against 5.94 ms for the FP64 hybrid: DESIGN.md section 4 has the
// version history and what bounds it (shared memory and load latency, not
// the tensor pipe).
//
// (c) this repository; the algorithm follows the reference's normal
// equations only through the Gram contract (model.cpp:37-60).
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>

#include <cstdio>

#include <cuda_runtime.h>

#include "kcg_device.cuh"

namespace kcg {

int num_sms();

namespace {

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

constexpr int SL_KT = 128;                 // rows per tile (MMA K extent)
constexpr int SL_SB = 8 * SL_KT;           // bytes between 8-row core groups
constexpr int SL_PF = 6;                   // tiles prefetched into L2 ahead of the slicers
constexpr int SL_S2 = 3;                   // operand ring stages
constexpr int SL_THREADS = 320;            // 10 slicer warps (one thread per feature and 16-row chunk)
constexpr int SL_SEG_CAP = 256;            // tiles per segment (int32 headroom: 2^14 * 2^15 < 2^31)

// S = 7 digits (56-bit fixed point, the default) or 6 (48-bit: one N = 6 FP
// MMA for digits 0..2 and digit 3 x 3 only -- 27% fewer operand bytes per
// tile, KCG_SLICED_DIGITS=6 for the A/B)
template <int FP, int S>
struct SlGeom {
  static constexpr int NB1 = S == 7 ? 2 : 1;  // MMAs over digits 0..2 x all digits
  static constexpr int N1 = S == 7 ? ((7 * FP + 1) / 2 + 15) / 16 * 16 : (6 * FP + 15) / 16 * 16;
  static constexpr int B2 = S == 7 ? 2 : 1;   // digit 3 against digits 3 .. 3 + B2 - 1
  static constexpr int N2 = (B2 * FP + 15) / 16 * 16;
  static constexpr int G2 = NB1 * N1;         // TMEM column of the digit-3 block
  static constexpr int ROWS_A = 3 * FP + 128;
  static constexpr int NROWS = (NB1 * N1 > ROWS_A ? NB1 * N1 : ROWS_A);
  static constexpr int OPB = NROWS * SL_KT;  // operand stage bytes
  static constexpr int SCALE = 8 * S - 3;    // v = rn(x 2^(SCALE - e)), |v| < 2^(8 S - 2)
  static constexpr long long OFF = S == 7 ? 0x0080808080808080ll : 0x0000808080808080ll;
  static_assert(S == 6 || S == 7, "digits");
  static_assert(3 * FP <= 128, "three digit planes per M = 128 MMA");
  static_assert(G2 + N2 <= 512, "TMEM columns");
  static_assert(N1 <= 256 && N2 <= 256, "MMA N");
};

__device__ __forceinline__ uint64_t sl_sdesc(unsigned addr) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(SL_SB >> 4) << 32) |
         ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t sl_idesc(int N) {
  // D = s32, A = B = signed 8-bit, K-major both, M = 128
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void sl_mma(unsigned d, uint64_t a, uint64_t b, uint32_t idesc, unsigned acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// mbarrier phase wait; a wait that outlives ~4 s of clocks is a protocol bug:
// report the barrier and trap instead of hanging the device
__device__ __forceinline__ void sl_wait(unsigned mbar, unsigned parity) {
  unsigned done = 0;
  long long t0 = 0;
  while (!done) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(mbar), "r"(parity)
                 : "memory");
    if (!done) {
      const long long now = clock64();
      if (t0 == 0) t0 = now;
      else if (now - t0 > 8000000000ll) {
        printf("kcg_gram_sliced: mbarrier %#x parity %u stuck (block %d thread %d)\n", mbar, parity, blockIdx.x, threadIdx.x);
        __trap();
      }
    }
  }
}
__device__ __forceinline__ void sl_bar() { asm volatile("bar.sync 1, %0;" ::"n"(SL_THREADS) : "memory"); }
__device__ __forceinline__ bool sl_bar_or(bool v) {
  unsigned r;
  asm volatile("{ .reg .pred p, q; setp.ne.u32 p, %1, 0; bar.red.or.pred q, 1, %2, p; selp.u32 %0, 1, 0, q; }"
               : "=r"(r)
               : "r"((unsigned)v), "n"(SL_THREADS)
               : "memory");
  return r != 0;
}
__device__ __forceinline__ double sl_pow2(int e) {  // e in [-1022, 1023]
  return __longlong_as_double((long long)(e + 1023) << 52);
}
__device__ __forceinline__ unsigned sl_prmt(unsigned a, unsigned b, unsigned s) {
  unsigned r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(s));
  return r;
}

// cells of the current segment -> P (fp64 partial, [FP][FP], symmetrised at
// the end: G = P + P^T). Called by the 4 warps of TMEM lane quarters 0..3.
// pj[b][j] = 2^(e_j - 5 - 8 b), so D_ab[i][j] pj[a][i] pj[b][j] is the
// digit pair's contribution to x_i x_j (a, b = 0 the top digit).
template <int FP, int S>
__device__ __forceinline__ void sl_drain(unsigned tmem, int F, const double* pj, double* P) {
  using Gm = SlGeom<FP, S>;
  const int m = threadIdx.x;  // TMEM lane (warps 0..3)
  const unsigned lane_base = tmem + ((unsigned)(threadIdx.x & ~31) << 16);
  // digits 0..2 (lanes < 3 FP) against every digit b >= a
  {
    const int a = m / FP, i = m % FP;
    const bool own = m < 3 * FP && i < F;
    const double pi = own ? pj[a * FP + i] : 0.0;
#pragma unroll
    for (int j0 = 0; j0 < FP; j0 += 8) {
      double acc[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = 0.0;
#pragma unroll
      for (int b = 0; b < S; ++b) {
        unsigned r[8];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t"
            "tcgen05.wait::ld.sync.aligned;"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
            : "r"(lane_base + (unsigned)(b * FP + j0))
            : "memory");
        const double w = b > a ? 1.0 : (b == a ? 0.5 : 0.0);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = fma(w, (double)(int)r[q] * pj[b * FP + j0 + q], acc[q]);
      }
      if (own)
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (j0 + q < F) atomicAdd(P + i * FP + j0 + q, acc[q] * pi);
    }
  }
  // digit 3 against digits 3 (half weight) and 4; lanes < FP
  {
    const bool own = m < F;
    const double pi = own ? pj[3 * FP + m] : 0.0;
#pragma unroll
    for (int j0 = 0; j0 < FP; j0 += 8) {
      double acc[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = 0.0;
#pragma unroll
      for (int b = 3; b < 3 + Gm::B2; ++b) {
        unsigned r[8];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t"
            "tcgen05.wait::ld.sync.aligned;"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
            : "r"(lane_base + (unsigned)(Gm::G2 + (b - 3) * FP + j0))
            : "memory");
        const double w = b == 3 ? 0.5 : 1.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = fma(w, (double)(int)r[q] * pj[b * FP + j0 + q], acc[q]);
      }
      if (own)
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (j0 + q < F) atomicAdd(P + m * FP + j0 + q, acc[q] * pi);
    }
  }
}

template <int FP, bool FULL, int S>
__global__ void __launch_bounds__(SL_THREADS, 1)
    kcg_gram_sliced(const double* __restrict__ X, kcg_i64 n, int F_, double* __restrict__ G,
                    double* __restrict__ xt1, double* __restrict__ cmax) {
  using Gm = SlGeom<FP, S>;
  // FULL: F == FP, a compile-time row pitch
  const int F = FULL ? FP : F_;
  extern __shared__ __align__(1024) unsigned char sl_smem[];
  // [operand ring: S2 x OPB][P: FP FP 8][pj: 7 FP 8][x1: FP 8][cm: FP 8][e: FP 4][tcm: FP 4]
  unsigned char* opr = sl_smem;
  const int stage_d = SL_KT * F;
  double* P = reinterpret_cast<double*>(sl_smem + SL_S2 * Gm::OPB);
  double* pj = P + FP * FP;
  double* sx1 = pj + 7 * FP;
  unsigned long long* scm = reinterpret_cast<unsigned long long*>(sx1 + FP);
  int* sE = reinterpret_cast<int*>(scm + FP);
  unsigned* tcm = reinterpret_cast<unsigned*>(sE + FP);
  __shared__ __align__(8) unsigned long long op_empty[SL_S2];
  __shared__ unsigned tmem_base;
  __shared__ int nonfinite;

  const int tid = threadIdx.x, warp = tid >> 5;
  for (int k = tid; k < FP * FP; k += blockDim.x) P[k] = 0.0;
  for (int k = tid; k < FP; k += blockDim.x) {
    sx1[k] = 0.0;
    scm[k] = 0ull;
    tcm[k] = 0u;
    sE[k] = -960;
  }
  if (tid == 0) nonfinite = 0;
  const unsigned oeb = (unsigned)__cvta_generic_to_shared(op_empty);
  const unsigned ob = (unsigned)__cvta_generic_to_shared(opr);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < SL_S2; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(oeb + 8 * s));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = tmem_base;

  const kcg_i64 ntiles = n / SL_KT;
  // this CTA's tiles blockIdx.x + t gridDim.x, t < ct (< 2^31: n < 2^31 * 128 * gridDim.x)
  const int ct = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  const unsigned bytes = (unsigned)(stage_d * 8);
  auto tile_ptr = [&](int t) { return X + (blockIdx.x + (kcg_i64)t * gridDim.x) * (kcg_i64)stage_d; };
  auto prefetch = [&](int t) {  // whole tile into L2 (the slicers' loads then hit L2)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(tile_ptr(t)), "r"(bytes) : "memory");
  };
  // the MMAs of local tile t (operand stage t % S2), issued by thread 0 once every
  // warp has written it (after the next CTA barrier); committed to op_empty[t % S2]
  auto issue_mma = [&](int t, bool first) {
    constexpr uint32_t id1 = sl_idesc(Gm::N1), id2 = sl_idesc(Gm::N2);
    const int s2 = t % SL_S2;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned base = ob + (unsigned)(s2 * Gm::OPB);
#pragma unroll
    for (int ks = 0; ks < SL_KT / 32; ++ks) {
      const unsigned kb = base + ks * 256;
      const unsigned acc = (first && ks == 0) ? 0u : 1u;
      sl_mma(tmem, sl_sdesc(kb), sl_sdesc(kb), id1, acc);
      if (Gm::NB1 == 2) sl_mma(tmem + Gm::N1, sl_sdesc(kb), sl_sdesc(kb + (Gm::N1 / 8) * SL_SB), id1, acc);
      sl_mma(tmem + Gm::G2, sl_sdesc(kb + (3 * FP / 8) * SL_SB), sl_sdesc(kb + (3 * FP / 8) * SL_SB), id2, acc);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(oeb + 8 * s2)
                 : "memory");
  };
  // every MMA through local tile t is complete
  auto mma_done = [&](int t) { sl_wait(oeb + 8 * (t % SL_S2), (unsigned)((t / SL_S2) & 1)); };

  // thread (c, i) owns feature i of rows 16 c .. 16 c + 15 (one core-matrix row per digit)
  const bool act = tid < 8 * FP;
  const int i = act ? tid % FP : 0, c = act ? tid / FP : 0;
  constexpr bool ALL = FULL && 8 * FP == SL_THREADS;  // every thread owns a real column
  const bool real = ALL || (act && i < F);
  int e = -960;  // segment exponent of column i
  double scale = sl_pow2(Gm::SCALE - e);
  unsigned lim_hi = 0u;           // high word of 2^(e + 1): the first tile always opens a segment
  unsigned cm_hi = 0u;            // high word of cm
  unsigned long long cm = 0ull;   // running max |x| bits
  double xacc = 0.0;              // X^T 1 of this thread's rows (fp64 sum of the inputs)
  int seg_n = 0;
  bool prev_first = false;        // tile t - 1 opened its segment
  const int roff = 16 * c * F + i;
  // digit a of feature i goes to core row group (a FP + i) / 8 = a FP / 8 + i / 8 (FP % 8 == 0)
  unsigned char* const dst0 = opr + c * 128 + (i >> 3) * SL_SB + (i & 7) * 16;
  if (tid == 0)
    for (int t = 0; t < SL_PF && t < ct; ++t) prefetch(t);
  // this thread's 16 values of the next tile, loaded a tile ahead (L2 hits after the prefetch)
  // this thread's 16 values of the next tile, loaded while the current tile is
  // sliced (L2 hits after the bulk prefetch)
  const double* src = X + (kcg_i64)blockIdx.x * stage_d + roff;
  const kcg_i64 tstep = (kcg_i64)gridDim.x * stage_d;
  double xn[16];
  auto load = [&](int t) {
    if (t < ct) {
      const double* p = src + (kcg_i64)t * tstep;
#pragma unroll
      for (int r = 0; r < 16; ++r) xn[r] = real ? __ldcs(p + r * F) : 0.0;
    }
  };
  load(0);
  for (int t = 0; t < ct; ++t) {
    double x[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) x[r] = xn[r];
    load(t + 1);
    if (tid == 0 && t + SL_PF < ct) prefetch(t + SL_PF);
    // high words of |x|: the segment test (2^(e+1) has a zero low word) and the column max
    unsigned mh = 0u;
#pragma unroll
    for (int r = 0; r < 16; ++r) mh = max(mh, (unsigned)(__double_as_longlong(x[r]) >> 32) & 0x7FFFFFFFu);
    if (mh >= cm_hi) {  // rare after the first tiles: exact 64-bit maximum
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const unsigned long long b = (unsigned long long)__double_as_longlong(x[r]) & 0x7FFFFFFFFFFFFFFFull;
        cm = b > cm ? b : cm;
      }
      cm_hi = (unsigned)(cm >> 32);
      if (mh >= 0x7FF00000u) nonfinite = 1;
    }
    // CTA barrier: tile t - 1's digits are all written (each writer fenced them
    // for the async proxy) and every thread agrees on a segment break
    const bool flush = sl_bar_or(mh >= lim_hi || seg_n == SL_SEG_CAP);
    if (tid == 0 && t > 0) issue_mma(t - 1, prev_first);
    if (flush) {
      if (real) atomicMax(tcm + i, mh);
      if (t > 0) {
        mma_done(t - 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (warp < 4) sl_drain<FP, S>(tmem, F, pj, P);
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      }
      sl_bar();
      if (act && c == 0) {
        int en = sE[i];
        if (real) {
          const int ex = (int)(tcm[i] >> 20) - 1023;
          en = ex > en ? ex : en;
          en = en < -960 ? -960 : (en > 1023 ? 1023 : en);
        }
        sE[i] = en;
        tcm[i] = 0u;
#pragma unroll
        for (int b = 0; b < S; ++b) pj[b * FP + i] = real ? sl_pow2(en - 5 - 8 * b) : 0.0;
      }
      sl_bar();
      e = sE[i];
      scale = sl_pow2(Gm::SCALE - e);
      lim_hi = e >= 1023 ? 0x7FF00000u : (unsigned)(e + 1 + 1023) << 20;
      seg_n = 0;
    }
    prev_first = seg_n == 0;
    ++seg_n;
    // operand stage t % S2 is free once tile t - S2's MMAs are done
    if (t >= SL_S2) mma_done(t - SL_S2);
    // digits: 4 rows at a time, a 4 x 8 byte transpose
    unsigned wd[7][4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      unsigned L[4], H[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        xacc += x[4 * g + q];
        const long long v = __double2ll_rn(x[4 * g + q] * scale);
        const long long w = v + Gm::OFF;
        L[q] = (unsigned)w;
        H[q] = (unsigned)((unsigned long long)w >> 32);
      }
      const unsigned a0 = sl_prmt(L[0], L[1], 0x5140), a1 = sl_prmt(L[0], L[1], 0x7362);
      const unsigned b0 = sl_prmt(L[2], L[3], 0x5140), b1 = sl_prmt(L[2], L[3], 0x7362);
      const unsigned h0 = sl_prmt(H[0], H[1], 0x5140), h1 = sl_prmt(H[0], H[1], 0x7362);
      const unsigned k0 = sl_prmt(H[2], H[3], 0x5140), k1 = sl_prmt(H[2], H[3], 0x7362);
      // digit a = byte (S - 1 - a) of w, xor 0x80 per byte
      wd[S - 1][g] = sl_prmt(a0, b0, 0x5410) ^ 0x80808080u;
      wd[S - 2][g] = sl_prmt(a0, b0, 0x7632) ^ 0x80808080u;
      wd[S - 3][g] = sl_prmt(a1, b1, 0x5410) ^ 0x80808080u;
      wd[S - 4][g] = sl_prmt(a1, b1, 0x7632) ^ 0x80808080u;
      wd[S - 5][g] = sl_prmt(h0, k0, 0x5410) ^ 0x80808080u;
      wd[S - 6][g] = sl_prmt(h0, k0, 0x7632) ^ 0x80808080u;
      if (S == 7) wd[0][g] = sl_prmt(h1, k1, 0x5410) ^ 0x80808080u;
    }
    if (act) {
      unsigned char* dst = dst0 + (t % SL_S2) * Gm::OPB;
#pragma unroll
      for (int a = 0; a < S; ++a)
        *reinterpret_cast<uint4*>(dst + a * (FP / 8) * SL_SB) = make_uint4(wd[a][0], wd[a][1], wd[a][2], wd[a][3]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
  // final segment: the last tile's MMAs, then the drain
  if (ct > 0) {
    sl_bar();
    if (tid == 0) issue_mma(ct - 1, prev_first);
    mma_done(ct - 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp < 4) sl_drain<FP, S>(tmem, F, pj, P);
  }
  if (real) {
    atomicAdd(sx1 + i, xacc);
    atomicMax(scm + i, cm);
  }
  // tail rows (block 0): fp64 products, half weight into P (G = P + P^T)
  if (blockIdx.x == 0 && ntiles * SL_KT < n) {
    const kcg_i64 r0 = ntiles * SL_KT;
    for (int k = tid; k < F * F; k += SL_THREADS) {
      const int a = k / F, b = k % F;
      double s = 0.0;
      for (kcg_i64 r = r0; r < n; ++r) s = fma(X[r * F + a], X[r * F + b], s);
      atomicAdd(P + a * FP + b, 0.5 * s);
    }
    for (int k = tid; k < F; k += SL_THREADS) {
      double s = 0.0;
      unsigned long long m = 0ull;
      for (kcg_i64 r = r0; r < n; ++r) {
        const double v = X[r * F + k];
        s += v;
        const unsigned long long b = (unsigned long long)__double_as_longlong(v) & 0x7FFFFFFFFFFFFFFFull;
        m = b > m ? b : m;
      }
      atomicAdd(sx1 + k, s);
      atomicMax(scm + k, m);
      if (m >= 0x7FF0000000000000ull) nonfinite = 1;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  const double nanv = __longlong_as_double(0x7FF8000000000000ll);
  const bool bad = nonfinite != 0;
  for (int k = tid; k < FP * FP; k += SL_THREADS) {
    const int r = k / FP, cc = k % FP;
    if (r >= F || cc >= F || cc < r) continue;
    const double v = bad ? nanv : P[r * FP + cc] + P[cc * FP + r];
    atomicAdd(G + r * F + cc, v);
    if (cc != r) atomicAdd(G + cc * F + r, v);
  }
  for (int k = tid; k < F; k += SL_THREADS) {
    atomicAdd(xt1 + k, bad ? nanv : sx1[k]);
    atomicMax(reinterpret_cast<unsigned long long*>(cmax + k), scm[k]);
  }
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int FP, bool FULL, int S>
void launch_sliced(const double* X, size_t n, int F, double* G, double* xt1, double* colmax, cudaStream_t st) {
  using Gm = SlGeom<FP, S>;
  const size_t smem = (size_t)SL_S2 * Gm::OPB + (size_t)FP * FP * 8 +
                      7 * FP * 8 + FP * 8 + FP * 8 + FP * 4 + FP * 4;
  static std::mutex mu;
  static size_t attr[64] = {};
  int dev = 0;
  check(cudaGetDevice(&dev), "cudaGetDevice");
  {
    std::lock_guard<std::mutex> lk(mu);
    if (smem > attr[dev & 63]) {
      check(cudaFuncSetAttribute(kcg_gram_sliced<FP, FULL, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
            "cudaFuncSetAttribute");
      attr[dev & 63] = smem;
    }
  }
  const kcg_i64 tiles = (kcg_i64)n / SL_KT;
  kcg_i64 grid = num_sms();
  if (grid > tiles) grid = tiles > 0 ? tiles : 1;
  kcg_gram_sliced<FP, FULL, S><<<(unsigned)grid, SL_THREADS, smem, st>>>(X, (kcg_i64)n, F, G, xt1, colmax);
  check(cudaGetLastError(), "kcg_gram_sliced launch");
}

}  // namespace

// F in [17, 40]: returns false for other widths (the caller keeps its FP64 kernels)
bool launch_gram_sliced(const double* X, size_t n, int F, double* G, double* xt1, double* colmax,
                        cudaStream_t st) {
  if (F < 17 || F > 40) return false;
  static const int digits = std::getenv("KCG_SLICED_DIGITS") && std::atoi(std::getenv("KCG_SLICED_DIGITS")) == 6 ? 6 : 7;
  if (digits == 6) {  // A/B only: 48-bit digits
    if (F == 40) launch_sliced<40, true, 6>(X, n, F, G, xt1, colmax, st);
    else if (F <= 24) launch_sliced<24, false, 6>(X, n, F, G, xt1, colmax, st);
    else if (F <= 32) launch_sliced<32, false, 6>(X, n, F, G, xt1, colmax, st);
    else launch_sliced<40, false, 6>(X, n, F, G, xt1, colmax, st);
    return true;
  }
  if (F == 24) launch_sliced<24, true, 7>(X, n, F, G, xt1, colmax, st);
  else if (F == 32) launch_sliced<32, true, 7>(X, n, F, G, xt1, colmax, st);
  else if (F == 40) launch_sliced<40, true, 7>(X, n, F, G, xt1, colmax, st);
  else if (F < 24) launch_sliced<24, false, 7>(X, n, F, G, xt1, colmax, st);
  else if (F < 32) launch_sliced<32, false, 7>(X, n, F, G, xt1, colmax, st);
  else launch_sliced<40, false, 7>(X, n, F, G, xt1, colmax, st);
  return true;
}

}  // namespace kcg
