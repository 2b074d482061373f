// Device image of one statement walk of the GPU enumeration oracle
// (enum_kernels.cu), compiled on the host per binding by enumerate.cpp.
//
// Mirrors the compiled fast path of the reference's enumerator
// (FastDomain / Row / FastGuard, enumerate.cpp:99-293): bounds, guards and
// access indices are integer rows c0 + sum_s c_s x_s over the statement's
// domain-variable slots with every parameter (and parameter-only floordiv)
// folded into c0 and rational coefficients scaled out by a common positive
// denominator `den`. Values are raw / den. Floor divisions over domain
// variables -- what the reference hands to its generic Walker
// (enumerate.cpp:31-90) -- are statement-level KeFd terms of the rows.
#pragma once

#include <stdint.h>

#define KE_MAXV 12  // domain variables per statement
#define KE_MAXG 8  // guards per statement
#define KE_MAXA 8  // global accesses per statement
#define KE_MAXD 4  // array rank
#define KE_MAXF 4  // floor divisions over domain variables per statement

// raw = c0 + sum_s c[s] x_s + sum_f cf[f] floor(raw(fd_f) / fd_f.div); value raw / den
struct KeRow {
  int64_t den;  // > 0
  int64_t c0;
  int64_t c[KE_MAXV];
  int64_t cf[KE_MAXF];
};

// floor((c0 + sum_s c_s x_s) / div) -- a floordiv atom over domain variables
// (the reference's parser allows them in loop bounds: `0 .. (i + 1) // 2`);
// its row has no floordiv terms of its own
struct KeFd {
  int64_t div;  // > 0: the atom's divisor times its row's den
  KeRow r;
};

struct KeGuard {
  int32_t depth;  // deepest slot referenced (the reference checks it there)
  int32_t divis;  // 1: ((raw % mod) + mod) % mod == rem (den == 1)
  int32_t op;     // relational: 0 <, 1 <=, 2 >, 3 >=, 4 == against 0
  int32_t pad;
  int64_t mod, rem;
  KeRow r;  // lhs - rhs (relational) or lhs (divisibility)
};

// target bitmaps of one global access (the whole array's footprint, shared
// by every access to the array): cell ids are row-major over a bounding box
// that contains every index the access can produce
struct KeMark {
  int32_t nd, fast;
  int64_t lo[KE_MAXD];
  int64_t ext[KE_MAXD];
  unsigned long long* cells;   // bit per box cell
  unsigned long long* others;  // bit per box cell of the non-fastest axes
  unsigned long long* fastp;   // bit per coordinate of the fastest axis
};

struct KeAccess {
  KeRow idx[KE_MAXD];  // integral rows (den == 1)
  KeMark m;
};

struct KeStmt {
  int32_t nv;     // domain variables
  int32_t nbox;   // leading levels with parameter-only bounds (flattened over threads)
  int32_t nbe;    // levels the threads enumerate: nbox, or the first empty box level
  int32_t inner;  // 1 when every box level is non-empty (leaves possible)
  int32_t ng, na;
  int32_t nf, pad_f;
  KeFd f[KE_MAXF];
  int64_t box_lo[KE_MAXV], box_ext[KE_MAXV];
  unsigned long long box_total;  // product of box_ext over the nbe levels
  KeRow lo[KE_MAXV], hi[KE_MAXV];  // bounds of the inner levels (hi exclusive)
  KeGuard g[KE_MAXG];
  KeAccess a[KE_MAXA];
  unsigned long long* out;  // [0] += leaves, [1] += visited (leaves + dead ends)
};
