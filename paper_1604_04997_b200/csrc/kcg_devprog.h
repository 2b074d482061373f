// Flat, POD image of a lowered program (kcg_host.hpp `Lowered`) for the
// ahead-of-time table interpreter. One copy lives in device global memory
// per program; every thread of a launch reads the same words (uniform,
// L1/L2-resident), so the interpreter never diverges on program structure.
#pragma once

#include <stdint.h>

#define KCG_MAX_PARAMS 8
#define KCG_MAX_OPS 256
#define KCG_MAX_ATOMS 32
#define KCG_MAX_MONOS 64
#define KCG_MAX_FACTORS 256
#define KCG_MAX_TERMS 512
#define KCG_MAX_EXPRS 96
#define KCG_MAX_ARGS 64
#define KCG_MAX_FD 32
#define KCG_MAX_CONS 32
#define KCG_MAX_KEYS 149

struct KcgWide {
  int64_t lo, hi;  // two's complement int128
};

struct KcgDevOp {
  int32_t code, dst, a, b, c;
};

struct KcgDevProg {
  int32_t n_params, n_atoms, n_monos, n_exprs;
  int32_t n_ops, n_cons, n_keys, pad;
  int64_t b64, b128;  // safe uniform parameter bounds (-1: no such path)
  KcgDevOp ops[KCG_MAX_OPS];
  int32_t fac_atom[KCG_MAX_FACTORS];
  int32_t fac_exp[KCG_MAX_FACTORS];
  KcgWide term_coef[KCG_MAX_TERMS];
  int32_t term_mono[KCG_MAX_TERMS];
  KcgWide expr_den[KCG_MAX_EXPRS];
  int32_t arg_expr[KCG_MAX_ARGS];
  KcgWide arg_scale[KCG_MAX_ARGS];
  KcgWide fd_den[KCG_MAX_FD];
  int32_t cons_div[KCG_MAX_CONS], cons_op[KCG_MAX_CONS], cons_expr[KCG_MAX_CONS];
  KcgWide cons_mod[KCG_MAX_CONS], cons_rem[KCG_MAX_CONS];
  int32_t key_schema[KCG_MAX_KEYS], key_expr[KCG_MAX_KEYS];
  KcgWide quot_mod[KCG_MAX_PARAMS], quot_rem[KCG_MAX_PARAMS];
};
