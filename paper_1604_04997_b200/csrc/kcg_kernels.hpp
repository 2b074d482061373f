// Ahead-of-time sm_100a kernels (kernels.cu) and their host launchers.
#pragma once

#include <cstddef>
#include <cstdint>

#include "kcg_devprog.h"

namespace kcg {

struct InterpEvalArgs {
  const int64_t* p[KCG_MAX_PARAMS];
  double* pred;
  uint8_t* status;
  int64_t* clo;
  int64_t* chi;
  int64_t n;
  int simulate;
  double alpha[KCG_MAX_KEYS];  // compact, one per program key
};

/// Table-interpreter evaluate + predict (KCG_ENGINE_INTERP).
void launch_interp_eval(const KcgDevProg* dprog, const KcgDevProg* dadmit,
                        const InterpEvalArgs& a, void* stream);

/// Materialised-X Gram: G += X^T X, xt1 += X^T 1, colmax = max(colmax,|X|).
void launch_gram(const double* X, size_t n, int F, size_t ld, double* G,
                 double* xt1, double* colmax, void* stream);

/// obj += sum (1 - X alpha)^2
void launch_residual(const double* X, size_t n, int F, size_t ld,
                     const double* alpha, double* obj, void* stream);

/// g += X^T (1 - X alpha)
void launch_residual_grad(const double* X, size_t n, int F, size_t ld,
                          const double* alpha, double* g, void* stream);

int num_sms();

}  // namespace kcg
