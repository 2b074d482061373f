// Ahead-of-time sm_100a kernels (kernels.cu) and their host launchers.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

#include "kcg_devprog.h"

struct KeStmt;  // kcg_enum_dev.h

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

/// Integer-sliced Gram on the int8 tensor cores (gram_sliced.cu); false
/// when F is outside its range (17..40).
bool launch_gram_sliced(const double* X, size_t n, int F, double* G, double* xt1,
                        double* colmax, cudaStream_t stream);

/// obj += sum (1 - X alpha)^2
void launch_residual(const double* X, size_t n, int F, size_t ld,
                     const double* alpha, double* obj, void* stream);

/// g += X^T (1 - X alpha)
void launch_residual_grad(const double* X, size_t n, int F, size_t ld,
                          const double* alpha, double* g, void* stream);

struct NoiseArgs {
  const int64_t* cols[KCG_MAX_PARAMS];  // parameter columns, sorted by name
  int n_params;
  int seg_len[KCG_MAX_PARAMS];
  unsigned char seg[KCG_MAX_PARAMS][48];  // "name=" (";name=" after the first)
  uint64_t prefix_hash;                   // FNV-1a state after "kernel|"
  uint64_t seed, counter;
  double sigma;
  double* t;                              // in: noiseless, out: noisy
  int64_t n;
};

/// simulate_time's multiplicative noise (simdevice.cpp:13-46, 96-102)
void launch_noise(const NoiseArgs& a, void* stream);

/// geometric_mean_error accumulation (model.cpp:119-133)
void launch_geomean(const double* pred, const double* actual, size_t n, double* log_sum,
                    unsigned long long* count, unsigned long long* bad, void* stream);

/// GPU enumeration oracle (enum_kernels.cu): one statement walk, and the
/// popcount / min / max set bit of a bitmap (out[0] +=, out[1] min=, out[2] max=)
void launch_enum_walk(const KeStmt* dev_stmt, unsigned long long box_total, cudaStream_t stream);
void launch_enum_bits(const unsigned long long* bm, unsigned long long words, unsigned long long* out,
                      cudaStream_t stream);

/// design rows x = RN(count) / T (row-major n x F; zero rows, counted in
/// *bad, for inadmissible points or T <= 0) from prop-major exact counts
void launch_form_rows(const int64_t* lo, const int64_t* hi, const uint8_t* status, const double* T, size_t n,
                      int F, double* X, unsigned long long* bad, void* stream);

/// grid descriptor -> SoA int64 bindings
void launch_grid_fill(int np, const int64_t* start, const int64_t* step, const uint64_t* count, uint64_t first,
                      size_t n, int64_t* const* cols, void* stream);

int num_sms();
// lane operations per second of one pipe (peaks.cu: 0 IMAD, 1 LOP3, 2 DFMA,
// 3 IMAD+LOP3 issue mix); synchronous on the current device
double measure_pipe_peak(int kind, unsigned long long iters);
double measure_stream(int R, int W, unsigned long long n);

}  // namespace kcg
