// kcg.hpp -- header-only C++ host API over the C ABI (kcg.h).
//
// This is the host side a C++ caller of the reference uses: RAII handles and
// batched overloads named after the reference API it replaces
// (proj/core/include/kernelcost):
//   kcg::Program                 <- extract_properties(k) output (props.hpp:37)
//   kcg::evaluate_properties()   <- evaluate_properties (props.hpp:49-50)
//   kcg::predict()               <- predict (model.hpp:61)
//   kcg::noiseless_time()        <- noiseless_time (simdevice.hpp:33)
//   kcg::argmin()                <- the autotuning sweep over kernel variants
//   kcg::fit_weights()           <- build_design_matrix + fit_weights
//                                   (model.hpp:43-49), Gram on the GPU
//   kcg::read_weights_json()     <- read_weights_json (jsonio.hpp:29)
// Errors are thrown as kcg::Error carrying the kcg_status code (1..11 ==
// kernelcost::Errc + 1). All device pointers are caller-owned.
#pragma once

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "kcg.h"

namespace kcg {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m)
      : std::runtime_error(std::string(kcg_status_str(c)) + ": " + m), code(c) {}
};

inline void check(int rc) {
  if (rc != KCG_OK) throw Error(rc, kcg_last_error());
}

inline void cuda_check(cudaError_t e) {
  if (e != cudaSuccess) throw Error(KCG_E_CUDA, cudaGetErrorString(e));
}

class Program {
 public:
  explicit Program(const std::string& text) { check(kcg_program_create(text.data(), text.size(), &h_)); }
  Program(const Program&) = delete;
  Program& operator=(const Program&) = delete;
  Program(Program&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  ~Program() { kcg_program_destroy(h_); }

  kcg_program* handle() const { return h_; }
  std::string name() const { return kcg_program_kernel_name(h_); }
  std::vector<std::string> params() const {
    std::vector<std::string> v;
    for (int i = 0; i < kcg_program_num_params(h_); ++i) v.emplace_back(kcg_program_param_name(h_, i));
    return v;
  }
  /// schema indices of the program's nonzero properties (column order of counts)
  std::vector<int> props() const {
    std::vector<int> v;
    for (int j = 0; j < kcg_program_num_props(h_); ++j) v.push_back(kcg_program_prop_schema_index(h_, j));
    return v;
  }

 private:
  kcg_program* h_ = nullptr;
};

struct ModelWeights {
  std::string device;
  std::vector<double> alpha = std::vector<double>(149, 0.0);
  std::vector<uint8_t> covered = std::vector<uint8_t>(149, 0);
  double objective = 0.0;
  uint64_t n_cases = 0;
};

inline ModelWeights read_weights_json(const std::string& path) {
  ModelWeights w;
  check(kcg_weights_read_json(path.c_str(), w.alpha.data(), w.covered.data(), &w.objective, &w.n_cases));
  return w;
}

inline void write_weights_json(const std::string& path, const ModelWeights& w) {
  check(kcg_weights_write_json(path.c_str(), w.device.c_str(), w.alpha.data(), w.covered.data(),
                               w.objective, w.n_cases));
}

/// Batched evaluate_properties: exact counts (int128 as lo/hi words,
/// prop-major [F][n]) and a status byte per binding.
inline void evaluate_properties(const Program& p, const int64_t* const* cols, size_t n,
                                int64_t* counts_lo, int64_t* counts_hi, uint8_t* status,
                                cudaStream_t s = nullptr) {
  check(kcg_eval_predict(p.handle(), cols, n, nullptr, nullptr, status, counts_lo, counts_hi, 0, s));
}

/// Batched predict: seconds per binding (NaN where status != 0).
inline void predict(const ModelWeights& w, const Program& p, const int64_t* const* cols, size_t n,
                    double* seconds, uint8_t* status = nullptr, cudaStream_t s = nullptr) {
  if (w.alpha.size() != static_cast<size_t>(kcg_schema_size()))
    throw Error(KCG_E_SCHEMA_MISMATCH, "weight vector does not match schema v1");
  check(kcg_eval_predict(p.handle(), cols, n, w.alpha.data(), seconds, status, nullptr, nullptr, 0, s));
}

/// Batched noiseless_time (simulate order: skip zero weights).
inline void noiseless_time(const std::vector<double>& alpha149, const Program& p, const int64_t* const* cols,
                           size_t n, double* seconds, cudaStream_t s = nullptr) {
  check(kcg_eval_predict(p.handle(), cols, n, alpha149.data(), seconds, nullptr, nullptr, nullptr, 1, s));
}

/// Autotuning sweep: best variant and its predicted time per size.
inline void argmin(const std::vector<const Program*>& variants, const ModelWeights& w,
                   const int64_t* const* cols, size_t n, int32_t* best, double* best_t,
                   double* preds = nullptr, cudaStream_t s = nullptr) {
  std::vector<const kcg_program*> h;
  for (const Program* v : variants) h.push_back(v->handle());
  check(kcg_argmin(h.data(), static_cast<int>(h.size()), cols, n, w.alpha.data(), best, best_t, preds, s));
}

struct FitResult {
  std::vector<double> alpha;  // one per design column
  int rank = 0;
  double objective = 0.0;
};

/// fit_weights over a materialised device design X [n x F] (rows p/T):
/// Gram on the FP64 tensor cores, host min-norm solve, `refine` semi-normal
/// refinement passes, objective from a residual pass.
inline FitResult fit_weights(const double* X, size_t n, int F, int refine = 1, cudaStream_t s = nullptr) {
  double *G, *xt1, *cm, *dalpha, *dg, *dobj;
  cuda_check(cudaMalloc(&G, sizeof(double) * (F * F + 4 * F + 1)));
  xt1 = G + F * F;
  cm = xt1 + F;
  dalpha = cm + F;
  dg = dalpha + F;
  dobj = dg + F;
  cuda_check(cudaMemsetAsync(G, 0, sizeof(double) * (F * F + 4 * F + 1), s));
  FitResult r;
  try {
    check(kcg_gram_accumulate(X, n, F, F, G, xt1, cm, s));
    std::vector<double> hG(F * F), h1(F), hm(F), hg(F);
    cuda_check(cudaMemcpyAsync(hG.data(), G, sizeof(double) * F * F, cudaMemcpyDeviceToHost, s));
    cuda_check(cudaMemcpyAsync(h1.data(), xt1, sizeof(double) * F, cudaMemcpyDeviceToHost, s));
    cuda_check(cudaMemcpyAsync(hm.data(), cm, sizeof(double) * F, cudaMemcpyDeviceToHost, s));
    cuda_check(cudaStreamSynchronize(s));
    r.alpha.assign(F, 0.0);
    check(kcg_solve_gram(F, hG.data(), h1.data(), hm.data(), r.alpha.data(), &r.rank));
    for (int it = 0; it < refine; ++it) {
      cuda_check(cudaMemcpyAsync(dalpha, r.alpha.data(), sizeof(double) * F, cudaMemcpyHostToDevice, s));
      cuda_check(cudaMemsetAsync(dg, 0, sizeof(double) * F, s));
      check(kcg_gram_residual_grad(X, n, F, F, dalpha, dg, s));
      cuda_check(cudaMemcpyAsync(hg.data(), dg, sizeof(double) * F, cudaMemcpyDeviceToHost, s));
      cuda_check(cudaStreamSynchronize(s));
      check(kcg_refine_gram(F, hG.data(), hm.data(), hg.data(), r.alpha.data()));
    }
    cuda_check(cudaMemcpyAsync(dalpha, r.alpha.data(), sizeof(double) * F, cudaMemcpyHostToDevice, s));
    check(kcg_residual_accumulate(X, n, F, F, dalpha, dobj, s));
    cuda_check(cudaMemcpyAsync(&r.objective, dobj, sizeof(double), cudaMemcpyDeviceToHost, s));
    cuda_check(cudaStreamSynchronize(s));
  } catch (...) {
    cudaFree(G);
    throw;
  }
  cudaFree(G);
  return r;
}

}  // namespace kcg
