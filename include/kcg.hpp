// kcg.hpp -- header-only C++ host API over the C ABI (kcg.h).
//
// This is the host side a C++ caller of the reference uses: RAII handles and
// batched overloads named after the reference API it replaces
// (proj/core/include/kernelcost):
//   kcg::Program                 <- extract_properties(k) output (props.hpp:37)
//   kcg::evaluate_properties()   <- evaluate_properties (props.hpp:49-50)
//   kcg::predict()               <- predict (model.hpp:61)
//   kcg::noiseless_time()        <- noiseless_time (simdevice.hpp:33)
//   kcg::predict_host()          <- the same over host vectors (chunked H2D / D2H inside)
//   kcg::argmin()                <- the autotuning sweep over kernel variants
//   kcg::fit_weights()           <- build_design_matrix + fit_weights
//                                   (model.hpp:43-49), Gram on the GPU
//   kcg::read_weights_json()     <- read_weights_json (jsonio.hpp:29)
//   kcg::prediction()            <- predict's Prediction{seconds, breakdown, warnings}
//   kcg::EnumProgram             <- enumerate_points (enumerate.hpp:23-24) on the GPU
//   kcg::Grid, predict_grid()    <- bulk grids from a lattice descriptor
//   kcg::Columns, write_columns  <- the kcg-columns v1 binary side format
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

/// Host-buffer predict over several programs sharing one set of bindings
/// (host_cols in programs[0]'s parameter order): returns programs x n
/// seconds, program-major. flags: KCG_HOST_PINNED for page-locked buffers.
inline std::vector<double> predict_host(const ModelWeights& w, const std::vector<const Program*>& programs,
                                        const int64_t* const* host_cols, size_t n,
                                        uint8_t* status = nullptr, unsigned flags = 0) {
  if (w.alpha.size() != static_cast<size_t>(kcg_schema_size()))
    throw Error(KCG_E_SCHEMA_MISMATCH, "weight vector does not match schema v1");
  std::vector<const kcg_program*> h;
  for (const Program* p : programs) h.push_back(p->handle());
  std::vector<double> out(programs.size() * n);
  check(kcg_eval_predict_host(h.data(), static_cast<int>(h.size()), host_cols, n, w.alpha.data(), out.data(),
                              status, flags));
  return out;
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

/// GPU enumeration oracle over a "kernelcost-enum v1" text (enum_text).
class EnumProgram {
 public:
  explicit EnumProgram(const std::string& text) { check(kcg_enum_program_create(text.data(), text.size(), &h_)); }
  EnumProgram(const EnumProgram&) = delete;
  EnumProgram& operator=(const EnumProgram&) = delete;
  ~EnumProgram() { kcg_enum_program_destroy(h_); }
  std::vector<std::string> params() const {
    std::vector<std::string> v;
    for (int i = 0; i < kcg_enum_program_num_params(h_); ++i) v.emplace_back(kcg_enum_program_param_name(h_, i));
    return v;
  }
  struct Tally {
    std::vector<__int128> counts = std::vector<__int128>(149, 0);  // schema order
    uint64_t points = 0;
  };
  /// enumerate_points at one binding (parameter declaration order)
  Tally enumerate_points(const std::vector<int64_t>& binding, uint64_t cap = 0, cudaStream_t s = nullptr) const {
    std::vector<int64_t> lo(149), hi(149);
    Tally t;
    check(kcg_enumerate_points(h_, binding.data(), cap, lo.data(), hi.data(), &t.points, s));
    for (int i = 0; i < 149; ++i)
      t.counts[i] = static_cast<__int128>((static_cast<unsigned __int128>(static_cast<uint64_t>(hi[i])) << 64) |
                                          static_cast<uint64_t>(lo[i]));
    return t;
  }

 private:
  kcg_enum_program* h_ = nullptr;
};

/// lattice of bindings: parameter j = start[j] + step[j] * d_j, last fastest
struct Grid {
  std::vector<int64_t> start, step;
  std::vector<uint64_t> count;
  kcg_grid c() const {
    kcg_grid g{};
    g.n_params = static_cast<int32_t>(start.size());
    for (size_t j = 0; j < start.size() && j < 8; ++j) {
      g.start[j] = start[j];
      g.step[j] = step[j];
      g.count[j] = count[j];
    }
    return g;
  }
};

inline void predict_grid(const ModelWeights& w, const Program& p, const Grid& grid, uint64_t first, size_t n,
                         double* seconds, uint8_t* status = nullptr, cudaStream_t s = nullptr) {
  const kcg_grid g = grid.c();
  check(kcg_eval_predict_grid(p.handle(), &g, first, n, w.alpha.data(), seconds, status, 0, s));
}

inline void grid_bindings(const Grid& grid, uint64_t first, size_t n, int64_t* const* cols, cudaStream_t s = nullptr) {
  const kcg_grid g = grid.c();
  check(kcg_grid_bindings(&g, first, n, cols, s));
}

/// a mapped kcg-columns v1 file
class Columns {
 public:
  explicit Columns(const std::string& path) { check(kcg_columns_open(path.c_str(), &h_)); }
  Columns(const Columns&) = delete;
  Columns& operator=(const Columns&) = delete;
  ~Columns() { kcg_columns_close(h_); }
  uint64_t rows() const { return kcg_columns_num_rows(h_); }
  int find(const std::string& name) const { return kcg_columns_find(h_, name.c_str()); }
  const void* data(int j) const { return kcg_columns_data(h_, j); }
  void load(int j, uint64_t row0, size_t n, void* dev, cudaStream_t s = nullptr) {
    check(kcg_columns_load(h_, j, row0, n, dev, s));
  }

 private:
  kcg_columns* h_ = nullptr;
};

inline void write_columns(const std::string& path, const std::vector<std::string>& names,
                          const std::vector<int>& dtypes, const std::vector<const void*>& host_cols,
                          uint64_t n_rows) {
  std::vector<const char*> nm;
  for (const auto& s : names) nm.push_back(s.c_str());
  check(kcg_columns_write(path.c_str(), static_cast<int>(names.size()), nm.data(), dtypes.data(),
                          host_cols.data(), n_rows));
}

/// predict's full result for one point (model.cpp:95-117) from its exact
/// counts (kcg::evaluate_properties output copied to the host: the F lo/hi
/// words of the point, program property order = schema order)
struct Prediction {
  double seconds = 0.0;
  std::vector<std::pair<std::string, double>> breakdown;
  std::vector<std::string> warnings;
};

inline Prediction prediction(const ModelWeights& w, const Program& p, const int64_t* lo, const int64_t* hi) {
  if (w.alpha.size() != static_cast<size_t>(kcg_schema_size()))
    throw Error(KCG_E_SCHEMA_MISMATCH, "weight vector does not match schema v1");
  Prediction out;
  const std::vector<int> props = p.props();
  for (size_t j = 0; j < props.size(); ++j) {
    const __int128 c = static_cast<__int128>((static_cast<unsigned __int128>(static_cast<uint64_t>(hi[j])) << 64) |
                                             static_cast<uint64_t>(lo[j]));
    if (c == 0) continue;
    const double count = static_cast<double>(c);  // round to nearest even
    const double part = w.alpha[props[j]] * count;
    out.seconds += part;
    out.breakdown.emplace_back(kcg_schema_key(props[j]), part);
    if (!w.covered[props[j]]) out.warnings.emplace_back(kcg_schema_key(props[j]));
  }
  return out;
}

}  // namespace kcg
