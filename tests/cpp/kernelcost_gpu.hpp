// Reference-side drop-in: the batched overloads a
// kernelcost maintainer adds next to evaluate_properties (props.hpp:49-50),
// predict (model.hpp:61) and fit_weights (model.hpp:48-49). The scalar
// signatures stay as they are; these take many bindings at once and run on
// the B200 through this repo's C ABI (include/kcg.h). Header-only; compiled
// against the reference's own headers and linked with libkcg.so by
// tests/cpp/ref_dropin.cpp (oracle/Makefile target _ref/ref_dropin).
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <string>
#include <utility>
#include <vector>

#include "../../include/kcg.h"
#include "kernelcost/error.hpp"
#include "kernelcost/ir.hpp"
#include "kernelcost/model.hpp"
#include "kernelcost/props.hpp"
#include "kernelcost/schema.hpp"

namespace kernelcost::gpu {

// kcg_status 1..11 are Errc + 1 (error.hpp:10-22 order); 100+ are the
// GPU-side codes (CUDA, JIT, unsupported, internal): invalid_argument here
inline void check(int rc) {
  if (rc == KCG_OK) return;
  if (rc >= 1 && rc <= 11) throw Error(static_cast<Errc>(rc - 1), kcg_last_error());
  throw Error(Errc::invalid_argument, std::string("kcg: ") + kcg_last_error());
}

inline void cuda(cudaError_t e) {
  if (e != cudaSuccess) throw Error(Errc::invalid_argument, cudaGetErrorString(e));
}

// the hand-off text of a symbolic PropertyVector (oracle/kcref_program.hpp
// program_text: params, assume constraints, nonzero entries, each printed
// with the reference's own str())
std::string program_text(const KernelIR& k, const PropertyVector& pv);

struct Program {  // one per kernel, reused for every grid
  kcg_program* h = nullptr;
  std::vector<int> keys;  // schema index of each of the program's counts
  explicit Program(const KernelIR& k) : Program(k, extract_properties(k)) {}  // symbolic extraction on the host
  Program(const KernelIR& k, const PropertyVector& symbolic) {
    const std::string t = program_text(k, symbolic);
    check(kcg_program_create(t.data(), t.size(), &h));
    for (int j = 0; j < kcg_program_num_props(h); ++j) keys.push_back(kcg_program_prop_schema_index(h, j));
  }
  Program(const Program&) = delete;
  Program& operator=(const Program&) = delete;
  ~Program() { kcg_program_destroy(h); }
  std::vector<std::string> params() const {
    std::vector<std::string> p;
    for (int i = 0; i < kcg_program_num_params(h); ++i) p.push_back(kcg_program_param_name(h, i));
    return p;
  }
};

inline void check_weights(const ModelWeights& w) {  // model.cpp:96-100
  if (w.schema_version != kSchemaVersion || w.alpha.size() != schema_size())
    throw Error(Errc::schema_mismatch, "weights schema");
}

// evaluate_properties + predict over n bindings (DEVICE SoA columns in
// Program::params() order). status[i] != 0 replaces the per-call
// E_ASSUMPTION_VIOLATED exception (props.cpp:264-266); pred[i] is NaN there.
inline void predict_batch(const Program& p, const ModelWeights& w, const int64_t* const* cols, size_t n,
                          double* pred, uint8_t* status, cudaStream_t s = nullptr) {
  check_weights(w);
  check(kcg_eval_predict(p.h, cols, n, w.alpha.data(), pred, status, nullptr, nullptr, /*simulate=*/0, s));
}

// Exact counts: lo / hi words of each count as int128, prop-major [keys][n]
inline void evaluate_properties_batch(const Program& p, const int64_t* const* cols, size_t n, int64_t* lo,
                                      int64_t* hi, uint8_t* status, cudaStream_t s = nullptr) {
  check(kcg_eval_predict(p.h, cols, n, nullptr, nullptr, status, lo, hi, 0, s));
}

// The same over HOST vectors -- the reference's own layout -- for every
// variant of a sweep in one call (each binding crosses PCIe once; the
// library overlaps H2D, one multi-variant kernel per chunk and D2H).
// cols follow ps[0]'s params(); returns variants x n predictions.
inline std::vector<double> predict_batch_host(const std::vector<const Program*>& ps, const ModelWeights& w,
                                              const std::vector<std::vector<int64_t>>& cols,
                                              std::vector<uint8_t>* status = nullptr) {
  check_weights(w);
  const size_t n = cols.empty() ? 0 : cols[0].size();
  std::vector<const kcg_program*> hs;
  for (const Program* p : ps) hs.push_back(p->h);
  std::vector<const int64_t*> c;
  for (const auto& v : cols) c.push_back(v.data());
  std::vector<double> pred(ps.size() * n);
  if (status) status->resize(ps.size() * n);
  check(kcg_eval_predict_host(hs.data(), static_cast<int>(hs.size()), c.data(), n, w.alpha.data(), pred.data(),
                              status ? status->data() : nullptr, 0));
  return pred;
}

// fit_weights (model.cpp:37-93) over measurements of several kernels, rows
// never materialised: per program the fused evaluate -> row -> Gram kernel
// over its bindings + measured times (DEVICE), scattered into the schema-
// wide statistics (rows of different kernels are disjoint), the host
// equilibrated minimum-norm solve, `refine` refinement steps with the
// double-double residual gradient over the reference's own rows, and the
// objective from a residual pass.
struct GramRows {
  const Program* p;
  const int64_t* const* cols;
  const double* T;
  size_t n;
};

inline std::pair<ModelWeights, FitReport> fit_weights_gram(const std::vector<GramRows>& parts,
                                                           const std::string& device, int refine = 2,
                                                           cudaStream_t s = nullptr) {
  const size_t K = schema_size();
  std::vector<double> G(K * K, 0.0), xt1(K, 0.0), cmax(K, 0.0);
  size_t rows = 0;
  double* d = nullptr;
  unsigned long long* bad = nullptr;
  cuda(cudaMalloc(&d, sizeof(double) * (K * K + 2 * K)));
  cuda(cudaMalloc(&bad, sizeof(unsigned long long)));
  std::vector<double> h(K * K + 2 * K);
  for (const GramRows& r : parts) {
    const size_t F = r.p->keys.size();
    cuda(cudaMemsetAsync(d, 0, sizeof(double) * (F * F + 2 * F), s));
    cuda(cudaMemsetAsync(bad, 0, sizeof(unsigned long long), s));
    check(kcg_gram_fused(r.p->h, r.cols, r.T, r.n, d, d + F * F, d + F * F + F, bad, s));
    unsigned long long nbad = 0;
    cuda(cudaMemcpyAsync(h.data(), d, sizeof(double) * (F * F + 2 * F), cudaMemcpyDeviceToHost, s));
    cuda(cudaMemcpyAsync(&nbad, bad, sizeof nbad, cudaMemcpyDeviceToHost, s));
    cuda(cudaStreamSynchronize(s));
    if (nbad) throw Error(Errc::assumption_violated, "inadmissible measurement rows");
    for (size_t a = 0; a < F; ++a) {
      const int ka = r.p->keys[a];
      for (size_t b = 0; b < F; ++b) G[ka * K + r.p->keys[b]] += h[a * F + b];
      xt1[ka] += h[F * F + a];
      cmax[ka] = std::max(cmax[ka], h[F * F + F + a]);
    }
    rows += r.n;
  }
  if (rows == 0) throw Error(Errc::empty_input, "no fit cases");
  std::vector<double> alpha(K, 0.0);
  int rank = 0;
  check(kcg_solve_gram(static_cast<int>(K), G.data(), xt1.data(), cmax.data(), alpha.data(), &rank));
  for (int it = 0; it < refine; ++it) {
    std::vector<double> g(K, 0.0);
    for (const GramRows& r : parts) {
      const size_t F = r.p->keys.size();
      cuda(cudaMemsetAsync(d, 0, sizeof(double) * F, s));
      check(kcg_residual_grad_fused(r.p->h, r.cols, r.T, r.n, alpha.data(), d, s));
      cuda(cudaMemcpyAsync(h.data(), d, sizeof(double) * F, cudaMemcpyDeviceToHost, s));
      cuda(cudaStreamSynchronize(s));
      for (size_t a = 0; a < F; ++a) g[r.p->keys[a]] += h[a];
    }
    check(kcg_refine_gram(static_cast<int>(K), G.data(), cmax.data(), g.data(), alpha.data()));
  }
  double obj = 0.0;
  for (const GramRows& r : parts) {
    cuda(cudaMemsetAsync(d, 0, sizeof(double), s));
    check(kcg_residual_fused(r.p->h, r.cols, r.T, r.n, alpha.data(), d, s));
    double o = 0;
    cuda(cudaMemcpyAsync(&o, d, sizeof o, cudaMemcpyDeviceToHost, s));
    cuda(cudaStreamSynchronize(s));
    obj += o;
  }
  cudaFree(d);
  cudaFree(bad);
  ModelWeights w;
  w.device = device;
  w.schema_version = kSchemaVersion;
  w.alpha = alpha;
  w.covered.assign(K, false);
  FitReport rep;
  for (size_t j = 0; j < K; ++j) {
    w.covered[j] = cmax[j] > 0.0;
    if (!w.covered[j]) rep.uncovered.push_back(schema_keys()[j]);
  }
  w.objective = rep.objective = obj;
  w.n_cases = rows;
  return {w, rep};
}

}  // namespace kernelcost::gpu
