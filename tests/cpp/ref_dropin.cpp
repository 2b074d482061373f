// The reference-side drop-in, compiled for real: the reference's own
// front end (parse_kernel, extract_properties, suite, campaign, fit) from
// oracle/_ref/libkernelcost_ref.a (the reference sources built in place)
// calls the GPU through tests/cpp/kernelcost_gpu.hpp
// and libkcg.so, in one process, and compares against the reference's own
// scalar calls:
//   * every symbolic suite kernel: Program(k) from program_text; all 406
//     manifest cases (suite.cpp) -- evaluate_properties_batch counts ==
//     evaluate_properties / extract_properties (bound) counts on all 149
//     keys, predict_batch == predict(w, bound).seconds bitwise, and an
//     inadmissible binding's status byte == the Errc the reference throws;
//   * predict_batch_host over the six matmul variants (one call, host
//     vectors) == per-point predict;
//   * fit_weights_gram over the simulated campaign of the 390 measurement
//     cases (run_campaign, sigma 0) vs fit_weights(build_design_matrix(..))
//     (model.cpp:11-93): weights within 1e-9 (equilibrated coordinates,
//     absolute 1e-13 for numerically-zero weights), objective to 1e-6.
// Prints one JSON object; exit code 0 iff every check passed.
//   ref_dropin
#include <cstdio>
#include <cstring>
#include <memory>
#include <map>
#include <random>
#include <set>
#include <string>
#include <vector>

#include "../../oracle/kcref_program.hpp"
#include "kernelcost/campaign.hpp"
#include "kernelcost/parser.hpp"
#include "kernelcost/simdevice.hpp"
#include "kernelcost/suite.hpp"
#include "kernelcost_gpu.hpp"

namespace kc = kernelcost;
namespace gpu = kernelcost::gpu;

std::string kernelcost::gpu::program_text(const KernelIR& k, const PropertyVector& pv) {
  return kcref::program_text(k, pv);
}

namespace {

__int128 to_i128(const kc::Rat& r) {
  const std::string s = boost::multiprecision::numerator(r).str();
  __int128 v = 0;
  size_t i = s[0] == '-' ? 1 : 0;
  for (; i < s.size(); ++i) v = v * 10 + (s[i] - '0');
  return s[0] == '-' ? -v : v;
}

struct DevCols {  // SoA int64 device columns in a Program's params() order
  std::vector<int64_t*> cols;
  std::vector<const int64_t*> ccols;
  DevCols(const gpu::Program& p, const std::vector<kc::Binding>& bs) {
    const auto names = p.params();
    for (const auto& nm : names) {
      std::vector<int64_t> h;
      for (const auto& b : bs) h.push_back(static_cast<int64_t>(b.at(nm)));
      int64_t* d = nullptr;
      gpu::cuda(cudaMalloc(&d, sizeof(int64_t) * std::max<size_t>(1, h.size())));
      gpu::cuda(cudaMemcpy(d, h.data(), sizeof(int64_t) * h.size(), cudaMemcpyHostToDevice));
      cols.push_back(d);
      ccols.push_back(d);
    }
  }
  ~DevCols() {
    for (auto* d : cols) cudaFree(d);
  }
};

}  // namespace

int main() {
  const kc::SuiteLibrary lib = kc::build_suite();
  const kc::SimDevice dev = kc::SimDevice::reference();
  kc::ModelWeights w;
  w.device = dev.name;
  w.schema_version = kc::kSchemaVersion;
  w.alpha = dev.alpha;
  w.covered.assign(kc::schema_size(), true);
  const kc::Int cap(20000000);
  std::vector<kc::SuiteCase> cases = lib.measurement_cases();
  for (const auto& c : lib.test_cases()) cases.push_back(c);

  std::map<std::string, kc::KernelIR> irs;
  std::map<std::string, kc::PropertyVector> syms;
  std::map<std::string, std::unique_ptr<gpu::Program>> progs;
  std::set<std::string> non_symbolic;
  long n_cases = 0, n_checked = 0, count_mismatch = 0, pred_mismatch = 0, err_mismatch = 0;
  std::map<std::string, std::vector<kc::Binding>> by_kernel;
  for (const auto& c : cases) by_kernel[c.kernel_id].push_back(c.binding);
  for (auto& [id, bs] : by_kernel) {
    const kc::KernelIR& k = irs.emplace(id, kc::parse_kernel(lib.find(id)->text)).first->second;
    try {
      syms[id] = kc::extract_properties(k);
    } catch (const kc::Error& e) {
      if (e.code() != kc::Errc::needs_binding) throw;
      non_symbolic.insert(id);
      n_cases += static_cast<long>(bs.size());
      continue;
    }
    progs[id] = std::make_unique<gpu::Program>(k, syms[id]);
    const gpu::Program& p = *progs[id];
    // plus one inadmissible binding (every parameter + 1) per kernel
    std::vector<kc::Binding> all = bs;
    kc::Binding bad = bs[0];
    for (auto& [nm, v] : bad) v = v + 1;
    all.push_back(bad);
    const size_t n = all.size(), F = p.keys.size();
    DevCols dc(p, all);
    double* dpred;
    uint8_t* dst;
    int64_t *dlo, *dhi;
    gpu::cuda(cudaMalloc(&dpred, sizeof(double) * n));
    gpu::cuda(cudaMalloc(&dst, n));
    gpu::cuda(cudaMalloc(&dlo, sizeof(int64_t) * F * n));
    gpu::cuda(cudaMalloc(&dhi, sizeof(int64_t) * F * n));
    gpu::predict_batch(p, w, dc.ccols.data(), n, dpred, dst);
    gpu::evaluate_properties_batch(p, dc.ccols.data(), n, dlo, dhi, nullptr);
    gpu::cuda(cudaDeviceSynchronize());
    std::vector<double> pred(n);
    std::vector<uint8_t> st(n);
    std::vector<int64_t> lo(F * n), hi(F * n);
    gpu::cuda(cudaMemcpy(pred.data(), dpred, sizeof(double) * n, cudaMemcpyDeviceToHost));
    gpu::cuda(cudaMemcpy(st.data(), dst, n, cudaMemcpyDeviceToHost));
    gpu::cuda(cudaMemcpy(lo.data(), dlo, sizeof(int64_t) * F * n, cudaMemcpyDeviceToHost));
    gpu::cuda(cudaMemcpy(hi.data(), dhi, sizeof(int64_t) * F * n, cudaMemcpyDeviceToHost));
    cudaFree(dpred);
    cudaFree(dst);
    cudaFree(dlo);
    cudaFree(dhi);
    for (size_t i = 0; i < n; ++i) {
      kc::PropertyVector bound;
      int ref_st = 0;
      try {
        bound = kc::evaluate_properties(k, syms[id], all[i]);
      } catch (const kc::Error& e) {
        ref_st = static_cast<int>(e.code()) + 1;  // Errc + 1 == kcg_status
      }
      if (i + 1 < n) ++n_cases;
      ++n_checked;
      if (ref_st != 0) {  // the per-point status byte says the same
        if (!(ref_st == KCG_E_ASSUMPTION_VIOLATED && st[i] == KCG_PT_ASSUMPTION_VIOLATED && pred[i] != pred[i]))
          ++err_mismatch;
        continue;
      }
      if (st[i] != KCG_PT_OK) {
        ++err_mismatch;
        continue;
      }
      std::vector<__int128> gpu_counts(kc::schema_size(), 0);
      for (size_t j = 0; j < F; ++j)
        gpu_counts[p.keys[j]] = static_cast<__int128>(
            (static_cast<unsigned __int128>(static_cast<uint64_t>(hi[j * n + i])) << 64) |
            static_cast<uint64_t>(lo[j * n + i]));
      for (size_t key = 0; key < kc::schema_size(); ++key) {
        const auto& e = bound.entries[key];
        const __int128 want = e.is_zero() ? 0 : to_i128(e.constant_value());
        if (want != gpu_counts[key]) ++count_mismatch;
      }
      const double want = kc::predict(w, bound).seconds;
      if (std::memcmp(&want, &pred[i], 8) != 0) ++pred_mismatch;
    }
  }

  // predict_batch_host: the six matmul variants over one host binding set
  const std::vector<std::string> vids = {"matmul_tiled_g12x12", "matmul_tiled_g14x14", "matmul_tiled_g16x16",
                                         "matmul_naive_g16x12", "matmul_naive_g16x14", "matmul_naive_g16x16"};
  std::vector<const gpu::Program*> vps;
  for (const auto& id : vids) {
    if (!progs.count(id)) {
      irs.emplace(id, kc::parse_kernel(lib.find(id)->text));
      syms[id] = kc::extract_properties(irs.at(id));
      progs[id] = std::make_unique<gpu::Program>(irs.at(id), syms[id]);
    }
    vps.push_back(progs[id].get());
  }
  std::mt19937_64 rng(7);
  const auto names = vps[0]->params();
  std::vector<std::vector<int64_t>> hcols(names.size());
  std::vector<kc::Binding> hb;
  for (int i = 0; i < 5000; ++i) {
    kc::Binding b;
    for (size_t j = 0; j < names.size(); ++j) {
      const int64_t v = 48 * static_cast<int64_t>(1 + rng() % 300) + (i % 41 == 0 ? 1 : 0);
      b[names[j]] = kc::Int(v);
      hcols[j].push_back(v);
    }
    hb.push_back(b);
  }
  std::vector<uint8_t> hst;
  const std::vector<double> hp = gpu::predict_batch_host(vps, w, hcols, &hst);
  long host_mismatch = 0, host_points = 0;
  for (size_t v = 0; v < vps.size(); ++v)
    for (size_t i = 0; i < hb.size(); ++i) {
      ++host_points;
      double want;
      try {
        want = kc::predict(w, kc::evaluate_properties(irs.at(vids[v]), syms[vids[v]], hb[i])).seconds;
      } catch (const kc::Error&) {
        if (hst[v * hb.size() + i] != KCG_PT_ASSUMPTION_VIOLATED) ++host_mismatch;
        continue;
      }
      if (std::memcmp(&want, &hp[v * hb.size() + i], 8) != 0) ++host_mismatch;
    }

  // fit_weights_gram vs the reference fit over the simulated campaign
  const kc::CampaignResult cr = kc::run_campaign(dev, lib, lib.measurement_cases(), cap);
  std::vector<kc::FitCase> fcases;
  std::map<std::string, std::vector<std::pair<kc::Binding, double>>> rows;
  for (const auto& r : cr.records) {
    if (!irs.count(r.kernel)) irs.emplace(r.kernel, kc::parse_kernel(lib.find(r.kernel)->text));
    fcases.push_back({kc::extract_properties(irs.at(r.kernel), r.binding, cap), r.time_s});
    rows[r.kernel].push_back({r.binding, r.time_s});
  }
  const kc::DesignMatrix dm = kc::build_design_matrix(fcases);
  const auto [wref, repref] = kc::fit_weights(dm, dev.name);
  std::vector<std::unique_ptr<DevCols>> keep;
  std::vector<double*> tbufs;
  std::vector<gpu::GramRows> parts;
  for (auto& [id, rs] : rows) {
    if (!progs.count(id)) {
      syms[id] = kc::extract_properties(irs.at(id));
      progs[id] = std::make_unique<gpu::Program>(irs.at(id), syms[id]);
    }
    std::vector<kc::Binding> bs;
    std::vector<double> ts;
    for (auto& [b, t] : rs) {
      bs.push_back(b);
      ts.push_back(t);
    }
    keep.push_back(std::make_unique<DevCols>(*progs[id], bs));
    double* dt = nullptr;
    gpu::cuda(cudaMalloc(&dt, sizeof(double) * ts.size()));
    gpu::cuda(cudaMemcpy(dt, ts.data(), sizeof(double) * ts.size(), cudaMemcpyHostToDevice));
    tbufs.push_back(dt);
    parts.push_back({progs[id].get(), keep.back()->ccols.data(), dt, ts.size()});
  }
  const auto [wg, repg] = gpu::fit_weights_gram(parts, dev.name);
  double fit_worst = 0.0;  // per-weight error in units of the tolerance (<= 1 passes)
  long cov_mismatch = 0;
  for (size_t j = 0; j < kc::schema_size(); ++j) {
    if (wg.covered[j] != wref.covered[j]) ++cov_mismatch;
    double cm = 0.0;
    for (const auto& row : dm.rows) cm = std::max(cm, std::fabs(row[j]));
    if (cm == 0.0) {
      if (wg.alpha[j] != 0.0) ++cov_mismatch;
      continue;
    }
    const double tol = 1e-9 * std::fabs(wref.alpha[j]) + 1e-13 / cm;
    fit_worst = std::max(fit_worst, std::fabs(wg.alpha[j] - wref.alpha[j]) / tol);
  }
  for (double* t : tbufs) cudaFree(t);
  const double obj_rel = std::fabs(wg.objective - wref.objective) / std::max(1e-300, std::fabs(wref.objective));
  const bool ok = count_mismatch == 0 && pred_mismatch == 0 && err_mismatch == 0 && host_mismatch == 0 &&
                  fit_worst <= 1.0 && cov_mismatch == 0 && (obj_rel <= 1e-6 || wg.objective < 1e-25);
  std::printf("{\"symbolic_kernels\": %zu, \"non_symbolic_kernels\": %zu, \"manifest_cases\": %ld, "
              "\"gpu_checked_points\": %ld, \"count_mismatches\": %ld, \"prediction_mismatches\": %ld, "
              "\"status_mismatches\": %ld, \"host_batch_points\": %ld, \"host_batch_mismatches\": %ld, "
              "\"fit_cases\": %zu, \"fit_worst_in_tolerance_units\": %.3g, \"fit_covered_mismatches\": %ld, "
              "\"fit_objective_ref\": %.6g, \"fit_objective_gpu\": %.6g, \"ok\": %s}\n",
              progs.size(), non_symbolic.size(), n_cases, n_checked, count_mismatch, pred_mismatch, err_mismatch,
              host_points, host_mismatch, fcases.size(), fit_worst, cov_mismatch, wref.objective, wg.objective,
              ok ? "true" : "false");
  return ok ? 0 : 1;
}
