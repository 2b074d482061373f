// C++ host-side driver of the kcg back end through include/kcg.hpp -- the
// path a C++ caller of the reference takes (no Python, no PyTorch).
//
//   kcg_host_driver eval <program.kcp> <weights.json> <bindings.bin> <out.bin>
//     bindings.bin: int64 n, int64 P, then P columns of n int64 (SoA)
//     out.bin:      n fp64 predictions, n status bytes, F*n int64 count low
//                   words, F*n int64 high words
//   kcg_host_driver grid <program.kcp> <weights.json> <dir>
//     predicts a lattice through kcg::predict_grid and through
//     kcg::grid_bindings -> kcg::Columns (a kcg-columns file round trip) ->
//     kcg::predict; prints "grid ok" when the two agree bitwise
//   kcg_host_driver enum <program.kce> <n>
//     kcg::EnumProgram::enumerate_points at every parameter = n; prints the
//     visited points and the nonzero counts
//   kcg_host_driver fit <X.bin> <out.bin>
//     X.bin: int64 n, int64 F, then n*F fp64 row-major; out: F fp64 alpha,
//     int64 rank, fp64 objective
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <vector>

#include "../../include/kcg.hpp"

static std::vector<char> slurp(const char* path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error(std::string("cannot open ") + path);
  return std::vector<char>(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
}

int eval(int argc, char** argv) {
  if (argc != 6) return 2;
  const std::vector<char> prog_text = slurp(argv[2]);
  kcg::Program prog(std::string(prog_text.begin(), prog_text.end()));
  const kcg::ModelWeights w = kcg::read_weights_json(argv[3]);
  const std::vector<char> raw = slurp(argv[4]);
  const int64_t* hdr = reinterpret_cast<const int64_t*>(raw.data());
  const int64_t n = hdr[0], P = hdr[1];
  if (P != static_cast<int64_t>(prog.params().size())) throw std::runtime_error("param count mismatch");
  const int F = static_cast<int>(prog.props().size());
  int64_t* dcols = nullptr;
  kcg::cuda_check(cudaMalloc(&dcols, sizeof(int64_t) * P * n));
  kcg::cuda_check(cudaMemcpy(dcols, hdr + 2, sizeof(int64_t) * P * n, cudaMemcpyHostToDevice));
  std::vector<const int64_t*> cols;
  for (int64_t j = 0; j < P; ++j) cols.push_back(dcols + j * n);
  double* dpred;
  uint8_t* dst;
  int64_t *dlo, *dhi;
  kcg::cuda_check(cudaMalloc(&dpred, sizeof(double) * n));
  kcg::cuda_check(cudaMalloc(&dst, n));
  kcg::cuda_check(cudaMalloc(&dlo, sizeof(int64_t) * F * n));
  kcg::cuda_check(cudaMalloc(&dhi, sizeof(int64_t) * F * n));
  kcg::predict(w, prog, cols.data(), n, dpred, dst);
  kcg::evaluate_properties(prog, cols.data(), n, dlo, dhi, nullptr);
  kcg::cuda_check(cudaDeviceSynchronize());
  std::vector<double> pred(n);
  std::vector<uint8_t> st(n);
  std::vector<int64_t> lo(F * n), hi(F * n);
  kcg::cuda_check(cudaMemcpy(pred.data(), dpred, sizeof(double) * n, cudaMemcpyDeviceToHost));
  kcg::cuda_check(cudaMemcpy(st.data(), dst, n, cudaMemcpyDeviceToHost));
  kcg::cuda_check(cudaMemcpy(lo.data(), dlo, sizeof(int64_t) * F * n, cudaMemcpyDeviceToHost));
  kcg::cuda_check(cudaMemcpy(hi.data(), dhi, sizeof(int64_t) * F * n, cudaMemcpyDeviceToHost));
  // the host-side Prediction of every admissible point == the GPU prediction
  int64_t mismatch = 0;
  std::vector<int64_t> plo(F), phi(F);
  for (int64_t i = 0; i < n; ++i) {
    if (st[i] != 0) continue;
    for (int j = 0; j < F; ++j) {
      plo[j] = lo[j * n + i];
      phi[j] = hi[j * n + i];
    }
    const kcg::Prediction pd = kcg::prediction(w, prog, plo.data(), phi.data());
    if (std::memcmp(&pd.seconds, &pred[i], 8) != 0) ++mismatch;
  }
  if (mismatch) {
    std::cout << "prediction mismatch: " << mismatch << "\n";
    return 1;
  }
  // the host-buffer entry point (pageable vectors) == the device path
  std::vector<const int64_t*> hcols;
  for (int64_t j = 0; j < P; ++j) hcols.push_back(hdr + 2 + j * n);
  std::vector<uint8_t> hst(n);
  const std::vector<double> hpred = kcg::predict_host(w, {&prog}, hcols.data(), n, hst.data());
  if (std::memcmp(hpred.data(), pred.data(), sizeof(double) * n) != 0 || hst != st) {
    std::cout << "predict_host differs from the device path\n";
    return 1;
  }
  std::ofstream out(argv[5], std::ios::binary);
  out.write(reinterpret_cast<const char*>(pred.data()), sizeof(double) * n);
  out.write(reinterpret_cast<const char*>(st.data()), n);
  out.write(reinterpret_cast<const char*>(lo.data()), sizeof(int64_t) * F * n);
  out.write(reinterpret_cast<const char*>(hi.data()), sizeof(int64_t) * F * n);
  cudaFree(dcols);
  cudaFree(dpred);
  cudaFree(dst);
  cudaFree(dlo);
  cudaFree(dhi);
  std::cout << "eval ok: " << prog.name() << " n=" << n << " F=" << F << "\n";
  return 0;
}

int grid(int argc, char** argv) {
  if (argc != 5) return 2;
  const std::vector<char> prog_text = slurp(argv[2]);
  kcg::Program prog(std::string(prog_text.begin(), prog_text.end()));
  const kcg::ModelWeights w = kcg::read_weights_json(argv[3]);
  const size_t P = prog.params().size();
  kcg::Grid g;
  for (size_t j = 0; j < P; ++j) {
    g.start.push_back(16 * static_cast<int64_t>(j + 1));
    g.step.push_back(16);
    g.count.push_back(40 + j);
  }
  size_t n = 1;
  for (auto c : g.count) n *= c;
  double *dp1, *dp2;
  int64_t* dcols;
  kcg::cuda_check(cudaMalloc(&dp1, sizeof(double) * n));
  kcg::cuda_check(cudaMalloc(&dp2, sizeof(double) * n));
  kcg::cuda_check(cudaMalloc(&dcols, sizeof(int64_t) * n * P));
  std::vector<int64_t*> cols;
  for (size_t j = 0; j < P; ++j) cols.push_back(dcols + j * n);
  kcg::predict_grid(w, prog, g, 0, n, dp1);
  kcg::grid_bindings(g, 0, n, cols.data());
  // through the side format: device -> host -> file -> mapped -> device
  std::vector<int64_t> host(n * P);
  kcg::cuda_check(cudaMemcpy(host.data(), dcols, sizeof(int64_t) * n * P, cudaMemcpyDeviceToHost));
  std::vector<std::string> names = prog.params();
  std::vector<int> dts(P, KCG_COL_INT64);
  std::vector<const void*> hc;
  for (size_t j = 0; j < P; ++j) hc.push_back(host.data() + j * n);
  const std::string path = std::string(argv[4]) + "/bindings.kcgcol";
  kcg::write_columns(path, names, dts, hc, n);
  kcg::cuda_check(cudaMemset(dcols, 0, sizeof(int64_t) * n * P));
  {
    kcg::Columns c(path);
    for (size_t j = 0; j < P; ++j) c.load(c.find(names[j]), 0, n, cols[j]);
  }
  kcg::predict(w, prog, reinterpret_cast<const int64_t* const*>(cols.data()), n, dp2);
  kcg::cuda_check(cudaDeviceSynchronize());
  std::vector<double> a(n), b(n);
  kcg::cuda_check(cudaMemcpy(a.data(), dp1, sizeof(double) * n, cudaMemcpyDeviceToHost));
  kcg::cuda_check(cudaMemcpy(b.data(), dp2, sizeof(double) * n, cudaMemcpyDeviceToHost));
  cudaFree(dp1);
  cudaFree(dp2);
  cudaFree(dcols);
  for (size_t i = 0; i < n; ++i)
    if (std::memcmp(&a[i], &b[i], 8) != 0) {
      std::cout << "grid mismatch at " << i << "\n";
      return 1;
    }
  std::cout << "grid ok: " << prog.name() << " n=" << n << "\n";
  return 0;
}

int enumerate(int argc, char** argv) {
  if (argc != 4) return 2;
  const std::vector<char> text = slurp(argv[2]);
  kcg::EnumProgram ep(std::string(text.begin(), text.end()));
  std::vector<int64_t> b(ep.params().size(), std::atoll(argv[3]));
  const kcg::EnumProgram::Tally t = ep.enumerate_points(b);
  std::cout << "points " << t.points << "\n";
  for (int i = 0; i < 149; ++i)
    if (t.counts[i]) std::cout << kcg_schema_key(i) << " " << static_cast<long long>(t.counts[i]) << "\n";
  return 0;
}

int fit(int argc, char** argv) {
  if (argc != 4) return 2;
  const std::vector<char> raw = slurp(argv[2]);
  const int64_t* hdr = reinterpret_cast<const int64_t*>(raw.data());
  const int64_t n = hdr[0], F = hdr[1];
  double* dX;
  kcg::cuda_check(cudaMalloc(&dX, sizeof(double) * n * F));
  kcg::cuda_check(cudaMemcpy(dX, hdr + 2, sizeof(double) * n * F, cudaMemcpyHostToDevice));
  const kcg::FitResult r = kcg::fit_weights(dX, n, static_cast<int>(F), 1);
  cudaFree(dX);
  std::ofstream out(argv[3], std::ios::binary);
  out.write(reinterpret_cast<const char*>(r.alpha.data()), sizeof(double) * F);
  const int64_t rank = r.rank;
  out.write(reinterpret_cast<const char*>(&rank), sizeof rank);
  out.write(reinterpret_cast<const char*>(&r.objective), sizeof(double));
  std::cout << "fit ok: F=" << F << " rank=" << r.rank << " objective=" << r.objective << "\n";
  return 0;
}

int main(int argc, char** argv) {
  try {
    if (argc > 1 && std::string(argv[1]) == "eval") return eval(argc, argv);
    if (argc > 1 && std::string(argv[1]) == "fit") return fit(argc, argv);
    if (argc > 1 && std::string(argv[1]) == "grid") return grid(argc, argv);
    if (argc > 1 && std::string(argv[1]) == "enum") return enumerate(argc, argv);
    std::cerr << "usage: kcg_host_driver eval|fit|grid|enum ...\n";
    return 2;
  } catch (const kcg::Error& e) {
    std::cerr << "kcg error: " << e.what() << "\n";
    return 3;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 4;
  }
}
