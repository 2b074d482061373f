// C++ host-side driver of the kcg back end through include/kcg.hpp -- the
// path a C++ caller of the reference takes (no Python, no PyTorch).
//
//   kcg_host_driver eval <program.kcp> <weights.json> <bindings.bin> <out.bin>
//     bindings.bin: int64 n, int64 P, then P columns of n int64 (SoA)
//     out.bin:      n fp64 predictions, n status bytes, F*n int64 count low
//                   words, F*n int64 high words
//   kcg_host_driver fit <X.bin> <out.bin>
//     X.bin: int64 n, int64 F, then n*F fp64 row-major; out: F fp64 alpha,
//     int64 rank, fp64 objective
#include <cstdio>
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
    std::cerr << "usage: kcg_host_driver eval|fit ...\n";
    return 2;
  } catch (const kcg::Error& e) {
    std::cerr << "kcg error: " << e.what() << "\n";
    return 3;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 4;
  }
}
