// ORACLE TEST INFRASTRUCTURE -- CPU timing of the reference's own hot path.
//
// Runs the reference library (compiled in place from /root/reference against
// oracle/shim: "reference code + shim bigint/COD") exactly as
// proj/benchmarks/bench.cpp:47-56 does -- symbolic extract_properties once per
// kernel, then per binding evaluate_properties + predict -- fanned out over
// std::thread workers (safe after single-threaded extraction).
//
//   kcref_bench autotune <threads> <n_sizes> [offset]
//       the 6 matmul variants at (n,m,l) = 336*(u,v,w), u,v,w in [1,551],
//       sizes enumerated in the GPU bench's order from `offset`
//   kcref_bench suite <threads> <n_points>
//       config 2: skinny (16u,128u,16u) and conv n=16u, u = 1..n/2
//   kcref_bench fit <n_rows> <n_cols>
//       config 3 shape through the reference API: test_model.cpp-style
//       synthetic FitCases (counts U{1..10000}, seed 4242, T = sum alpha c
//       over the 16 simdev-v1 weights + log-uniform extras), then
//       build_design_matrix + fit_weights (model.cpp:11-93); rows/s
//   kcref_bench config1
//       config 1 through the reference API, as the CLI runs it: the
//       simulate campaign over the 390 measurement cases (run_campaign,
//       sigma 0), fit (bound extract_properties per record,
//       build_design_matrix, fit_weights), eval of the 16 test cases
//       (extract + predict); seconds per phase, 1 thread
//   kcref_bench enumerate <kernel_id> <n>
//       enumerate_points (enumerate.cpp:371-456) at the binding n (every
//       parameter = n), single-threaded like the reference; visited points/s
// Prints one JSON object: points, seconds, points_per_s, threads, checksum.
#include <atomic>
#include <map>
#include <cmath>
#include <random>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#include "kernelcost/campaign.hpp"
#include "kernelcost/enumerate.hpp"
#include "kernelcost/model.hpp"
#include "kernelcost/parser.hpp"
#include "kernelcost/props.hpp"
#include "kernelcost/simdevice.hpp"
#include "kernelcost/suite.hpp"

namespace kc = kernelcost;

namespace {

struct Kern {
  kc::KernelIR ir;
  kc::PropertyVector sym;
};

}  // namespace

int main(int argc, char** argv) {
  if (argc < 4 && !(argc == 2 && std::string(argv[1]) == "config1")) {
    std::fprintf(stderr, "usage: kcref_bench autotune|suite <threads> <n> [offset] | config1 | fit <rows> <cols> | enumerate <id> <n>\n");
    return 2;
  }
  const std::string mode = argv[1];
  if (mode == "config1") {
    using clk = std::chrono::steady_clock;
    const kc::SuiteLibrary lib = kc::build_suite();
    const kc::SimDevice dev = kc::SimDevice::reference();
    const kc::Int cap(20000000);
    const auto t0 = clk::now();
    const kc::CampaignResult cr = kc::run_campaign(dev, lib, lib.measurement_cases(), cap);
    const auto t1 = clk::now();
    std::map<std::string, kc::KernelIR> irs;
    auto ir = [&](const std::string& id) -> const kc::KernelIR& {
      auto it = irs.find(id);
      if (it == irs.end()) it = irs.emplace(id, kc::parse_kernel(lib.find(id)->text)).first;
      return it->second;
    };
    std::vector<kc::FitCase> cases;
    for (const auto& r : cr.records) cases.push_back({kc::extract_properties(ir(r.kernel), r.binding, cap), r.time_s});
    const kc::DesignMatrix d = kc::build_design_matrix(cases);
    auto [w, rep] = kc::fit_weights(d, dev.name);
    const auto t2 = clk::now();
    double acc = 0;
    int n_eval = 0;
    for (const auto& c : lib.test_cases()) {
      acc += kc::predict(w, kc::extract_properties(ir(c.kernel_id), c.binding, cap)).seconds;
      ++n_eval;
    }
    const auto t3 = clk::now();
    auto s = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
    std::printf("{\"cases\": %zu, \"test_cases\": %d, \"simulate_s\": %.6f, \"fit_s\": %.6f, \"eval_s\": %.6f, "
                "\"total_s\": %.6f, \"objective\": %.6g, \"checksum\": %.17g, \"threads\": 1}\n",
                cr.records.size(), n_eval, s(t0, t1), s(t1, t2), s(t2, t3), s(t0, t3), rep.objective, acc);
    return 0;
  }
  if (mode == "fit") {
    const long rows = std::atol(argv[2]);
    const int F = std::atoi(argv[3]);
    const kc::SimDevice dev = kc::SimDevice::reference();
    std::vector<std::pair<std::string, double>> w;
    const auto& keys = kc::schema_keys();
    for (size_t i = 0; i < keys.size() && static_cast<int>(w.size()) < F; ++i)
      if (dev.alpha[i] != 0) w.emplace_back(keys[i], dev.alpha[i]);
    std::mt19937_64 rng(4242);
    for (size_t i = 0; i < keys.size() && static_cast<int>(w.size()) < F; ++i)
      if (dev.alpha[i] == 0)
        w.emplace_back(keys[i], std::exp(std::log(1e-13) + (std::log(1e-9) - std::log(1e-13)) *
                                                               std::uniform_real_distribution<double>(0, 1)(rng)));
    std::vector<kc::FitCase> cases;
    cases.reserve(rows);
    for (long r = 0; r < rows; ++r) {
      kc::PropertyVector pv;
      double t = 0;
      for (const auto& [key, alpha] : w) {
        const long c = static_cast<long>(1 + rng() % 10000);
        pv.at(key) = kc::CountExpr::from_int(kc::Int(c));
        t += alpha * static_cast<double>(c);
      }
      cases.push_back({std::move(pv), t});
    }
    const auto t0 = std::chrono::steady_clock::now();
    const kc::DesignMatrix d = kc::build_design_matrix(cases);
    const auto t1 = std::chrono::steady_clock::now();
    auto [fw, rep] = kc::fit_weights(d, dev.name);
    const auto t2 = std::chrono::steady_clock::now();
    const double sb = std::chrono::duration<double>(t1 - t0).count();
    const double sf = std::chrono::duration<double>(t2 - t1).count();
    std::printf("{\"rows\": %ld, \"cols\": %d, \"build_s\": %.6f, \"fit_s\": %.6f, \"rows_per_s\": %.6g, "
                "\"objective\": %.6g, \"threads\": 1}\n",
                rows, F, sb, sf, rows / (sb + sf), rep.objective);
    return 0;
  }
  if (mode == "enumerate") {
    const kc::SuiteLibrary lib = kc::build_suite();
    const kc::KernelIR k = kc::parse_kernel(lib.find(argv[2])->text);
    kc::Binding b;
    for (const auto& p : k.params) b[p.name] = kc::Int(std::atol(argv[3]));
    const auto t0 = std::chrono::steady_clock::now();
    const kc::EnumTally t = kc::enumerate_points(k, b, kc::Int("1000000000000"));
    const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const double pts = t.points.convert_to<double>();
    std::printf("{\"points\": %.0f, \"seconds\": %.6f, \"points_per_s\": %.6g, \"threads\": 1}\n", pts, sec,
                pts / sec);
    return 0;
  }
  const int threads = std::max(1, std::atoi(argv[2]));
  const long n = std::atol(argv[3]);
  const long offset = argc > 4 ? std::atol(argv[4]) : 0;

  const kc::SuiteLibrary lib = kc::build_suite();
  const kc::SimDevice dev = kc::SimDevice::reference();
  kc::ModelWeights w;
  w.device = dev.name;
  w.schema_version = kc::kSchemaVersion;
  w.alpha = dev.alpha;
  w.covered.assign(kc::schema_size(), true);

  std::vector<std::string> ids;
  if (mode == "autotune")
    ids = {"matmul_tiled_g12x12", "matmul_tiled_g14x14", "matmul_tiled_g16x16",
           "matmul_naive_g16x12", "matmul_naive_g16x14", "matmul_naive_g16x16"};
  else
    ids = {"matmul_skinny_g16x16", "conv_g16x16"};
  std::vector<Kern> ks;
  for (const auto& id : ids) {
    kc::KernelIR k = kc::parse_kernel(lib.find(id)->text);
    kc::PropertyVector pv = kc::extract_properties(k);
    ks.push_back({std::move(k), std::move(pv)});
  }

  std::atomic<long> points{0};
  std::vector<double> sums(threads, 0.0);
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      const long b = n * t / threads, e = n * (t + 1) / threads;
      double acc = 0;
      long local = 0;
      for (long i = b; i < e; ++i) {
        if (mode == "autotune") {
          const long s = offset + i;
          const long u = s / (551L * 551L) + 1, v = (s / 551L) % 551L + 1, x = s % 551L + 1;
          const kc::Binding bind{{"n", kc::Int(336 * u)}, {"m", kc::Int(336 * v)},
                                 {"l", kc::Int(336 * x)}};
          double best = 1e300;
          for (const auto& k : ks) {
            const kc::PropertyVector bound = kc::evaluate_properties(k.ir, k.sym, bind);
            const double sec = kc::predict(w, bound).seconds;
            if (sec < best) best = sec;
            ++local;
          }
          acc += best;
        } else {
          const long u = i / 2 + 1;
          const Kern& k = ks[i % 2];
          kc::Binding bind;
          if (i % 2 == 0)
            bind = {{"n", kc::Int(16 * u)}, {"m", kc::Int(128 * u)}, {"l", kc::Int(16 * u)}};
          else
            bind = {{"n", kc::Int(16 * u)}};
          const kc::PropertyVector bound = kc::evaluate_properties(k.ir, k.sym, bind);
          acc += kc::predict(w, bound).seconds;
          ++local;
        }
      }
      sums[t] = acc;
      points += local;
    });
  }
  for (auto& th : pool) th.join();
  const double sec =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  double checksum = 0;
  for (double s : sums) checksum += s;
  std::printf("{\"points\": %ld, \"seconds\": %.6f, \"points_per_s\": %.6g, \"threads\": %d, "
              "\"checksum\": %.17g}\n",
              points.load(), sec, points.load() / sec, threads, checksum);
  return 0;
}
