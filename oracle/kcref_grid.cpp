// ORACLE TEST INFRASTRUCTURE -- the front-end extension (kcref_extract.hpp)
// run over the reference's whole suite:
//
//   kcref_grid <programs_dir | -> [<extra.json> <kernels.txt>]   (- : skip the suite)
//
//  * every suite kernel the reference extracts symbolically: the extension's
//    PropertyVector must equal extract_properties(k) entry for entry
//    (CountExpr::str());
//  * every kernel it rejects (fd_stencil, nbody): the extension's symbolic
//    PV, bound at each oracle-lattice binding the 2e7 enumeration cap
//    admits, must equal the reference's bound mode extract_properties(k, b,
//    cap) on all 149 keys; its program_text is written to
//    <programs_dir>/<id>.kcp (replacing the round-1 interpolated files);
//  * extra kernels (tests/gen/halo_kernels.txt, "----"-separated): the same
//    bound-mode check over n = 16 u; their program_text, enum_text and the
//    reference's bound-mode counts go to <extra.json> (tests/golden/
//    halo_kernels.json) for the GPU tests.
// Prints one JSON object; exit 0 iff every comparison held.
#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "json.hpp"
#include "kcref_extract.hpp"
#include "kcref_program.hpp"
#include "kernelcost/parser.hpp"
#include "kernelcost/suite.hpp"

namespace kc = kernelcost;

namespace {

bool same_pv(const kc::PropertyVector& a, const kc::PropertyVector& b) {
  for (size_t i = 0; i < a.entries.size(); ++i)
    if (a.entries[i].str() != b.entries[i].str()) return false;
  return true;
}

// bound-mode check of a symbolic PV: returns (#bindings compared, #mismatches)
std::pair<int, int> check_bound(const kc::KernelIR& k, const kc::PropertyVector& pv,
                                const std::vector<kc::Binding>& bs) {
  int n = 0, bad = 0;
  for (const auto& b : bs) {
    kc::PropertyVector ref;
    try {
      ref = kc::extract_properties(k, b, kc::Int(20000000));
    } catch (const kc::Error& e) {
      if (e.code() == kc::Errc::cap_exceeded || e.code() == kc::Errc::assumption_violated) continue;
      throw;
    }
    const kc::PropertyVector got = kc::evaluate_properties(k, pv, b);
    ++n;
    if (!same_pv(got, ref)) {
      ++bad;
      std::fprintf(stderr, "%s: bound-mode mismatch\n", k.name.c_str());
    }
  }
  return {n, bad};
}

}  // namespace

int main(int argc, char** argv) {
  if (argc != 2 && argc != 4) {
    std::fprintf(stderr, "usage: kcref_grid <programs_dir> [<extra.json> <kernels.txt>]\n");
    return 2;
  }
  const std::string pdir = argv[1];
  const kc::SuiteLibrary lib = kc::build_suite();
  int sym_equal = 0, sym_differ = 0, extended = 0, still_failing = 0, bound_checked = 0, bound_bad = 0;
  std::string ext_ids;
  auto emit = [&](const kc::KernelIR& k, const kc::PropertyVector& pv) {
    std::ofstream(pdir + "/" + k.name + ".kcp") << kcref::program_text(k, pv);
    ext_ids += (ext_ids.empty() ? "\"" : ", \"") + k.name + "\"";
  };
  for (const auto& sk : lib.kernels) {
    if (pdir == "-") break;  // extra kernels only
    const kc::KernelIR k = kc::parse_kernel(sk.text);
    kc::PropertyVector ref;
    bool ref_ok = true;
    try {
      ref = kc::extract_properties(k);
    } catch (const kc::Error& e) {
      if (e.code() != kc::Errc::needs_binding) throw;
      ref_ok = false;
    }
    kc::PropertyVector ext;
    try {
      ext = kcref::extract_properties_grid(k);
    } catch (const kc::Error& e) {
      if (ref_ok || e.code() != kc::Errc::needs_binding) throw;
      ++still_failing;
      continue;
    }
    if (ref_ok) {
      (same_pv(ref, ext) ? sym_equal : sym_differ)++;
      continue;
    }
    ++extended;
    // the oracle lattice (sample_oracle_binding, seed 0x5eed as acceptance.cpp)
    // plus every lattice point n = unit * u up to the cap
    std::vector<kc::Binding> bs;
    std::mt19937_64 rng(0x5eed);
    for (int i = 0; i < 20; ++i) bs.push_back(kc::sample_oracle_binding(sk, rng));
    for (const auto& od : sk.oracle)
      for (long u = 1; u <= 160; ++u) bs.push_back({{od.param, od.unit * u}});
    const auto [n, bad] = check_bound(k, ext, bs);
    bound_checked += n;
    bound_bad += bad;
    emit(k, ext);
  }
  if (argc == 4) {  // extra kernels: every parameter n = 16 u
    using json = nlohmann::ordered_json;
    std::ifstream in(argv[3]);
    std::stringstream ss;
    ss << in.rdbuf();
    const std::string all = ss.str();
    json ks = json::array();
    for (size_t b0 = 0; b0 < all.size();) {
      size_t e = all.find("\n----\n", b0);
      const std::string text = all.substr(b0, e == std::string::npos ? std::string::npos : e - b0 + 1);
      b0 = e == std::string::npos ? all.size() : e + 6;
      const kc::KernelIR k = kc::parse_kernel(text);
      bool ref_ok = true;
      try {
        (void)kc::extract_properties(k);
      } catch (const kc::Error&) {
        ref_ok = false;
      }
      const kc::PropertyVector ext = kcref::extract_properties_grid(k);
      std::vector<kc::Binding> bs;
      json bound = json::array();
      for (long u = 1; u <= 512; ++u) {
        kc::Binding b;
        for (const auto& p : k.params) b[p.name] = kc::Int(16 * u);
        kc::PropertyVector ref;
        try {
          ref = kc::extract_properties(k, b, kc::Int(20000000));
        } catch (const kc::Error&) {
          continue;
        }
        bs.push_back(b);
        json c = json::object();
        for (size_t i = 0; i < ref.entries.size(); ++i)
          if (!ref.entries[i].is_zero()) c[kc::schema_keys()[i]] = ref.entries[i].str();
        bound.push_back(json{{"n", 16 * u}, {"counts", c}});
      }
      const auto [n, bad] = check_bound(k, ext, bs);
      bound_checked += n;
      bound_bad += bad;
      if (!ref_ok) ++extended;
      ks.push_back(json{{"id", k.name}, {"reference_symbolic", ref_ok}, {"source", text},
                        {"program", kcref::program_text(k, ext)}, {"enum_text", kcref::enum_text(k)},
                        {"bound_mode", bound}});
    }
    std::ofstream(argv[2]) << json{{"kernels", ks}}.dump(1) << "\n";
  }
  std::printf("{\"symbolic_equal\": %d, \"symbolic_differ\": %d, \"extended\": %d, \"still_needs_binding\": %d, "
              "\"bound_mode_bindings_compared\": %d, \"bound_mode_mismatches\": %d, \"written\": [%s]}\n",
              sym_equal, sym_differ, extended, still_failing, bound_checked, bound_bad, ext_ids.c_str());
  return sym_differ == 0 && bound_bad == 0 && still_failing == 0 ? 0 : 1;
}
