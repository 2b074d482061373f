// ORACLE TEST INFRASTRUCTURE -- BASELINE config 2 through the reference.
//
//   kcref_config2 <kernel_id> <mode sym|bound> <u0> <u1> <keys> <out.bin>
//
// For u in [u0, u1) evaluates the test kernel at the config-2 binding
// (suite.cpp:527-552 shapes):
//   matmul_skinny_g16x16  n = 16u, m = 128u, l = 16u
//   conv_g16x16           n = 16u
//   fd_stencil_g16x16     n = 16u
//   nbody_g256            n = 256u
// mode sym:   extract_properties(k) once, then evaluate_properties(k, pv, b)
//             per point (props.cpp:259-271) -- the symbolic path;
// mode bound: extract_properties(k, b, cap 2e7) per point -- bound mode,
//             enumerating what the front end cannot count symbolically.
// then predict (model.cpp:95-117) with the simdev-v1 weights. <keys> is the
// comma-separated schema indices of the GPU program's keys (its property
// order); the tool fails if the reference produces a nonzero count on any
// other key. Per point it appends to <out.bin>, for each key, the count as a
// little-endian two's-complement int128 (lo, hi int64), then the prediction's
// IEEE bits: the layout tests/gen/gen_config2.py hashes block by block and
// tests/test_config2.py rebuilds from the GPU's counts lo/hi columns.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "kernelcost/model.hpp"
#include "kernelcost/parser.hpp"
#include "kernelcost/props.hpp"
#include "kernelcost/schema.hpp"
#include "kernelcost/simdevice.hpp"
#include "kernelcost/suite.hpp"

namespace kc = kernelcost;

namespace {

__int128 to_i128(const kc::Int& v) {
  const std::string s = v.str();
  __int128 r = 0;
  size_t i = 0;
  const bool neg = !s.empty() && s[0] == '-';
  if (neg) i = 1;
  for (; i < s.size(); ++i) r = r * 10 + (s[i] - '0');
  return neg ? -r : r;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc != 7) {
    std::fprintf(stderr, "usage: kcref_config2 <kernel_id> sym|bound <u0> <u1> <keys> <out.bin>\n");
    return 2;
  }
  const std::string id = argv[1], mode = argv[2];
  const long u0 = std::atol(argv[3]), u1 = std::atol(argv[4]);
  std::vector<int> keys;
  {
    std::stringstream ss(argv[5]);
    std::string tok;
    while (std::getline(ss, tok, ',')) keys.push_back(std::atoi(tok.c_str()));
  }
  std::vector<bool> listed(kc::schema_size(), false);
  for (int k : keys) listed[k] = true;
  const kc::SuiteLibrary lib = kc::build_suite();
  const kc::KernelIR ir = kc::parse_kernel(lib.find(id)->text);
  const kc::SimDevice dev = kc::SimDevice::reference();
  kc::ModelWeights w;
  w.device = dev.name;
  w.schema_version = kc::kSchemaVersion;
  w.alpha = dev.alpha;
  w.covered.assign(kc::schema_size(), true);
  kc::PropertyVector sym;
  if (mode == "sym") sym = kc::extract_properties(ir);
  FILE* out = std::fopen(argv[6], "wb");
  if (!out) return 3;
  std::vector<int64_t> rec(keys.size() * 2 + 1);
  for (long u = u0; u < u1; ++u) {
    kc::Binding b;
    if (id == "matmul_skinny_g16x16")
      b = {{"n", kc::Int(16 * u)}, {"m", kc::Int(128 * u)}, {"l", kc::Int(16 * u)}};
    else if (id == "nbody_g256")
      b = {{"n", kc::Int(256 * u)}};
    else
      b = {{"n", kc::Int(16 * u)}};
    const kc::PropertyVector bound =
        mode == "sym" ? kc::evaluate_properties(ir, sym, b) : kc::extract_properties(ir, b, kc::Int(20000000));
    for (size_t i = 0; i < bound.entries.size(); ++i)
      if (!listed[i] && !bound.entries[i].is_zero()) {
        std::fprintf(stderr, "%s u=%ld: nonzero count on unlisted key %s\n", id.c_str(), u, kc::schema_keys()[i].c_str());
        return 4;
      }
    for (size_t j = 0; j < keys.size(); ++j) {
      const auto& e = bound.entries[keys[j]];
      __int128 v = 0;
      if (!e.is_zero()) {
        const kc::Rat r = e.constant_value();
        if (boost::multiprecision::denominator(r) != 1) return 5;
        v = to_i128(boost::multiprecision::numerator(r));
      }
      rec[2 * j] = static_cast<int64_t>(static_cast<uint64_t>(v));
      rec[2 * j + 1] = static_cast<int64_t>(v >> 64);
    }
    const double sec = kc::predict(w, bound).seconds;
    std::memcpy(&rec[2 * keys.size()], &sec, 8);
    std::fwrite(rec.data(), 8, rec.size(), out);
  }
  std::fclose(out);
  return 0;
}
