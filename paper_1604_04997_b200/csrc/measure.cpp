// Measurement I/O (the data format on the input side of
// the fit): the reference's measurement CSV and raw-runs CSV
// (csvio.cpp:104-225), detected by header like the CLI's read_any_csv
// (kernelcost.cpp:116-126), returned as per-kernel SoA columns ready to be
// copied to the GPU for the fused Gram / residual / predict kernels.
#include <algorithm>
#include <cerrno>
#include <cstdlib>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/kcg.h"
#include "kcg_host.hpp"

struct kcg_measurements {
  struct Kernel {
    std::string name;
    std::vector<std::string> params;  // sorted (std::map order of Binding)
    std::vector<std::vector<int64_t>> cols;
    std::vector<double> times;
  };
  std::vector<Kernel> kernels;  // sorted by name
};

namespace kcg {

namespace {

// fields of one CSV line (no quoting in the measurement format): every
// separator ends a field, so "a,,b," has four fields
std::vector<std::string> split(const std::string& line, char sep) {
  std::vector<std::string> fields;
  size_t start = 0;
  for (;;) {
    const size_t end = line.find(sep, start);
    fields.emplace_back(line, start, end == std::string::npos ? std::string::npos : end - start);
    if (end == std::string::npos) return fields;
    start = end + 1;
  }
}

[[noreturn]] void bad(const std::string& path, int line, const std::string& what) {
  throw KcgError(KCG_E_PARSE, path + ": line " + std::to_string(line) + ": " + what);
}

// parse_binding (csvio.cpp:86-102) restricted to int64 values
std::map<std::string, int64_t> parse_binding(const std::string& s, const std::string& path, int line) {
  std::map<std::string, int64_t> b;
  if (s.empty()) return b;
  for (const std::string& part : split(s, ';')) {
    const size_t eq = part.find('=');
    if (eq == std::string::npos || eq == 0) bad(path, line, "bad binding entry '" + part + "'");
    const std::string v = part.substr(eq + 1);
    char* end = nullptr;
    errno = 0;
    const long long x = std::strtoll(v.c_str(), &end, 10);
    if (v.empty() || *end != '\0') bad(path, line, "bad binding value '" + part + "'");
    if (errno == ERANGE)
      throw KcgError(KCG_E_UNSUPPORTED, path + ": line " + std::to_string(line) +
                                            ": binding value beyond int64 '" + part + "'");
    b[part.substr(0, eq)] = x;
  }
  return b;
}

double parse_time(const std::string& s, const std::string& path, int line) {
  char* end = nullptr;
  const double t = std::strtod(s.c_str(), &end);
  if (s.empty() || *end != '\0') bad(path, line, "bad time '" + s + "'");
  return t;
}

struct Rec {
  std::string kernel;
  std::map<std::string, int64_t> binding;
  double time;
};

std::string binding_text(const std::map<std::string, int64_t>& b) {
  std::string out;
  for (const auto& [k, v] : b) {
    if (!out.empty()) out += ';';
    out += k + "=" + std::to_string(v);
  }
  return out;
}

}  // namespace

kcg_measurements* read_measurements(const std::string& path, int discard) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw KcgError(KCG_E_IO, "cannot open: " + path);
  std::string line, header;
  std::getline(in, header);
  if (!header.empty() && header.back() == '\r') header.pop_back();
  const bool raw = header == "kernel,binding,group_config,run_index,time_s";
  if (!raw && header != "kernel,binding,group_config,time_s")
    throw KcgError(KCG_E_PARSE, path + ": unexpected header '" + header + "'");
  std::vector<Rec> recs;
  // raw runs: (kernel, binding text, group) -> (run index, time)
  std::map<std::tuple<std::string, std::string, std::string>, std::vector<std::pair<int, double>>> groups;
  std::map<std::tuple<std::string, std::string, std::string>, std::map<std::string, int64_t>> gbind;
  int line_no = 1;
  while (std::getline(in, line)) {
    ++line_no;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty()) continue;
    const auto f = split(line, ',');
    if (f.size() != (raw ? 5u : 4u))
      bad(path, line_no, "expected " + std::to_string(raw ? 5 : 4) + " fields, got " + std::to_string(f.size()));
    auto b = parse_binding(f[1], path, line_no);
    if (!raw) {
      recs.push_back({f[0], std::move(b), parse_time(f[3], path, line_no)});
    } else {
      char* end = nullptr;
      const long idx = std::strtol(f[3].c_str(), &end, 10);
      if (f[3].empty() || *end != '\0') bad(path, line_no, "bad run index '" + f[3] + "'");
      const auto key = std::make_tuple(f[0], binding_text(b), f[2]);
      groups[key].emplace_back(static_cast<int>(idx), parse_time(f[4], path, line_no));
      gbind[key] = std::move(b);
    }
  }
  if (raw) {
    if (discard < 0) throw KcgError(KCG_E_INVALID_ARGUMENT, "negative discard count");
    for (auto& [key, samples] : groups) {  // reduce_raw_runs (csvio.cpp:192-225)
      std::sort(samples.begin(), samples.end());
      if (samples.size() <= static_cast<size_t>(discard))
        throw KcgError(KCG_E_INVALID_ARGUMENT, "need more than " + std::to_string(discard) +
                                                   " runs, got " + std::to_string(samples.size()));
      double best = samples[discard].second;
      for (size_t i = discard; i < samples.size(); ++i) best = std::min(best, samples[i].second);
      recs.push_back({std::get<0>(key), gbind[key], best});
    }
  }
  auto m = std::make_unique<kcg_measurements>();
  std::map<std::string, size_t> idx;
  for (const Rec& r : recs) {
    auto it = idx.find(r.kernel);
    if (it == idx.end()) {
      kcg_measurements::Kernel k;
      k.name = r.kernel;
      for (const auto& [p, v] : r.binding) k.params.push_back(p);
      k.cols.resize(k.params.size());
      it = idx.emplace(r.kernel, m->kernels.size()).first;
      m->kernels.push_back(std::move(k));
    }
    auto& k = m->kernels[it->second];
    if (r.binding.size() != k.params.size())
      throw KcgError(KCG_E_INVALID_ARGUMENT, "kernel '" + r.kernel + "' has bindings over different parameters");
    size_t j = 0;
    for (const auto& [p, v] : r.binding) {
      if (p != k.params[j])
        throw KcgError(KCG_E_INVALID_ARGUMENT, "kernel '" + r.kernel + "' has bindings over different parameters");
      k.cols[j++].push_back(v);
    }
    k.times.push_back(r.time);
  }
  std::sort(m->kernels.begin(), m->kernels.end(),
            [](const kcg_measurements::Kernel& a, const kcg_measurements::Kernel& b) { return a.name < b.name; });
  return m.release();
}

}  // namespace kcg

namespace {
thread_local std::string g_err;
}

extern "C" {

int kcg_measurements_read_csv(const char* path, int discard, kcg_measurements** out) {
  if (!path || !out) return KCG_E_INVALID_ARGUMENT;
  *out = nullptr;
  try {
    *out = kcg::read_measurements(path, discard);
    return KCG_OK;
  } catch (const kcg::KcgError& e) {
    kcg_set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    kcg_set_last_error(e.what());
    return KCG_E_INTERNAL;
  }
}

void kcg_measurements_destroy(kcg_measurements* m) { delete m; }

int kcg_measurements_num_kernels(const kcg_measurements* m) {
  return m ? static_cast<int>(m->kernels.size()) : -1;
}

const char* kcg_measurements_kernel(const kcg_measurements* m, int i) {
  return m && i >= 0 && i < static_cast<int>(m->kernels.size()) ? m->kernels[i].name.c_str() : nullptr;
}

size_t kcg_measurements_num_rows(const kcg_measurements* m, int i) {
  return m && i >= 0 && i < static_cast<int>(m->kernels.size()) ? m->kernels[i].times.size() : 0;
}

int kcg_measurements_num_params(const kcg_measurements* m, int i) {
  return m && i >= 0 && i < static_cast<int>(m->kernels.size()) ? static_cast<int>(m->kernels[i].params.size())
                                                                  : -1;
}

const char* kcg_measurements_param_name(const kcg_measurements* m, int i, int j) {
  if (!m || i < 0 || i >= static_cast<int>(m->kernels.size())) return nullptr;
  const auto& k = m->kernels[i];
  return j >= 0 && j < static_cast<int>(k.params.size()) ? k.params[j].c_str() : nullptr;
}

const int64_t* kcg_measurements_column(const kcg_measurements* m, int i, int j) {
  if (!m || i < 0 || i >= static_cast<int>(m->kernels.size())) return nullptr;
  const auto& k = m->kernels[i];
  return j >= 0 && j < static_cast<int>(k.cols.size()) ? k.cols[j].data() : nullptr;
}

const double* kcg_measurements_times(const kcg_measurements* m, int i) {
  return m && i >= 0 && i < static_cast<int>(m->kernels.size()) ? m->kernels[i].times.data() : nullptr;
}

}  // extern "C"
