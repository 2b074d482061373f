// extern "C" boundary (include/kcg.h): program handles, launch dispatch,
// host-side solve and weights I/O. No exception crosses this file's
// functions; failures become KCG_E_* codes plus kcg_last_error().
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <limits>
#include <memory>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/kcg.h"
#include "json.hpp"
#include "kcg_codegen.hpp"
#include "kcg_host.hpp"
#include "kcg_kernels.hpp"

using kcg::i128;
using kcg::KcgError;

struct kcg_program {
  kcg::Symbolic sym;
  kcg::Lowered low;
  std::vector<std::string> param_names;
  int engine = KCG_ENGINE_JIT;
  KcgDevProg* dprog = nullptr;  // device image (interpreter), lazily uploaded
  KcgDevProg* dadmit = nullptr; // admissibility-only image (beyond the count bound)
  bool dprog_ok = true;         // fits the interpreter's static tables
  std::string jit_src;
  std::string jit_src_kind;
  void* jit_eval = nullptr;
  void* jit_eval_gen = nullptr;
  void* jit_eval_tma = nullptr;
  void* jit_eval_grid = nullptr;
  void* jit_eval_grid_gen = nullptr;
  void* jit_gram = nullptr;
  void* jit_resid = nullptr;
  void* jit_rgrad = nullptr;
  uint64_t uid = next_uid();  // identity for caches keyed by program sets
  static uint64_t next_uid() {
    static std::atomic<uint64_t> c{1};
    return c++;
  }
};

namespace {

thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
std::atomic<unsigned> g_host_last_path{0};

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

}  // namespace

extern "C" void kcg_set_last_error(const char* msg) { g_last_error = msg ? msg : ""; }

namespace {

// NVTX range per C-ABI phase (visible in Nsight Systems / ncu
// --nvtx); a no-op unless a tool is attached (nvtx3 is header-only)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const KcgError& e) {
    return fail(e.code, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(KCG_E_INVALID_ARGUMENT, e.what());
  } catch (const std::exception& e) {
    return fail(KCG_E_CUDA, e.what());
  }
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw KcgError(KCG_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void require_device() {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    throw KcgError(KCG_E_CUDA, "no CUDA device available (the kcg back end has no CPU fallback)");
}

// byte-exact image of the generated `struct KcgArgs` (natural C alignment)
// progs[v]'s parameter j lives in launch column pmaps[v][j] (progs[0]'s
// declaration order); every program must have the same parameter names
void variant_maps(const kcg_program* const* progs, int V, std::vector<const kcg::Lowered*>& lows,
                  std::vector<std::vector<int>>& pmaps) {
  const kcg_program* p0 = progs[0];
  if (!p0) throw KcgError(KCG_E_INVALID_ARGUMENT, "null program");
  const int np = p0->low.n_params;
  for (int v = 0; v < V; ++v) {
    const kcg_program* p = progs[v];
    if (!p || p->low.n_params != np)
      throw KcgError(KCG_E_INVALID_ARGUMENT, "the programs must share the parameter set");
    std::vector<int> map(np);
    for (int j = 0; j < np; ++j) {
      auto it = std::find(p0->param_names.begin(), p0->param_names.end(), p->param_names[j]);
      if (it == p0->param_names.end())
        throw KcgError(KCG_E_INVALID_ARGUMENT, "the programs must share the parameter set");
      map[j] = static_cast<int>(it - p0->param_names.begin());
    }
    lows.push_back(&p->low);
    pmaps.push_back(map);
  }
}

struct ArgBuf {
  std::vector<unsigned char> b;
  template <class T>
  void push(const T& v) {
    const size_t al = alignof(T);
    while (b.size() % al) b.push_back(0);
    const auto* p = reinterpret_cast<const unsigned char*>(&v);
    b.insert(b.end(), p, p + sizeof(T));
  }
  void finish() {
    while (b.size() % 8) b.push_back(0);
  }
};

unsigned grid_for(size_t n, int threads = 256, int per_sm = 8) {
  const size_t need = (n + threads - 1) / threads;
  const size_t cap = static_cast<size_t>(kcg::num_sms()) * per_sm;
  return static_cast<unsigned>(std::max<size_t>(1, std::min(need, cap)));
}

KcgWide wide(i128 v) { return {static_cast<int64_t>(v), static_cast<int64_t>(v >> 64)}; }

bool build_devprog(const kcg::Lowered& L, KcgDevProg& d) {
  std::memset(&d, 0, sizeof d);
  if (L.n_params > KCG_MAX_PARAMS || static_cast<int>(L.ops.size()) > KCG_MAX_OPS ||
      L.n_atoms > KCG_MAX_ATOMS || L.n_monos > KCG_MAX_MONOS ||
      static_cast<int>(L.factors.size()) > KCG_MAX_FACTORS ||
      static_cast<int>(L.terms.size()) > KCG_MAX_TERMS || L.n_exprs > KCG_MAX_EXPRS ||
      static_cast<int>(L.args.size()) > KCG_MAX_ARGS ||
      static_cast<int>(L.floordiv_den.size()) > KCG_MAX_FD ||
      static_cast<int>(L.cons.size()) > KCG_MAX_CONS ||
      static_cast<int>(L.keys.size()) > KCG_MAX_KEYS)
    return false;
  d.n_params = L.n_params;
  d.n_atoms = L.n_atoms;
  d.n_monos = L.n_monos;
  d.n_exprs = L.n_exprs;
  d.n_ops = static_cast<int32_t>(L.ops.size());
  d.n_cons = static_cast<int32_t>(L.cons.size());
  d.n_keys = static_cast<int32_t>(L.keys.size());
  d.b64 = L.b64;
  d.b128 = L.b128;
  for (size_t i = 0; i < L.ops.size(); ++i)
    d.ops[i] = {L.ops[i].code, L.ops[i].dst, L.ops[i].a, L.ops[i].b, L.ops[i].c};
  for (size_t i = 0; i < L.factors.size(); ++i) {
    d.fac_atom[i] = L.factors[i].first;
    d.fac_exp[i] = L.factors[i].second;
  }
  for (size_t i = 0; i < L.terms.size(); ++i) {
    d.term_coef[i] = wide(L.terms[i].coef);
    d.term_mono[i] = L.terms[i].mono;
  }
  for (size_t i = 0; i < L.exprs.size(); ++i) d.expr_den[i] = wide(L.exprs[i].D);
  for (size_t i = 0; i < L.args.size(); ++i) {
    d.arg_expr[i] = L.args[i].expr;
    d.arg_scale[i] = wide(L.args[i].scale);
  }
  for (size_t i = 0; i < L.floordiv_den.size(); ++i) d.fd_den[i] = wide(L.floordiv_den[i]);
  for (size_t i = 0; i < L.cons.size(); ++i) {
    d.cons_div[i] = L.cons[i].divisibility;
    d.cons_op[i] = L.cons[i].op;
    d.cons_expr[i] = L.cons[i].expr;
    d.cons_mod[i] = wide(L.cons[i].mod);
    d.cons_rem[i] = wide(L.cons[i].rem);
  }
  if (L.quot_mod.size() > KCG_MAX_PARAMS) return false;
  for (size_t i = 0; i < L.quot_mod.size(); ++i) {
    d.quot_mod[i] = wide(L.quot_mod[i]);
    d.quot_rem[i] = wide(L.quot_rem[i]);
  }
  for (size_t i = 0; i < L.keys.size(); ++i) {
    d.key_schema[i] = L.keys[i].schema;
    d.key_expr[i] = L.keys[i].expr;
  }
  return true;
}

std::vector<int> identity(int n) {
  std::vector<int> v(n);
  for (int i = 0; i < n; ++i) v[i] = i;
  return v;
}

std::string kname(const char* base, const kcg_program* p) {
  std::string s = base;
  for (char c : p->sym.kernel) s.push_back(std::isalnum(static_cast<unsigned char>(c)) ? c : '_');
  return s;
}

void compact_alpha(const kcg_program* p, const double* alpha149, double* out) {
  for (size_t j = 0; j < p->low.keys.size(); ++j)
    out[j] = alpha149 ? alpha149[p->low.keys[j].schema] : 0.0;
}

// alpha (compact) -> the folded weights of the GEN = 0 predict kernels
// (kcg::predict_fold); *finite says whether both sets are finite (the
// precondition of the unconditional-accumulation kernels)
std::vector<double> folded_alpha(const kcg_program* p, const std::vector<double>& al, bool* finite) {
  std::vector<double> f(al);
  bool fin = true;
  for (size_t j = 0; j < p->low.keys.size(); ++j) {
    f[j] = al[j] * kcg::predict_fold(p->low, static_cast<int>(j));
    fin = fin && std::isfinite(al[j]) && std::isfinite(f[j]);
  }
  if (finite) *finite = fin;
  return f;
}

// symmetric eigen-decomposition (cyclic Jacobi), A row-major n x n
void jacobi_eigen(int n, std::vector<double>& A, std::vector<double>& V, std::vector<double>& w) {
  V.assign(static_cast<size_t>(n) * n, 0.0);
  for (int i = 0; i < n; ++i) V[i * n + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0, diag = 0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) (i == j ? diag : off) += A[i * n + j] * A[i * n + j];
    if (off <= 1e-34 * diag || off == 0) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A[p * n + q];
        if (apq == 0) continue;
        const double app = A[p * n + p], aqq = A[q * n + q];
        const double theta = (aqq - app) / (2 * apq);
        const double t = (theta >= 0 ? 1 : -1) / (std::fabs(theta) + std::sqrt(theta * theta + 1));
        const double c = 1 / std::sqrt(t * t + 1), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double akp = A[k * n + p], akq = A[k * n + q];
          A[k * n + p] = c * akp - s * akq;
          A[k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = A[p * n + k], aqk = A[q * n + k];
          A[p * n + k] = c * apk - s * aqk;
          A[q * n + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = V[k * n + p], vkq = V[k * n + q];
          V[k * n + p] = c * vkp - s * vkq;
          V[k * n + q] = s * vkp + c * vkq;
        }
      }
  }
  w.resize(n);
  for (int i = 0; i < n; ++i) w[i] = A[i * n + i];
}

// minimum-norm solution of (D G D) y = D b over covered columns; returns
// x = D y (unscaled coordinates) and the numerical rank
int solve_equilibrated(int F, const double* G, const double* colmax, const double* b,
                       std::vector<double>& x) {
  std::vector<int> cols;
  for (int j = 0; j < F; ++j)
    if (colmax[j] > 0.0) cols.push_back(j);
  x.assign(F, 0.0);
  const int n = static_cast<int>(cols.size());
  if (n == 0) return 0;
  std::vector<double> s(n), A(static_cast<size_t>(n) * n), rhs(n);
  for (int i = 0; i < n; ++i) s[i] = 1.0 / colmax[cols[i]];  // model.cpp:71-76
  for (int i = 0; i < n; ++i) {
    rhs[i] = b[cols[i]] * s[i];
    for (int j = 0; j < n; ++j) A[i * n + j] = G[cols[i] * F + cols[j]] * s[i] * s[j];
  }
  std::vector<double> V, w;
  jacobi_eigen(n, A, V, w);
  double wmax = 0;
  for (double v : w) wmax = std::max(wmax, std::fabs(v));
  const double tol = wmax * n * std::numeric_limits<double>::epsilon() * 64;
  int rank = 0;
  std::vector<double> y(n, 0.0);
  for (int k = 0; k < n; ++k) {
    if (w[k] <= tol) continue;
    ++rank;
    double proj = 0;
    for (int i = 0; i < n; ++i) proj += V[i * n + k] * rhs[i];
    proj /= w[k];
    for (int i = 0; i < n; ++i) y[i] += V[i * n + k] * proj;
  }
  for (int i = 0; i < n; ++i) x[cols[i]] = y[i] * s[i];  // alpha = x * scale
  return rank;
}

}  // namespace

extern "C" {

int kcg_schema_size(void) { return static_cast<int>(kcg::schema_keys().size()); }

const char* kcg_schema_key(int index) {
  const auto& k = kcg::schema_keys();
  return index >= 0 && index < static_cast<int>(k.size()) ? k[index].c_str() : nullptr;
}

int kcg_schema_index(const char* key) { return key ? kcg::schema_index(key) : -1; }

const char* kcg_schema_version(void) { return "v1"; }

int kcg_program_create(const char* text, size_t len, kcg_program** out) {
  if (!text || !out) return fail(KCG_E_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  return guarded([&] {
    auto p = std::make_unique<kcg_program>();
    p->sym = kcg::parse_program_text(std::string(text, len));
    p->low = kcg::lower(p->sym);
    if (p->low.n_params > KCG_MAX_PARAMS)
      throw KcgError(KCG_E_UNSUPPORTED, "more than 8 parameters");
    p->param_names = p->sym.params;
    if (const char* e = std::getenv("KCG_ENGINE"); e && std::string(e) == "interp")
      p->engine = KCG_ENGINE_INTERP;
    *out = p.release();
    return KCG_OK;
  });
}

void kcg_program_destroy(kcg_program* prog) {
  if (!prog) return;
  if (prog->dprog) cudaFree(prog->dprog);
  if (prog->dadmit) cudaFree(prog->dadmit);
  delete prog;
}

int kcg_program_num_params(const kcg_program* p) { return p ? p->low.n_params : -1; }

const char* kcg_program_param_name(const kcg_program* p, int i) {
  return p && i >= 0 && i < p->low.n_params ? p->param_names[i].c_str() : nullptr;
}

int kcg_program_num_props(const kcg_program* p) {
  return p ? static_cast<int>(p->low.keys.size()) : -1;
}

int kcg_program_prop_schema_index(const kcg_program* p, int j) {
  return p && j >= 0 && j < static_cast<int>(p->low.keys.size()) ? p->low.keys[j].schema : -1;
}

const char* kcg_program_kernel_name(const kcg_program* p) { return p ? p->sym.kernel.c_str() : nullptr; }

int kcg_program_safe_bounds(const kcg_program* p, int64_t* b64, int64_t* b128) {
  if (!p) return fail(KCG_E_INVALID_ARGUMENT, "null program");
  if (b64) *b64 = p->low.b64;
  if (b128) *b128 = p->low.b128;
  return KCG_OK;
}

int kcg_program_set_engine(kcg_program* p, int engine) {
  if (!p || (engine != KCG_ENGINE_JIT && engine != KCG_ENGINE_INTERP))
    return fail(KCG_E_INVALID_ARGUMENT, "bad engine");
  p->engine = engine;
  return KCG_OK;
}

int kcg_program_set_gram_basis(kcg_program* p, int enable) {
  if (!p) return fail(KCG_E_INVALID_ARGUMENT, "null program");
  if (p->low.gram_basis != (enable != 0)) {
    p->low.gram_basis = enable != 0;
    p->jit_gram = p->jit_resid = nullptr;  // respecialise on next use (modules stay cached)
  }
  return KCG_OK;
}

const char* kcg_program_jit_source(kcg_program* p) {
  if (!p) return nullptr;
  if (p->jit_src.empty())
    p->jit_src = kcg::codegen({&p->low}, {identity(p->low.n_params)}, p->low.n_params,
                              kcg::JitKind::eval, kname("kcg_eval_", p));
  return p->jit_src.c_str();
}

const char* kcg_program_jit_source_kind(kcg_program* p, int kind) {
  if (!p || kind < 0 || kind > 5) return nullptr;
  if (kind == 0) return kcg_program_jit_source(p);
  const int np = p->low.n_params;
  if (kind == 4) {  // the evaluator as host C++ (kcg_host_eval), e.g. for a CPU baseline
    p->jit_src_kind = kcg::codegen({&p->low}, {identity(np)}, np, kcg::JitKind::host_eval, "kcg_host_eval");
    return p->jit_src_kind.c_str();
  }
  if (kind == 3) {  // argmin over this single variant
    p->jit_src_kind = kcg::codegen({&p->low}, {identity(np)}, np, kcg::JitKind::argmin, "kcg_argmin");
    return p->jit_src_kind.c_str();
  }
  p->jit_src_kind = kcg::codegen({&p->low}, {identity(np)}, np,
                                 kind == 1 ? kcg::JitKind::gram : kind == 2 ? kcg::JitKind::residual
                                                                            : kcg::JitKind::residual_grad,
                                 kname(kind == 1 ? "kcg_gram_" : kind == 2 ? "kcg_resid_" : "kcg_rgrad_", p));
  return p->jit_src_kind.c_str();
}

int kcg_jit_compile_check(const char* src, const char* name) {
  if (!src || !name) return fail(KCG_E_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    kcg::jit_compile_only(src, name);
    return KCG_OK;
  });
}

int kcg_eval_predict(const kcg_program* cp, const int64_t* const* param_cols, size_t n,
                     const double* alpha, double* pred_out, uint8_t* status_out,
                     int64_t* counts_lo, int64_t* counts_hi, int simulate, void* stream) {
  kcg_program* p = const_cast<kcg_program*>(cp);
  if (!p) return fail(KCG_E_INVALID_ARGUMENT, "null program");
  if (pred_out && !alpha) return fail(KCG_E_INVALID_ARGUMENT, "alpha required for predictions");
  if (p->low.n_params > 0 && !param_cols) return fail(KCG_E_INVALID_ARGUMENT, "null param_cols");
  return guarded([&] {
    const NvtxRange nvtx_range("kcg_eval_predict");
    require_device();
    if (n == 0) return KCG_OK;
    const int np = p->low.n_params;
    const int F = static_cast<int>(p->low.keys.size());
    if (p->engine == KCG_ENGINE_INTERP) {
      if (!p->dprog && p->dprog_ok) {
        auto img = std::make_unique<KcgDevProg>();
        p->dprog_ok = build_devprog(p->low, *img);
        if (p->dprog_ok) {
          cuda_check(cudaMalloc(&p->dprog, sizeof(KcgDevProg)), "cudaMalloc");
          cuda_check(cudaMemcpy(p->dprog, img.get(), sizeof(KcgDevProg), cudaMemcpyHostToDevice),
                     "cudaMemcpy");
          if (p->low.admit && build_devprog(*p->low.admit, *img)) {
            cuda_check(cudaMalloc(&p->dadmit, sizeof(KcgDevProg)), "cudaMalloc");
            cuda_check(cudaMemcpy(p->dadmit, img.get(), sizeof(KcgDevProg), cudaMemcpyHostToDevice),
                       "cudaMemcpy");
          }
        }
      }
      if (!p->dprog_ok)
        throw KcgError(KCG_E_UNSUPPORTED, "program exceeds the interpreter's static tables");
      kcg::InterpEvalArgs a{};
      for (int j = 0; j < np; ++j) a.p[j] = param_cols[j];
      a.pred = pred_out;
      a.status = status_out;
      a.clo = counts_lo;
      a.chi = counts_hi;
      a.n = static_cast<int64_t>(n);
      a.simulate = simulate;
      compact_alpha(p, alpha, a.alpha);
      kcg::launch_interp_eval(p->dprog, p->dadmit, a, stream);
      ++g_launches;
      return KCG_OK;
    }
    if (!p->jit_eval) {
      const std::string nm = kname("kcg_eval_", p);
      p->jit_eval = kcg::jit_kernel(kcg_program_jit_source(p), nm);
      p->jit_eval_gen = kcg::jit_kernel(kcg_program_jit_source(p), nm + "_gen");
      p->jit_eval_tma = kcg::jit_kernel(kcg_program_jit_source(p), nm + "_tma");
    }
    ArgBuf ab;
    for (int j = 0; j < std::max(np, 1); ++j) ab.push<const void*>(j < np ? param_cols[j] : nullptr);
    ab.push<void*>(pred_out);
    ab.push<void*>(status_out);
    ab.push<void*>(counts_lo);
    ab.push<void*>(counts_hi);
    ab.push<int64_t>(static_cast<int64_t>(n));
    ab.push<int32_t>(simulate);
    // inputs 16-byte aligned: TMA bulk copies / vector loads; outputs
    // aligned: 16-byte prediction stores and 4-byte status stores
    bool vec = true;
    for (int j = 0; j < np; ++j) vec = vec && reinterpret_cast<uintptr_t>(param_cols[j]) % 16 == 0;
    const bool vout = (reinterpret_cast<uintptr_t>(pred_out) % 16 == 0) &&
                      (reinterpret_cast<uintptr_t>(status_out) % 4 == 0);
    ab.push<int32_t>(vec ? 1 : 0);
    ab.push<int32_t>(vout ? 1 : 0);
    std::vector<double> al(std::max(F, 1), 0.0);
    compact_alpha(p, alpha, al.data());
    // finite weights: the skip rules cannot change the sum (GEN = 0 kernel)
    bool finite = true;
    const std::vector<double> alf = folded_alpha(p, al, &finite);
    for (double v : al) ab.push<double>(v);
    for (double v : alf) ab.push<double>(v);
    ab.finish();
    static const bool no_tma = std::getenv("KCG_NO_TMA") != nullptr;
    const size_t tiles = n / kcg::kTmaPointsPerTile;
    if (finite && vec && !no_tma && tiles >= static_cast<size_t>(kcg::num_sms())) {
      // TMA-staged persistent kernel: tma_ctas_per_sm() CTAs per SM
      const unsigned grid = static_cast<unsigned>(
          std::min<size_t>(tiles, static_cast<size_t>(kcg::num_sms()) * kcg::tma_ctas_per_sm()));
      kcg::launch_jit(p->jit_eval_tma, ab.b.data(), ab.b.size(), grid, 256, stream,
                      kcg::tma_smem_bytes(np));
    } else {
      kcg::launch_jit(finite ? p->jit_eval : p->jit_eval_gen, ab.b.data(), ab.b.size(),
                      grid_for((n + 3) / 4), 256, stream);
    }
    ++g_launches;
    return KCG_OK;
  });
}

const char* kcg_multi_jit_source(const kcg_program* const* progs, int V, int argmin) {
  static thread_local std::string src;
  if (!progs || V < 1) return nullptr;
  try {
    std::vector<const kcg::Lowered*> lows;
    std::vector<std::vector<int>> pmaps;
    variant_maps(progs, V, lows, pmaps);
    src = kcg::codegen(lows, pmaps, progs[0]->low.n_params, argmin ? kcg::JitKind::multi_argmin : kcg::JitKind::multi,
                       (argmin ? "kcg_multiam_v" : "kcg_multi_v") + std::to_string(V));
  } catch (const KcgError& e) {
    fail(e.code, e.what());
    return nullptr;
  }
  return src.c_str();
}

}  // extern "C"

namespace {

// One-pass multi-program launch (kcg_eval_predict_multi / kcg_argmin).
// Returns false when the one-pass kernel does not apply (non-finite weights
// or shared products, an interpreter-engine program): the caller falls back.
// The generated source and kernel handles are cached per program set.
struct MultiKey {
  std::vector<uint64_t> uids;
  bool argmin;
  bool operator<(const MultiKey& o) const { return std::tie(uids, argmin) < std::tie(o.uids, o.argmin); }
};
struct MultiEntry {
  std::string src, name;
  kcg::MultiPlan plan;
  std::map<std::string, void*> kernels;  // per kernel name (and device: handles are context-independent)
};

bool launch_multi(const kcg_program* const* progs, int V, const int64_t* const* param_cols, size_t n,
                  const double* alpha, double* pred, size_t ldp, uint8_t* status, size_t lds, int32_t* best,
                  double* best_t, void* stream, bool argmin) {
  std::vector<const kcg::Lowered*> lows;
  std::vector<std::vector<int>> pmaps;
  variant_maps(progs, V, lows, pmaps);
  const int np = progs[0]->low.n_params;
  bool ok = !std::getenv("KCG_NO_MULTI");
  std::vector<std::vector<double>> als(V), alfs(V);
  for (int v = 0; v < V && ok; ++v) {
    als[v].assign(std::max<size_t>(1, progs[v]->low.keys.size()), 0.0);
    compact_alpha(progs[v], alpha, als[v].data());
    bool fin = true;
    alfs[v] = folded_alpha(progs[v], als[v], &fin);
    ok = ok && fin && progs[v]->engine == KCG_ENGINE_JIT;
  }
  if (!ok) return false;
  static std::mutex mu;
  static std::map<MultiKey, std::shared_ptr<MultiEntry>> cache;
  MultiKey key{{}, argmin};
  for (int v = 0; v < V; ++v) key.uids.push_back(progs[v]->uid);
  std::shared_ptr<MultiEntry> e;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) e = it->second;
  }
  if (!e) {
    e = std::make_shared<MultiEntry>();
    e->name = (argmin ? "kcg_multiam_v" : "kcg_multi_v") + std::to_string(V);
    e->src = kcg::codegen(lows, pmaps, np, argmin ? kcg::JitKind::multi_argmin : kcg::JitKind::multi, e->name);
    e->plan = kcg::multi_plan(lows, pmaps, np);
    std::lock_guard<std::mutex> lock(mu);
    if (cache.size() >= 256) cache.clear();  // bounded (program sets of one process)
    cache[key] = e;
  }
  // shared products (multi_plan): alpha (x) constant count; alpha * 2^k
  std::vector<double> shk, shw;
  for (const auto& [schema, c] : e->plan.kprods) shk.push_back(alpha[schema] * static_cast<double>(static_cast<int64_t>(c)));
  for (const auto& [schema, c, m] : e->plan.wprods) {
    shw.push_back(alpha[schema] * static_cast<double>(c));
    if (!std::isfinite(shw.back())) return false;
  }
  bool vec = true;
  for (int j = 0; j < np; ++j) vec = vec && reinterpret_cast<uintptr_t>(param_cols[j]) % 16 == 0;
  static const bool no_tma = std::getenv("KCG_NO_TMA") != nullptr;
  const size_t tiles = n / static_cast<size_t>(kcg::multi_tile());
  const bool tma = vec && !no_tma && np > 0 && tiles >= static_cast<size_t>(kcg::num_sms());
  const bool extra = argmin ? pred != nullptr : status != nullptr;  // _p / _st kernels
  // bulk-store variant: every program's output row 16-byte aligned
  static const bool no_bulk = std::getenv("KCG_MULTI_BULK") && std::string(std::getenv("KCG_MULTI_BULK")) == "0";
  const bool bulk = tma && !argmin && !no_bulk && V <= kcg::multi_bulk_vmax() &&
                    reinterpret_cast<uintptr_t>(pred) % 16 == 0 && ldp % 2 == 0;
  const std::string kname = e->name + (tma ? (bulk ? "_tmab" : "_tma") : "") + (extra ? (argmin ? "_p" : "_st") : "");
  void* k = nullptr;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = e->kernels.find(kname);
    if (it != e->kernels.end()) k = it->second;
  }
  if (!k) {
    k = kcg::jit_kernel(e->src, kname);
    std::lock_guard<std::mutex> lock(mu);
    e->kernels[kname] = k;
  }
  ArgBuf ab;
  for (int j = 0; j < std::max(np, 1); ++j) ab.push<const void*>(j < np ? param_cols[j] : nullptr);
  ab.push<void*>(pred);
  ab.push<void*>(status);
  ab.push<void*>(best);
  ab.push<void*>(best_t);
  ab.push<int64_t>(static_cast<int64_t>(n));
  ab.push<int64_t>(static_cast<int64_t>(ldp));
  ab.push<int64_t>(static_cast<int64_t>(lds));
  for (int v = 0; v < V; ++v)
    for (double x : als[v]) ab.push<double>(x);
  for (int v = 0; v < V; ++v)
    for (double x : alfs[v]) ab.push<double>(x);
  for (double x : shk) ab.push<double>(x);
  if (shk.empty()) ab.push<double>(0.0);
  for (double x : shw) ab.push<double>(x);
  if (shw.empty()) ab.push<double>(0.0);
  ab.finish();
  if (bulk) {
    const unsigned grid = static_cast<unsigned>(
        std::min<size_t>(tiles, static_cast<size_t>(kcg::num_sms()) * kcg::multi_bulk_ctas()));
    kcg::launch_jit(k, ab.b.data(), ab.b.size(), grid, 256, stream, kcg::multi_bulk_smem_bytes(np, V));
  } else if (tma) {
    const unsigned grid = static_cast<unsigned>(
        std::min<size_t>(tiles, static_cast<size_t>(kcg::num_sms()) * kcg::multi_ctas_per_sm(argmin)));
    kcg::launch_jit(k, ab.b.data(), ab.b.size(), grid, 256, stream, kcg::multi_smem_bytes(np, argmin));
  } else {
    kcg::launch_jit(k, ab.b.data(), ab.b.size(), grid_for(n), 256, stream);
  }
  ++g_launches;
  return true;
}

}  // namespace

extern "C" {

int kcg_eval_predict_multi(const kcg_program* const* progs, int V, const int64_t* const* param_cols, size_t n,
                           const double* alpha, double* pred_out, size_t ld_pred, uint8_t* status_out,
                           size_t ld_status, void* stream) {
  if (!progs || V < 1 || !alpha || (!pred_out && !status_out))
    return fail(KCG_E_INVALID_ARGUMENT, "bad multi eval arguments");
  if ((pred_out && ld_pred < n) || (status_out && ld_status < n))
    return fail(KCG_E_INVALID_ARGUMENT, "output leading dimension below n_points");
  return guarded([&] {
    const NvtxRange nvtx_range("kcg_eval_predict_multi");
    require_device();
    std::vector<const kcg::Lowered*> lows;
    std::vector<std::vector<int>> pmaps;
    variant_maps(progs, V, lows, pmaps);
    const int np = progs[0]->low.n_params;
    if (np > 0 && !param_cols) throw KcgError(KCG_E_INVALID_ARGUMENT, "null param_cols");
    if (n == 0) return KCG_OK;
    if (pred_out && launch_multi(progs, V, param_cols, n, alpha, pred_out, ld_pred, status_out, ld_status, nullptr,
                                 nullptr, stream, false))
      return KCG_OK;
    // non-finite weights (skip rules matter), the interpreter engine or
    // status-only calls: one kcg_eval_predict per program (same results)
    for (int v = 0; v < V; ++v) {
      std::vector<const int64_t*> cols(std::max(np, 1), nullptr);
      for (int j = 0; j < progs[v]->low.n_params; ++j) cols[j] = param_cols[pmaps[v][j]];
      const int rc = kcg_eval_predict(progs[v], cols.data(), n, alpha, pred_out ? pred_out + v * ld_pred : nullptr,
                                      status_out ? status_out + v * ld_status : nullptr, nullptr, nullptr, 0, stream);
      if (rc != KCG_OK) throw KcgError(rc, g_last_error);
    }
    return KCG_OK;
  });
}

int kcg_argmin(const kcg_program* const* progs, int V, const int64_t* const* param_cols,
               size_t n, const double* alpha, int32_t* best_idx, double* best_t,
               double* preds_out, void* stream) {
  if (!progs || V < 1 || !alpha || !best_idx || !best_t)
    return fail(KCG_E_INVALID_ARGUMENT, "bad argmin arguments");
  return guarded([&] {
    const NvtxRange nvtx_range("kcg_argmin");
    require_device();
    if (n == 0) return KCG_OK;
    if (progs[0] && progs[0]->low.n_params > 0 && !param_cols)
      throw KcgError(KCG_E_INVALID_ARGUMENT, "null param_cols");
    // the one-pass kernel with the argmin epilogue (KCG_ARGMIN_LEGACY=1: the
    // round-1 grid-stride argmin kernel below)
    static const bool legacy = std::getenv("KCG_ARGMIN_LEGACY") != nullptr;
    if (!legacy && launch_multi(progs, V, param_cols, n, alpha, preds_out, n, nullptr, 0, best_idx, best_t, stream,
                                true))
      return KCG_OK;
    const kcg_program* p0 = progs[0];
    const int np = p0->low.n_params;
    std::vector<const kcg::Lowered*> lows;
    std::vector<std::vector<int>> pmaps;
    std::string name = "kcg_argmin";
    for (int v = 0; v < V; ++v) {
      const kcg_program* p = progs[v];
      if (!p || p->low.n_params != np)
        throw KcgError(KCG_E_INVALID_ARGUMENT, "argmin variants must share the parameter set");
      std::vector<int> map(np);
      for (int j = 0; j < np; ++j) {
        auto it = std::find(p0->param_names.begin(), p0->param_names.end(), p->param_names[j]);
        if (it == p0->param_names.end())
          throw KcgError(KCG_E_INVALID_ARGUMENT, "argmin variants must share the parameter set");
        map[j] = static_cast<int>(it - p0->param_names.begin());
      }
      lows.push_back(&p->low);
      pmaps.push_back(map);
    }
    const std::string src = kcg::codegen(lows, pmaps, np, kcg::JitKind::argmin, name);
    void* k = kcg::jit_kernel(src, name);
    ArgBuf ab;
    for (int j = 0; j < std::max(np, 1); ++j) ab.push<const void*>(j < np ? param_cols[j] : nullptr);
    ab.push<void*>(best_idx);
    ab.push<void*>(best_t);
    ab.push<void*>(preds_out);
    ab.push<int64_t>(static_cast<int64_t>(n));
    // per-variant compact weights in one device buffer: as given (wide
    // path), then folded (fast path, predict_fold); cached per device and
    // weight set (small, reused across sweeps)
    std::vector<double> host;
    std::vector<size_t> off(V), offf(V);
    std::vector<std::vector<double>> alfs(V);
    for (int v = 0; v < V; ++v) {
      std::vector<double> al(std::max<size_t>(1, progs[v]->low.keys.size()), 0.0);
      compact_alpha(progs[v], alpha, al.data());
      bool fin = true;
      alfs[v] = folded_alpha(progs[v], al, &fin);
      if (!fin) throw KcgError(KCG_E_INVALID_ARGUMENT, "argmin requires finite weights");
      off[v] = host.size();
      host.insert(host.end(), al.begin(), al.end());
    }
    for (int v = 0; v < V; ++v) {
      offf[v] = host.size();
      host.insert(host.end(), alfs[v].begin(), alfs[v].end());
    }
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    static std::mutex mu;
    static std::vector<std::tuple<int, std::vector<double>, double*>> cache;
    double* dw = nullptr;
    {
      std::lock_guard<std::mutex> lock(mu);
      for (auto& [d, h, ptr] : cache)
        if (d == dev && h == host) dw = ptr;
      if (!dw) {
        cuda_check(cudaMalloc(&dw, host.size() * sizeof(double)), "cudaMalloc");
        cuda_check(cudaMemcpy(dw, host.data(), host.size() * sizeof(double), cudaMemcpyHostToDevice),
                   "cudaMemcpy");
        if (cache.size() >= 64) {  // bound the cache: drop the oldest set
          cudaFree(std::get<2>(cache.front()));
          cache.erase(cache.begin());
        }
        cache.emplace_back(dev, host, dw);
      }
    }
    for (int v = 0; v < V; ++v) ab.push<const void*>(dw + off[v]);
    for (int v = 0; v < V; ++v) ab.push<const void*>(dw + offf[v]);
    ab.finish();
    kcg::launch_jit(k, ab.b.data(), ab.b.size(), grid_for(n), 256, stream);
    ++g_launches;
    return KCG_OK;
  });
}

}  // extern "C"

namespace {

long long env_ll(const char* name, long long dflt, long long lo, long long hi) {
  const char* e = std::getenv(name);
  if (!e || !*e) return dflt;
  const long long v = std::atoll(e);
  return v < lo ? lo : (v > hi ? hi : v);
}

// Host copies between pageable caller buffers and the pinned staging: a
// persistent pool of threads that split every batch of segments into 2 MB
// parts (spawning threads per copy cost more than the copies themselves)
struct CopySeg {
  void* dst;
  const void* src;
  size_t bytes;
};

class CopyPool {
 public:
  CopyPool() {
    const unsigned T = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    for (unsigned t = 1; t < T; ++t) workers_.emplace_back([this] { work(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  // copies every segment; returns when all are done
  void run(const std::vector<CopySeg>& segs) {
    size_t total = 0;
    for (const CopySeg& g : segs) total += g.bytes;
    if (workers_.empty() || total < (8u << 20)) {
      for (const CopySeg& g : segs) std::memcpy(g.dst, g.src, g.bytes);
      return;
    }
    std::lock_guard<std::mutex> one_batch(run_mu_);  // callers on several devices share the pool
    std::unique_lock<std::mutex> lk(mu_);
    // a worker that woke late for the previous batch may still be scanning it
    done_cv_.wait(lk, [&] { return active_ == 0; });
    parts_.clear();
    for (const CopySeg& g : segs)
      for (size_t o = 0; o < g.bytes; o += kPart)
        parts_.push_back({static_cast<char*>(g.dst) + o, static_cast<const char*>(g.src) + o,
                          std::min(kPart, g.bytes - o)});
    next_.store(0);
    finished_ = 0;
    ++gen_;
    lk.unlock();
    cv_.notify_all();
    drain();
    lk.lock();
    done_cv_.wait(lk, [&] { return finished_ == parts_.size() && active_ == 0; });
  }

 private:
  static constexpr size_t kPart = 2u << 20;
  void drain() {
    size_t mine = 0;
    for (;;) {
      const size_t p = next_.fetch_add(1);
      if (p >= parts_.size()) break;
      std::memcpy(parts_[p].dst, parts_[p].src, parts_[p].bytes);
      ++mine;
    }
    std::lock_guard<std::mutex> lk(mu_);
    finished_ += mine;
    if (finished_ == parts_.size()) done_cv_.notify_all();
  }
  void work() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        ++active_;
      }
      drain();
      std::lock_guard<std::mutex> lk(mu_);
      --active_;
      done_cv_.notify_all();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex run_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  std::vector<CopySeg> parts_;
  std::atomic<size_t> next_{0};
  size_t finished_ = 0;
  unsigned active_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

CopyPool& copy_pool() {
  static CopyPool pool;
  return pool;
}

// per-device streams and staging of kcg_eval_predict_host, kept across calls
// (cudaHostAlloc of ~1 GB costs more than a whole call)
struct HostPipe {
  int slots = 0;
  size_t dev_bytes = 0, host_bytes = 0;
  std::vector<cudaStream_t> streams;
  std::vector<cudaEvent_t> events;
  std::vector<char*> dev, host;
  std::mutex mu;  // one host call per device at a time
  void ensure(int S, size_t dbytes, size_t hbytes) {
    while (slots < S) {
      cudaStream_t s;
      cudaEvent_t e;
      cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
      cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
      streams.push_back(s);
      events.push_back(e);
      dev.push_back(nullptr);
      host.push_back(nullptr);
      ++slots;
    }
    // slots added by a later call with more streams start null: (re)allocate
    // every slot that is missing or smaller than this call needs
    if (dbytes > dev_bytes) {
      for (auto& d : dev) {
        if (d) cudaFree(d);
        d = nullptr;
      }
      dev_bytes = dbytes;
    }
    for (int b = 0; b < slots; ++b)
      if (!dev[b] && dev_bytes > 0) cuda_check(cudaMalloc(&dev[b], dev_bytes), "cudaMalloc");
    if (hbytes > host_bytes) {
      for (auto& h : host) {
        if (h) cudaFreeHost(h);
        h = nullptr;
      }
      host_bytes = hbytes;
    }
    if (hbytes > 0)
      for (int b = 0; b < slots; ++b)
        if (!host[b]) cuda_check(cudaHostAlloc(&host[b], host_bytes, cudaHostAllocDefault), "cudaHostAlloc");
  }
};

HostPipe& host_pipe(int dev) {
  static std::mutex mu;
  static std::vector<std::unique_ptr<HostPipe>> pipes;
  std::lock_guard<std::mutex> lock(mu);
  if (pipes.size() <= static_cast<size_t>(dev)) pipes.resize(dev + 1);
  if (!pipes[dev]) pipes[dev].reset(new HostPipe());
  return *pipes[dev];
}

}  // namespace

extern "C" {

int kcg_eval_predict_host(const kcg_program* const* progs, int V, const int64_t* const* host_cols, size_t n,
                          const double* alpha, double* pred_out, uint8_t* status_out, unsigned flags) {
  if (!progs || V < 1 || !alpha || (!pred_out && !status_out))
    return fail(KCG_E_INVALID_ARGUMENT, "bad host eval arguments");
  return guarded([&] {
    const NvtxRange nvtx_range("kcg_eval_predict_host");
    require_device();
    const kcg_program* p0 = progs[0];
    const int np = p0->low.n_params;
    if (np > 0 && !host_cols) throw KcgError(KCG_E_INVALID_ARGUMENT, "null host_cols");
    std::vector<std::vector<int>> maps(V);
    for (int v = 0; v < V; ++v) {
      const kcg_program* p = progs[v];
      if (!p || p->low.n_params != np)
        throw KcgError(KCG_E_INVALID_ARGUMENT, "host eval programs must share the parameter set");
      maps[v].resize(np);
      for (int j = 0; j < np; ++j) {
        auto it = std::find(p0->param_names.begin(), p0->param_names.end(), p->param_names[j]);
        if (it == p0->param_names.end())
          throw KcgError(KCG_E_INVALID_ARGUMENT, "host eval programs must share the parameter set");
        maps[v][j] = static_cast<int>(it - p0->param_names.begin());
      }
    }
    if (n == 0) return KCG_OK;
    const bool pinned = (flags & KCG_HOST_PINNED) != 0;
    const size_t chunk = std::min<size_t>(n, static_cast<size_t>(env_ll("KCG_HOST_CHUNK", 1 << 22, 1024, 1ll << 28)));
    const int S = static_cast<int>(env_ll("KCG_HOST_STREAMS", 3, 1, 8));
    // pinned callers: one 2D D2H copy per chunk for all programs (KCG_HOST_2D=0: one per program)
    // cudaMemcpy2DAsync rejects a pitch above cudaDevAttrMaxPitch (2^31 - 1
    // on current parts): n * 8 must fit, else one 1D copy per program
    // (KCG_HOST_MAX_PITCH lowers the limit for tests of the fallback)
    int max_pitch = 0, cur_dev = 0;
    cuda_check(cudaGetDevice(&cur_dev), "cudaGetDevice");
    cuda_check(cudaDeviceGetAttribute(&max_pitch, cudaDevAttrMaxPitch, cur_dev), "cudaDeviceGetAttribute");
    const long long pitch_cap = env_ll("KCG_HOST_MAX_PITCH", max_pitch, 8, max_pitch);
    const bool copy2d = env_ll("KCG_HOST_2D", 1, 0, 1) == 1 && n * 8 <= static_cast<unsigned long long>(pitch_cap);
    // several programs: one kcg_eval_predict_multi per chunk (KCG_HOST_ONEPASS=0: one launch per program)
    const bool onepass = V > 1 && pred_out && env_ll("KCG_HOST_ONEPASS", 1, 0, 1) == 1;
    // slot layout: np binding columns, V prediction columns, V status columns
    const size_t in_b = static_cast<size_t>(std::max(np, 1)) * chunk * 8;
    const size_t pred_b = pred_out ? static_cast<size_t>(V) * chunk * 8 : 0;
    const size_t st_b = status_out ? static_cast<size_t>(V) * chunk : 0;
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    HostPipe& hp = host_pipe(dev);
    std::lock_guard<std::mutex> lock(hp.mu);
    hp.ensure(S, in_b + pred_b + st_b, pinned ? 0 : in_b + pred_b + st_b);
    std::vector<size_t> busy_c0(S), busy_m(S, 0);
    auto unstage = [&](int b) {  // the slot's results: pinned staging -> caller
      cuda_check(cudaEventSynchronize(hp.events[b]), "cudaEventSynchronize");
      const size_t c0 = busy_c0[b], m = busy_m[b];
      busy_m[b] = 0;
      if (pinned || m == 0) return;
      std::vector<CopySeg> segs;
      for (int v = 0; v < V; ++v) {
        if (pred_out) segs.push_back({pred_out + v * n + c0, hp.host[b] + in_b + v * chunk * 8, m * 8});
        if (status_out) segs.push_back({status_out + v * n + c0, hp.host[b] + in_b + pred_b + v * chunk, m});
      }
      copy_pool().run(segs);
    };
    // on any failure, let the in-flight copies finish before the staging can
    // be reused or freed by a later call
    try {
      for (size_t k = 0, c0 = 0; c0 < n; ++k, c0 += chunk) {
        const int b = static_cast<int>(k % S);
        unstage(b);
        const size_t m = std::min(chunk, n - c0);
        cudaStream_t st = hp.streams[b];
        char* d = hp.dev[b];
        char* h = pinned ? nullptr : hp.host[b];
        if (!pinned) {
          std::vector<CopySeg> segs;
          for (int j = 0; j < np; ++j) segs.push_back({h + j * chunk * 8, host_cols[j] + c0, m * 8});
          copy_pool().run(segs);
        }
        for (int j = 0; j < np; ++j) {
          const void* src = pinned ? static_cast<const void*>(host_cols[j] + c0) : h + j * chunk * 8;
          cuda_check(cudaMemcpyAsync(d + j * chunk * 8, src, m * 8, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync H2D");
        }
        if (onepass) {  // every program in one launch: the chunk's bindings read once
          std::vector<const int64_t*> cols(std::max(np, 1), nullptr);
          for (int j = 0; j < np; ++j) cols[j] = reinterpret_cast<const int64_t*>(d + j * chunk * 8);
          const int rc = kcg_eval_predict_multi(
              progs, V, cols.data(), m, alpha, pred_out ? reinterpret_cast<double*>(d + in_b) : nullptr, chunk,
              status_out ? reinterpret_cast<uint8_t*>(d + in_b + pred_b) : nullptr, chunk, st);
          if (rc != KCG_OK) throw KcgError(rc, g_last_error);
        }
        for (int v = 0; v < V; ++v) {
          double* dp = pred_out ? reinterpret_cast<double*>(d + in_b + v * chunk * 8) : nullptr;
          uint8_t* ds = status_out ? reinterpret_cast<uint8_t*>(d + in_b + pred_b + v * chunk) : nullptr;
          if (!onepass) {
            std::vector<const int64_t*> cols(std::max(np, 1), nullptr);
            for (int j = 0; j < np; ++j) cols[j] = reinterpret_cast<const int64_t*>(d + maps[v][j] * chunk * 8);
            const int rc = kcg_eval_predict(progs[v], cols.data(), m, alpha, dp, ds, nullptr, nullptr, 0, st);
            if (rc != KCG_OK) throw KcgError(rc, g_last_error);
          }
          if (pred_out && !(pinned && copy2d))
            cuda_check(cudaMemcpyAsync(pinned ? static_cast<void*>(pred_out + v * n + c0) : h + in_b + v * chunk * 8, dp,
                                       m * 8, cudaMemcpyDeviceToHost, st),
                       "cudaMemcpyAsync D2H");
          if (status_out)
            cuda_check(cudaMemcpyAsync(pinned ? static_cast<void*>(status_out + v * n + c0) : h + in_b + pred_b + v * chunk,
                                       ds, m, cudaMemcpyDeviceToHost, st),
                       "cudaMemcpyAsync D2H");
        }
        if (pred_out && pinned && copy2d)  // all programs' predictions of the chunk in one copy
          cuda_check(cudaMemcpy2DAsync(pred_out + c0, n * 8, d + in_b, chunk * 8, m * 8, V, cudaMemcpyDeviceToHost, st),
                     "cudaMemcpy2DAsync D2H");
        cuda_check(cudaEventRecord(hp.events[b], st), "cudaEventRecord");
        busy_c0[b] = c0;
        busy_m[b] = m;
      }
      const size_t nch = (n + chunk - 1) / chunk;
      for (size_t k = nch > static_cast<size_t>(S) ? nch - S : 0; k < nch; ++k) unstage(static_cast<int>(k % S));
    } catch (...) {
      for (int b = 0; b < S; ++b) cudaStreamSynchronize(hp.streams[b]);
      throw;
    }
    g_host_last_path = (pinned ? KCG_HOST_PINNED : 0u) | (pinned && copy2d && pred_out ? KCG_HOST_PATH_2D : 0u) |
                       (onepass ? KCG_HOST_PATH_ONEPASS : 0u);
    return KCG_OK;
  });
}

unsigned kcg_host_last_path(void) { return g_host_last_path.load(); }

int kcg_gram_accumulate(const double* X, size_t n, int F, size_t ld, double* G, double* xt1,
                        double* colmax, void* stream) {
  if (!X || !G || !xt1 || !colmax || ld < static_cast<size_t>(F))
    return fail(KCG_E_INVALID_ARGUMENT, "bad gram arguments");
  return guarded([&] {
    const NvtxRange nvtx_range("kcg_gram_accumulate");
    require_device();
    static const bool no_wide = std::getenv("KCG_NO_WIDE_DMMA") != nullptr;  // A/B knob
    // F <= KCG_DMMA_MAXF (default 72): the row-split DMMA kernel (one CTA per
    // SM from F = 49); wider: one specialisation per width
    static const long long row_split_max = env_ll("KCG_DMMA_MAXF", 72, 48, 72);
    if (!no_wide && F > row_split_max && F <= 160 && ld == static_cast<size_t>(F) &&
        reinterpret_cast<uintptr_t>(X) % 16 == 0 && n >= 32) {
      static const bool grouped = env_ll("KCG_WIDE_GROUPED", 1, 0, 1) == 1;
      if (grouped) {
        // block-run groups x row-split warps (one CTA per SM), rows shared via L2
        const std::string name = "kcg_gram_group_" + std::to_string(F);
        void* k = kcg::jit_kernel(kcg::gram_group_source(F, name), name);
        struct {
          const double* X;
          int64_t n;
          double *G, *xt1, *cmax;
        } args{X, static_cast<int64_t>(n), G, xt1, colmax};
        const int NGr = kcg::gram_group_count(F);
        const size_t tiles = std::max<size_t>(1, n / 64);
        const size_t per = std::max<size_t>(1, std::min<size_t>(tiles, static_cast<size_t>(kcg::num_sms()) / NGr));
        void* argv[] = {&args.X, &args.n, &args.G, &args.xt1, &args.cmax};
        kcg::launch_jit_argv(k, argv, static_cast<unsigned>(per * NGr), 256, stream, kcg::gram_group_smem(F));
        ++g_launches;
        return KCG_OK;
      }
      // wide design on the tensor cores: one NVRTC specialisation per width
      const std::string name = "kcg_gram_wide_" + std::to_string(F);
      void* k = kcg::jit_kernel(kcg::gram_wide_source(F, name), name);
      struct {
        const double* X;
        int64_t n;
        double *G, *xt1, *cmax;
      } args{X, static_cast<int64_t>(n), G, xt1, colmax};
      const size_t tiles = n / 32;
      const unsigned grid = static_cast<unsigned>(
          std::max<size_t>(1, std::min<size_t>(tiles, static_cast<size_t>(kcg::num_sms()) * kcg::gram_wide_ctas(F))));
      void* argv[] = {&args.X, &args.n, &args.G, &args.xt1, &args.cmax};
      kcg::launch_jit_argv(k, argv, grid, 32 * kcg::gram_wide_warps(F), stream, kcg::gram_wide_smem(F));
      ++g_launches;
      return KCG_OK;
    }
    kcg::launch_gram(X, n, F, ld, G, xt1, colmax, stream);
    ++g_launches;
    return KCG_OK;
  });
}

int kcg_gram_accumulate_sliced(const double* X, size_t n, int F, size_t ld, double* G, double* xt1,
                               double* colmax, void* stream) {
  if (!X || !G || !xt1 || !colmax || F < 17 || F > 40 || ld != static_cast<size_t>(F) ||
      reinterpret_cast<uintptr_t>(X) % 16 != 0)
    return fail(KCG_E_INVALID_ARGUMENT, "sliced gram: needs 17 <= n_cols <= 40, ld == n_cols, 16-byte aligned X");
  return guarded([&] {
    const NvtxRange nvtx_range("kcg_gram_accumulate_sliced");
    require_device();
    if (n == 0) return KCG_OK;
    kcg::launch_gram_sliced(X, n, F, G, xt1, colmax, static_cast<cudaStream_t>(stream));
    ++g_launches;
    return KCG_OK;
  });
}

namespace {

// Fused Gram / residual for programs whose design rows stay wider than 48
// columns even over the monomial basis: a register-resident row of that
// width would spill (and takes NVRTC minutes to compile), so rows are
// formed in HBM chunk by chunk -- exact counts (eval kernel), then
// x = RN(count) / T (kcg_form_rows) -- and reduced by the materialised-X
// kernels (per-width DMMA Gram, residual). Same statistics as the fused path.
constexpr size_t kWideChunk = 1 << 18;

bool fused_too_wide(const kcg_program* p) {
  return kcg::gram_basis(p->low).width(static_cast<int>(p->low.keys.size())) > 48;
}

void chunked_rows(const kcg_program* p, const int64_t* const* param_cols, const double* T, size_t n,
                  unsigned long long* bad_rows, void* stream, const std::function<void(const double*, size_t)>& reduce) {
  const int np = p->low.n_params;
  const int F = static_cast<int>(p->low.keys.size());
  const size_t chunk = std::min(n, kWideChunk);
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  void* buf = nullptr;
  const size_t bytes = chunk * (8 * F * 3 + 1) + 64;
  cuda_check(cudaMallocAsync(&buf, bytes, st), "cudaMallocAsync");
  int64_t* lo = static_cast<int64_t*>(buf);
  int64_t* hi = lo + chunk * F;
  double* X = reinterpret_cast<double*>(hi + chunk * F);
  uint8_t* status = reinterpret_cast<uint8_t*>(X + chunk * F);
  try {
    std::vector<const int64_t*> cols(std::max(np, 1), nullptr);
    for (size_t c0 = 0; c0 < n; c0 += chunk) {
      const size_t m = std::min(chunk, n - c0);
      for (int j = 0; j < np; ++j) cols[j] = param_cols[j] + c0;
      const int rc = kcg_eval_predict(p, cols.data(), m, nullptr, nullptr, status, lo, hi, 0, stream);
      if (rc != KCG_OK) throw KcgError(rc, kcg_last_error());
      kcg::launch_form_rows(lo, hi, status, T + c0, m, F, X, bad_rows, stream);
      reduce(X, m);
    }
  } catch (...) {
    cudaFreeAsync(buf, st);
    throw;
  }
  cuda_check(cudaFreeAsync(buf, st), "cudaFreeAsync");
}

}  // namespace

namespace {
// CTAs per SM a persistent fused kernel launches: its register-cap target,
// but no more than shared memory lets reside at once (a grid beyond that
// runs a second wave that starts only when the first has finished its whole
// share of the tiles). The HBM-bound fused Gram and residual showed no
// difference (profiles/ab_fused_grid.sh); the FP64-bound refinement
// gradient uses it
int resident_ctas(int want, size_t smem) {
  const int fit = static_cast<int>((228u * 1024u) / (smem + 1024u));
  return std::max(1, std::min(want, fit));
}
}  // namespace

int kcg_gram_fused(const kcg_program* cp, const int64_t* const* param_cols, const double* T,
                   size_t n, double* G, double* xt1, double* colmax,
                   unsigned long long* bad_rows, void* stream) {
  kcg_program* p = const_cast<kcg_program*>(cp);
  if (!p || !T || !G || !xt1 || !colmax) return fail(KCG_E_INVALID_ARGUMENT, "bad gram arguments");
  return guarded([&] {
    const NvtxRange nvtx_range("kcg_gram_fused");
    require_device();
    if (n == 0) return KCG_OK;
    const int np = p->low.n_params;
    if (fused_too_wide(p)) {
      const int F = static_cast<int>(p->low.keys.size());
      chunked_rows(p, param_cols, T, n, bad_rows, stream, [&](const double* X, size_t m) {
        const int rc = kcg_gram_accumulate(X, m, F, F, G, xt1, colmax, stream);
        if (rc != KCG_OK) throw KcgError(rc, kcg_last_error());
      });
      return KCG_OK;
    }
    if (!p->jit_gram) {
      const std::string name = kname("kcg_gram_", p);
      p->jit_gram = kcg::jit_kernel(
          kcg::codegen({&p->low}, {identity(np)}, np, kcg::JitKind::gram, name), name);
    }
    ArgBuf ab;
    for (int j = 0; j < std::max(np, 1); ++j) ab.push<const void*>(j < np ? param_cols[j] : nullptr);
    ab.push<const void*>(T);
    ab.push<void*>(G);
    ab.push<void*>(xt1);
    ab.push<void*>(colmax);
    ab.push<void*>(bad_rows);
    ab.push<int64_t>(static_cast<int64_t>(n));
    bool vec = reinterpret_cast<uintptr_t>(T) % 16 == 0;
    for (int j = 0; j < np; ++j) vec = vec && reinterpret_cast<uintptr_t>(param_cols[j]) % 16 == 0;
    ab.push<int32_t>(vec ? 1 : 0);
    ab.finish();
    // persistent TMA-streamed kernel (2 CTAs/SM for the DMMA variant)
    kcg::launch_jit(p->jit_gram, ab.b.data(), ab.b.size(), kcg::num_sms() * kcg::fused_ctas_per_sm(p->low, true), 256, stream,
                    kcg::fused_smem_bytes(np, p->low, true));
    ++g_launches;
    return KCG_OK;
  });
}

int kcg_residual_accumulate(const double* X, size_t n, int F, size_t ld, const double* alpha,
                            double* obj, void* stream) {
  if (!X || !alpha || !obj || ld < static_cast<size_t>(F))
    return fail(KCG_E_INVALID_ARGUMENT, "bad residual arguments");
  return guarded([&] {
    const NvtxRange nvtx_range("kcg_residual_accumulate");
    require_device();
    kcg::launch_residual(X, n, F, ld, alpha, obj, stream);
    ++g_launches;
    return KCG_OK;
  });
}

int kcg_gram_residual_grad(const double* X, size_t n, int F, size_t ld, const double* alpha,
                           double* g, void* stream) {
  if (!X || !alpha || !g || ld < static_cast<size_t>(F))
    return fail(KCG_E_INVALID_ARGUMENT, "bad residual arguments");
  return guarded([&] {
    const NvtxRange nvtx_range("kcg_gram_residual_grad");
    require_device();
    kcg::launch_residual_grad(X, n, F, ld, alpha, g, stream);
    ++g_launches;
    return KCG_OK;
  });
}

int kcg_residual_fused(const kcg_program* cp, const int64_t* const* param_cols, const double* T,
                       size_t n, const double* alpha, double* obj, void* stream) {
  kcg_program* p = const_cast<kcg_program*>(cp);
  if (!p || !T || !alpha || !obj) return fail(KCG_E_INVALID_ARGUMENT, "bad residual arguments");
  return guarded([&] {
    const NvtxRange nvtx_range("kcg_residual_fused");
    require_device();
    if (n == 0) return KCG_OK;
    const int np = p->low.n_params;
    const int F = static_cast<int>(p->low.keys.size());
    if (fused_too_wide(p)) {
      std::vector<double> al(std::max(F, 1), 0.0);
      compact_alpha(p, alpha, al.data());
      double* da = nullptr;
      cuda_check(cudaMallocAsync(&da, sizeof(double) * al.size(), static_cast<cudaStream_t>(stream)), "cudaMallocAsync");
      cuda_check(cudaMemcpyAsync(da, al.data(), sizeof(double) * al.size(), cudaMemcpyHostToDevice,
                                 static_cast<cudaStream_t>(stream)), "cudaMemcpyAsync");
      chunked_rows(p, param_cols, T, n, nullptr, stream, [&](const double* X, size_t m) {
        const int rc = kcg_residual_accumulate(X, m, F, F, da, obj, stream);
        if (rc != KCG_OK) throw KcgError(rc, kcg_last_error());
      });
      cuda_check(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "residual");  // al outlives the copy
      cudaFreeAsync(da, static_cast<cudaStream_t>(stream));
      return KCG_OK;
    }
    if (!p->jit_resid) {
      const std::string name = kname("kcg_resid_", p);
      p->jit_resid = kcg::jit_kernel(
          kcg::codegen({&p->low}, {identity(np)}, np, kcg::JitKind::residual, name), name);
    }
    ArgBuf ab;
    for (int j = 0; j < std::max(np, 1); ++j) ab.push<const void*>(j < np ? param_cols[j] : nullptr);
    ab.push<const void*>(T);
    ab.push<void*>(obj);
    ab.push<int64_t>(static_cast<int64_t>(n));
    bool vec = reinterpret_cast<uintptr_t>(T) % 16 == 0;
    for (int j = 0; j < np; ++j) vec = vec && reinterpret_cast<uintptr_t>(param_cols[j]) % 16 == 0;
    ab.push<int32_t>(vec ? 1 : 0);
    std::vector<double> al(std::max(F, 1), 0.0);
    compact_alpha(p, alpha, al.data());
    const kcg::GramBasis gb = kcg::gram_basis(p->low);
    if (gb.reduced) {
      // x . alpha = sum_b u_b * beta_b with beta_b = sum_j alpha_j A_jb
      std::vector<double> beta(gb.monos.size(), 0.0);
      for (int j = 0; j < F; ++j)
        for (const auto& [b, c] : gb.terms[j]) beta[b] += al[j] * c;
      al.assign(std::max(F, 1), 0.0);
      std::copy(beta.begin(), beta.end(), al.begin());
    }
    for (double v : al) ab.push<double>(v);
    ab.finish();
    kcg::launch_jit(p->jit_resid, ab.b.data(), ab.b.size(), kcg::num_sms() * kcg::fused_ctas_per_sm(p->low, false), 256, stream,
                    kcg::fused_smem_bytes(np, p->low, false));
    ++g_launches;
    return KCG_OK;
  });
}

int kcg_residual_grad_fused(const kcg_program* cp, const int64_t* const* param_cols, const double* T, size_t n,
                            const double* alpha, double* g, void* stream) {
  return kcg_residual_grad_obj_fused(cp, param_cols, T, n, alpha, g, nullptr, stream);
}

int kcg_residual_grad_obj_fused(const kcg_program* cp, const int64_t* const* param_cols, const double* T, size_t n,
                                const double* alpha, double* g, double* r2, void* stream) {
  kcg_program* p = const_cast<kcg_program*>(cp);
  if (!p || !T || !alpha || !g) return fail(KCG_E_INVALID_ARGUMENT, "bad residual-gradient arguments");
  return guarded([&] {
    const NvtxRange nvtx_range("kcg_residual_grad_fused");
    require_device();
    if (n == 0) return KCG_OK;
    const int np = p->low.n_params;
    const int F = static_cast<int>(p->low.keys.size());
    std::vector<double> al(std::max(F, 1), 0.0);
    compact_alpha(p, alpha, al.data());
    if (F > 48) {  // rows in HBM chunk by chunk (as the wide fused Gram)
      double* da = nullptr;
      cuda_check(cudaMallocAsync(&da, sizeof(double) * al.size(), static_cast<cudaStream_t>(stream)), "cudaMallocAsync");
      cuda_check(cudaMemcpyAsync(da, al.data(), sizeof(double) * al.size(), cudaMemcpyHostToDevice,
                                 static_cast<cudaStream_t>(stream)), "cudaMemcpyAsync");
      chunked_rows(p, param_cols, T, n, nullptr, stream, [&](const double* X, size_t m) {
        int rc = kcg_gram_residual_grad(X, m, F, F, da, g, stream);
        if (rc == KCG_OK && r2) rc = kcg_residual_accumulate(X, m, F, F, da, r2, stream);
        if (rc != KCG_OK) throw KcgError(rc, kcg_last_error());
      });
      cuda_check(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "residual grad");
      cudaFreeAsync(da, static_cast<cudaStream_t>(stream));
      return KCG_OK;
    }
    if (!p->jit_rgrad) {
      const std::string name = kname("kcg_rgrad_", p);
      p->jit_rgrad = kcg::jit_kernel(
          kcg::codegen({&p->low}, {identity(np)}, np, kcg::JitKind::residual_grad, name), name);
    }
    ArgBuf ab;
    for (int j = 0; j < std::max(np, 1); ++j) ab.push<const void*>(j < np ? param_cols[j] : nullptr);
    ab.push<const void*>(T);
    ab.push<void*>(g);
    ab.push<void*>(r2);
    ab.push<int64_t>(static_cast<int64_t>(n));
    bool vec = reinterpret_cast<uintptr_t>(T) % 16 == 0;
    for (int j = 0; j < np; ++j) vec = vec && reinterpret_cast<uintptr_t>(param_cols[j]) % 16 == 0;
    ab.push<int32_t>(vec ? 1 : 0);
    // per group: A_g = sum_j 2^k_j alpha_j as a double-double (hi, lo)
    const kcg::RGradGroups rg = kcg::rgrad_groups(p->low);
    const size_t G = rg.base.size();
    std::vector<double> ahi(std::max<size_t>(G, 1), 0.0), alo(std::max<size_t>(G, 1), 0.0);
    for (int j = 0; j < F; ++j) {
      const auto [g, k] = rg.of_key[j];
      const double b = std::ldexp(al[j], k);
      const double s = ahi[g] + b, bb = s - ahi[g];
      const double e = (ahi[g] - (s - bb)) + (b - bb);
      const double lo = alo[g] + e;
      ahi[g] = s + lo;
      alo[g] = lo - (ahi[g] - s);
    }
    for (double v : ahi) ab.push<double>(v);
    for (double v : alo) ab.push<double>(v);
    ab.finish();
    // grid: the CTAs that are resident at once (the persistent loop's stride);
    // the register cap (__launch_bounds__) may ask for more than shared
    // memory admits (a second wave of CTAs would start only after the first
    // finished its whole share)
    const size_t rg_smem = kcg::fused_smem_bytes(np, p->low, false, true);
    static const int grid_ctas_env = static_cast<int>(env_ll("KCG_RGRAD_GRID", 0, 0, 8));
    const int grid_ctas = grid_ctas_env ? grid_ctas_env : resident_ctas(kcg::rgrad_ctas_per_sm(), rg_smem);
    kcg::launch_jit(p->jit_rgrad, ab.b.data(), ab.b.size(), kcg::num_sms() * grid_ctas, 256, stream, rg_smem);
    ++g_launches;
    return KCG_OK;
  });
}

int kcg_simulate_time(const kcg_program* cp, const int64_t* const* param_cols, size_t n,
                      const double* alpha, double sigma, uint64_t seed, uint64_t run,
                      double* times_out, uint8_t* status_out, void* stream) {
  kcg_program* p = const_cast<kcg_program*>(cp);
  if (!p || !alpha || !times_out) return fail(KCG_E_INVALID_ARGUMENT, "bad simulate arguments");
  const int rc = kcg_eval_predict(cp, param_cols, n, alpha, times_out, status_out, nullptr, nullptr,
                                  /*simulate=*/1, stream);
  if (rc != KCG_OK || sigma == 0.0 || n == 0) return rc;  // simdevice.cpp:99
  return guarded([&] {
    const NvtxRange nvtx_range("kcg_simulate_time");
    kcg::NoiseArgs a{};
    const int np = p->low.n_params;
    std::vector<int> order(np);
    for (int j = 0; j < np; ++j) order[j] = j;
    std::sort(order.begin(), order.end(),
              [&](int x, int y) { return p->param_names[x] < p->param_names[y]; });
    for (int k = 0; k < np; ++k) {
      const std::string seg = (k ? ";" : "") + p->param_names[order[k]] + "=";
      if (seg.size() > sizeof(a.seg[0])) throw KcgError(KCG_E_UNSUPPORTED, "parameter name too long");
      std::memcpy(a.seg[k], seg.data(), seg.size());
      a.seg_len[k] = static_cast<int>(seg.size());
      a.cols[k] = param_cols[order[k]];
    }
    a.n_params = np;
    uint64_t h = 1469598103934665603ull;  // fnv1a(kernel + "|"), simdevice.cpp:23-30
    for (unsigned char c : p->sym.kernel + "|") {
      h ^= c;
      h *= 1099511628211ull;
    }
    a.prefix_hash = h;
    a.seed = seed;
    a.counter = run;
    a.sigma = sigma;
    a.t = times_out;
    a.n = static_cast<int64_t>(n);
    kcg::launch_noise(a, stream);
    ++g_launches;
    return KCG_OK;
  });
}

int kcg_geomean_accumulate(const double* pred, const double* actual, size_t n, double* log_sum,
                           unsigned long long* count, unsigned long long* bad, void* stream) {
  if (!pred || !actual || !log_sum || !count || !bad)
    return fail(KCG_E_INVALID_ARGUMENT, "bad geomean arguments");
  return guarded([&] {
    const NvtxRange nvtx_range("kcg_geomean_accumulate");
    require_device();
    kcg::launch_geomean(pred, actual, n, log_sum, count, bad, stream);
    ++g_launches;
    return KCG_OK;
  });
}

int kcg_solve_gram(int F, const double* G, const double* xt1, const double* colmax,
                   double* alpha_out, int* rank_out) {
  if (F < 1 || !G || !xt1 || !colmax || !alpha_out)
    return fail(KCG_E_INVALID_ARGUMENT, "bad solve arguments");
  return guarded([&] {
    const NvtxRange nvtx_range("kcg_solve_gram");
    std::vector<double> x;
    const int r = solve_equilibrated(F, G, colmax, xt1, x);
    std::copy(x.begin(), x.end(), alpha_out);
    if (rank_out) *rank_out = r;
    return KCG_OK;
  });
}

int kcg_refine_gram(int F, const double* G, const double* colmax, const double* g,
                    double* alpha) {
  if (F < 1 || !G || !colmax || !g || !alpha)
    return fail(KCG_E_INVALID_ARGUMENT, "bad refine arguments");
  return guarded([&] {
    const NvtxRange nvtx_range("kcg_refine_gram");
    std::vector<double> dx;
    solve_equilibrated(F, G, colmax, g, dx);
    for (int j = 0; j < F; ++j)
      if (colmax[j] > 0.0) alpha[j] += dx[j];
    return KCG_OK;
  });
}

int kcg_weights_read_json(const char* path, double* alpha, uint8_t* covered, double* objective,
                          uint64_t* n_cases) {
  if (!path || !alpha || !covered) return fail(KCG_E_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw KcgError(KCG_E_IO, std::string("cannot open: ") + path);
    nlohmann::json j;
    try {
      j = nlohmann::json::parse(in);
    } catch (const nlohmann::json::exception& e) {
      throw KcgError(KCG_E_PARSE, std::string(path) + ": " + e.what());
    }
    try {
      const std::string ver = j.at("schema_version").get<std::string>();
      if (ver != "v1")
        throw KcgError(KCG_E_SCHEMA_MISMATCH,
                       std::string(path) + ": schema '" + ver + "', expected 'v1'");
      const int K = kcg_schema_size();
      std::fill(alpha, alpha + K, 0.0);
      std::fill(covered, covered + K, 0);
      for (const auto& [key, val] : j.at("weights").items()) {
        const int i = kcg::schema_index(key);
        if (i < 0) throw KcgError(KCG_E_SCHEMA_MISMATCH, "unknown property key '" + key + "'");
        alpha[i] = val.get<double>();
        covered[i] = 1;
      }
      if (j.contains("covered"))
        for (const auto& [key, val] : j.at("covered").items()) {
          const int i = kcg::schema_index(key);
          if (i < 0) throw KcgError(KCG_E_SCHEMA_MISMATCH, "unknown property key '" + key + "'");
          covered[i] = val.get<bool>() ? 1 : 0;
        }
      if (objective) *objective = j.contains("fit") ? j["fit"].value("objective", 0.0) : 0.0;
      if (n_cases) *n_cases = j.contains("fit") ? j["fit"].value("n_cases", uint64_t{0}) : 0;
    } catch (const nlohmann::json::exception& e) {
      throw KcgError(KCG_E_PARSE, std::string(path) + ": " + e.what());
    }
    return KCG_OK;
  });
}

int kcg_weights_write_json(const char* path, const char* device, const double* alpha,
                           const uint8_t* covered, double objective, uint64_t n_cases) {
  if (!path || !alpha || !covered) return fail(KCG_E_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    nlohmann::json weights = nlohmann::json::object(), cov = nlohmann::json::object();
    const auto& keys = kcg::schema_keys();
    for (size_t i = 0; i < keys.size(); ++i) {
      weights[keys[i]] = alpha[i];
      cov[keys[i]] = static_cast<bool>(covered[i]);
    }
    nlohmann::json out;
    out["device"] = device ? device : "";
    out["schema_version"] = "v1";
    out["weights"] = weights;
    out["covered"] = cov;
    out["fit"] = {{"objective", objective}, {"n_cases", n_cases}};
    const std::string tmp = std::string(path) + ".tmp";
    {
      std::ofstream o(tmp, std::ios::binary | std::ios::trunc);
      if (!o) throw KcgError(KCG_E_IO, "cannot open for writing: " + tmp);
      o << out.dump(2) << "\n";
      if (!o.flush()) throw KcgError(KCG_E_IO, "write failed: " + tmp);
    }
    if (std::rename(tmp.c_str(), path) != 0)
      throw KcgError(KCG_E_IO, "cannot rename " + tmp + " to " + path);
    return KCG_OK;
  });
}

const char* kcg_status_str(int s) {
  switch (s) {
    case KCG_OK: return "OK";
    case KCG_E_PARSE: return "E_PARSE";
    case KCG_E_NEEDS_BINDING: return "E_NEEDS_BINDING";
    case KCG_E_NEEDS_FALLBACK: return "E_NEEDS_FALLBACK";
    case KCG_E_CAP_EXCEEDED: return "E_CAP_EXCEEDED";
    case KCG_E_TYPE_CONFLICT: return "E_TYPE_CONFLICT";
    case KCG_E_ASSUMPTION_VIOLATED: return "E_ASSUMPTION_VIOLATED";
    case KCG_E_SCHEMA_MISMATCH: return "E_SCHEMA_MISMATCH";
    case KCG_E_NONPOSITIVE_TIME: return "E_NONPOSITIVE_TIME";
    case KCG_E_EMPTY: return "E_EMPTY";
    case KCG_E_IO: return "E_IO";
    case KCG_E_INVALID_ARGUMENT: return "E_INVALID_ARGUMENT";
    case KCG_E_CUDA: return "E_CUDA";
    case KCG_E_JIT: return "E_JIT";
    case KCG_E_UNSUPPORTED: return "E_UNSUPPORTED";
    case KCG_E_INTERNAL: return "E_INTERNAL";
  }
  return "E_UNKNOWN";
}

const char* kcg_point_status_str(int s) {
  switch (s) {
    case KCG_PT_OK: return "OK";
    case KCG_PT_ASSUMPTION_VIOLATED: return "E_ASSUMPTION_VIOLATED";
    case KCG_PT_NONINTEGRAL: return "NONINTEGRAL";
    case KCG_PT_OVERFLOW: return "OVERFLOW";
    case KCG_PT_COUNT_WIDE: return "COUNT_WIDE";
  }
  return "UNKNOWN";
}

const char* kcg_last_error(void) { return g_last_error.c_str(); }

uint64_t kcg_launch_count(void) { return g_launches.load(); }

int kcg_measure_pipe_peak(int kind, uint64_t iters, double* lane_ops_per_s) {
  if (kind < 0 || kind > 3 || iters == 0 || !lane_ops_per_s)
    return fail(KCG_E_INVALID_ARGUMENT, "bad pipe-peak arguments");
  return guarded([&] {
    require_device();
    *lane_ops_per_s = kcg::measure_pipe_peak(kind, iters);
    return KCG_OK;
  });
}

int kcg_measure_stream(int n_read, int n_write, uint64_t n_points, double* bytes_per_s) {
  if (n_read < 0 || n_write < 0 || n_points < 2 || !bytes_per_s)
    return fail(KCG_E_INVALID_ARGUMENT, "bad stream arguments");
  return guarded([&] {
    require_device();
    try {
      *bytes_per_s = kcg::measure_stream(n_read, n_write, n_points);
    } catch (const std::runtime_error& e) {
      throw KcgError(KCG_E_UNSUPPORTED, e.what());
    }
    return KCG_OK;
  });
}

}  // extern "C"

// ---- GPU enumeration oracle --------------------------------------------------

struct kcg_enum_program {
  kcg::EnumSymbolic e;
};

extern "C" {

int kcg_enum_program_create(const char* text, size_t len, kcg_enum_program** out) {
  if (!text || !out) return fail(KCG_E_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  return guarded([&] {
    auto p = std::make_unique<kcg_enum_program>();
    p->e = kcg::parse_enum_text(std::string(text, len));
    *out = p.release();
    return KCG_OK;
  });
}

void kcg_enum_program_destroy(kcg_enum_program* p) { delete p; }

int kcg_enum_program_num_params(const kcg_enum_program* p) { return p ? p->e.n_params : -1; }

const char* kcg_enum_program_param_name(const kcg_enum_program* p, int i) {
  return p && i >= 0 && i < p->e.n_params ? p->e.sym.params[i].c_str() : nullptr;
}

int kcg_enumerate_points(const kcg_enum_program* p, const int64_t* binding, uint64_t cap, int64_t* lo,
                         int64_t* hi, uint64_t* points, void* stream) {
  if (!p || (!binding && p->e.n_params > 0) || !lo || !hi)
    return fail(KCG_E_INVALID_ARGUMENT, "bad enumerate arguments");
  return guarded([&] {
    const NvtxRange nvtx_range("kcg_enumerate_points");
    require_device();
    std::vector<i128> c(kcg::schema_keys().size(), 0);
    const int launches = kcg::enumerate_points(p->e, binding, cap, c.data(), points, stream);
    for (size_t i = 0; i < c.size(); ++i) {
      lo[i] = static_cast<int64_t>(c[i]);
      hi[i] = static_cast<int64_t>(c[i] >> 64);
    }
    g_launches += static_cast<uint64_t>(launches);
    return KCG_OK;
  });
}

}  // extern "C"

// ---- grid descriptors ----------------------------------------------------------

namespace {

// validates the lattice and [first, first + n) against it
void check_grid(const kcg_grid* g, uint64_t first, size_t n) {
  if (!g || g->n_params < 0 || g->n_params > 8) throw KcgError(KCG_E_INVALID_ARGUMENT, "bad grid descriptor");
  unsigned __int128 total = 1;
  for (int j = 0; j < g->n_params; ++j) {
    if (g->count[j] == 0) throw KcgError(KCG_E_INVALID_ARGUMENT, "grid count must be >= 1");
    total *= g->count[j];
    if (total > (static_cast<unsigned __int128>(1) << 64)) throw KcgError(KCG_E_INVALID_ARGUMENT, "grid has more than 2^64 points");
    const i128 last = static_cast<i128>(g->start[j]) + static_cast<i128>(g->step[j]) * static_cast<i128>(g->count[j] - 1);
    if (last > INT64_MAX || last < INT64_MIN) throw KcgError(KCG_E_INVALID_ARGUMENT, "grid values exceed int64");
  }
  if (static_cast<unsigned __int128>(first) + n > total)
    throw KcgError(KCG_E_INVALID_ARGUMENT, "points beyond the end of the grid");
}

}  // namespace

extern "C" {

int kcg_grid_bindings(const kcg_grid* g, uint64_t first, size_t n, int64_t* const* cols, void* stream) {
  return guarded([&] {
    const NvtxRange nvtx_range("kcg_grid_bindings");
    check_grid(g, first, n);
    if (g->n_params > 0 && !cols) throw KcgError(KCG_E_INVALID_ARGUMENT, "null columns");
    require_device();
    if (n == 0 || g->n_params == 0) return KCG_OK;
    kcg::launch_grid_fill(g->n_params, g->start, g->step, g->count, first, n, cols, stream);
    ++g_launches;
    return KCG_OK;
  });
}

int kcg_eval_predict_grid(const kcg_program* cp, const kcg_grid* g, uint64_t first, size_t n,
                          const double* alpha, double* pred_out, uint8_t* status_out, int simulate,
                          void* stream) {
  kcg_program* p = const_cast<kcg_program*>(cp);
  if (!p) return fail(KCG_E_INVALID_ARGUMENT, "null program");
  if (pred_out && !alpha) return fail(KCG_E_INVALID_ARGUMENT, "alpha required for predictions");
  return guarded([&] {
    const NvtxRange nvtx_range("kcg_eval_predict_grid");
    check_grid(g, first, n);
    const int np = p->low.n_params;
    if (g->n_params != np) throw KcgError(KCG_E_INVALID_ARGUMENT, "grid parameter count != program's");
    require_device();
    if (n == 0) return KCG_OK;
    const int F = static_cast<int>(p->low.keys.size());
    if (!p->jit_eval_grid) {
      const std::string nm = kname("kcg_eval_", p);
      p->jit_eval_grid = kcg::jit_kernel(kcg_program_jit_source(p), nm + "_grid");
      p->jit_eval_grid_gen = kcg::jit_kernel(kcg_program_jit_source(p), nm + "_grid_gen");
    }
    const unsigned grid = grid_for((n + 3) / 4);
    ArgBuf ab;
    for (int j = 0; j < std::max(np, 1); ++j) ab.push<const void*>(nullptr);  // KcgArgs.p (unused)
    ab.push<void*>(pred_out);
    ab.push<void*>(status_out);
    ab.push<void*>(nullptr);  // clo
    ab.push<void*>(nullptr);  // chi
    ab.push<int64_t>(static_cast<int64_t>(n));
    ab.push<int32_t>(simulate);
    ab.push<int32_t>(0);  // vec
    const bool vout = (reinterpret_cast<uintptr_t>(pred_out) % 16 == 0) &&
                      (reinterpret_cast<uintptr_t>(status_out) % 4 == 0);
    ab.push<int32_t>(vout ? 1 : 0);
    std::vector<double> al(std::max(F, 1), 0.0);
    compact_alpha(p, alpha, al.data());
    bool finite = true;
    const std::vector<double> alf = folded_alpha(p, al, &finite);
    for (double v : al) ab.push<double>(v);
    for (double v : alf) ab.push<double>(v);
    ab.finish();  // end of the embedded KcgArgs
    const int NP = std::max(np, 1);
    for (int j = 0; j < NP; ++j) ab.push<int64_t>(j < np ? g->start[j] : 0);
    for (int j = 0; j < NP; ++j) ab.push<int64_t>(j < np ? g->step[j] : 0);
    for (int j = 0; j < NP; ++j) ab.push<uint64_t>(j < np ? g->count[j] : 1);
    // digits of the per-step advance 4 * gridDim * blockDim (mod the lattice size)
    uint64_t adv = 4ull * grid * 256ull, dig[8] = {0};
    for (int j = np - 1; j >= 0; --j) {
      dig[j] = adv % g->count[j];
      adv /= g->count[j];
    }
    for (int j = 0; j < NP; ++j) ab.push<uint64_t>(j < np ? dig[j] : 0);
    ab.push<uint64_t>(first);
    ab.finish();
    kcg::launch_jit(finite ? p->jit_eval_grid : p->jit_eval_grid_gen, ab.b.data(), ab.b.size(), grid, 256,
                    stream);
    ++g_launches;
    return KCG_OK;
  });
}

}  // extern "C"

// ---- kcg-columns v1 ----------------------------------------------------------

extern "C" {

int kcg_columns_write(const char* path, int n_cols, const char* const* names, const int* dtypes,
                      const void* const* host_cols, uint64_t n_rows) {
  return guarded([&] {
    kcg::columns_write(path, n_cols, names, dtypes, host_cols, n_rows);
    return KCG_OK;
  });
}

int kcg_columns_open(const char* path, kcg_columns** out) {
  if (!out) return fail(KCG_E_INVALID_ARGUMENT, "null out");
  *out = nullptr;
  return guarded([&] {
    *out = kcg::columns_open(path);
    return KCG_OK;
  });
}

void kcg_columns_close(kcg_columns* c) { delete c; }

uint64_t kcg_columns_num_rows(const kcg_columns* c) { return c ? c->n_rows : 0; }

int kcg_columns_num_cols(const kcg_columns* c) { return c ? static_cast<int>(c->cols.size()) : -1; }

const char* kcg_columns_name(const kcg_columns* c, int j) {
  return c && j >= 0 && j < static_cast<int>(c->cols.size()) ? c->cols[j].name.c_str() : nullptr;
}

int kcg_columns_dtype(const kcg_columns* c, int j) {
  return c && j >= 0 && j < static_cast<int>(c->cols.size()) ? c->cols[j].dtype : -1;
}

int kcg_columns_find(const kcg_columns* c, const char* name) {
  if (!c || !name) return -1;
  for (size_t j = 0; j < c->cols.size(); ++j)
    if (c->cols[j].name == name) return static_cast<int>(j);
  return -1;
}

const void* kcg_columns_data(const kcg_columns* c, int j) {
  return c && j >= 0 && j < static_cast<int>(c->cols.size())
             ? static_cast<const char*>(c->map) + c->cols[j].offset
             : nullptr;
}

int kcg_columns_load(kcg_columns* c, int j, uint64_t row0, size_t n, void* dev, void* stream) {
  return guarded([&] {
    const NvtxRange nvtx_range("kcg_columns_load");
    require_device();
    kcg::columns_load(c, j, row0, n, dev, stream);
    return KCG_OK;
  });
}

}  // extern "C"
