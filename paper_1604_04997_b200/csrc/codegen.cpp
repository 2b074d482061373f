// JIT specialisation: lowered programs -> straight-line CUDA source.
//
// Each program becomes `kcg_body_<v><T>()`, the exact evaluation of its
// admissibility (AssumeCtx::admits, decide.cpp:153-170) and nonzero property
// entries (evaluate_properties, props.cpp:259-271) with every coefficient,
// denominator and modulus a compile-time constant, instantiated for
// T = int64 (fast path) and T = int128 (wide path). The kernels around the
// bodies implement fused evaluate+predict, argmin over variants, and the
// fused design-row Gram / residual reductions.
#include <sstream>

#include "kcg_codegen.hpp"

namespace kcg {

namespace {

const char* kDeviceHelpers =
#include "kcg_device_src.inc"
    ;

std::string lit(i128 v) {
  const int64_t lo = static_cast<int64_t>(v);
  const int64_t hi = static_cast<int64_t>(v >> 64);
  std::ostringstream os;
  if (static_cast<i128>(lo) == v) {
    if (lo == INT64_MIN)
      os << "kcg_const<T>((kcg_i64)0x8000000000000000ull, -1ll)";
    else
      os << "((T)" << lo << "ll)";
  } else {
    os << "kcg_const<T>((kcg_i64)" << static_cast<uint64_t>(lo) << "ull, "
       << hi << "ll)";
  }
  return os.str();
}

const char* cmp_str(int op) {
  switch (op) {
    case 0: return "<";
    case 1: return "<=";
    case 2: return ">";
    case 3: return ">=";
    default: return "==";
  }
}

void emit_body(std::ostringstream& os, const Lowered& L, int v) {
  os << "template <class T>\n__device__ __forceinline__ int kcg_body_" << v
     << "(const kcg_i64* __restrict__ p, T* __restrict__ cnt) {\n";
  for (const LOp& op : L.ops) {
    switch (op.code) {
      case OP_VAR:
        os << "  const T a" << op.dst << " = (T)p[" << op.a << "];\n";
        break;
      case OP_MONO: {
        os << "  const T m" << op.dst << " = ";
        bool first = true;
        for (int i = op.a; i < op.b; ++i)
          for (int k = 0; k < L.factors[i].second; ++k) {
            os << (first ? "" : " * ") << "a" << L.factors[i].first;
            first = false;
          }
        os << ";\n";
        break;
      }
      case OP_EXPR: {
        os << "  const T e" << op.dst << " = ";
        if (op.a == op.b) os << "(T)0";
        for (int i = op.a; i < op.b; ++i) {
          const LTerm& t = L.terms[i];
          if (i != op.a) os << " + ";
          if (t.mono < 0) {
            os << lit(t.coef);
          } else if (t.coef == 1) {
            os << "m" << t.mono;
          } else if (t.coef == -1) {
            os << "(-m" << t.mono << ")";
          } else {
            os << lit(t.coef) << " * m" << t.mono;
          }
        }
        os << ";\n";
        break;
      }
      case OP_FLOORDIV:
        os << "  const T a" << op.dst << " = kcg_floordiv<T>(e" << op.a << ", "
           << lit(L.floordiv_den[op.c]) << ");\n";
        break;
      case OP_MIN:
      case OP_MAX: {
        os << "  T a" << op.dst << ";\n  {\n";
        for (int i = op.a; i < op.b; ++i) {
          const LArg& g = L.args[i];
          os << "    const T v" << (i - op.a) << " = e" << g.expr;
          if (g.scale != 1) os << " * " << lit(g.scale);
          os << ";\n";
        }
        os << "    a" << op.dst << " = v0;\n";
        for (int i = op.a + 1; i < op.b; ++i)
          os << "    if (v" << (i - op.a) << (op.code == OP_MIN ? " < " : " > ")
             << "a" << op.dst << ") a" << op.dst << " = v" << (i - op.a) << ";\n";
        os << "  }\n";
        break;
      }
    }
  }
  // admissibility
  for (const LCons& c : L.cons) {
    const LExpr& ex = L.exprs[c.expr];
    if (!c.divisibility) {
      os << "  if (!(e" << c.expr << " " << cmp_str(c.op)
         << " (T)0)) return KCG_PT_ASSUMPTION_VIOLATED;\n";
    } else {
      os << "  {\n";
      if (ex.D != 1) {
        os << "    if (e" << c.expr << " % " << lit(ex.D)
           << " != (T)0) return KCG_PT_NONINTEGRAL;\n";
        os << "    const T v = e" << c.expr << " / " << lit(ex.D) << ";\n";
      } else {
        os << "    const T v = e" << c.expr << ";\n";
      }
      os << "    if (kcg_posmod<T>(v, " << lit(c.mod) << ") != " << lit(c.rem)
         << ") return KCG_PT_ASSUMPTION_VIOLATED;\n  }\n";
    }
  }
  // property values, schema order
  for (size_t j = 0; j < L.keys.size(); ++j) {
    const LExpr& ex = L.exprs[L.keys[j].expr];
    const int e = L.keys[j].expr;
    if (ex.D != 1) {
      os << "  if (e" << e << " % " << lit(ex.D)
         << " != (T)0) return KCG_PT_NONINTEGRAL;\n";
      os << "  cnt[" << j << "] = e" << e << " / " << lit(ex.D) << ";\n";
    } else {
      os << "  cnt[" << j << "] = e" << e << ";\n";
    }
  }
  os << "  return KCG_PT_OK;\n}\n\n";
}

// param range classification: 0 = negative (inadmissible), 1 = fast int64,
// 2 = wide int128, 3 = beyond the wide bound
void emit_classify(std::ostringstream& os, const Lowered& L, int v,
                   const std::vector<int>& pmap) {
  os << "__device__ __forceinline__ int kcg_class_" << v
     << "(const kcg_i64* p) {\n";
  os << "  if ((";
  for (int j = 0; j < L.n_params; ++j) os << (j ? " | " : "") << "p[" << pmap[j] << "]";
  if (L.n_params == 0) os << "0ll";
  os << ") < 0) return 0;\n";
  if (L.b64 >= 0) {
    os << "  if (";
    for (int j = 0; j < L.n_params; ++j)
      os << (j ? " && " : "") << "p[" << pmap[j] << "] <= " << L.b64 << "ll";
    if (L.n_params == 0) os << "true";
    os << ") return 1;\n";
  }
  if (L.b128 >= 0) {
    os << "  if (";
    for (int j = 0; j < L.n_params; ++j)
      os << (j ? " && " : "") << "p[" << pmap[j] << "] <= " << L.b128 << "ll";
    if (L.n_params == 0) os << "true";
    os << ") return 2;\n";
  }
  os << "  return 3;\n}\n\n";
}

void emit_gather(std::ostringstream& os, int v, const Lowered& L,
                 const std::vector<int>& pmap) {
  // variant parameter vector in its own declaration order
  os << "    kcg_i64 q" << v << "[" << (L.n_params ? L.n_params : 1) << "];\n";
  for (int j = 0; j < L.n_params; ++j)
    os << "    q" << v << "[" << j << "] = p[" << pmap[j] << "];\n";
}

}  // namespace

std::string codegen(const std::vector<const Lowered*>& progs,
                    const std::vector<std::vector<int>>& pmaps, int n_cols,
                    JitKind kind, const std::string& name) {
  std::ostringstream os;
  os << "// generated by kcg codegen\n" << kDeviceHelpers << "\n";
  for (size_t v = 0; v < progs.size(); ++v) {
    emit_body(os, *progs[v], static_cast<int>(v));
    emit_classify(os, *progs[v], static_cast<int>(v), pmaps[v]);
  }
  const int NP = n_cols > 0 ? n_cols : 1;

  if (kind == JitKind::eval) {
    const Lowered& L = *progs[0];
    const int F = static_cast<int>(L.keys.size());
    const int FA = F > 0 ? F : 1;
    os << "struct KcgArgs { const kcg_i64* p[" << NP << "]; double* pred; "
          "unsigned char* status; kcg_i64* clo; kcg_i64* chi; kcg_i64 n; int sim; "
          "double alpha["
       << FA << "]; };\n";
    os << "extern \"C\" __global__ void __launch_bounds__(256) " << name
       << "(const __grid_constant__ KcgArgs a) {\n"
          "  const kcg_i64 stride = (kcg_i64)gridDim.x * blockDim.x;\n"
          "  for (kcg_i64 i = (kcg_i64)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {\n"
          "    kcg_i64 p["
       << NP << "];\n";
    for (int j = 0; j < n_cols; ++j) os << "    p[" << j << "] = __ldcs(a.p[" << j << "] + i);\n";
    os << "    int st; double s = 0.0;\n"
          "    const int cls = kcg_class_0(p);\n"
          "    if (cls == 0) { st = KCG_PT_ASSUMPTION_VIOLATED; }\n"
          "    else if (cls == 1) {\n"
          "      kcg_i64 c["
       << FA << "];\n      st = kcg_body_0<kcg_i64>(p, c);\n"
          "      if (st == KCG_PT_OK) {\n";
    for (int j = 0; j < F; ++j) os << "        s = kcg_accum(s, a.alpha[" << j << "], c[" << j << "], a.sim);\n";
    os << "        if (a.clo) {\n";
    for (int j = 0; j < F; ++j) os << "          __stcs(a.clo + (kcg_i64)" << j << " * a.n + i, c[" << j << "]);\n";
    os << "          if (a.chi) {\n";
    for (int j = 0; j < F; ++j) os << "            __stcs(a.chi + (kcg_i64)" << j << " * a.n + i, kcg_hi64(c[" << j << "]));\n";
    os << "          }\n        }\n      }\n    } else if (cls == 2) {\n"
          "      kcg_i128 c["
       << FA << "];\n      st = kcg_body_0<kcg_i128>(p, c);\n"
          "      if (st == KCG_PT_OK) {\n";
    for (int j = 0; j < F; ++j) os << "        s = kcg_accum(s, a.alpha[" << j << "], c[" << j << "], a.sim);\n";
    os << "        if (a.clo) {\n";
    for (int j = 0; j < F; ++j) {
      os << "          a.clo[(kcg_i64)" << j << " * a.n + i] = (kcg_i64)c[" << j << "];\n";
      os << "          if (a.chi) a.chi[(kcg_i64)" << j << " * a.n + i] = kcg_hi64(c[" << j
         << "]); else if (!kcg_fits_i64(c[" << j << "])) st = KCG_PT_COUNT_WIDE;\n";
    }
    os << "        }\n      }\n    } else { st = KCG_PT_OVERFLOW; }\n"
          "    if (a.pred) __stcs(a.pred + i, (st == KCG_PT_OK || st == KCG_PT_COUNT_WIDE) ? s : kcg_nan());\n"
          "    if (a.status) a.status[i] = (unsigned char)st;\n"
          "  }\n}\n";
    return os.str();
  }

  if (kind == JitKind::argmin) {
    const int V = static_cast<int>(progs.size());
    os << "struct KcgArgs { const kcg_i64* p[" << NP << "]; int* best; double* best_t; "
          "double* preds; kcg_i64 n; const double* alpha[" << V << "]; };\n";
    os << "extern \"C\" __global__ void __launch_bounds__(256) " << name
       << "(const __grid_constant__ KcgArgs a) {\n"
          "  const kcg_i64 stride = (kcg_i64)gridDim.x * blockDim.x;\n"
          "  for (kcg_i64 i = (kcg_i64)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {\n"
          "    kcg_i64 p["
       << NP << "];\n";
    for (int j = 0; j < n_cols; ++j) os << "    p[" << j << "] = __ldcs(a.p[" << j << "] + i);\n";
    os << "    int best = -1; double best_t = __longlong_as_double(0x7ff0000000000000ll);\n";
    for (int v = 0; v < V; ++v) {
      const Lowered& L = *progs[v];
      const int F = static_cast<int>(L.keys.size());
      const int FA = F > 0 ? F : 1;
      os << "    {\n      double s = 0.0; int st;\n"
            "      const int cls = kcg_class_"
         << v << "(p);\n";
      emit_gather(os, v, L, pmaps[v]);
      os << "      if (cls == 0) st = KCG_PT_ASSUMPTION_VIOLATED;\n"
            "      else if (cls == 1) { kcg_i64 c["
         << FA << "]; st = kcg_body_" << v << "<kcg_i64>(q" << v
         << ", c); if (st == KCG_PT_OK) {\n";
      for (int j = 0; j < F; ++j) os << "        s = kcg_accum(s, a.alpha[" << v << "][" << j << "], c[" << j << "], 0);\n";
      os << "      } }\n      else if (cls == 2) { kcg_i128 c[" << FA << "]; st = kcg_body_" << v
         << "<kcg_i128>(q" << v << ", c); if (st == KCG_PT_OK) {\n";
      for (int j = 0; j < F; ++j) os << "        s = kcg_accum(s, a.alpha[" << v << "][" << j << "], c[" << j << "], 0);\n";
      os << "      } }\n      else st = KCG_PT_OVERFLOW;\n"
            "      if (st == KCG_PT_OK && s < best_t) { best_t = s; best = "
         << v << "; }\n"
                 "      if (a.preds) __stcs(a.preds + (kcg_i64)"
         << v << " * a.n + i, st == KCG_PT_OK ? s : kcg_nan());\n    }\n";
    }
    os << "    __stcs(a.best + i, best);\n    __stcs(a.best_t + i, best_t);\n  }\n}\n";
    return os.str();
  }

  // fused design-row reductions (gram / residual)
  const Lowered& L = *progs[0];
  const int F = static_cast<int>(L.keys.size());
  const int FA = F > 0 ? F : 1;
  const int NG = F * (F + 1) / 2;
  os << "template <class T> __device__ __forceinline__ int kcg_row(const kcg_i64* p, double t, double* x) {\n"
        "  T c["
     << FA << "];\n  const int st = kcg_body_0<T>(p, c);\n  if (st != KCG_PT_OK) return st;\n";
  for (int j = 0; j < F; ++j)
    os << "  x[" << j << "] = (c[" << j << "] != 0) ? __ddiv_rn(kcg_to_double(c[" << j
       << "]), t) : 0.0;\n";
  os << "  return KCG_PT_OK;\n}\n";
  os << "__device__ __forceinline__ int kcg_row_any(const kcg_i64* p, double t, double* x) {\n"
        "  if (!(t > 0.0)) return KCG_PT_ASSUMPTION_VIOLATED;\n"
        "  const int cls = kcg_class_0(p);\n"
        "  if (cls == 1) return kcg_row<kcg_i64>(p, t, x);\n"
        "  if (cls == 2) return kcg_row<kcg_i128>(p, t, x);\n"
        "  return cls == 0 ? KCG_PT_ASSUMPTION_VIOLATED : KCG_PT_OVERFLOW;\n}\n";
  if (kind == JitKind::gram) {
    os << "struct KcgArgs { const kcg_i64* p[" << NP
       << "]; const double* t; double* G; double* xt1; double* cmax; "
          "unsigned long long* bad; kcg_i64 n; };\n";
    os << "extern \"C\" __global__ void __launch_bounds__(256) " << name
       << "(const __grid_constant__ KcgArgs a) {\n"
          "  double g["
       << (NG ? NG : 1) << "], s1[" << FA << "], mx[" << FA << "];\n"
          "  #pragma unroll\n  for (int k = 0; k < "
       << NG << "; ++k) g[k] = 0.0;\n  #pragma unroll\n  for (int k = 0; k < " << F
       << "; ++k) { s1[k] = 0.0; mx[k] = 0.0; }\n"
          "  unsigned long long bad = 0;\n"
          "  const kcg_i64 stride = (kcg_i64)gridDim.x * blockDim.x;\n"
          "  for (kcg_i64 i = (kcg_i64)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {\n"
          "    kcg_i64 p["
       << NP << "];\n";
    for (int j = 0; j < n_cols; ++j) os << "    p[" << j << "] = __ldcs(a.p[" << j << "] + i);\n";
    os << "    double x[" << FA << "];\n"
          "    if (kcg_row_any(p, __ldcs(a.t + i), x) != KCG_PT_OK) { ++bad; continue; }\n";
    int k = 0;
    for (int r = 0; r < F; ++r) {
      os << "    s1[" << r << "] += x[" << r << "]; mx[" << r << "] = fmax(mx[" << r
         << "], fabs(x[" << r << "]));\n";
      for (int c = r; c < F; ++c, ++k)
        os << "    g[" << k << "] = fma(x[" << r << "], x[" << c << "], g[" << k << "]);\n";
    }
    os << "  }\n"
          "  // warp reduce, then one atomic per warp and value\n"
          "  #pragma unroll\n  for (int o = 16; o > 0; o >>= 1) {\n"
          "    #pragma unroll\n    for (int k = 0; k < "
       << NG << "; ++k) g[k] += __shfl_down_sync(0xffffffffu, g[k], o);\n"
          "    #pragma unroll\n    for (int k = 0; k < "
       << F << "; ++k) { s1[k] += __shfl_down_sync(0xffffffffu, s1[k], o); "
          "mx[k] = fmax(mx[k], __shfl_down_sync(0xffffffffu, mx[k], o)); }\n"
          "    bad += __shfl_down_sync(0xffffffffu, bad, o);\n  }\n"
          "  if ((threadIdx.x & 31) == 0) {\n";
    k = 0;
    for (int r = 0; r < F; ++r) {
      os << "    atomicAdd(a.xt1 + " << r << ", s1[" << r << "]);\n";
      os << "    atomicMax((unsigned long long*)(a.cmax + " << r << "), (unsigned long long)__double_as_longlong(mx[" << r << "]));\n";
      for (int c = r; c < F; ++c, ++k) {
        os << "    atomicAdd(a.G + " << (r * F + c) << ", g[" << k << "]);\n";
        if (c != r) os << "    atomicAdd(a.G + " << (c * F + r) << ", g[" << k << "]);\n";
      }
    }
    os << "    if (a.bad && bad) atomicAdd(a.bad, bad);\n  }\n}\n";
    return os.str();
  }

  // residual: obj += (1 - x . alpha)^2
  os << "struct KcgArgs { const kcg_i64* p[" << NP
     << "]; const double* t; double* obj; kcg_i64 n; double alpha[" << FA << "]; };\n";
  os << "extern \"C\" __global__ void __launch_bounds__(256) " << name
     << "(const __grid_constant__ KcgArgs a) {\n"
        "  double acc = 0.0;\n"
        "  const kcg_i64 stride = (kcg_i64)gridDim.x * blockDim.x;\n"
        "  for (kcg_i64 i = (kcg_i64)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {\n"
        "    kcg_i64 p["
     << NP << "];\n";
  for (int j = 0; j < n_cols; ++j) os << "    p[" << j << "] = __ldcs(a.p[" << j << "] + i);\n";
  os << "    double x[" << FA << "];\n"
        "    if (kcg_row_any(p, __ldcs(a.t + i), x) != KCG_PT_OK) continue;\n"
        "    double pr = 0.0;\n";
  for (int j = 0; j < F; ++j) os << "    pr = fma(x[" << j << "], a.alpha[" << j << "], pr);\n";
  os << "    const double r = 1.0 - pr;\n    acc = fma(r, r, acc);\n  }\n"
        "  #pragma unroll\n  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);\n"
        "  if ((threadIdx.x & 31) == 0) atomicAdd(a.obj, acc);\n}\n";
  return os.str();
}

}  // namespace kcg
