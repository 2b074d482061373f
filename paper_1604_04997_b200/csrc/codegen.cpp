// JIT specialisation: lowered programs -> straight-line CUDA source.
//
// Each program v becomes two exact evaluators of its admissibility
// (AssumeCtx::admits, decide.cpp:153-170) and nonzero property entries
// (evaluate_properties, props.cpp:259-271) with every coefficient,
// denominator and modulus a compile-time constant:
//   kcg_fast_<v>  int64, used when every parameter is in [0, b64]. When
//                 b64 < 2^32 parameters and congruence quotients are handled
//                 as 32-bit unsigned values (one IMAD.WIDE per first product,
//                 32-bit quotients instead of 64-bit division sequences).
//   kcg_wide_<v>  int128, out of line (__noinline__) so it does not inflate
//                 the fast path's register allocation; parameters in
//                 (b64, b128].
// The kernels around them: fused evaluate+predict (4 points per thread,
// 16-byte vector loads/stores), argmin over variants, and the fused
// design-row Gram / residual reductions.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <map>
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
    os << "kcg_const<T>((kcg_i64)" << static_cast<uint64_t>(lo) << "ull, " << hi << "ll)";
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

constexpr int64_t kU32 = 0xffffffffll;

// fast: T = kcg_i64; small: every parameter <= b64 < 2^32
// gb != nullptr: kcg_widem_<v> -- same checks, but writes the basis values
// u[b] = double(mono_b) (gram_basis) instead of the counts.
void emit_body(std::ostringstream& os, const Lowered& L, int v, bool fast,
               const char* wide_name = "kcg_wide_", const GramBasis* gb = nullptr) {
  const bool small = fast && L.b64 >= 0 && L.b64 <= kU32;
  std::vector<bool> atom_u32(L.n_atoms, false);  // value known in [0, 2^32)
  if (gb)
    os << "__device__ __noinline__ int kcg_widem_" << v
       << "(const kcg_i64* __restrict__ p, double* __restrict__ u) {\n  typedef kcg_i128 T;\n";
  else if (fast)
    os << "__device__ __forceinline__ int kcg_fast_" << v
       << "(const kcg_i64* __restrict__ p, kcg_i64* __restrict__ cnt) {\n  typedef kcg_i64 T;\n";
  else
    os << "__device__ __noinline__ int " << wide_name << v
       << "(const kcg_i64* __restrict__ p, kcg_i128* __restrict__ cnt) {\n  typedef kcg_i128 T;\n";
  for (const LOp& op : L.ops) {
    switch (op.code) {
      case OP_VAR:
        if (small) {
          os << "  const unsigned u" << op.dst << " = (unsigned)p[" << op.a << "];\n";
          atom_u32[op.dst] = true;
        }
        os << "  const T a" << op.dst << " = (T)p[" << op.a << "];\n";
        break;
      case OP_QUOT: {
        const i128 M = L.quot_mod[op.c], R = L.quot_rem[op.c];
        if (small && M <= kU32) {
          // admissible points have p = M q + R with 0 <= R <= p < 2^32
          os << "  const unsigned u" << op.dst << " = ((unsigned)p[" << op.a << "] - "
             << static_cast<uint64_t>(R) << "u) / " << static_cast<uint64_t>(M) << "u;\n";
          os << "  const T a" << op.dst << " = (T)u" << op.dst << ";\n";
          atom_u32[op.dst] = true;
        } else {
          os << "  const T a" << op.dst << " = kcg_floordiv<T>((T)p[" << op.a << "] - " << lit(R)
             << ", " << lit(M) << ");\n";
        }
        break;
      }
      case OP_MONO: {
        std::vector<int> f;
        for (int i = op.a; i < op.b; ++i)
          for (int k = 0; k < L.factors[i].second; ++k) f.push_back(L.factors[i].first);
        os << "  const T m" << op.dst << " = ";
        size_t start = 0;
        if (f.size() >= 2 && atom_u32[f[0]] && atom_u32[f[1]]) {
          os << "(T)((kcg_u64)u" << f[0] << " * u" << f[1] << ")";
          start = 2;
        } else {
          os << "a" << f[0];
          start = 1;
        }
        for (size_t k = start; k < f.size(); ++k) os << " * a" << f[k];
        os << ";\n";
        break;
      }
      case OP_EXPR: {
        os << "  const T e" << op.dst << " = ";
        if (op.a == op.b) os << "(T)0";
        for (int i = op.a; i < op.b; ++i) {
          const LTerm& t = L.terms[i];
          if (i != op.a) os << " + ";
          if (t.mono < 0)
            os << lit(t.coef);
          else if (t.coef == 1)
            os << "m" << t.mono;
          else if (t.coef == -1)
            os << "(-m" << t.mono << ")";
          else
            os << lit(t.coef) << " * m" << t.mono;
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
          os << "    if (v" << (i - op.a) << (op.code == OP_MIN ? " < " : " > ") << "a" << op.dst
             << ") a" << op.dst << " = v" << (i - op.a) << ";\n";
        os << "  }\n";
        break;
      }
    }
  }
  // admissibility
  for (const LCons& c : L.cons) {
    if (c.divisibility == 2) {
      // congruence facts folded into p = M q + R
      if (small && atom_u32[c.expr] && c.rem == 0 && c.mod <= kU32)
        os << "  if ((unsigned)p[" << c.op << "] != " << static_cast<uint64_t>(c.mod) << "u * u"
           << c.expr << ") return KCG_PT_ASSUMPTION_VIOLATED;\n";
      else
        os << "  if ((T)p[" << c.op << "] - " << lit(c.rem) << " != " << lit(c.mod) << " * a"
           << c.expr << ") return KCG_PT_ASSUMPTION_VIOLATED;\n";
      continue;
    }
    const LExpr& ex = L.exprs[c.expr];
    if (!c.divisibility) {
      os << "  if (!(e" << c.expr << " " << cmp_str(c.op)
         << " (T)0)) return KCG_PT_ASSUMPTION_VIOLATED;\n";
    } else {
      os << "  {\n";
      if (ex.D != 1) {
        os << "    if (e" << c.expr << " % " << lit(ex.D) << " != (T)0) return KCG_PT_NONINTEGRAL;\n";
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
    if (gb) {
      if (ex.D != 1)
        os << "  if (e" << e << " % " << lit(ex.D) << " != (T)0) return KCG_PT_NONINTEGRAL;\n";
      continue;
    }
    if (ex.D != 1) {
      os << "  if (e" << e << " % " << lit(ex.D) << " != (T)0) return KCG_PT_NONINTEGRAL;\n";
      os << "  cnt[" << j << "] = e" << e << " / " << lit(ex.D) << ";\n";
    } else {
      os << "  cnt[" << j << "] = e" << e << ";\n";
    }
  }
  if (gb)
    for (size_t b = 0; b < gb->monos.size(); ++b)
      os << "  u[" << b << "] = " << (gb->monos[b] < 0 ? std::string("1.0") : "kcg_to_double(m" + std::to_string(gb->monos[b]) + ")")
         << ";\n";
  os << "  return KCG_PT_OK;\n}\n\n";
}

}  // namespace

// Predict folding: a key whose count is C * mono with C = 2^k > 1 (and the
// count-to-double trick applies: |C|, |mono| < 2^53) contributes
// RN(alpha * RN(C * mono)) = RN((alpha * C) * mono), since C * mono and
// alpha * C are exact. The GEN = 0 predict kernels therefore take
// alpha_f = alpha * C and skip the DMUL that forms the count.
double predict_fold(const Lowered& L, int j) {
  const LExpr& ex = L.exprs[L.keys[j].expr];
  if (ex.D != 1 || ex.term_end - ex.term_begin != 1) return 1.0;
  const LTerm& t = L.terms[ex.term_begin];
  const long double two53 = std::ldexp(1.0L, 53);
  if (t.mono < 0 || t.coef <= 1 || static_cast<long double>(t.coef) >= two53 ||
      t.mono >= static_cast<int>(L.mono_bound64.size()) || !(L.mono_bound64[t.mono] < two53))
    return 1.0;
  if ((t.coef & (t.coef - 1)) != 0) return 1.0;
  return static_cast<double>(t.coef);
}

namespace {

// Fast path (every parameter in [0, b64]), branch-free: admissibility and
// integrality are folded into flags, the status is selected at the end.
//   dbl = false: kcg_fasti_<v> writes the exact int64 counts;
//   dbl = true : kcg_fastd_<v> writes RN(double(count)) only (predict). A key
//                that is one monomial times a constant C with |C| and the
//                monomial's bound below 2^53 gets C (x) double(mono): both
//                factors are exact doubles, so the single rounding of their
//                product equals RN(C * mono) -- no 64-bit constant multiply.
//   gb != null: kcg_fastm_<v> writes the basis values double(mono_b) (the
//                fused Gram / residual rows) and checks key integrality only.
//   fold      : kcg_fastp_<v>, kcg_fastd_ with power-of-two constants left
//                out (predict_fold: the kernel's weights carry them).
void emit_fast(std::ostringstream& os, const Lowered& L, int v, bool dbl,
               const GramBasis* gb = nullptr, bool fold = false) {
  const bool small = L.b64 >= 0 && L.b64 <= kU32;
  const long double two53 = std::ldexp(1.0L, 53);
  std::vector<bool> atom_u32(L.n_atoms, false);
  if (gb || fold) dbl = true;
  os << "__device__ __forceinline__ int kcg_fast" << (gb ? "m_" : fold ? "p_" : dbl ? "d_" : "i_") << v
     << "(const kcg_i64* __restrict__ p, " << (dbl ? "double" : "kcg_i64")
     << "* __restrict__ cnt) {\n  typedef kcg_i64 T;\n  bool ok = true, integral = true;\n";
  // which exprs are needed as integers
  std::vector<bool> need_expr(L.n_exprs, false), need_mono_d(L.n_monos, false);
  std::vector<int> key_fast(L.keys.size(), -1);  // mono id for the DMUL trick
  if (gb)
    for (int m : gb->monos)
      if (m >= 0) need_mono_d[m] = true;
  for (size_t j = 0; j < L.keys.size(); ++j) {
    const LExpr& ex = L.exprs[L.keys[j].expr];
    if (gb) {
      if (ex.D != 1) need_expr[L.keys[j].expr] = true;
      continue;
    }
    bool trick = dbl && ex.D == 1 && ex.term_end - ex.term_begin == 1;
    if (trick) {
      const LTerm& t = L.terms[ex.term_begin];
      const i128 ac = t.coef < 0 ? -t.coef : t.coef;
      trick = t.mono >= 0 && static_cast<long double>(ac) < two53 &&
              t.mono < static_cast<int>(L.mono_bound64.size()) && L.mono_bound64[t.mono] < two53;
      if (trick) {
        key_fast[j] = t.mono;
        need_mono_d[t.mono] = true;
      }
    }
    if (!trick) need_expr[L.keys[j].expr] = true;
  }
  for (const LCons& c : L.cons)
    if (c.divisibility != 2) need_expr[c.expr] = true;
  for (const LOp& op : L.ops)
    if (op.code == OP_FLOORDIV) need_expr[op.a] = true;
    else if (op.code == OP_MIN || op.code == OP_MAX)
      for (int i = op.a; i < op.b; ++i) need_expr[L.args[i].expr] = true;
  for (const LOp& op : L.ops) {
    switch (op.code) {
      case OP_VAR:
        if (small) {
          os << "  const unsigned u" << op.dst << " = (unsigned)p[" << op.a << "];\n";
          atom_u32[op.dst] = true;
        }
        os << "  const T a" << op.dst << " = (T)p[" << op.a << "];\n";
        break;
      case OP_QUOT: {
        const i128 M = L.quot_mod[op.c], R = L.quot_rem[op.c];
        if (small && M <= kU32) {
          os << "  const unsigned u" << op.dst << " = ((unsigned)p[" << op.a << "] - "
             << static_cast<uint64_t>(R) << "u) / " << static_cast<uint64_t>(M) << "u;\n";
          os << "  const T a" << op.dst << " = (T)u" << op.dst << ";\n";
          atom_u32[op.dst] = true;
        } else {
          os << "  const T a" << op.dst << " = kcg_floordiv<T>((T)p[" << op.a << "] - " << lit(R)
             << ", " << lit(M) << ");\n";
        }
        break;
      }
      case OP_MONO: {
        std::vector<int> f;
        for (int i = op.a; i < op.b; ++i)
          for (int k = 0; k < L.factors[i].second; ++k) f.push_back(L.factors[i].first);
        os << "  const T m" << op.dst << " = ";
        size_t start;
        if (f.size() >= 2 && atom_u32[f[0]] && atom_u32[f[1]]) {
          os << "(T)((kcg_u64)u" << f[0] << " * u" << f[1] << ")";
          start = 2;
        } else {
          os << "a" << f[0];
          start = 1;
        }
        for (size_t k = start; k < f.size(); ++k) os << " * a" << f[k];
        os << ";\n";
        if (need_mono_d[op.dst]) os << "  const double dm" << op.dst << " = __ll2double_rn(m" << op.dst << ");\n";
        break;
      }
      case OP_EXPR: {
        if (!need_expr[op.dst]) break;
        os << "  const T e" << op.dst << " = ";
        if (op.a == op.b) os << "(T)0";
        for (int i = op.a; i < op.b; ++i) {
          const LTerm& t = L.terms[i];
          if (i != op.a) os << " + ";
          if (t.mono < 0)
            os << lit(t.coef);
          else if (t.coef == 1)
            os << "m" << t.mono;
          else if (t.coef == -1)
            os << "(-m" << t.mono << ")";
          else
            os << lit(t.coef) << " * m" << t.mono;
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
          os << "    a" << op.dst << " = (v" << (i - op.a) << (op.code == OP_MIN ? " < " : " > ") << "a"
             << op.dst << ") ? v" << (i - op.a) << " : a" << op.dst << ";\n";
        os << "  }\n";
        break;
      }
    }
  }
  for (const LCons& c : L.cons) {
    if (c.divisibility == 2) {
      if (small && atom_u32[c.expr] && c.rem == 0 && c.mod <= kU32)
        os << "  ok &= (unsigned)p[" << c.op << "] == " << static_cast<uint64_t>(c.mod) << "u * u" << c.expr << ";\n";
      else
        os << "  ok &= (T)p[" << c.op << "] - " << lit(c.rem) << " == " << lit(c.mod) << " * a" << c.expr << ";\n";
      continue;
    }
    const LExpr& ex = L.exprs[c.expr];
    if (!c.divisibility) {
      os << "  ok &= e" << c.expr << " " << cmp_str(c.op) << " (T)0;\n";
    } else if (ex.D != 1) {
      os << "  { const bool di = (e" << c.expr << " % " << lit(ex.D) << ") == (T)0; integral &= di;"
         << " ok &= !di || kcg_posmod<T>(e" << c.expr << " / " << lit(ex.D) << ", " << lit(c.mod)
         << ") == " << lit(c.rem) << "; }\n";
    } else {
      os << "  ok &= kcg_posmod<T>(e" << c.expr << ", " << lit(c.mod) << ") == " << lit(c.rem) << ";\n";
    }
  }
  if (gb) {
    for (size_t j = 0; j < L.keys.size(); ++j) {
      const int e = L.keys[j].expr;
      if (L.exprs[e].D != 1) os << "  integral &= (e" << e << " % " << lit(L.exprs[e].D) << ") == (T)0;\n";
    }
    for (size_t b = 0; b < gb->monos.size(); ++b)
      os << "  cnt[" << b << "] = " << (gb->monos[b] < 0 ? std::string("1.0") : "dm" + std::to_string(gb->monos[b]))
         << ";\n";
  }
  for (size_t j = 0; j < (gb ? 0 : L.keys.size()); ++j) {
    const int e = L.keys[j].expr;
    const LExpr& ex = L.exprs[e];
    if (key_fast[j] >= 0) {
      const i128 C = L.terms[ex.term_begin].coef;
      if (C == 1 || (fold && predict_fold(L, static_cast<int>(j)) != 1.0))
        os << "  cnt[" << j << "] = dm" << key_fast[j] << ";\n";
      else
        os << "  cnt[" << j << "] = __dmul_rn(" << static_cast<long long>(C) << ".0, dm" << key_fast[j] << ");\n";
      continue;
    }
    std::string val = "e" + std::to_string(e);
    if (ex.D != 1) {
      os << "  integral &= (e" << e << " % " << lit(ex.D) << ") == (T)0;\n";
      val = "(e" + std::to_string(e) + " / " + lit(ex.D) + ")";
    }
    if (dbl)
      os << "  cnt[" << j << "] = __ll2double_rn(" << val << ");\n";
    else
      os << "  cnt[" << j << "] = " << val << ";\n";
  }
  os << "  return ok ? (integral ? KCG_PT_OK : KCG_PT_NONINTEGRAL) : KCG_PT_ASSUMPTION_VIOLATED;\n}\n\n";
}

// parameter range class: 0 negative (inadmissible), 1 fast, 2 wide, 3 overflow
void emit_classify(std::ostringstream& os, const Lowered& L, int v, const std::vector<int>& pmap) {
  os << "__device__ __forceinline__ int kcg_class_" << v << "(const kcg_i64* p) {\n";
  if (L.b64 >= 0 && L.b64 <= kU32 && L.n_params > 0) {
    // class 1 <=> all high words zero and every low word <= b64
    os << "  if (((";
    for (int j = 0; j < L.n_params; ++j) os << (j ? " | " : "") << "p[" << pmap[j] << "]";
    os << ") >> 32) == 0 && ";
    for (int j = 0; j < L.n_params; ++j)
      os << (j ? " && " : "") << "(unsigned)p[" << pmap[j] << "] <= " << L.b64 << "u";
    os << ") return 1;\n";
  }
  os << "  if ((";
  for (int j = 0; j < L.n_params; ++j) os << (j ? " | " : "") << "p[" << pmap[j] << "]";
  if (L.n_params == 0) os << "0ll";
  os << ") < 0) return 0;\n";
  for (int pass = 0; pass < 2; ++pass) {
    const int64_t b = pass == 0 ? L.b64 : L.b128;
    if (b < 0) continue;
    os << "  if (";
    for (int j = 0; j < L.n_params; ++j) os << (j ? " && " : "") << "p[" << pmap[j] << "] <= " << b << "ll";
    if (L.n_params == 0) os << "true";
    os << ") return " << (pass + 1) << ";\n";
  }
  os << "  return 3;\n}\n\n";
}

// gather program v's parameters (its declaration order) from the launch's columns
void emit_gather(std::ostringstream& os, const char* dst, const char* src, const Lowered& L,
                 const std::vector<int>& pmap, const char* indent) {
  os << indent << "kcg_i64 " << dst << "[" << (L.n_params ? L.n_params : 1) << "];\n";
  for (int j = 0; j < L.n_params; ++j)
    os << indent << dst << "[" << j << "] = " << src << "[" << pmap[j] << "];\n";
}

// point evaluator for the eval kernel: status + prediction (+ counts).
// GEN = 0: every compact weight is finite, so skipping zero counts
//          (model.cpp:106-111) or zero weights (simdevice.cpp:84-88) cannot
//          change the sum (adding +-0.0 to a sum that starts at +0.0 is an
//          identity) and the accumulation is unconditional.
// GEN = 1: general case, the skip rule is applied per key.
void emit_eval_point(std::ostringstream& os, const Lowered& L) {
  const int F = static_cast<int>(L.keys.size());
  const int FA = F > 0 ? F : 1;
  os << "struct KcgRes { double s; int st; };\n";
  // wide path body (inlined into the out-of-line entry points below): the
  // parameters come from the binding columns (kcg_point_slow) or from a
  // grid descriptor (kcg_point_slow_g); writes counts when requested.
  // The entry points take only the argument struct and the index: passing
  // the parameter values across the noinline call as extra 64-bit arguments
  // was miscompiled at the 64-register cap (caller spill slot overwritten,
  // found by the 1000-program fuzz).
  os << "__device__ __forceinline__ KcgRes kcg_point_slow_body(const KcgArgs& a, kcg_i64 i, const kcg_i64* pin) {\n"
        "  kcg_i64 p["
     << (L.n_params ? L.n_params : 1) << "];\n";
  for (int j = 0; j < L.n_params; ++j) os << "  p[" << j << "] = pin[" << j << "];\n";
  os << "  KcgRes r; r.s = kcg_nan();\n"
        "  const int cls = kcg_class_0(p);\n"
        "  if (cls == 0) { r.st = KCG_PT_ASSUMPTION_VIOLATED; return r; }\n";
  if (L.admit && L.admit->b128 >= 0) {
    // beyond the count bound: still decide admissibility first (props.cpp:263-266)
    os << "  if (cls == 3) {\n    r.st = KCG_PT_OVERFLOW;\n    if (";
    for (int j = 0; j < L.n_params; ++j) os << (j ? " && " : "") << "p[" << j << "] <= " << L.admit->b128 << "ll";
    if (L.n_params == 0) os << "true";
    os << ") {\n      kcg_i128 none[1];\n      const int a0 = kcg_admit_0(p, none);\n"
          "      if (a0 != KCG_PT_OK) r.st = a0;\n    }\n    return r;\n  }\n";
  } else {
    os << "  if (cls == 3) { r.st = KCG_PT_OVERFLOW; return r; }\n";
  }
  os << "  kcg_i128 c["
     << FA << "];\n  r.st = kcg_wide_0(p, c);\n  if (r.st != KCG_PT_OK) return r;\n  double s = 0.0;\n";
  for (int j = 0; j < F; ++j) os << "  s = kcg_accum(s, a.alpha[" << j << "], c[" << j << "], a.sim);\n";
  os << "  r.s = s;\n  if (a.clo) {\n";
  for (int j = 0; j < F; ++j)
    os << "    a.clo[(kcg_i64)" << j << " * a.n + i] = (kcg_i64)c[" << j << "];\n"
       << "    if (a.chi) a.chi[(kcg_i64)" << j << " * a.n + i] = kcg_hi64(c[" << j
       << "]); else if (!kcg_fits_i64(c[" << j << "])) r.st = KCG_PT_COUNT_WIDE;\n";
  os << "  }\n  return r;\n}\n";
  os << "__device__ __noinline__ KcgRes kcg_point_slow(const KcgArgs& a, kcg_i64 i) {\n"
        "  kcg_i64 p["
     << (L.n_params ? L.n_params : 1) << "];\n";
  for (int j = 0; j < L.n_params; ++j) os << "  p[" << j << "] = a.p[" << j << "][i];\n";
  os << "  return kcg_point_slow_body(a, i, p);\n}\n";
  // fast path only; returns -1 when the point needs kcg_point_slow
  os << "template <int GEN>\n__device__ __forceinline__ int kcg_point_fast(const kcg_i64* p, const KcgArgs& a, kcg_i64 i, double& out) {\n"
        "  if (kcg_class_0(p) != 1) return -1;\n"
        "  if (a.clo) {\n    kcg_i64 c["
     << FA << "];\n    const int st = kcg_fasti_0(p, c);\n    if (st != KCG_PT_OK) return st;\n"
              "    double s = 0.0;\n";
  for (int j = 0; j < F; ++j)
    os << "    s = GEN ? kcg_accum(s, a.alpha[" << j << "], c[" << j << "], a.sim) : "
       << "__dadd_rn(s, __dmul_rn(a.alpha[" << j << "], kcg_to_double(c[" << j << "])));\n";
  os << "    out = s;\n";
  for (int j = 0; j < F; ++j) {
    os << "    __stcs(a.clo + (kcg_i64)" << j << " * a.n + i, c[" << j << "]);\n";
    os << "    if (a.chi) __stcs(a.chi + (kcg_i64)" << j << " * a.n + i, kcg_hi64(c[" << j << "]));\n";
  }
  os << "    return KCG_PT_OK;\n  }\n  double c[" << FA << "];\n"
        "  if (GEN == 0) {  // folded power-of-two count constants (predict_fold)\n"
        "    const int st = kcg_fastp_0(p, c);\n    double s = 0.0;\n";
  for (int j = 0; j < F; ++j) os << "    s = __dadd_rn(s, __dmul_rn(a.alpha_f[" << j << "], c[" << j << "]));\n";
  os << "    out = s;\n    return st;\n  }\n  const int st = kcg_fastd_0(p, c);\n"
        "  double s = 0.0;\n";
  for (int j = 0; j < F; ++j) os << "  s = kcg_accum(s, a.alpha[" << j << "], c[" << j << "], a.sim);\n";
  os << "  out = s;\n  return st;\n}\n";
}

// Grid-descriptor kernel: bindings are never read from HBM. Point i of the
// lattice has parameter j = start_j + step_j * d_j with (d_0..d_{P-1}) the
// mixed-radix digits of first + i (last parameter fastest). Each thread
// handles 4 consecutive points per step: the digits are decoded once and
// then advanced by odometer increments (+1 inside the quad, + the digits of
// 4 * gridDim * blockDim between steps), so no division runs per point.
int min_blocks();

void emit_grid_kernel(std::ostringstream& os, int n_cols, const std::string& name, int gen) {
  const int NP = n_cols > 0 ? n_cols : 1;
  if (!gen) {  // shared by the two variants: emitted once
    os << "struct KcgGridArgs { KcgArgs a; kcg_i64 start[" << NP << "]; kcg_i64 step[" << NP
       << "]; kcg_u64 count[" << NP << "]; kcg_u64 sdig[" << NP << "]; kcg_u64 first; };\n";
    os << "__device__ __forceinline__ void kcg_odo_add(kcg_u64* d, const kcg_u64* add, const kcg_u64* cnt) {\n"
          "  kcg_u64 c = 0;\n  #pragma unroll\n  for (int j = "
       << n_cols - 1 << "; j >= 0; --j) {\n"
          "    kcg_u64 t = d[j] + add[j] + c;\n    c = t >= cnt[j];\n    d[j] = c ? t - cnt[j] : t;\n  }\n}\n";
    os << "__device__ __forceinline__ void kcg_odo_inc(kcg_u64* d, const kcg_u64* cnt) {\n"
          "  #pragma unroll\n  for (int j = "
       << n_cols - 1 << "; j >= 0; --j) {\n    if (++d[j] < cnt[j]) return;\n    d[j] = 0;\n  }\n}\n";
    // out-of-line wide path of the grid kernels: re-derives the binding of
    // lattice point first + i (rare; the divisions do not matter)
    os << "__device__ __noinline__ KcgRes kcg_point_slow_g(const KcgGridArgs& g, kcg_i64 i) {\n"
          "  kcg_i64 p["
       << NP << "];\n  kcg_u64 r = g.first + (kcg_u64)i;\n  #pragma unroll\n  for (int j = " << n_cols - 1
       << "; j >= 0; --j) { p[j] = g.start[j] + g.step[j] * (kcg_i64)(r % g.count[j]); r /= g.count[j]; }\n"
          "  return kcg_point_slow_body(g.a, i, p);\n}\n";
  }
  // 2 CTAs/SM: the 4-point odometer state plus the exact evaluation need
  // ~100 registers; the 64-register cap of the streaming kernels spills
  os << "extern \"C\" __global__ void __launch_bounds__(256, 2) " << name
     << "(const __grid_constant__ KcgGridArgs g) {\n"
        "  const KcgArgs& a = g.a;\n"
        "  const kcg_i64 tid = (kcg_i64)blockIdx.x * blockDim.x + threadIdx.x;\n"
        "  const kcg_i64 stride = (kcg_i64)gridDim.x * blockDim.x;\n"
        "  const kcg_i64 nq = (a.n + 3) >> 2;\n"
        "  if (tid >= nq) return;\n"
        "  kcg_u64 d["
     << NP << "];\n  { kcg_u64 r = g.first + 4 * (kcg_u64)tid;\n    #pragma unroll\n    for (int j = " << n_cols - 1
     << "; j >= 0; --j) { d[j] = r % g.count[j]; r /= g.count[j]; } }\n"
        "  for (kcg_i64 v = tid; v < nq; v += stride) {\n"
        "    kcg_u64 e["
     << NP << "];\n    #pragma unroll\n    for (int j = 0; j < " << n_cols << "; ++j) e[j] = d[j];\n"
        "    double s[4]; int st[4];\n"
        "    #pragma unroll\n"
        "    for (int u = 0; u < 4; ++u) {\n"
        "      kcg_i64 p["
     << NP << "];\n      #pragma unroll\n      for (int j = 0; j < " << n_cols
     << "; ++j) p[j] = g.start[j] + g.step[j] * (kcg_i64)e[j];\n"
        "      s[u] = kcg_nan();\n"
        "      st[u] = kcg_point_fast<"
     << gen << ">(p, a, 4 * v + u, s[u]);\n"
        "      if (st[u] < 0 && 4 * v + u < a.n) { const KcgRes r = kcg_point_slow_g(g, 4 * v + u); s[u] = r.s; st[u] = r.st; }\n"
        "      if (st[u] != KCG_PT_OK && st[u] != KCG_PT_COUNT_WIDE) s[u] = kcg_nan();\n"
        "      if (u < 3) kcg_odo_inc(e, g.count);\n"
        "    }\n"
        "    if (a.vout && 4 * v + 3 < a.n) {\n"
        "      if (a.pred) {\n"
        "        __stcs(reinterpret_cast<double2*>(a.pred) + 2 * v, make_double2(s[0], s[1]));\n"
        "        __stcs(reinterpret_cast<double2*>(a.pred) + 2 * v + 1, make_double2(s[2], s[3]));\n"
        "      }\n"
        "      if (a.status) reinterpret_cast<unsigned*>(a.status)[v] =\n"
        "          (unsigned)st[0] | ((unsigned)st[1] << 8) | ((unsigned)st[2] << 16) | ((unsigned)st[3] << 24);\n"
        "    } else {\n"
        "      #pragma unroll\n"
        "      for (int u = 0; u < 4; ++u)\n"
        "        if (4 * v + u < a.n) {\n"
        "          if (a.pred) a.pred[4 * v + u] = s[u];\n"
        "          if (a.status) a.status[4 * v + u] = (unsigned char)st[u];\n"
        "        }\n"
        "    }\n"
        "    kcg_odo_add(d, g.sdig, g.count);\n"
        "  }\n}\n";
}

int min_blocks() {
  // occupancy target of the eval kernels (blocks of 256 per SM); the
  // register cap it implies is the main tuning knob (KCG_MIN_BLOCKS)
  const char* e = std::getenv("KCG_MIN_BLOCKS");
  const int v = e ? std::atoi(e) : 4;
  return v >= 1 && v <= 8 ? v : 4;
}

// TMA-staged eval kernel (persistent, 2 CTAs/SM): one elected thread streams
// tiles of 1024 points per parameter column into a ring of shared-memory
// stages with cp.async.bulk (SASS UBLKCP) completing on an mbarrier; the
// 256 threads evaluate 4 points each from shared memory while the next
// stages are in flight, so the bytes in flight no longer depend on the
// register budget of the exact integer evaluation.
constexpr int kTmaTile = 1024;

int env_int(const char* name, int dflt, int lo, int hi);

// ring depth of the fused (bindings + T) kernels: 64 KB when two CTAs also
// hold 35 KB of DMMA row buffers each, 96 KB otherwise (3 stages for P = 3)
// Register-path fused kernels (residual, basis Gram) evaluate one row at a
// time straight from the stage (~80 registers) and run 3 CTAs per SM with a
// 64 KB ring each (measured: Gram 5.35 -> 6.12 TB/s, residual 6.25 -> 7.0
// TB/s); the DMMA Gram keeps 2 CTAs (its row buffers need the shared memory).
int fused_ctas(bool dmma) { return env_int("KCG_FUSED_CTAS", dmma ? 2 : 3, 1, 4); }
// the refinement gradient (FP64-bound, not HBM-bound) has its own defaults:
// profiles/ab_rgrad_knobs.sh
// (64-register cap and rows tid + 256 u: 7.71 -> 6.86 ms per 1e9 rows with
// the grid at the resident CTA count)
int rgrad_ctas() { return env_int("KCG_RGRAD_CTAS", 4, 1, 4); }
bool rgrad_strided() { return env_int("KCG_RGRAD_STRIDED", 1, 0, 1) == 1; }
bool fused_rowwise(bool dmma) { return env_int("KCG_FUSED_ROWWISE", dmma ? 0 : 1, 0, 1) == 1; }
// row order and unroll of the row-wise consumer: the Gram is fastest with
// rows tid + 256 u fully unrolled (6.17 -> 6.45 TB/s), the residual with
// rows 4 tid + u rolled (7.01 vs 6.82 TB/s) -- profiles/ab_fused.sh
int fused_unroll(bool gram) { return env_int("KCG_FUSED_UNROLL", gram ? 4 : 1, 1, 4); }
bool fused_strided(bool gram) { return env_int("KCG_FUSED_STRIDED", gram ? 1 : 0, 0, 1) == 1; }

int fused_stages(int n_cols, bool dmma) {
  const int per = (n_cols + 1) * 1024 * 8;
  const int s = (env_int("KCG_FUSED_RING_KB", 64, 16, 200) * 1024) / per;
  return s < 2 ? 2 : (s > 8 ? 8 : s);
}

int env_int(const char* name, int dflt, int lo, int hi) {
  const char* e = std::getenv(name);
  const int v = e ? std::atoi(e) : dflt;
  return v >= lo && v <= hi ? v : dflt;
}

// per-CTA ring size (KB) and CTAs per SM of the TMA kernel (tuning knobs)
// one point at a time from the stage: ~80 registers, 3 CTAs/SM with a 64 KB
// ring each (measured on the headline step: 1.92e11 -> 2.13e11 points/s);
// KCG_TMA_ROWWISE=0 restores the 4-points-in-registers consumer (2 CTAs/SM)
bool tma_rowwise() { return env_int("KCG_TMA_ROWWISE", 1, 0, 1) == 1; }
int tma_ring_kb() { return env_int("KCG_TMA_RING_KB", tma_rowwise() ? 64 : 96, 16, 200); }
int tma_ctas() { return env_int("KCG_TMA_CTAS", tma_rowwise() ? 3 : 2, 1, 4); }
int tma_unroll() { return env_int("KCG_TMA_UNROLL", 4, 1, 4); }  // 1 -> 4: 2.10e11 -> 2.18e11 points/s
int argmin_ctas() { return env_int("KCG_ARGMIN_CTAS", 0, 0, 8); }  // 0: no register cap
bool argmin_prefetch() { return env_int("KCG_ARGMIN_PREFETCH", 1, 0, 1) == 1; }

// points per TMA stage of the eval kernel (row-wise consumers: a multiple
// of the 256-thread CTA)
int tma_tile() { return tma_rowwise() ? 256 * env_int("KCG_TMA_TILE_Q", 4, 1, 8) : kTmaTile; }

int tma_stages(int n_cols) {
  const int per = (n_cols > 0 ? n_cols : 1) * tma_tile() * 8;
  int s = (tma_ring_kb() * 1024) / per;
  return s < 2 ? 2 : (s > 8 ? 8 : s);
}

void emit_tma_kernel(std::ostringstream& os, int n_cols, const std::string& name) {
  const int NP = n_cols > 0 ? n_cols : 1;
  const int S = tma_stages(n_cols);
  os << "extern \"C\" __global__ void __launch_bounds__(256, " << tma_ctas() << ") " << name
     << "(const __grid_constant__ KcgArgs a) {\n"
        "  constexpr int TP = "
     << tma_tile() << ", S = " << S << ", NP = " << NP
     << ";\n"
        "  extern __shared__ __align__(128) unsigned char kcg_smem[];\n"
        "  kcg_i64* buf = reinterpret_cast<kcg_i64*>(kcg_smem);\n"
        "  __shared__ __align__(8) unsigned long long full[S];\n"
        "  __shared__ unsigned reads[S];  // row-wise variant: warps done with stage s\n"
        "  if (threadIdx.x < S) reads[threadIdx.x] = 0;\n"
        "  const kcg_i64 ntiles = a.n / TP;\n"
        "  const unsigned fb = (unsigned)__cvta_generic_to_shared(full);\n"
        "  const unsigned bb = (unsigned)__cvta_generic_to_shared(buf);\n"
        "  if (threadIdx.x == 0) {\n"
        "    for (int s = 0; s < S; ++s)\n"
        "      asm volatile(\"mbarrier.init.shared::cta.b64 [%0], 1;\" :: \"r\"(fb + 8 * s));\n"
        "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n"
        "  }\n"
        "  __syncthreads();\n"
        "  auto issue = [&](int s, kcg_i64 tile) {\n"
        "    asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n"
        "    asm volatile(\"mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\" :: \"r\"(fb + 8 * s), \"r\"(NP * TP * 8) : \"memory\");\n"
        "    for (int j = 0; j < NP; ++j)\n"
        "      asm volatile(\"cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\"\n"
        "                   :: \"r\"(bb + (unsigned)((s * NP + j) * TP * 8)), \"l\"(a.p[j] + tile * TP), \"r\"(TP * 8), \"r\"(fb + 8 * s) : \"memory\");\n"
        "  };\n"
        "  if (threadIdx.x == 0)\n"
        "    for (int s = 0; s < S; ++s) {\n"
        "      const kcg_i64 t = blockIdx.x + (kcg_i64)s * gridDim.x;\n"
        "      if (t < ntiles) issue(s, t);\n"
        "    }\n"
        "  for (kcg_i64 k = 0;; ++k) {\n"
        "    const kcg_i64 tile = blockIdx.x + k * gridDim.x;\n"
        "    if (tile >= ntiles) break;\n"
        "    const int s = (int)(k % S);\n"
        "    const unsigned parity = (unsigned)((k / S) & 1);\n"
        "    {\n"
        "      unsigned done = 0;\n"
        "      while (!done)\n"
        "        asm volatile(\"{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }\"\n"
        "                     : \"=r\"(done) : \"r\"(fb + 8 * s), \"r\"(parity) : \"memory\");\n"
        "    }\n"
        << (tma_rowwise()
                ? std::string(
                      "    // one point at a time straight from the stage (points tid + 256 u:\n"
                      "    // conflict-free loads, coalesced stores), ~80 registers -> 3 CTAs/SM\n"
                      "    const kcg_i64 rb = tile * TP;\n"
                      "    #pragma unroll " + std::to_string(tma_unroll()) + "\n"
                      "    for (int u = 0; u < TP / 256; ++u) {\n"
                      "      const int o = u * 256 + threadIdx.x;\n"
                      "      kcg_i64 q[NP];\n"
                      "      #pragma unroll\n"
                      "      for (int j = 0; j < NP; ++j) q[j] = buf[(s * NP + j) * TP + o];\n"
                      "      double r = kcg_nan();\n"
                      "      int st = kcg_point_fast<0>(q, a, rb + o, r);\n"
                      "      if (st < 0) { const KcgRes x = kcg_point_slow(a, rb + o); r = x.s; st = x.st; }\n"
                      "      if (st != KCG_PT_OK && st != KCG_PT_COUNT_WIDE) r = kcg_nan();\n"
                      "      if (a.pred) __stcs(a.pred + rb + o, r);\n"
                      "      if (a.status) a.status[rb + o] = (unsigned char)st;\n"
                      "    }\n"
                      "    __syncwarp();\n"
                      "    if ((threadIdx.x & 31) == 0) {\n"
                      "      if (kcg_ring_release(&reads[s], blockDim.x / 32)) {\n"
                      "        const kcg_i64 nt = blockIdx.x + (k + S) * gridDim.x;\n"
                      "        if (nt < ntiles) issue(s, nt);\n"
                      "      }\n"
                      "    }\n"
                      "    continue;\n")
                : std::string()) <<
        "    kcg_i64 q[4][NP];\n"
        "    #pragma unroll\n"
        "    for (int j = 0; j < NP; ++j) {\n"
        "      const longlong2* src = reinterpret_cast<const longlong2*>(buf + (s * NP + j) * TP) + 2 * threadIdx.x;\n"
        "      const longlong2 x = src[0], y = src[1];\n"
        "      q[0][j] = x.x; q[1][j] = x.y; q[2][j] = y.x; q[3][j] = y.y;\n"
        "    }\n"
        "    __syncthreads();  // stage s fully read: refill it\n"
        "    if (threadIdx.x == 0) {\n"
        "      const kcg_i64 nt = blockIdx.x + (k + S) * gridDim.x;\n"
        "      if (nt < ntiles) issue(s, nt);\n"
        "    }\n"
        "    const kcg_i64 base = tile * TP + 4 * threadIdx.x;\n"
        "    double r[4]; int st[4];\n"
        "    #pragma unroll\n"
        "    for (int u = 0; u < 4; ++u) { r[u] = kcg_nan(); st[u] = kcg_point_fast<0>(q[u], a, base + u, r[u]); }\n"
        "    if ((st[0] | st[1] | st[2] | st[3]) < 0) {\n"
        "      #pragma unroll\n"
        "      for (int u = 0; u < 4; ++u)\n"
        "        if (st[u] < 0) { const KcgRes x = kcg_point_slow(a, base + u); r[u] = x.s; st[u] = x.st; }\n"
        "    }\n"
        "    #pragma unroll\n"
        "    for (int u = 0; u < 4; ++u)\n"
        "      if (st[u] != KCG_PT_OK && st[u] != KCG_PT_COUNT_WIDE) r[u] = kcg_nan();\n"
        "    if (a.vout) {\n"
        "      if (a.pred) {\n"
        "        __stcs(reinterpret_cast<double2*>(a.pred + base), make_double2(r[0], r[1]));\n"
        "        __stcs(reinterpret_cast<double2*>(a.pred + base) + 1, make_double2(r[2], r[3]));\n"
        "      }\n"
        "      if (a.status) reinterpret_cast<unsigned*>(a.status)[base >> 2] =\n"
        "          (unsigned)st[0] | ((unsigned)st[1] << 8) | ((unsigned)st[2] << 16) | ((unsigned)st[3] << 24);\n"
        "    } else {\n"
        "      #pragma unroll\n"
        "      for (int u = 0; u < 4; ++u) {\n"
        "        if (a.pred) __stcs(a.pred + base + u, r[u]);\n"
        "        if (a.status) a.status[base + u] = (unsigned char)st[u];\n"
        "      }\n"
        "    }\n"
        "  }\n"
        "  // tail (n % TP points): scalar\n"
        "  for (kcg_i64 i = ntiles * TP + (kcg_i64)blockIdx.x * blockDim.x + threadIdx.x; i < a.n;\n"
        "       i += (kcg_i64)gridDim.x * blockDim.x) {\n"
        "    kcg_i64 p[NP];\n";
  for (int j = 0; j < n_cols; ++j) os << "    p[" << j << "] = a.p[" << j << "][i];\n";
  os << "    double r = kcg_nan();\n    int st = kcg_point_fast<0>(p, a, i, r);\n"
        "    if (st < 0) { const KcgRes x = kcg_point_slow(a, i); r = x.s; st = x.st; }\n"
        "    if (st != KCG_PT_OK && st != KCG_PT_COUNT_WIDE) r = kcg_nan();\n"
        "    if (a.pred) a.pred[i] = r;\n"
        "    if (a.status) a.status[i] = (unsigned char)st;\n"
        "  }\n}\n";
}

void emit_eval_kernel(std::ostringstream& os, int n_cols, const std::string& name, int gen) {
  const int NP = n_cols > 0 ? n_cols : 1;
  os << "extern \"C\" __global__ void __launch_bounds__(256, " << min_blocks() << ") " << name
     << "(const __grid_constant__ KcgArgs a) {\n"
        "  const kcg_i64 tid = (kcg_i64)blockIdx.x * blockDim.x + threadIdx.x;\n"
        "  const kcg_i64 stride = (kcg_i64)gridDim.x * blockDim.x;\n"
        "  kcg_i64 done = 0;\n"
        "  if (a.vec && a.vout) {\n"
        "    // 4 consecutive points per thread: two 16-byte loads per column,\n"
        "    // two 16-byte streaming stores of predictions, one 4-byte status store\n"
        "    const kcg_i64 nv = a.n >> 2;\n"
        "    for (kcg_i64 v = tid; v < nv; v += stride) {\n"
        "      kcg_i64 q[4]["
     << NP << "];\n";
  for (int j = 0; j < n_cols; ++j)
    os << "      { const longlong2 x = __ldcs(reinterpret_cast<const longlong2*>(a.p[" << j
       << "]) + 2 * v); const longlong2 y = __ldcs(reinterpret_cast<const longlong2*>(a.p[" << j
       << "]) + 2 * v + 1);\n"
          "        q[0]["
       << j << "] = x.x; q[1][" << j << "] = x.y; q[2][" << j << "] = y.x; q[3][" << j << "] = y.y; }\n";
  os << "      double s[4]; int st[4];\n"
        "      #pragma unroll\n"
        "      for (int u = 0; u < 4; ++u) { s[u] = kcg_nan(); st[u] = kcg_point_fast<"
     << gen << ">(q[u], a, 4 * v + u, s[u]); }\n"
               "      if ((st[0] | st[1] | st[2] | st[3]) < 0) {\n"
               "        #pragma unroll\n"
               "        for (int u = 0; u < 4; ++u)\n"
               "          if (st[u] < 0) { const KcgRes r = kcg_point_slow(a, 4 * v + u); s[u] = r.s; st[u] = r.st; }\n"
               "      }\n"
               "      #pragma unroll\n"
               "      for (int u = 0; u < 4; ++u)\n"
               "        if (st[u] != KCG_PT_OK && st[u] != KCG_PT_COUNT_WIDE) s[u] = kcg_nan();\n"
               "      if (a.pred) {\n"
               "        __stcs(reinterpret_cast<double2*>(a.pred) + 2 * v, make_double2(s[0], s[1]));\n"
               "        __stcs(reinterpret_cast<double2*>(a.pred) + 2 * v + 1, make_double2(s[2], s[3]));\n"
               "      }\n"
               "      if (a.status) reinterpret_cast<unsigned*>(a.status)[v] =\n"
               "          (unsigned)st[0] | ((unsigned)st[1] << 8) | ((unsigned)st[2] << 16) | ((unsigned)st[3] << 24);\n"
               "    }\n"
               "    done = nv << 2;\n"
               "  }\n"
               "  for (kcg_i64 i = done + tid; i < a.n; i += stride) {\n"
               "    kcg_i64 p["
     << NP << "];\n";
  for (int j = 0; j < n_cols; ++j) os << "    p[" << j << "] = __ldcs(a.p[" << j << "] + i);\n";
  os << "    double s = kcg_nan();\n    int st = kcg_point_fast<" << gen
     << ">(p, a, i, s);\n"
        "    if (st < 0) { const KcgRes r = kcg_point_slow(a, i); s = r.s; st = r.st; }\n"
        "    if (st != KCG_PT_OK && st != KCG_PT_COUNT_WIDE) s = kcg_nan();\n"
        "    if (a.pred) __stcs(a.pred + i, s);\n"
        "    if (a.status) a.status[i] = (unsigned char)st;\n"
        "  }\n}\n";
}

}  // namespace

int tma_ctas_per_sm() { return tma_ctas(); }


GramBasis gram_basis(const Lowered& L) {
  GramBasis g;
  std::map<int, int> idx;
  const int F = static_cast<int>(L.keys.size());
  g.terms.resize(F);
  for (int j = 0; j < F; ++j) {
    const LExpr& ex = L.exprs[L.keys[j].expr];
    for (int t = ex.term_begin; t < ex.term_end; ++t) {
      const LTerm& lt = L.terms[t];
      auto it = idx.find(lt.mono);
      if (it == idx.end()) {
        it = idx.emplace(lt.mono, static_cast<int>(g.monos.size())).first;
        g.monos.push_back(lt.mono);
      }
      const long double c = static_cast<long double>(lt.coef) / static_cast<long double>(ex.D);
      g.terms[j].emplace_back(it->second, static_cast<double>(c));
    }
    if (g.terms[j].size() != 1) g.compound.push_back(j);
  }
  // A key with several terms is expanded without cancellation only when
  // every term is a positive coefficient times a monomial of parameters /
  // congruence quotients (both >= 0 at admissible points): then every
  // product in A Gu A^T is non-negative and the expansion is as accurate as
  // the direct sum. Otherwise (e.g. n^3/6 - n^2/2 + n/3) keep one column per key.
  std::vector<bool> nonneg_atom(L.n_atoms, false), nonneg_mono(L.n_monos, false);
  for (const LOp& op : L.ops) {
    if (op.code == OP_VAR || op.code == OP_QUOT) nonneg_atom[op.dst] = true;
    if (op.code == OP_MONO) {
      bool nn = true;
      for (int i = op.a; i < op.b; ++i) nn = nn && nonneg_atom[L.factors[i].first];
      nonneg_mono[op.dst] = nn;
    }
  }
  bool safe = true;
  for (int j : g.compound) {
    const LExpr& ex = L.exprs[L.keys[j].expr];
    for (int t = ex.term_begin; t < ex.term_end; ++t)
      safe = safe && L.terms[t].coef > 0 && (L.terms[t].mono < 0 || nonneg_mono[L.terms[t].mono]);
  }
  // the basis pays when it is narrower than the key set; the expansion
  // tables stay small (F <= 64) and the compound-key maxima few
  g.reduced = L.gram_basis && safe && g.monos.size() < static_cast<size_t>(F) && F <= 64 &&
              g.compound.size() <= 8;
  return g;
}

namespace {
// Refinement-gradient groups: keys whose ORIGINAL counts differ by a power
// of two (same parameter monomial, or both constants) have design columns
// x_j = RN(2^k c_base) / T = 2^k RN(c_base) / T exactly, so one division per
// group forms them all, the residual needs one double-double term per group
// (weight A_g = sum_j 2^k_j alpha_j) and g_j = 2^k_j sum_i x_base r_i.
// Tiled matmul g16: 9 keys -> 4 groups ({store, minls, local, addsub, mul,
// barrier} over n m l, load 9/8 n m l, groups n l / 256, const).
}  // namespace

RGradGroups rgrad_groups(const Lowered& L) {
  RGradGroups R;
  const int F = static_cast<int>(L.keys.size());
  R.of_key.assign(F, {-1, 0});
  auto shape_eq = [&](const LKey& a, const LKey& b) {
    if (a.form == 0 || b.form == 0) return false;
    if ((a.form == 1) != (b.form == 1)) return false;
    return a.form == 1 || a.pexp == b.pexp;
  };
  // log2(ca / cb) if it is an integer power of two, else INT_MIN
  auto pow2_ratio = [](const LKey& a, const LKey& b) -> int {
    try {
      const i128 num = checked_mul(a.coef, b.coef_den), den = checked_mul(a.coef_den, b.coef);
      if (num <= 0 || den <= 0) return INT_MIN;
      int e = 0;
      i128 n = num, d = den;
      while (n % 2 == 0 && n > d) { n /= 2; ++e; }
      while (d % 2 == 0 && d > n) { d /= 2; --e; }
      return n == d ? e : INT_MIN;
    } catch (const KcgError&) {
      return INT_MIN;
    }
  };
  for (int j = 0; j < F; ++j) {
    if (R.of_key[j].first >= 0) continue;
    std::vector<int> mem{j};
    for (int k = j + 1; k < F; ++k)
      if (R.of_key[k].first < 0 && shape_eq(L.keys[j], L.keys[k]) && pow2_ratio(L.keys[k], L.keys[j]) != INT_MIN)
        mem.push_back(k);
    int base = j;  // the smallest count of the group: every other member is 2^k (k >= 0) times it
    for (int k : mem)
      if (pow2_ratio(L.keys[k], L.keys[base]) < 0) base = k;
    const int g = static_cast<int>(R.base.size());
    R.base.push_back(base);
    for (int k : mem) R.of_key[k] = {g, k == base ? 0 : pow2_ratio(L.keys[k], L.keys[base])};
  }
  return R;
}

namespace {

// register-accumulator fused Gram for narrow rows, DMMA otherwise
constexpr int kRegGramMax = 6;
bool gram_dmma(int W) { return W > kRegGramMax && W <= 48; }
}  // namespace

size_t fused_smem_bytes(int n_cols, const Lowered& L, bool gram, bool per_key) {
  const int W = per_key ? static_cast<int>(L.keys.size()) : gram_basis(L).width(static_cast<int>(L.keys.size()));
  const int WA = W > 0 ? W : 1;
  const int NB = (W + 7) / 8, LDX = NB * 8 + 1;
  size_t b = static_cast<size_t>(fused_stages(n_cols, gram && gram_dmma(W))) * (n_cols + 1) * kTmaTile * 8;
  if (gram && gram_dmma(W))
    b += static_cast<size_t>(8) * 32 * LDX * 8;  // DMMA row buffers (also the slow-path rows)
  else
    b += static_cast<size_t>(256) * WA * 8;      // slow-path rows
  return b;
}

int fused_ctas_per_sm(const Lowered& L, bool gram) {
  return fused_ctas(gram && gram_dmma(gram_basis(L).width(static_cast<int>(L.keys.size()))));
}

int rgrad_ctas_per_sm() { return rgrad_ctas(); }

size_t tma_smem_bytes(int n_cols) {
  return static_cast<size_t>(tma_stages(n_cols)) * (n_cols > 0 ? n_cols : 1) * tma_tile() * 8;
}

// ---------------------------------------------------------------------------
// One-pass multi-program evaluate + predict (kcg_eval_predict_multi).
//
// The autotuning sweep evaluates V variants over the same sizes. One
// program per launch re-reads every size's bindings V times (config 4: 24 B
// x 6 per size, 2.65x the unique bytes). This kernel streams each size's
// bindings once through the TMA ring and writes all V predictions (and
// status bytes): HBM traffic per size is 8 P + 8 V (+ V) bytes.
//   * fast path: one range check against the smallest int64-safe bound of
//     all variants, then each variant's branch-free kcg_fastp_<v> + its
//     folded-weight inner product, straight-line; quotients and monomials
//     that several variants share are CSE'd by the compiler;
//   * anything else (negative / beyond an int64 bound / int128 counts):
//     kcg_mslow, out of line, which reloads the size's bindings from the
//     columns and writes every variant's outputs itself (no parameter values
//     or local addresses cross the call, see kcg_point_slow);
//   * weights: one flat table of compact weights per variant in the
//     argument struct (constant bank): as given (wide path), folded (fast).
// measured on the config-4 lattice (profiles/gpu_r02_multi*.sh): one CTA
// per SM with a 72 KB ring (3 stages) 2.40-2.50 ms; 2 CTAs x 96 KB 2.74,
// 3 CTAs x 64 KB 2.57-2.83, 1 CTA x 192 KB 2.89; loading the thread's
// whole share of a stage up front (KCG_MULTI_PREFETCH=1) 2.60
// The argmin epilogue writes 12 B per size instead of 48: there the kernel
// is latency-bound and more CTAs pay (1 CTA x 72 KB 2.25 ms, 2 CTAs 1.90,
// 3 CTAs x 64 KB 1.65; KCG_MULTIAM_CTAS / KCG_MULTIAM_RING_KB)
int multi_ctas(bool argmin = false) {
  return argmin ? env_int("KCG_MULTIAM_CTAS", 3, 1, 4) : env_int("KCG_MULTI_CTAS", 1, 1, 4);
}
int multi_ring_kb(bool argmin = false) {
  return argmin ? env_int("KCG_MULTIAM_RING_KB", 64, 16, 200) : env_int("KCG_MULTI_RING_KB", 72, 16, 200);
}
int multi_tile() { return 256 * env_int("KCG_MULTI_TILE_Q", 4, 1, 8); }
int multi_ctas_per_sm(bool argmin) { return multi_ctas(argmin); }
bool multi_share() { return env_int("KCG_MULTI_SHARE", 1, 0, 1) == 1; }
bool multi_prefetch() { return env_int("KCG_MULTI_PREFETCH", 0, 0, 1) == 1; }
// bulk-store variant (pred mode): predictions staged per warp in shared
// memory and written by cp.async.bulk (profiles/stream_store_ab.cu: the
// 3-read:6-write mix reaches 6.1-6.2 TB/s with bulk stores against
// 5.2-5.8 with 16-byte streaming stores)
// measured (profiles/gpu_r02_bulk*.sh, config-4 lattice): per-warp 1 KB bulk
// stores with one staging buffer, 2 CTAs x 48 KB ring per SM: 2.055-2.08 ms
// against 2.17 for the 16-byte-store kernel; double-buffered staging at one
// CTA per SM 2.46, 3 CTAs with a 16 KB ring 2.38
int multi_obuf() { return env_int("KCG_MULTI_OBUF", 1, 1, 2); }
int multi_bulk_ctas() { return env_int("KCG_MULTI_BULK_CTAS", 2, 1, 3); }
int multi_bulk_ring_kb() { return env_int("KCG_MULTI_BULK_RING_KB", 48, 16, 200); }
bool multi_bulk_cta() { return env_int("KCG_MULTI_BULK_CTA", 0, 0, 1) == 1; }  // one 8 KB store per row per stage
int multi_bulk_vmax() { return 10; }
int multi_stages(int n_cols, bool argmin) {
  const int per = (n_cols > 0 ? n_cols : 1) * multi_tile() * 8;
  const int s = (multi_ring_kb(argmin) * 1024) / per;
  return s < 2 ? 2 : (s > 8 ? 8 : s);
}
size_t multi_smem_bytes(int n_cols, bool argmin) {
  return static_cast<size_t>(multi_stages(n_cols, argmin)) * (n_cols > 0 ? n_cols : 1) * multi_tile() * 8;
}
int multi_bulk_stages(int n_cols) {
  const int per = (n_cols > 0 ? n_cols : 1) * multi_tile() * 8;
  const int s = (multi_bulk_ring_kb() * 1024) / per;
  return s < 2 ? 2 : (s > 8 ? 8 : s);
}
size_t multi_bulk_smem_bytes(int n_cols, int V) {
  return static_cast<size_t>(multi_bulk_stages(n_cols)) * (n_cols > 0 ? n_cols : 1) * multi_tile() * 8 +
         static_cast<size_t>(multi_obuf()) * V * multi_tile() * 8;  // 8 warps x OB x [V][TP / 8]
}

// Which products the one-pass kernel forms once per point and shares:
//   * form-1 keys (constant count C): alpha_key (x) RN(C) is a constant of
//     the launch, computed on the host (shk[]): the kernel only adds it;
//   * form-2 keys (count = 2^k * a parameter monomial): RN(count) =
//     2^k * RN(mono) and alpha (x) RN(count) = (alpha * 2^k) (x) RN(mono)
//     (alpha * 2^k is exact when finite), so every program whose key has
//     the same (schema key, 2^k, monomial) uses one product sh[t] =
//     shw[t] (x) RN(mono), the monomial an exact u64 product of the
//     parameters (valid on the fast path: every parameter <= min_v b64_v,
//     and bmin^deg < 2^64 is checked here).
// Both are bitwise what the per-program kernel adds for that key.
MultiPlan multi_plan(const std::vector<const Lowered*>& progs, const std::vector<std::vector<int>>& pmaps,
                     int n_cols) {
  MultiPlan P;
  const int V = static_cast<int>(progs.size());
  P.bmin = INT64_MAX;
  P.all_small = true;
  for (int v = 0; v < V; ++v) {
    P.bmin = std::min<int64_t>(P.bmin, progs[v]->b64);
    P.all_small = P.all_small && progs[v]->b64 >= 0 && progs[v]->b64 <= kU32;
  }
  P.use.resize(V);
  const long double two62 = std::ldexp(1.0L, 62), two64 = std::ldexp(1.0L, 64);
  for (int v = 0; v < V; ++v) {
    const Lowered& L = *progs[v];
    P.use[v].assign(L.keys.size(), {0, -1});
    if (!multi_share()) continue;
    for (size_t k = 0; k < L.keys.size(); ++k) {
      const LKey& key = L.keys[k];
      if (key.form == 1 && static_cast<long double>(key.coef < 0 ? -key.coef : key.coef) < two62) {
        int t = -1;
        for (size_t i = 0; i < P.kprods.size(); ++i)
          if (P.kprods[i].first == key.schema && P.kprods[i].second == key.coef) t = static_cast<int>(i);
        if (t < 0) {
          t = static_cast<int>(P.kprods.size());
          P.kprods.push_back({key.schema, key.coef});
        }
        P.use[v][k] = {1, t};
      } else if (key.form == 2 && P.bmin >= 0 && n_cols > 0 &&
                 static_cast<long double>(key.coef) < std::ldexp(1.0L, 1000)) {
        std::vector<int> ex(n_cols, 0);
        int deg = 0;
        for (int j = 0; j < L.n_params; ++j) {
          ex[pmaps[v][j]] += key.pexp[j];
          deg += key.pexp[j];
        }
        if (std::pow(static_cast<long double>(std::max<int64_t>(P.bmin, 1)), deg) >= two64) continue;
        int m = -1;
        for (size_t i = 0; i < P.monos.size(); ++i)
          if (P.monos[i] == ex) m = static_cast<int>(i);
        if (m < 0) {
          m = static_cast<int>(P.monos.size());
          P.monos.push_back(ex);
        }
        int t = -1;
        for (size_t i = 0; i < P.wprods.size(); ++i)
          if (std::get<0>(P.wprods[i]) == key.schema && std::get<1>(P.wprods[i]) == key.coef &&
              std::get<2>(P.wprods[i]) == m)
            t = static_cast<int>(i);
        if (t < 0) {
          t = static_cast<int>(P.wprods.size());
          P.wprods.emplace_back(key.schema, key.coef, m);
        }
        P.use[v][k] = {2, t};
      }
    }
  }
  return P;
}

// argmin = true: the config-4 autotuning epilogue instead of the prediction
// stores -- per size the lowest-index variant with status OK and the
// smallest prediction (best = -1, best_t = +inf if none), optionally all
// predictions too (kernels <name>[_tma] and <name>[_tma]_p)
void emit_multi(std::ostringstream& os, const std::vector<const Lowered*>& progs,
                const std::vector<std::vector<int>>& pmaps, int n_cols, const std::string& name, bool argmin) {
  const int V = static_cast<int>(progs.size());
  const int NP = n_cols > 0 ? n_cols : 1;
  const MultiPlan P = multi_plan(progs, pmaps, n_cols);
  std::vector<int> off(V);
  int tot = 0;
  for (int v = 0; v < V; ++v) {
    off[v] = tot;
    tot += std::max<int>(1, static_cast<int>(progs[v]->keys.size()));
  }
  const int NK = std::max<int>(1, static_cast<int>(P.kprods.size()));
  const int NW = std::max<int>(1, static_cast<int>(P.wprods.size()));
  os << "struct KcgMArgs { const kcg_i64* p[" << NP << "]; double* pred; unsigned char* status; int* best; "
        "double* best_t; kcg_i64 n; kcg_i64 ldp; kcg_i64 lds; double al[" << tot << "]; double alf[" << tot
     << "]; double shk[" << NK << "]; double shw[" << NW << "]; };\n";
  // combined fast-path range: every parameter in [0, min_v b64_v]
  os << "__device__ __forceinline__ bool kcg_mfast(const kcg_i64* p) {\n";
  if (P.bmin < 0 || n_cols == 0) {
    os << "  return " << (P.bmin >= 0 ? "true" : "false") << ";\n}\n";
  } else if (P.all_small) {
    os << "  return ((";
    for (int j = 0; j < n_cols; ++j) os << (j ? " | " : "") << "p[" << j << "]";
    os << ") >> 32) == 0";
    for (int j = 0; j < n_cols; ++j) os << " && (unsigned)p[" << j << "] <= " << P.bmin << "u";
    os << ";\n}\n";
  } else {
    os << "  return ";
    for (int j = 0; j < n_cols; ++j)
      os << (j ? " && " : "") << "p[" << j << "] >= 0 && p[" << j << "] <= " << P.bmin << "ll";
    os << ";\n}\n";
  }
  // variant v on the fast path: SH = 1 uses the shared products sh[] (only
  // valid when kcg_mfast holds), SH = 0 the program's own products
  for (int v = 0; v < V; ++v) {
    const Lowered& L = *progs[v];
    const int F = static_cast<int>(L.keys.size());
    // NS = 0 (argmin without predictions): the raw sum, no NaN select --
    // the epilogue tests the status itself
    os << "template <int SH, int NS = 1>\n__device__ __forceinline__ int kcg_mfastv_" << v
       << "(const kcg_i64* p, const KcgMArgs& a, const double* sh, double& out) {\n";
    emit_gather(os, "q", "p", L, pmaps[v], "  ");
    os << "  double c[" << std::max(F, 1) << "];\n  const int st = kcg_fastp_" << v << "(q, c);\n  double s = 0.0;\n";
    for (int j = 0; j < F; ++j) {
      const auto [form, t] = P.use[v][j];
      const std::string own = "__dmul_rn(a.alf[" + std::to_string(off[v] + j) + "], c[" + std::to_string(j) + "])";
      if (form == 1)
        os << "  s = __dadd_rn(s, a.shk[" << t << "]);\n";
      else if (form == 2)
        os << "  s = __dadd_rn(s, SH ? sh[" << t << "] : " << own << ");\n";
      else
        os << "  s = __dadd_rn(s, " << own << ");\n";
    }
    // one opaque select (a plain ?: is pushed into every admissibility
    // check as a pair of FSELs on the result: 18 per variant)
    os << "  if (NS)\n    asm(\"{ .reg .pred p; setp.eq.s32 p, %1, 0; selp.f64 %0, %2, 0d7FF8000000000000, p; }\"\n"
          "        : \"=d\"(out) : \"r\"(st), \"d\"(s));\n  else\n    out = s;\n  return st;\n}\n";
  }
  // out-of-line: every variant of size i, any parameter range
  // ob != nullptr (bulk-store kernels): predictions go to the warp's
  // shared-memory staging block ob[v * 128 + li] instead of global memory
  os << "__device__ __noinline__ void kcg_mslow(const KcgMArgs& a, kcg_i64 i, double* ob, int li, int rs) {\n  kcg_i64 p[" << NP << "];\n"
        "  int bi = -1;\n  double bt = __longlong_as_double(0x7ff0000000000000ll);\n";
  for (int j = 0; j < n_cols; ++j) os << "  p[" << j << "] = a.p[" << j << "][i];\n";
  for (int v = 0; v < V; ++v) {
    const Lowered& L = *progs[v];
    const int F = static_cast<int>(L.keys.size());
    os << "  {\n    double s = kcg_nan();\n    int st;\n    const int cls = kcg_class_" << v << "(p);\n";
    emit_gather(os, "q", "p", L, pmaps[v], "    ");
    os << "    if (cls == 1) {\n      st = kcg_mfastv_" << v << "<0>(p, a, nullptr, s);\n    } else if (cls == 2) {\n"
       << "      kcg_i128 c[" << std::max(F, 1) << "];\n      st = kcg_wide_" << v << "(q, c);\n"
       << "      if (st == KCG_PT_OK) {\n        double t = 0.0;\n";
    for (int j = 0; j < F; ++j) os << "        t = kcg_accum(t, a.al[" << off[v] + j << "], c[" << j << "], 0);\n";
    os << "        s = t;\n      }\n    } else if (cls == 0) {\n      st = KCG_PT_ASSUMPTION_VIOLATED;\n"
          "    } else {\n      st = KCG_PT_OVERFLOW;\n";
    if (L.admit && L.admit->b128 >= 0) {
      // beyond the count bound: admissibility still decides first (props.cpp:263-266)
      os << "      if (";
      for (int j = 0; j < L.n_params; ++j) os << (j ? " && " : "") << "q[" << j << "] <= " << L.admit->b128 << "ll";
      if (L.n_params == 0) os << "true";
      os << ") {\n        kcg_i128 none[1];\n        const int a0 = kcg_admit_" << v
         << "(q, none);\n        if (a0 != KCG_PT_OK) st = a0;\n      }\n";
    }
    os << "    }\n    if (st != KCG_PT_OK) s = kcg_nan();\n"
       << "    if (ob) ob[" << v << " * rs + li] = s;\n    else if (a.pred) a.pred[(kcg_i64)" << v << " * a.ldp + i] = s;\n"
       << "    if (a.status) a.status[(kcg_i64)" << v << " * a.lds + i] = (unsigned char)st;\n"
       << "    if (st == KCG_PT_OK && s < bt) { bt = s; bi = " << v << "; }\n  }\n";
  }
  os << "  if (a.best) { a.best[i] = bi; a.best_t[i] = bt; }\n}\n";
  // one size from registers: shared products, then every variant -- one
  // basic block (no per-variant branches), so the V independent
  // accumulation chains interleave
  // BULK > 0: predictions to the shared staging block ob[v * BULK + li]
  os << "template <int ST, int BULK = 0>\n__device__ __forceinline__ void kcg_msize(const kcg_i64* p, const KcgMArgs& a, "
        "kcg_i64 i, double* ob = nullptr, int li = 0) {\n"
        "  if (!kcg_mfast(p)) { kcg_mslow(a, i, BULK ? ob : nullptr, li, BULK); return; }\n";
  for (size_t m = 0; m < P.monos.size(); ++m) {
    os << "  const double dm" << m << " = __ull2double_rn(";
    bool first = true;
    for (int j = 0; j < n_cols; ++j)
      for (int e = 0; e < P.monos[m][j]; ++e) {
        os << (first ? "" : " * ") << "(kcg_u64)p[" << j << "]";
        first = false;
      }
    if (first) os << "1ull";
    os << ");\n";
  }
  os << "  double sh[" << NW << "];\n";
  for (size_t t = 0; t < P.wprods.size(); ++t)
    os << "  sh[" << t << "] = __dmul_rn(a.shw[" << t << "], dm" << std::get<2>(P.wprods[t]) << ");\n";
  for (int v = 0; v < V; ++v)
    os << "  double s" << v << ";\n  const int st" << v << " = kcg_mfastv_" << v << "<1, " << (argmin ? "ST" : "1")
       << ">(p, a, sh, s" << v << ");\n";
  // ST: pred mode -- status bytes too; argmin mode -- all predictions too
  if (!argmin) {
    os << "  if (BULK) {\n";
    for (int v = 0; v < V; ++v) os << "    ob[" << v << " * BULK + li] = s" << v << ";\n";
    os << "  } else {\n";
    for (int v = 0; v < V; ++v) os << "    __stcs(a.pred + (kcg_i64)" << v << " * a.ldp + i, s" << v << ");\n";
    os << "  }\n  if (ST) {\n";
    for (int v = 0; v < V; ++v) os << "    a.status[(kcg_i64)" << v << " * a.lds + i] = (unsigned char)st" << v << ";\n";
    os << "  }\n}\n";
  } else {
    // lowest index wins ties (strict <); a non-OK variant holds NaN, which
    // never compares below
    os << "  int bi = -1;\n  double bt = __longlong_as_double(0x7ff0000000000000ll);\n";
    for (int v = 0; v < V; ++v)
      os << "  if (st" << v << " == KCG_PT_OK && s" << v << " < bt) { bt = s" << v << "; bi = " << v << "; }\n";
    os << "  __stcs(a.best + i, bi);\n  __stcs(a.best_t + i, bt);\n  if (ST) {\n";
    for (int v = 0; v < V; ++v) os << "    __stcs(a.pred + (kcg_i64)" << v << " * a.ldp + i, s" << v << ");\n";
    os << "  }\n}\n";
  }
  for (int stv = 0; stv < 2; ++stv) {
    const std::string sfx = stv ? (argmin ? "_p" : "_st") : "";
    // plain grid-stride kernel (unaligned columns, small n)
    os << "extern \"C\" __global__ void __launch_bounds__(256) " << name << sfx << "(const __grid_constant__ KcgMArgs a) {\n"
          "  for (kcg_i64 i = (kcg_i64)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += (kcg_i64)gridDim.x * blockDim.x) {\n"
          "    kcg_i64 p[" << NP << "];\n";
    for (int j = 0; j < n_cols; ++j) os << "    p[" << j << "] = __ldcs(a.p[" << j << "] + i);\n";
    os << "    kcg_msize<" << stv << ">(p, a, i);\n  }\n}\n";
    // TMA ring kernel (persistent): one elected thread streams TP-point
    // tiles of every column into the ring; each warp releases a stage when
    // done and the last one refills it (as kcg_eval_<k>_tma)
    const int S = multi_stages(n_cols, argmin);
    os << "extern \"C\" __global__ void __launch_bounds__(256, " << multi_ctas(argmin) << ") " << name << "_tma" << sfx
       << "(const __grid_constant__ KcgMArgs a) {\n"
          "  constexpr int TP = " << multi_tile() << ", S = " << S << ", NP = " << NP << ";\n"
          "  extern __shared__ __align__(128) unsigned char kcg_smem[];\n"
          "  kcg_i64* buf = reinterpret_cast<kcg_i64*>(kcg_smem);\n"
          "  __shared__ __align__(8) unsigned long long full[S];\n"
          "  __shared__ unsigned reads[S];\n"
          "  if (threadIdx.x < S) reads[threadIdx.x] = 0;\n"
          "  const kcg_i64 ntiles = a.n / TP;\n"
          "  const unsigned fb = (unsigned)__cvta_generic_to_shared(full);\n"
          "  const unsigned bb = (unsigned)__cvta_generic_to_shared(buf);\n"
          "  if (threadIdx.x == 0) {\n"
          "    for (int s = 0; s < S; ++s)\n"
          "      asm volatile(\"mbarrier.init.shared::cta.b64 [%0], 1;\" :: \"r\"(fb + 8 * s));\n"
          "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n"
          "  }\n"
          "  __syncthreads();\n"
          "  auto issue = [&](int s, kcg_i64 tile) {\n"
          "    asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n"
          "    asm volatile(\"mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\" :: \"r\"(fb + 8 * s), \"r\"(NP * TP * 8) : \"memory\");\n"
          "    for (int j = 0; j < NP; ++j)\n"
          "      asm volatile(\"cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\"\n"
          "                   :: \"r\"(bb + (unsigned)((s * NP + j) * TP * 8)), \"l\"(a.p[j] + tile * TP), \"r\"(TP * 8), \"r\"(fb + 8 * s) : \"memory\");\n"
          "  };\n"
          "  if (threadIdx.x == 0)\n"
          "    for (int s = 0; s < S; ++s) {\n"
          "      const kcg_i64 t = blockIdx.x + (kcg_i64)s * gridDim.x;\n"
          "      if (t < ntiles) issue(s, t);\n"
          "    }\n"
          "  for (kcg_i64 k = 0;; ++k) {\n"
          "    const kcg_i64 tile = blockIdx.x + k * gridDim.x;\n"
          "    if (tile >= ntiles) break;\n"
          "    const int s = (int)(k % S);\n"
          "    const unsigned parity = (unsigned)((k / S) & 1);\n"
          "    {\n"
          "      unsigned done = 0;\n"
          "      while (!done)\n"
          "        asm volatile(\"{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }\"\n"
          "                     : \"=r\"(done) : \"r\"(fb + 8 * s), \"r\"(parity) : \"memory\");\n"
          "    }\n"
          "    const kcg_i64 rb = tile * TP;\n";
    // the warp is done with stage s: the last warp to arrive refills it
    const char* release =
        "    __syncwarp();\n"
        "    if ((threadIdx.x & 31) == 0) {\n"
        "      if (kcg_ring_release(&reads[s], blockDim.x / 32)) {\n"
        "        const kcg_i64 nt = blockIdx.x + (k + S) * gridDim.x;\n"
        "        if (nt < ntiles) issue(s, nt);\n"
        "      }\n"
        "    }\n";
    if (multi_prefetch()) {
      // the thread's share of the stage (TP / 256 points) is loaded up
      // front and the stage released before any evaluation: the refill
      // overlaps this stage's work, and the shared-memory latency is paid
      // once (ncu: the first use of the LDS result was the top stall of
      // the one-point-at-a-time loop)
      os << "    kcg_i64 q[TP / 256][NP];\n"
            "    #pragma unroll\n"
            "    for (int u = 0; u < TP / 256; ++u)\n"
            "      #pragma unroll\n"
            "      for (int j = 0; j < NP; ++j) q[u][j] = buf[(s * NP + j) * TP + u * 256 + threadIdx.x];\n"
         << release
         << "    #pragma unroll\n"
            "    for (int u = 0; u < TP / 256; ++u) kcg_msize<" << stv << ">(q[u], a, rb + u * 256 + threadIdx.x);\n"
            "  }\n";
    } else {
      os << "    #pragma unroll 1\n"
            "    for (int u = 0; u < TP / 256; ++u) {\n"
            "      const int o = u * 256 + threadIdx.x;\n"
            "      kcg_i64 q[NP];\n"
            "      #pragma unroll\n"
            "      for (int j = 0; j < NP; ++j) q[j] = buf[(s * NP + j) * TP + o];\n"
            "      kcg_msize<" << stv << ">(q, a, rb + o);\n"
            "    }\n"
         << release << "  }\n";
    }
    os <<           "  for (kcg_i64 i = ntiles * TP + (kcg_i64)blockIdx.x * blockDim.x + threadIdx.x; i < a.n;\n"
          "       i += (kcg_i64)gridDim.x * blockDim.x) {\n"
          "    kcg_i64 p[NP];\n";
    for (int j = 0; j < n_cols; ++j) os << "    p[" << j << "] = a.p[" << j << "][i];\n";
    os << "    kcg_msize<" << stv << ">(p, a, i);\n  }\n}\n";
    if (argmin || V > multi_bulk_vmax() || n_cols == 0) continue;
    // bulk-store TMA kernel (<name>_tmab[_st]): warp w owns points
    // [PW w, PW w + PW) of each TP-point stage (PW = TP / 8); its lanes
    // evaluate points PW w + lane + 32 u into the warp's staging block
    // [V][PW] in shared memory, then lane 0 writes the block's V rows to
    // global memory with cp.async.bulk (PW * 8 bytes each), after the
    // block's previous stores have read it -- no CTA barrier, warps drift
    // freely. KCG_MULTI_BULK_CTA=1: one CTA-wide [V][TP] block, one TP * 8
    // byte store per row per stage, two barriers per stage.
    const int SB = multi_bulk_stages(n_cols), OB = multi_obuf(), TPB = multi_tile(), PW = TPB / 8;
    os << "extern \"C\" __global__ void __launch_bounds__(256, " << multi_bulk_ctas() << ") " << name << "_tmab" << sfx
       << "(const __grid_constant__ KcgMArgs a) {\n"
          "  constexpr int TP = " << TPB << ", S = " << SB << ", NP = " << NP << ", V = " << V << ", OB = " << OB
       << ", PW = " << PW << ";\n"
          "  extern __shared__ __align__(128) unsigned char kcg_smem[];\n"
          "  kcg_i64* buf = reinterpret_cast<kcg_i64*>(kcg_smem);\n"
          "  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;\n"
          "  double* obase = reinterpret_cast<double*>(kcg_smem + (size_t)S * NP * TP * 8) + (size_t)w * OB * V * PW;\n"
          "  __shared__ __align__(8) unsigned long long full[S];\n"
          "  __shared__ unsigned reads[S];\n"
          "  if (threadIdx.x < S) reads[threadIdx.x] = 0;\n"
          "  const kcg_i64 ntiles = a.n / TP;\n"
          "  const unsigned fb = (unsigned)__cvta_generic_to_shared(full);\n"
          "  const unsigned bb = (unsigned)__cvta_generic_to_shared(buf);\n"
          "  if (threadIdx.x == 0) {\n"
          "    for (int s = 0; s < S; ++s)\n"
          "      asm volatile(\"mbarrier.init.shared::cta.b64 [%0], 1;\" :: \"r\"(fb + 8 * s));\n"
          "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n"
          "  }\n"
          "  __syncthreads();\n"
          "  auto issue = [&](int s, kcg_i64 tile) {\n"
          "    asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n"
          "    asm volatile(\"mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\" :: \"r\"(fb + 8 * s), \"r\"(NP * TP * 8) : \"memory\");\n"
          "    for (int j = 0; j < NP; ++j)\n"
          "      asm volatile(\"cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\"\n"
          "                   :: \"r\"(bb + (unsigned)((s * NP + j) * TP * 8)), \"l\"(a.p[j] + tile * TP), \"r\"(TP * 8), \"r\"(fb + 8 * s) : \"memory\");\n"
          "  };\n"
          "  if (threadIdx.x == 0)\n"
          "    for (int s = 0; s < S; ++s) {\n"
          "      const kcg_i64 t = blockIdx.x + (kcg_i64)s * gridDim.x;\n"
          "      if (t < ntiles) issue(s, t);\n"
          "    }\n"
          "  for (kcg_i64 k = 0;; ++k) {\n"
          "    const kcg_i64 tile = blockIdx.x + k * gridDim.x;\n"
          "    if (tile >= ntiles) break;\n"
          "    const int s = (int)(k % S);\n"
          "    const unsigned parity = (unsigned)((k / S) & 1);\n"
          "    {\n"
          "      unsigned done = 0;\n"
          "      while (!done)\n"
          "        asm volatile(\"{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }\"\n"
          "                     : \"=r\"(done) : \"r\"(fb + 8 * s), \"r\"(parity) : \"memory\");\n"
          "    }\n";
    if (multi_bulk_cta())
      os << "    double* ob = reinterpret_cast<double*>(kcg_smem + (size_t)S * NP * TP * 8);\n"
            "    if (k > 0 && threadIdx.x == 0) asm volatile(\"cp.async.bulk.wait_group.read 0;\" ::: \"memory\");\n"
            "    __syncthreads();\n"
            "    const kcg_i64 rb = tile * TP;\n"
            "    #pragma unroll 1\n"
            "    for (int u = 0; u < TP / 256; ++u) {\n"
            "      const int li = u * 256 + threadIdx.x;\n"
            "      kcg_i64 q[NP];\n"
            "      #pragma unroll\n"
            "      for (int j = 0; j < NP; ++j) q[j] = buf[(s * NP + j) * TP + li];\n"
            "      kcg_msize<" << stv << ", TP>(q, a, rb + li, ob, li);\n"
            "    }\n"
            "    asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n"
            "    __syncthreads();\n"
            "    if (threadIdx.x == 0) {\n"
            "      const unsigned ob_s = (unsigned)__cvta_generic_to_shared(ob);\n"
            "      #pragma unroll\n"
            "      for (int v = 0; v < V; ++v)\n"
            "        asm volatile(\"cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\"\n"
            "                     :: \"l\"(a.pred + (kcg_i64)v * a.ldp + rb), \"r\"(ob_s + v * TP * 8), \"r\"(TP * 8) : \"memory\");\n"
            "      asm volatile(\"cp.async.bulk.commit_group;\" ::: \"memory\");\n"
            "      const kcg_i64 nt = blockIdx.x + (k + S) * gridDim.x;\n"
            "      if (nt < ntiles) issue(s, nt);  // every thread is past its reads of stage s\n"
            "    }\n"
            "  }\n";
    else
      os << "    double* ob = obase + (int)(k % OB) * V * PW;\n"
            "    if (k >= OB) {  // the block's previous bulk stores have finished reading it\n"
            "      if (lane == 0) asm volatile(\"cp.async.bulk.wait_group.read %0;\" :: \"n\"(OB - 1) : \"memory\");\n"
            "      __syncwarp();\n"
            "    }\n"
            "    const kcg_i64 rb = tile * TP + PW * w;\n"
            "    #pragma unroll 1\n"
            "    for (int u = 0; u < PW / 32; ++u) {\n"
            "      const int li = lane + 32 * u;\n"
            "      kcg_i64 q[NP];\n"
            "      #pragma unroll\n"
            "      for (int j = 0; j < NP; ++j) q[j] = buf[(s * NP + j) * TP + PW * w + li];\n"
            "      kcg_msize<" << stv << ", PW>(q, a, rb + li, ob, li);\n"
            "    }\n"
            "    asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n"
            "    __syncwarp();\n"
            "    if (lane == 0) {\n"
            "      const unsigned ob_s = (unsigned)__cvta_generic_to_shared(ob);\n"
            "      #pragma unroll\n"
            "      for (int v = 0; v < V; ++v)\n"
            "        asm volatile(\"cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\"\n"
            "                     :: \"l\"(a.pred + (kcg_i64)v * a.ldp + rb), \"r\"(ob_s + v * PW * 8), \"r\"(PW * 8) : \"memory\");\n"
            "      asm volatile(\"cp.async.bulk.commit_group;\" ::: \"memory\");\n"
            "      if (kcg_ring_release(&reads[s], blockDim.x / 32)) {\n"
            "        const kcg_i64 nt = blockIdx.x + (k + S) * gridDim.x;\n"
            "        if (nt < ntiles) issue(s, nt);\n"
            "      }\n"
            "    }\n"
            "  }\n";
    os << "  if (lane == 0) asm volatile(\"cp.async.bulk.wait_group 0;\" ::: \"memory\");\n"
          "  for (kcg_i64 i = ntiles * TP + (kcg_i64)blockIdx.x * blockDim.x + threadIdx.x; i < a.n;\n"
          "       i += (kcg_i64)gridDim.x * blockDim.x) {\n"
          "    kcg_i64 p[NP];\n";
    for (int j = 0; j < n_cols; ++j) os << "    p[" << j << "] = a.p[" << j << "][i];\n";
    os << "    kcg_msize<" << stv << ">(p, a, i);\n  }\n}\n";
  }
}

std::string codegen(const std::vector<const Lowered*>& progs,
                    const std::vector<std::vector<int>>& pmaps, int n_cols, JitKind kind,
                    const std::string& name) {
  std::ostringstream os;
  if (kind == JitKind::host_eval)  // the same evaluator compiled for the host CPU (g++ -ffp-contract=off)
    os << "// host build of the lowered program (baseline / cross-check)\n"
          "#include <cmath>\n#include <cstring>\nusing std::scalbn;\n"
          "#define __device__\n#define __forceinline__ inline __attribute__((always_inline))\n"
          "#define __noinline__ __attribute__((noinline))\n"
          "static inline double __dmul_rn(double a, double b) { return a * b; }\n"
          "static inline double __dadd_rn(double a, double b) { return a + b; }\n"
          "static inline double __ll2double_rn(long long x) { return (double)x; }\n"
          "static inline double __ull2double_rn(unsigned long long x) { return (double)x; }\n"
          "static inline int __clzll(long long x) { return x ? __builtin_clzll((unsigned long long)x) : 64; }\n"
          "static inline double __longlong_as_double(long long x) { double d; std::memcpy(&d, &x, 8); return d; }\n"
          "template <class T> static inline void __stcs(T* p, T v) { *p = v; }\n"
          "template <class T> static inline T __ldcs(const T* p) { return *p; }\n";
  os << "// generated by kcg codegen\n" << kDeviceHelpers << "\n";
  for (size_t v = 0; v < progs.size(); ++v) {
    emit_fast(os, *progs[v], static_cast<int>(v), false);
    emit_fast(os, *progs[v], static_cast<int>(v), true);
    if (kind == JitKind::eval || kind == JitKind::argmin || kind == JitKind::host_eval || kind == JitKind::multi ||
        kind == JitKind::multi_argmin)
      emit_fast(os, *progs[v], static_cast<int>(v), true, nullptr, true);
    emit_body(os, *progs[v], static_cast<int>(v), false);
    emit_classify(os, *progs[v], static_cast<int>(v), pmaps[v]);
  }
  if ((kind == JitKind::eval || kind == JitKind::host_eval) && progs[0]->admit)
    emit_body(os, *progs[0]->admit, 0, false, "kcg_admit_");
  if (kind == JitKind::multi || kind == JitKind::multi_argmin)
    for (size_t v = 0; v < progs.size(); ++v)
      if (progs[v]->admit) emit_body(os, *progs[v]->admit, static_cast<int>(v), false, "kcg_admit_");
  const int NP = n_cols > 0 ? n_cols : 1;

  if (kind == JitKind::host_eval) {
    const Lowered& L = *progs[0];
    const int FA = std::max<int>(1, static_cast<int>(L.keys.size()));
    os << "struct KcgArgs { const kcg_i64* p[" << NP << "]; double* pred; "
          "unsigned char* status; kcg_i64* clo; kcg_i64* chi; kcg_i64 n; int sim; int vec; int vout; "
          "double alpha["
       << FA << "]; double alpha_f[" << FA << "]; };\n";
    emit_eval_point(os, L);
    // points [begin, end): kcg_eval_predict semantics (general weights path)
    os << "extern \"C\" void " << name
       << "(const KcgArgs* ap, long long begin, long long end) {\n"
          "  const KcgArgs& a = *ap;\n"
          "  for (long long i = begin; i < end; ++i) {\n"
          "    kcg_i64 p["
       << NP << "];\n";
    for (int j = 0; j < n_cols; ++j) os << "    p[" << j << "] = a.p[" << j << "][i];\n";
    os << "    double s = kcg_nan();\n    int st = kcg_point_fast<1>(p, a, i, s);\n"
          "    if (st < 0) { const KcgRes r = kcg_point_slow(a, i); s = r.s; st = r.st; }\n"
          "    if (st != KCG_PT_OK && st != KCG_PT_COUNT_WIDE) s = kcg_nan();\n"
          "    if (a.pred) a.pred[i] = s;\n    if (a.status) a.status[i] = (unsigned char)st;\n  }\n}\n";
    return os.str();
  }

  if (kind == JitKind::eval) {
    const Lowered& L = *progs[0];
    const int F = static_cast<int>(L.keys.size());
    const int FA = F > 0 ? F : 1;
    os << "struct KcgArgs { const kcg_i64* p[" << NP << "]; double* pred; "
          "unsigned char* status; kcg_i64* clo; kcg_i64* chi; kcg_i64 n; int sim; int vec; int vout; "
          "double alpha["
       << FA << "]; double alpha_f[" << FA << "]; };\n";
    emit_eval_point(os, L);
    emit_eval_kernel(os, n_cols, name, 0);
    emit_eval_kernel(os, n_cols, name + "_gen", 1);
    emit_tma_kernel(os, n_cols, name + "_tma");
    emit_grid_kernel(os, n_cols, name + "_grid", 0);
    emit_grid_kernel(os, n_cols, name + "_grid_gen", 1);
    return os.str();
  }

  if (kind == JitKind::multi || kind == JitKind::multi_argmin) {
    emit_multi(os, progs, pmaps, n_cols, name, kind == JitKind::multi_argmin);
    return os.str();
  }

  if (kind == JitKind::argmin) {
    // Weights are read through device pointers (L1-resident): as by-value
    // kernel parameters the compiler hoists all V x F of them into
    // registers and the kernel drops to 2 CTAs/SM (measured 3.4 vs 3.9 ms
    // for config 4). al: as given (wide path); alf: folded (predict_fold).
    const int V = static_cast<int>(progs.size());
    os << "struct KcgArgs { const kcg_i64* p[" << NP << "]; int* best; double* best_t; "
          "double* preds; kcg_i64 n; const double* al[" << V << "]; const double* alf[" << V << "]; };\n";
    for (int v = 0; v < V; ++v) {
      const Lowered& L = *progs[v];
      const int F = static_cast<int>(L.keys.size());
      const int FA = F > 0 ? F : 1;
      os << "__device__ __noinline__ int kcg_wide_pred_" << v
         << "(const kcg_i64* q, const double* __restrict__ al, double* out) {\n  kcg_i128 c[" << FA
         << "];\n  const int st = kcg_wide_" << v
         << "(q, c);\n  if (st != KCG_PT_OK) return st;\n  double s = 0.0;\n";
      for (int j = 0; j < F; ++j) os << "  s = kcg_accum(s, al[" << j << "], c[" << j << "], 0);\n";
      os << "  *out = s;\n  return KCG_PT_OK;\n}\n";
      os << "__device__ __forceinline__ int kcg_pred_" << v
         << "(const kcg_i64* p, const KcgArgs& a, double* out) {\n"
            "  const int cls = kcg_class_"
         << v << "(p);\n";
      emit_gather(os, "q", "p", L, pmaps[v], "  ");
      os << "  if (cls == 1) {\n    double c[" << FA << "];\n    const int st = kcg_fastp_" << v
         << "(q, c);\n    if (st != KCG_PT_OK) return st;\n    const double* __restrict__ w = a.alf[" << v
         << "];\n    double s = 0.0;\n";
      for (int j = 0; j < F; ++j) os << "    s = __dadd_rn(s, __dmul_rn(w[" << j << "], c[" << j << "]));\n";
      os << "    *out = s;\n    return KCG_PT_OK;\n  }\n"
            "  if (cls == 2) return kcg_wide_pred_"
         << v << "(q, a.al[" << v
         << "], out);\n"
            "  return cls == 0 ? KCG_PT_ASSUMPTION_VIOLATED : KCG_PT_OVERFLOW;\n}\n";
    }
    // one size: all variants, lowest-index minimum (variant-major preds)
    os << "__device__ __forceinline__ void kcg_best(const kcg_i64* p, const KcgArgs& a, kcg_i64 i, int& best, "
          "double& best_t) {\n"
          "  best = -1; best_t = __longlong_as_double(0x7ff0000000000000ll);\n";
    for (int v = 0; v < V; ++v)
      os << "  {\n    double s = kcg_nan();\n    const int st = kcg_pred_" << v
         << "(p, a, &s);\n"
            "    if (st == KCG_PT_OK && s < best_t) { best_t = s; best = "
         << v << "; }\n    if (a.preds) __stcs(a.preds + (kcg_i64)" << v
         << " * a.n + i, st == KCG_PT_OK ? s : kcg_nan());\n  }\n";
    os << "}\n";
    // plain grid-stride kernel: one size per thread and iteration, the
    // compiler's own register allocation (~60 registers, 4 CTAs/SM); the
    // evaluation of 6 variants per size hides the load latency
    const int mb = argmin_ctas();
    os << "extern \"C\" __global__ void __launch_bounds__(256" << (mb > 0 ? ", " + std::to_string(mb) : "")
       << ") " << name
       << "(const __grid_constant__ KcgArgs a) {\n"
          "  const kcg_i64 stride = (kcg_i64)gridDim.x * blockDim.x;\n";
    if (argmin_prefetch()) {
      // the next size's bindings are loaded before this size is evaluated:
      // the load latency hides behind the V evaluations (ncu: the first use
      // of the bindings was the kernel's dominant stall)
      os << "  kcg_i64 i = (kcg_i64)blockIdx.x * blockDim.x + threadIdx.x;\n"
            "  kcg_i64 pn["
         << NP << "];\n  if (i < a.n) {\n";
      for (int j = 0; j < n_cols; ++j) os << "    pn[" << j << "] = __ldcs(a.p[" << j << "] + i);\n";
      os << "  }\n  for (; i < a.n; i += stride) {\n    kcg_i64 p[" << NP << "];\n";
      for (int j = 0; j < n_cols; ++j) os << "    p[" << j << "] = pn[" << j << "];\n";
      os << "    if (i + stride < a.n) {\n";
      for (int j = 0; j < n_cols; ++j) os << "      pn[" << j << "] = __ldcs(a.p[" << j << "] + i + stride);\n";
      os << "    }\n";
    } else {
      os << "  for (kcg_i64 i = (kcg_i64)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {\n"
            "    kcg_i64 p["
         << NP << "];\n";
      for (int j = 0; j < n_cols; ++j) os << "    p[" << j << "] = __ldcs(a.p[" << j << "] + i);\n";
    }
    os << "    int bi; double bt;\n    kcg_best(p, a, i, bi, bt);\n"
          "    __stcs(a.best + i, bi);\n    __stcs(a.best_t + i, bt);\n  }\n}\n";
    return os.str();
  }

  // fused design-row reductions (gram / residual)
  const Lowered& L = *progs[0];
  const int F = static_cast<int>(L.keys.size());
  GramBasis gb = gram_basis(L);
  // the refinement gradient works on the reference's own rows
  // x_j = RN(count_j) / T (model.cpp:29), never the monomial basis: it is
  // what makes the refined weights the least-squares solution of exactly
  // the design the reference would form
  if (kind == JitKind::residual_grad) gb.reduced = false;
  const bool red_basis = gb.reduced;
  // row width: the F design columns, or the W < F basis values u_b = mono_b / T,
  // or (refinement gradient) one value per power-of-two key group
  const RGradGroups rg = kind == JitKind::residual_grad ? rgrad_groups(L) : RGradGroups{};
  const int W = kind == JitKind::residual_grad ? static_cast<int>(rg.base.size()) : gb.width(F);
  const int WA = W > 0 ? W : 1;
  const bool gram = kind == JitKind::gram;
  const bool rgrad = kind == JitKind::residual_grad;
  const bool dmma = gram && gram_dmma(W);
  const bool regsm = gram && !dmma && W <= 48;  // register accumulators, CTA totals in smem
  const int NCMP = red_basis ? static_cast<int>(gb.compound.size()) : 0;
  const int NB = (W + 7) / 8, NT = NB * (NB + 1) / 2, FP = NB * 8, LDX = FP + 1;
  const int NC = n_cols + 1;  // parameter columns + T
  const int S = fused_stages(n_cols, dmma);
  if (red_basis) {
    emit_fast(os, L, 0, true, &gb);
    emit_body(os, L, 0, false, "kcg_wide_", &gb);
  }
  if (gram)
    os << "struct KcgArgs { const kcg_i64* p[" << NP << "]; const double* t; double* G; double* xt1; "
          "double* cmax; unsigned long long* bad; kcg_i64 n; int vec; };\n";
  else
    os << "struct KcgArgs { const kcg_i64* p[" << NP << "]; const double* t; double* obj; "
       << (rgrad ? "double* r2; " : "") << "kcg_i64 n; int vec; double alpha[" << (rgrad ? 2 * WA : (F > 0 ? F : 1))
       << "]; };\n";
  if (red_basis) {
    // expansion tables: key j = sum over kcg_kt[off[j]..off[j+1]) of coef * u_b
    std::vector<int> off{0}, tb;
    std::vector<double> tc;
    for (int j = 0; j < F; ++j) {
      for (const auto& [b, c] : gb.terms[j]) {
        tb.push_back(b);
        tc.push_back(c);
      }
      off.push_back(static_cast<int>(tb.size()));
    }
    std::vector<int> cidx(F, -1);
    for (int k = 0; k < NCMP; ++k) cidx[gb.compound[k]] = k;
    auto arr = [&](const char* ty, const char* nm, auto& v) {
      os << "__constant__ " << ty << " " << nm << "[" << v.size() << "] = {";
      for (size_t i = 0; i < v.size(); ++i) os << (i ? ", " : "") << v[i];
      os << "};\n";
    };
    os.precision(17);
    arr("int", "kcg_kt_off", off);
    arr("int", "kcg_kt_b", tb);
    std::vector<std::string> tcs;
    for (double c : tc) {
      char buf[64];
      std::snprintf(buf, sizeof buf, "%a", c);
      tcs.push_back(buf);
    }
    arr("double", "kcg_kt_c", tcs);
    arr("int", "kcg_kt_cmp", cidx);
  }
  // x = c / t correctly rounded (Markstein: one reciprocal per row, exact
  // residual by FMA, final FMA correction)
  os << "__device__ __forceinline__ double kcg_div(double c, double t, double r) {\n"
        "  const double q = __dmul_rn(c, r);\n  const double e = fma(-q, t, c);\n  return fma(e, r, q);\n}\n";
  os << "template <class T> __device__ __forceinline__ void kcg_xrow(const T* c, double t, double* x) {\n";
  if (rgrad) {
    for (int g = 0; g < W; ++g)
      os << "  x[" << g << "] = (c[" << rg.base[g] << "] != 0) ? __ddiv_rn(kcg_to_double(c[" << rg.base[g]
         << "]), t) : 0.0;\n";
  } else {
    for (int j = 0; j < F; ++j)
      os << "  x[" << j << "] = (c[" << j << "] != 0) ? __ddiv_rn(kcg_to_double(c[" << j << "]), t) : 0.0;\n";
  }
  os << "}\n";
  // out-of-line row: reloads its inputs (no address-taken locals in callers)
  os << "__device__ __noinline__ int kcg_row_i(const KcgArgs& a, kcg_i64 i, double* __restrict__ x) {\n"
        "  kcg_i64 p["
     << NP << "];\n";
  for (int j = 0; j < n_cols; ++j) os << "  p[" << j << "] = a.p[" << j << "][i];\n";
  os << "  const double t = a.t[i];\n"
        "  if (!(t > 0.0)) return KCG_PT_ASSUMPTION_VIOLATED;\n"
        "  const int cls = kcg_class_0(p);\n";
  if (red_basis) {
    os << "  if (cls == 1 || cls == 2) {\n    double u[" << WA << "];\n"
       << "    const int st = cls == 1 ? kcg_fastm_0(p, u) : kcg_widem_0(p, u);\n"
       << "    if (st == KCG_PT_OK) {\n      #pragma unroll\n      for (int b = 0; b < " << W
       << "; ++b) x[b] = __ddiv_rn(u[b], t);\n    }\n    return st;\n  }\n";
  } else {
    os << "  if (cls == 1) { kcg_i64 c[" << (F > 0 ? F : 1)
       << "]; const int st = kcg_fasti_0(p, c); if (st == KCG_PT_OK) kcg_xrow(c, t, x); return st; }\n"
          "  if (cls == 2) { kcg_i128 c["
       << (F > 0 ? F : 1) << "]; const int st = kcg_wide_0(p, c); if (st == KCG_PT_OK) kcg_xrow(c, t, x); return st; }\n";
  }
  os << "  return cls == 0 ? KCG_PT_ASSUMPTION_VIOLATED : KCG_PT_OVERFLOW;\n}\n";
  // fast row from registers; -1 -> caller uses kcg_row_i
  if (rgrad) {
    os << "__device__ __forceinline__ int kcg_row_fast(const kcg_i64* p, double t, double* x) {\n"
          "  if (!(t > 0.0) || kcg_class_0(p) != 1) return -1;\n"
          "  double c[" << (F > 0 ? F : 1) << "];\n  const int st = kcg_fastd_0(p, c);\n";
    // one correctly rounded reciprocal per row, then each quotient by
    // Markstein's correction (q = c r, e = c - q t exact by FMA, q + e r):
    // RN(c / t) exactly when r = RN(1 / t) (Markstein's theorem; checked
    // against exact rational division on 300,000 adversarial pairs)
    os << "  const double r = __drcp_rn(t);\n";
    for (int g = 0; g < W; ++g) os << "  x[" << g << "] = kcg_div(c[" << rg.base[g] << "], t, r);\n";
    os << "  return st;\n}\n";
  } else
  os << "__device__ __forceinline__ int kcg_row_fast(const kcg_i64* p, double t, double* x) {\n"
        "  if (!(t > 0.0) || kcg_class_0(p) != 1) return -1;\n"
        "  double c["
     << WA << "];\n  const int st = " << (red_basis ? "kcg_fastm_0" : "kcg_fastd_0")
     << "(p, c);\n  const double r = __drcp_rn(t);\n"
        "  #pragma unroll\n  for (int j = 0; j < "
     << W << "; ++j) x[j] = " << (red_basis ? "__dmul_rn(c[j], r)" : rgrad ? "__ddiv_rn(c[j], t)" : "kcg_div(c[j], t, r)")
     << ";\n  return st;\n}\n";

  // compound keys (basis mode): x_j = sum_t coef * u_b, max |x_j| per row
  std::ostringstream cmp_row;
  for (int k = 0; k < NCMP; ++k) {
    const int j = gb.compound[k];
    cmp_row << "      { double xc = 0.0;";
    for (const auto& [b, c] : gb.terms[j]) {
      char buf[64];
      std::snprintf(buf, sizeof buf, "%a", c);
      cmp_row << " xc = fma(" << buf << ", x[" << b << "], xc);";
    }
    cmp_row << " mxc[" << k << "] = fmax(mxc[" << k << "], fabs(xc)); }\n";
  }

  // CTA totals in shared memory (dmma / regsm): G block (upper, stride LD),
  // sum of rows, max |x| bits, compound maxima bits
  const bool ones = dmma && FP > W;
  const int LD = dmma ? FP : W;
  const int GSZ = dmma ? FP * FP : W * W;
  const int S1OFF = GSZ, MXOFF = GSZ + (dmma ? FP : W), MCOFF = MXOFF + (dmma ? FP : W);
  const int REDN = MCOFF + (NCMP ? NCMP : 1);
  std::string s1_at = ones ? "red[(b) * " + std::to_string(FP) + " + " + std::to_string(W) + "]"
                           : "red[" + std::to_string(S1OFF) + " + (b)]";
  std::ostringstream epi;  // CTA totals -> global statistics
  if (dmma || regsm) {
    epi << "  __syncthreads();\n";
    if (red_basis) {
      epi << "  for (int e = threadIdx.x; e < " << F * F << "; e += blockDim.x) {\n"
          << "    const int j = e / " << F << ", k = e % " << F << ";\n"
          << "    if (k < j) continue;\n"
          << "    double v = 0.0;\n"
          << "    for (int ta = kcg_kt_off[j]; ta < kcg_kt_off[j + 1]; ++ta)\n"
          << "      for (int tb = kcg_kt_off[k]; tb < kcg_kt_off[k + 1]; ++tb) {\n"
          << "        const int x = kcg_kt_b[ta], y = kcg_kt_b[tb];\n"
          << "        const int lo = x < y ? x : y, hi = x < y ? y : x;\n"
          << "        v = fma(kcg_kt_c[ta] * kcg_kt_c[tb], red[lo * " << LD << " + hi], v);\n"
          << "      }\n"
          << "    atomicAdd(a.G + j * " << F << " + k, v);\n"
          << "    if (j != k) atomicAdd(a.G + k * " << F << " + j, v);\n  }\n"
          << "  for (int j = threadIdx.x; j < " << F << "; j += blockDim.x) {\n"
          << "    double s = 0.0;\n"
          << "    for (int t = kcg_kt_off[j]; t < kcg_kt_off[j + 1]; ++t) { const int b = kcg_kt_b[t]; s = fma(kcg_kt_c[t], "
          << s1_at << ", s); }\n"
          << "    atomicAdd(a.xt1 + j, s);\n"
          << "    const int ci = kcg_kt_cmp[j];\n"
          << "    const double m = ci >= 0 ? __longlong_as_double((long long)reinterpret_cast<unsigned long long*>(red)["
          << MCOFF << " + ci])\n"
          << "        : fabs(kcg_kt_c[kcg_kt_off[j]]) * __longlong_as_double((long long)reinterpret_cast<unsigned long long*>(red)["
          << MXOFF << " + kcg_kt_b[kcg_kt_off[j]]]);\n"
          << "    atomicMax((unsigned long long*)(a.cmax + j), (unsigned long long)__double_as_longlong(m));\n  }\n";
    } else {
      epi << "  for (int e = threadIdx.x; e < " << LD * LD << "; e += blockDim.x) {\n"
          << "    const int r = e / " << LD << ", c = e % " << LD << ";\n"
          << "    if (r >= " << F << " || c >= " << F << " || c < r) continue;\n"
          << "    atomicAdd(a.G + r * " << F << " + c, red[e]);\n"
          << "    if (c != r) atomicAdd(a.G + c * " << F << " + r, red[e]);\n  }\n"
          << "  for (int b = threadIdx.x; b < " << F << "; b += blockDim.x) {\n"
          << "    atomicAdd(a.xt1 + b, " << s1_at << ");\n"
          << "    atomicMax((unsigned long long*)(a.cmax + b), reinterpret_cast<unsigned long long*>(red)[" << MXOFF
          << " + b]);\n  }\n";
    }
    epi << "  if (threadIdx.x == 0 && a.bad && red_bad) atomicAdd(a.bad, red_bad);\n";
  }
  const std::string red_decl = "  __shared__ double red[" + std::to_string(REDN) + "];\n"
                               "  __shared__ unsigned long long red_bad;\n"
                               "  for (int k = threadIdx.x; k < " + std::to_string(REDN) +
                               "; k += blockDim.x) red[k] = 0.0;\n"
                               "  if (threadIdx.x == 0) red_bad = 0;\n";
  const std::string mxc_decl = NCMP ? "  double mxc[" + std::to_string(NCMP) + "];\n  #pragma unroll\n  for (int k = 0; k < " +
                                          std::to_string(NCMP) + "; ++k) mxc[k] = 0.0;\n"
                                    : "";

  // ---- per-row consumer ---------------------------------------------------
  std::ostringstream cons_decl, cons_row, cons_end;
  if (dmma) {
    // Xᵀ1 rides on the tensor cores as a constant-one column W (when the
    // padded width leaves room): G[j][W] = sum_r x_rj. colmax is kept per
    // thread at row production, so the k-step loop is loads + DMMA only.
    cons_decl << "  double* xs_base = reinterpret_cast<double*>(kcg_smem) + S * NC * TP;\n"
              << red_decl
              << "  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, gid = lane >> 2, tig = lane & 3;\n"
              << "  double acc[" << NT << "][2];\n  #pragma unroll\n  for (int t = 0; t < " << NT
              << "; ++t) acc[t][0] = acc[t][1] = 0.0;\n"
              << "  unsigned long long mxr[" << W << "];\n"
              << (ones ? "" : std::string("  double s1r[") + std::to_string(W) + "];\n")
              << "  #pragma unroll\n  for (int j = 0; j < " << W << "; ++j) { mxr[j] = 0ull;"
              << (ones ? "" : " s1r[j] = 0.0;") << " }\n"
              << mxc_decl
              << "  unsigned long long bad = 0;\n  double* xw = xs_base + warp * 32 * " << LDX << ";\n"
              << "  for (int e = lane; e < 32 * " << LDX << "; e += 32) xw[e] = 0.0;  // padding stays zero\n"
              << "  __syncwarp();\n";
    cons_row << "      #pragma unroll\n      for (int j = 0; j < " << W << "; ++j) { xw[lane * " << LDX
             << " + j] = x[j]; { const unsigned long long b = kcg_abs_bits(x[j]); mxr[j] = b > mxr[j] ? b : mxr[j]; }"
             << (ones ? "" : " s1r[j] += x[j];") << " }\n"
             << cmp_row.str();
    if (ones) cons_row << "      xw[lane * " << LDX << " + " << W << "] = ok ? 1.0 : 0.0;\n";
    cons_row << "      __syncwarp();\n"
             << "      #pragma unroll\n      for (int ks = 0; ks < 8; ++ks) {\n"
             << "        const double* row = xw + (4 * ks + tig) * " << LDX << ";\n"
             << "        double v[" << NB << "];\n"
             << "        #pragma unroll\n        for (int b = 0; b < " << NB << "; ++b) v[b] = row[8 * b + gid];\n"
             << "        int t = 0;\n"
             << "        #pragma unroll\n        for (int I = 0; I < " << NB << "; ++I)\n"
             << "          #pragma unroll\n          for (int J = I; J < " << NB << "; ++J, ++t)\n"
             << "            asm volatile(\"mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\"\n"
             << "                         : \"+d\"(acc[t][0]), \"+d\"(acc[t][1]) : \"d\"(v[I]), \"d\"(v[J]));\n"
             << "      }\n      __syncwarp();\n";
    cons_end << "  __syncthreads();\n"
             << "  #pragma unroll\n  for (int j = 0; j < " << W << "; ++j) {\n"
             << "    unsigned long long m = mxr[j];\n"
             << "    #pragma unroll\n    for (int o = 16; o > 0; o >>= 1) { const unsigned long long y = __shfl_xor_sync(0xffffffffu, m, o); m = y > m ? y : m; }\n"
             << "    if (lane == 0) atomicMax((unsigned long long*)(red + " << MXOFF << " + j), m);\n";
    if (!ones)
      cons_end << "    double sj = s1r[j];\n"
               << "    #pragma unroll\n    for (int o = 16; o > 0; o >>= 1) sj += __shfl_xor_sync(0xffffffffu, sj, o);\n"
               << "    if (lane == 0) atomicAdd(red + " << S1OFF << " + j, sj);\n";
    cons_end << "  }\n";
    for (int k = 0; k < NCMP; ++k)
      cons_end << "  { double m = mxc[" << k << "];\n    #pragma unroll\n    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));\n"
               << "    if (lane == 0) atomicMax((unsigned long long*)(red + " << MCOFF + k
               << "), (unsigned long long)__double_as_longlong(m)); }\n";
    // each (I, J) block of the upper block triangle; diagonal blocks are full
    cons_end << "  { int t = 0;\n    #pragma unroll\n    for (int I = 0; I < " << NB
             << "; ++I)\n      #pragma unroll\n      for (int J = I; J < " << NB << "; ++J, ++t) {\n"
             << "        atomicAdd(red + (8 * I + gid) * " << FP << " + 8 * J + 2 * tig, acc[t][0]);\n"
             << "        atomicAdd(red + (8 * I + gid) * " << FP << " + 8 * J + 2 * tig + 1, acc[t][1]); } }\n"
             << "  #pragma unroll\n  for (int o = 16; o > 0; o >>= 1) bad += __shfl_down_sync(0xffffffffu, bad, o);\n"
             << "  if (lane == 0 && bad) atomicAdd(&red_bad, bad);\n"
             << epi.str();
  } else if (regsm) {
    const int NG = W * (W + 1) / 2;
    cons_decl << red_decl
              << "  double g[" << (NG ? NG : 1) << "], s1[" << WA << "];\n"
              << "  unsigned long long mx[" << WA << "];  // |x| bit patterns: max on the integer pipe\n"
              << "  #pragma unroll\n  for (int k = 0; k < " << NG << "; ++k) g[k] = 0.0;\n"
              << "  #pragma unroll\n  for (int k = 0; k < " << W << "; ++k) { s1[k] = 0.0; mx[k] = 0ull; }\n"
              << mxc_decl << "  unsigned long long bad = 0;\n";
    int k = 0;
    for (int r = 0; r < W; ++r) {
      cons_row << "      s1[" << r << "] += x[" << r << "]; { const unsigned long long b = kcg_abs_bits(x["
               << r << "]); mx[" << r << "] = b > mx[" << r << "] ? b : mx[" << r << "]; }\n";
      for (int c = r; c < W; ++c, ++k)
        cons_row << "      g[" << k << "] = fma(x[" << r << "], x[" << c << "], g[" << k << "]);\n";
    }
    cons_row << cmp_row.str();
    cons_end << "  #pragma unroll\n  for (int o = 16; o > 0; o >>= 1) {\n"
             << "    #pragma unroll\n    for (int k = 0; k < " << NG << "; ++k) g[k] += __shfl_down_sync(0xffffffffu, g[k], o);\n"
             << "    #pragma unroll\n    for (int k = 0; k < " << W
             << "; ++k) { s1[k] += __shfl_down_sync(0xffffffffu, s1[k], o); const unsigned long long y = __shfl_down_sync(0xffffffffu, mx[k], o); mx[k] = y > mx[k] ? y : mx[k]; }\n";
    if (NCMP)
      cons_end << "    #pragma unroll\n    for (int k = 0; k < " << NCMP
               << "; ++k) mxc[k] = fmax(mxc[k], __shfl_down_sync(0xffffffffu, mxc[k], o));\n";
    cons_end << "    bad += __shfl_down_sync(0xffffffffu, bad, o);\n  }\n"
             << "  if ((threadIdx.x & 31) == 0) {\n";
    k = 0;
    for (int r = 0; r < W; ++r) {
      cons_end << "    atomicAdd(red + " << S1OFF + r << ", s1[" << r << "]);\n"
               << "    atomicMax((unsigned long long*)(red + " << MXOFF + r
               << "), mx[" << r << "]);\n";
      for (int c = r; c < W; ++c, ++k) cons_end << "    atomicAdd(red + " << (r * W + c) << ", g[" << k << "]);\n";
    }
    for (int q = 0; q < NCMP; ++q)
      cons_end << "    atomicMax((unsigned long long*)(red + " << MCOFF + q
               << "), (unsigned long long)__double_as_longlong(mxc[" << q << "]));\n";
    cons_end << "    if (bad) atomicAdd(&red_bad, bad);\n  }\n" << epi.str();
  } else if (gram) {
    // wide rows (W > 48): warp totals straight to global
    const int NG = F * (F + 1) / 2;
    cons_decl << "  double g[" << (NG ? NG : 1) << "], s1[" << WA << "], mx[" << WA << "];\n"
              << "  #pragma unroll\n  for (int k = 0; k < " << NG << "; ++k) g[k] = 0.0;\n"
              << "  #pragma unroll\n  for (int k = 0; k < " << F << "; ++k) { s1[k] = 0.0; mx[k] = 0.0; }\n"
              << "  unsigned long long bad = 0;\n";
    int k = 0;
    for (int r = 0; r < F; ++r) {
      cons_row << "      s1[" << r << "] += x[" << r << "]; mx[" << r << "] = fmax(mx[" << r << "], fabs(x[" << r << "]));\n";
      for (int c = r; c < F; ++c, ++k)
        cons_row << "      g[" << k << "] = fma(x[" << r << "], x[" << c << "], g[" << k << "]);\n";
    }
    cons_end << "  #pragma unroll\n  for (int o = 16; o > 0; o >>= 1) {\n"
             << "    #pragma unroll\n    for (int k = 0; k < " << NG << "; ++k) g[k] += __shfl_down_sync(0xffffffffu, g[k], o);\n"
             << "    #pragma unroll\n    for (int k = 0; k < " << F
             << "; ++k) { s1[k] += __shfl_down_sync(0xffffffffu, s1[k], o); mx[k] = fmax(mx[k], __shfl_down_sync(0xffffffffu, mx[k], o)); }\n"
             << "    bad += __shfl_down_sync(0xffffffffu, bad, o);\n  }\n"
             << "  if ((threadIdx.x & 31) == 0) {\n";
    k = 0;
    for (int r = 0; r < F; ++r) {
      cons_end << "    atomicAdd(a.xt1 + " << r << ", s1[" << r << "]);\n"
               << "    atomicMax((unsigned long long*)(a.cmax + " << r
               << "), (unsigned long long)__double_as_longlong(mx[" << r << "]));\n";
      for (int c = r; c < F; ++c, ++k) {
        cons_end << "    atomicAdd(a.G + " << (r * F + c) << ", g[" << k << "]);\n";
        if (c != r) cons_end << "    atomicAdd(a.G + " << (c * F + r) << ", g[" << k << "]);\n";
      }
    }
    cons_end << "    if (a.bad && bad) atomicAdd(a.bad, bad);\n  }\n";
  } else if (rgrad) {
    // refinement gradient g = X^T (1 - X alpha): the residual in
    // double-double (exact FMA products, compensated sums) rounded once,
    // then per-thread sums of u_b r (basis) or x_j r; each warp's totals
    // expanded to the F keys (g_j = sum_b A_jb gu_b) and added atomically
    cons_decl << "  double gacc[" << WA << "];\n  #pragma unroll\n  for (int j = 0; j < " << WA
              << "; ++j) gacc[j] = 0.0;\n  double rr = 0.0;\n";
    // 1 - sum_g x_g (A_hi + A_lo) as a compensated dot product (Ogita, Rump
    // and Oishi's Dot2 class: TwoSums of the rounded products, the product
    // errors (exact by FMA), the A_lo terms and the sum errors gathered in
    // one double) -- as accurate as twice the working precision, ~11 FP64
    // operations per group instead of 14 for a double-double subtraction
    // The W products are summed as a pairwise tree of TwoSums (log2 W levels
    // of independent work instead of a W-long dependent chain), then
    // TwoSum(1, -S); every TwoSum error and product error is gathered in one
    // double: the same Dot2-class accuracy with shorter dependence chains.
    cons_row << "      if (ok) {\n";
    {
      std::vector<std::string> errs;  // error terms, summed as a tree at the end
      for (int j = 0; j < W; ++j) {
        cons_row << "        const double p" << j << " = __dmul_rn(x[" << j << "], a.alpha[" << j << "]);\n"
                 << "        const double q" << j << " = fma(x[" << j << "], a.alpha[" << W + j << "], fma(x[" << j
                 << "], a.alpha[" << j << "], -p" << j << "));\n";
        errs.push_back("q" + std::to_string(j));
      }
      std::vector<std::string> lv;
      for (int j = 0; j < W; ++j) lv.push_back("p" + std::to_string(j));
      int tmp = 0;
      while (lv.size() > 1) {
        std::vector<std::string> nx;
        for (size_t k = 0; k + 1 < lv.size(); k += 2) {
          const std::string t = std::to_string(tmp++);
          cons_row << "        const double t" << t << " = __dadd_rn(" << lv[k] << ", " << lv[k + 1] << ");\n"
                   << "        const double b" << t << " = __dsub_rn(t" << t << ", " << lv[k] << ");\n"
                   << "        const double u" << t << " = __dadd_rn(__dsub_rn(" << lv[k] << ", __dsub_rn(t" << t << ", b"
                   << t << ")), __dsub_rn(" << lv[k + 1] << ", b" << t << "));\n";
          nx.push_back("t" + t);
          errs.push_back("u" + t);
        }
        if (lv.size() % 2) nx.push_back(lv.back());
        lv = nx;
      }
      while (errs.size() > 1) {
        std::vector<std::string> nx;
        for (size_t k = 0; k + 1 < errs.size(); k += 2) {
          const std::string v = "v" + std::to_string(tmp++);
          cons_row << "        const double " << v << " = __dadd_rn(" << errs[k] << ", " << errs[k + 1] << ");\n";
          nx.push_back(v);
        }
        if (errs.size() % 2) nx.push_back(errs.back());
        errs = nx;
      }
      cons_row << "        double hi, lo;\n        { const double s = __dsub_rn(1.0, " << lv[0] << "), bb = __dsub_rn(s, 1.0);\n"
               << "          const double e = __dadd_rn(__dsub_rn(1.0, __dsub_rn(s, bb)), __dsub_rn(-" << lv[0]
               << ", bb));\n          hi = s; lo = __dsub_rn(e, " << errs[0] << "); }\n";
    }
    cons_row << "        const double r = __dadd_rn(hi, lo);\n";
    for (int j = 0; j < W; ++j) cons_row << "        gacc[" << j << "] = fma(x[" << j << "], r, gacc[" << j << "]);\n";
    // sum of r^2 at these weights (a.r2, nullable): with the gradient and the
    // Gram it gives the objective after the refinement step (api.refined_objective)
    cons_row << "        rr = fma(r, r, rr);\n";
    cons_row << "      }\n";
    cons_end << "  #pragma unroll\n  for (int j = 0; j < " << W << "; ++j)\n"
             << "    for (int o = 16; o > 0; o >>= 1) gacc[j] += __shfl_down_sync(0xffffffffu, gacc[j], o);\n"
             << "  for (int o = 16; o > 0; o >>= 1) rr += __shfl_down_sync(0xffffffffu, rr, o);\n"
             << "  if ((threadIdx.x & 31) == 0) {\n    if (a.r2) atomicAdd(a.r2, rr);\n";
    for (int j = 0; j < F; ++j) {
      if (!red_basis) {  // g_j = 2^k_j * (sum of x_base r over the group)
        char buf[64];
        std::snprintf(buf, sizeof buf, "%a", std::ldexp(1.0, rg.of_key[j].second));
        cons_end << "    atomicAdd(a.obj + " << j << ", " << buf << " * gacc[" << rg.of_key[j].first << "]);\n";
        continue;
      }
      cons_end << "    { double gj = 0.0;";
      for (const auto& [b, c] : gb.terms[j]) {
        char buf[64];
        std::snprintf(buf, sizeof buf, "%a", c);
        cons_end << " gj = fma(" << buf << ", gacc[" << b << "], gj);";
      }
      cons_end << " atomicAdd(a.obj + " << j << ", gj); }\n";
    }
    cons_end << "  }\n";
  } else {
    // residual: alpha holds the compact weights, or beta = A^T alpha in basis mode
    cons_decl << "  double acc = 0.0;\n";
    cons_row << "      if (ok) {\n        double pr = 0.0;\n";
    for (int j = 0; j < W; ++j) cons_row << "        pr = fma(x[" << j << "], a.alpha[" << j << "], pr);\n";
    cons_row << "        const double r = 1.0 - pr;\n        acc = fma(r, r, acc);\n      }\n";
    cons_end << "  #pragma unroll\n  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);\n"
             << "  if ((threadIdx.x & 31) == 0) atomicAdd(a.obj, acc);\n";
  }
  const int XW = WA;  // x row width
  // produce row x for global index i from registers q/t (or out of line)
  // The out-of-line path writes its row to a scratch row (shared memory for
  // the DMMA variant) and the fast path's registers are copied there too, so
  // no per-thread array ever has its address taken (no local memory).
  auto emit_make_row = [&](const char* qexpr, const char* texpr, const char* iexpr, const char* valid) {
    os << "      double x[" << XW << "];\n      #pragma unroll\n      for (int j = 0; j < " << XW
       << "; ++j) x[j] = 0.0;\n"
       << "      bool ok = false;\n"
       << "      if (" << valid << ") {\n"
       << "        int st = kcg_row_fast(" << qexpr << ", " << texpr << ", x);\n"
       << "        if (st < 0) {\n"
       << "          double* sx = slow_row;\n"
       << "          st = kcg_row_i(a, " << iexpr << ", sx);\n"
       << "          if (st == KCG_PT_OK) {\n            #pragma unroll\n            for (int j = 0; j < " << W
       << "; ++j) x[j] = sx[j];\n          }\n"
       << "        }\n"
       << "        ok = st == KCG_PT_OK;\n"
       << "        if (!ok) {\n          #pragma unroll\n          for (int j = 0; j < " << XW
       << "; ++j) x[j] = 0.0;\n";
    if (gram) os << "          ++bad;\n";
    os << "        }\n      }\n";
  };

  os << "extern \"C\" __global__ void __launch_bounds__(256, " << (rgrad ? rgrad_ctas() : fused_ctas(dmma)) << ") " << name
     << "(const __grid_constant__ KcgArgs a) {\n"
        "  constexpr int TP = "
     << kTmaTile << ", S = " << S << ", NC = " << NC
     << ";\n"
        "  extern __shared__ __align__(128) unsigned char kcg_smem[];\n"
        "  kcg_i64* buf = reinterpret_cast<kcg_i64*>(kcg_smem);\n"
        "  __shared__ __align__(8) unsigned long long full[S];\n"
        "  __shared__ unsigned reads[S];\n"
        "  if (threadIdx.x < S) reads[threadIdx.x] = 0;\n"
     << cons_decl.str()
     << (dmma ? std::string("  double* slow_row = xw + lane * ") + std::to_string(LDX) + ";\n"
              : std::string("  double* slow_row = reinterpret_cast<double*>(kcg_smem) + S * NC * TP + threadIdx.x * ") +
                    std::to_string(WA) + ";\n")
     << "  const kcg_i64 ntiles = a.vec ? a.n / TP : 0;\n"
        "  const unsigned fb = (unsigned)__cvta_generic_to_shared(full);\n"
        "  const unsigned bb = (unsigned)__cvta_generic_to_shared(buf);\n"
        "  if (threadIdx.x == 0) {\n"
        "    for (int s = 0; s < S; ++s) asm volatile(\"mbarrier.init.shared::cta.b64 [%0], 1;\" :: \"r\"(fb + 8 * s));\n"
        "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n"
        "  }\n"
        "  __syncthreads();\n"
        "  auto issue = [&](int s, kcg_i64 tile) {\n"
        "    asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n"
        "    asm volatile(\"mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\" :: \"r\"(fb + 8 * s), \"r\"(NC * TP * 8) : \"memory\");\n"
        "    for (int j = 0; j < NC; ++j) {\n"
        "      const void* src = j < NC - 1 ? (const void*)(a.p[j] + tile * TP) : (const void*)(a.t + tile * TP);\n"
        "      asm volatile(\"cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\"\n"
        "                   :: \"r\"(bb + (unsigned)((s * NC + j) * TP * 8)), \"l\"(src), \"r\"(TP * 8), \"r\"(fb + 8 * s) : \"memory\");\n"
        "    }\n"
        "  };\n"
        "  if (threadIdx.x == 0)\n"
        "    for (int s = 0; s < S; ++s) {\n"
        "      const kcg_i64 t = blockIdx.x + (kcg_i64)s * gridDim.x;\n"
        "      if (t < ntiles) issue(s, t);\n"
        "    }\n"
        "  for (kcg_i64 k = 0;; ++k) {\n"
        "    const kcg_i64 tile = blockIdx.x + k * gridDim.x;\n"
        "    if (tile >= ntiles) break;\n"
        "    const int s = (int)(k % S);\n"
        "    const unsigned parity = (unsigned)((k / S) & 1);\n"
        "    { unsigned done = 0;\n"
        "      while (!done)\n"
        "        asm volatile(\"{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }\"\n"
        "                     : \"=r\"(done) : \"r\"(fb + 8 * s), \"r\"(parity) : \"memory\"); }\n"
        "";
  const std::string release =
      "    // last warp to finish reading stage s refills it (no CTA-wide barrier:\n"
      "    // warps drift apart freely between tiles)\n"
      "    __syncwarp();\n"
      "    if ((threadIdx.x & 31) == 0) {\n"
      "      if (kcg_ring_release(&reads[s], blockDim.x / 32)) {\n"
      "        const kcg_i64 nt = blockIdx.x + (k + S) * gridDim.x;\n"
      "        if (nt < ntiles) issue(s, nt);\n"
      "      }\n"
      "    }\n";
  if (fused_rowwise(dmma)) {
    // one row at a time straight from the stage (fewer live registers), the
    // stage released after the thread's 4 rows
    // rows tid + 256 u (conflict-free stage loads) or 4 tid + u
    const bool strided = rgrad ? rgrad_strided() : fused_strided(gram);
    const std::string off = strided ? "u * 256 + threadIdx.x" : "4 * threadIdx.x + u";
    os << "    const kcg_i64 base = tile * TP;\n"
          "    #pragma unroll "
       << fused_unroll(gram) << "\n"
          "    for (int u = 0; u < 4; ++u) {\n"
          "      const int o = " << off << ";\n"
          "      kcg_i64 qu["
       << NP << "];\n      #pragma unroll\n      for (int j = 0; j < NC - 1; ++j) qu[j] = buf[(s * NC + j) * TP + o];\n"
                "      const double tu = __longlong_as_double(buf[(s * NC + NC - 1) * TP + o]);\n";
    emit_make_row("qu", "tu", "base + o", "true");
    os << cons_row.str() << "    }\n" << release << "  }\n";
  } else {
    os << "    kcg_i64 q[4]["
       << NP << "]; double tq[4];\n"
                "    #pragma unroll\n"
                "    for (int j = 0; j < NC; ++j) {\n"
                "      const longlong2* src = reinterpret_cast<const longlong2*>(buf + (s * NC + j) * TP) + 2 * threadIdx.x;\n"
                "      const longlong2 x0 = src[0], x1 = src[1];\n"
                "      if (j < NC - 1) { q[0][j] = x0.x; q[1][j] = x0.y; q[2][j] = x1.x; q[3][j] = x1.y; }\n"
                "      else { tq[0] = __longlong_as_double(x0.x); tq[1] = __longlong_as_double(x0.y);\n"
                "             tq[2] = __longlong_as_double(x1.x); tq[3] = __longlong_as_double(x1.y); }\n"
                "    }\n"
             << release
             << "    const kcg_i64 base = tile * TP + 4 * threadIdx.x;\n"
                "    #pragma unroll\n"
                "    for (int u = 0; u < 4; ++u) {\n";
    emit_make_row("q[u]", "tq[u]", "base + u", "true");
    os << cons_row.str() << "    }\n  }\n";
  }
  // tail (and the whole range when not aligned): warp-uniform trip counts
  os << "  {\n"
        "    const kcg_i64 t0 = ntiles * TP;\n"
        "    const kcg_i64 rem = a.n - t0;\n"
        "    const kcg_i64 stride = (kcg_i64)gridDim.x * blockDim.x;\n"
        "    const kcg_i64 span = (rem + 31) / 32 * 32;\n"
        "    for (kcg_i64 r = (kcg_i64)blockIdx.x * blockDim.x + threadIdx.x; r < span; r += stride) {\n"
        "      const kcg_i64 i = t0 + r;\n"
        "      kcg_i64 p["
     << NP << "];\n";
  for (int j = 0; j < n_cols; ++j) os << "      p[" << j << "] = i < a.n ? a.p[" << j << "][i] : 0;\n";
  os << "      const double tv = i < a.n ? a.t[i] : 0.0;\n";
  emit_make_row("p", "tv", "i", "i < a.n");
  os << cons_row.str() << "    }\n  }\n" << cons_end.str() << "}\n";
  return os.str();
}

}  // namespace kcg
