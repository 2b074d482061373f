// Host-side program representation for the kcg back end.
//
// A `Program` is the reference front end's symbolic output for one kernel
// (parameters, assume constraints, nonzero PropertyVector entries as
// CountExpr polynomials) lowered to an integer program the GPU evaluates
// exactly:
//   * every CountExpr (countexpr.hpp:55-117) becomes an integer-coefficient
//     polynomial over atom numerators divided by one static denominator D;
//   * atoms are parameters, floor divisions by constants and n-ary min/max
//     (countexpr.hpp:20-34), scheduled in dependency order;
//   * assume constraints (LinCmp, linexpr.hpp:62-77) become integer forms
//     evaluated per point exactly like AssumeCtx::admits (decide.cpp:153-170).
// Exactness: evaluation is exact in int64 when every parameter is <= b64
// and in int128 when <= b128 (static magnitude analysis, `bounds()`);
// beyond that the point reports KCG_PT_OVERFLOW.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace kcg {

using i128 = __int128;
using u128 = unsigned __int128;

/// sets the calling thread's kcg_last_error() text (capi.cpp)
}  // namespace kcg
extern "C" void kcg_set_last_error(const char* msg);
namespace kcg {

struct KcgError : std::runtime_error {
  int code;
  KcgError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

std::string i128_str(i128 v);
i128 checked_add(i128 a, i128 b);
i128 checked_mul(i128 a, i128 b);
i128 gcd128(i128 a, i128 b);
i128 lcm128(i128 a, i128 b);

/// Exact rational with 128-bit numerator/denominator, normalised; every
/// operation throws KcgError(KCG_E_UNSUPPORTED) instead of overflowing.
struct Q {
  i128 n = 0, d = 1;
  Q() = default;
  Q(i128 v) : n(v), d(1) {}
  Q(i128 num, i128 den);
  bool is_zero() const { return n == 0; }
  bool is_int() const { return d == 1; }
  Q operator+(const Q& o) const;
  Q operator-(const Q& o) const;
  Q operator*(const Q& o) const;
  Q operator-() const { Q r; r.n = -n; r.d = d; return r; }
  bool operator==(const Q& o) const { return n == o.n && d == o.d; }
  std::string str() const;
};

// ---------------------------------------------------------------------------
// Symbolic layer (parsed text)

enum class AtomKind : int { var = 0, floordiv = 1, min = 2, max = 3, quot = 4 };

struct Mono {
  std::vector<std::pair<int, int>> f;  // (atom id, exponent), sorted by atom id
  bool operator<(const Mono& o) const { return f < o.f; }
  bool operator==(const Mono& o) const { return f == o.f; }
};

using Poly = std::map<Mono, Q>;

struct AtomDef {
  AtomKind kind = AtomKind::var;
  int param = -1;          // var
  int num = -1;            // floordiv numerator poly id
  i128 den = 1;            // floordiv denominator (> 0)
  std::vector<int> args;   // min/max argument poly ids
  i128 qmod = 1, qrem = 0; // quot: (param - qrem) / qmod
  std::string key;         // canonical text (identity)
};

enum class CmpOp : int { lt = 0, le = 1, gt = 2, ge = 3, eq = 4 };

struct Constraint {
  bool divisibility = false;
  CmpOp op = CmpOp::eq;
  int poly = -1;       // relational: lhs - rhs; divisibility: lhs
  i128 mod = 0, rem = 0;
  bool absorbed = false;  // folded into a quot atom's exactness check
  std::string text;
};

struct Symbolic {
  std::string kernel;
  std::vector<std::string> params;
  std::vector<AtomDef> atoms;
  std::vector<Poly> polys;
  std::vector<Constraint> cons;
  std::vector<std::pair<int, int>> props;  // (schema index, poly id), schema order
};

Symbolic parse_program_text(const std::string& text);

// ---------------------------------------------------------------------------
// Enumeration program ("kernelcost-enum v1", oracle/kcref_program.hpp
// enum_text): what enumerate_points (enumerate.cpp:371-456) walks. Variables
// of `sym` are the kernel parameters followed by every domain variable name;
// polys are LinExpr / CountExpr texts parsed by the same front end.

struct EnumVar {
  std::string name;
  int lo = -1, hi = -1;  // poly ids; hi exclusive
};

struct EnumAccess {
  int array = -1;
  bool store = false;
  int stride = -1;  // lane_stride_signed poly (global arrays), -1 for local
  std::vector<int> idx;  // poly ids
};

struct EnumStmt {
  bool barrier = false;
  std::vector<EnumVar> vars;
  std::vector<int> guards;  // indices into sym.cons
  std::vector<EnumAccess> acc;
  std::vector<std::pair<int, i128>> ops;  // (schema index, count per point)
};

struct EnumArray {
  std::string name;
  bool global = true;
  int bits = 32, nd = 1, fast = 0;
};

struct EnumSymbolic {
  Symbolic sym;     // sym.params = kernel params + domain variables
  int n_params = 0; // the kernel's own parameters (binding order)
  std::vector<int> assumes;  // indices into sym.cons
  std::vector<EnumArray> arrays;
  std::vector<int> groups;   // group-axis extent polys
  std::vector<EnumStmt> stmts;
};

EnumSymbolic parse_enum_text(const std::string& text);

/// kcg-columns v1 side format (columns.cpp)
}  // namespace kcg
struct kcg_columns {  // a mapped file (include/kcg.h)
  int fd = -1;
  void* map = nullptr;
  size_t map_len = 0;
  bool registered = false;  // mapping page-locked for DMA
  uint64_t n_rows = 0;
  struct Col {
    std::string name;
    int dtype;
    uint64_t offset, nbytes;
  };
  std::vector<Col> cols;
  void* pending = nullptr;  // cudaEvent_t of the last async copy out of the mapping
  ~kcg_columns();
};
namespace kcg {
void columns_write(const char* path, int n_cols, const char* const* names, const int* dtypes,
                   const void* const* data, uint64_t n_rows);
kcg_columns* columns_open(const char* path);
void columns_load(kcg_columns* h, int j, uint64_t row0, size_t n, void* dev, void* stream);

/// enumerate_points at one binding (enumerate.cpp): counts149 gets the bound
/// property vector, points_out the visited points. Synchronous on `stream`
/// (a cudaStream_t). Throws KcgError (E_ASSUMPTION_VIOLATED, E_CAP_EXCEEDED,
/// E_UNSUPPORTED, E_CUDA ...). Returns the number of kernels launched.
int enumerate_points(const EnumSymbolic& E, const int64_t* binding, uint64_t cap, i128* counts149,
                      uint64_t* points_out, void* stream);

// ---------------------------------------------------------------------------
// Lowered integer program

enum OpCode : int32_t {
  OP_VAR = 0,       // atom[dst] = param[a]
  OP_MONO = 1,      // mono[dst] = prod factors[a..b)
  OP_EXPR = 2,      // expr[dst] = sum terms[a..b)
  OP_FLOORDIV = 3,  // atom[dst] = floor(expr[a] / big[c])
  OP_MIN = 4,       // atom[dst] = min over args[a..b) of expr*scale
  OP_MAX = 5,
  OP_QUOT = 6       // atom[dst] = floor((param[a] - quot_rem[c]) / quot_mod[c])
};

struct LOp {
  int32_t code, dst, a, b, c;
};

struct LTerm {
  i128 coef;
  int32_t mono;  // -1: constant term
};

struct LExpr {
  int32_t term_begin, term_end;
  i128 D;  // value = numerator / D
};

struct LArg {
  int32_t expr;
  i128 scale;  // Dm / D_expr
};

struct LCons {
  int32_t divisibility;  // 0 relational, 1 divisibility, 2 quot exactness
  int32_t op;            // relational: CmpOp; quot: parameter index
  int32_t expr;          // relational/divisibility: expr; quot: atom id
  i128 mod, rem;
};

struct LKey {
  int32_t schema, expr;
  // the key's ORIGINAL polynomial (before congruence substitution), when it
  // is one term: form 1 = the constant `coef`; form 2 = coef * prod_j
  // param_j^pexp[j] with coef a positive power of two (the multi-program
  // kernel shares such products across programs); form 3 = the same
  // monomial shape with any rational coefficient coef / coef_den (the
  // refinement gradient groups keys whose counts differ by powers of two);
  // 0 = anything else
  int form = 0;
  i128 coef = 0, coef_den = 1;
  std::vector<int> pexp;
};

struct Lowered {
  int n_params = 0, n_atoms = 0, n_monos = 0, n_exprs = 0;
  std::vector<LOp> ops;
  std::vector<std::pair<int32_t, int32_t>> factors;  // (atom, exp)
  std::vector<LTerm> terms;
  std::vector<LExpr> exprs;
  std::vector<LArg> args;
  std::vector<i128> floordiv_den;  // per floordiv op (index in op.c)
  std::vector<LCons> cons;
  std::vector<LKey> keys;          // schema order
  std::vector<i128> atom_den;      // value = numerator / atom_den
  std::vector<i128> quot_mod, quot_rem;  // per OP_QUOT (index in op.c)
  int64_t b64 = 0, b128 = 0;       // safe uniform parameter bounds
  bool gram_basis = true;          // fused Gram/residual over the monomial basis when narrower
  std::vector<long double> mono_bound64;  // |monomial| bound when params <= b64
  // admissibility-only lowering (no properties): decides E_ASSUMPTION_VIOLATED
  // for points whose counts are beyond the 128-bit bound (admits() is checked
  // before any count in props.cpp:263-269)
  std::shared_ptr<Lowered> admit;
};

Lowered lower(const Symbolic& s);

/// Magnitude bound of the largest intermediate when all |params| <= B.
long double max_intermediate(const Lowered& L, long double B,
                             std::vector<long double>* mono_bounds = nullptr);

// ---------------------------------------------------------------------------
// Schema v1 (schema.cpp:16-38)

const std::vector<std::string>& schema_keys();
int schema_index(const std::string& key);

}  // namespace kcg
