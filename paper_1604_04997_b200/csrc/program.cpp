// Parsing and lowering of front-end programs (see kcg_host.hpp).
//
// Input syntax is exactly what the reference prints:
//   CountExpr::str()  prefix polynomials  (countexpr.cpp:385-416; atom keys
//                     countexpr.cpp:25-49)
//   LinCmp::str()     infix constraints   (linexpr.cpp:97-155)
#include <algorithm>
#include <cctype>
#include <cmath>
#include <functional>
#include <set>
#include <sstream>

#include "../../include/kcg.h"
#include "kcg_host.hpp"

namespace kcg {

// ---------------------------------------------------------------------------
// 128-bit helpers

std::string i128_str(i128 v) {
  if (v == 0) return "0";
  const bool neg = v < 0;
  u128 u = neg ? -static_cast<u128>(v) : static_cast<u128>(v);
  std::string s;
  while (u) {
    s.push_back(static_cast<char>('0' + static_cast<int>(u % 10)));
    u /= 10;
  }
  if (neg) s.push_back('-');
  std::reverse(s.begin(), s.end());
  return s;
}

i128 checked_add(i128 a, i128 b) {
  i128 r;
  if (__builtin_add_overflow(a, b, &r))
    throw KcgError(KCG_E_UNSUPPORTED, "program constant exceeds 128 bits");
  return r;
}

i128 checked_mul(i128 a, i128 b) {
  i128 r;
  if (__builtin_mul_overflow(a, b, &r))
    throw KcgError(KCG_E_UNSUPPORTED, "program constant exceeds 128 bits");
  return r;
}

i128 gcd128(i128 a, i128 b) {
  if (a < 0) a = -a;
  if (b < 0) b = -b;
  while (b) {
    const i128 t = a % b;
    a = b;
    b = t;
  }
  return a;
}

i128 lcm128(i128 a, i128 b) {
  if (a == 0 || b == 0) return 0;
  return checked_mul(a / gcd128(a, b), b < 0 ? -b : b);
}

Q::Q(i128 num, i128 den) {
  if (den == 0) throw KcgError(KCG_E_PARSE, "zero denominator");
  if (den < 0) {
    num = -num;
    den = -den;
  }
  const i128 g = gcd128(num, den);
  n = g ? num / g : 0;
  d = g ? den / g : 1;
  if (n == 0) d = 1;
}

Q Q::operator+(const Q& o) const {
  if (d == o.d) return Q(checked_add(n, o.n), d);
  const i128 g = gcd128(d, o.d);
  const i128 l = checked_mul(d / g, o.d);
  return Q(checked_add(checked_mul(n, l / d), checked_mul(o.n, l / o.d)), l);
}

Q Q::operator-(const Q& o) const { return *this + (-o); }

Q Q::operator*(const Q& o) const {
  const i128 g1 = gcd128(n, o.d), g2 = gcd128(o.n, d);
  const i128 a = g1 ? n / g1 : n, bd = g1 ? o.d / g1 : o.d;
  const i128 b = g2 ? o.n / g2 : o.n, ad = g2 ? d / g2 : d;
  return Q(checked_mul(a, b), checked_mul(ad, bd));
}

std::string Q::str() const {
  return d == 1 ? i128_str(n) : i128_str(n) + "/" + i128_str(d);
}

// ---------------------------------------------------------------------------
// Schema v1: loads, stores over s32/s64/s128 x 15 classes, minls, local,
// flops, barrier, groups, const (schema.cpp:16-38; README "Property schema")

const std::vector<std::string>& schema_keys() {
  static const std::vector<std::string> keys = [] {
    const char* classes[] = {"uniform", "1/1", "1/2", "2/2",  "1/3",
                             "2/3",     "3/3", "1/4", "2/4",  "3/4",
                             "4/4",     "1/>4", "2/>4", "3/>4", "4/>4"};
    const char* sizes[] = {"s32", "s64", "s128"};
    std::vector<std::string> k;
    for (const char* dir : {"load", "store"})
      for (const char* sz : sizes)
        for (const char* c : classes)
          k.push_back(std::string("mem.global.") + dir + "." + sz + "." + c);
    for (const char* sz : sizes)
      for (const char* c : classes)
        k.push_back(std::string("mem.minls.") + sz + "." + c);
    k.push_back("mem.local.load");
    for (const char* dt : {"f32", "f64"})
      for (const char* op : {"addsub", "mul", "div", "pow", "special"})
        k.push_back(std::string("flop.") + dt + "." + op);
    k.push_back("sync.barrier");
    k.push_back("launch.groups");
    k.push_back("launch.const");
    return k;
  }();
  return keys;
}

int schema_index(const std::string& key) {
  static const std::map<std::string, int> idx = [] {
    std::map<std::string, int> m;
    const auto& k = schema_keys();
    for (size_t i = 0; i < k.size(); ++i) m.emplace(k[i], static_cast<int>(i));
    return m;
  }();
  auto it = idx.find(key);
  return it == idx.end() ? -1 : it->second;
}

// ---------------------------------------------------------------------------
// Polynomial algebra over interned atoms

namespace {

[[noreturn]] void parse_fail(const std::string& what) {
  throw KcgError(KCG_E_PARSE, what);
}

bool parse_int(const std::string& s, i128& out) {
  size_t i = 0;
  bool neg = false;
  if (i < s.size() && (s[i] == '-' || s[i] == '+')) {
    neg = s[i] == '-';
    ++i;
  }
  if (i >= s.size()) return false;
  i128 v = 0;
  for (; i < s.size(); ++i) {
    if (!std::isdigit(static_cast<unsigned char>(s[i]))) return false;
    v = checked_add(checked_mul(v, 10), s[i] - '0');
  }
  out = neg ? -v : v;
  return true;
}

bool parse_rat(const std::string& s, Q& out) {
  const size_t slash = s.find('/');
  i128 n, d = 1;
  if (slash == std::string::npos) {
    if (!parse_int(s, n)) return false;
  } else {
    if (!parse_int(s.substr(0, slash), n) || !parse_int(s.substr(slash + 1), d))
      return false;
    if (d <= 0) return false;
  }
  out = Q(n, d);
  return true;
}

Poly poly_const(const Q& c) {
  Poly p;
  if (!c.is_zero()) p.emplace(Mono{}, c);
  return p;
}

void poly_add_term(Poly& p, const Mono& m, const Q& c) {
  if (c.is_zero()) return;
  auto it = p.find(m);
  if (it == p.end()) {
    p.emplace(m, c);
  } else {
    it->second = it->second + c;
    if (it->second.is_zero()) p.erase(it);
  }
}

Poly poly_add(const Poly& a, const Poly& b, const Q& scale_b = Q(1)) {
  Poly r = a;
  for (const auto& [m, c] : b) poly_add_term(r, m, c * scale_b);
  return r;
}

Mono mono_mul(const Mono& a, const Mono& b) {
  Mono r;
  size_t i = 0, j = 0;
  while (i < a.f.size() || j < b.f.size()) {
    if (j >= b.f.size() || (i < a.f.size() && a.f[i].first < b.f[j].first)) {
      r.f.push_back(a.f[i++]);
    } else if (i >= a.f.size() || b.f[j].first < a.f[i].first) {
      r.f.push_back(b.f[j++]);
    } else {
      r.f.push_back({a.f[i].first, a.f[i].second + b.f[j].second});
      ++i;
      ++j;
    }
  }
  return r;
}

Poly poly_mul(const Poly& a, const Poly& b) {
  Poly r;
  for (const auto& [ma, ca] : a)
    for (const auto& [mb, cb] : b) poly_add_term(r, mono_mul(ma, mb), ca * cb);
  return r;
}

struct Builder {
  Symbolic s;
  std::map<std::string, int> atom_ids;

  int intern_atom(AtomDef a) {
    auto it = atom_ids.find(a.key);
    if (it != atom_ids.end()) return it->second;
    const int id = static_cast<int>(s.atoms.size());
    atom_ids.emplace(a.key, id);
    s.atoms.push_back(std::move(a));
    return id;
  }

  int add_poly(Poly p) {
    s.polys.push_back(std::move(p));
    return static_cast<int>(s.polys.size()) - 1;
  }

  Poly atom_poly(int id) {
    Poly p;
    p.emplace(Mono{{{id, 1}}}, Q(1));
    return p;
  }

  Poly var(const std::string& name) {
    auto it = std::find(s.params.begin(), s.params.end(), name);
    if (it == s.params.end()) parse_fail("unbound variable '" + name + "'");
    AtomDef a;
    a.kind = AtomKind::var;
    a.param = static_cast<int>(it - s.params.begin());
    a.key = name;
    return atom_poly(intern_atom(std::move(a)));
  }

  Poly floordiv(Poly num, i128 den, const std::string& key) {
    if (den <= 0) parse_fail("floordiv requires a positive denominator");
    AtomDef a;
    a.kind = AtomKind::floordiv;
    a.num = add_poly(std::move(num));
    a.den = den;
    a.key = key;
    return atom_poly(intern_atom(std::move(a)));
  }

  Poly minmax(AtomKind k, std::vector<Poly> args, const std::string& key) {
    if (args.size() < 2) parse_fail("min/max needs at least two arguments");
    AtomDef a;
    a.kind = k;
    for (auto& p : args) a.args.push_back(add_poly(std::move(p)));
    a.key = key;
    return atom_poly(intern_atom(std::move(a)));
  }

  // ---- CountExpr::str() prefix syntax ----
  struct Node {
    bool list = false;
    std::string tok;
    std::vector<Node> kids;
    size_t begin = 0, end = 0;  // source span
  };

  static Node parse_sexpr(const std::string& t, size_t& i) {
    while (i < t.size() && std::isspace(static_cast<unsigned char>(t[i]))) ++i;
    if (i >= t.size()) parse_fail("unexpected end of expression");
    Node n;
    n.begin = i;
    if (t[i] == '(') {
      n.list = true;
      ++i;
      while (true) {
        while (i < t.size() && std::isspace(static_cast<unsigned char>(t[i]))) ++i;
        if (i >= t.size()) parse_fail("unbalanced '('");
        if (t[i] == ')') {
          ++i;
          break;
        }
        n.kids.push_back(parse_sexpr(t, i));
      }
      if (n.kids.empty() || n.kids[0].list) parse_fail("bad list head");
    } else if (t[i] == ')') {
      parse_fail("unexpected ')'");
    } else {
      const size_t b = i;
      while (i < t.size() && !std::isspace(static_cast<unsigned char>(t[i])) &&
             t[i] != '(' && t[i] != ')')
        ++i;
      n.tok = t.substr(b, i - b);
    }
    n.end = i;
    return n;
  }

  Poly eval_node(const Node& n, const std::string& src) {
    if (!n.list) {
      Q c;
      if (parse_rat(n.tok, c)) return poly_const(c);
      return var(n.tok);
    }
    const std::string& head = n.kids[0].tok;
    const size_t nk = n.kids.size();
    if (head == "+") {
      Poly r;
      for (size_t i = 1; i < nk; ++i) r = poly_add(r, eval_node(n.kids[i], src));
      return r;
    }
    if (head == "*") {
      Poly r = poly_const(Q(1));
      for (size_t i = 1; i < nk; ++i) r = poly_mul(r, eval_node(n.kids[i], src));
      return r;
    }
    if (head == "^") {
      if (nk != 3 || n.kids[2].list) parse_fail("bad power");
      i128 e;
      if (!parse_int(n.kids[2].tok, e) || e < 0 || e > 64) parse_fail("bad exponent");
      const Poly base = eval_node(n.kids[1], src);
      Poly r = poly_const(Q(1));
      for (i128 i = 0; i < e; ++i) r = poly_mul(r, base);
      return r;
    }
    const std::string key = src.substr(n.begin, n.end - n.begin);
    if (head == "floordiv") {
      if (nk != 3 || n.kids[2].list) parse_fail("bad floordiv");
      i128 den;
      if (!parse_int(n.kids[2].tok, den)) parse_fail("bad floordiv denominator");
      return floordiv(eval_node(n.kids[1], src), den, key);
    }
    if (head == "min" || head == "max") {
      std::vector<Poly> args;
      for (size_t i = 1; i < nk; ++i) args.push_back(eval_node(n.kids[i], src));
      return minmax(head == "min" ? AtomKind::min : AtomKind::max, std::move(args), key);
    }
    parse_fail("unknown operator '" + head + "'");
  }

  Poly count_expr(const std::string& text) {
    size_t i = 0;
    Node n = parse_sexpr(text, i);
    while (i < text.size() && std::isspace(static_cast<unsigned char>(text[i]))) ++i;
    if (i != text.size()) parse_fail("trailing text after expression: " + text);
    return eval_node(n, text);
  }

  // ---- LinExpr::str() infix syntax ----
  struct Lex {
    const std::string& t;
    size_t i = 0;
    explicit Lex(const std::string& s) : t(s) {}
    void ws() {
      while (i < t.size() && std::isspace(static_cast<unsigned char>(t[i]))) ++i;
    }
    bool eat(const char* s) {
      ws();
      const size_t n = std::char_traits<char>::length(s);
      if (t.compare(i, n, s) == 0) {
        i += n;
        return true;
      }
      return false;
    }
    bool peek_digit() {
      ws();
      return i < t.size() && std::isdigit(static_cast<unsigned char>(t[i]));
    }
    i128 integer() {
      ws();
      const size_t b = i;
      while (i < t.size() && std::isdigit(static_cast<unsigned char>(t[i]))) ++i;
      i128 v;
      if (b == i || !parse_int(t.substr(b, i - b), v)) parse_fail("expected integer in '" + t + "'");
      return v;
    }
    std::string ident() {
      ws();
      const size_t b = i;
      while (i < t.size() && (std::isalnum(static_cast<unsigned char>(t[i])) || t[i] == '_')) ++i;
      if (b == i) parse_fail("expected identifier in '" + t + "'");
      return t.substr(b, i - b);
    }
    bool done() {
      ws();
      return i >= t.size();
    }
  };

  Poly lin_factor(Lex& lx) {
    if (lx.eat("(")) {
      const size_t b = lx.i;
      Poly inner = lin_expr(lx);
      const size_t e = lx.i;
      if (!lx.eat(")")) parse_fail("expected ')' in '" + lx.t + "'");
      if (!lx.eat("//")) parse_fail("expected '//' in '" + lx.t + "'");
      const i128 den = lx.integer();
      std::string body = lx.t.substr(b, e - b);
      while (!body.empty() && std::isspace(static_cast<unsigned char>(body.back()))) body.pop_back();
      return floordiv(std::move(inner), den, "(lin-floordiv (" + body + ") " + i128_str(den) + ")");
    }
    return var(lx.ident());
  }

  Poly lin_term(Lex& lx) {
    if (lx.peek_digit()) {
      i128 n = lx.integer(), d = 1;
      const size_t save = lx.i;
      if (!lx.eat("//") && lx.eat("/")) {
        d = lx.integer();
      } else {
        lx.i = save;
      }
      const Q c(n, d);
      if (lx.eat("*")) return poly_mul(poly_const(c), lin_factor(lx));
      return poly_const(c);
    }
    return lin_factor(lx);
  }

  Poly lin_expr(Lex& lx) {
    Q sign(1);
    if (lx.eat("-")) sign = Q(-1);
    Poly r = poly_mul(poly_const(sign), lin_term(lx));
    while (true) {
      if (lx.eat("+")) {
        r = poly_add(r, lin_term(lx));
      } else {
        const size_t save = lx.i;
        lx.ws();
        if (lx.i < lx.t.size() && lx.t[lx.i] == '-') {
          ++lx.i;
          r = poly_add(r, lin_term(lx), Q(-1));
        } else {
          lx.i = save;
          break;
        }
      }
    }
    return r;
  }

  Poly lin(const std::string& text) {
    Lex lx(text);
    Poly p = lin_expr(lx);
    if (!lx.done()) parse_fail("trailing text in affine expression '" + text + "'");
    return p;
  }

  void constraint(const std::string& text) {
    Constraint c;
    c.text = text;
    const size_t pct = text.find(" % ");
    if (pct != std::string::npos) {
      const size_t eq = text.find(" == ", pct);
      if (eq == std::string::npos) parse_fail("bad divisibility constraint '" + text + "'");
      c.divisibility = true;
      c.poly = add_poly(lin(text.substr(0, pct)));
      if (!parse_int(text.substr(pct + 3, eq - pct - 3), c.mod) || c.mod <= 0 ||
          !parse_int(text.substr(eq + 4), c.rem))
        parse_fail("bad divisibility constraint '" + text + "'");
    } else {
      static const std::pair<const char*, CmpOp> ops[] = {
          {" <= ", CmpOp::le}, {" >= ", CmpOp::ge}, {" == ", CmpOp::eq},
          {" < ", CmpOp::lt},  {" > ", CmpOp::gt}};
      size_t at = std::string::npos, len = 0;
      for (const auto& [s, op] : ops) {
        const size_t p = text.find(s);
        if (p != std::string::npos) {
          at = p;
          len = std::char_traits<char>::length(s);
          c.op = op;
          break;
        }
      }
      if (at == std::string::npos) parse_fail("no comparison in constraint '" + text + "'");
      c.poly = add_poly(poly_add(lin(text.substr(0, at)), lin(text.substr(at + len)), Q(-1)));
    }
    s.cons.push_back(std::move(c));
  }
};

std::string trim(const std::string& s) {
  size_t b = 0, e = s.size();
  while (b < e && std::isspace(static_cast<unsigned char>(s[b]))) ++b;
  while (e > b && std::isspace(static_cast<unsigned char>(s[e - 1]))) --e;
  return s.substr(b, e - b);
}

}  // namespace

Symbolic parse_program_text(const std::string& text) {
  Builder b;
  std::istringstream in(text);
  std::string line;
  bool header = false, ended = false;
  std::set<int> seen;
  int last_schema = -1;
  bool sorted = true;
  std::vector<std::pair<int, std::string>> props;
  while (std::getline(in, line)) {
    line = trim(line);
    if (line.empty() || line[0] == '#') continue;
    if (!header) {
      if (line != "kernelcost-program v1") parse_fail("missing 'kernelcost-program v1' header");
      header = true;
      continue;
    }
    if (ended) parse_fail("text after 'end'");
    const size_t sp = line.find(' ');
    const std::string kw = line.substr(0, sp);
    const std::string rest = sp == std::string::npos ? "" : trim(line.substr(sp + 1));
    if (kw == "kernel") {
      b.s.kernel = rest;
    } else if (kw == "param") {
      if (rest.empty()) parse_fail("empty param name");
      if (std::find(b.s.params.begin(), b.s.params.end(), rest) != b.s.params.end())
        parse_fail("duplicate param '" + rest + "'");
      b.s.params.push_back(rest);
    } else if (kw == "assume") {
      b.constraint(rest);
    } else if (kw == "prop") {
      const size_t sp2 = rest.find(' ');
      if (sp2 == std::string::npos) parse_fail("prop line needs key and expression");
      const std::string key = rest.substr(0, sp2);
      const int idx = schema_index(key);
      if (idx < 0) throw KcgError(KCG_E_SCHEMA_MISMATCH, "unknown property key '" + key + "'");
      if (!seen.insert(idx).second) parse_fail("duplicate property '" + key + "'");
      if (idx < last_schema) sorted = false;
      last_schema = idx;
      props.emplace_back(idx, trim(rest.substr(sp2 + 1)));
    } else if (kw == "end") {
      ended = true;
    } else {
      parse_fail("unknown line '" + line + "'");
    }
  }
  if (!header) parse_fail("empty program");
  if (!ended) parse_fail("missing 'end'");
  (void)sorted;
  std::sort(props.begin(), props.end());
  for (const auto& [idx, expr] : props) {
    Poly p = b.count_expr(expr);
    if (p.empty()) continue;  // identically zero entries are omitted
    b.s.props.emplace_back(idx, b.add_poly(std::move(p)));
  }
  return std::move(b.s);
}

// ---------------------------------------------------------------------------
// Enumeration program text (oracle/kcref_program.hpp enum_text)

namespace {

std::vector<std::string> split_bar(const std::string& s) {
  std::vector<std::string> out;
  size_t b = 0;
  while (true) {
    const size_t e = s.find(" | ", b);
    out.push_back(trim(s.substr(b, e == std::string::npos ? std::string::npos : e - b)));
    if (e == std::string::npos) break;
    b = e + 3;
  }
  return out;
}

}  // namespace

EnumSymbolic parse_enum_text(const std::string& text) {
  std::vector<std::string> lines;
  {
    std::istringstream in(text);
    std::string line;
    while (std::getline(in, line)) {
      line = trim(line);
      if (!line.empty() && line[0] != '#') lines.push_back(line);
    }
  }
  if (lines.empty() || lines[0] != "kernelcost-enum v1") parse_fail("missing 'kernelcost-enum v1' header");
  auto kw_rest = [](const std::string& l, std::string& rest) {
    const size_t sp = l.find(' ');
    rest = sp == std::string::npos ? "" : trim(l.substr(sp + 1));
    return l.substr(0, sp);
  };
  EnumSymbolic E;
  Builder b;
  // pass 1: parameters, then every domain-variable name as a further variable
  std::string rest;
  for (const auto& l : lines) {
    const std::string kw = kw_rest(l, rest);
    if (kw == "param") {
      if (rest.empty() || std::find(b.s.params.begin(), b.s.params.end(), rest) != b.s.params.end())
        parse_fail("bad or duplicate param '" + rest + "'");
      b.s.params.push_back(rest);
    }
  }
  E.n_params = static_cast<int>(b.s.params.size());
  for (const auto& l : lines) {
    const std::string kw = kw_rest(l, rest);
    if (kw != "var") continue;
    const std::string name = rest.substr(0, rest.find(' '));
    if (std::find(b.s.params.begin(), b.s.params.end(), name) == b.s.params.end()) b.s.params.push_back(name);
  }
  std::map<std::string, int> array_ids;
  EnumStmt* cur = nullptr;
  bool ended = false;
  for (size_t li = 1; li < lines.size(); ++li) {
    const std::string& l = lines[li];
    const std::string kw = kw_rest(l, rest);
    if (ended) parse_fail("text after 'end'");
    if (kw == "kernel") {
      b.s.kernel = rest;
    } else if (kw == "param") {
    } else if (kw == "assume") {
      b.constraint(rest);
      E.assumes.push_back(static_cast<int>(b.s.cons.size()) - 1);
    } else if (kw == "array") {
      std::istringstream is(rest);
      EnumArray a;
      std::string space;
      if (!(is >> a.name >> space >> a.bits >> a.nd >> a.fast) || (space != "global" && space != "local") ||
          a.nd < 1 || a.fast < 0 || a.fast >= a.nd)
        parse_fail("bad array line '" + l + "'");
      a.global = space == "global";
      array_ids[a.name] = static_cast<int>(E.arrays.size());
      E.arrays.push_back(a);
    } else if (kw == "group") {
      E.groups.push_back(b.add_poly(b.lin(rest)));
    } else if (kw == "stmt") {
      if (cur) parse_fail("nested 'stmt'");
      if (rest != "assign" && rest != "barrier") parse_fail("bad stmt kind '" + rest + "'");
      E.stmts.emplace_back();
      cur = &E.stmts.back();
      cur->barrier = rest == "barrier";
    } else if (kw == "endstmt") {
      if (!cur) parse_fail("'endstmt' outside a statement");
      cur = nullptr;
    } else if (kw == "end") {
      if (cur) parse_fail("'end' inside a statement");
      ended = true;
    } else {
      if (!cur) parse_fail("unknown line '" + l + "'");
      if (kw == "var") {
        const size_t sp = rest.find(' ');
        const auto parts = split_bar(sp == std::string::npos ? "" : rest.substr(sp + 1));
        if (parts.size() != 2) parse_fail("bad var line '" + l + "'");
        EnumVar v;
        v.name = rest.substr(0, sp);
        v.lo = b.add_poly(b.lin(parts[0]));
        v.hi = b.add_poly(b.lin(parts[1]));
        cur->vars.push_back(v);
      } else if (kw == "guard") {
        b.constraint(rest);
        cur->guards.push_back(static_cast<int>(b.s.cons.size()) - 1);
      } else if (kw == "access") {
        const auto parts = split_bar(rest);
        std::istringstream is(parts[0]);
        std::string arr, dir, stride;
        is >> arr >> dir;
        std::getline(is, stride);
        stride = trim(stride);
        auto it = array_ids.find(arr);
        if (it == array_ids.end() || (dir != "load" && dir != "store") || stride.empty())
          parse_fail("bad access line '" + l + "'");
        EnumAccess a;
        a.array = it->second;
        a.store = dir == "store";
        if (E.arrays[a.array].global) a.stride = b.add_poly(b.count_expr(stride));
        for (size_t k = 1; k < parts.size(); ++k) a.idx.push_back(b.add_poly(b.lin(parts[k])));
        if (static_cast<int>(a.idx.size()) != E.arrays[a.array].nd) parse_fail("access rank mismatch in '" + l + "'");
        cur->acc.push_back(std::move(a));
      } else if (kw == "op") {
        std::istringstream is(rest);
        std::string key, cnt;
        is >> key >> cnt;
        const int idx = schema_index(key);
        i128 v;
        if (idx < 0 || !parse_int(cnt, v)) parse_fail("bad op line '" + l + "'");
        cur->ops.emplace_back(idx, v);
      } else {
        parse_fail("unknown line '" + l + "'");
      }
    }
  }
  if (!ended) parse_fail("missing 'end'");
  E.sym = std::move(b.s);
  return E;
}

// ---------------------------------------------------------------------------
// Congruence substitution
//
// A parameter with divisibility facts p % m_i == r_i (AssumeCtx::add_constraint
// distils the same facts, decide.cpp:33-45) satisfies p = M*q + R at every
// admissible binding, with (M, R) their CRT combination. Substituting that
// into every property polynomial is an exact identity on the admissible set
// and typically clears all denominators (9/8 l m n with l,m,n = 16 q_*
// becomes 4608 q_l q_m q_n), so the GPU evaluates the counts with no
// division at all. Constraints keep the original parameters; inadmissible
// points are rejected before any count is formed.

namespace {

bool ext_crt(i128 m1, i128 r1, i128 m2, i128 r2, i128& M, i128& R) {
  // x = r1 (m1), x = r2 (m2)
  i128 a = m1, b = m2, x0 = 1, x1 = 0;
  while (b) {
    const i128 q = a / b;
    i128 t = a - q * b; a = b; b = t;
    t = x0 - q * x1; x0 = x1; x1 = t;
  }
  const i128 g = a;  // m1 * x0 = g (mod m2)
  if ((r2 - r1) % g != 0) return false;
  const i128 m2g = m2 / g;
  i128 k = ((r2 - r1) / g) % m2g;
  k = (k * (x0 % m2g)) % m2g;
  if (k < 0) k += m2g;
  M = checked_mul(m1 / g, m2);
  R = ((r1 + checked_mul(m1, k)) % M + M) % M;
  return true;
}

Poly poly_subst_atom(const Poly& p, int atom, const Poly& repl) {
  Poly out;
  for (const auto& [m, c] : p) {
    Poly term = poly_const(c);
    Mono rest;
    int e_sub = 0;
    for (const auto& [a, e] : m.f) {
      if (a == atom)
        e_sub = e;
      else
        rest.f.push_back({a, e});
    }
    Poly restp;
    restp.emplace(rest, Q(1));
    term = poly_mul(term, restp);
    for (int k = 0; k < e_sub; ++k) term = poly_mul(term, repl);
    out = poly_add(out, term);
  }
  return out;
}

Symbolic substitute_congruences(const Symbolic& in) {
  Symbolic s = in;
  const int np = static_cast<int>(s.params.size());
  std::vector<i128> M(np, 1), R(np, 0);
  std::vector<bool> ok(np, true);
  std::vector<std::vector<size_t>> used(np);
  for (size_t ci = 0; ci < s.cons.size(); ++ci) {
    const Constraint& c = s.cons[ci];
    if (!c.divisibility) continue;
    const Poly& p = s.polys[c.poly];
    int var_atom = -1;
    i128 k = 0;
    bool shape = true;
    for (const auto& [m, q] : p) {
      if (!q.is_int()) { shape = false; break; }
      if (m.f.empty()) { k = q.n; continue; }
      if (m.f.size() != 1 || m.f[0].second != 1 || q.n != 1 ||
          s.atoms[m.f[0].first].kind != AtomKind::var || var_atom >= 0) {
        shape = false;
        break;
      }
      var_atom = m.f[0].first;
    }
    if (!shape || var_atom < 0) continue;
    const int par = s.atoms[var_atom].param;
    const i128 r = ((c.rem - k) % c.mod + c.mod) % c.mod;
    i128 nm, nr;
    if (!ext_crt(M[par], R[par], c.mod, r, nm, nr)) {
      ok[par] = false;  // never admissible; leave the checks to reject it
      continue;
    }
    M[par] = nm;
    R[par] = nr;
    used[par].push_back(ci);
  }
  for (int par = 0; par < np; ++par) {
    if (!ok[par] || M[par] <= 1) continue;
    int var_atom = -1;
    for (size_t a = 0; a < s.atoms.size(); ++a)
      if (s.atoms[a].kind == AtomKind::var && s.atoms[a].param == par) var_atom = static_cast<int>(a);
    if (var_atom < 0) continue;
    AtomDef q;
    q.kind = AtomKind::quot;
    q.param = par;
    q.qmod = M[par];
    q.qrem = R[par];
    q.key = "(quot " + s.params[par] + " " + i128_str(M[par]) + " " + i128_str(R[par]) + ")";
    const int qid = static_cast<int>(s.atoms.size());
    s.atoms.push_back(q);
    for (size_t ci : used[par]) s.cons[ci].absorbed = true;
    Poly repl;
    repl.emplace(Mono{{{qid, 1}}}, Q(M[par]));
    if (R[par] != 0) repl.emplace(Mono{}, Q(R[par]));
    std::vector<bool> is_cons(s.polys.size(), false);
    for (const Constraint& c : s.cons) is_cons[c.poly] = true;
    for (size_t i = 0; i < s.polys.size(); ++i)
      if (!is_cons[i]) s.polys[i] = poly_subst_atom(s.polys[i], var_atom, repl);
  }
  return s;
}

}  // namespace

// ---------------------------------------------------------------------------
// Lowering

Lowered lower(const Symbolic& s_in) {
  const Symbolic s = substitute_congruences(s_in);
  Lowered L;
  L.n_params = static_cast<int>(s.params.size());
  L.n_atoms = static_cast<int>(s.atoms.size());
  L.atom_den.assign(s.atoms.size(), 0);

  std::map<Mono, int> mono_ids;
  std::vector<Mono> monos;
  std::vector<int> expr_of_poly(s.polys.size(), -1);
  std::vector<int> atom_state(s.atoms.size(), 0);  // 0 new, 1 visiting, 2 done
  std::vector<int> mono_done;

  std::function<int(int)> visit_poly;
  std::function<void(int)> visit_atom;

  auto visit_mono = [&](const Mono& m) -> int {
    auto it = mono_ids.find(m);
    if (it != mono_ids.end()) return it->second;
    for (const auto& [a, e] : m.f) visit_atom(a);
    const int id = static_cast<int>(monos.size());
    monos.push_back(m);
    mono_ids.emplace(m, id);
    LOp op{OP_MONO, id, static_cast<int32_t>(L.factors.size()), 0, 0};
    for (const auto& [a, e] : m.f) L.factors.push_back({a, e});
    op.b = static_cast<int32_t>(L.factors.size());
    L.ops.push_back(op);
    return id;
  };

  visit_atom = [&](int a) {
    if (atom_state[a] == 2) return;
    if (atom_state[a] == 1) throw KcgError(KCG_E_PARSE, "cyclic atom");
    atom_state[a] = 1;
    const AtomDef& ad = s.atoms[a];
    switch (ad.kind) {
      case AtomKind::var:
        L.atom_den[a] = 1;
        L.ops.push_back({OP_VAR, a, ad.param, 0, 0});
        break;
      case AtomKind::quot:
        L.atom_den[a] = 1;
        L.quot_mod.push_back(ad.qmod);
        L.quot_rem.push_back(ad.qrem);
        L.ops.push_back({OP_QUOT, a, ad.param, 0, static_cast<int32_t>(L.quot_mod.size() - 1)});
        break;
      case AtomKind::floordiv: {
        const int e = visit_poly(ad.num);
        L.atom_den[a] = 1;
        const i128 den = checked_mul(L.exprs[e].D, ad.den);
        L.floordiv_den.push_back(den);
        L.ops.push_back({OP_FLOORDIV, a, e, 0,
                         static_cast<int32_t>(L.floordiv_den.size() - 1)});
        break;
      }
      case AtomKind::min:
      case AtomKind::max: {
        std::vector<int> es;
        i128 Dm = 1;
        for (int p : ad.args) {
          es.push_back(visit_poly(p));
          Dm = lcm128(Dm, L.exprs[es.back()].D);
        }
        L.atom_den[a] = Dm;
        LOp op{ad.kind == AtomKind::min ? OP_MIN : OP_MAX, a,
               static_cast<int32_t>(L.args.size()), 0, 0};
        for (int e : es) L.args.push_back({e, Dm / L.exprs[e].D});
        op.b = static_cast<int32_t>(L.args.size());
        L.ops.push_back(op);
        break;
      }
    }
    atom_state[a] = 2;
  };

  visit_poly = [&](int pid) -> int {
    if (expr_of_poly[pid] >= 0) return expr_of_poly[pid];
    const Poly& p = s.polys[pid];
    // effective coefficient of each term: c / prod(atom_den^e)
    std::vector<std::pair<Q, int>> eff;
    i128 D = 1;
    for (const auto& [m, c] : p) {
      const int mid = m.f.empty() ? -1 : visit_mono(m);
      i128 den = 1;
      for (const auto& [a, e] : m.f)
        for (int k = 0; k < e; ++k) den = checked_mul(den, L.atom_den[a]);
      const Q q = c * Q(1, den);
      eff.emplace_back(q, mid);
      D = lcm128(D, q.d);
    }
    LExpr ex;
    ex.D = D;
    ex.term_begin = static_cast<int32_t>(L.terms.size());
    for (const auto& [q, mid] : eff) L.terms.push_back({checked_mul(q.n, D / q.d), mid});
    ex.term_end = static_cast<int32_t>(L.terms.size());
    const int id = static_cast<int>(L.exprs.size());
    L.exprs.push_back(ex);
    L.ops.push_back({OP_EXPR, id, ex.term_begin, ex.term_end, 0});
    expr_of_poly[pid] = id;
    return id;
  };

  for (size_t a = 0; a < s.atoms.size(); ++a) {
    if (s.atoms[a].kind != AtomKind::quot) continue;
    visit_atom(static_cast<int>(a));
    L.cons.push_back({2, s.atoms[a].param, static_cast<int32_t>(a), s.atoms[a].qmod, s.atoms[a].qrem});
  }
  for (const auto& c : s.cons) {
    if (c.absorbed) continue;
    const int e = visit_poly(c.poly);
    L.cons.push_back({c.divisibility ? 1 : 0, static_cast<int32_t>(c.op), e, c.mod, c.rem});
  }
  for (const auto& [schema, pid] : s.props) L.keys.push_back({schema, visit_poly(pid), 0, 0, 1, {}});
  // one-term original polynomials (s_in: the text as written, before the
  // congruence substitution rewrote parameters as quotients)
  for (size_t k = 0; k < L.keys.size() && k < s_in.props.size(); ++k) {
    const Poly& P = s_in.polys[s_in.props[k].second];
    if (P.size() != 1) continue;
    const Mono& m = P.begin()->first;
    const Q& q = P.begin()->second;
    if (q.n == 0) continue;
    LKey& key = L.keys[k];
    if (m.f.empty()) {
      if (!q.is_int()) continue;
      key.form = 1;
      key.coef = q.n;
      continue;
    }
    bool params_only = q.n > 0;
    std::vector<int> ex(L.n_params, 0);
    for (const auto& [a, e] : m.f) {
      if (s_in.atoms[a].kind != AtomKind::var) params_only = false;
      else ex[s_in.atoms[a].param] += e;
    }
    if (!params_only) continue;
    key.form = q.is_int() && (q.n & (q.n - 1)) == 0 ? 2 : 3;
    key.coef = q.n;
    key.coef_den = q.d;
    key.pexp = ex;
  }
  L.n_monos = static_cast<int>(monos.size());
  L.n_exprs = static_cast<int>(L.exprs.size());
  // atoms only reachable from nothing keep den 0; give them a sane value
  for (auto& d : L.atom_den)
    if (d == 0) d = 1;

  // safe uniform bounds (binary search on the magnitude analysis)
  auto search = [&](long double limit) -> int64_t {
    if (max_intermediate(L, 0) >= limit) return -1;
    int64_t lo = 0, hi = (int64_t(1) << 62);
    if (max_intermediate(L, static_cast<long double>(hi)) < limit) return hi;
    while (lo < hi) {
      const int64_t mid = lo + (hi - lo + 1) / 2;
      if (max_intermediate(L, static_cast<long double>(mid)) < limit)
        lo = mid;
      else
        hi = mid - 1;
    }
    return lo;
  };
  L.b64 = search(std::ldexp(1.0L, 62));
  L.b128 = search(std::ldexp(1.0L, 125));
  if (L.b64 >= 0) max_intermediate(L, static_cast<long double>(L.b64), &L.mono_bound64);
  if (!s_in.props.empty()) {
    Symbolic only = s_in;
    only.props.clear();
    L.admit = std::make_shared<Lowered>(lower(only));
  }
  return L;
}

long double max_intermediate(const Lowered& L, long double B,
                             std::vector<long double>* mono_bounds) {
  auto absq = [](i128 v) -> long double {
    return static_cast<long double>(v < 0 ? -v : v);
  };
  std::vector<long double> atom(L.n_atoms, 0), mono(L.n_monos, 0), expr(L.n_exprs, 0);
  long double worst = 0;
  auto see = [&](long double v) {
    if (v > worst) worst = v;
  };
  for (const LOp& op : L.ops) {
    switch (op.code) {
      case OP_VAR:
        atom[op.dst] = B;
        break;
      case OP_MONO: {
        long double m = 1;
        for (int i = op.a; i < op.b; ++i)
          for (int k = 0; k < L.factors[i].second; ++k) {
            m *= std::max<long double>(1, atom[L.factors[i].first]);
            see(m);
          }
        mono[op.dst] = m;
        break;
      }
      case OP_EXPR: {
        long double sum = 0;
        for (int i = op.a; i < op.b; ++i) {
          const LTerm& t = L.terms[i];
          const long double v = absq(t.coef) * (t.mono < 0 ? 1 : mono[t.mono]);
          see(v);
          sum += v;
          see(sum);
        }
        see(absq(L.exprs[op.dst].D));
        expr[op.dst] = sum;
        break;
      }
      case OP_QUOT:
        atom[op.dst] = (B + absq(L.quot_rem[op.c])) / absq(L.quot_mod[op.c]) + 1;
        see(B + absq(L.quot_rem[op.c]));
        break;
      case OP_FLOORDIV:
        atom[op.dst] = expr[op.a] / absq(L.floordiv_den[op.c]) + 1;
        see(absq(L.floordiv_den[op.c]));
        break;
      case OP_MIN:
      case OP_MAX: {
        long double m = 0;
        for (int i = op.a; i < op.b; ++i) {
          const long double v = expr[L.args[i].expr] * absq(L.args[i].scale);
          see(v);
          m = std::max(m, v);
        }
        atom[op.dst] = m;
        break;
      }
    }
  }
  for (const LCons& c : L.cons) see(2 * absq(c.mod) + absq(c.rem));
  if (mono_bounds) *mono_bounds = mono;
  return worst;
}

}  // namespace kcg
