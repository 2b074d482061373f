// GPU enumeration oracle, host side: enumerate_points
// (proj/core/src/enumerate.cpp:371-456) at one binding.
//
//   1. admissibility (AssumeCtx::admits, decide.cpp:153-170): every raw
//      assume constraint, then params >= 0;
//   2. per assign / barrier statement (walk_stmts order): the domain is
//      compiled to integer rows at the binding like RowCompiler
//      (enumerate.cpp:111-164) and walked on the GPU (enum_kernels.cu),
//      which counts leaves and visited points and marks the cells of the
//      statement's global accesses;
//   3. the tally (enumerate.cpp:407-455) runs here in exact 128-bit
//      arithmetic with the reference's classification rule
//      (classify_ratio, classify.cpp:15-25) and key names (schema.cpp:62-69).
// The GPU replaces only the walk -- the part that is O(domain size).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "kcg_enum_dev.h"
#include "kcg_host.hpp"
#include "kcg_kernels.hpp"

#include "../../include/kcg.h"

namespace kcg {

namespace {

i128 floor_q(const Q& q) {  // floor(n / d), d > 0
  i128 f = q.n / q.d;
  if (q.n % q.d != 0 && q.n < 0) f -= 1;
  return f;
}

struct Evaluator {
  const Symbolic& s;
  const std::vector<Q>* vals;  // per variable, nullptr entries = unbound

  // exact value of poly at the bound variables; throws for unbound ones
  Q poly(int id) const {
    Q r(0);
    for (const auto& [m, c] : s.polys[id]) {
      Q t = c;
      for (const auto& [atom, e] : m.f) {
        const Q a = this->atom(atom);
        for (int k = 0; k < e; ++k) t = t * a;
      }
      r = r + t;
    }
    return r;
  }
  Q atom(int id) const {
    const AtomDef& a = s.atoms[id];
    switch (a.kind) {
      case AtomKind::var: {
        const Q& v = (*vals)[a.param];
        if (v.d == 0) throw KcgError(KCG_E_UNSUPPORTED, "expression needs domain variable '" + s.params[a.param] + "'");
        return v;
      }
      case AtomKind::floordiv: {  // floor(num / den), numeric.hpp:24-31
        const Q v = poly(a.num);
        return Q(floor_q(Q(v.n, checked_mul(v.d, a.den))));
      }
      case AtomKind::min:
      case AtomKind::max: {
        Q best = poly(a.args[0]);
        for (size_t i = 1; i < a.args.size(); ++i) {
          const Q v = poly(a.args[i]);
          const i128 sg = (v - best).n;
          if (a.kind == AtomKind::min ? sg < 0 : sg > 0) best = v;
        }
        return best;
      }
      default:
        throw KcgError(KCG_E_UNSUPPORTED, "unsupported atom in enumeration program");
    }
  }
  // variables (atom params) the poly references, recursively
  void vars(int id, std::vector<int>& out) const {
    for (const auto& [m, c] : s.polys[id])
      for (const auto& [atom, e] : m.f) atom_vars(atom, out);
  }
  void atom_vars(int id, std::vector<int>& out) const {
    const AtomDef& a = s.atoms[id];
    if (a.kind == AtomKind::var) out.push_back(a.param);
    if (a.kind == AtomKind::floordiv) vars(a.num, out);
    for (int g : a.args) vars(g, out);
  }
};

bool fits64(i128 v) { return v >= -(static_cast<i128>(1) << 62) && v <= (static_cast<i128>(1) << 62); }

// row c0 + sum c_s x_s (over den) of a linear poly: parameters and
// parameter-only floordiv atoms fold into c0 (RowCompiler::compile)
KeRow compile_row(const Evaluator& ev, int poly, const std::map<int, int>& slot, int n_params, int* depth,
                  bool integral, std::vector<KeFd>* fds = nullptr) {
  Q c0(0);
  std::vector<std::pair<int, Q>> tm;
  std::vector<std::pair<int, Q>> tf;  // (statement fd index, coefficient)
  int fd_depth = -1;
  for (const auto& [m, c] : ev.s.polys[poly]) {
    if (m.f.empty()) {
      c0 = c0 + c;
      continue;
    }
    if (m.f.size() != 1 || m.f[0].second != 1)
      throw KcgError(KCG_E_UNSUPPORTED, "non-linear term in a domain expression");
    const int atom = m.f[0].first;
    const AtomDef& a = ev.s.atoms[atom];
    if (a.kind == AtomKind::var && a.param >= n_params) {
      auto it = slot.find(a.param);
      if (it == slot.end()) throw KcgError(KCG_E_UNSUPPORTED, "variable outside its statement's domain");
      tm.emplace_back(it->second, c);
      continue;
    }
    std::vector<int> vs;
    ev.atom_vars(atom, vs);
    bool domain = false;
    for (int v : vs) domain = domain || v >= n_params;
    if (!domain) {
      c0 = c0 + c * ev.atom(atom);
      continue;
    }
    // floor division over domain variables (the reference's Walker case,
    // enumerate.cpp:31-90): one statement-level term floor(row / div)
    if (a.kind != AtomKind::floordiv || !fds)
      throw KcgError(KCG_E_UNSUPPORTED, "min/max or nested floordiv over a domain variable");
    int din = -1;
    KeFd fd;
    std::memset(&fd, 0, sizeof fd);
    fd.r = compile_row(ev, a.num, slot, n_params, &din, false, nullptr);
    const i128 div = checked_mul(fd.r.den, a.den);
    if (!fits64(div)) throw KcgError(KCG_E_UNSUPPORTED, "floordiv divisor exceeds 64 bits");
    fd.div = static_cast<int64_t>(div);
    int f = -1;
    for (size_t i = 0; i < fds->size(); ++i)
      if (std::memcmp(&(*fds)[i], &fd, sizeof fd) == 0) f = static_cast<int>(i);
    if (f < 0) {
      if (static_cast<int>(fds->size()) >= KE_MAXF)
        throw KcgError(KCG_E_UNSUPPORTED, "more than 4 floor divisions over domain variables in a statement");
      f = static_cast<int>(fds->size());
      fds->push_back(fd);
    }
    tf.emplace_back(f, c);
    fd_depth = std::max(fd_depth, din);
  }
  i128 L = c0.d;
  for (const auto& [s, c] : tm) L = lcm128(L, c.d);
  for (const auto& [f, c] : tf) L = lcm128(L, c.d);
  if (integral && L != 1) throw KcgError(KCG_E_UNSUPPORTED, "array index / divisibility operand is not integral");
  KeRow r;
  std::memset(&r, 0, sizeof r);
  const i128 n0 = checked_mul(c0.n, L / c0.d);
  if (!fits64(L) || !fits64(n0)) throw KcgError(KCG_E_UNSUPPORTED, "domain row exceeds 64 bits");
  r.den = static_cast<int64_t>(L);
  r.c0 = static_cast<int64_t>(n0);
  int d = -1;
  for (const auto& [s, c] : tm) {
    const i128 v = checked_add(static_cast<i128>(r.c[s]), checked_mul(c.n, L / c.d));
    if (!fits64(v)) throw KcgError(KCG_E_UNSUPPORTED, "domain row exceeds 64 bits");
    r.c[s] = static_cast<int64_t>(v);
    if (r.c[s] != 0) d = std::max(d, s);
  }
  for (const auto& [f, c] : tf) {
    const i128 v = checked_add(static_cast<i128>(r.cf[f]), checked_mul(c.n, L / c.d));
    if (!fits64(v)) throw KcgError(KCG_E_UNSUPPORTED, "domain row exceeds 64 bits");
    r.cf[f] = static_cast<int64_t>(v);
    if (r.cf[f] != 0) d = std::max(d, fd_depth);
  }
  if (depth) *depth = d;
  return r;
}

struct Interval {
  i128 lo, hi;  // inclusive; lo > hi = empty
};

i128 floor_div128(i128 a, i128 d) {  // d > 0
  i128 q = a / d;
  if (a % d != 0 && a < 0) q -= 1;
  return q;
}

// range of a row's raw value over variable intervals (floor-division terms
// over the range of their own rows)
Interval row_range(const KeRow& r, const std::vector<Interval>& iv, int nv, const std::vector<KeFd>* fds = nullptr) {
  i128 lo = r.c0, hi = r.c0;
  for (int s = 0; s < nv; ++s) {
    if (r.c[s] == 0) continue;
    const i128 a = checked_mul(r.c[s], iv[s].lo), b = checked_mul(r.c[s], iv[s].hi);
    lo = checked_add(lo, std::min(a, b));
    hi = checked_add(hi, std::max(a, b));
  }
  for (int f = 0; f < KE_MAXF; ++f) {
    if (r.cf[f] == 0) continue;
    if (!fds || f >= static_cast<int>(fds->size())) throw KcgError(KCG_E_INTERNAL, "floordiv term without definition");
    const KeFd& fd = (*fds)[f];
    const Interval in = row_range(fd.r, iv, nv);
    const i128 flo = floor_div128(in.lo, fd.div), fhi = floor_div128(in.hi, fd.div);
    const i128 a = checked_mul(r.cf[f], flo), b = checked_mul(r.cf[f], fhi);
    lo = checked_add(lo, std::min(a, b));
    hi = checked_add(hi, std::max(a, b));
  }
  return {lo, hi};
}

i128 ceil_div128(i128 a, i128 d) {  // d > 0
  i128 q = a / d;
  if (a % d != 0 && a > 0) q += 1;
  return q;
}

std::string classify_ratio(i128 s, i128 cells, i128 fill) {  // classify.cpp:15-25
  if (s == 0) return "uniform";
  if (s == 1) return "1/1";
  if (fill <= 0) throw KcgError(KCG_E_INVALID_ARGUMENT, "empty footprint in classification");
  i128 q = (checked_mul(cells, s) + fill - 1) / fill;
  q = std::max<i128>(1, std::min<i128>(4, q));
  return i128_str(q) + "/" + (s > 4 ? std::string(">4") : i128_str(s));
}

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw KcgError(KCG_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

}  // namespace

int enumerate_points(const EnumSymbolic& E, const int64_t* binding, uint64_t cap, i128* counts149,
                      uint64_t* points_out, void* stream_) {
  const cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const Symbolic& s = E.sym;
  const int P = E.n_params;
  std::vector<Q> vals(s.params.size(), Q());
  for (auto& v : vals) v.d = 0;  // unbound marker
  for (int j = 0; j < P; ++j) vals[j] = Q(binding[j]);
  const Evaluator ev{s, &vals};

  // 1. admissibility: raw constraints, then params >= 0
  for (int ci : E.assumes) {
    const Constraint& c = s.cons[ci];
    const Q v = ev.poly(c.poly);
    bool ok;
    if (c.divisibility) {
      if (!v.is_int()) throw KcgError(KCG_E_INVALID_ARGUMENT, "divisibility operand is not an integer");
      i128 m = v.n % c.mod;
      if (m < 0) m += c.mod;
      ok = m == c.rem;
    } else {
      const i128 sg = v.n;
      switch (c.op) {
        case CmpOp::lt: ok = sg < 0; break;
        case CmpOp::le: ok = sg <= 0; break;
        case CmpOp::gt: ok = sg > 0; break;
        case CmpOp::ge: ok = sg >= 0; break;
        default: ok = sg == 0;
      }
    }
    if (!ok) throw KcgError(KCG_E_ASSUMPTION_VIOLATED, "binding violates the kernel's assumptions");
  }
  for (int j = 0; j < P; ++j)
    if (binding[j] < 0) throw KcgError(KCG_E_ASSUMPTION_VIOLATED, "binding violates the kernel's assumptions");

  const int NS = static_cast<int>(E.stmts.size());
  // 2a. compile every statement at the binding; union of index boxes per array
  std::vector<KeStmt> hs(NS);
  std::vector<bool> empty_dom(NS, false);
  const int NA = static_cast<int>(E.arrays.size());
  std::vector<std::vector<Interval>> abox(NA);
  std::vector<std::vector<std::pair<int, std::vector<Interval>>>> acc_iv(NS);  // per global access: idx ranges
  for (int si = 0; si < NS; ++si) {
    const EnumStmt& st = E.stmts[si];
    KeStmt& k = hs[si];
    std::memset(&k, 0, sizeof k);
    const int nv = static_cast<int>(st.vars.size());
    if (nv > KE_MAXV) throw KcgError(KCG_E_UNSUPPORTED, "statement domain deeper than 12 variables");
    std::map<int, int> slot;
    std::vector<KeFd> fds;  // floor divisions over this statement's domain variables
    k.nv = nv;
    std::vector<Interval> iv(nv);
    bool box = true;
    k.nbox = 0;
    for (int l = 0; l < nv; ++l) {
      const int vid = static_cast<int>(std::find(s.params.begin(), s.params.end(), st.vars[l].name) - s.params.begin());
      int dl, dh;
      k.lo[l] = compile_row(ev, st.vars[l].lo, slot, P, &dl, false, &fds);
      k.hi[l] = compile_row(ev, st.vars[l].hi, slot, P, &dh, false, &fds);
      slot[vid] = l;
      const Interval rl = row_range(k.lo[l], iv, nv, &fds), rh = row_range(k.hi[l], iv, nv, &fds);
      const i128 lmin = ceil_div128(rl.lo, k.lo[l].den), hmax = ceil_div128(rh.hi, k.hi[l].den);
      iv[l] = {lmin, hmax - 1};
      if (box && dl < 0 && dh < 0) {
        const i128 lo = ceil_div128(k.lo[l].c0, k.lo[l].den), hi = ceil_div128(k.hi[l].c0, k.hi[l].den);
        k.box_lo[l] = static_cast<int64_t>(lo);
        k.box_ext[l] = static_cast<int64_t>(std::max<i128>(0, hi - lo));
        ++k.nbox;
      } else {
        box = false;
      }
      if (!fits64(iv[l].lo) || !fits64(iv[l].hi)) throw KcgError(KCG_E_UNSUPPORTED, "domain bound exceeds 64 bits");
    }
    // guards: depth of the deepest variable; parameter-only guards decide emptiness
    for (int ci : st.guards) {
      const Constraint& c = s.cons[ci];
      KeGuard g;
      std::memset(&g, 0, sizeof g);
      int depth;
      g.r = compile_row(ev, c.poly, slot, P, &depth, c.divisibility, &fds);
      g.depth = depth;
      g.divis = c.divisibility ? 1 : 0;
      g.op = static_cast<int>(c.op);
      g.mod = static_cast<int64_t>(c.mod);
      g.rem = static_cast<int64_t>(c.rem);
      if (depth < 0) {
        const i128 v = g.r.c0;
        bool pass;
        if (g.divis) {
          i128 m = v % c.mod;
          if (m < 0) m += c.mod;
          pass = m == c.rem;
        } else {
          pass = c.op == CmpOp::lt ? v < 0 : c.op == CmpOp::le ? v <= 0 : c.op == CmpOp::gt ? v > 0
                 : c.op == CmpOp::ge ? v >= 0 : v == 0;
        }
        if (!pass) empty_dom[si] = true;
        continue;
      }
      if (k.ng >= KE_MAXG) throw KcgError(KCG_E_UNSUPPORTED, "more than 8 guards in a statement");
      // magnitude: |raw| over the domain box must stay within 64 bits
      const Interval gr = row_range(g.r, iv, nv, &fds);
      if (!fits64(gr.lo) || !fits64(gr.hi)) throw KcgError(KCG_E_UNSUPPORTED, "guard value exceeds 64 bits");
      k.g[k.ng++] = g;
    }
    for (int l = 0; l < nv; ++l) {
      const Interval a = row_range(k.lo[l], iv, nv, &fds), b = row_range(k.hi[l], iv, nv, &fds);
      if (!fits64(a.lo) || !fits64(a.hi) || !fits64(b.lo) || !fits64(b.hi))
        throw KcgError(KCG_E_UNSUPPORTED, "domain bound exceeds 64 bits");
    }
    // box levels the threads enumerate: up to the first empty one
    k.nbe = k.nbox;
    k.inner = 1;
    unsigned long long total = 1;
    for (int l = 0; l < k.nbox; ++l) {
      if (k.box_ext[l] == 0) {
        k.nbe = l;
        k.inner = 0;
        break;
      }
      if (total > ~0ull / static_cast<unsigned long long>(k.box_ext[l]))
        throw KcgError(KCG_E_UNSUPPORTED, "domain box exceeds 2^64 points");
      total *= static_cast<unsigned long long>(k.box_ext[l]);
    }
    k.box_total = empty_dom[si] ? 0 : total;
    bool nonempty_iv = true;
    for (int l = 0; l < nv; ++l) nonempty_iv = nonempty_iv && iv[l].lo <= iv[l].hi;
    // global accesses: index rows and their ranges
    for (const EnumAccess& a : st.acc) {
      if (!E.arrays[a.array].global || st.barrier) continue;
      if (k.na >= KE_MAXA) throw KcgError(KCG_E_UNSUPPORTED, "more than 8 global accesses in a statement");
      KeAccess& A = k.a[k.na++];
      std::memset(&A, 0, sizeof A);
      if (static_cast<int>(a.idx.size()) > KE_MAXD) throw KcgError(KCG_E_UNSUPPORTED, "array rank above 4");
      std::vector<Interval> r;
      for (size_t d = 0; d < a.idx.size(); ++d) {
        A.idx[d] = compile_row(ev, a.idx[d], slot, P, nullptr, true, &fds);
        const Interval x = row_range(A.idx[d], iv, nv, &fds);
        if (!fits64(x.lo) || !fits64(x.hi)) throw KcgError(KCG_E_UNSUPPORTED, "array index exceeds 64 bits");
        r.push_back(x);
      }
      A.m.nd = static_cast<int>(a.idx.size());
      A.m.fast = E.arrays[a.array].fast;
      if (nonempty_iv && k.box_total > 0 && k.inner) {
        auto& bx = abox[a.array];
        if (bx.empty()) {
          bx = r;
        } else {
          for (size_t d = 0; d < r.size(); ++d) {
            bx[d].lo = std::min(bx[d].lo, r[d].lo);
            bx[d].hi = std::max(bx[d].hi, r[d].hi);
          }
        }
      }
      acc_iv[si].emplace_back(a.array, r);
    }
    k.nf = static_cast<int32_t>(fds.size());
    for (size_t f = 0; f < fds.size(); ++f) k.f[f] = fds[f];
  }

  // 2b. bitmaps per touched global array
  struct ArrBits {
    unsigned long long cells_w = 0, others_w = 0, fast_w = 0;
    unsigned long long *cells = nullptr, *others = nullptr, *fastp = nullptr;
    std::vector<int64_t> lo, ext;
  };
  std::vector<ArrBits> ab(NA);
  std::vector<DevBuf> bufs;
  bufs.reserve(4 * NA + 4);
  size_t free_b = 0, total_b = 0;
  cuda_ok(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
  size_t bitmap_bytes = 0;
  for (int ai = 0; ai < NA; ++ai) {
    if (abox[ai].empty()) continue;
    ArrBits& B = ab[ai];
    i128 cells = 1, others = 1, fast = 1;
    for (size_t d = 0; d < abox[ai].size(); ++d) {
      const i128 e = abox[ai][d].hi - abox[ai][d].lo + 1;
      B.lo.push_back(static_cast<int64_t>(abox[ai][d].lo));
      B.ext.push_back(static_cast<int64_t>(e));
      cells = checked_mul(cells, e);
      if (static_cast<int>(d) == E.arrays[ai].fast)
        fast = e;
      else
        others = checked_mul(others, e);
    }
    if (cells > (static_cast<i128>(1) << 46)) throw KcgError(KCG_E_UNSUPPORTED, "array footprint box too large for a bitmap");
    B.cells_w = static_cast<unsigned long long>((cells + 63) / 64);
    B.others_w = static_cast<unsigned long long>((others + 63) / 64);
    B.fast_w = static_cast<unsigned long long>((fast + 63) / 64);
    bitmap_bytes += 8 * (B.cells_w + B.others_w + B.fast_w);
  }
  if (bitmap_bytes > free_b / 2) throw KcgError(KCG_E_UNSUPPORTED, "footprint bitmaps exceed half of free device memory");
  for (int ai = 0; ai < NA; ++ai) {
    ArrBits& B = ab[ai];
    if (!B.cells_w) continue;
    for (auto [pp, w] : {std::pair<unsigned long long**, unsigned long long>{&B.cells, B.cells_w},
                         {&B.others, B.others_w}, {&B.fastp, B.fast_w}}) {
      bufs.emplace_back();
      cuda_ok(cudaMallocAsync(&bufs.back().p, 8 * w, stream), "cudaMallocAsync");
      cuda_ok(cudaMemsetAsync(bufs.back().p, 0, 8 * w, stream), "cudaMemsetAsync");
      *pp = static_cast<unsigned long long*>(bufs.back().p);
    }
  }
  // counters: per statement (leaves, visited), per array (pop, min, max) x 3
  const size_t nctr = 2 * NS + 9 * NA;
  std::vector<unsigned long long> hctr(nctr, 0);
  for (int ai = 0; ai < NA; ++ai)
    for (int q = 0; q < 3; ++q) hctr[2 * NS + 9 * ai + 3 * q + 1] = ~0ull;
  DevBuf dctr, dst;
  cuda_ok(cudaMallocAsync(&dctr.p, 8 * std::max<size_t>(nctr, 1), stream), "cudaMallocAsync");
  cuda_ok(cudaMemcpyAsync(dctr.p, hctr.data(), 8 * nctr, cudaMemcpyHostToDevice, stream), "cudaMemcpyAsync");
  auto* ctr = static_cast<unsigned long long*>(dctr.p);
  for (int si = 0; si < NS; ++si) {
    KeStmt& k = hs[si];
    k.out = ctr + 2 * si;
    int na = 0;
    for (const auto& [ai, r] : acc_iv[si]) {
      KeMark& M = k.a[na++].m;
      const ArrBits& B = ab[ai];
      for (int d = 0; d < M.nd; ++d) {
        M.lo[d] = B.cells_w ? B.lo[d] : 0;
        M.ext[d] = B.cells_w ? B.ext[d] : 1;
      }
      M.cells = B.cells;
      M.others = B.others;
      M.fastp = B.fastp;
    }
    if (!k.inner) k.na = 0;  // no leaves, nothing to mark
  }
  cuda_ok(cudaMallocAsync(&dst.p, sizeof(KeStmt) * std::max(NS, 1), stream), "cudaMallocAsync");
  cuda_ok(cudaMemcpyAsync(dst.p, hs.data(), sizeof(KeStmt) * NS, cudaMemcpyHostToDevice, stream), "cudaMemcpyAsync");
  int launches = 0;
  for (int si = 0; si < NS; ++si) {
    launch_enum_walk(static_cast<const KeStmt*>(dst.p) + si, hs[si].box_total, stream);
    launches += hs[si].box_total > 0;
  }
  for (int ai = 0; ai < NA; ++ai) {
    const ArrBits& B = ab[ai];
    if (!B.cells_w) continue;
    launches += 3;
    unsigned long long* o = ctr + 2 * NS + 9 * ai;
    launch_enum_bits(B.cells, B.cells_w, o, stream);
    launch_enum_bits(B.others, B.others_w, o + 3, stream);
    launch_enum_bits(B.fastp, B.fast_w, o + 6, stream);
  }
  cuda_ok(cudaMemcpyAsync(hctr.data(), dctr.p, 8 * nctr, cudaMemcpyDeviceToHost, stream), "cudaMemcpyAsync");
  cuda_ok(cudaStreamSynchronize(stream), "enumeration");
  for (auto& b : bufs) {
    cudaFreeAsync(b.p, stream);
    b.p = nullptr;
  }
  cudaFreeAsync(dctr.p, stream);
  dctr.p = nullptr;
  cudaFreeAsync(dst.p, stream);
  dst.p = nullptr;

  // 3. tally (enumerate.cpp:407-455)
  unsigned long long points = 0;
  for (int si = 0; si < NS; ++si) points += hctr[2 * si + 1];
  if (points_out) *points_out = points;
  if (cap && points > cap)
    throw KcgError(KCG_E_CAP_EXCEEDED, "enumeration exceeded cap of " + std::to_string(cap) + " points");
  std::vector<i128> out(schema_keys().size(), 0);
  auto add = [&](const std::string& key, i128 v) {
    const int i = schema_index(key);
    if (i < 0) throw KcgError(KCG_E_SCHEMA_MISMATCH, "key '" + key + "' not in schema v1");
    out[i] = checked_add(out[i], v);
  };
  std::map<std::pair<int, std::string>, std::pair<i128, i128>> ls;
  for (int si = 0; si < NS; ++si) {
    const EnumStmt& st = E.stmts[si];
    const i128 n = static_cast<i128>(hctr[2 * si]);
    if (n == 0) continue;
    for (const EnumAccess& a : st.acc) {
      const EnumArray& arr = E.arrays[a.array];
      if (!arr.global) {
        if (!a.store) add("mem.local.load", n);
        continue;
      }
      const unsigned long long* o = hctr.data() + 2 * NS + 9 * a.array;
      const i128 nf = static_cast<i128>(o[0]);
      const i128 fill = nf == 0 ? 0 : checked_mul(static_cast<i128>(o[8] - o[7] + 1), static_cast<i128>(o[3]));
      const Q sr = ev.poly(a.stride);
      if (!sr.is_int()) throw KcgError(KCG_E_INVALID_ARGUMENT, "lane stride does not evaluate to an integer");
      const i128 sv = sr.n < 0 ? -sr.n : sr.n;
      const std::string cls = classify_ratio(sv, nf, fill);
      add(std::string("mem.global.") + (a.store ? "store" : "load") + ".s" + std::to_string(arr.bits) + "." + cls, n);
      auto& pr = ls[{arr.bits, cls}];
      (a.store ? pr.second : pr.first) += n;
    }
  }
  for (const auto& [kc, pr] : ls) {
    const i128 m = std::min(pr.first, pr.second);
    if (m > 0) add("mem.minls.s" + std::to_string(kc.first) + "." + kc.second, m);
  }
  for (int si = 0; si < NS; ++si) {
    const EnumStmt& st = E.stmts[si];
    const i128 n = static_cast<i128>(hctr[2 * si]);
    if (st.barrier) {
      add("sync.barrier", n);
    } else {
      for (const auto& [key, per] : st.ops) out[key] = checked_add(out[key], checked_mul(per, n));
    }
  }
  i128 groups = 1;
  for (int g : E.groups) {
    const Q v = ev.poly(g);
    if (!v.is_int()) throw KcgError(KCG_E_INVALID_ARGUMENT, "group extent does not evaluate to an integer");
    groups = checked_mul(groups, v.n);
  }
  out[schema_index("launch.groups")] = groups;
  out[schema_index("launch.const")] = 1;
  std::copy(out.begin(), out.end(), counts149);
  return launches;
}

}  // namespace kcg
