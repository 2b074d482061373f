// Reference-side front-end extension: symbolic
// extraction for kernels the reference's extract_properties(k) rejects only
// because of footprint analysis -- fd_stencil and nbody. It is the
// reference's own pipeline (props.cpp:102-247, restated with the public API
// of counting.hpp / footprint.hpp / classify.hpp / decide.hpp) with two
// semantics-preserving rules, and it is what kcref_export prints into
// paper_1604_04997_b200/programs/{fd_stencil_g16x16,nbody_g256}.kcp:
//
//  1. Stride before footprint. The reference computes the array footprint
//     before classifying any access (props.cpp:211-212 array_stat), and the
//     footprint throws needs_binding when the per-axis images of the
//     accesses differ (footprint.cpp:421-430). classify_symbolic /
//     classify_ratio return "uniform" / "1/1" for a lane stride of 0 / 1
//     without looking at cells or fill (classify.cpp:15-17, 31-32), so for
//     such accesses the footprint is skipped. Exactly the classes the
//     reference's bound mode produces at every binding.
//  2. Contained-box union. When the accesses' per-axis images differ, but
//     one access's image box contains every other access's box (dense
//     step-1 axes, min/max containment proven by DecideCtx) and its axes
//     draw on disjoint variables, the union of the boxes IS that box: its
//     cells and stride fill are the footprint (nbody's pos: axis images
//     {0}, {1}, {2} and [0, 2] -> cells = fill = 3n at every n).
//  Anything else still throws needs_binding, as the reference does.
#pragma once

#include <map>
#include <string>
#include <vector>

#include "kernelcost/classify.hpp"
#include "kernelcost/counting.hpp"
#include "kernelcost/decide.hpp"
#include "kernelcost/error.hpp"
#include "kernelcost/footprint.hpp"
#include "kernelcost/ir.hpp"
#include "kernelcost/props.hpp"
#include "kernelcost/schema.hpp"
#include "kernelcost/typing.hpp"

namespace kcref {

namespace detail {

namespace kc = kernelcost;

// rule 2: the footprint of an array whose access boxes are all contained in
// one of them (throws needs_binding otherwise)
inline kc::Footprint contained_box_footprint(const kc::KernelIR& k, const kc::ArrayDecl& arr,
                                             const kc::AssumeCtx& actx) {
  std::vector<std::vector<kc::AxisImage>> boxes;
  for (const auto& acc : kc::collect_accesses(k)) {
    if (acc.array != &arr) continue;
    const kc::StmtDomain dom = kc::stmt_domain(k, *acc.stmt, acc.enclosing);
    std::vector<kc::AxisImage> axes;
    for (const auto& idx : *acc.indices) axes.push_back(kc::index_image(idx, dom, actx));
    boxes.push_back(std::move(axes));
  }
  if (boxes.empty()) throw kc::Error(kc::Errc::invalid_argument, "array '" + arr.name + "' has no accesses");
  const kc::DecideCtx dc(actx);
  auto contains = [&](const std::vector<kc::AxisImage>& big, const std::vector<kc::AxisImage>& small) {
    if (big.size() != small.size()) return false;
    for (size_t i = 0; i < big.size(); ++i) {
      if (big[i].step != 1) return false;  // a dense interval holds every value between its ends
      if (!dc.proves_nonneg(small[i].min - big[i].min)) return false;
      if (!dc.proves_nonneg(big[i].max - small[i].max)) return false;
    }
    return true;
  };
  for (const auto& cand : boxes) {
    bool all = true;
    for (const auto& b : boxes) all = all && contains(cand, b);
    if (!all) continue;
    std::map<std::string, int> seen;  // |box| = product of the axis cardinalities
    bool disjoint = true;
    for (const auto& ax : cand)
      for (const auto& v : ax.support) disjoint = disjoint && ++seen[v] == 1;
    if (!disjoint) continue;
    kc::Footprint fp;
    fp.array = &arr;
    fp.axes = cand;
    fp.cells = kc::CountExpr::from_int(1);
    for (const auto& ax : fp.axes) fp.cells = fp.cells * ax.card;
    return fp;
  }
  throw kc::Error(kc::Errc::needs_binding, "array '" + arr.name + "': no access box contains the others");
}

}  // namespace detail

// extract_properties(k) (props.hpp:37) with rules 1 and 2 above: equal to it
// wherever it succeeds, and symbolic for fd_stencil / nbody where it throws
inline kernelcost::PropertyVector extract_properties_grid(const kernelcost::KernelIR& k) {
  namespace kc = kernelcost;
  const kc::AssumeCtx actx = kc::build_assume_ctx(k);
  const kc::TypeMap tm = kc::infer_types(k);
  kc::PropertyVector out;
  std::map<const kc::Stmt*, kc::CountExpr> counts;
  auto stmt_count = [&](const kc::Stmt& s, const std::vector<const kc::Stmt*>& chain) {
    auto it = counts.find(&s);
    if (it != counts.end()) return it->second;
    const kc::CountExpr c = kc::count_points(kc::stmt_domain(k, s, chain), actx);
    counts.emplace(&s, c);
    return c;
  };
  kc::walk_stmts(k, [&](const kc::Stmt& s, const std::vector<const kc::Stmt*>& chain) {
    if (s.kind == kc::Stmt::Kind::assign) {
      const kc::CountExpr n = stmt_count(s, chain);
      for (const auto& [key, per_point] : kc::rhs_op_counts(*s.rhs, tm))
        out.at(key) = out.at(key) + n.scaled(kc::Rat(per_point));
    } else if (s.kind == kc::Stmt::Kind::barrier) {
      out.at("sync.barrier") = out.at("sync.barrier") + stmt_count(s, chain);
    }
  });
  struct ArrStat {
    kc::CountExpr cells, fill;
  };
  std::map<const kc::ArrayDecl*, ArrStat> stats;
  auto array_stat = [&](const kc::ArrayDecl* a) -> const ArrStat& {
    auto it = stats.find(a);
    if (it != stats.end()) return it->second;
    kc::Footprint f;
    try {
      f = kc::access_footprint(k, *a, actx);
    } catch (const kc::Error& err) {
      if (err.code() != kc::Errc::needs_binding && err.code() != kc::Errc::needs_fallback) throw;
      f = detail::contained_box_footprint(k, *a, actx);  // rule 2
    }
    return stats.emplace(a, ArrStat{f.cells, kc::fill_footprint(f)}).first->second;
  };
  const kc::DecideCtx dc(actx);
  std::map<std::pair<int, std::string>, std::pair<kc::CountExpr, kc::CountExpr>> ls;
  for (const auto& acc : kc::collect_accesses(k)) {
    const kc::CountExpr n = counts.at(acc.stmt);
    if (n.is_zero()) continue;
    if (acc.array->space == kc::Space::local) {
      if (!acc.is_store) out.at("mem.local.load") = out.at("mem.local.load") + n;
      continue;
    }
    const kc::CountExpr stride = kc::lane_stride(k, acc, actx);
    std::string cls;
    if (stride.is_zero())
      cls = "uniform";  // rule 1: classify.cpp:31
    else if (stride.is_constant() && stride.constant_value() == 1)
      cls = "1/1";      // rule 1: classify.cpp:32
    else {
      const ArrStat& st = array_stat(acc.array);
      cls = kc::classify_symbolic(stride, st.cells, st.fill, dc);
    }
    const int bits = kc::dtype_bits(acc.array->dtype);
    const std::string key = kc::global_key(acc.is_store, bits, cls);
    out.at(key) = out.at(key) + n;
    auto& pair = ls[{bits, cls}];
    if (acc.is_store)
      pair.second = pair.second + n;
    else
      pair.first = pair.first + n;
  }
  for (const auto& [kcls, pair] : ls) {
    if (pair.first.is_zero() || pair.second.is_zero()) continue;
    out.at(kc::minls_key(kcls.first, kcls.second)) = kc::make_min(pair.first, pair.second, dc);
  }
  kc::CountExpr groups = kc::CountExpr::from_int(1);
  for (const kc::AxisDecl* ax : k.group_axes()) groups = groups * kc::to_count(ax->extent, actx);
  out.at("launch.groups") = groups;
  out.at("launch.const") = kc::CountExpr::from_int(1);
  return out;
}

}  // namespace kcref
