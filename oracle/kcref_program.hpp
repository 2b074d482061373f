// ORACLE TEST INFRASTRUCTURE (reference side of the boundary).
//
// `program_text` is the ~20-line function a kernelcost maintainer adds on the
// reference side to hand a symbolic PropertyVector to the GPU path: it prints
// the kernel's parameters, its `assume` constraints (LinCmp::str(),
// linexpr.cpp:146-155) and every nonzero schema entry as CountExpr::str()
// (countexpr.cpp:385-416). The GPU library's kcg_program_create() parses this
// text (include/kcg.h). INTEGRATION.md shows the same function.
#pragma once

#include <string>

#include "kernelcost/counting.hpp"
#include "kernelcost/footprint.hpp"
#include "kernelcost/ir.hpp"
#include "kernelcost/props.hpp"
#include "kernelcost/schema.hpp"
#include "kernelcost/typing.hpp"

namespace kcref {

inline std::string program_text(const kernelcost::KernelIR& k,
                                const kernelcost::PropertyVector& pv) {
  std::string s = "kernelcost-program v1\nkernel " + k.name + "\n";
  for (const auto& p : k.params) s += "param " + p.name + "\n";
  for (const auto& c : k.assumptions) s += "assume " + c.str() + "\n";
  const auto& keys = kernelcost::schema_keys();
  for (size_t i = 0; i < pv.entries.size(); ++i)
    if (!pv.entries[i].is_zero())
      s += "prop " + keys[i] + " " + pv.entries[i].str() + "\n";
  s += "end\n";
  return s;
}

// `enum_text` hands the GPU enumeration oracle (kcg_enumerate_points,
// include/kcg.h) what enumerate_points (enumerate.cpp:371-456) walks: for
// every assign/barrier statement in walk_stmts order its StmtDomain
// (stmt_domain, counting.hpp:33-34: vars with LinExpr bounds, guards as
// LinCmp), its global/local accesses in collect_accesses order with the
// signed lane stride (lane_stride_signed, footprint.hpp:58) and index
// LinExprs, and its rhs_op_counts (props.hpp:31); arrays with space, element
// bits and fastest layout axis; group-axis extents. Every expression is
// printed with the reference's own str() (linexpr.cpp:100-126,
// countexpr.cpp:385-416).
inline std::string enum_text(const kernelcost::KernelIR& k) {
  namespace kc = kernelcost;
  const kc::AssumeCtx actx = kc::build_assume_ctx(k);
  const kc::TypeMap tm = kc::infer_types(k);
  std::string s = "kernelcost-enum v1\nkernel " + k.name + "\n";
  for (const auto& p : k.params) s += "param " + p.name + "\n";
  for (const auto& c : k.assumptions) s += "assume " + c.str() + "\n";
  for (const auto& a : k.arrays)
    s += "array " + a.name + " " + (a.space == kc::Space::global ? "global" : "local") + " " +
         std::to_string(kc::dtype_bits(a.dtype)) + " " + std::to_string(a.shape.size()) + " " +
         std::to_string(kc::fastest_axis(a)) + "\n";
  for (const kc::AxisDecl* ax : k.group_axes()) s += "group " + ax->extent.str() + "\n";
  const std::vector<kc::AccessRef> accs = kc::collect_accesses(k);
  kc::walk_stmts(k, [&](const kc::Stmt& st, const std::vector<const kc::Stmt*>& chain) {
    if (st.kind != kc::Stmt::Kind::assign && st.kind != kc::Stmt::Kind::barrier) return;
    const kc::StmtDomain d = kc::stmt_domain(k, st, chain);
    s += std::string("stmt ") + (st.kind == kc::Stmt::Kind::assign ? "assign" : "barrier") + "\n";
    for (const auto& v : d.vars) s += "var " + v.name + " " + v.lower.str() + " | " + v.upper_excl.str() + "\n";
    for (const auto& g : d.guards) s += "guard " + g.str() + "\n";
    for (const auto& acc : accs) {
      if (acc.stmt != &st) continue;
      s += "access " + acc.array->name + (acc.is_store ? " store " : " load ") +
           (acc.array->space == kc::Space::global ? kc::lane_stride_signed(k, acc, actx).str()
                                                  : std::string("-"));
      for (const auto& idx : *acc.indices) s += " | " + idx.str();
      s += "\n";
    }
    if (st.kind == kc::Stmt::Kind::assign)
      for (const auto& [key, per_point] : kc::rhs_op_counts(*st.rhs, tm))
        s += "op " + key + " " + per_point.str() + "\n";
    s += "endstmt\n";
  });
  s += "end\n";
  return s;
}

}  // namespace kcref
