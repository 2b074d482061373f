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

#include "kernelcost/ir.hpp"
#include "kernelcost/props.hpp"
#include "kernelcost/schema.hpp"

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

}  // namespace kcref
