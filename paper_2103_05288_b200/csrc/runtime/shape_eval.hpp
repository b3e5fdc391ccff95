#pragma once

#include <vector>

#include "../host/compiler.hpp"

namespace disc::rt {

// Evaluates shape instructions [from, to) into `regs`; input_dims[i] are graph input i's dims.
void eval_shape_range(const CompiledPlan& plan, int from, int to,
                      const std::vector<const std::vector<int64_t>*>& input_dims, std::vector<int64_t>& regs);

inline int64_t resolve(const ScalarRef& r, const std::vector<int64_t>& regs) {
  if (r.is_const) return r.value;
  if (r.reg < 0 || r.reg >= static_cast<int>(regs.size())) throw InternalError("shape register out of range");
  return regs[r.reg];
}

inline std::vector<int64_t> resolve_all(const std::vector<ScalarRef>& refs, const std::vector<int64_t>& regs) {
  std::vector<int64_t> v;
  v.reserve(refs.size());
  for (const auto& r : refs) v.push_back(resolve(r, regs));
  return v;
}

}  // namespace disc::rt
