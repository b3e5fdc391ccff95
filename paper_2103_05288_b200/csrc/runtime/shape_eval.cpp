// Host shape program interpreter (EvalShape; reference executor.cpp:303-341).  Shape
// computation stays on the host by design (paper: shapes on CPU, kernels on device).
#include "../capi_common.hpp"
#include "shape_eval.hpp"

namespace disc::rt {

void eval_shape_range(const CompiledPlan& plan, int from, int to,
                      const std::vector<const std::vector<int64_t>*>& input_dims, std::vector<int64_t>& regs) {
  const auto& prog = plan.shape_program.instrs;
  for (int k = from; k < to; ++k) {
    const ShapeInstr& si = prog[k];
    switch (si.kind) {
      case ShapeInstrKind::kReadInputDim:
        regs[si.dest] = (*input_dims[si.input])[si.axis];
        break;
      case ShapeInstrKind::kReadScalar:
        regs[si.dest] = plan.literals.at(si.tensor).at(si.index);
        break;
      case ShapeInstrKind::kLoadConst:
        regs[si.dest] = si.value;
        break;
      case ShapeInstrKind::kBinOp: {
        const int64_t a = regs[si.lhs], b = regs[si.rhs];
        int64_t r = 0;
        switch (si.op) {
          case ShapeBinOp::kAdd: r = a + b; break;
          case ShapeBinOp::kSub: r = a - b; break;
          case ShapeBinOp::kMul: r = a * b; break;
          case ShapeBinOp::kDivFloor:
            if (b == 0) throw RuntimeError("shape computation divided by zero");
            r = a / b;
            break;
          case ShapeBinOp::kCeilDiv:
            if (b <= 0) throw RuntimeError("shape ceil_div by non-positive stride");
            r = (a + b - 1) / b;
            break;
          case ShapeBinOp::kMax: r = a > b ? a : b; break;
        }
        regs[si.dest] = r;
        break;
      }
      case ShapeInstrKind::kBindDim:
        break;  // the register already holds the symbol's value
    }
  }
}

}  // namespace disc::rt

namespace disc_capi {
std::vector<int64_t> eval_shape_program(const disc::CompiledPlan& plan,
                                        const std::vector<std::vector<int64_t>>& input_dims) {
  if (input_dims.size() < plan.inputs.size()) throw disc::RuntimeError("missing input dims");
  std::vector<int64_t> regs(plan.shape_program.num_regs, 0);
  std::vector<const std::vector<int64_t>*> ptrs;
  for (const auto& d : input_dims) ptrs.push_back(&d);
  for (size_t i = 0; i < plan.inputs.size(); ++i)
    if (input_dims[i].size() != plan.inputs[i].dims.size())
      throw disc::RuntimeError("input " + plan.inputs[i].id + " rank mismatch");
  disc::rt::eval_shape_range(plan, 0, static_cast<int>(plan.shape_program.instrs.size()), ptrs, regs);
  return regs;
}
}  // namespace disc_capi
