// disc-b200 host IR: errors, symbolic shapes, the framework graph and the DHLO hub IR.
//
// Clean-room re-statement of the reference's public C++ surface so that code written
// against it keeps compiling: names follow /root/reference/proj/include/disc/
// {error,shape,framework,dhlo}.hpp; the layout and implementation here are our own.
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace disc {

// ---------------------------------------------------------------------------
// Errors (reference error.hpp:25-63). Classes map to CLI exit codes 2/3/4.
enum class ErrorClass { kUsage, kParse, kValidation, kCompile, kRuntime, kInternal };
const char* error_class_name(ErrorClass c);

class Error : public std::runtime_error {
 public:
  Error(ErrorClass c, const std::string& m) : std::runtime_error(m), cls_(c) {}
  ErrorClass error_class() const { return cls_; }

 private:
  ErrorClass cls_;
};
#define DISC_ERROR_KIND(Name, Cls) \
  struct Name : Error {            \
    explicit Name(const std::string& m) : Error(ErrorClass::Cls, m) {} \
  };
DISC_ERROR_KIND(ParseError, kParse)
DISC_ERROR_KIND(ValidationError, kValidation)
DISC_ERROR_KIND(CompileError, kCompile)
DISC_ERROR_KIND(RuntimeError, kRuntime)
DISC_ERROR_KIND(InternalError, kInternal)
#undef DISC_ERROR_KIND

// ---------------------------------------------------------------------------
// Shapes (reference shape.hpp:28-125).
enum class ElementType { kF32, kI64 };
inline const char* element_type_name(ElementType t) { return t == ElementType::kF32 ? "f32" : "i64"; }

// A dimension: a non-negative constant, or a symbol id (dense, per graph).
class SymbolicDim {
 public:
  SymbolicDim() = default;
  static SymbolicDim Const(int64_t v) {
    if (v < 0) throw InternalError("SymbolicDim: negative constant dim");
    SymbolicDim d;
    d.v_ = v;
    return d;
  }
  static SymbolicDim Sym(int id) {
    if (id < 0) throw InternalError("SymbolicDim: negative symbol id");
    SymbolicDim d;
    d.sym_ = id;
    return d;
  }
  bool is_const() const { return sym_ < 0; }
  bool is_sym() const { return sym_ >= 0; }
  int64_t size() const {
    if (is_sym()) throw InternalError("SymbolicDim: size() on symbolic dim");
    return v_;
  }
  int sym_id() const {
    if (is_const()) throw InternalError("SymbolicDim: sym_id() on constant dim");
    return sym_;
  }
  bool operator==(const SymbolicDim& o) const {
    return is_sym() ? o.sym_ == sym_ : (o.is_const() && o.v_ == v_);
  }
  bool operator!=(const SymbolicDim& o) const { return !(*this == o); }
  std::string str() const { return is_sym() ? "s" + std::to_string(sym_) : std::to_string(v_); }

 private:
  int64_t v_ = 0;
  int sym_ = -1;
};

struct ShapeVector {
  std::vector<SymbolicDim> dims;
  ShapeVector() = default;
  explicit ShapeVector(std::vector<SymbolicDim> d) : dims(std::move(d)) {}
  int rank() const { return static_cast<int>(dims.size()); }
  bool is_static() const {
    for (const auto& d : dims)
      if (d.is_sym()) return false;
    return true;
  }
  int64_t static_numel() const {
    int64_t n = 1;
    for (const auto& d : dims) n *= d.size();
    return n;
  }
  bool operator==(const ShapeVector& o) const { return dims == o.dims; }
  bool operator!=(const ShapeVector& o) const { return !(dims == o.dims); }
  std::string str() const;
  static ShapeVector all_const(const std::vector<int64_t>& v);
};

struct GraphValue {
  std::string id;
  ShapeVector shape;
  ElementType etype = ElementType::kF32;
};

// ---------------------------------------------------------------------------
// Framework-level graph (reference framework.hpp:28-92).
enum class FwOpKind {
  kAdd, kSub, kMul, kDiv, kExp, kTanh, kNeg, kMaximum, kReduceSum, kReduceMax,
  kTranspose, kReshape, kBroadcast, kSlice, kPad, kSplit, kConcat, kMatMul, kSoftmax,
};
const char* fw_op_name(FwOpKind k);

struct NodeAttrs {
  std::vector<int64_t> axes, perm, starts, limits, strides, low, high, interior;
  float pad_value = 0.0f;
  std::vector<int64_t> broadcast_dims;
  std::vector<SymbolicDim> target_shape;
  int64_t num_splits = 0;
  int64_t axis = 0;
};

struct FrameworkNode {
  std::string id;
  FwOpKind op = FwOpKind::kAdd;
  std::vector<std::string> inputs, outputs;
  NodeAttrs attrs;
};

struct FrameworkGraph {
  std::string name;
  std::vector<GraphValue> inputs;
  std::vector<std::string> outputs;
  std::vector<FrameworkNode> nodes;
  std::vector<std::string> symbol_names;
  std::map<std::string, ShapeVector> tensor_shapes;
  const ShapeVector& shape_of(const std::string& id) const;
  bool is_input(const std::string& id) const;
};

FrameworkGraph parse_graph(const std::string& json_text);

// ---------------------------------------------------------------------------
// DHLO hub IR (reference dhlo.hpp:35-131).
enum class DhloOpKind {
  kAdd, kSub, kMul, kDiv, kMaximum, kExp, kTanh, kNeg, kReduceSum, kReduceMax,
  kTranspose, kDynamicBroadcastInDim, kDynamicReshape, kDynamicSlice, kDynamicPad,
  kConcat, kMatMul, kConstant, kShapeOf, kExtractDim, kScalarArith,
};
enum class ScalarArithKind { kAdd, kSub, kMul, kDiv, kCeilDiv };

const char* dhlo_kind_name(DhloOpKind k);
std::optional<DhloOpKind> dhlo_kind_from_name(const std::string& s);
const char* scalar_arith_name(ScalarArithKind k);
std::optional<ScalarArithKind> scalar_arith_from_name(const std::string& s);

bool is_elementwise_binary(DhloOpKind k);
bool is_elementwise_unary(DhloOpKind k);
bool is_reduce(DhloOpKind k);
bool is_index_plumbing(DhloOpKind k);
inline bool is_compute_op(DhloOpKind k) { return !is_index_plumbing(k); }

struct Literal {
  ElementType etype = ElementType::kF32;
  std::vector<int64_t> dims;
  std::vector<float> f32;
  std::vector<int64_t> i64;
  int64_t numel() const {
    int64_t n = 1;
    for (int64_t d : dims) n *= d;
    return n;
  }
};

struct DhloOp {
  std::string id;
  DhloOpKind kind = DhloOpKind::kAdd;
  std::vector<std::string> inputs;
  ShapeVector shape;
  ElementType etype = ElementType::kF32;
  std::vector<int64_t> dims_attr;  // reduce axes | transpose perm | broadcast_dims
  int64_t axis = 0;                // concat
  int64_t index = 0;               // extract_dim
  ScalarArithKind arith = ScalarArithKind::kAdd;
  Literal literal;
};

struct SymbolOrigin {
  enum class Kind { kInputDim, kDerived };
  Kind kind = Kind::kInputDim;
  int input = -1;
  int dim = -1;
  std::string op_id;
};

struct DhloGraph {
  std::string name;
  std::vector<GraphValue> inputs;
  std::vector<std::string> outputs;
  std::vector<DhloOp> ops;
  std::vector<SymbolOrigin> symbols;

  int new_symbol(SymbolOrigin o) {
    symbols.push_back(std::move(o));
    return static_cast<int>(symbols.size()) - 1;
  }
  const DhloOp* find_op(const std::string& id) const;
  const GraphValue* find_input(const std::string& id) const;
  const ShapeVector& value_shape(const std::string& id) const;
  ElementType value_etype(const std::string& id) const;
};

std::vector<std::string> verify(const DhloGraph& g);
std::string print_text(const DhloGraph& g);
std::string to_json(const DhloGraph& g);
DhloGraph dhlo_from_json(const std::string& text);

// Size of a data-argument prefix of an op's operand list: index operands (slice
// starts/limits/strides, broadcast/reshape shape tensors, pad value/edges) follow it.
size_t data_arg_count(const DhloOp& op);

}  // namespace disc
