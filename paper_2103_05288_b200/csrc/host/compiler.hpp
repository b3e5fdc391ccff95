// disc-b200 compile pipeline: constraints, lowering, shape analysis, fusion planning,
// buffer planning and the compile-time-generated runtime flow (CompiledPlan).
//
// API surface mirrors the reference headers (constraint_set.hpp, lowering.hpp,
// shape_analysis.hpp, passes.hpp, fusion.hpp, buffer_plan.hpp, runtime_program.hpp,
// codegen.hpp) so callers of the reference compile unchanged; the plan JSON produced
// is byte-identical to the reference's (tests/test_compiler_parity.py).
#pragma once

#include <functional>
#include <future>
#include <memory>
#include <mutex>
#include <set>

#include "ir.hpp"

namespace disc {

// ---------------------------------------------------------------------------
// Shape constraints (reference constraint_set.hpp:39-109).
class ConstraintSet {
 public:
  void union_dims(const SymbolicDim& a, const SymbolicDim& b, const std::string& context);
  bool same_dim(const SymbolicDim& a, const SymbolicDim& b) const { return canonical(a) == canonical(b); }
  std::optional<int64_t> const_of(int sym) const;
  int rep_of(int sym) const;
  SymbolicDim canonical(const SymbolicDim& d) const;
  bool same_dims(const ShapeVector& a, const ShapeVector& b) const;

  void link_size(const ShapeVector& a, const ShapeVector& b);
  bool same_size(const ShapeVector& a, const ShapeVector& b) const;
  std::string size_key(const ShapeVector& s) const;

  std::string dump() const;
  std::string partition_fingerprint(int num_symbols) const;
  int num_size_links() const { return static_cast<int>(links_.size()); }

 private:
  // Union-find node: parent, interned constant (-1 if a symbol), smallest symbol in class.
  struct Node {
    int parent;
    int64_t value;
    int min_sym;
  };
  std::vector<Node> nodes_;
  std::map<int, int> by_sym_;
  std::map<int64_t, int> by_const_;
  std::vector<std::pair<ShapeVector, ShapeVector>> links_;
  std::map<std::string, std::string> key_root_;  // size-key union-find, rebuilt eagerly

  int sym_node(int sym);
  int const_node(int64_t v);
  int root(int n) const;
  int root_compress(int n);
  void rebuild_size_classes();
  std::string size_class(const std::string& key) const;
};

// ---------------------------------------------------------------------------
// Lowering (reference lowering.hpp:27-42).
struct LoweringOptions {
  bool symbolize_inputs = true;
  bool inject_constraints = true;
};
std::pair<DhloGraph, ConstraintSet> lower_to_dhlo(const FrameworkGraph& g, const LoweringOptions& o = {});

// ---------------------------------------------------------------------------
// Shape analysis + host shape program (reference shape_analysis.hpp:31-125).
enum class OpClass {
  kElementwiseSameShape, kUnaryShapePreserving, kTranspose, kReduce, kMatMul, kConcat,
  kSizePreservingOnly, kBroadcast, kOpaque, kIndexPlumbing,
};
OpClass op_class(DhloOpKind k);
ConstraintSet infer(const DhloGraph& g, const ConstraintSet& seed);
DhloGraph canonicalize_dims(const DhloGraph& g, const ConstraintSet& cs);

enum class ShapeInstrKind { kReadInputDim, kReadScalar, kLoadConst, kBinOp, kBindDim };
enum class ShapeBinOp { kAdd, kSub, kMul, kDivFloor, kCeilDiv, kMax };

struct ShapeInstr {
  ShapeInstrKind kind = ShapeInstrKind::kLoadConst;
  int dest = -1;
  int input = -1;
  int axis = 0;
  std::string tensor;
  int index = 0;
  int64_t value = 0;
  ShapeBinOp op = ShapeBinOp::kAdd;
  int lhs = -1, rhs = -1;
  int sym = -1;
};

struct ShapeProgram {
  std::vector<ShapeInstr> instrs;
  int num_regs = 0;
  std::map<int, int> sym_reg;
  bool empty() const { return instrs.empty(); }
};

struct ScalarRef {
  bool is_const = true;
  int64_t value = 0;
  int reg = -1;
  static ScalarRef Const(int64_t v) { return {true, v, -1}; }
  static ScalarRef Reg(int r) { return {false, 0, r}; }
};

class ShapeProgramBuilder {
 public:
  ShapeProgramBuilder(const DhloGraph& g, const ConstraintSet& cs) : g_(g), cs_(cs) {}
  void bind_all();
  ScalarRef resolve_scalar(const std::string& tensor_id, int index);
  ScalarRef dim_ref(const SymbolicDim& d);
  ScalarRef binop(ShapeBinOp op, ScalarRef a, ScalarRef b);
  const ShapeProgram& program() const { return prog_; }
  const std::set<std::string>& referenced_literals() const { return literals_; }

 private:
  const DhloGraph& g_;
  const ConstraintSet& cs_;
  ShapeProgram prog_;
  std::set<std::string> literals_;
  std::map<int64_t, int> const_reg_;
  int new_reg() { return prog_.num_regs++; }
  int to_reg(const ScalarRef& r, const std::string& literal = "", int lit_index = 0);
  void bind_derived(const DhloOp& op);
  void emit(ShapeInstr si) { prog_.instrs.push_back(std::move(si)); }
};

ShapeProgram emit_shape_program(const DhloGraph& g, const ConstraintSet& cs);

// ---------------------------------------------------------------------------
// Passes (reference passes.hpp:29-53).
struct PassState {
  DhloGraph graph;
  ConstraintSet constraints;
};
struct Pass {
  std::string name;
  std::function<void(PassState&)> run;
};
using StageObserver = std::function<void(const std::string&, const PassState&)>;
PassState run_pipeline(PassState state, const std::vector<Pass>& passes, const StageObserver& obs = nullptr);
void simplify_broadcast(DhloGraph& g, const ConstraintSet& cs);
Pass make_simplify_broadcast_pass();

// ---------------------------------------------------------------------------
// Fusion (reference fusion.hpp:28-90).
enum class RootKind { kElementwiseLoop, kReduceRoot };

struct FusionGroup {
  int id = 0;
  std::vector<std::string> members;
  RootKind root = RootKind::kElementwiseLoop;
  std::string reduce_member;
  std::vector<std::string> external_inputs, external_outputs;
  std::string signature;
};

std::string pattern_signature(const DhloGraph& g, const std::vector<std::string>& members);
std::string whole_graph_signature(const DhloGraph& g);
uint64_t fnv1a64(const std::string& s);
std::string digest_hex(const std::string& s);
bool is_fusible_kind(DhloOpKind k);
std::vector<FusionGroup> fuse(const DhloGraph& g, const ConstraintSet& cs);

enum class GuardKind { kTotalDivisibleBy4, kBroadcastIdentity, kAlways };
struct KernelVersion {
  int id = 0;
  bool vectorized4 = false;
  bool implicit_broadcast = false;
  std::vector<GuardKind> guards;
};
struct KernelSpec {
  int kernel_id = 0;
  FusionGroup group;
  std::vector<KernelVersion> versions;
  static int64_t tile_for(int64_t total) { return total >= (int64_t{1} << 16) ? 1024 : 256; }
};
std::vector<KernelSpec> specialize(const DhloGraph& g, const std::vector<FusionGroup>& groups,
                                   const ConstraintSet& cs);

// ---------------------------------------------------------------------------
// Buffer planning (reference buffer_plan.hpp:31-62).
struct SchedulePoint {
  enum class Kind { kKernel, kLibrary };
  Kind kind = Kind::kKernel;
  int kernel_id = -1;
  std::string op_id;
  std::vector<std::string> inputs, outputs;
};

struct BufferAssignment {
  struct LogicalBuffer {
    int id = 0;
    std::string value_id;
    ShapeVector shape;
    bool is_output = false;
    int def_point = -1;
    int last_use_point = -1;
    int alias_of = -1;
  };
  std::vector<LogicalBuffer> buffers;
  std::map<std::string, int> buffer_of_value;
  std::map<int, std::vector<int>> deallocs_after_point;
  int aliased_allocs = 0;
};
BufferAssignment plan_buffers(const DhloGraph& g, const std::vector<SchedulePoint>& schedule,
                              const ConstraintSet& cs);

// ---------------------------------------------------------------------------
// The compiled runtime flow (reference runtime_program.hpp:32-153).
struct TapeRef {
  enum class Kind { kExternal, kMember };
  Kind kind = Kind::kExternal;
  int index = 0;
};

struct TapeInstr {
  std::string op_id;
  DhloOpKind kind = DhloOpKind::kAdd;
  std::vector<TapeRef> args;
  std::vector<ScalarRef> out_dims;
  std::vector<int64_t> dims;
  std::vector<ScalarRef> slice_starts, slice_strides;
  std::vector<ScalarRef> pad_low, pad_high, pad_interior;
  float pad_value = 0.0f;
  int64_t axis = 0;
};

struct GuardTest {
  enum class Kind { kTotalDivisibleBy4, kRefEqual, kNever, kAlways };
  Kind kind = Kind::kAlways;
  ScalarRef a, b;
};

struct VersionArtifact {
  int id = 0;
  bool vectorized4 = false;
  bool implicit_broadcast = false;
  std::vector<GuardTest> guards;
};

struct KernelArtifact {
  int kernel_id = 0;
  std::string name;
  RootKind root = RootKind::kElementwiseLoop;
  bool standalone = false;
  std::vector<TapeInstr> tape;
  std::vector<std::vector<ScalarRef>> external_input_dims;
  std::vector<int> output_tape_indices;
  std::vector<ScalarRef> space_dims;
  std::vector<VersionArtifact> versions;
  std::string signature;
};

struct SizeExpr {
  int64_t const_elems = 1;
  std::vector<int> regs;
};

enum class InstrKind {
  kBindInput, kEvalShape, kAlloc, kDealloc, kAlias, kSelectVersion, kComputeLaunch,
  kLaunch, kLibraryCall, kBindOutput,
};
const char* instr_kind_name(InstrKind k);

struct Instr {
  InstrKind kind = InstrKind::kBindInput;
  int a = -1;
  int b = -1;
  SizeExpr size;
  std::vector<int> arg_bufs, out_bufs;
  int fixed_version = -1;
  int64_t fixed_tile = -1, fixed_blocks = -1;
  std::vector<ScalarRef> lib_dims;
  bool reserve = false;
};

struct CompiledPlan {
  int plan_version = 1;
  std::string graph_name;
  std::string signature_digest;
  int64_t eager_op_count = 0;
  struct PlanInput {
    std::string id;
    std::vector<std::string> declared;
    std::vector<ScalarRef> dims;
  };
  struct PlanOutput {
    std::string id;
    int buffer = -1;
    std::vector<ScalarRef> dims;
  };
  std::vector<PlanInput> inputs;
  std::vector<PlanOutput> outputs;
  ShapeProgram shape_program;
  std::map<std::string, std::vector<int64_t>> literals;
  std::vector<KernelArtifact> kernels;
  std::vector<Instr> instrs;
  int num_buffers = 0;
  std::vector<std::string> buffer_values;

  int64_t host_instruction_count() const { return static_cast<int64_t>(instrs.size()); }
  int eval_shape_count() const {
    int n = 0;
    for (const auto& i : instrs) n += i.kind == InstrKind::kEvalShape;
    return n;
  }
};

std::string plan_to_json(const CompiledPlan& plan);
CompiledPlan plan_from_json(const std::string& text);
std::vector<std::string> check_plan(const CompiledPlan& plan);

// ---------------------------------------------------------------------------
// Compiler entry points (reference codegen.hpp:32-83).
struct CompileOptions {
  bool inject_constraints = true;
  bool enable_fusion = true;
  bool static_fallback = false;
};
using TextDumper = std::function<void(const std::string& stage, const std::string& text)>;

CompiledPlan compile_graph(const FrameworkGraph& g, const CompileOptions& opts = {},
                           const TextDumper& dump = nullptr);
CompiledPlan static_specialize(const FrameworkGraph& g, const CompileOptions& opts = {},
                               const TextDumper& dump = nullptr);
std::string cache_key(const FrameworkGraph& g, const CompileOptions& opts);

struct CompilerStats {
  int64_t compile_count = 0;
  int64_t cache_hits = 0;
};

// Shape-agnostic plan cache; concurrent compiles of one signature coalesce.
class Compiler {
 public:
  explicit Compiler(CompileOptions defaults = {}) : defaults_(defaults) {}
  std::shared_ptr<const CompiledPlan> compile(const FrameworkGraph& g) { return compile(g, defaults_); }
  std::shared_ptr<const CompiledPlan> compile(const FrameworkGraph& g, const CompileOptions& opts);
  CompilerStats stats() const {
    std::lock_guard<std::mutex> lk(mu_);
    return stats_;
  }

 private:
  CompileOptions defaults_;
  mutable std::mutex mu_;
  std::map<std::string, std::shared_future<std::shared_ptr<const CompiledPlan>>> cache_;
  CompilerStats stats_;
};

}  // namespace disc
