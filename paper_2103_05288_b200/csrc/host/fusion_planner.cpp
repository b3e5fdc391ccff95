// Fusion planner: greedy reverse-topological growth of kLoop / kInput groups under the
// op-class rules, same-size proofs and convexity; shape-agnostic pattern signatures;
// multi-version kernel specs.  Ordering (seed order, ascending candidate scan with
// restart, group reversal) follows the reference fusion.cpp:28-403.
#include <algorithm>
#include <cstdio>
#include <sstream>

#include "compiler.hpp"

namespace disc {

uint64_t fnv1a64(const std::string& s) {
  // NB: the reference seeds with 1469598103934665603 (the FNV-1a offset basis missing its
  // last digit, fusion.cpp:29); digests and plan signatures depend on it.
  uint64_t h = 1469598103934665603ull;
  for (unsigned char ch : s) h = (h ^ ch) * 0x100000001b3ull;
  return h;
}

std::string digest_hex(const std::string& s) {
  char buf[17];
  std::snprintf(buf, sizeof buf, "%016llx", static_cast<unsigned long long>(fnv1a64(s)));
  return buf;
}

bool is_fusible_kind(DhloOpKind k) {
  return is_elementwise_binary(k) || is_elementwise_unary(k) || is_reduce(k) ||
         k == DhloOpKind::kDynamicBroadcastInDim || k == DhloOpKind::kDynamicSlice;
}

namespace {

// Producer/consumer adjacency over op positions (graph inputs are not nodes).
struct Adjacency {
  std::map<std::string, int> pos;
  std::vector<std::vector<int>> producers, consumers;
  explicit Adjacency(const DhloGraph& g) : producers(g.ops.size()), consumers(g.ops.size()) {
    for (size_t i = 0; i < g.ops.size(); ++i) pos[g.ops[i].id] = static_cast<int>(i);
    for (size_t i = 0; i < g.ops.size(); ++i)
      for (const auto& a : g.ops[i].inputs) {
        auto it = pos.find(a);
        if (it == pos.end()) continue;
        producers[i].push_back(it->second);
        consumers[it->second].push_back(static_cast<int>(i));
      }
  }
};

// At most one reduce; every non-reduce member same-size with the iteration space (the
// reduce input for kInput groups); after the reduce only broadcasts of the reduce
// result and at most one elementwise epilogue.
bool admissible(const DhloGraph& g, const Adjacency& adj, const ConstraintSet& cs, const std::set<int>& m) {
  int red = -1;
  for (int i : m)
    if (is_reduce(g.ops[i].kind)) {
      if (red >= 0) return false;
      red = i;
    }
  const ShapeVector space = red >= 0 ? g.value_shape(g.ops[red].inputs[0]) : g.ops[*m.begin()].shape;
  for (int i : m) {
    const ShapeVector& s = i == red ? g.value_shape(g.ops[i].inputs[0]) : g.ops[i].shape;
    if (!cs.same_size(s, space)) return false;
  }
  if (red < 0) return true;

  std::set<int> after;
  std::vector<int> stack = {red};
  while (!stack.empty()) {
    int cur = stack.back();
    stack.pop_back();
    for (int u : adj.consumers[cur])
      if (m.count(u) && after.insert(u).second) stack.push_back(u);
  }
  int epilogues = 0;
  for (int i : after) {
    const DhloOp& op = g.ops[i];
    if (op.kind == DhloOpKind::kDynamicBroadcastInDim) {
      if (op.inputs[0] != g.ops[red].id) return false;
    } else if (is_elementwise_binary(op.kind) || is_elementwise_unary(op.kind)) {
      if (++epilogues > 1) return false;
    } else {
      return false;
    }
  }
  return true;
}

// Convex: no non-member both depends on a member and feeds a member (paths through
// index plumbing count).
bool convex(const DhloGraph& g, const Adjacency& adj, const std::set<int>& m) {
  const int n = static_cast<int>(g.ops.size());
  std::vector<char> below(n, 0), above(n, 0);
  for (int i = 0; i < n; ++i) {
    if (m.count(i)) {
      below[i] = 1;
      continue;
    }
    for (int p : adj.producers[i])
      if (below[p]) {
        below[i] = 1;
        break;
      }
  }
  for (int i = n - 1; i >= 0; --i) {
    if (m.count(i)) {
      above[i] = 1;
      continue;
    }
    for (int c : adj.consumers[i])
      if (above[c]) {
        above[i] = 1;
        break;
      }
  }
  for (int i = 0; i < n; ++i)
    if (!m.count(i) && below[i] && above[i]) return false;
  return true;
}

void op_signature(std::ostringstream& os, const DhloOp& op, const std::map<std::string, int>& member,
                  std::map<std::string, int>& external) {
  os << dhlo_kind_name(op.kind) << "/r" << op.shape.rank();
  if (!op.dims_attr.empty()) {
    os << "/a[";
    for (size_t i = 0; i < op.dims_attr.size(); ++i) os << (i ? "," : "") << op.dims_attr[i];
    os << "]";
  }
  if (op.kind == DhloOpKind::kConcat) os << "/x" << op.axis;
  if (op.kind == DhloOpKind::kExtractDim) os << "/i" << op.index;
  if (op.kind == DhloOpKind::kScalarArith) os << "/" << scalar_arith_name(op.arith);
  os << "(";
  for (size_t i = 0; i < op.inputs.size(); ++i) {
    if (i) os << ",";
    auto it = member.find(op.inputs[i]);
    if (it != member.end()) {
      os << "m" << it->second;
    } else {
      auto ins = external.emplace(op.inputs[i], static_cast<int>(external.size()));
      os << "e" << ins.first->second;
    }
  }
  os << ");";
}

}  // namespace

std::string pattern_signature(const DhloGraph& g, const std::vector<std::string>& members) {
  std::map<std::string, int> member, external;
  for (size_t i = 0; i < members.size(); ++i) member[members[i]] = static_cast<int>(i);
  std::ostringstream os;
  for (const auto& id : members) {
    const DhloOp* op = g.find_op(id);
    if (!op) throw InternalError("signature: unknown member " + id);
    op_signature(os, *op, member, external);
  }
  return os.str();
}

std::string whole_graph_signature(const DhloGraph& g) {
  std::vector<std::string> all;
  for (const auto& op : g.ops) all.push_back(op.id);
  std::ostringstream os;
  os << pattern_signature(g, all) << "|inputs:";
  std::map<int, int> order;
  for (const auto& in : g.inputs) {
    os << "[";
    for (const auto& d : in.shape.dims) {
      if (d.is_const()) {
        os << "c" << d.size() << ",";
      } else {
        auto ins = order.emplace(d.sym_id(), static_cast<int>(order.size()));
        os << "p" << ins.first->second << ",";
      }
    }
    os << "]";
  }
  os << "|literals:";
  for (const auto& op : g.ops) {
    if (op.kind != DhloOpKind::kConstant) continue;
    std::ostringstream lit;
    lit << op.id << ":";
    for (int64_t d : op.literal.dims) lit << d << ",";
    lit << ":";
    if (op.literal.etype == ElementType::kF32)
      for (float f : op.literal.f32) lit << f << ",";
    else
      for (int64_t v : op.literal.i64) lit << v << ",";
    os << digest_hex(lit.str());
  }
  std::map<std::string, int> pos;
  for (size_t i = 0; i < g.ops.size(); ++i) pos[g.ops[i].id] = static_cast<int>(i);
  os << "|outputs:";
  for (const auto& o : g.outputs) {
    auto it = pos.find(o);
    if (it != pos.end()) {
      os << "m" << it->second << ",";
      continue;
    }
    for (size_t i = 0; i < g.inputs.size(); ++i)
      if (g.inputs[i].id == o) os << "in" << i << ",";
  }
  return os.str();
}

std::vector<FusionGroup> fuse(const DhloGraph& g, const ConstraintSet& cs) {
  const Adjacency adj(g);
  const int n = static_cast<int>(g.ops.size());
  auto fusible = [&](int i) { return g.ops[i].etype == ElementType::kF32 && is_fusible_kind(g.ops[i].kind); };

  // Slices of one source (a lowered Split) are siblings even with no edge between them.
  std::map<std::string, std::vector<int>> sibling_slices;
  for (int i = 0; i < n; ++i)
    if (g.ops[i].kind == DhloOpKind::kDynamicSlice && fusible(i)) sibling_slices[g.ops[i].inputs[0]].push_back(i);

  auto frontier = [&](const std::set<int>& m) {
    std::set<int> f;
    for (int i : m) {
      for (int p : adj.producers[i])
        if (fusible(p)) f.insert(p);
      for (int c : adj.consumers[i])
        if (fusible(c)) f.insert(c);
      if (g.ops[i].kind == DhloOpKind::kDynamicSlice) {
        auto it = sibling_slices.find(g.ops[i].inputs[0]);
        if (it != sibling_slices.end()) f.insert(it->second.begin(), it->second.end());
      }
    }
    for (int i : m) f.erase(i);
    return f;
  };

  std::vector<char> taken(n, 0);
  std::vector<FusionGroup> groups;
  for (int seed = n - 1; seed >= 0; --seed) {
    if (taken[seed] || !fusible(seed)) continue;
    std::set<int> m = {seed};
    for (bool grown = true; grown;) {
      grown = false;
      for (int c : frontier(m)) {  // ascending: smallest index first, restart on success
        if (taken[c]) continue;
        std::set<int> trial = m;
        trial.insert(c);
        if (!admissible(g, adj, cs, trial) || !convex(g, adj, trial)) continue;
        m = std::move(trial);
        grown = true;
        break;
      }
    }

    FusionGroup grp;
    grp.id = static_cast<int>(groups.size());
    for (int i : m) {
      taken[i] = 1;
      grp.members.push_back(g.ops[i].id);
      if (is_reduce(g.ops[i].kind)) {
        grp.root = RootKind::kReduceRoot;
        grp.reduce_member = g.ops[i].id;
      }
    }
    std::set<std::string> inside(grp.members.begin(), grp.members.end()), seen;
    for (int i : m) {
      const DhloOp& op = g.ops[i];
      for (size_t a = 0; a < data_arg_count(op); ++a) {
        const std::string& v = op.inputs[a];
        if (inside.count(v) || !seen.insert(v).second) continue;
        grp.external_inputs.push_back(v);
      }
    }
    for (int i : m) {
      bool visible = std::find(g.outputs.begin(), g.outputs.end(), g.ops[i].id) != g.outputs.end();
      for (int c : adj.consumers[i])
        visible = visible || (!m.count(c) && g.ops[c].etype == ElementType::kF32 && is_compute_op(g.ops[c].kind));
      if (visible) grp.external_outputs.push_back(g.ops[i].id);
    }
    grp.signature = pattern_signature(g, grp.members);
    groups.push_back(std::move(grp));
  }
  std::reverse(groups.begin(), groups.end());
  for (size_t i = 0; i < groups.size(); ++i) groups[i].id = static_cast<int>(i);
  return groups;
}

std::vector<KernelSpec> specialize(const DhloGraph& g, const std::vector<FusionGroup>& groups,
                                   const ConstraintSet&) {
  std::vector<KernelSpec> specs;
  for (const auto& grp : groups) {
    KernelSpec spec;
    spec.kernel_id = grp.id;
    spec.group = grp;
    bool bcast = std::any_of(grp.members.begin(), grp.members.end(), [&](const std::string& id) {
      return g.find_op(id)->kind == DhloOpKind::kDynamicBroadcastInDim;
    });
    int next = 0;
    KernelVersion v4;
    v4.id = next++;
    v4.vectorized4 = true;
    if (bcast) v4.guards.push_back(GuardKind::kBroadcastIdentity);
    v4.guards.push_back(GuardKind::kTotalDivisibleBy4);
    spec.versions.push_back(v4);
    if (bcast) {
      KernelVersion nb;
      nb.id = next++;
      nb.guards = {GuardKind::kBroadcastIdentity};
      spec.versions.push_back(nb);
    }
    KernelVersion scalar;
    scalar.id = next++;
    scalar.implicit_broadcast = bcast;
    scalar.guards = {GuardKind::kAlways};
    spec.versions.push_back(scalar);
    specs.push_back(std::move(spec));
  }
  return specs;
}

}  // namespace disc
