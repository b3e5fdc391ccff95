// C ABI, compile side: graph -> plan, plan JSON I/O, stage dumps, shape evaluation.
#include <cstdlib>
#include <cstring>
#include <memory>

#include "capi_common.hpp"
#include "host/compiler.hpp"
#include "json.hpp"

using namespace disc;

namespace disc_capi {
thread_local std::string g_error;
thread_local int g_error_class = -1;

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}
}  // namespace disc_capi

using disc_capi::dup;
using disc_capi::guard;

struct disc_compiler_s {
  explicit disc_compiler_s(CompileOptions o) : c(o) {}
  Compiler c;
};

namespace {
CompileOptions opts(int inject, int fusion, int static_fb) {
  CompileOptions o;
  o.inject_constraints = inject != 0;
  o.enable_fusion = fusion != 0;
  o.static_fallback = static_fb != 0;
  return o;
}
disc_plan wrap(std::shared_ptr<const CompiledPlan> p) { return new disc_plan_s(std::move(p)); }
}  // namespace

extern "C" {

const char* disc_last_error(void) { return disc_capi::g_error.c_str(); }
int disc_last_error_class(void) { return disc_capi::g_error_class; }
void disc_free(void* p) { std::free(p); }
const char* disc_version(void) { return "disc-b200 0.1 (sm_100a)"; }

int disc_compile_graph(const char* graph_json, int inject, int fusion, int static_fb, disc_plan* out) {
  return guard([&] {
    FrameworkGraph g = parse_graph(graph_json);
    *out = wrap(std::make_shared<const CompiledPlan>(compile_graph(g, opts(inject, fusion, static_fb))));
  });
}

int disc_static_specialize(const char* graph_json, disc_plan* out) {
  return guard([&] {
    FrameworkGraph g = parse_graph(graph_json);
    *out = wrap(std::make_shared<const CompiledPlan>(static_specialize(g)));
  });
}

int disc_compiler_create(int inject, int fusion, int static_fb, disc_compiler* out) {
  return guard([&] { *out = new disc_compiler_s(opts(inject, fusion, static_fb)); });
}
void disc_compiler_destroy(disc_compiler c) { delete c; }

int disc_compiler_compile(disc_compiler c, const char* graph_json, disc_plan* out) {
  return guard([&] {
    FrameworkGraph g = parse_graph(graph_json);
    *out = wrap(c->c.compile(g));
  });
}

void disc_compiler_stats(disc_compiler c, int64_t* compile_count, int64_t* cache_hits) {
  CompilerStats s = c->c.stats();
  *compile_count = s.compile_count;
  *cache_hits = s.cache_hits;
}

int disc_cache_key(const char* graph_json, int inject, int fusion, int static_fb, char** out) {
  return guard([&] { *out = dup(cache_key(parse_graph(graph_json), opts(inject, fusion, static_fb))); });
}

int disc_dump_stage(const char* graph_json, int inject, int fusion, const char* stage, char** out) {
  return guard([&] {
    static const char* const kStages[] = {"dhlo", "constraints", "simplified", "fused", "program"};
    bool known = false;
    for (const char* s : kStages) known = known || std::strcmp(s, stage) == 0;
    if (!known)
      throw Error(ErrorClass::kUsage, std::string("unknown stage ") + stage +
                                          " (dhlo|constraints|simplified|fused|program)");
    FrameworkGraph g = parse_graph(graph_json);
    std::string want = stage, got;
    compile_graph(g, opts(inject, fusion, 0), [&](const std::string& st, const std::string& text) {
      if (st == want) got = text;
    });
    *out = dup(got);
  });
}

int disc_lower_dhlo_json(const char* graph_json, char** out) {
  return guard([&] { *out = dup(to_json(lower_to_dhlo(parse_graph(graph_json)).first)); });
}

int disc_dhlo_roundtrip(const char* dhlo_json, char** out) {
  return guard([&] { *out = dup(to_json(dhlo_from_json(dhlo_json))); });
}

int disc_plan_from_json(const char* plan_json, disc_plan* out) {
  return guard([&] { *out = wrap(std::make_shared<const CompiledPlan>(plan_from_json(plan_json))); });
}

int disc_plan_to_json(disc_plan p, char** out) {
  return guard([&] { *out = dup(plan_to_json(*p->plan)); });
}

int disc_plan_check(disc_plan p, char** diags) {
  return guard([&] { *diags = dup(nlohmann::json(check_plan(*p->plan)).dump()); });
}

void disc_plan_retain(disc_plan p) { p->refs.fetch_add(1); }
const void* disc_plan_identity(disc_plan p) { return p ? p->plan.get() : nullptr; }
void disc_plan_release(disc_plan p) {
  if (p && p->refs.fetch_sub(1) == 1) delete p;
}

int disc_plan_num_inputs(disc_plan p) { return static_cast<int>(p->plan->inputs.size()); }
const char* disc_plan_input_name(disc_plan p, int i) { return p->plan->inputs.at(i).id.c_str(); }
int disc_plan_input_rank(disc_plan p, int i) { return static_cast<int>(p->plan->inputs.at(i).dims.size()); }
int disc_plan_num_outputs(disc_plan p) { return static_cast<int>(p->plan->outputs.size()); }
const char* disc_plan_output_name(disc_plan p, int i) { return p->plan->outputs.at(i).id.c_str(); }
int disc_plan_num_kernels(disc_plan p) { return static_cast<int>(p->plan->kernels.size()); }
int64_t disc_plan_eager_op_count(disc_plan p) { return p->plan->eager_op_count; }
int64_t disc_plan_host_instruction_count(disc_plan p) { return p->plan->host_instruction_count(); }
const char* disc_plan_input_declared(disc_plan p, int i, int d) {
  const auto& in = p->plan->inputs;
  if (i < 0 || i >= static_cast<int>(in.size()) || d < 0 || d >= static_cast<int>(in[i].declared.size())) return nullptr;
  return in[i].declared[d].c_str();
}
const char* disc_plan_signature(disc_plan p) { return p->plan->signature_digest.c_str(); }

int disc_plan_eval_shapes(disc_plan p, int n, const int64_t* const* dims, const int* ranks, int64_t* regs,
                          int cap, int* nregs) {
  return guard([&] {
    std::vector<std::vector<int64_t>> in(n);
    for (int i = 0; i < n; ++i) in[i].assign(dims[i], dims[i] + ranks[i]);
    std::vector<int64_t> r = disc_capi::eval_shape_program(*p->plan, in);
    *nregs = static_cast<int>(r.size());
    for (int i = 0; i < cap && i < static_cast<int>(r.size()); ++i) regs[i] = r[i];
  });
}

}  // extern "C"
