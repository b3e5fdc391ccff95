// TEST INFRASTRUCTURE ONLY -- never linked into, loaded by, or called from the product path.
//
// A C-ABI shim over the *unmodified* reference DISC artifact (arXiv 2103.05288 desk-scale
// re-creation), compiled from /root/reference/proj/src/*.cpp by oracle/Makefile into
// oracle/_ref/libdisc_ref.so.  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load it, and only as the checker / the CPU
// baseline being timed.
//
// What it exposes (all reference entry points, nothing re-implemented):
//   * compile_graph + plan_to_json                  (codegen.cpp:688, runtime_program.cpp:182)
//   * Compiler (plan cache) stats                    (codegen.cpp:766-802)
//   * lower_to_dhlo + to_json / print_text goldens   (lowering.cpp:734, dhlo_json.cpp:54)
//   * the TextDumper stages (dump-ir)                (codegen.cpp:624-684)
//   * Executor::run over a parsed plan               (executor.cpp:221-465)
//   * run_kernel / guard_passes per version          (executor.cpp:78-219)
//   * eval_eager (framework level)                   (interpreter.cpp:222-378)
//   * the test utilities' RandomGraphGen / make_binding / random_symbols
//     (tests/testutil.hpp:86-432), so the reference's seeds replay bit-exactly.
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "disc/codegen.hpp"
#include "disc/executor.hpp"
#include "disc/framework.hpp"
#include "disc/interpreter.hpp"
#include "disc/lowering.hpp"
#include "disc/runtime_program.hpp"

#include <any>
#include <cmath>
#include <fstream>
#include <functional>
#include <json.hpp>
#include <map>
#include <set>
#include <sstream>

#define DISC_FIXTURE_DIR "/nonexistent"
// The generator keeps its JSON in private members; open them up so the shim can hand
// the exact generated graph text back to Python (the class itself is used unmodified).
#define private public
#include "testutil.hpp"
#undef private

namespace {

thread_local std::string g_err;

char* dup_string(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.data(), s.size() + 1);
  return p;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const disc::Error& e) {
    g_err = std::string("error[") + disc::error_class_name(e.error_class()) + "]: " + e.what();
    switch (e.error_class()) {
      case disc::ErrorClass::kUsage: return 2;
      case disc::ErrorClass::kParse:
      case disc::ErrorClass::kValidation:
      case disc::ErrorClass::kCompile: return 3;
      default: return 4;
    }
  } catch (const std::exception& e) {
    g_err = std::string("error[internal]: ") + e.what();
    return 4;
  }
}

disc::CompileOptions make_opts(int inject, int fusion, int static_fb) {
  disc::CompileOptions o;
  o.inject_constraints = inject != 0;
  o.enable_fusion = fusion != 0;
  o.static_fallback = static_fb != 0;
  return o;
}

disc::Binding make_inputs(int n, const char* const* names, const float* const* data,
                          const int64_t* const* dims, const int* ranks) {
  disc::Binding b;
  for (int i = 0; i < n; ++i) {
    std::vector<int64_t> d(dims[i], dims[i] + ranks[i]);
    int64_t numel = 1;
    for (int64_t x : d) numel *= x;
    std::vector<float> v(data[i], data[i] + numel);
    b[names[i]] = disc::ConcreteTensor::from_f32(d, std::move(v));
  }
  return b;
}

}  // namespace

struct dref_result {
  std::vector<disc::ConcreteTensor> tensors;
  std::vector<std::string> names;
  disc::ExecStats stats;
  std::vector<disc::BufferEvent> events;
};

struct dref_plan {
  disc::CompiledPlan plan;
};

struct dref_executor {
  disc::Executor exec;
};

struct dref_compiler {
  explicit dref_compiler(disc::CompileOptions o) : c(o) {}
  disc::Compiler c;
};

struct dref_rng {
  explicit dref_rng(uint64_t s) : rng(s) {}
  std::mt19937_64 rng;
};

extern "C" {

const char* dref_last_error() { return g_err.c_str(); }
void dref_free(void* p) { std::free(p); }

// --- compile side -----------------------------------------------------------

int dref_compile(const char* graph_json, int inject, int fusion, int static_fb, char** plan_json) {
  return guarded([&] {
    auto g = disc::parse_graph(graph_json);
    *plan_json = dup_string(disc::plan_to_json(disc::compile_graph(g, make_opts(inject, fusion, static_fb))));
  });
}

int dref_static_specialize(const char* graph_json, char** plan_json) {
  return guarded([&] {
    auto g = disc::parse_graph(graph_json);
    *plan_json = dup_string(disc::plan_to_json(disc::static_specialize(g)));
  });
}

int dref_cache_key(const char* graph_json, int inject, int fusion, int static_fb, char** key) {
  return guarded([&] {
    auto g = disc::parse_graph(graph_json);
    *key = dup_string(disc::cache_key(g, make_opts(inject, fusion, static_fb)));
  });
}

// stage in {dhlo, constraints, simplified, fused, program}
int dref_dump_stage(const char* graph_json, int inject, int fusion, const char* stage, char** text) {
  return guarded([&] {
    auto g = disc::parse_graph(graph_json);
    std::string wanted = stage, captured;
    disc::compile_graph(g, make_opts(inject, fusion, 0),
                        [&](const std::string& st, const std::string& t) {
                          if (st == wanted) captured = t;
                        });
    *text = dup_string(captured);
  });
}

int dref_lower_dhlo_json(const char* graph_json, char** dhlo_json) {
  return guarded([&] {
    auto g = disc::parse_graph(graph_json);
    auto [d, cs] = disc::lower_to_dhlo(g);
    *dhlo_json = dup_string(disc::to_json(d));
  });
}

int dref_roundtrip_plan(const char* plan_json, char** out) {
  return guarded([&] { *out = dup_string(disc::plan_to_json(disc::plan_from_json(plan_json))); });
}

int dref_compiler_new(int inject, int fusion, int static_fb, dref_compiler** out) {
  return guarded([&] { *out = new dref_compiler(make_opts(inject, fusion, static_fb)); });
}
void dref_compiler_free(dref_compiler* c) { delete c; }
int dref_compiler_compile(dref_compiler* c, const char* graph_json, char** plan_json) {
  return guarded([&] {
    auto g = disc::parse_graph(graph_json);
    auto p = c->c.compile(g);
    if (plan_json) *plan_json = dup_string(disc::plan_to_json(*p));
  });
}
void dref_compiler_stats(dref_compiler* c, int64_t* compile_count, int64_t* cache_hits) {
  auto s = c->c.stats();
  *compile_count = s.compile_count;
  *cache_hits = s.cache_hits;
}

// --- run side ---------------------------------------------------------------

int dref_plan_load(const char* plan_json, dref_plan** out) {
  return guarded([&] {
    auto p = std::make_unique<dref_plan>();
    p->plan = disc::plan_from_json(plan_json);
    *out = p.release();
  });
}
void dref_plan_free(dref_plan* p) { delete p; }

dref_executor* dref_executor_new() { return new dref_executor(); }
void dref_executor_free(dref_executor* e) { delete e; }

int dref_executor_run(dref_executor* e, const dref_plan* p, int n, const char* const* names,
                      const float* const* data, const int64_t* const* dims, const int* ranks,
                      dref_result** out) {
  return guarded([&] {
    auto r = std::make_unique<dref_result>();
    disc::Binding b = make_inputs(n, names, data, dims, ranks);
    disc::ExecResult res = e->exec.run(p->plan, b);
    r->tensors = std::move(res.outputs);
    r->stats = res.stats;
    r->events = std::move(res.buffer_events);
    for (const auto& o : p->plan.outputs) r->names.push_back(o.id);
    *out = r.release();
  });
}

// Times `reps` runs of the same binding; returns seconds of wall time.
int dref_executor_time(dref_executor* e, const dref_plan* p, int n, const char* const* names,
                       const float* const* data, const int64_t* const* dims, const int* ranks,
                       int reps, double* seconds) {
  return guarded([&] {
    disc::Binding b = make_inputs(n, names, data, dims, ranks);
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) e->exec.run(p->plan, b);
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

int dref_eval_eager(const char* graph_json, int n, const char* const* names,
                    const float* const* data, const int64_t* const* dims, const int* ranks,
                    dref_result** out) {
  return guarded([&] {
    auto g = disc::parse_graph(graph_json);
    auto r = std::make_unique<dref_result>();
    disc::EagerStats st;
    r->tensors = disc::eval_eager(g, make_inputs(n, names, data, dims, ranks), &st);
    r->names = g.outputs;
    r->stats.launch_count = st.op_count;
    r->stats.peak_bytes = st.peak_bytes;
    *out = r.release();
  });
}

// run_kernel on one artifact/version with caller-provided externals and registers.
int dref_run_kernel(const dref_plan* p, int kernel, int version, int n, const float* const* data,
                    const int64_t* const* dims, const int* ranks, const int64_t* regs,
                    int nregs, dref_result** out) {
  return guarded([&] {
    const auto& art = p->plan.kernels.at(kernel);
    const disc::VersionArtifact* v = nullptr;
    for (const auto& x : art.versions)
      if (x.id == version) v = &x;
    if (!v) throw disc::InternalError("no such version");
    std::vector<disc::ConcreteTensor> ext;
    for (int i = 0; i < n; ++i) {
      std::vector<int64_t> d(dims[i], dims[i] + ranks[i]);
      int64_t numel = 1;
      for (int64_t x : d) numel *= x;
      ext.push_back(disc::ConcreteTensor::from_f32(d, std::vector<float>(data[i], data[i] + numel)));
    }
    std::vector<const disc::ConcreteTensor*> ptrs;
    for (const auto& t : ext) ptrs.push_back(&t);
    auto r = std::make_unique<dref_result>();
    r->tensors = disc::run_kernel(art, *v, ptrs, std::vector<int64_t>(regs, regs + nregs));
    *out = r.release();
  });
}

int dref_guard_passes(const dref_plan* p, int kernel, int version, const int64_t* regs, int nregs) {
  const auto& art = p->plan.kernels.at(kernel);
  for (const auto& x : art.versions)
    if (x.id == version) return disc::guard_passes(art, x, std::vector<int64_t>(regs, regs + nregs)) ? 1 : 0;
  return -1;
}

int dref_result_count(const dref_result* r) { return static_cast<int>(r->tensors.size()); }
int dref_result_rank(const dref_result* r, int i) { return r->tensors[i].rank(); }
const int64_t* dref_result_dims(const dref_result* r, int i) { return r->tensors[i].dims.data(); }
const float* dref_result_data(const dref_result* r, int i) { return r->tensors[i].f32.data(); }
// launch_count, library_calls, host_instruction_count, peak_bytes, alloc_calls,
// allocator_cache_hits, aliased_allocs
void dref_result_stats(const dref_result* r, int64_t* s7, double* ms2) {
  const auto& s = r->stats;
  int64_t v[7] = {s.launch_count, s.library_calls, s.host_instruction_count, s.peak_bytes,
                  s.alloc_calls, s.allocator_cache_hits, s.aliased_allocs};
  std::memcpy(s7, v, sizeof(v));
  if (ms2) {
    ms2[0] = s.host_ms;
    ms2[1] = s.kernel_ms;
  }
}
int dref_result_num_events(const dref_result* r) { return static_cast<int>(r->events.size()); }
void dref_result_event(const dref_result* r, int i, int* four) {
  const auto& e = r->events[i];
  four[0] = e.logical;
  four[1] = e.physical;
  four[2] = e.alloc_instr;
  four[3] = e.dealloc_instr;
}
void dref_result_free(dref_result* r) { delete r; }

// --- reference test utilities (seed-exact) ----------------------------------

dref_rng* dref_rng_new(uint64_t seed) { return new dref_rng(seed); }
void dref_rng_free(dref_rng* r) { delete r; }

int dref_random_graph(uint64_t seed, int max_nodes, char** graph_json) {
  return guarded([&] {
    disc::testing::RandomGraphGen gen(seed);
    gen.generate(max_nodes);
    // Rebuild the exact text generate() parsed (testutil.hpp:189-196).
    nlohmann::json g;
    g["name"] = "random";
    g["inputs"] = gen.inputs_;
    g["nodes"] = gen.nodes_;
    nlohmann::json outputs = nlohmann::json::array();
    for (const auto& t : gen.tensors_)
      if (!gen.consumed_.count(t.id)) outputs.push_back(t.id);
    if (outputs.empty()) outputs.push_back(gen.tensors_.back().id);
    g["outputs"] = outputs;
    *graph_json = dup_string(g.dump());
  });
}

// random_symbols(g, rng, allow_zero) -> {"name": value, ...}
int dref_random_symbols(dref_rng* rng, const char* graph_json, int allow_zero, char** syms_json) {
  return guarded([&] {
    auto g = disc::parse_graph(graph_json);
    auto m = disc::testing::random_symbols(g, rng->rng, allow_zero != 0);
    nlohmann::json j = nlohmann::json::object();
    for (const auto& [k, v] : m) j[k] = v;
    *syms_json = dup_string(j.dump());
  });
}

// make_binding(g, syms, seed): the reference's input tensors (names in graph input order).
int dref_make_binding(const char* graph_json, const char* syms_json, uint64_t seed,
                      dref_result** out) {
  return guarded([&] {
    auto g = disc::parse_graph(graph_json);
    std::map<std::string, int64_t> syms;
    auto parsed = nlohmann::json::parse(syms_json);
    for (auto it = parsed.begin(); it != parsed.end(); ++it) syms[it.key()] = it.value().get<int64_t>();
    disc::Binding b = disc::testing::make_binding(g, syms, seed);
    auto r = std::make_unique<dref_result>();
    for (const auto& in : g.inputs) {
      r->tensors.push_back(b.at(in.id));
      r->names.push_back(in.id);
    }
    *out = r.release();
  });
}

}  // extern "C"
