// `disc` command-line tool over the C ABI (include/disc_b200.h): the reference CLI's
// subcommands, options, output lines, session-stats file and exit codes
// (tools/disc_main.cpp:138-368, pinned by tests/cli_test.cmake), with plans executed by
// the B200 device executor.  Differences, by design:
//   * `run --eager` runs the graph unfused (one device launch per op) instead of the
//     reference's host interpreter (the interpreter is not part of the product);
//   * `bench` times the device executor (inputs resident in HBM, synchronized wall clock,
//     device kernel time from CUDA events).
// Exit codes: 0 ok, 2 usage, 3 parse/validation/compile, 4 runtime/internal.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <json.hpp>
#include <map>
#include <memory>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "disc_b200.h"
#include "disc_cuda.h"

namespace {

using nlohmann::json;

// A failure with its exit code and the "error[<class>]: message" line.
struct Failure {
  int code;
  std::string line;
};
[[noreturn]] void usage_error(const std::string& msg) { throw Failure{2, "error[usage]: " + msg}; }
[[noreturn]] void runtime_error(const std::string& msg) { throw Failure{4, "error[runtime]: " + msg}; }
// Library status -> Failure (disc_last_error already carries the class prefix).
void check(int rc) {
  if (rc != 0) throw Failure{rc, disc_last_error()};
}

// ---------------------------------------------------------------------------
// Argument parsing: one subcommand, its positionals, flags and valued options
// (`--opt v`, `--opt=v`, `-o v`; repeatable options collect every value).
struct Spec {
  std::vector<std::string> positionals;                 // required, in order
  std::map<std::string, std::string> flags;             // spelling -> canonical name
  std::map<std::string, std::string> options;           // spelling -> canonical name
};

struct Parsed {
  std::map<std::string, std::string> pos;
  std::map<std::string, bool> flag;
  std::map<std::string, std::vector<std::string>> opt;
  bool has(const std::string& k) const { return opt.count(k) && !opt.at(k).empty(); }
  std::string get(const std::string& k, const std::string& dflt = "") const { return has(k) ? opt.at(k).back() : dflt; }
  bool on(const std::string& k) const { return flag.count(k) && flag.at(k); }
};

Parsed parse_args(const Spec& spec, int argc, char** argv, int first) {
  Parsed p;
  size_t npos = 0;
  for (int i = first; i < argc; ++i) {
    std::string a = argv[i], val;
    bool has_val = false;
    if (a.size() > 1 && a[0] == '-') {
      const size_t eq = a.find('=');
      if (eq != std::string::npos) {
        val = a.substr(eq + 1);
        a = a.substr(0, eq);
        has_val = true;
      }
      if (auto f = spec.flags.find(a); f != spec.flags.end()) {
        if (has_val) usage_error(a + " takes no value");
        p.flag[f->second] = true;
      } else if (auto o = spec.options.find(a); o != spec.options.end()) {
        if (!has_val) {
          if (i + 1 >= argc) usage_error(a + " requires a value");
          val = argv[++i];
        }
        p.opt[o->second].push_back(val);
      } else {
        usage_error("unknown option " + a);
      }
    } else {
      if (npos >= spec.positionals.size()) usage_error("unexpected argument " + a);
      p.pos[spec.positionals[npos++]] = a;
    }
  }
  if (npos < spec.positionals.size()) usage_error(spec.positionals[npos] + " is required");
  return p;
}

// ---------------------------------------------------------------------------
// Files: text, tensors (`shape: d0,d1,...` line + little-endian f32, tensor_io.cpp:25-61)
std::string slurp(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) usage_error("cannot open " + path);
  std::ostringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

void spill(const std::string& path, const std::string& text) {
  std::ofstream f(path, std::ios::binary);
  if (!f) usage_error("cannot write " + path);
  f << text;
}

struct HostTensor {
  std::vector<int64_t> dims;
  std::vector<float> data;
  std::string shape_str() const {
    std::string s = "[";
    for (size_t i = 0; i < dims.size(); ++i) s += (i ? "," : "") + std::to_string(dims[i]);
    return s + "]";
  }
};

HostTensor read_tensor(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) runtime_error("cannot open tensor file " + path);
  std::string header;
  if (!std::getline(f, header)) runtime_error(path + ": missing header line");
  if (header.rfind("shape:", 0) != 0) runtime_error(path + ": header must start with 'shape:'");
  HostTensor t;
  std::stringstream ss(header.substr(6));
  for (std::string tok; std::getline(ss, tok, ',');) {
    const size_t a = tok.find_first_not_of(" \t\r");
    if (a == std::string::npos) continue;
    try {
      t.dims.push_back(std::stoll(tok.substr(a)));
    } catch (const std::exception&) {
      runtime_error(path + ": bad dim '" + tok + "'");
    }
  }
  int64_t n = 1;
  for (int64_t d : t.dims) n *= d;
  t.data.resize(static_cast<size_t>(n));
  f.read(reinterpret_cast<char*>(t.data.data()), n * 4);
  if (f.gcount() != n * 4) runtime_error(path + ": expected " + std::to_string(n * 4) + " data bytes");
  return t;
}

void write_tensor(const std::string& path, const HostTensor& t) {
  std::ofstream f(path, std::ios::binary);
  if (!f) runtime_error("cannot write tensor file " + path);
  f << "shape:";
  for (size_t i = 0; i < t.dims.size(); ++i) f << (i ? "," : " ") << t.dims[i];
  f << "\n";
  f.write(reinterpret_cast<const char*>(t.data.data()), static_cast<std::streamsize>(t.data.size() * 4));
}

// ---------------------------------------------------------------------------
// Session stats: a JSON object persisted across invocations (--stats-file, else
// $DISC_STATS_FILE, else ./disc_stats.json).
struct Session {
  std::string path;
  json j = json::object();
  explicit Session(const std::string& flag) {
    const char* env = std::getenv("DISC_STATS_FILE");
    path = !flag.empty() ? flag : env ? env : "disc_stats.json";
    std::ifstream f(path);
    if (!f) return;
    try {
      json r;
      f >> r;
      if (r.is_object()) j = r;
    } catch (...) {
    }
  }
  void add(const char* k, int64_t d) { j[k] = j.value(k, int64_t{0}) + d; }
  // ExecStats order of disc_executor_stats: launch_count, library_calls,
  // host_instruction_count, peak_bytes, alloc_calls, allocator_cache_hits, aliased_allocs
  void merge_run(const int64_t s[7]) {
    add("launch_count", s[0]);
    add("library_calls", s[1]);
    add("alloc_calls", s[4]);
    add("allocator_cache_hits", s[5]);
    add("aliased_allocs", s[6]);
    j["peak_bytes"] = std::max(j.value("peak_bytes", int64_t{0}), s[3]);
    j["host_instruction_count"] = s[2];
  }
  void save() const { spill(path, j.dump(2)); }
};

// ---------------------------------------------------------------------------
// Library handles
struct Plan {
  disc_plan p = nullptr;
  ~Plan() {
    if (p) disc_plan_release(p);
  }
};

struct Exec {
  disc_executor e = nullptr;
  Exec() { check(disc_executor_create(0, nullptr, &e)); }
  ~Exec() {
    if (e) disc_executor_destroy(e);
  }
};

struct DeviceBuffer {
  void* ptr = nullptr;
  ~DeviceBuffer() {
    if (ptr) disc_cuda_free(ptr, nullptr);
  }
};

struct CompileFlags {
  int inject = 1, fusion = 1, static_fallback = 0;
};

CompileFlags compile_flags(const Parsed& a) {
  CompileFlags f;
  f.inject = !a.on("no-injected-constraints");
  f.fusion = !a.on("no-fusion");
  f.static_fallback = a.on("static-fallback");
  return f;
}

// Pipeline stage texts (dhlo, constraints, simplified, fused, program), the reference
// compile dumper's stages; written to $DISC_DUMP_DIR/<stage>.txt when set.
const std::vector<std::string> kStages = {"dhlo", "constraints", "simplified", "fused", "program"};

void dump_dir_stages(const std::string& graph, const CompileFlags& f) {
  const char* dir = std::getenv("DISC_DUMP_DIR");
  if (!dir || !*dir) return;
  std::filesystem::create_directories(dir);
  for (const auto& st : kStages) {
    char* text = nullptr;
    check(disc_dump_stage(graph.c_str(), f.inject, f.fusion, st.c_str(), &text));
    spill(std::string(dir) + "/" + st + ".txt", text);
    disc_free(text);
  }
}

// Runs a plan on host tensors; returns the outputs (host) and the run's ExecStats.
std::vector<HostTensor> run_plan(disc_plan plan, const std::map<std::string, HostTensor>& binding, int64_t stats[7]) {
  std::vector<const char*> names;
  std::vector<const void*> data;
  std::vector<const int64_t*> dims;
  std::vector<int> ranks;
  for (const auto& [id, t] : binding) {
    names.push_back(id.c_str());
    data.push_back(t.data.data());
    dims.push_back(t.dims.data());
    ranks.push_back(static_cast<int>(t.dims.size()));
  }
  Exec ex;
  check(disc_executor_run(ex.e, plan, static_cast<int>(names.size()), names.data(), data.data(), dims.data(),
                          ranks.data(), 1));
  std::vector<HostTensor> outs(disc_executor_num_outputs(ex.e));
  for (size_t i = 0; i < outs.size(); ++i) {
    const float* dptr = nullptr;
    const int64_t* od = nullptr;
    int rank = 0;
    check(disc_executor_output(ex.e, static_cast<int>(i), &dptr, &od, &rank));
    outs[i].dims.assign(od, od + rank);
    int64_t n = 1;
    for (int64_t d : outs[i].dims) n *= d;
    outs[i].data.resize(static_cast<size_t>(n));
    if (n) check(disc_executor_copy_output(ex.e, static_cast<int>(i), outs[i].data.data(), 1));
  }
  check(disc_executor_synchronize(ex.e));
  double ms[2];
  check(disc_executor_stats(ex.e, stats, ms));
  return outs;
}

std::map<std::string, HostTensor> load_inputs(const std::vector<std::string>& specs) {
  std::map<std::string, HostTensor> b;
  for (const auto& s : specs) {
    const size_t eq = s.find('=');
    if (eq == std::string::npos) usage_error("--input expects id=path, got " + s);
    b[s.substr(0, eq)] = read_tensor(s.substr(eq + 1));
  }
  return b;
}

// Synthetic inputs of a shape binding: declared dims with symbols substituted, values
// uniform [0.25, 2) from mt19937_64(seed) in input order (disc_main.cpp:113-136).
std::map<std::string, HostTensor> synth_inputs(disc_plan plan, const json& shape, uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<float> dist(0.25f, 2.0f);
  std::map<std::string, HostTensor> b;
  for (int i = 0; i < disc_plan_num_inputs(plan); ++i) {
    HostTensor t;
    for (int d = 0; d < disc_plan_input_rank(plan, i); ++d) {
      const std::string e = disc_plan_input_declared(plan, i, d);
      if (!e.empty() && std::isdigit(static_cast<unsigned char>(e[0])))
        t.dims.push_back(std::stoll(e));
      else if (shape.contains(e))
        t.dims.push_back(shape[e].get<int64_t>());
      else
        usage_error("shape binding is missing symbol " + e);
    }
    int64_t n = 1;
    for (int64_t d : t.dims) n *= d;
    t.data.resize(static_cast<size_t>(n));
    for (float& v : t.data) v = dist(rng);
    b[disc_plan_input_name(plan, i)] = std::move(t);
  }
  return b;
}

// ---------------------------------------------------------------------------
// Subcommands
int do_compile(const Parsed& a) {
  const std::string graph_path = a.pos.at("graph"), out = a.get("output", "plan.json");
  const std::string graph = slurp(graph_path);
  const CompileFlags f = compile_flags(a);
  Plan plan;
  check(disc_compile_graph(graph.c_str(), f.inject, f.fusion, f.static_fallback, &plan.p));
  dump_dir_stages(graph, f);
  char* text = nullptr;
  check(disc_plan_to_json(plan.p, &text));
  spill(out, text);
  disc_free(text);
  Session s(a.get("stats-file"));
  s.add("compile_count", 1);
  s.j["host_instruction_count"] = disc_plan_host_instruction_count(plan.p);
  s.save();
  std::cout << "compiled " << graph_path << " -> " << out << " (signature " << disc_plan_signature(plan.p) << ", "
            << disc_plan_num_kernels(plan.p) << " kernels, " << disc_plan_host_instruction_count(plan.p)
            << " host instructions)\n";
  return 0;
}

int do_run(const Parsed& a) {
  const std::string file = a.pos.at("file");
  const auto binding = load_inputs(a.opt.count("input") ? a.opt.at("input") : std::vector<std::string>{});
  const bool eager = a.on("eager");
  Plan plan;
  if (eager)  // unfused: one launch per op (the reference interprets the graph eagerly)
    check(disc_compile_graph(slurp(file).c_str(), 1, 0, 0, &plan.p));
  else
    check(disc_plan_from_json(slurp(file).c_str(), &plan.p));
  int64_t stats[7] = {};
  const auto outs = run_plan(plan.p, binding, stats);
  if (!eager) {
    Session s(a.get("stats-file"));
    s.merge_run(stats);
    s.save();
  }
  const std::string out_dir = a.get("out-dir");
  for (size_t i = 0; i < outs.size(); ++i) {
    const std::string id = disc_plan_output_name(plan.p, static_cast<int>(i));
    std::cout << "output " << id << " shape=" << outs[i].shape_str() << "\n";
    if (!out_dir.empty()) {
      std::filesystem::create_directories(out_dir);
      write_tensor(out_dir + "/" + id + ".tensor", outs[i]);
    }
  }
  return 0;
}

double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

int do_bench(const Parsed& a) {
  Plan plan;
  check(disc_plan_from_json(slurp(a.pos.at("plan")).c_str(), &plan.p));
  json shapes;
  try {
    shapes = json::parse(slurp(a.get("shapes")));
  } catch (const json::exception& e) {
    usage_error(std::string("--shapes file is not JSON: ") + e.what());
  }
  if (!shapes.is_array()) usage_error("--shapes file must be a JSON array");
  int reps = 20;
  try {
    reps = std::max(std::stoi(a.get("reps", "20")), 20);
  } catch (const std::exception&) {
    usage_error("--reps expects an integer");
  }
  const bool as_json = a.on("json");
  std::cout << "note: timings are B200 device-executor medians (inputs resident in HBM); they are not\n"
               "comparable with the CPU reference executor's.\n";
  Exec ex;
  check(disc_executor_set_timing(ex.e, 1));
  json report = json::array();
  int64_t last[7] = {};
  const int64_t eager_ops = disc_plan_eager_op_count(plan.p);
  for (size_t si = 0; si < shapes.size(); ++si) {
    const auto binding = synth_inputs(plan.p, shapes[si], 0x9E3779B9u + si);
    std::vector<DeviceBuffer> bufs(binding.size());
    std::vector<const char*> names;
    std::vector<const void*> data;
    std::vector<const int64_t*> dims;
    std::vector<int> ranks;
    size_t k = 0;
    for (const auto& [id, t] : binding) {
      const size_t bytes = t.data.size() * 4;
      if (bytes) {
        if (disc_cuda_malloc(bytes, nullptr, &bufs[k].ptr) != 0 ||
            disc_cuda_memcpy(bufs[k].ptr, t.data.data(), bytes, 0 | DISC_MEMCPY_NOW, nullptr) != 0)
          runtime_error(std::string("input upload: ") + disc_cuda_last_error());
      }
      names.push_back(id.c_str());
      data.push_back(bufs[k++].ptr);
      dims.push_back(t.dims.data());
      ranks.push_back(static_cast<int>(t.dims.size()));
    }
    check(disc_cuda_stream_synchronize(nullptr));
    std::vector<double> wall, host, kernel;
    for (int r = 0; r < reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      check(disc_executor_run(ex.e, plan.p, static_cast<int>(names.size()), names.data(), data.data(), dims.data(),
                              ranks.data(), 0));
      check(disc_executor_synchronize(ex.e));
      wall.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
      double ms[2];
      check(disc_executor_stats(ex.e, last, ms));
      host.push_back(ms[0]);
      kernel.push_back(ms[1]);
    }
    const double ratio = eager_ops > 0 ? static_cast<double>(last[0] + last[1]) / static_cast<double>(eager_ops) : 0.0;
    if (as_json) {
      report.push_back(json{{"binding", shapes[si]},
                            {"wall_ms", median(wall)},
                            {"host_ms", median(host)},
                            {"kernel_ms", median(kernel)},
                            {"launch_count", last[0]},
                            {"library_calls", last[1]},
                            {"eager_op_count", eager_ops},
                            {"launch_ratio", ratio}});
    } else {
      std::cout << "shape " << shapes[si].dump() << " wall_ms=" << median(wall) << " host_ms=" << median(host)
                << " kernel_ms=" << median(kernel) << " launch_count=" << last[0] << " library_calls=" << last[1]
                << " eager_op_count=" << eager_ops << " launch_ratio=" << ratio << "\n";
    }
  }
  if (as_json) std::cout << report.dump(2) << "\n";
  Session s(a.get("stats-file"));
  s.merge_run(last);
  s.save();
  return 0;
}

int do_dump_ir(const Parsed& a) {
  const std::string stage = a.get("stage");
  if (std::find(kStages.begin(), kStages.end(), stage) == kStages.end())
    usage_error("unknown stage " + stage + " (dhlo|constraints|simplified|fused|program)");
  const std::string graph = slurp(a.pos.at("graph"));
  const CompileFlags f = compile_flags(a);
  char* text = nullptr;
  check(disc_dump_stage(graph.c_str(), f.inject, f.fusion, stage.c_str(), &text));
  dump_dir_stages(graph, f);
  std::cout << text;
  disc_free(text);
  return 0;
}

int do_stats(const Parsed& a) {
  const Session s(a.get("stats-file"));
  static const char* keys[] = {"compile_count", "cache_hits",  "launch_count",
                               "library_calls", "peak_bytes",  "host_instruction_count",
                               "alloc_calls",   "allocator_cache_hits", "aliased_allocs"};
  if (a.on("json")) {
    json out = json::object();
    for (const char* k : keys) out[k] = s.j.value(k, int64_t{0});
    std::cout << out.dump(2) << "\n";
  } else {
    for (const char* k : keys) std::cout << k << "=" << s.j.value(k, int64_t{0}) << "\n";
  }
  return 0;
}

struct Command {
  const char* name;
  const char* help;
  Spec spec;
  int (*fn)(const Parsed&);
};

std::vector<Command> commands() {
  const std::map<std::string, std::string> stats_opt = {{"--stats-file", "stats-file"}};
  auto with = [](std::map<std::string, std::string> m, const std::map<std::string, std::string>& more) {
    m.insert(more.begin(), more.end());
    return m;
  };
  return {
      {"compile", "compile a graph JSON into a plan",
       {{"graph"},
        {{"--static-fallback", "static-fallback"}, {"--no-injected-constraints", "no-injected-constraints"},
         {"--no-fusion", "no-fusion"}},
        with({{"-o", "output"}, {"--output", "output"}}, stats_opt)},
       do_compile},
      {"run", "execute a plan (or a graph unfused with --eager) on the GPU",
       {{"file"}, {{"--eager", "eager"}}, with({{"--input", "input"}, {"--out-dir", "out-dir"}}, stats_opt)},
       do_run},
      {"bench", "run a plan over a list of shape bindings",
       {{"plan"}, {{"--json", "json"}}, with({{"--shapes", "shapes"}, {"--reps", "reps"}}, stats_opt)},
       do_bench},
      {"dump-ir", "print one pipeline stage",
       {{"graph"}, {{"--no-injected-constraints", "no-injected-constraints"}, {"--no-fusion", "no-fusion"}},
        {{"--stage", "stage"}}},
       do_dump_ir},
      {"stats", "print session stats as key=value", {{}, {{"--json", "json"}}, stats_opt}, do_stats},
  };
}

void print_help(const std::vector<Command>& cmds) {
  std::cout << "disc: dynamic-shape fused-kernel compiler (B200 executor)\n"
               "usage: disc <command> [args]\n";
  for (const auto& c : cmds) std::cout << "  " << c.name << "\t" << c.help << "\n";
}

}  // namespace

int main(int argc, char** argv) {
  const auto cmds = commands();
  if (argc >= 2 && (!std::strcmp(argv[1], "-h") || !std::strcmp(argv[1], "--help"))) {
    print_help(cmds);
    return 0;
  }
  try {
    if (argc < 2) usage_error("a subcommand is required (compile|run|bench|dump-ir|stats)");
    for (const auto& c : cmds) {
      if (std::strcmp(argv[1], c.name) != 0) continue;
      for (int i = 2; i < argc; ++i)
        if (!std::strcmp(argv[i], "-h") || !std::strcmp(argv[i], "--help")) {
          std::cout << "disc " << c.name << ": " << c.help << "\n";
          return 0;
        }
      const Parsed p = parse_args(c.spec, argc, argv, 2);
      if (!std::strcmp(c.name, "bench") && !p.has("shapes")) usage_error("--shapes is required");
      if (!std::strcmp(c.name, "dump-ir") && !p.has("stage")) usage_error("--stage is required");
      return c.fn(p);
    }
    usage_error(std::string("unknown subcommand ") + argv[1]);
  } catch (const Failure& f) {
    std::cerr << f.line << "\n";
    return f.code;
  } catch (const std::exception& e) {
    std::cerr << "error[internal]: " << e.what() << "\n";
    return 4;
  }
}
