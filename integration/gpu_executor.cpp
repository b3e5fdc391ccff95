// The reference-side binding a maintainer adds to put the reference's runtime on B200:
// a replacement for the reference's src/executor.cpp that implements the same
// declarations (include/disc/executor.hpp:74-95) over libdisc_b200.so's C ABI.
//
//   disc::Executor::run   (executor.hpp:79; reference body executor.cpp:221-465)
//       -> disc_executor_run(inputs_on_host=1) + disc_executor_{output,copy_output,stats,event}
//   disc::run_kernel      (executor.hpp:87-89; reference body executor.cpp:137-219)
//       -> disc_executor_run_kernel on device copies of the externals
//   disc::guard_passes    (executor.hpp:92-93; executor.cpp:78-98) -> disc_guard_passes
//   disc::resolve_ref     (executor.hpp:95; executor.cpp:46-51)    -> the register read
//
// Build (integration/Makefile): every reference source except src/executor.cpp, plus this
// file, linked with -ldisc_b200.  Nothing else in the reference changes -- its tests
// (tests/acceptance_main.cpp) construct `Executor` and call `run_kernel` exactly as
// before, and now run on the GPU.  Plans cross the boundary as the reference's own plan
// JSON (plan_to_json), which disc_plan_from_json reads byte-compatibly.
//
// Not part of the B200 package: it is written against the reference's headers.

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <list>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "disc/error.hpp"
#include "disc/executor.hpp"
#include "disc/runtime_program.hpp"
#include "disc_b200.h"
#include "disc_cuda.h"

namespace disc {
namespace {

// C ABI status -> the reference's exception classes (error.hpp:25-63), with the bare
// reference message (disc_last_error() carries "error[<class>]: <message>").
void check(int rc) {
  if (rc == 0) return;
  std::string msg = disc_last_error();
  const std::string::size_type p = msg.find("]: ");
  if (msg.rfind("error[", 0) == 0 && p != std::string::npos) msg = msg.substr(p + 3);
  switch (static_cast<ErrorClass>(disc_last_error_class())) {
    case ErrorClass::kParse: throw ParseError(msg);
    case ErrorClass::kValidation: throw ValidationError(msg);
    case ErrorClass::kCompile: throw CompileError(msg);
    case ErrorClass::kRuntime: throw RuntimeError(msg);
    default: throw InternalError(msg);
  }
}

void cuda(int rc, const char* what) {
  if (rc != 0) throw RuntimeError(std::string(what) + ": " + disc_cuda_last_error());
}

int device_ordinal() {
  static const int dev = [] {
    const char* e = std::getenv("DISC_DEVICE");
    return e ? std::atoi(e) : 0;
  }();
  return dev;
}

// One device executor per host thread: the reference's contract is one Executor per
// thread (executor.hpp:74-76) and runs on a thread are sequential, so every
// disc::Executor object of a thread shares it (its caching allocator persists like the
// reference's).  Destroyed at thread exit.
struct ThreadExecutor {
  disc_executor e = nullptr;
  void* stream = nullptr;
  ~ThreadExecutor() {
    if (e) disc_executor_destroy(e);
    if (stream) disc_cuda_stream_destroy(stream);
  }
  disc_executor get() {
    if (!e) {
      cuda(disc_cuda_set_device(device_ordinal()), "set device");
      cuda(disc_cuda_stream_create(&stream), "stream");
      check(disc_executor_create(device_ordinal(), stream, &e));
    }
    return e;
  }
};
thread_local ThreadExecutor t_exec;

// Plan handles keyed by the plan's JSON bytes (a CompiledPlan has no identity of its own
// that survives copies), bounded LRU per thread.
class PlanCache {
 public:
  ~PlanCache() {
    for (auto& [_, h] : order_) disc_plan_release(h);
  }
  disc_plan get(const CompiledPlan& plan) {
    std::string text = plan_to_json(plan);
    auto it = index_.find(text);
    if (it != index_.end()) {
      order_.splice(order_.begin(), order_, it->second);
      return it->second->second;
    }
    disc_plan h = nullptr;
    check(disc_plan_from_json(text.c_str(), &h));
    order_.emplace_front(text, h);
    index_[order_.front().first] = order_.begin();
    if (order_.size() > kMax) {
      index_.erase(order_.back().first);
      disc_plan_release(order_.back().second);
      order_.pop_back();
    }
    return h;
  }

 private:
  static constexpr size_t kMax = 64;
  std::list<std::pair<std::string, disc_plan>> order_;
  std::unordered_map<std::string, std::list<std::pair<std::string, disc_plan>>::iterator> index_;
};
thread_local PlanCache t_plans;

ConcreteTensor fetch_output(disc_executor e, int i) {
  const float* dptr = nullptr;
  const int64_t* d = nullptr;
  int rank = 0;
  check(disc_executor_output(e, i, &dptr, &d, &rank));
  ConcreteTensor t = ConcreteTensor::zeros_f32(std::vector<int64_t>(d, d + rank));
  if (!t.f32.empty()) check(disc_executor_copy_output(e, i, t.f32.data(), /*dst_on_host=*/1));
  return t;
}

// Device copies of host tensors for run_kernel (released when it returns).
struct DeviceStaging {
  void* stream;
  std::vector<void*> ptrs;
  explicit DeviceStaging(void* s) : stream(s) {}
  ~DeviceStaging() {
    disc_cuda_stream_synchronize(stream);
    for (void* p : ptrs) disc_cuda_free(p, stream);
  }
  const float* put(const ConcreteTensor& t) {
    const size_t bytes = t.f32.size() * sizeof(float);
    void* p = nullptr;
    cuda(disc_cuda_malloc(bytes ? bytes : 16, stream, &p), "device allocation");
    ptrs.push_back(p);
    if (bytes) cuda(disc_cuda_memcpy(p, t.f32.data(), bytes, /*h2d*/ 0, stream), "h2d");
    return static_cast<const float*>(p);
  }
};

}  // namespace

ExecResult Executor::run(const CompiledPlan& plan, const Binding& inputs) {
  disc_executor e = t_exec.get();
  disc_plan p = t_plans.get(plan);
  std::vector<const char*> names;
  std::vector<const void*> data;
  std::vector<const int64_t*> dims;
  std::vector<int> ranks;
  for (const auto& [name, t] : inputs) {  // Binding = map<string, ConcreteTensor>
    names.push_back(name.c_str());
    data.push_back(t.f32.data());
    dims.push_back(t.dims.data());
    ranks.push_back(static_cast<int>(t.dims.size()));
  }
  check(disc_executor_run(e, p, static_cast<int>(names.size()), names.data(), data.data(), dims.data(),
                          ranks.data(), /*inputs_on_host=*/1));
  ExecResult r;
  for (int i = 0; i < disc_executor_num_outputs(e); ++i) r.outputs.push_back(fetch_output(e, i));
  int64_t s[7];
  double ms[2];
  check(disc_executor_stats(e, s, ms));
  r.stats.launch_count = s[0];
  r.stats.library_calls = s[1];
  r.stats.host_instruction_count = s[2];
  r.stats.peak_bytes = s[3];
  r.stats.alloc_calls = s[4];
  r.stats.allocator_cache_hits = s[5];
  r.stats.aliased_allocs = s[6];
  r.stats.host_ms = ms[0];
  r.stats.kernel_ms = ms[1];
  for (int i = 0; i < disc_executor_num_events(e); ++i) {
    int four[4];
    check(disc_executor_event(e, i, four));
    r.buffer_events.push_back({four[0], four[1], four[2], four[3]});
  }
  return r;
}

std::vector<ConcreteTensor> run_kernel(const KernelArtifact& art, const VersionArtifact& version,
                                       const std::vector<const ConcreteTensor*>& externals,
                                       const std::vector<int64_t>& regs) {
  disc_executor e = t_exec.get();
  CompiledPlan holder;  // the artifact crosses as a one-kernel plan
  holder.kernels.push_back(art);
  disc_plan p = t_plans.get(holder);
  DeviceStaging staged(t_exec.stream);
  std::vector<const float*> ext;
  std::vector<const int64_t*> dims;
  std::vector<int> ranks;
  for (const ConcreteTensor* t : externals) {
    ext.push_back(staged.put(*t));
    dims.push_back(t->dims.data());
    ranks.push_back(static_cast<int>(t->dims.size()));
  }
  check(disc_executor_run_kernel(e, p, 0, version.id, static_cast<int>(ext.size()), ext.data(), dims.data(),
                                 ranks.data(), regs.data(), static_cast<int>(regs.size())));
  std::vector<ConcreteTensor> out;
  for (int i = 0; i < disc_executor_num_outputs(e); ++i) out.push_back(fetch_output(e, i));
  return out;
}

bool guard_passes(const KernelArtifact& art, const VersionArtifact& version, const std::vector<int64_t>& regs) {
  CompiledPlan holder;
  holder.kernels.push_back(art);
  const int rc = disc_guard_passes(t_plans.get(holder), 0, version.id, regs.data(), static_cast<int>(regs.size()));
  if (rc < 0) check(rc);
  return rc == 1;
}

int64_t resolve_ref(const ScalarRef& r, const std::vector<int64_t>& regs) {
  if (r.is_const) return r.value;
  if (r.reg < 0 || r.reg >= static_cast<int>(regs.size())) throw InternalError("shape register out of range");
  return regs[static_cast<size_t>(r.reg)];
}

}  // namespace disc
