// C ABI, runtime side: executors over a device + stream (include/disc_b200.h).
#include <chrono>
#include <cstring>

#include "capi_common.hpp"
#include "disc_cuda.h"
#include "runtime/runtime_flow.hpp"
#include "runtime/launcher.hpp"
#include "runtime/shape_eval.hpp"

using namespace disc;
using disc_capi::guard;

namespace disc::rt {
struct PreparedPlan {};  // per-plan device lowering cache (launch binding is per shape)
std::shared_ptr<const PreparedPlan> prepare_plan(const CompiledPlan&) { return std::make_shared<PreparedPlan>(); }
}  // namespace disc::rt

struct disc_executor_s {
  disc_executor_s(int device, void* stream) : ex(device, stream) {}
  rt::DeviceExecutor ex;
};

namespace {
int64_t bytes_of(const int64_t* dims, int rank) {
  int64_t n = 1;
  for (int i = 0; i < rank; ++i) n *= dims[i];
  return n * 4;
}
}  // namespace

extern "C" {

int disc_executor_create(int device, void* stream, disc_executor* out) {
  return guard([&] {
    int n = 0;
    if (disc_cuda_device_count(&n) != 0 || n == 0)
      throw RuntimeError(std::string("no CUDA device available: ") + disc_cuda_last_error());
    *out = new disc_executor_s(device, stream);
  });
}

void disc_executor_destroy(disc_executor e) { delete e; }

int disc_executor_set_stream(disc_executor e, void* stream) {
  return guard([&] { e->ex.set_stream(stream); });
}

int disc_executor_run(disc_executor e, disc_plan p, int n, const char* const* names, const void* const* data,
                      const int64_t* const* dims, const int* ranks, int on_host) {
  return guard([&] {
    std::vector<rt::InputBinding> in(n);
    for (int i = 0; i < n; ++i) {
      in[i].name = names[i];
      in[i].dims.assign(dims[i], dims[i] + ranks[i]);
      in[i].ptr = on_host ? e->ex.stage_input(i, data[i], bytes_of(dims[i], ranks[i]))
                          : static_cast<const float*>(data[i]);
    }
    e->ex.run(*p->plan, in, false, p->serial);
  });
}

int disc_executor_run_batch(disc_executor e, disc_plan p, int n_requests, int n_inputs, const char* const* names,
                            const void* const* data, const int64_t* const* dims, const int* ranks, int on_host) {
  return guard([&] {
    std::vector<rt::InputBinding> in(n_inputs);
    for (int r = 0; r < n_requests; ++r) {
      for (int i = 0; i < n_inputs; ++i) {
        const int k = r * n_inputs + i;
        in[i].name = names[i];
        in[i].dims.assign(dims[k], dims[k] + ranks[k]);
        in[i].ptr = on_host ? e->ex.stage_input(i, data[k], bytes_of(dims[k], ranks[k]))
                            : static_cast<const float*>(data[k]);
      }
      e->ex.run(*p->plan, in, r > 0, p->serial);
    }
  });
}

int disc_executor_run_stream(disc_executor e, int n_requests, const disc_plan* plans, const int* input_offsets,
                             const char* const* names, const void* const* data, const int64_t* const* dims,
                             const int* ranks, int on_host) {
  return guard([&] {
    std::vector<rt::InputBinding> in;
    for (int r = 0; r < n_requests; ++r) {
      const int i0 = input_offsets[r], n = input_offsets[r + 1] - i0;
      in.resize(n);
      for (int i = 0; i < n; ++i) {
        const int k = i0 + i;
        in[i].name = names[k];
        in[i].dims.assign(dims[k], dims[k] + ranks[k]);
        in[i].ptr = on_host ? e->ex.stage_input(i, data[k], bytes_of(dims[k], ranks[k]))
                            : static_cast<const float*>(data[k]);
      }
      e->ex.run(*plans[r]->plan, in, r > 0, plans[r]->serial);
    }
  });
}

int disc_executors_run_interleaved(const disc_executor* exs, int n_exec, int n_requests, const int* which,
                                   const disc_plan* plans, const int* input_offsets, const char* const* names,
                                   const void* const* data, const int64_t* const* dims, const int* ranks,
                                   int on_host) {
  return guard([&] {
    std::vector<rt::InputBinding> in;
    std::vector<char> started(n_exec, 0);
    for (int r = 0; r < n_requests; ++r) {
      const int x = which[r];
      if (x < 0 || x >= n_exec) throw disc::Error(disc::ErrorClass::kUsage, "executor index out of range");
      disc_executor e = exs[x];
      const int i0 = input_offsets[r], n = input_offsets[r + 1] - i0;
      in.resize(n);
      for (int i = 0; i < n; ++i) {
        const int k = i0 + i;
        in[i].name = names[k];
        in[i].dims.assign(dims[k], dims[k] + ranks[k]);
        in[i].ptr = on_host ? e->ex.stage_input(i, data[k], bytes_of(dims[k], ranks[k]))
                            : static_cast<const float*>(data[k]);
      }
      e->ex.run(*plans[r]->plan, in, started[x] != 0, plans[r]->serial);
      started[x] = 1;
    }
  });
}

int disc_executor_run_grouped(disc_executor e, int n_requests, const disc_plan* plans, const int* input_offsets,
                              const char* const* names, const void* const* data, const int64_t* const* dims,
                              const int* ranks, int on_host) {
  return guard([&] {
    std::vector<const CompiledPlan*> ps(n_requests);
    std::vector<uint64_t> serials(n_requests);
    for (int r = 0; r < n_requests; ++r) {
      ps[r] = plans[r]->plan.get();
      serials[r] = plans[r]->serial;
    }
    e->ex.run_grouped_batch(n_requests, ps.data(), serials.data(), input_offsets, names, data, dims, ranks,
                            on_host != 0);
  });
}

int disc_executor_set_graphs(disc_executor e, int on) {
  return guard([&] { e->ex.set_graphs(on != 0); });
}

int64_t disc_executor_graph_replays(disc_executor e) { return e->ex.graph_replays(); }

int disc_executor_set_host_threads(disc_executor e, int n) {
  return guard([&] {
    e->ex.wait_issued();
    e->ex.set_host_threads(n);
  });
}

int disc_executor_num_requests(disc_executor e) { return static_cast<int>(e->ex.request_outputs().size()); }

int disc_executor_num_request_outputs(disc_executor e, int r) {
  const auto& ro = e->ex.request_outputs();
  return r >= 0 && r < static_cast<int>(ro.size()) ? static_cast<int>(ro[r].size()) : -1;
}

int disc_executor_request_output(disc_executor e, int r, int i, const float** dptr, const int64_t** dims, int* rank) {
  return guard([&] {
    const auto& o = e->ex.request_outputs().at(r).at(i);
    *dptr = o.ptr;
    *dims = o.dims.data();
    *rank = static_cast<int>(o.dims.size());
  });
}

int disc_executor_copy_request_output(disc_executor e, int r, int i, void* dst, int dst_on_host) {
  return guard([&] {
    e->ex.wait_issued();
    const auto& o = e->ex.request_outputs().at(r).at(i);
    int64_t n = 1;
    for (int64_t d : o.dims) n *= d;
    if (n == 0) return;
    if (disc_cuda_memcpy(dst, o.ptr, static_cast<size_t>(n * 4), dst_on_host ? 1 : 2, e->ex.stream()) != 0)
      throw RuntimeError(std::string("output copy: ") + disc_cuda_last_error());
    if (dst_on_host == 1 && disc_cuda_stream_synchronize(e->ex.stream()) != 0)
      throw RuntimeError(std::string("stream sync: ") + disc_cuda_last_error());
  });
}

int disc_executor_request_stats(disc_executor e, int r, int64_t* s7) {
  return guard([&] {
    const auto& s = e->ex.request_stats().at(r);
    int64_t v[7] = {s.launch_count, s.library_calls, s.host_instruction_count, s.peak_bytes,
                    s.alloc_calls, s.allocator_cache_hits, s.aliased_allocs};
    std::memcpy(s7, v, sizeof v);
  });
}

int disc_executor_num_outputs(disc_executor e) { return static_cast<int>(e->ex.outputs().size()); }

int disc_executor_output(disc_executor e, int i, const float** dptr, const int64_t** dims, int* rank) {
  return guard([&] {
    const auto& o = e->ex.outputs().at(i);
    *dptr = o.ptr;
    *dims = o.dims.data();
    *rank = static_cast<int>(o.dims.size());
  });
}

int disc_executor_copy_output(disc_executor e, int i, void* dst, int dst_on_host) {
  return guard([&] {
    e->ex.wait_issued();
    const auto& o = e->ex.outputs().at(i);
    int64_t n = 1;
    for (int64_t d : o.dims) n *= d;
    if (n == 0) return;
    if (disc_cuda_memcpy(dst, o.ptr, static_cast<size_t>(n * 4), dst_on_host ? 1 : 2, e->ex.stream()) != 0)
      throw RuntimeError(std::string("output copy: ") + disc_cuda_last_error());
    if (dst_on_host == 1 && disc_cuda_stream_synchronize(e->ex.stream()) != 0)
      throw RuntimeError(std::string("stream sync: ") + disc_cuda_last_error());
  });
}

int disc_executor_synchronize(disc_executor e) {
  return guard([&] {
    e->ex.wait_issued();
    if (disc_cuda_stream_synchronize(e->ex.stream()) != 0)
      throw RuntimeError(std::string("device error: ") + disc_cuda_last_error());
  });
}

int disc_executor_stats(disc_executor e, int64_t* s7, double* ms2) {
  e->ex.finish_timing();
  const auto& s = e->ex.stats();
  int64_t v[7] = {s.launch_count, s.library_calls, s.host_instruction_count, s.peak_bytes,
                  s.alloc_calls, s.allocator_cache_hits, s.aliased_allocs};
  std::memcpy(s7, v, sizeof v);
  if (ms2) {
    ms2[0] = s.host_ms;
    ms2[1] = s.kernel_ms;
  }
  return 0;
}

int disc_executor_num_events(disc_executor e) { return static_cast<int>(e->ex.events().size()); }

int disc_executor_event(disc_executor e, int i, int* four) {
  const auto& ev = e->ex.events().at(i);
  four[0] = ev.logical;
  four[1] = ev.physical;
  four[2] = ev.alloc_instr;
  four[3] = ev.dealloc_instr;
  return 0;
}

int64_t disc_executor_device_launches(disc_executor e) { return e->ex.device_launches(); }

int disc_executor_num_records(disc_executor e) {
  e->ex.finish_timing();
  return static_cast<int>(e->ex.launch_records().size());
}

int disc_executor_record(disc_executor e, int i, int* instr, int* kernel, int64_t* bytes, double* ms,
                         int* device_kernels, const char** schedule) {
  return guard([&] {
    const auto& r = e->ex.launch_records().at(i);
    *instr = r.instr;
    *kernel = r.kernel;
    *bytes = r.bytes;
    *ms = r.ms;
    *device_kernels = r.device_kernels;
    *schedule = r.schedule.c_str();
  });
}

int64_t disc_executor_algorithmic_bytes(disc_executor e) { return e->ex.algorithmic_bytes(); }

int disc_executor_set_timing(disc_executor e, int enabled) {
  return guard([&] {
    e->ex.wait_issued();
    e->ex.set_timing(enabled != 0);
  });
}

int disc_executor_set_async_flush(disc_executor e, int on) {
  return guard([&] { e->ex.set_async_flush(on != 0); });
}

int disc_executor_wait_issued(disc_executor e) {
  return guard([&] { e->ex.wait_issued(); });
}

int disc_executor_set_schedule(disc_executor e, const char* s) {
  return guard([&] {
    std::string v = s ? s : "auto";
    rt::SchedulePref p;
    if (v == "auto") p = rt::SchedulePref::kAuto;
    else if (v == "materialize") p = rt::SchedulePref::kMaterialize;
    else if (v == "fused") p = rt::SchedulePref::kFusedOnly;
    else if (v == "twopass") p = rt::SchedulePref::kTwoPass;
    else if (v == "atomic") p = rt::SchedulePref::kAtomic;
    else throw Error(ErrorClass::kUsage, "unknown schedule " + v);
    e->ex.set_schedule(p);
  });
}

int disc_executor_set_cache_budget(disc_executor e, int64_t bytes) {
  e->ex.set_cache_budget(bytes);
  return 0;
}

int disc_executor_reserve(disc_executor e, int64_t bytes) {
  return guard([&] { e->ex.reserve(bytes); });
}

int disc_executor_run_kernel(disc_executor e, disc_plan p, int kernel, int version, int n_ext, const float* const* ext,
                             const int64_t* const* ext_dims, const int* ext_ranks, const int64_t* regs, int n_regs) {
  return guard([&] {
    const KernelArtifact& art = p->plan->kernels.at(kernel);
    const VersionArtifact* v = nullptr;
    for (const auto& x : art.versions)
      if (x.id == version) v = &x;
    if (!v) throw InternalError("no such version");
    std::vector<rt::DevTensor> ex;
    for (int i = 0; i < n_ext; ++i) ex.push_back({ext[i], std::vector<int64_t>(ext_dims[i], ext_dims[i] + ext_ranks[i])});
    e->ex.run_kernel(art, *v, ex, std::vector<int64_t>(regs, regs + n_regs));
  });
}

int disc_plan_capture_programs(disc_plan p, int n, const char* const* names, const int64_t* const* dims,
                               const int* ranks, char** json) {
  disc_cuda_set_capture(1);
  int rc = guard([&] {
    rt::DeviceExecutor ex(0, nullptr);
    std::vector<rt::InputBinding> in(n);
    for (int i = 0; i < n; ++i) {
      in[i].name = names[i];
      in[i].dims.assign(dims[i], dims[i] + ranks[i]);
      void* fake = nullptr;
      disc_cuda_malloc(static_cast<size_t>(bytes_of(dims[i], ranks[i])), nullptr, &fake);
      in[i].ptr = static_cast<const float*>(fake);
    }
    ex.run(*p->plan, in);
    disc_cuda_capture_records(json);
  });
  disc_cuda_set_capture(0);
  return rc;
}

int disc_plan_group_dry_run(int n_requests, const disc_plan* plans, const int* input_offsets, const char* const* names,
                            const int64_t* const* dims, const int* ranks, int host_threads, char** json) {
  disc_cuda_set_capture(1);
  int rc = guard([&] {
    rt::DeviceExecutor ex(0, nullptr);
    ex.set_host_threads(host_threads);
    const int total = input_offsets[n_requests];
    std::vector<const void*> data(std::max(total, 1));
    for (int k = 0; k < total; ++k) {
      void* fake = nullptr;
      disc_cuda_malloc(static_cast<size_t>(bytes_of(dims[k], ranks[k])), nullptr, &fake);
      data[k] = fake;
    }
    std::vector<const CompiledPlan*> ps(n_requests);
    std::vector<uint64_t> serials(n_requests);
    for (int r = 0; r < n_requests; ++r) {
      ps[r] = plans[r]->plan.get();
      serials[r] = plans[r]->serial;
    }
    disc_cuda_set_capture(2);  // launches unrecorded (mode 2): the output is only the flush plan
    ex.run_grouped_batch(n_requests, ps.data(), serials.data(), input_offsets, names, data.data(), dims, ranks, false);
    disc_cuda_capture_records(json);
  });
  disc_cuda_set_capture(0);
  return rc;
}

int disc_plan_host_overhead(disc_plan p, int n, const char* const* names, const int64_t* const* dims,
                            const int* ranks, int iters, double* us_per_run) {
  disc_cuda_set_capture(2);
  int rc = guard([&] {
    rt::DeviceExecutor ex(0, nullptr);
    std::vector<rt::InputBinding> in(n);
    for (int i = 0; i < n; ++i) {
      in[i].name = names[i];
      in[i].dims.assign(dims[i], dims[i] + ranks[i]);
      void* fake = nullptr;
      disc_cuda_malloc(static_cast<size_t>(bytes_of(dims[i], ranks[i])), nullptr, &fake);
      in[i].ptr = static_cast<const float*>(fake);
    }
    ex.run(*p->plan, in, false, p->serial);
    auto t0 = std::chrono::steady_clock::now();
    for (int k = 0; k < iters; ++k) ex.run(*p->plan, in, false, p->serial);
    *us_per_run = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / iters;
  });
  disc_cuda_set_capture(0);
  return rc;
}

int disc_plan_algorithmic_bytes(disc_plan p, int n, const char* const* names, const int64_t* const* dims,
                                const int* ranks, int64_t* bytes) {
  return guard([&] {
    const CompiledPlan& plan = *p->plan;
    std::vector<rt::InputBinding> in(n);
    for (int i = 0; i < n; ++i) {
      in[i].name = names[i];
      in[i].dims.assign(dims[i], dims[i] + ranks[i]);
    }
    const std::vector<int64_t> regs = disc_capi::eval_shape_program(plan, [&] {
      std::vector<std::vector<int64_t>> d(plan.inputs.size());
      for (size_t k = 0; k < plan.inputs.size(); ++k)
        for (const auto& b : in)
          if (b.name == plan.inputs[k].id) d[k] = b.dims;
      return d;
    }());
    int64_t total = 0;
    for (const auto& ins : plan.instrs) {
      if (ins.kind == InstrKind::kLaunch) {
        const KernelArtifact& art = plan.kernels.at(ins.a);
        const VersionArtifact* ver = nullptr;
        for (const auto& v : art.versions)
          if (ins.fixed_version >= 0 ? v.id == ins.fixed_version
                                     : disc_guard_passes(p, ins.a, v.id, regs.data(), static_cast<int>(regs.size())) == 1) {
            ver = &v;
            break;
          }
        if (!ver) throw RuntimeError("no kernel version guard matched");
        std::vector<std::vector<int64_t>> ext;
        for (const auto& d : art.external_input_dims) ext.push_back(rt::resolve_all(d, regs));
        total += rt::launch_bytes_estimate(art, *ver, ext, regs);
      } else if (ins.kind == InstrKind::kLibraryCall) {
        const int64_t m = rt::resolve(ins.lib_dims[0], regs), k = rt::resolve(ins.lib_dims[1], regs),
                      q = rt::resolve(ins.lib_dims[2], regs);
        total += 4 * (m * k + k * q + m * q);
      }
    }
    *bytes = total;
  });
}

int disc_guard_passes(disc_plan p, int kernel, int version, const int64_t* regs, int n_regs) {
  const KernelArtifact& art = p->plan->kernels.at(kernel);
  std::vector<int64_t> r(regs, regs + n_regs);
  for (const auto& v : art.versions) {
    if (v.id != version) continue;
    for (const auto& g : v.guards) {
      if (g.kind == GuardTest::Kind::kNever) return 0;
      if (g.kind == GuardTest::Kind::kRefEqual && rt::resolve(g.a, r) != rt::resolve(g.b, r)) return 0;
      if (g.kind == GuardTest::Kind::kTotalDivisibleBy4) {
        int64_t total = 1;
        for (const auto& d : art.space_dims) total *= rt::resolve(d, r);
        if (total % 4 != 0) return 0;
      }
    }
    return 1;
  }
  return -1;
}

}  // extern "C"
