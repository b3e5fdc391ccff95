// C ABI of the device layer (include/disc_cuda.h): streams, stream-ordered memory,
// events and the kernel launches the runtime flow issues.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "disc_cuda.h"
#include "../kernels/program.cuh"

namespace disc_launch {
cudaError_t loop(const disc_loop_launch& L, cudaStream_t s);
cudaError_t reduce(const disc_reduce_launch& L, cudaStream_t s);
cudaError_t col_pass(const disc_reduce_launch& L, cudaStream_t s);
cudaError_t finalize_columns(const disc_reduce_launch& L, cudaStream_t s);
cudaError_t pad(const disc_pad_launch& P, cudaStream_t s);
cudaError_t concat(const disc_concat_launch& C, cudaStream_t s);
cudaError_t gemm(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c, cudaStream_t s);
cudaError_t fill_uniform(float* dst, int64_t n, uint64_t seed, float lo, float hi, cudaStream_t s);
cudaError_t flush(void* p, size_t bytes, cudaStream_t s);
cudaError_t spin(uint64_t ns, cudaStream_t s);
void set_pdl(int mode);
int pdl_mode();
}  // namespace disc_launch

// Generated fast paths (patterns_gen.cu): straight-line kernels for known program
// structures, keyed by (schedule kind, structural hash of the lowered program).
namespace disc_spec {
struct Entry {
  int kind;        // 0 loop, 1 row (pre+post), 2 column pass (pre)
  uint64_t key;
  cudaError_t (*launch)(const void* launch, int vec, cudaStream_t s);
};
const Entry* lookup(int kind, uint64_t key);
int count();
}  // namespace disc_spec

namespace {
thread_local std::string t_err;
std::atomic<int64_t> g_launches{0};
std::atomic<int64_t> g_spec_launches{0};
bool g_spec_enabled = true;

// Capture mode (host-only dry run used by the pattern generator): device calls become
// no-ops, allocations return fake aligned addresses, launches are recorded.
bool g_capture = false;
bool g_capture_record = true;  // capture mode 2: dry run without recording (host timing)
uint64_t g_fake_next = uint64_t{1} << 36;
std::vector<std::string> g_records;

uint64_t mix(uint64_t h, uint64_t v) {
  for (int i = 0; i < 8; ++i) {
    h ^= (v >> (8 * i)) & 0xff;
    h *= 1099511628211ull;
  }
  return h;
}

// Structure of a program: everything except pointers and load bindings.
uint64_t program_hash(const disc_program& P) {
  uint64_t h = 14695981039346656037ull;
  h = mix(h, P.n_instr);
  h = mix(h, P.n_slots);
  h = mix(h, P.n_loads);
  h = mix(h, P.n_outs);
  for (int i = 0; i < P.n_instr; ++i) {
    const disc_instr& I = P.code[i];
    const int op = I.op <= DISC_I_LOAD_CONST ? 0 : I.op;
    h = mix(h, (uint64_t)op | ((uint64_t)I.a << 8) | ((uint64_t)I.b << 16) | ((uint64_t)I.flags << 24) |
                   ((uint64_t)I.dst << 32) | ((uint64_t)I.load << 40) | ((uint64_t)I.out << 48));
  }
  for (int l = 0; l < P.n_loads; ++l) h = mix(h, 0x100 + disc_dev::load_class(P.loads[l]));
  return h;
}

std::string program_text(const disc_program& P) {
  std::string s = "{\"slots\":" + std::to_string(P.n_slots) + ",\"loads\":" + std::to_string(P.n_loads) +
                  ",\"outs\":" + std::to_string(P.n_outs) + ",\"code\":[";
  for (int i = 0; i < P.n_instr; ++i) {
    const disc_instr& I = P.code[i];
    const int op = I.op <= DISC_I_LOAD_CONST ? 0 : I.op;
    s += (i ? ",[" : "[") + std::to_string(op) + "," + std::to_string(I.a) + "," + std::to_string(I.b) + "," +
         std::to_string(I.flags) + "," + std::to_string(I.dst) + "," + std::to_string(I.load) + "," +
         std::to_string(I.out) + "]";
  }
  s += "],\"lclass\":[";
  for (int l = 0; l < P.n_loads; ++l) s += (l ? "," : "") + std::to_string(disc_dev::load_class(P.loads[l]));
  return s + "]}";
}

uint64_t launch_key(int kind, const disc_program& a, const disc_program* b) {
  uint64_t h = mix(1469598103934665603ull, kind);
  h = mix(h, program_hash(a));
  if (b) h = mix(h, program_hash(*b));
  return h;
}

void record(const std::string& kind, uint64_t key, const std::string& body) {
  if (!g_capture_record) return;
  char hex[32];
  std::snprintf(hex, sizeof hex, "%016llx", static_cast<unsigned long long>(key));
  g_records.push_back("{\"kind\":\"" + kind + "\",\"key\":\"" + hex + "\"," + body + "}");
}

int check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return 0;
  t_err = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return 4;
}
cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

int counted(cudaError_t e, const char* what, int n = 1) {
  if (e == cudaSuccess) g_launches.fetch_add(n, std::memory_order_relaxed);
  return check(e, what);
}
}  // namespace

extern "C" {

const char* disc_cuda_last_error(void) { return t_err.c_str(); }

int disc_cuda_device_count(int* n) {
  if (g_capture) {
    *n = 1;
    return 0;
  }
  return check(cudaGetDeviceCount(n), "cudaGetDeviceCount");
}
int disc_cuda_set_device(int device) {
  if (g_capture) return 0;
  return check(cudaSetDevice(device), "cudaSetDevice");
}

int disc_cuda_device_info(int device, int* sm_count, int64_t* l2_bytes, int64_t* hbm_bytes) {
  if (g_capture) {
    *sm_count = 148;
    *l2_bytes = 126 << 20;
    *hbm_bytes = int64_t{180} << 30;
    return 0;
  }
  cudaDeviceProp p;
  if (int rc = check(cudaGetDeviceProperties(&p, device), "cudaGetDeviceProperties")) return rc;
  *sm_count = p.multiProcessorCount;
  *l2_bytes = p.l2CacheSize;
  *hbm_bytes = static_cast<int64_t>(p.totalGlobalMem);
  return 0;
}

int disc_cuda_stream_create(void** stream) {
  cudaStream_t s;
  int rc = check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
  *stream = s;
  return rc;
}
int disc_cuda_stream_destroy(void* stream) { return check(cudaStreamDestroy(S(stream)), "cudaStreamDestroy"); }
int disc_cuda_stream_synchronize(void* stream) {
  if (g_capture) return 0;
  return check(cudaStreamSynchronize(S(stream)), "cudaStreamSynchronize");
}
int disc_cuda_device_synchronize(void) { return check(cudaDeviceSynchronize(), "cudaDeviceSynchronize"); }

int disc_cuda_malloc(size_t bytes, void* stream, void** dptr) {
  if (g_capture) {
    *dptr = reinterpret_cast<void*>(g_fake_next);
    g_fake_next += (bytes + 4095) / 4096 * 4096 + 4096;
    return 0;
  }
  return check(cudaMallocAsync(dptr, bytes ? bytes : 16, S(stream)), "cudaMallocAsync");
}
int disc_cuda_free(void* dptr, void* stream) {
  if (g_capture) return 0;
  return check(cudaFreeAsync(dptr, S(stream)), "cudaFreeAsync");
}
int disc_cuda_host_alloc(size_t bytes, void** hptr) { return check(cudaMallocHost(hptr, bytes ? bytes : 16), "cudaMallocHost"); }
int disc_cuda_host_free(void* hptr) { return check(cudaFreeHost(hptr), "cudaFreeHost"); }

int disc_cuda_memcpy(void* dst, const void* src, size_t bytes, int kind, void* stream) {
  if (!bytes || g_capture) return 0;
  static const cudaMemcpyKind kinds[] = {cudaMemcpyHostToDevice, cudaMemcpyDeviceToHost, cudaMemcpyDeviceToDevice,
                                         cudaMemcpyDefault};
  return check(cudaMemcpyAsync(dst, src, bytes, kinds[kind & 3], S(stream)), "cudaMemcpyAsync");
}
int disc_cuda_memset(void* dst, int value, size_t bytes, void* stream) {
  if (g_capture) return 0;
  return check(cudaMemsetAsync(dst, value, bytes, S(stream)), "cudaMemsetAsync");
}

int disc_cuda_event_create(void** ev) {
  if (g_capture) {
    *ev = reinterpret_cast<void*>(g_fake_next++);
    return 0;
  }
  cudaEvent_t e;
  int rc = check(cudaEventCreate(&e), "cudaEventCreate");
  *ev = e;
  return rc;
}
int disc_cuda_event_destroy(void* ev) {
  if (g_capture) return 0;
  return check(cudaEventDestroy(static_cast<cudaEvent_t>(ev)), "cudaEventDestroy"); }
int disc_cuda_event_record(void* ev, void* stream) {
  if (g_capture) return 0;
  return check(cudaEventRecord(static_cast<cudaEvent_t>(ev), S(stream)), "cudaEventRecord");
}
int disc_cuda_stream_wait_event(void* stream, void* ev) {
  if (g_capture) return 0;
  return check(cudaStreamWaitEvent(S(stream), static_cast<cudaEvent_t>(ev), 0), "cudaStreamWaitEvent");
}
int disc_cuda_event_synchronize(void* ev) {
  return check(cudaEventSynchronize(static_cast<cudaEvent_t>(ev)), "cudaEventSynchronize");
}
int disc_cuda_event_elapsed_ms(void* a, void* b, float* ms) {
  return check(cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(a), static_cast<cudaEvent_t>(b)), "cudaEventElapsedTime");
}

int disc_cuda_launch_loop(const disc_loop_launch* l, void* stream) {
  if (l->total <= 0) return 0;
  const uint64_t key = launch_key(0, l->prog, nullptr);
  if (g_capture) {
    if (g_capture_record) record("loop", key, "\"vec\":" + std::to_string(l->vec) + ",\"pre\":" + program_text(l->prog));
    else if (g_spec_enabled && !l->wide) (void)disc_spec::lookup(0, key);
    return 0;
  }
  if (g_spec_enabled && !l->wide)
    if (const disc_spec::Entry* e = disc_spec::lookup(0, key)) {
      g_spec_launches.fetch_add(1, std::memory_order_relaxed);
      return counted(e->launch(l, l->vec, S(stream)), "launch loop (generated)");
    }
  return counted(disc_launch::loop(*l, S(stream)), "launch loop");
}

int disc_cuda_launch_reduce(const disc_reduce_launch* l, void* stream) {
  const bool row = l->schedule == DISC_SCHED_ROW;
  const bool col = l->schedule == DISC_SCHED_COL_SINGLE || l->schedule == DISC_SCHED_COL_TWOPASS ||
                   l->schedule == DISC_SCHED_COL_ATOMIC;
  const uint64_t key = row ? launch_key(1, l->pre, &l->post) : launch_key(2, l->pre, nullptr);
  if (g_capture) {
    if (!g_capture_record) {
      if (g_spec_enabled && (row || col)) (void)disc_spec::lookup(row ? 1 : 2, key);
      return 0;
    }
    if (row || col)
      record(row ? "row" : "col", key,
             "\"vec\":" + std::to_string(l->vec) + ",\"pre\":" + program_text(l->pre) +
                 (row ? ",\"post\":" + program_text(l->post) : std::string()));
    return 0;
  }
  const disc_spec::Entry* e = (g_spec_enabled && !l->wide && (row || col)) ? disc_spec::lookup(row ? 1 : 2, key) : nullptr;
  if (e) g_spec_launches.fetch_add(1, std::memory_order_relaxed);
  if (!col) return counted(e ? e->launch(l, l->vec, S(stream)) : disc_launch::reduce(*l, S(stream)), "launch reduce");
  if (l->K * l->C <= 0) return 0;
  if (l->schedule == DISC_SCHED_COL_ATOMIC) {
    if (int rc = check(cudaMemsetAsync(l->workspace, 0, sizeof(double) * l->K * l->C, S(stream)), "workspace memset"))
      return rc;
  }
  if (int rc = counted(e ? e->launch(l, l->vec, S(stream)) : disc_launch::col_pass(*l, S(stream)), "launch column pass"))
    return rc;
  if (l->schedule == DISC_SCHED_COL_SINGLE) return 0;
  return counted(disc_launch::finalize_columns(*l, S(stream)), "launch column finalize");
}

int disc_cuda_launch_pad(const disc_pad_launch* l, void* stream) {
  if (g_capture) return 0;
  if (l->total <= 0) return 0;
  return counted(disc_launch::pad(*l, S(stream)), "launch pad");
}
int disc_cuda_launch_concat(const disc_concat_launch* l, void* stream) {
  if (g_capture) return 0;
  return counted(disc_launch::concat(*l, S(stream)), "launch concat");
}
int disc_cuda_gemm(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c, void* stream) {
  if (g_capture) return 0;
  return counted(disc_launch::gemm(m, k, n, a, b, c, S(stream)), "launch gemm");
}
int disc_cuda_fill_uniform(float* dst, int64_t n, uint64_t seed, float lo, float hi, void* stream) {
  return counted(disc_launch::fill_uniform(dst, n, seed, lo, hi, S(stream)), "launch fill");
}
int disc_cuda_flush_l2(void* scratch, size_t bytes, void* stream) {
  return counted(disc_launch::flush(scratch, bytes, S(stream)), "launch flush");
}
int disc_cuda_spin(uint64_t microseconds, void* stream) {
  return counted(disc_launch::spin(microseconds * 1000ull, S(stream)), "launch spin");
}
int64_t disc_cuda_kernel_launches(void) { return g_launches.load(); }

int disc_cuda_set_pdl(int mode) {
  disc_launch::set_pdl(mode < 0 ? 0 : (mode > 2 ? 2 : mode));
  return 0;
}
int disc_cuda_pdl_mode(void) { return disc_launch::pdl_mode(); }

int disc_cuda_set_specialization(int enabled) {
  g_spec_enabled = enabled != 0;
  return 0;
}
int64_t disc_cuda_specialized_launches(void) { return g_spec_launches.load(); }
int disc_cuda_num_specializations(void) { return disc_spec::count(); }

int disc_cuda_set_capture(int enabled) {
  g_capture = enabled != 0;
  g_capture_record = enabled == 1;
  if (g_capture) g_records.clear();
  return 0;
}
int disc_cuda_capture_records(char** json) {
  std::string s = "[";
  for (size_t i = 0; i < g_records.size(); ++i) s += (i ? ",\n" : "\n") + g_records[i];
  s += "\n]";
  *json = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(*json, s.c_str(), s.size() + 1);
  return 0;
}

}  // extern "C"
