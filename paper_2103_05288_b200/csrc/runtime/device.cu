// C ABI of the device layer (include/disc_cuda.h): streams, stream-ordered memory,
// events and the kernel launches the runtime flow issues.
#include <atomic>
#include <cstdio>
#include <string>

#include "disc_cuda.h"

namespace disc_launch {
cudaError_t loop(const disc_loop_launch& L, cudaStream_t s);
cudaError_t reduce(const disc_reduce_launch& L, cudaStream_t s);
cudaError_t pad(const disc_pad_launch& P, cudaStream_t s);
cudaError_t concat(const disc_concat_launch& C, cudaStream_t s);
cudaError_t gemm(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c, cudaStream_t s);
cudaError_t fill_uniform(float* dst, int64_t n, uint64_t seed, float lo, float hi, cudaStream_t s);
cudaError_t flush(void* p, size_t bytes, cudaStream_t s);
}  // namespace disc_launch

namespace {
thread_local std::string t_err;
std::atomic<int64_t> g_launches{0};

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

int disc_cuda_device_count(int* n) { return check(cudaGetDeviceCount(n), "cudaGetDeviceCount"); }
int disc_cuda_set_device(int device) { return check(cudaSetDevice(device), "cudaSetDevice"); }

int disc_cuda_device_info(int device, int* sm_count, int64_t* l2_bytes, int64_t* hbm_bytes) {
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
int disc_cuda_stream_synchronize(void* stream) { return check(cudaStreamSynchronize(S(stream)), "cudaStreamSynchronize"); }
int disc_cuda_device_synchronize(void) { return check(cudaDeviceSynchronize(), "cudaDeviceSynchronize"); }

int disc_cuda_malloc(size_t bytes, void* stream, void** dptr) {
  return check(cudaMallocAsync(dptr, bytes ? bytes : 16, S(stream)), "cudaMallocAsync");
}
int disc_cuda_free(void* dptr, void* stream) { return check(cudaFreeAsync(dptr, S(stream)), "cudaFreeAsync"); }
int disc_cuda_host_alloc(size_t bytes, void** hptr) { return check(cudaMallocHost(hptr, bytes ? bytes : 16), "cudaMallocHost"); }
int disc_cuda_host_free(void* hptr) { return check(cudaFreeHost(hptr), "cudaFreeHost"); }

int disc_cuda_memcpy(void* dst, const void* src, size_t bytes, int kind, void* stream) {
  if (!bytes) return 0;
  static const cudaMemcpyKind kinds[] = {cudaMemcpyHostToDevice, cudaMemcpyDeviceToHost, cudaMemcpyDeviceToDevice,
                                         cudaMemcpyDefault};
  return check(cudaMemcpyAsync(dst, src, bytes, kinds[kind & 3], S(stream)), "cudaMemcpyAsync");
}
int disc_cuda_memset(void* dst, int value, size_t bytes, void* stream) {
  return check(cudaMemsetAsync(dst, value, bytes, S(stream)), "cudaMemsetAsync");
}

int disc_cuda_event_create(void** ev) {
  cudaEvent_t e;
  int rc = check(cudaEventCreate(&e), "cudaEventCreate");
  *ev = e;
  return rc;
}
int disc_cuda_event_destroy(void* ev) { return check(cudaEventDestroy(static_cast<cudaEvent_t>(ev)), "cudaEventDestroy"); }
int disc_cuda_event_record(void* ev, void* stream) {
  return check(cudaEventRecord(static_cast<cudaEvent_t>(ev), S(stream)), "cudaEventRecord");
}
int disc_cuda_event_synchronize(void* ev) {
  return check(cudaEventSynchronize(static_cast<cudaEvent_t>(ev)), "cudaEventSynchronize");
}
int disc_cuda_event_elapsed_ms(void* a, void* b, float* ms) {
  return check(cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(a), static_cast<cudaEvent_t>(b)), "cudaEventElapsedTime");
}

int disc_cuda_launch_loop(const disc_loop_launch* l, void* stream) {
  if (l->total <= 0) return 0;
  return counted(disc_launch::loop(*l, S(stream)), "launch loop");
}
int disc_cuda_launch_reduce(const disc_reduce_launch* l, void* stream) {
  int n = (l->schedule == DISC_SCHED_COL_TWOPASS || l->schedule == DISC_SCHED_COL_ATOMIC) ? 2 : 1;
  return counted(disc_launch::reduce(*l, S(stream)), "launch reduce", n);
}
int disc_cuda_launch_pad(const disc_pad_launch* l, void* stream) {
  if (l->total <= 0) return 0;
  return counted(disc_launch::pad(*l, S(stream)), "launch pad");
}
int disc_cuda_launch_concat(const disc_concat_launch* l, void* stream) {
  return counted(disc_launch::concat(*l, S(stream)), "launch concat");
}
int disc_cuda_gemm(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c, void* stream) {
  return counted(disc_launch::gemm(m, k, n, a, b, c, S(stream)), "launch gemm");
}
int disc_cuda_fill_uniform(float* dst, int64_t n, uint64_t seed, float lo, float hi, void* stream) {
  return counted(disc_launch::fill_uniform(dst, n, seed, lo, hi, S(stream)), "launch fill");
}
int disc_cuda_flush_l2(void* scratch, size_t bytes, void* stream) {
  return counted(disc_launch::flush(scratch, bytes, S(stream)), "launch flush");
}
int64_t disc_cuda_kernel_launches(void) { return g_launches.load(); }

}  // extern "C"
