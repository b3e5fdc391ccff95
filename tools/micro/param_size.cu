// Launch cost vs kernel parameter size (host submit rate and device back-to-back time).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a param_size.cu -o param_size && ./param_size
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

template <int N>
struct P {
  float* out;
  int pad[N];
};

template <int N>
__global__ void k(const __grid_constant__ P<N> p) {
  if (threadIdx.x == 0 && blockIdx.x == 0) p.out[0] += p.pad[N - 1];
}

template <int N>
void run(const char* name, bool pdl) {
  P<N> p{};
  cudaMalloc(&p.out, 16);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  for (int i = 0; i < 200; ++i) cudaLaunchKernelEx(&cfg, k<N>, p);
  cudaStreamSynchronize(s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int n = 2000;
  cudaEventRecord(a, s);
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < n; ++i) cudaLaunchKernelEx(&cfg, k<N>, p);
  auto t1 = std::chrono::steady_clock::now();
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("%-8s pdl=%d  host %.2f us/launch  device %.2f us/kernel (back-to-back)\n", name, pdl,
         std::chrono::duration<double, std::micro>(t1 - t0).count() / n, ms * 1e3 / n);
  cudaStreamDestroy(s);
  cudaFree(p.out);
}

int main() {
  for (int pdl = 0; pdl < 2; ++pdl) {
    run<14>("64B", pdl);
    run<126>("512B", pdl);
    run<1150>("4.6KB", pdl);
    run<2300>("9.2KB", pdl);
  }
  return 0;
}
