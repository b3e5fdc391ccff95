// Standalone (non-fusible) data-movement artifacts and the library GEMM:
//   pad    -> output-driven gather (eval_pad, reference kernels.cpp:125-147)
//   concat -> output-driven gather (eval_concat, kernels.cpp:196-232)
//   gemm   -> f32 in/out with f64 accumulation (eval_matmul, kernels.cpp:261-303)
// Transpose and reshape run through the fused loop kernel as single-load programs.
#include <cstdint>
#include <cstdlib>
#include <dlfcn.h>
#include <string>

#include "disc_cuda.h"
#include "kernels.cuh"

namespace disc_dev {

// Grouped 2-D copies (request-queue flush, device.cu): reshape D2D copies and concat
// parts of many requests in ONE launch.  Item g copies rows x cols floats from src (row
// stride src_ld) to dst (row stride dst_ld); CTAs [block_off[g], block_off[g+1]) stride
// over its float4 (or float) elements.
__global__ void __launch_bounds__(256) k_copy2d_g(const __grid_constant__ disc_group G) {
  const int b = blockIdx.x, g = group_of(G, b);
  const disc_copy2d* items = reinterpret_cast<const disc_copy2d*>(G.table);
  const disc_copy2d it = items[g];
  const int lb = b - G.block_off[g], nb = G.block_off[g + 1] - G.block_off[g];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const bool v4 = ((it.cols | it.src_ld | it.dst_ld) & 3) == 0 &&
                  ((reinterpret_cast<uintptr_t>(it.src) | reinterpret_cast<uintptr_t>(it.dst)) & 15) == 0;
  if (v4) {
    const int64_t c4 = it.cols >> 2, n = it.rows * c4;
    for (int64_t f = static_cast<int64_t>(lb) * blockDim.x + threadIdx.x; f < n; f += static_cast<int64_t>(nb) * blockDim.x) {
      const int64_t r = it.rows == 1 ? 0 : f / c4, c = f - r * c4;
      reinterpret_cast<float4*>(it.dst + r * it.dst_ld)[c] = __ldg(reinterpret_cast<const float4*>(it.src + r * it.src_ld) + c);
    }
  } else {
    const int64_t n = it.rows * it.cols;
    for (int64_t f = static_cast<int64_t>(lb) * blockDim.x + threadIdx.x; f < n; f += static_cast<int64_t>(nb) * blockDim.x) {
      const int64_t r = it.rows == 1 ? 0 : f / it.cols, c = f - r * it.cols;
      it.dst[r * it.dst_ld + c] = __ldg(it.src + r * it.src_ld + c);
    }
  }
}

__global__ void __launch_bounds__(256) k_pad(const __grid_constant__ disc_pad_launch P) {
  for (int64_t f = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; f < P.total;
       f += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t rem = f, src = 0, in_stride = 1;
    bool inside = true;
    for (int d = P.rank - 1; d >= 0; --d) {
      const int64_t c = rem % P.out_dims[d];
      rem /= P.out_dims[d];
      const int64_t t = c - P.low[d];
      if (t < 0 || t % P.step[d] != 0) {
        inside = false;
      } else {
        const int64_t i = t / P.step[d];
        if (i >= P.in_dims[d]) inside = false;
        src += i * in_stride;
      }
      in_stride *= P.in_dims[d];
    }
    P.out[f] = inside ? __ldg(P.in + src) : P.value;
  }
}

__global__ void __launch_bounds__(256) k_concat(const __grid_constant__ disc_concat_launch C) {
  int64_t span = 0;
  for (int p = 0; p < C.n_parts; ++p) span += C.part_axis[p];
  const int64_t total = C.outer * span * C.inner;
  for (int64_t f = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; f < total;
       f += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = f % C.inner;
    const int64_t rest = f / C.inner;
    int64_t a = rest % span;
    const int64_t o = rest / span;
    int p = 0;
    while (a >= C.part_axis[p]) a -= C.part_axis[p++];
    const float v = __ldg(C.parts[p] + (o * C.part_axis[p] + a) * C.inner + i);
    C.out[(o * C.axis_total + C.axis_offset + (f / C.inner) % span) * C.inner + i] = v;
  }
}

// 32x32 output tile per 256-thread block (each thread 4 outputs in a column strip),
// K staged through shared memory in 32-wide slices; f64 accumulation.
constexpr int kT = 32;
__global__ void __launch_bounds__(256) k_gemm(int64_t m, int64_t k, int64_t n, const float* __restrict__ a,
                                              const float* __restrict__ b, float* __restrict__ c) {
  __shared__ float As[kT][kT + 1];
  __shared__ float Bs[kT][kT + 1];
  const int tx = threadIdx.x % kT, ty = threadIdx.x / kT;  // ty in [0, 8)
  const int64_t row0 = static_cast<int64_t>(blockIdx.y) * kT, col = static_cast<int64_t>(blockIdx.x) * kT + tx;
  double acc[4] = {0, 0, 0, 0};
  for (int64_t k0 = 0; k0 < k; k0 += kT) {
    for (int r = ty; r < kT; r += 8) {
      const int64_t ar = row0 + r, ac = k0 + tx;
      As[r][tx] = (ar < m && ac < k) ? a[ar * k + ac] : 0.f;
      const int64_t br = k0 + r;
      Bs[r][tx] = (br < k && col < n) ? b[br * n + col] : 0.f;
    }
    __syncthreads();
    const int kk = static_cast<int>(k - k0 < kT ? k - k0 : kT);
    for (int p = 0; p < kk; ++p) {
      const double bv = Bs[p][tx];
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i] += static_cast<double>(As[ty + 8 * i][p]) * bv;
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = row0 + ty + 8 * i;
    if (r < m && col < n) c[r * n + col] = static_cast<float>(acc[i]);
  }
}

__global__ void k_widen(const float* __restrict__ in, double* __restrict__ out, int64_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<double>(__ldg(in + i));
}
__global__ void k_narrow(const double* __restrict__ in, float* __restrict__ out, int64_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<float>(in[i]);
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__global__ void k_fill_uniform(float* dst, int64_t n, uint64_t seed, float lo, float hi) {
  const float span = hi - lo;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t r = mix64(seed * 0x9E3779B97F4A7C15ull + static_cast<uint64_t>(i));
    const float u = static_cast<float>(r >> 40) * (1.0f / 16777216.0f);  // [0, 1)
    float v = lo + u * span;
    dst[i] = v < hi ? v : lo;
  }
}

__global__ void k_flush(uint4* p, int64_t n, uint32_t salt) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = make_uint4(salt, static_cast<uint32_t>(i), salt, 0u);
}
// Read pass over the (long since written back) start of the flush buffer: evicts the
// dirty lines the write pass left in L2, so their write-back is paid here and not inside
// the next timed kernel.  The sum goes to p[0].w only if impossible (keeps the loads).
__global__ void k_flush_read(uint4* p, int64_t n) {
  uint32_t acc = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    acc ^= __ldcg(p + i).y;
  if (acc == 0xFFFFFFFFu && n > 0) p[0].w = acc;
}

// Holds the stream for `ns` nanoseconds (globaltimer), so that host submissions queue up
// behind it and per-launch events then time device execution only.
__global__ void k_spin(uint64_t ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

}  // namespace disc_dev

namespace disc_launch {

using namespace disc_dev;

static int grid_for(int64_t n, int threads, int cap) {
  const int64_t want = (n + threads - 1) / threads;
  return static_cast<int>(want < cap ? (want > 0 ? want : 1) : cap);
}

cudaError_t pad(const disc_pad_launch& P, cudaStream_t s) {
  if (P.total <= 0) return cudaSuccess;
  k_pad<<<grid_for(P.total, 256, 148 * 16), 256, 0, s>>>(P);
  return cudaGetLastError();
}

cudaError_t concat(const disc_concat_launch& C, cudaStream_t s) {
  int64_t span = 0;
  for (int p = 0; p < C.n_parts; ++p) span += C.part_axis[p];
  const int64_t total = C.outer * span * C.inner;
  if (total <= 0) return cudaSuccess;
  k_concat<<<grid_for(total, 256, 148 * 16), 256, 0, s>>>(C);
  return cudaGetLastError();
}

// Grouped copies: the table (H.dev_table) holds H.n disc_copy2d items.
cudaError_t copy2d_group(const HostGroup& H, cudaStream_t s) {
  disc_group G;
  H.fill(G);  // records are disc_copy2d items read in place (no staging)
  int64_t off = 0;
  for (int i = 0; i < H.n; ++i) {
    const disc_copy2d& it = H.at<disc_copy2d>(i);
    G.block_off[i] = static_cast<int32_t>(off);
    const int64_t n = it.rows * it.cols;
    if (n > 0) off += std::min<int64_t>((n + 4095) / 4096, 256);
  }
  G.block_off[H.n] = static_cast<int32_t>(off);
  if (off == 0) return cudaSuccess;
  const cudaError_t e = launch_k(k_copy2d_g, dim3(static_cast<unsigned>(off)), dim3(256), 0, s, G);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// kLibraryCall GEMM with the reference's numerics: eval_matmul
// (kernels.cpp:261-303) accumulates f32 products in f64.  Operands are widened to f64 on the
// device and multiplied by cuBLAS DGEMM (B200 FP64 tensor cores), the product rounded back
// to f32 -- the same exact f64 products and f64 sums as the reference, in another order.
// (SGEMM's f32 accumulation misses the 1e-5 floored tolerance under cancellation at K=768:
// 4.9e-5 measured.)  cuBLAS is loaded lazily with dlopen, so the library only needs it when
// a plan has a library call; DISC_GEMM=simt selects the f64-accumulating SIMT kernel below
// (also used when cuBLAS cannot be loaded).
namespace {
struct Cublas {
  void* handle = nullptr;  // cublasHandle_t
  int (*create)(void**) = nullptr;
  int (*set_stream)(void*, cudaStream_t) = nullptr;
  int (*dgemm)(void*, int, int, int, int, int, const double*, const double*, int, const double*, int, const double*,
               double*, int) = nullptr;
  bool ok = false;
};
Cublas* cublas() {
  thread_local Cublas c;
  thread_local bool tried = false;
  if (tried) return c.ok ? &c : nullptr;
  tried = true;
  const char* mode = std::getenv("DISC_GEMM");
  if (mode && std::string(mode) == "simt") return nullptr;
  void* lib = dlopen("libcublas.so.12", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) return nullptr;
  c.create = reinterpret_cast<int (*)(void**)>(dlsym(lib, "cublasCreate_v2"));
  c.set_stream = reinterpret_cast<int (*)(void*, cudaStream_t)>(dlsym(lib, "cublasSetStream_v2"));
  c.dgemm = reinterpret_cast<decltype(c.dgemm)>(dlsym(lib, "cublasDgemm_v2"));
  if (!c.create || !c.set_stream || !c.dgemm || c.create(&c.handle) != 0) return nullptr;
  c.ok = true;
  return &c;
}
}  // namespace

bool gemm_uses_cublas() { return cublas() != nullptr; }

// `ws`: f64 workspace of m*k + k*n + m*n doubles (the caller's scratch); null: one
// stream-ordered allocation, released on every path.
cudaError_t gemm(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c, double* ws,
                 cudaStream_t s) {
  if (m <= 0 || n <= 0) return cudaSuccess;
  if (Cublas* cb = cublas(); cb && k > 0 && m < (int64_t{1} << 31) && n < (int64_t{1} << 31) && k < (int64_t{1} << 31)) {
    double* own = nullptr;
    if (!ws) {
      if (cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&own), sizeof(double) * (m * k + k * n + m * n), s))
        return e;
      ws = own;
    }
    double *a64 = ws, *b64 = ws + m * k, *c64 = ws + m * k + k * n;
    k_widen<<<grid_for(m * k, 256, 148 * 16), 256, 0, s>>>(a, a64, m * k);
    k_widen<<<grid_for(k * n, 256, 148 * 16), 256, 0, s>>>(b, b64, k * n);
    // row-major C[m,n] = A[m,k] B[k,n]  ==  column-major C^T = B^T A^T
    const double one = 1.0, zero = 0.0;
    int st = cb->set_stream(cb->handle, s);
    if (st == 0)
      st = cb->dgemm(cb->handle, 0 /*N*/, 0 /*N*/, static_cast<int>(n), static_cast<int>(m), static_cast<int>(k), &one,
                     b64, static_cast<int>(n), a64, static_cast<int>(k), &zero, c64, static_cast<int>(n));
    k_narrow<<<grid_for(m * n, 256, 148 * 16), 256, 0, s>>>(c64, c, m * n);
    if (own) cudaFreeAsync(own, s);
    if (st != 0) return cudaErrorUnknown;
    return cudaGetLastError();
  }
  dim3 grid(static_cast<unsigned>((n + kT - 1) / kT), static_cast<unsigned>((m + kT - 1) / kT));
  k_gemm<<<grid, 256, 0, s>>>(m, k, n, a, b, c);
  return cudaGetLastError();
}

cudaError_t fill_uniform(float* dst, int64_t n, uint64_t seed, float lo, float hi, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  k_fill_uniform<<<grid_for(n, 256, 148 * 32), 256, 0, s>>>(dst, n, seed, lo, hi);
  return cudaGetLastError();
}

cudaError_t flush(void* p, size_t bytes, cudaStream_t s) {
  static uint32_t salt = 1;
  const int64_t n = static_cast<int64_t>(bytes / 16);
  if (n <= 0) return cudaSuccess;
  k_flush<<<grid_for(n, 256, 148 * 32), 256, 0, s>>>(static_cast<uint4*>(p), n, salt++);
  k_flush_read<<<grid_for(n / 2, 256, 148 * 32), 256, 0, s>>>(static_cast<uint4*>(p), n / 2);
  return cudaGetLastError();
}

cudaError_t spin(uint64_t ns, cudaStream_t s) {
  k_spin<<<1, 32, 0, s>>>(ns);
  return cudaGetLastError();
}

}  // namespace disc_launch
