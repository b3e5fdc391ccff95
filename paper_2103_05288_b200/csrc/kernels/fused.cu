// Fused tape kernels for sm_100a: elementwise loops (kLoop groups) and reduce-rooted
// schedules (kInput groups: row, column two-pass/atomic, generic), all driven by the
// by-value lowered tape (disc_program).  Memory-bound: no tensor cores; 128-bit
// coalesced accesses along the contiguous dimension, f64 accumulation for reductions
// (the reference's reduce semantics, kernels.cpp:46-54, 234-259).
#include <cfloat>
#include <cmath>

#include "program.cuh"

namespace disc_dev {

constexpr int kLoopThreads = 256;

// ---------------------------------------------------------------------------
// kLoop: one program over the flat space, grid-stride over VEC-element chunks.
template <int VEC, bool WIDE>
__global__ void __launch_bounds__(kLoopThreads) k_loop(const __grid_constant__ disc_loop_launch L) {
  using T = typename Vec<VEC>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* slots = reinterpret_cast<T*>(smem_raw) + threadIdx.x;
  const int64_t chunks = L.total / VEC;
  const int64_t step = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; c < chunks; c += step)
    run_program<VEC, WIDE>(L.prog, c * VEC, slots, blockDim.x, 0.f);
}

// ---------------------------------------------------------------------------
// Reduction helpers (f64, reference order-insensitive within f64 rounding).
__device__ __forceinline__ double red_identity(int kind) { return kind == DISC_REDUCE_SUM ? 0.0 : -INFINITY; }
__device__ __forceinline__ double red_step(int kind, double acc, double v) {
  return kind == DISC_REDUCE_SUM ? acc + v : ((acc < v) ? v : acc);  // std::max(acc, v)
}
__device__ __forceinline__ double red_join(int kind, double a, double b) {
  // Joins partials: sum adds; max keeps NaN out (partials never hold NaN).
  return kind == DISC_REDUCE_SUM ? a + b : ((a < b) ? b : a);
}
__device__ __forceinline__ double red_accumulate(int kind, double acc, float v) { return red_step(kind, acc, (double)v); }
__device__ __forceinline__ double red_accumulate(int kind, double acc, float4 v) {
  acc = red_step(kind, acc, (double)v.x);
  acc = red_step(kind, acc, (double)v.y);
  acc = red_step(kind, acc, (double)v.z);
  return red_step(kind, acc, (double)v.w);
}

// ---------------------------------------------------------------------------
// Row schedule: reduce arg collapsed to [K rows, R]; G threads per row (power of two).
// Optional fused epilogue (post program) re-evaluated per element with the row value.
template <int VEC, bool WIDE>
__global__ void __launch_bounds__(1024) k_row(const __grid_constant__ disc_reduce_launch L) {
  using T = typename Vec<VEC>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double warp_part[32];
  __shared__ float row_val[32];
  T* slots = reinterpret_cast<T*>(smem_raw) + threadIdx.x;
  const int G = L.group;
  const int lane = threadIdx.x & (G - 1);
  const int sub = threadIdx.x / G;
  const int rpb = blockDim.x / G;
  const int64_t rows = L.K;
  const int64_t chunks = L.R / VEC;
  const int kind = L.kind;
  const bool fuse_post = L.post.n_instr > 0;

  for (int64_t base = static_cast<int64_t>(blockIdx.x) * rpb; base < rows; base += static_cast<int64_t>(gridDim.x) * rpb) {
    const int64_t row = base + sub;
    const bool valid = row < rows;
    double acc = red_identity(kind);
    if (valid) {
      const int64_t f0 = row * L.R;
      for (int64_t c = lane; c < chunks; c += G) {
        T v = run_program<VEC, WIDE>(L.pre, f0 + c * VEC, slots, blockDim.x, 0.f);
        acc = red_accumulate(kind, acc, v);
      }
    }
    // Reduce within the G-thread group.
    const int width = G < 32 ? G : 32;
    for (int o = width / 2; o > 0; o >>= 1) acc = red_join(kind, acc, __shfl_xor_sync(0xffffffffu, acc, o, width));
    float result;
    if (G <= 32) {
      result = static_cast<float>(acc);
    } else {
      const int warp = threadIdx.x >> 5;
      if ((threadIdx.x & 31) == 0) warp_part[warp] = acc;
      __syncthreads();
      const int wpr = G >> 5;  // warps per row group
      if (lane == 0) {
        double t = warp_part[sub * wpr];
        for (int w = 1; w < wpr; ++w) t = red_join(kind, t, warp_part[sub * wpr + w]);
        row_val[sub] = static_cast<float>(t);
      }
      __syncthreads();
      result = row_val[sub];
    }
    if (valid) {
      if (lane == 0 && L.red_out) L.red_out[row] = result;
      if (fuse_post) {
        const int64_t f0 = row * L.R;
        for (int64_t c = lane; c < chunks; c += G) run_program<VEC, WIDE>(L.post, f0 + c * VEC, slots, blockDim.x, result);
      }
    }
    if (G > 32) __syncthreads();  // warp_part/row_val reuse next iteration
  }
}

// ---------------------------------------------------------------------------
// Column schedule: reduce arg collapsed to [K, R, C], reduce over R, C contiguous.
// Block = 32 (along C chunks) x 8 (along R); grid.x = K * ceil(C/VEC/32), grid.y = splits.
constexpr int kColX = 32, kColY = 8;

template <int VEC, bool WIDE>
__global__ void __launch_bounds__(kColX* kColY) k_col(const __grid_constant__ disc_reduce_launch L) {
  using T = typename Vec<VEC>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double part[kColY][kColX][VEC];
  const int tid = threadIdx.y * kColX + threadIdx.x;
  T* slots = reinterpret_cast<T*>(smem_raw) + tid;
  const int kind = L.kind;
  const int64_t cchunks = L.C / VEC;
  const int64_t tiles = (cchunks + kColX - 1) / kColX;
  const int64_t k = blockIdx.x / tiles;
  const int64_t cc = (blockIdx.x % tiles) * kColX + threadIdx.x;
  const int64_t per = (L.R + L.splits - 1) / L.splits;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * per;
  const int64_t r1 = r0 + per < L.R ? r0 + per : L.R;

  double acc[VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i) acc[i] = red_identity(kind);
  if (cc < cchunks) {
    for (int64_t r = r0 + threadIdx.y; r < r1; r += kColY) {
      const int64_t f = (k * L.R + r) * L.C + cc * VEC;
      T v = run_program<VEC, WIDE>(L.pre, f, slots, kColX * kColY, 0.f);
      if constexpr (VEC == 1) {
        acc[0] = red_step(kind, acc[0], (double)v);
      } else {
        acc[0] = red_step(kind, acc[0], (double)v.x);
        acc[1] = red_step(kind, acc[1], (double)v.y);
        acc[2] = red_step(kind, acc[2], (double)v.z);
        acc[3] = red_step(kind, acc[3], (double)v.w);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < VEC; ++i) part[threadIdx.y][threadIdx.x][i] = acc[i];
  __syncthreads();
  if (threadIdx.y == 0 && cc < cchunks) {
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      double t = part[0][threadIdx.x][i];
      for (int y = 1; y < kColY; ++y) t = red_join(kind, t, part[y][threadIdx.x][i]);
      const int64_t o = k * L.C + cc * VEC + i;
      switch (L.schedule) {
        case DISC_SCHED_COL_SINGLE:
          if (L.red_out) L.red_out[o] = static_cast<float>(t);
          break;
        case DISC_SCHED_COL_TWOPASS:
          L.workspace[static_cast<int64_t>(blockIdx.y) * L.K * L.C + o] = t;
          break;
        default:  // DISC_SCHED_COL_ATOMIC (sum only)
          atomicAdd(L.workspace + o, t);
          break;
      }
    }
  }
}

// Finalize split-R partials: ordered join over splits (two-pass) or cast (atomic).
__global__ void k_col_finalize(const __grid_constant__ disc_reduce_launch L) {
  const int64_t n = L.K * L.C;
  for (int64_t o = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; o < n;
       o += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double t;
    if (L.schedule == DISC_SCHED_COL_TWOPASS) {
      t = L.workspace[o];
      for (int s = 1; s < L.splits; ++s) t = red_join(L.kind, t, L.workspace[static_cast<int64_t>(s) * n + o]);
    } else {
      t = L.workspace[o];
    }
    L.red_out[o] = static_cast<float>(t);
  }
}

// ---------------------------------------------------------------------------
// Generic schedule: arbitrary reduced-axis mask; one thread per output element.
__global__ void __launch_bounds__(kLoopThreads) k_reduce_generic(const __grid_constant__ disc_reduce_launch L) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* slots = reinterpret_cast<float*>(smem_raw) + threadIdx.x;
  const int r = L.g_rank;
  int64_t kept_dims[DISC_MAX_RANK], red_dims[DISC_MAX_RANK], kept_str[DISC_MAX_RANK], red_str[DISC_MAX_RANK];
  int nk = 0, nr = 0;
  int64_t stride = 1;
  int64_t str[DISC_MAX_RANK];
  for (int d = r - 1; d >= 0; --d) {
    str[d] = stride;
    stride *= L.g_dims[d];
  }
  for (int d = 0; d < r; ++d) {
    if ((L.g_mask >> d) & 1) {
      red_dims[nr] = L.g_dims[d];
      red_str[nr++] = str[d];
    } else {
      kept_dims[nk] = L.g_dims[d];
      kept_str[nk++] = str[d];
    }
  }
  const int64_t outs = L.K, inner = L.R;
  for (int64_t o = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; o < outs;
       o += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t base = 0, rem = o;
    for (int i = nk - 1; i >= 0; --i) {
      base += (rem % kept_dims[i]) * kept_str[i];
      rem /= kept_dims[i];
    }
    double acc = red_identity(L.kind);
    for (int64_t j = 0; j < inner; ++j) {
      int64_t f = base, rj = j;
      for (int i = nr - 1; i >= 0; --i) {
        f += (rj % red_dims[i]) * red_str[i];
        rj /= red_dims[i];
      }
      float v = run_program<1, true>(L.pre, f, slots, kLoopThreads, 0.f);
      acc = red_step(L.kind, acc, (double)v);
    }
    if (L.red_out) L.red_out[o] = static_cast<float>(acc);
  }
}

}  // namespace disc_dev

// ---------------------------------------------------------------------------
// Host launchers (called by the C ABI in runtime/device.cu).
namespace disc_launch {

using namespace disc_dev;

static int sm_count() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

template <typename K>
static cudaError_t set_smem(K kernel, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
}

cudaError_t loop(const disc_loop_launch& L, cudaStream_t s) {
  if (L.total <= 0) return cudaSuccess;
  const int64_t chunks = L.total / L.vec;
  const int64_t want = (chunks + kLoopThreads - 1) / kLoopThreads;
  const int grid = static_cast<int>(want < sm_count() * 16 ? want : sm_count() * 16);
  const size_t smem = static_cast<size_t>(L.prog.n_slots) * kLoopThreads * (L.vec == 4 ? 16 : 4);
  auto go = [&](auto kernel) {
    cudaError_t e = set_smem(kernel, smem);
    if (e != cudaSuccess) return e;
    kernel<<<grid, kLoopThreads, smem, s>>>(L);
    return cudaGetLastError();
  };
  if (L.vec == 4) return L.wide ? go(k_loop<4, true>) : go(k_loop<4, false>);
  return L.wide ? go(k_loop<1, true>) : go(k_loop<1, false>);
}

cudaError_t reduce(const disc_reduce_launch& L, cudaStream_t s) {
  const int slots = L.pre.n_slots > L.post.n_slots ? L.pre.n_slots : L.post.n_slots;
  const size_t esz = L.vec == 4 ? 16 : 4;
  if (L.schedule == DISC_SCHED_ROW) {
    if (L.K <= 0) return cudaSuccess;
    const int block = L.group > 256 ? L.group : 256;
    const int rpb = block / L.group;
    const int64_t groups = (L.K + rpb - 1) / rpb;
    const int64_t cap = static_cast<int64_t>(sm_count()) * (2048 / block) * 4;
    const int grid = static_cast<int>(groups < cap ? groups : cap);
    const size_t smem = static_cast<size_t>(slots) * block * esz;
    auto go = [&](auto kernel) {
      cudaError_t e = set_smem(kernel, smem);
      if (e != cudaSuccess) return e;
      kernel<<<grid, block, smem, s>>>(L);
      return cudaGetLastError();
    };
    if (L.vec == 4) return L.wide ? go(k_row<4, true>) : go(k_row<4, false>);
    return L.wide ? go(k_row<1, true>) : go(k_row<1, false>);
  }
  if (L.schedule == DISC_SCHED_GENERIC) {
    if (L.K <= 0) return cudaSuccess;
    const int64_t want = (L.K + kLoopThreads - 1) / kLoopThreads;
    const int grid = static_cast<int>(want < sm_count() * 8 ? want : sm_count() * 8);
    const size_t smem = static_cast<size_t>(slots) * kLoopThreads * 4;
    cudaError_t e = set_smem(k_reduce_generic, smem);
    if (e != cudaSuccess) return e;
    k_reduce_generic<<<grid, kLoopThreads, smem, s>>>(L);
    return cudaGetLastError();
  }
  // Column schedules.
  if (L.K * L.C <= 0) return cudaSuccess;
  if (L.schedule == DISC_SCHED_COL_ATOMIC) {
    cudaError_t e = cudaMemsetAsync(L.workspace, 0, sizeof(double) * L.K * L.C, s);
    if (e != cudaSuccess) return e;
  }
  const int64_t tiles = (L.C / L.vec + kColX - 1) / kColX;
  dim3 grid(static_cast<unsigned>(L.K * tiles), static_cast<unsigned>(L.splits));
  dim3 block(kColX, kColY);
  const size_t smem = static_cast<size_t>(slots) * kColX * kColY * esz;
  auto go = [&](auto kernel) {
    cudaError_t e = set_smem(kernel, smem);
    if (e != cudaSuccess) return e;
    kernel<<<grid, block, smem, s>>>(L);
    return cudaGetLastError();
  };
  cudaError_t e;
  if (L.vec == 4) e = L.wide ? go(k_col<4, true>) : go(k_col<4, false>);
  else e = L.wide ? go(k_col<1, true>) : go(k_col<1, false>);
  if (e != cudaSuccess || L.schedule == DISC_SCHED_COL_SINGLE) return e;
  const int64_t n = L.K * L.C;
  const int64_t want = (n + 255) / 256;
  k_col_finalize<<<static_cast<int>(want < sm_count() * 8 ? want : sm_count() * 8), 256, 0, s>>>(L);
  return cudaGetLastError();
}

}  // namespace disc_launch
