// Launchers of the fused tape kernels (interpreter instantiation); the kernel templates
// live in kernels.cuh.  Memory-bound schedules: no tensor cores; 128-bit coalesced
// accesses, CH chunks in flight per thread, f64 accumulation for reductions (the
// reference's reduce semantics, kernels.cpp:46-54, 234-259).
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "kernels.cuh"

// Chunks per thread per interpreter dispatch (the dispatch cost is paid once per
// instruction per CH*VEC elements); A/B knob at build time.
#ifndef DISC_INTERP_CH
#define DISC_INTERP_CH 2
#endif


namespace disc_dev {

__device__ __forceinline__ double red_identity(int kind) { return kind == DISC_REDUCE_SUM ? 0.0 : -INFINITY; }
__device__ __forceinline__ double red_step(int kind, double acc, double v) {
  return kind == DISC_REDUCE_SUM ? acc + v : ((acc < v) ? v : acc);  // std::max(acc, v)
}
__device__ __forceinline__ double red_join(int kind, double a, double b) {
  return kind == DISC_REDUCE_SUM ? a + b : ((a < b) ? b : a);
}

// Finalize split-R partials (two-pass) or cast the f64 atomic accumulators.  A block owns
// 256/lpo outputs with lpo lanes each (lpo grows with the split count, so a few outputs
// over many splits still spread across the block); lane s joins splits s, s+lpo, ... in
// order, then the lanes are joined by a fixed tree (deterministic for a given split count).
__device__ __host__ inline int finalize_lanes(int splits) {
  int l = 8;
  while (l < 256 && l * 4 < splits) l <<= 1;
  return l;
}

// Outputs of a column launch: K*C, or K*fold_cout when folded (fold super-columns each).
__device__ __host__ inline int64_t col_outputs(const disc_reduce_launch& L) {
  return L.fold > 1 ? L.K * L.fold_cout : L.K * L.C;
}

__device__ __forceinline__ void finalize_body(const disc_reduce_launch& L, const int bx, const int gx) {
  __shared__ double part[256];
  pdl_enter(L.pre);
  const int64_t nws = L.K * L.C;  // workspace columns per split
  const int64_t n = col_outputs(L);
  const int F = L.fold > 1 ? L.fold : 1;
  const int64_t cout = F > 1 ? L.fold_cout : 0;
  const int lpo = finalize_lanes(L.splits * F), opb = 256 / lpo;
  const int ox = threadIdx.x / lpo, sl = threadIdx.x % lpo;
  for (int64_t base = static_cast<int64_t>(bx) * opb; base < n; base += static_cast<int64_t>(gx) * opb) {
    const int64_t o = base + ox;
    if (L.schedule != DISC_SCHED_COL_TWOPASS) {  // atomic: one f64 sum per (super-)column
      if (sl == 0 && o < n) {
        double t = L.workspace[o];
        for (int j = 1; j < F; ++j) t = red_join(L.kind, t, L.workspace[o + j * cout]);
        L.red_out[o] = static_cast<float>(t);
      }
      continue;
    }
    double t = red_identity(L.kind);
    if (o < n)
      for (int e = sl; e < L.splits * F; e += lpo) {  // (split, fold) pairs in a fixed order
        const int s = e / F, j = e - s * F;
        t = red_join(L.kind, t, L.workspace[static_cast<int64_t>(s) * nws + o + j * cout]);
      }
    part[threadIdx.x] = t;
    __syncthreads();
    for (int w = lpo / 2; w > 0; w >>= 1) {
      if (sl < w) part[threadIdx.x] = red_join(L.kind, part[threadIdx.x], part[threadIdx.x + w]);
      __syncthreads();
    }
    if (sl == 0 && o < n) L.red_out[o] = static_cast<float>(part[threadIdx.x]);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) k_col_finalize(const __grid_constant__ disc_reduce_launch L) {
  finalize_body(L, blockIdx.x, gridDim.x);
}
__global__ void __launch_bounds__(256) k_col_finalize_g(const __grid_constant__ disc_group G) {
  __shared__ __align__(16) unsigned char desc[desc_bytes<disc_reduce_launch>()];
  const int b = blockIdx.x, g = group_of(G, b);
  const disc_reduce_launch& L = group_stage<disc_reduce_launch>(G, g, desc);
  finalize_body(L, b - G.block_off[g], G.block_off[g + 1] - G.block_off[g]);
}

// ---------------------------------------------------------------------------
// Generic schedule: arbitrary reduced-axis mask; one thread per output element; the
// program runs on the flat index (W = 1 view: row = f).
__global__ void __launch_bounds__(kLoopThreads) k_reduce_generic(const __grid_constant__ disc_reduce_launch L) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ float consts[DISC_MAX_LOADS];
  float* slots = reinterpret_cast<float*>(smem_raw) + threadIdx.x;
  pdl_enter(L.pre);
  hoist_consts(L.pre, consts);
  __syncthreads();
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
      TileCtx t{f, 0, 1, 1, 1};
      float v[1];
      run_tile<1, 1, true>(L.pre, t, v, slots, kLoopThreads, consts, 0.f);
      acc = red_step(L.kind, acc, (double)v[0]);
    }
    if (L.red_out) L.red_out[o] = static_cast<float>(acc);
  }
}

}  // namespace disc_dev

// ---------------------------------------------------------------------------
// Host launchers (called by the C ABI in runtime/device.cu).
namespace disc_dev {

static int g_pdl = 1;
static thread_local bool t_capturing = false;  // stream capture in progress on this thread
bool pdl_enabled() { return g_pdl != 0 && !t_capturing; }
void set_capturing(bool on) { t_capturing = on; }

int group_waves() {
  static const int w = [] {
    const char* e = std::getenv("DISC_GROUP_WAVES");
    const int v = e ? std::atoi(e) : 16;
    return v > 0 ? v : 16;
  }();
  return w;
}

namespace {
struct OccKey {
  int device;
  const void* kernel;
  int block;
  size_t smem;
  bool operator==(const OccKey& o) const {
    return device == o.device && kernel == o.kernel && block == o.block && smem == o.smem;
  }
};
struct OccKeyHash {
  size_t operator()(const OccKey& k) const {
    uint64_t h = reinterpret_cast<uintptr_t>(k.kernel) * 0x9E3779B97F4A7C15ull;
    h ^= (static_cast<uint64_t>(k.block) << 40) ^ (static_cast<uint64_t>(k.device) << 56) ^ k.smem;
    return static_cast<size_t>(h ^ (h >> 29));
  }
};
}  // namespace

// Resident CTAs per SM for (device, kernel, block, dynamic smem): the full tuple is the key.
int resident_ctas(const void* kernel, int block, size_t smem) {
  thread_local std::unordered_map<OccKey, int, OccKeyHash> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const OccKey key{dev, kernel, block, smem};
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, block, smem) != cudaSuccess || n < 1) n = 1;
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, n);
  return n;
}

bool col_mb() {
  static const bool on = [] {
    const char* e = std::getenv("DISC_COL_MB");
    return e && std::atoi(e) != 0;
  }();
  return on;
}

cudaError_t raise_smem_limit(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<OccKey, size_t, OccKeyHash> limit;  // (device, kernel) -> attribute set
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  size_t& cur = limit[OccKey{dev, kernel, 0, 0}];
  if (cur >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  if (e == cudaSuccess) cur = bytes;
  return e;
}

}  // namespace disc_dev

namespace disc_launch {

using namespace disc_dev;

void set_pdl(int mode) { g_pdl = mode; }
int pdl_mode() { return g_pdl; }

cudaError_t loop(const disc_loop_launch& L, cudaStream_t s, const HostGroup* g) {
  return loop_pass<Interp, DISC_INTERP_CH>(L, s, true, g);
}

cudaError_t col_pass(const disc_reduce_launch& L, cudaStream_t s, const HostGroup* g);

inline int64_t finalize_blocks(const disc_reduce_launch& L) {
  const int64_t n = col_outputs(L);
  const int64_t opb = 256 / finalize_lanes(L.splits * (L.fold > 1 ? L.fold : 1));
  const int64_t want = (n + opb - 1) / opb;
  return want < sm_count() * 8 ? want : sm_count() * 8;
}

cudaError_t finalize_columns(const disc_reduce_launch& L, cudaStream_t s, const HostGroup* g) {
  if (g) {  // members are two-pass / atomic launches
    disc_group G;
    g->fill(G);  // the column pass's records: reduce geometry, pointers and pre.flags included
    int64_t off = 0;
    for (int i = 0; i < g->n; ++i) {
      G.block_off[i] = static_cast<int32_t>(off);
      const disc_reduce_launch& M = g->at<disc_reduce_launch>(i);
      if (M.K * M.C > 0 && M.schedule != DISC_SCHED_COL_SINGLE) off += finalize_blocks(M);
    }
    G.block_off[g->n] = static_cast<int32_t>(off);
    if (off == 0) return cudaSuccess;
    const cudaError_t e = launch_k(k_col_finalize_g, dim3(static_cast<unsigned>(off)), dim3(256), 0, s, G);
    return e != cudaSuccess ? e : cudaGetLastError();
  }
  if (L.schedule == DISC_SCHED_COL_SINGLE) return cudaSuccess;
  const cudaError_t e = launch_k(k_col_finalize, dim3(static_cast<int>(finalize_blocks(L))), dim3(256), 0, s, L);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t reduce(const disc_reduce_launch& L, cudaStream_t s, const HostGroup* g) {
  if (L.schedule == DISC_SCHED_ROW) {
    return row_pass<Interp, Interp, DISC_INTERP_CH>(L, s, true, g);
  }
  if (L.schedule == DISC_SCHED_GENERIC) {
    if (g) return cudaErrorInvalidValue;  // never grouped (device layer issues these one by one)
    if (L.K <= 0) return cudaSuccess;
    const int slots = L.pre.n_slots;
    const int64_t want = (L.K + kLoopThreads - 1) / kLoopThreads;
    const int grid = static_cast<int>(want < sm_count() * 8 ? want : sm_count() * 8);
    const size_t smem = static_cast<size_t>(slots) * kLoopThreads * 4;
    cudaError_t e = set_smem(k_reduce_generic, smem);
    if (e != cudaSuccess) return e;
    e = launch_k(k_reduce_generic, dim3(grid), dim3(kLoopThreads), smem, s, L);
    return e != cudaSuccess ? e : cudaGetLastError();
  }
  return col_pass(L, s, g);  // column schedules: the device layer adds memset/finalize
}

cudaError_t col_pass(const disc_reduce_launch& L, cudaStream_t s, const HostGroup* g) {
  return col_pass_t<Interp, DISC_INTERP_CH>(L, s, true, g);
}

}  // namespace disc_launch
