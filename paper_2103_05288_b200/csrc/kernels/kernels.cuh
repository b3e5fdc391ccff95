// Kernel templates for the fused schedules, parameterised by a "program" functor:
//   Interp       -- the generic tape interpreter (program.cuh, run_tile), and
//   generated    -- straight-line code for a known program structure (patterns_gen.cu),
// so both share one schedule implementation.  See fused.cu for the launchers.
#pragma once

#include <algorithm>
#include <cstddef>
#include <cfloat>
#include <cmath>
#include <type_traits>

#include "program.cuh"
#include "../desc_ranges.hpp"

namespace disc_dev {

// Programmatic dependent launch: every fused kernel is launched with programmatic stream
// serialization, so its launch overlaps the previous kernel.  The kernel must not touch
// global memory before pdl_enter()'s wait (which returns once the preceding grid has
// completed and flushed).  With DISC_PROG_PDL_EARLY it then lets its own dependents
// launch at once (their CTAs become resident and wait); otherwise as this grid retires.
__device__ __forceinline__ void pdl_enter(const disc_program& P) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (P.flags & DISC_PROG_PDL_EARLY) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Program functors: run<VEC, CH, WIDE>(program, tile, acc, ...).  kSplitFull: the schedule
// instantiates a guard-free body for full tiles (generated programs); the interpreter
// keeps one body.
struct Interp {
  static constexpr bool kSplitFull = false;
  static constexpr int kPipe = 0;  // no load/compute split
  static constexpr bool kXuHeavy = false;
  static constexpr int kMaxRowMinBlocks = 0;  // see k_row_mb
  template <int VEC, int CH, typename Ctx>
  __device__ __forceinline__ static void prefetch(const disc_program&, const Ctx&) {}
  template <int VEC, int CH, bool WIDE, typename Ctx>
  __device__ __forceinline__ static void run(const disc_program& P, const Ctx& t, typename Vec<VEC>::T (&acc)[CH],
                                             typename Vec<VEC>::T* slots, int stride, const float* consts, float red) {
    if constexpr (Ctx::kRows) {  // row tiles: one single-chunk interpreter pass per row
      using T = typename Vec<VEC>::T;
#pragma unroll
      for (int c = 0; c < CH; ++c)
        if (t.has(c)) {
          const TileCtx t1{t.row + c * t.cstride, t.col0, t.W, t.cstride, 1, nullptr};
          run_tile<VEC, 1, WIDE>(P, t1, reinterpret_cast<T(&)[1]>(acc[c]), slots, stride, consts, red);
        }
    } else {
      const Tile<int64_t, false, false, Ctx::kStaged> t64{t.row, t.col0, t.W, t.cstride, t.nvalid, t.cache, t.slot_stride};
      run_tile<VEC, CH, WIDE>(P, t64, acc, slots, stride, consts, red);
    }
  }
};

template <bool WIDE>
using IndexT = typename std::conditional<WIDE, int64_t, int32_t>::type;


// Reduction helpers.  Sums accumulate in f64 (the reference's semantics); max is exact in
// f32 (max of f32 values cast to f64 == cast of the f32 max), with std::max's NaN rule.
template <int KIND>
struct Red {
  using Acc = typename std::conditional<KIND == DISC_REDUCE_SUM, double, float>::type;
  __device__ __forceinline__ static Acc identity() {
    if constexpr (KIND == DISC_REDUCE_SUM) return 0.0;
    else return -INFINITY;
  }
  __device__ __forceinline__ static Acc step(Acc acc, float v) {
    if constexpr (KIND == DISC_REDUCE_SUM) return acc + static_cast<double>(v);
    else return (acc < v) ? v : acc;  // std::max(acc, v)
  }
  __device__ __forceinline__ static Acc join(Acc a, Acc b) {
    if constexpr (KIND == DISC_REDUCE_SUM) return a + b;
    else return (a < b) ? b : a;  // partials never hold NaN
  }
  __device__ __forceinline__ static Acc acc(Acc a, float v) { return step(a, v); }
  __device__ __forceinline__ static Acc acc(Acc a, float4 v) { return step(step(step(step(a, v.x), v.y), v.z), v.w); }
};

// Per-thread partial accumulator of a reduce pass.  Default: the Red accumulator (f64
// sum: one f32->f64 conversion + DADD per element).  COMP (programs heavy on the XU pipe,
// which also executes the f32->f64 conversions, e.g. tanh/exp prologues): a compensated
// f32 pair (Knuth TwoSum, error <= eps|sum| + O(n eps^2) sum|v|, i.e. f64-grade for these
// lengths) on the FMA pipe, converted to f64 once when the pass ends.
#ifndef DISC_COMP_SUM
#define DISC_COMP_SUM 0  // A/B on B200: no gain on the tanh column reduce, -3% softmax
#endif
template <int KIND, bool COMP>
struct PartAcc {
  using RD = Red<KIND>;
  using T = typename RD::Acc;
  __device__ __forceinline__ static T identity() { return RD::identity(); }
  __device__ __forceinline__ static T add(T a, float v) { return RD::step(a, v); }
  __device__ __forceinline__ static T add(T a, float4 v) { return RD::acc(a, v); }
  __device__ __forceinline__ static typename RD::Acc to(T a) { return a; }
};
struct F2 {
  float s, c;
};
template <>
struct PartAcc<DISC_REDUCE_SUM, true> {
  using T = F2;
  __device__ __forceinline__ static T identity() { return {0.f, 0.f}; }
  __device__ __forceinline__ static T add(T a, float v) {
    const float t = __fadd_rn(a.s, v);
    const float bp = __fsub_rn(t, a.s);
    const float ap = __fsub_rn(t, bp);
    const float err = __fadd_rn(__fsub_rn(a.s, ap), __fsub_rn(v, bp));
    return {t, __fadd_rn(a.c, err)};
  }
  __device__ __forceinline__ static T add(T a, float4 v) { return add(add(add(add(a, v.x), v.y), v.z), v.w); }
  __device__ __forceinline__ static double to(T a) { return static_cast<double>(a.s) + static_cast<double>(a.c); }
};
// f32 -> f64 on the integer pipe (XU-bound column passes: the XU executes both the tanh
// prologue's MUFU ops and F2F.F64.F32, ncu s9: XU 75.6% of peak, ALU 28%).  Exact for
// normal floats (the f64 exponent is the f32 one rebiased, the mantissa shifted); zeros,
// subnormals, infinities and NaNs (exponent field 0 or 255) take the hardware conversion,
// for the whole warp when any lane has one, so the result is bit-identical to (double)v.
#ifndef DISC_INT_CVT
#define DISC_INT_CVT 0  // A/B s10 on B200: column reduce 4181 -> 3556 GB/s (the ALU work and the vote cost more than the XU relief); off
#endif
__device__ __forceinline__ double f2d_bits(float v, bool& special) {
  const uint32_t u = __float_as_uint(v);
  const uint32_t e = u & 0x7f800000u;
  special |= (e == 0u) | (e == 0x7f800000u);
  const uint32_t hi = (((u & 0x7fffffffu) >> 3) + 0x38000000u) | (u & 0x80000000u);
  return __hiloint2double(static_cast<int>(hi), static_cast<int>(u << 29));
}
__device__ __forceinline__ void f2d4(const float4& v, double (&d)[4]) {
  bool sp = false;
  d[0] = f2d_bits(v.x, sp);
  d[1] = f2d_bits(v.y, sp);
  d[2] = f2d_bits(v.z, sp);
  d[3] = f2d_bits(v.w, sp);
  if (__any_sync(__activemask(), sp)) {
    d[0] = static_cast<double>(v.x);
    d[1] = static_cast<double>(v.y);
    d[2] = static_cast<double>(v.z);
    d[3] = static_cast<double>(v.w);
  }
}

template <typename Prog>
constexpr bool comp_sum() {
  if constexpr (DISC_COMP_SUM == 0) return false;
  else return Prog::kXuHeavy;
}

// Chunks of a tile inside the row: CH chunks spaced cstride apart starting at col0.
template <int CH>
__device__ __forceinline__ int chunks_in_row(int64_t left, int64_t cstride) {
  int n = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) n += left > c * cstride;
  return n;
}

constexpr int kLoopThreads = 256;
constexpr int kCH = 2;  // chunks per thread per dispatch

// ---------------------------------------------------------------------------
// Grouped launches: ONE kernel covers n independent launches that share a kernel
// instantiation (same program structure / schedule template), e.g. the same plan
// kernel of many variable-shape requests.  Launch g owns CTAs [block_off[g],
// block_off[g+1]) and runs exactly the single-launch body with (local block, local
// grid), so results are identical to n separate launches.  Its launch descriptor lives
// in a device table (uploaded by the device layer) and is staged into shared memory
// once per CTA; the CTA -> launch map is a binary search over the offsets held in
// __grid_constant__ parameter space.
#ifndef DISC_ROW_PIPE
#define DISC_ROW_PIPE 0  // software-pipelined reduce pass in row kernels (A/B on B200: slower, off)
#endif
#ifndef DISC_MAX_GROUP
#define DISC_MAX_GROUP 1024
#endif
#define DISC_GROUP_SEGS 8
struct disc_group {
  const unsigned char* table;  // n descriptors, `stride` bytes apart
  int32_t stride;
  int32_t n;
  int32_t nseg;                       // descriptor ranges a CTA stages, in 16 B units:
  uint16_t seg[DISC_GROUP_SEGS][3];   // (offset in the descriptor, count, offset in the record)
  int32_t block_off[DISC_MAX_GROUP + 1];
};

// Item of a grouped 2-D copy (reshape copies, concat parts): rows x cols floats.
struct disc_copy2d {
  const float* src;
  float* dst;
  int64_t rows, cols, src_ld, dst_ld;
};

__device__ __forceinline__ int group_of(const disc_group& G, int b) {
  int lo = 0, hi = G.n;  // block_off[lo] <= b < block_off[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (G.block_off[mid] <= b) lo = mid;
    else hi = mid;
  }
  return lo;
}

template <typename Launch>
constexpr int desc_bytes() { return (static_cast<int>(sizeof(Launch)) + 15) / 16 * 16; }

// Copies descriptor g into shared memory (16 B per thread per step).  The table was
// written by a copy ordered before the previous kernel in the stream, so it may be read
// before griddepcontrol.wait.
template <typename Launch>
__device__ __forceinline__ const Launch& group_stage(const disc_group& G, int g, unsigned char* buf) {
  // member g's record holds only the descriptor ranges the kernel reads (desc_ranges.hpp),
  // packed back to back; they are unpacked to their offsets in the descriptor
  const uint4* src = reinterpret_cast<const uint4*>(G.table + static_cast<int64_t>(g) * G.stride);
  uint4* dst = reinterpret_cast<uint4*>(buf);
  for (int k = 0; k < G.nseg; ++k) {
    const int o = G.seg[k][0], c = G.seg[k][1], so = G.seg[k][2];
    for (int i = threadIdx.x; i < c; i += blockDim.x) dst[o + i] = __ldg(src + so + i);
  }
  __syncthreads();
  return *reinterpret_cast<const Launch*>(buf);
}

// Host: the staged ranges of a group's descriptors (desc_ranges.hpp): the union over the
// members -- their used prefixes -- so interpreter groups, whose members may differ in
// program length, stage every member's instructions and loads.
inline void max_counts(disc_program& m, const disc_program& p) {
  m.n_instr = std::max(m.n_instr, p.n_instr);
  m.n_loads = std::max(m.n_loads, p.n_loads);
}
inline void group_counts(disc_loop_launch& m, const disc_loop_launch& L) { max_counts(m.prog, L.prog); }
inline void group_counts(disc_reduce_launch& m, const disc_reduce_launch& L) {
  max_counts(m.pre, L.pre);
  max_counts(m.post, L.post);
}
// Fills (nseg, seg, stride) of a compact member record for `n` descriptors.
template <typename Launch>
inline void group_segments(const void* const* members, int n, int32_t* nseg, uint16_t (*seg)[3], int32_t* stride) {
  Launch m;
  disc_desc::copy_used(&m, *static_cast<const Launch*>(members[0]));
  for (int i = 1; i < n; ++i) group_counts(m, *static_cast<const Launch*>(members[i]));
  disc_desc::Range r[disc_desc::kMaxRanges];
  const int nr = disc_desc::ranges(m, r);
  int ns = 0, rec = 0;
  for (int i = 0; i < nr; ++i) {
    if (!r[i].len) continue;
    const int o = static_cast<int>(r[i].off / 16), e = static_cast<int>((r[i].off + r[i].len + 15) / 16);
    if (ns > 0 && seg[ns - 1][0] + seg[ns - 1][1] >= o) {  // merge adjacent
      const int s0 = seg[ns - 1][0], add = std::max(e, s0 + seg[ns - 1][1]) - (s0 + seg[ns - 1][1]);
      seg[ns - 1][1] = static_cast<uint16_t>(seg[ns - 1][1] + add);
      rec += add;
      continue;
    }
    seg[ns][0] = static_cast<uint16_t>(o);
    seg[ns][1] = static_cast<uint16_t>(e - o);
    seg[ns][2] = static_cast<uint16_t>(rec);
    rec += e - o;
    ++ns;
  }
  *nseg = ns;
  *stride = rec * 16;
}

// ---------------------------------------------------------------------------
// kLoop: the space viewed as [rows, W].  A warp tile covers 32/lpr rows x (lpr*CH*VEC)
// columns: lpr lanes share a row (lane l takes chunks l, l+lpr, ... so every access is
// coalesced), narrow rows pack several per warp.  Grid-stride over warp tiles.
template <int VEC, bool WIDE, typename Prog, int CH>
__device__ __forceinline__ void loop_body(const disc_loop_launch& L, const int bx, const int gx) {
  using T = typename Vec<VEC>::T;
  using I = IndexT<WIDE>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ float consts[DISC_MAX_LOADS];
  T* slots = reinterpret_cast<T*>(smem_raw) + threadIdx.x;
  pdl_enter(L.prog);
  hoist_consts(L.prog, consts);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int lpr = L.lpr;
  const int rpw = 32 / lpr;
  const int sub = lane / lpr;
  const I W = static_cast<I>(L.W), rows = static_cast<I>(L.rows);
  const I cstride = static_cast<I>(lpr) * VEC;
  const I span = cstride * CH;
  const I tpr = (W + span - 1) / span;
  const I nrg = (rows + rpw - 1) / rpw;
  const int64_t warps = static_cast<int64_t>(gx) * (blockDim.x >> 5);
  const int64_t tile = static_cast<int64_t>(bx) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  // (row group, column tile) advanced incrementally: one division per thread, not per tile.
  I rg = static_cast<I>(tile / tpr), tc = static_cast<I>(tile - static_cast<int64_t>(rg) * tpr);
  const I drg = static_cast<I>(warps / tpr), dtc = static_cast<I>(warps - static_cast<int64_t>(drg) * tpr);
  const I lane_col = static_cast<I>(lane & (lpr - 1)) * VEC;
  if constexpr (Prog::kPipe > 0) {
    // Software pipeline: the next grid-stride tile's streaming loads are issued before
    // the current tile computes (one tile of loads in flight per thread while the
    // math runs; registers: kPipe x CH x VEC).
    using LD = typename Prog::template Loads<VEC, CH>;
    I row = rg * rpw + sub, col0 = tc * span + lane_col;
    int nv = (rg < nrg && row < rows) ? chunks_in_row<CH>(W - col0, cstride) : 0;
    LD cur;
    if (nv > 0) Prog::template load<VEC, CH, WIDE>(L.prog, Tile<I, false>{row, col0, W, cstride, nv}, cur);
    while (rg < nrg) {
      I nrg_ = rg + drg, ntc = tc + dtc;
      if (ntc >= tpr) {
        ntc -= tpr;
        ++nrg_;
      }
      const I nrow = nrg_ * rpw + sub, ncol0 = ntc * span + lane_col;
      const int nnv = (nrg_ < nrg && nrow < rows) ? chunks_in_row<CH>(W - ncol0, cstride) : 0;
      LD nxt;
      if (nnv > 0) Prog::template load<VEC, CH, WIDE>(L.prog, Tile<I, false>{nrow, ncol0, W, cstride, nnv}, nxt);
      T acc[CH];
      if (nv == CH)
        Prog::template run_loaded<VEC, CH, WIDE>(L.prog, Tile<I, true>{row, col0, W, cstride, CH}, cur, acc, slots,
                                                 kLoopThreads, consts, 0.f);
      else if (CH > 1 && nv > 0)
        Prog::template run_loaded<VEC, CH, WIDE>(L.prog, Tile<I, false>{row, col0, W, cstride, nv}, cur, acc, slots,
                                                 kLoopThreads, consts, 0.f);
      cur = nxt;
      rg = nrg_;
      tc = ntc;
      row = nrow;
      col0 = ncol0;
      nv = nnv;
    }
    return;
  }
  const bool prefetch = L.prefetch != 0;
  for (; rg < nrg;) {
    const I row = rg * rpw + sub;
    const I col0 = tc * span + lane_col;
    if (prefetch) {  // next grid-stride tile of this warp
      I ntc = tc + dtc, nrg_ = rg + drg;
      if (ntc >= tpr) {
        ntc -= tpr;
        ++nrg_;
      }
      const I nrow = nrg_ * rpw + sub, ncol0 = ntc * span + lane_col;
      if (nrow < rows) {
        const int nnv = chunks_in_row<CH>(W - ncol0, cstride);
        Prog::template prefetch<VEC, CH>(L.prog, Tile<I, false>{nrow, ncol0, W, cstride, nnv});
      }
    }
    if (row < rows) {
      const int nv = chunks_in_row<CH>(W - col0, cstride);
      T acc[CH];
      if (!Prog::kSplitFull) {
        if (nv > 0) Prog::template run<VEC, CH, WIDE>(L.prog, Tile<I, false>{row, col0, W, cstride, nv}, acc, slots,
                                                       kLoopThreads, consts, 0.f);
      } else if (nv == CH) {
        Prog::template run<VEC, CH, WIDE>(L.prog, Tile<I, true>{row, col0, W, cstride, CH}, acc, slots, kLoopThreads,
                                          consts, 0.f);
      } else if (CH > 1 && nv > 0) {
        Prog::template run<VEC, CH, WIDE>(L.prog, Tile<I, false>{row, col0, W, cstride, nv}, acc, slots,
                                          kLoopThreads, consts, 0.f);
      }
    }
    rg += drg;
    tc += dtc;
    if (tc >= tpr) {
      tc -= tpr;
      ++rg;
    }
  }
}

// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// Row schedule: reduce arg collapsed to [K rows, R]; G threads per row (power of two);
// thread `lane` of a row takes chunks lane, lane+G, ... (coalesced across the group).
// Optional fused epilogue (post program) re-evaluated per element with the row value.
// Shared-memory slots hold the block's rpb rows back to back (slot-major):
//   row cache (FILL/READ)  loads the epilogue re-reads stay on chip;
//   staged (L.stage)       short rows: the block copies its contiguous span of every
//                          identity input into the slots (coalesced, 16 B when aligned),
//                          programs read/write slots, outputs are copied out the same way.

// TMA bulk copies (cp.async.bulk, 1-D) into shared memory, completing on an mbarrier.
__device__ __forceinline__ uint32_t sh_addr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sh_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sh_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "DISC_MBAR_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra DISC_MBAR_WAIT_%=;\n"
      "}\n" ::"r"(sh_addr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   sh_addr(dst)),
               "l"(src), "r"(bytes), "r"(sh_addr(bar))
               : "memory");
}
// Generic-proxy accesses of a buffer before the async proxy (TMA) overwrites it.
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

#ifndef DISC_COPY_BATCH
#define DISC_COPY_BATCH 1  // A/B s13 (4): staged short rows stay 2-3x slower than unstaged; off
#endif
// Copies n floats global -> shared (or back), 16 B per access when both ends allow it.
__device__ __forceinline__ void copy_span(float* __restrict__ dst, const float* __restrict__ src, int64_t n,
                                          bool to_global) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
    const int64_t n4 = n >> 2;
#if DISC_COPY_BATCH > 1
    // DISC_COPY_BATCH float4 loads per thread issued before any store (memory-level
    // parallelism: the plain loop waits for each load before its store)
    constexpr int U = DISC_COPY_BATCH;
    for (int64_t i0 = tid; i0 < n4; i0 += static_cast<int64_t>(nt) * U) {
      float4 r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + static_cast<int64_t>(u) * nt;
        if (i < n4) r[u] = to_global ? reinterpret_cast<const float4*>(src)[i] : __ldg(reinterpret_cast<const float4*>(src) + i);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + static_cast<int64_t>(u) * nt;
        if (i < n4) reinterpret_cast<float4*>(dst)[i] = r[u];
      }
    }
#else
    for (int64_t i = tid; i < n4; i += nt) {
      const float4 v = to_global ? reinterpret_cast<const float4*>(src)[i] : __ldg(reinterpret_cast<const float4*>(src) + i);
      reinterpret_cast<float4*>(dst)[i] = v;
    }
#endif
    for (int64_t i = (n4 << 2) + tid; i < n; i += nt) dst[i] = to_global ? src[i] : __ldg(src + i);
  } else {
    for (int64_t i = tid; i < n; i += nt) dst[i] = to_global ? src[i] : __ldg(src + i);
  }
}

#ifndef DISC_ROW_L2PF
#define DISC_ROW_L2PF 1  // A/B s20 on B200 (rows with exp/tanh in the reduce pass only): sweep 4947 -> 4976, softmax 4112 -> 4238, BERT 5444 -> 5480-5526 GB/s
#endif
#ifndef DISC_UNAL_HT_TILES
#define DISC_UNAL_HT_TILES 0  // A/B s17 on B200: S=17 2935 -> 3233 GB/s but S=65 3443 -> 3338, C1 and the sweep flat; off
#endif
template <int VEC, bool WIDE, int KIND, typename Pre, typename Post, int CH, bool STAGED, bool UNAL>
__device__ __forceinline__ void row_body(const disc_reduce_launch& L, const int bx, const int gx) {
  using RD = Red<KIND>;
  using Acc = typename RD::Acc;
  using T = typename Vec<VEC>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ Acc warp_part[32];
  __shared__ float row_val[32];
  __shared__ float consts[2][DISC_MAX_LOADS];
  const int G = L.group;
  const int lane = threadIdx.x & (G - 1);
  const int sub = threadIdx.x / G;
  const int rpb = blockDim.x / G;
  // Dynamic smem: [cache_loads slots of slot_stride floats][interpreter slots].
  // float4 body + scalar head/tail per row: a separate instantiation (UNAL), so aligned
  // kernels keep their register budget (30 vs 58 registers for a plain row sum)
  const bool unal = UNAL && VEC == 4 && L.unaligned;
  const int64_t rrow = L.row_pitch ? L.row_pitch : unal ? (L.R + 6) / 4 * 4 : L.R;  // row pitch in the row cache
  const int64_t slot_stride = (static_cast<int64_t>(rpb) * rrow + 3) / 4 * 4;
  const int64_t cache_floats = slot_stride * L.cache_loads;
  float* const cache0 = reinterpret_cast<float*>(smem_raw);
  float* row_cache = L.cache_loads ? cache0 + sub * rrow : nullptr;
  T* slots = reinterpret_cast<T*>(reinterpret_cast<float*>(smem_raw) + cache_floats) + threadIdx.x;
  pdl_enter(L.pre);
  hoist_consts(L.pre, consts[0]);
  hoist_consts(L.post, consts[1]);
  __syncthreads();
  using I = IndexT<WIDE>;
  const int64_t rows = L.K;
  const I R = static_cast<I>(L.R);
  const I sst = static_cast<I>(slot_stride);
  const bool fuse_post = L.post.n_instr > 0;
  const I cstride = static_cast<I>(G) * VEC;
  const I span = cstride * CH;

  // TMA staging (L.stage == 2): the staged inputs of block-iteration i+1 are copied by
  // bulk copies (one per operand, issued by thread 0) into the other half of a double
  // buffer while iteration i computes from shared memory; no registers hold loads in
  // flight.  A block span whose size or source is not 16 B aligned falls back to copy_span.
  __shared__ __align__(8) uint64_t tma_bar[2];
  const bool tma = STAGED && L.stage == 2;
  const int64_t stage_floats = tma ? cache_floats : 0;
  auto tma_issue = [&](int64_t b, int st) -> bool {  // thread 0; false = not TMA-able
    const int64_t n = (rows - b < rpb ? rows - b : rpb) * L.R;
    const uint32_t bytes = static_cast<uint32_t>(n * 4);
    if (bytes % 16) return false;
    uint32_t seen = 0, total = 0;
    for (int pass = 0; pass < 2; ++pass) {  // pass 0: checks and byte count; pass 1: copies
      seen = 0;
      for (int q = 0; q < 2; ++q) {
        const disc_program& P = q ? L.post : L.pre;
        for (int l = 0; l < P.n_loads; ++l) {
          const int k = P.cache_slot[l];
          if (k < 0 || k == L.arg_slot || ((seen >> k) & 1)) continue;
          seen |= 1u << k;
          const float* src = P.loads[l].ptr + b * L.R;
          if (pass == 0) {
            if (reinterpret_cast<uintptr_t>(src) & 15) return false;
            total += bytes;
          } else {
            bulk_g2s(cache0 + st * stage_floats + k * slot_stride, src, bytes, &tma_bar[st]);
          }
        }
      }
      if (pass == 0) {
        fence_proxy_async();  // earlier generic reads/writes of this buffer
        mbar_expect_tx(&tma_bar[st], total);
      }
    }
    return true;
  };
  __shared__ int tma_ok[2];
  uint32_t tma_phase = 0;  // bit s: parity of the next wait on barrier s
  if (tma) {
    if (threadIdx.x == 0) {
      mbar_init(&tma_bar[0], 1);
      mbar_init(&tma_bar[1], 1);
      mbar_fence_init();
      const int64_t b0 = static_cast<int64_t>(bx) * rpb;
      if (b0 < rows) tma_ok[0] = tma_issue(b0, 0);
    }
    __syncthreads();
  }
  int it = 0;
  for (int64_t base = static_cast<int64_t>(bx) * rpb; base < rows; base += static_cast<int64_t>(gx) * rpb, ++it) {
    const int64_t n_el = (rows - base < rpb ? rows - base : rpb) * L.R;
#if DISC_ROW_L2PF
    // only compiled into rows whose reduce pass evaluates exp/tanh (softmax-like fused
    // epilogues): the code alone changes ptxas's allocation of the plain row kernels
    if constexpr (!STAGED && Pre::kXuHeavy) {
      // L2 prefetch of this block's NEXT rows (grid stride) for every streamed operand of the
      // reduce pass: one prefetch per 128 B line, no registers held, so the next iteration's
      // loads hit L2 while this one's epilogue runs (fused rows load nothing in pass 2)
      const int64_t nb = base + static_cast<int64_t>(gx) * rpb;
      if (nb < rows && L.post.n_instr > 0 && L.arg_slot >= 0) {  // argument-cached epilogues only (A/B s18)
        const int64_t nn = (rows - nb < rpb ? rows - nb : rpb) * L.R;
        for (int l = 0; l < L.pre.n_loads; ++l) {
          if (L.pre.loads[l].mode != DISC_LOAD_IDENTITY) continue;
          const float* p = L.pre.loads[l].ptr + nb * L.R;
          for (int64_t i = static_cast<int64_t>(threadIdx.x) * 32; i < nn; i += static_cast<int64_t>(blockDim.x) * 32)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(p + i));
        }
      }
    }
#endif

    if (tma) {
      const int st = it & 1;
      const int64_t nb = base + static_cast<int64_t>(gx) * rpb;
      if (threadIdx.x == 0 && nb < rows) tma_ok[st ^ 1] = tma_issue(nb, st ^ 1);  // prefetch the next
      float* const c0 = cache0 + st * stage_floats;
      if (!tma_ok[st]) {  // synchronous copy of this span (unaligned / odd-sized)
        uint32_t seen = 0;
        for (int q = 0; q < 2; ++q) {
          const disc_program& P = q ? L.post : L.pre;
          for (int l = 0; l < P.n_loads; ++l) {
            const int k = P.cache_slot[l];
            if (k < 0 || k == L.arg_slot || ((seen >> k) & 1)) continue;
            seen |= 1u << k;
            copy_span(c0 + k * slot_stride, P.loads[l].ptr + base * L.R, n_el, false);
          }
        }
        __syncthreads();
      } else {
        mbar_wait(&tma_bar[st], (tma_phase >> st) & 1);
        tma_phase ^= 1u << st;
      }
      row_cache = c0 + sub * rrow;
    } else if constexpr (STAGED) {  // copy the block's rows of every staged input into its slot
      uint32_t pre_slots = 0;
      for (int l = 0; l < L.pre.n_loads; ++l) {
        const int k = L.pre.cache_slot[l];
        if (k >= 0 && !((pre_slots >> k) & 1)) {
          pre_slots |= 1u << k;
          copy_span(cache0 + k * slot_stride, L.pre.loads[l].ptr + base * L.R, n_el, false);
        }
      }
      for (int l = 0; l < L.post.n_loads; ++l) {
        const int k = L.post.cache_slot[l];
        if (k >= 0 && k != L.arg_slot && !((pre_slots >> k) & 1)) {  // the arg slot is written, not copied
          pre_slots |= 1u << k;
          copy_span(cache0 + k * slot_stride, L.post.loads[l].ptr + base * L.R, n_el, false);
        }
      }
      __syncthreads();
    }
    const I row = static_cast<I>(base + sub);
    const bool valid = base + sub < rows;
    // body columns [h, Rb): h = first column whose flat index is 16 B aligned
    I h = 0, Rb = R;
    if (unal) {
      h = static_cast<I>((4 - (static_cast<int64_t>(base + sub) * L.R) % 4) % 4);
      Rb = h + (R - h) / 4 * 4;
      if (L.cache_loads) row_cache = cache0 + sub * rrow + ((4 - h) & 3);  // body aligned in smem too
    }
    // one accumulator per chunk position: CH independent f64 add chains per thread,
    // joined in a fixed order (deterministic)
    using PA = PartAcc<KIND, comp_sum<Pre>()>;
    typename PA::T part[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) part[c] = PA::identity();
    if constexpr (DISC_ROW_PIPE && Pre::kPipe > 0 && !STAGED) {
      // Software pipeline (generated programs): the next span's loads are issued before
      // the current span is evaluated and accumulated.
      using LD = typename Pre::template Loads<VEC, CH>;
      if (valid) {
        I col0 = static_cast<I>(lane) * VEC;
        int nv = col0 < R ? chunks_in_row<CH>(R - col0, cstride) : 0;
        LD cur;
        if (nv == CH) Pre::template load<VEC, CH, WIDE>(L.pre, Tile<I, true>{row, col0, R, cstride, CH, row_cache, sst}, cur);
        else if (nv > 0) Pre::template load<VEC, CH, WIDE>(L.pre, Tile<I, false>{row, col0, R, cstride, nv, row_cache, sst}, cur);
        while (nv > 0) {
          const I ncol = col0 + span;
          const int nnv = ncol < R ? chunks_in_row<CH>(R - ncol, cstride) : 0;
          LD nxt;
          if (nnv == CH)
            Pre::template load<VEC, CH, WIDE>(L.pre, Tile<I, true>{row, ncol, R, cstride, CH, row_cache, sst}, nxt);
          else if (nnv > 0)
            Pre::template load<VEC, CH, WIDE>(L.pre, Tile<I, false>{row, ncol, R, cstride, nnv, row_cache, sst}, nxt);
          T v[CH];
          if (nv == CH) {
            Pre::template run_loaded<VEC, CH, WIDE>(L.pre, Tile<I, true>{row, col0, R, cstride, CH, row_cache, sst}, cur, v,
                                                    slots, blockDim.x, consts[0], 0.f);
#pragma unroll
            for (int c = 0; c < CH; ++c) part[c] = PA::add(part[c], v[c]);
          } else {
            Pre::template run_loaded<VEC, CH, WIDE>(L.pre, Tile<I, false>{row, col0, R, cstride, nv, row_cache, sst}, cur, v,
                                                    slots, blockDim.x, consts[0], 0.f);
#pragma unroll
            for (int c = 0; c < CH; ++c)
              if (c < nv) part[c] = PA::add(part[c], v[c]);
          }
          if (L.arg_slot >= 0 && row_cache) {
#pragma unroll
            for (int c = 0; c < CH; ++c)
              if (c < nv) st_cache(row_cache + L.arg_slot * sst + col0 + c * cstride, v[c]);
          }
          cur = nxt;
          col0 = ncol;
          nv = nnv;
        }
      }
    } else if (valid) {
      // reduce-argument cache (fused epilogue reads the pre value back from smem)
      float* const arg_cache = (L.arg_slot >= 0 && row_cache) ? row_cache + L.arg_slot * sst : nullptr;
      for (I col0 = h + static_cast<I>(lane) * VEC; col0 < Rb; col0 += span) {
        const int nv = chunks_in_row<CH>(Rb - col0, cstride);
        T v[CH];
        if (Pre::kSplitFull && nv == CH) {
          Pre::template run<VEC, CH, WIDE>(L.pre, Tile<I, true, false, STAGED>{row, col0, R, cstride, CH, row_cache, sst}, v, slots,
                                           blockDim.x, consts[0], 0.f);
#pragma unroll
          for (int c = 0; c < CH; ++c) part[c] = PA::add(part[c], v[c]);
        } else {
          Pre::template run<VEC, CH, WIDE>(L.pre, Tile<I, false, false, STAGED>{row, col0, R, cstride, nv, row_cache, sst}, v, slots,
                                           blockDim.x, consts[0], 0.f);
#pragma unroll
          for (int c = 0; c < CH; ++c)
            if (c < nv) part[c] = PA::add(part[c], v[c]);
        }
        if (arg_cache) {
#pragma unroll
          for (int c = 0; c < CH; ++c)
            if (c < nv) st_cache(arg_cache + col0 + c * cstride, v[c]);
        }
      }
      if constexpr (UNAL && VEC == 4 && !STAGED) {
        if (unal && DISC_UNAL_HT_TILES && Pre::kSplitFull && G == 1) {
          // thread per row (generated programs): head [0, h) and tail [Rb, R) as two scalar
          // tiles of <= 3 elements, each with its loads issued together (2 dependent round
          // trips instead of up to 6); same accumulation order as the element loop below
          float hv[4], tv[4];
          if (h > 0)
            Pre::template run<1, 4, WIDE>(L.pre, Tile<I, false>{row, 0, R, 1, static_cast<int>(h), row_cache, sst}, hv,
                                          nullptr, 0, consts[0], 0.f);
          if (R > Rb)
            Pre::template run<1, 4, WIDE>(L.pre, Tile<I, false>{row, Rb, R, 1, static_cast<int>(R - Rb), row_cache, sst},
                                          tv, nullptr, 0, consts[0], 0.f);
#pragma unroll
          for (int c = 0; c < 3; ++c)
            if (c < h) {
              part[0] = PA::add(part[0], hv[c]);
              if (arg_cache) st_cache(arg_cache + c, hv[c]);
            }
#pragma unroll
          for (int c = 0; c < 3; ++c)
            if (c < R - Rb) {
              part[0] = PA::add(part[0], tv[c]);
              if (arg_cache) st_cache(arg_cache + Rb + c, tv[c]);
            }
        } else if (unal) {  // scalar head [0, h) and tail [Rb, R)
          for (I e = static_cast<I>(lane); e < h + (R - Rb); e += static_cast<I>(G)) {
            const I c = e < h ? e : Rb + (e - h);
            float vs[1];
            Pre::template run<1, 1, WIDE>(L.pre, Tile<I, false>{row, c, R, 1, 1, row_cache, sst}, vs,
                                          reinterpret_cast<float*>(slots), blockDim.x * 4, consts[0], 0.f);
            part[0] = PA::add(part[0], vs[0]);
            if (arg_cache) st_cache(arg_cache + c, vs[0]);
          }
        }
      }
    }
    Acc acc = PA::to(part[0]);
#pragma unroll
    for (int c = 1; c < CH; ++c) acc = RD::join(acc, PA::to(part[c]));
    const int width = G < 32 ? G : 32;
    for (int o = width / 2; o > 0; o >>= 1) acc = RD::join(acc, __shfl_xor_sync(0xffffffffu, acc, o, width));
    float result;
    if (G <= 32) {
      result = static_cast<float>(acc);
    } else {
      const int warp = threadIdx.x >> 5;
      if ((threadIdx.x & 31) == 0) warp_part[warp] = acc;
      __syncthreads();
      const int wpr = G >> 5;
      if (lane == 0) {
        Acc s = warp_part[sub * wpr];
        for (int w = 1; w < wpr; ++w) s = RD::join(s, warp_part[sub * wpr + w]);
        row_val[sub] = static_cast<float>(s);
      }
      __syncthreads();
      result = row_val[sub];
    }
    if (valid) {
      if (lane == 0 && L.red_out) L.red_out[row] = result;
      if (fuse_post) {
        for (I col0 = h + static_cast<I>(lane) * VEC; col0 < Rb; col0 += span) {
          const int nv = chunks_in_row<CH>(Rb - col0, cstride);
          T v[CH];
          if (Post::kSplitFull && nv == CH)
            Post::template run<VEC, CH, WIDE>(L.post, Tile<I, true, false, STAGED>{row, col0, R, cstride, CH, row_cache, sst}, v,
                                              slots, blockDim.x, consts[1], result);
          else
            Post::template run<VEC, CH, WIDE>(L.post, Tile<I, false, false, STAGED>{row, col0, R, cstride, nv, row_cache, sst}, v,
                                              slots, blockDim.x, consts[1], result);
        }
        if constexpr (UNAL && VEC == 4 && !STAGED) {
          if (unal && DISC_UNAL_HT_TILES && Post::kSplitFull && G == 1) {
            float hv[4], tv[4];
            if (h > 0)
              Post::template run<1, 4, WIDE>(L.post, Tile<I, false>{row, 0, R, 1, static_cast<int>(h), row_cache, sst}, hv,
                                             nullptr, 0, consts[1], result);
            if (R > Rb)
              Post::template run<1, 4, WIDE>(L.post, Tile<I, false>{row, Rb, R, 1, static_cast<int>(R - Rb), row_cache, sst},
                                             tv, nullptr, 0, consts[1], result);
          } else if (unal) {
            for (I e = static_cast<I>(lane); e < h + (R - Rb); e += static_cast<I>(G)) {
              const I c = e < h ? e : Rb + (e - h);
              float vs[1];
              Post::template run<1, 1, WIDE>(L.post, Tile<I, false>{row, c, R, 1, 1, row_cache, sst}, vs,
                                             reinterpret_cast<float*>(slots), blockDim.x * 4, consts[1], result);
            }
          }
        }
      }
    }
    if constexpr (STAGED) {  // copy every staged output slot back, then free the slots
      __syncthreads();
      if (tma) continue;  // outputs went to global memory; the barrier frees this half
      for (int o = 0; o < L.pre.n_outs; ++o)
        if (L.pre.out_slot[o] >= 0)
          copy_span(L.pre.outs[o] + base * L.R, cache0 + L.pre.out_slot[o] * slot_stride, n_el, true);
      for (int o = 0; o < L.post.n_outs; ++o)
        if (L.post.out_slot[o] >= 0)
          copy_span(L.post.outs[o] + base * L.R, cache0 + L.post.out_slot[o] * slot_stride, n_el, true);
      __syncthreads();
    } else if (G > 32) {
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// Short rows (R < 32 floats, scalar, generated programs): one thread per row evaluates its
// whole row at once -- MAXR chunks of one element, fully unrolled and predicated (c < R),
// values in registers -- and reduces them with ONE sequential accumulator (the reference's
// own order, kernels.cpp:234-259).  No column loop, no per-chunk partials; the fused
// epilogue reads the cached reduce argument this thread wrote (no barrier).
//
// Warp-staged variant (STG, L.stage == 3): a thread-per-row warp reads 32 rows whose
// elements sit R floats apart -- every load instruction touches ~R different lines, so
// the L1 replays it ~R times and the kernel is issue/L1-bound (ncu: DRAM 33-42%, issue
// slots 82-88%).  Instead each warp copies its 32 rows' contiguous span of every identity
// operand into shared memory with 128-bit coalesced loads (all of a lane's loads issued
// before any store: up to MAXR/4 x 16 B in flight per thread), the rows are evaluated
// from shared memory (odd R: bank-conflict-free), staged outputs are copied back the same
// way.  Only __syncwarp between the phases: no block barrier, warps stay independent.
template <int U>
__device__ __forceinline__ void warp_copy(float* __restrict__ dst, const float* __restrict__ src, int n, int lane,
                                          bool to_global) {
  const int n4 = n >> 2;
  float4 r[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int i = lane + 32 * u;
    if (i < n4) r[u] = to_global ? reinterpret_cast<const float4*>(src)[i] : __ldg(reinterpret_cast<const float4*>(src) + i);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int i = lane + 32 * u;
    if (i < n4) reinterpret_cast<float4*>(dst)[i] = r[u];
  }
  for (int i = (n4 << 2) + lane; i < n; i += 32) dst[i] = to_global ? src[i] : __ldg(src + i);
}

// Rows per thread of the narrowest short rows (MAXR 8, unstaged): RPT rows' loads are
// issued before any of them is reduced, so a thread keeps RPT x R loads in flight instead
// of R (2-7 floats).  Shared memory (the argument cache) holds RPT x blockDim rows.
#ifndef DISC_SHORT_RPT
#define DISC_SHORT_RPT 1  // A/B s4 on B200 at 4: S=2 2457 -> 1735, S=7 5170 -> 4076 GB/s (56 vs 31 registers, 4x argument cache)
#endif
template <int MAXR, bool STG>
constexpr int short_rpt() { return (!STG && MAXR <= 8) ? DISC_SHORT_RPT : 1; }

template <int KIND, typename Pre, typename Post, int MAXR, bool STG = false>
__device__ __forceinline__ void row_short_body(const disc_reduce_launch& L, const int bx, const int gx) {
  using RD = Red<KIND>;
  using Acc = typename RD::Acc;
  using I = int32_t;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ float consts[2][DISC_MAX_LOADS];
  constexpr int RPT = short_rpt<MAXR, STG>();
  const int rpb = blockDim.x;
  const int64_t slot_stride = (static_cast<int64_t>(rpb) * RPT * L.R + 3) / 4 * 4;
  if constexpr (RPT > 1) {
    pdl_enter(L.pre);
    hoist_consts(L.pre, consts[0]);
    hoist_consts(L.post, consts[1]);
    __syncthreads();
    float* const cache0 = reinterpret_cast<float*>(smem_raw);
    const I R = static_cast<I>(L.R), sst = static_cast<I>(slot_stride);
    const bool fuse_post = L.post.n_instr > 0;
    const int64_t span = static_cast<int64_t>(rpb) * RPT;
    for (int64_t base = static_cast<int64_t>(bx) * span; base < L.K; base += static_cast<int64_t>(gx) * span) {
      float v[RPT][MAXR];
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        const int64_t r64 = base + u * rpb + threadIdx.x;
        float* const rc = L.cache_loads ? cache0 + (u * rpb + threadIdx.x) * L.R : nullptr;
        if (r64 < L.K)
          Pre::template run<1, MAXR, false>(L.pre, Tile<I, false>{static_cast<I>(r64), 0, R, 1, static_cast<int>(R), rc, sst},
                                            v[u], nullptr, 0, consts[0], 0.f);
      }
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        const int64_t r64 = base + u * rpb + threadIdx.x;
        if (r64 >= L.K) continue;
        const I row = static_cast<I>(r64);
        float* const rc = L.cache_loads ? cache0 + (u * rpb + threadIdx.x) * L.R : nullptr;
        float* const ac = (L.arg_slot >= 0 && rc) ? rc + L.arg_slot * slot_stride : nullptr;
        Acc acc = RD::identity();
#pragma unroll
        for (int c = 0; c < MAXR; ++c)
          if (c < R) {
            acc = RD::step(acc, v[u][c]);
            if (ac) ac[c] = v[u][c];
          }
        const float result = static_cast<float>(acc);
        if (L.red_out) L.red_out[row] = result;
        if (fuse_post) {
          float w[MAXR];
          Post::template run<1, MAXR, false>(L.post, Tile<I, false>{row, 0, R, 1, static_cast<int>(R), rc, sst}, w,
                                             nullptr, 0, consts[1], result);
        }
      }
    }
    return;
  }
  float* const cache0 = reinterpret_cast<float*>(smem_raw);
  pdl_enter(L.pre);
  hoist_consts(L.pre, consts[0]);
  hoist_consts(L.post, consts[1]);
  __syncthreads();
  const I R = static_cast<I>(L.R), sst = static_cast<I>(slot_stride);
  float* const row_cache = L.cache_loads ? cache0 + threadIdx.x * L.R : nullptr;
  float* const arg_cache = (L.arg_slot >= 0 && row_cache) ? row_cache + L.arg_slot * slot_stride : nullptr;
  const bool fuse_post = L.post.n_instr > 0;
  const int lane = threadIdx.x & 31;
  const int64_t wofs = static_cast<int64_t>(threadIdx.x & ~31) * L.R;  // this warp's rows in a slot
  for (int64_t base = static_cast<int64_t>(bx) * rpb; base < L.K; base += static_cast<int64_t>(gx) * rpb) {
    const int64_t r64 = base + threadIdx.x;
    int nw = 0;  // this warp's element count (warp-uniform)
    if constexpr (STG) {
      const int64_t w0 = base + (threadIdx.x & ~31);
      const int64_t nr = L.K - w0 < 32 ? L.K - w0 : 32;
      if (nr <= 0) continue;  // the whole warp is past the end
      nw = static_cast<int>(nr * L.R);
      uint32_t seen = 0;
      for (int q = 0; q < 2; ++q) {
        const disc_program& P = q ? L.post : L.pre;
        for (int l = 0; l < P.n_loads; ++l) {
          const int k = P.cache_slot[l];
          if (k < 0 || k == L.arg_slot || P.loads[l].mode != DISC_LOAD_IDENTITY || ((seen >> k) & 1)) continue;
          seen |= 1u << k;
          warp_copy<MAXR / 4>(cache0 + k * slot_stride + wofs, P.loads[l].ptr + w0 * L.R, nw, lane, false);
        }
      }
      __syncwarp();
    }
    if (r64 < L.K) {
      const I row = static_cast<I>(r64);
      float v[MAXR];
      Pre::template run<1, MAXR, false>(L.pre, Tile<I, false, false, STG>{row, 0, R, 1, static_cast<int>(R), row_cache, sst},
                                        v, nullptr, 0, consts[0], 0.f);
      Acc acc = RD::identity();
#pragma unroll
      for (int c = 0; c < MAXR; ++c)
        if (c < R) {
          acc = RD::step(acc, v[c]);
          if (arg_cache) arg_cache[c] = v[c];
        }
      const float result = static_cast<float>(acc);
      if (L.red_out) L.red_out[row] = result;
      if (fuse_post) {
        float w[MAXR];
        Post::template run<1, MAXR, false>(L.post, Tile<I, false, false, STG>{row, 0, R, 1, static_cast<int>(R), row_cache, sst},
                                           w, nullptr, 0, consts[1], result);
      }
    }
    if constexpr (STG) {
      __syncwarp();
      const int64_t w0 = base + (threadIdx.x & ~31);
      for (int q = 0; q < 2; ++q) {
        const disc_program& P = q ? L.post : L.pre;
        for (int o = 0; o < P.n_outs; ++o)
          if (P.out_slot[o] >= 0)
            warp_copy<MAXR / 4>(P.outs[o] + w0 * L.R, cache0 + P.out_slot[o] * slot_stride + wofs, nw, lane, true);
      }
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------------------
// Column schedule: reduce arg collapsed to [K, R, C], reduce over R, C contiguous; viewed
// as rows k*R + r of width C.  A thread owns VEC columns; lpc = L.group lanes span a row
// segment of lpc*VEC columns and a warp covers 32/lpc rows (narrow C packs many rows per
// warp).  Each step a thread evaluates CH rows (row tiles: CH loads in flight for the
// same columns), so only VEC accumulators are live.  8 warps per block; grid.x = K *
// ceil(C / (lpc*VEC)), grid.y = R splits.  Per-thread partials are joined per column
// through shared memory in a fixed order (deterministic).
constexpr int kColThreads = 256;
#ifndef DISC_COL_PIPE
#define DISC_COL_PIPE 0  // software-pipelined full steps in the column pass (A/B s2 on B200: 3144 vs 3858 GB/s, off)
#endif

template <int VEC, bool WIDE, int KIND, typename Pre, int CH>
__device__ __forceinline__ void col_body(const disc_reduce_launch& L, const int bx, const int by) {
  using T = typename Vec<VEC>::T;
  using RD = Red<KIND>;
  using Acc = typename RD::Acc;
  using I = IndexT<WIDE>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ Acc part[kColThreads][VEC];
  __shared__ float consts[DISC_MAX_LOADS];
  const int tid = threadIdx.x;
  T* slots = reinterpret_cast<T*>(smem_raw) + tid;
  pdl_enter(L.pre);
  hoist_consts(L.pre, consts);
  __syncthreads();
  // Q = L.group lanes per row segment (any 1..256): thread tid takes column chunk tid % Q
  // of row slot tid / Q, so a warp reads consecutive chunks across row boundaries (one
  // contiguous span when the tile is the whole row); the 256 % Q leftover threads idle.
  const int Q = L.group;
  const int rows_per_pass = kColThreads / Q;
  const int sub = tid / Q, lc = tid - sub * Q;
  const int warp = sub < rows_per_pass ? 0 : 1;  // 1: an idle leftover thread
  const int64_t span = static_cast<int64_t>(Q) * VEC;
  const int64_t tiles = (L.C + span - 1) / span;
  const int64_t k = bx / tiles;
  const int64_t tile0 = (bx - k * tiles) * span;
  const int64_t col0 = tile0 + lc * VEC;
  const int64_t per = (L.R + L.splits - 1) / L.splits;
  const int64_t r0 = static_cast<int64_t>(by) * per;
  const int64_t r1 = r0 + per < L.R ? r0 + per : L.R;

  using PA = PartAcc<KIND, comp_sum<Pre>()>;
  typename PA::T acc[VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i) acc[i] = PA::identity();
  constexpr bool kIntCvt = DISC_INT_CVT && VEC == 4 && KIND == DISC_REDUCE_SUM && Pre::kXuHeavy && !comp_sum<Pre>();
  auto add = [&](const T& v) {
    if constexpr (VEC == 1) {
      acc[0] = PA::add(acc[0], v);
    } else if constexpr (kIntCvt) {
      double d[4];
      f2d4(v, d);
      acc[0] += d[0];
      acc[1] += d[1];
      acc[2] += d[2];
      acc[3] += d[3];
    } else {
      acc[0] = PA::add(acc[0], v.x);
      acc[1] = PA::add(acc[1], v.y);
      acc[2] = PA::add(acc[2], v.z);
      acc[3] = PA::add(acc[3], v.w);
    }
  };
  if (col0 < L.C && warp == 0) {
    const int64_t step = static_cast<int64_t>(rows_per_pass) * CH;
    int64_t r = r0 + sub;
#if DISC_COL_PIPE
    if constexpr (Pre::kPipe > 0) {
      // Software pipeline over full steps: the next step's streaming loads are issued
      // before the current step computes (CH x VEC floats in flight per thread while the
      // prologue math runs -- the tanh prologue of C3 is long).
      using LD = typename Pre::template Loads<VEC, CH>;
      auto tile = [&](int64_t rr) {
        return Tile<I, true, true>{static_cast<I>(k * L.R + rr), static_cast<I>(col0), static_cast<I>(L.C),
                                   static_cast<I>(rows_per_pass), CH};
      };
      if (r + (CH - 1) * rows_per_pass < r1) {
        LD cur;
        Pre::template load<VEC, CH, WIDE>(L.pre, tile(r), cur);
        for (;;) {
          const int64_t rn = r + step;
          const bool more = rn + (CH - 1) * rows_per_pass < r1;
          LD nxt;
          if (more) Pre::template load<VEC, CH, WIDE>(L.pre, tile(rn), nxt);
          T v[CH];
          Pre::template run_loaded<VEC, CH, WIDE>(L.pre, tile(r), cur, v, slots, kColThreads, consts, 0.f);
#pragma unroll
          for (int c = 0; c < CH; ++c) add(v[c]);
          r = rn;
          if (!more) break;
          cur = nxt;
        }
      }
    }
#endif
    // full steps: all CH rows inside [r0, r1)
    for (; r + (CH - 1) * rows_per_pass < r1; r += step) {
      T v[CH];
      Pre::template run<VEC, CH, WIDE>(
          L.pre, Tile<I, true, true>{static_cast<I>(k * L.R + r), static_cast<I>(col0), static_cast<I>(L.C),
                                     static_cast<I>(rows_per_pass), CH},
          v, slots, kColThreads, consts, 0.f);
#pragma unroll
      for (int c = 0; c < CH; ++c) add(v[c]);
    }
    if (r < r1) {  // last partial step
      const int nv = static_cast<int>((r1 - r + rows_per_pass - 1) / rows_per_pass);
      T v[CH];
      Pre::template run<VEC, CH, WIDE>(
          L.pre, Tile<I, false, true>{static_cast<I>(k * L.R + r), static_cast<I>(col0), static_cast<I>(L.C),
                                      static_cast<I>(rows_per_pass), nv},
          v, slots, kColThreads, consts, 0.f);
#pragma unroll
      for (int c = 0; c < CH; ++c)
        if (c < nv) add(v[c]);
    }
    // folded launch (L.fold > 1, K == 1): the partial last super row -- its first
    // fold_tail * fold_cout columns are real rows -- evaluated element by element, once per
    // column (the first row slot of warp 0), in the last split
    if (L.fold > 1 && L.fold_tail > 0 && by == L.splits - 1 && warp == 0 && sub == 0) {
      const int64_t lim = static_cast<int64_t>(L.fold_tail) * L.fold_cout;
#pragma unroll
      for (int j = 0; j < VEC; ++j)
        if (col0 + j < lim) {
          float vs[1];
          Pre::template run<1, 1, WIDE>(
              L.pre, Tile<I, false, true>{static_cast<I>(L.R), static_cast<I>(col0 + j), static_cast<I>(L.C), 1, 1},
              vs, reinterpret_cast<float*>(smem_raw) + tid, kColThreads, consts, 0.f);
          acc[j] = PA::add(acc[j], vs[0]);
        }
    }
  }
#pragma unroll
  for (int i = 0; i < VEC; ++i) part[tid][i] = PA::to(acc[i]);
  __syncthreads();
  // Column j of the tile: lane lc = j/VEC of each row slot, element j%VEC.
  for (int j = tid; j < span; j += kColThreads) {
    const int64_t col = tile0 + j;
    if (col >= L.C) continue;
    const int jl = j / VEC, e = j % VEC;
    Acc s = RD::identity();
    for (int u = 0; u < rows_per_pass; ++u) s = RD::join(s, part[u * Q + jl][e]);  // row slots in order
    const int64_t o = k * L.C + col;
    switch (L.schedule) {
      case DISC_SCHED_COL_SINGLE:
        if (L.red_out) L.red_out[o] = static_cast<float>(s);
        break;
      case DISC_SCHED_COL_TWOPASS:
        L.workspace[static_cast<int64_t>(by) * L.K * L.C + o] = static_cast<double>(s);
        break;
      default:  // DISC_SCHED_COL_ATOMIC (sum only)
        atomicAdd(L.workspace + o, static_cast<double>(s));
        break;
    }
  }
}

// ---------------------------------------------------------------------------
// Kernels: single launch (descriptor in parameter space) and grouped launch.
template <int VEC, bool WIDE, typename Prog, int CH = kCH>
__global__ void __launch_bounds__(kLoopThreads, 4) k_loop(const __grid_constant__ disc_loop_launch L) {
  loop_body<VEC, WIDE, Prog, CH>(L, blockIdx.x, gridDim.x);
}
template <int VEC, bool WIDE, typename Prog, int CH = kCH>
__global__ void __launch_bounds__(kLoopThreads, 4) k_loop_g(const __grid_constant__ disc_group G) {
  __shared__ __align__(16) unsigned char desc[desc_bytes<disc_loop_launch>()];
  const int b = blockIdx.x, g = group_of(G, b);
  const disc_loop_launch& L = group_stage<disc_loop_launch>(G, g, desc);
  loop_body<VEC, WIDE, Prog, CH>(L, b - G.block_off[g], G.block_off[g + 1] - G.block_off[g]);
}

template <int VEC, bool WIDE, int KIND, typename Pre, typename Post, int CH = kCH, bool STAGED = false, bool UNAL = false>
__global__ void __launch_bounds__(1024) k_row(const __grid_constant__ disc_reduce_launch L) {
  row_body<VEC, WIDE, KIND, Pre, Post, CH, STAGED, UNAL>(L, blockIdx.x, gridDim.x);
}
template <int VEC, bool WIDE, int KIND, typename Pre, typename Post, int CH = kCH, bool STAGED = false, bool UNAL = false>
__global__ void __launch_bounds__(1024) k_row_g(const __grid_constant__ disc_group G) {
  __shared__ __align__(16) unsigned char desc[desc_bytes<disc_reduce_launch>()];
  const int b = blockIdx.x, g = group_of(G, b);
  const disc_reduce_launch& L = group_stage<disc_reduce_launch>(G, g, desc);
  row_body<VEC, WIDE, KIND, Pre, Post, CH, STAGED, UNAL>(L, b - G.block_off[g], G.block_off[g + 1] - G.block_off[g]);
}
// Max-reduce rows of generated programs with two or more streamed operands (BERT's scaled +
// masked scores): <= 256 threads and 6 resident blocks (<= 40 registers).  A/B: that row
// kernel 5522 -> 6155 GB/s, while the single-stream softmax max row loses (5038 -> 4802),
// so the choice is per pattern (Pre::kMaxRowMinBlocks) and per launch (block <= 256).
template <int VEC, bool WIDE, typename Pre, typename Post, int CH, bool STAGED, bool UNAL>
__global__ void __launch_bounds__(256, 6) k_row_mb(const __grid_constant__ disc_reduce_launch L) {
  row_body<VEC, WIDE, DISC_REDUCE_MAX, Pre, Post, CH, STAGED, UNAL>(L, blockIdx.x, gridDim.x);
}
template <int VEC, bool WIDE, typename Pre, typename Post, int CH, bool STAGED, bool UNAL>
__global__ void __launch_bounds__(256, 6) k_row_g_mb(const __grid_constant__ disc_group G) {
  __shared__ __align__(16) unsigned char desc[desc_bytes<disc_reduce_launch>()];
  const int b = blockIdx.x, g = group_of(G, b);
  const disc_reduce_launch& L = group_stage<disc_reduce_launch>(G, g, desc);
  row_body<VEC, WIDE, DISC_REDUCE_MAX, Pre, Post, CH, STAGED, UNAL>(L, b - G.block_off[g],
                                                                   G.block_off[g + 1] - G.block_off[g]);
}

template <int KIND, typename Pre, typename Post, int MAXR, bool STG = false>
__global__ void __launch_bounds__(256) k_row_short(const __grid_constant__ disc_reduce_launch L) {
  row_short_body<KIND, Pre, Post, MAXR, STG>(L, blockIdx.x, gridDim.x);
}
template <int KIND, typename Pre, typename Post, int MAXR, bool STG = false>
__global__ void __launch_bounds__(256) k_row_short_g(const __grid_constant__ disc_group G) {
  __shared__ __align__(16) unsigned char desc[desc_bytes<disc_reduce_launch>()];
  const int b = blockIdx.x, g = group_of(G, b);
  const disc_reduce_launch& L = group_stage<disc_reduce_launch>(G, g, desc);
  row_short_body<KIND, Pre, Post, MAXR, STG>(L, b - G.block_off[g], G.block_off[g + 1] - G.block_off[g]);
}

// Sum rows at <= 256 threads capped at 6 resident blocks (<= 40 registers) -- A/B knob
// DISC_SUM_ROW_MB (the fused softmax epilogue runs at 64 registers, 50% occupancy).
#ifndef DISC_SMB_BLOCKS
#define DISC_SMB_BLOCKS 6
#endif
template <int VEC, bool WIDE, typename Pre, typename Post, int CH, bool STAGED, bool UNAL>
__global__ void __launch_bounds__(256, DISC_SMB_BLOCKS) k_row_smb(const __grid_constant__ disc_reduce_launch L) {
  row_body<VEC, WIDE, DISC_REDUCE_SUM, Pre, Post, CH, STAGED, UNAL>(L, blockIdx.x, gridDim.x);
}
template <int VEC, bool WIDE, typename Pre, typename Post, int CH, bool STAGED, bool UNAL>
__global__ void __launch_bounds__(256, DISC_SMB_BLOCKS) k_row_g_smb(const __grid_constant__ disc_group G) {
  __shared__ __align__(16) unsigned char desc[desc_bytes<disc_reduce_launch>()];
  const int b = blockIdx.x, g = group_of(G, b);
  const disc_reduce_launch& L = group_stage<disc_reduce_launch>(G, g, desc);
  row_body<VEC, WIDE, DISC_REDUCE_SUM, Pre, Post, CH, STAGED, UNAL>(L, b - G.block_off[g],
                                                                   G.block_off[g + 1] - G.block_off[g]);
}

template <int VEC, bool WIDE, int KIND, typename Pre, int CH = kCH>
__global__ void __launch_bounds__(kColThreads, 4) k_col(const __grid_constant__ disc_reduce_launch L) {
  col_body<VEC, WIDE, KIND, Pre, CH>(L, blockIdx.x, blockIdx.y);
}
// Grouped column pass: launch g's 2-D grid (K * col tiles, splits) is flattened x-major.
#ifndef DISC_COL_MINB
#define DISC_COL_MINB 4  // resident blocks of the grouped column pass (4: <= 64 registers)
#endif
template <int VEC, bool WIDE, int KIND, typename Pre, int CH = kCH>
__global__ void __launch_bounds__(kColThreads, DISC_COL_MINB) k_col_g(const __grid_constant__ disc_group G) {
  __shared__ __align__(16) unsigned char desc[desc_bytes<disc_reduce_launch>()];
  const int b = blockIdx.x, g = group_of(G, b);
  const disc_reduce_launch& L = group_stage<disc_reduce_launch>(G, g, desc);
  const int local = b - G.block_off[g];
  const int64_t span = static_cast<int64_t>(L.group) * L.vec;
  const int gx = static_cast<int>(L.K * ((L.C + span - 1) / span));
  col_body<VEC, WIDE, KIND, Pre, CH>(L, local % gx, local / gx);
}
// The same at 6 resident blocks (<= 40 registers) -- A/B knob DISC_COL_MB.
template <int VEC, bool WIDE, int KIND, typename Pre, int CH = kCH>
__global__ void __launch_bounds__(kColThreads, 6) k_col_g_mb(const __grid_constant__ disc_group G) {
  __shared__ __align__(16) unsigned char desc[desc_bytes<disc_reduce_launch>()];
  const int b = blockIdx.x, g = group_of(G, b);
  const disc_reduce_launch& L = group_stage<disc_reduce_launch>(G, g, desc);
  const int local = b - G.block_off[g];
  const int64_t span = static_cast<int64_t>(L.group) * L.vec;
  const int gx = static_cast<int>(L.K * ((L.C + span - 1) / span));
  col_body<VEC, WIDE, KIND, Pre, CH>(L, local % gx, local / gx);
}

// ---------------------------------------------------------------------------
// Host-side launch configuration shared by the interpreter and generated kernels.
// SM count of the calling thread's current device (cached per thread and device).
inline int sm_count() {
  thread_local int dev_cached = -1, n_cached = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return n_cached;
  if (dev != dev_cached) {
    int v = 148;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess) n_cached = v;
    dev_cached = dev;
  }
  return n_cached;
}

// Raises `kernel`'s dynamic shared-memory limit on the current device to at least `bytes`
// (fused.cu).  The attribute is shared by every thread launching the kernel, so it only
// ever grows (per device and kernel, under a lock): a concurrent launch needing less can
// never see it lowered under its feet.
cudaError_t raise_smem_limit(const void* kernel, size_t bytes);

template <typename K>
inline cudaError_t set_smem(K kernel, size_t bytes, size_t threshold = 40 * 1024) {
  if (bytes <= threshold) return cudaSuccess;
  return raise_smem_limit(reinterpret_cast<const void*>(kernel), bytes);
}

// Host side of a grouped launch: the members' host descriptors (full layout, for grid and
// shared-memory sizing) and the uploaded device table of compact member records.
struct HostGroup {
  const void* const* members;
  int n;
  const unsigned char* dev_table;
  int32_t stride;               // record bytes
  int32_t nseg;
  uint16_t seg[DISC_GROUP_SEGS][3];
  template <typename T>
  const T& at(int i) const { return *static_cast<const T*>(members[i]); }
  void fill(disc_group& G) const {
    G.table = dev_table;
    G.stride = stride;
    G.n = n;
    G.nseg = nseg;
    for (int k = 0; k < nseg; ++k)
      for (int j = 0; j < 3; ++j) G.seg[k][j] = seg[k][j];
  }
};
// Grouped kernels hold a descriptor in static shared memory: opt in to more dynamic
// shared memory earlier than single launches do.
constexpr size_t kGroupSmemThreshold = 24 * 1024;

// Resident CTAs per SM for (kernel, block, dynamic smem); grid-stride kernels are sized
// to exactly one wave (SM count x this).  Cached per host thread.
int resident_ctas(const void* kernel, int block, size_t smem);

// PDL mode (disc_cuda_set_pdl); launches go through cudaLaunchKernelEx.  Off while this
// thread captures a CUDA graph (set_capturing).
bool pdl_enabled();
void set_capturing(bool on);

template <typename Arg>
inline cudaError_t launch_k(void (*kernel)(Arg), dim3 grid, dim3 block, size_t smem, cudaStream_t s, const Arg& a) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, a);
}

template <int CH>
inline int64_t loop_blocks_wanted(const disc_loop_launch& L) {
  if (L.total <= 0) return 0;
  const int64_t span = static_cast<int64_t>(L.lpr) * CH * L.vec;
  const int64_t rpw = 32 / L.lpr;
  const int64_t tiles = ((L.rows + rpw - 1) / rpw) * ((L.W + span - 1) / span);
  const int64_t warps_per_block = kLoopThreads / 32;
  return (tiles + warps_per_block - 1) / warps_per_block;
}
template <int CH>
inline size_t loop_smem(const disc_loop_launch& L, bool use_slots) {
  return use_slots ? static_cast<size_t>(L.prog.n_slots) * CH * kLoopThreads * (L.vec == 4 ? 16 : 4) : 0;
}

// use_slots = false for generated programs (values live in registers, no slot smem).
template <int CH = kCH, typename K>
inline cudaError_t launch_loop_with(K kernel, const disc_loop_launch& L, cudaStream_t s, bool use_slots = true) {
  if (L.total <= 0) return cudaSuccess;
  const int64_t want = loop_blocks_wanted<CH>(L);
  const size_t smem = loop_smem<CH>(L, use_slots);
  cudaError_t e = set_smem(kernel, smem);
  if (e != cudaSuccess) return e;
  const int64_t cap = static_cast<int64_t>(sm_count()) * resident_ctas(reinterpret_cast<const void*>(kernel), kLoopThreads, smem);
  const int grid = static_cast<int>(want < cap ? want : cap);
  e = launch_k(kernel, dim3(grid), dim3(kLoopThreads), smem, s, L);
  return e != cudaSuccess ? e : cudaGetLastError();
}

inline int row_block(const disc_reduce_launch& L) { return L.group > 256 ? L.group : 256; }
template <int CH>
inline size_t row_smem(const disc_reduce_launch& L, bool use_slots) {
  const int slots = L.pre.n_slots > L.post.n_slots ? L.pre.n_slots : L.post.n_slots;
  const int block = row_block(L);
  const int rpb = block / L.group;
  const int64_t rrow = L.row_pitch ? L.row_pitch : (L.vec == 4 && L.unaligned) ? (L.R + 6) / 4 * 4 : L.R;
  const int rpt = (L.short_rows && L.short_rows <= 8 && L.stage != 3) ? short_rpt<8, false>() : 1;  // row_short_body
  const size_t cache = static_cast<size_t>((static_cast<int64_t>(rpb) * rpt * rrow + 3) / 4 * 4) * L.cache_loads * 4 *
                       (L.stage == 2 ? 2 : 1);  // TMA staging: double buffer
  return cache + (use_slots ? static_cast<size_t>(slots) * CH * block * (L.vec == 4 ? 16 : 4) : 0);
}

template <int CH = kCH, typename K>
inline cudaError_t launch_row_with(K kernel, const disc_reduce_launch& L, cudaStream_t s, bool use_slots = true) {
  if (L.K <= 0) return cudaSuccess;
  const int block = row_block(L);
  const int rpb = block / L.group;
  const int64_t groups = (L.K + rpb - 1) / rpb;
  const size_t smem = row_smem<CH>(L, use_slots);
  cudaError_t e = set_smem(kernel, smem);
  if (e != cudaSuccess) return e;
  const int64_t cap = static_cast<int64_t>(sm_count()) * resident_ctas(reinterpret_cast<const void*>(kernel), block, smem);
  const int grid = static_cast<int>(groups < cap ? groups : cap);
  e = launch_k(kernel, dim3(grid), dim3(block), smem, s, L);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// Column pass only (the finalize kernel is launched by the caller).
template <int CH = kCH, typename K>
inline cudaError_t launch_col_with(K kernel, const disc_reduce_launch& L, cudaStream_t s, bool use_slots = true) {
  const int64_t span = static_cast<int64_t>(L.group) * L.vec;
  const int64_t tiles = (L.C + span - 1) / span;
  dim3 grid(static_cast<unsigned>(L.K * tiles), static_cast<unsigned>(L.splits));
  const size_t smem = use_slots ? static_cast<size_t>(L.pre.n_slots) * CH * kColThreads * (L.vec == 4 ? 16 : 4) : 0;
  cudaError_t e = set_smem(kernel, smem);
  if (e != cudaSuccess) return e;
  e = launch_k(kernel, grid, dim3(kColThreads), smem, s, L);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// Grouped launches (see disc_group).  The group's CTAs are concatenated in table order.
// CTA budget: a few waves of the kernel shared by all members in proportion to their
// work units (warp tiles / row groups), every member >= 1 CTA and never more than it can
// use or than one wave (its single-launch grid).  Members grid-stride over their units,
// so per-CTA startup (descriptor staging, dependency wait) is amortised over many units
// instead of every member paying a full wave.
int group_waves();  // DISC_GROUP_WAVES (default 16; A/B on C2: 1 -> 3453, 4 -> 4855, 8 -> 5211, 16 -> 5225 GB/s)

inline void group_blocks(const int64_t* units, int n, int64_t cap, int32_t* off) {
  int64_t total = 0;
  for (int i = 0; i < n; ++i) total += units[i] > 0 ? units[i] : 0;
  const int64_t budget = static_cast<int64_t>(group_waves()) * cap;
  int64_t o = 0;
  for (int i = 0; i < n; ++i) {
    off[i] = static_cast<int32_t>(o);
    if (units[i] <= 0) continue;
    int64_t b = total <= budget ? units[i] : (budget * units[i] + total - 1) / total;
    b = std::max<int64_t>(1, std::min({b, units[i], cap}));
    o += b;
  }
  off[n] = static_cast<int32_t>(o);
}
template <int CH = kCH, typename K>
inline cudaError_t launch_loop_group(K kernel, const HostGroup& H, cudaStream_t s, bool use_slots) {
  disc_group G;
  H.fill(G);
  size_t smem = 0;
  for (int i = 0; i < H.n; ++i) smem = std::max(smem, loop_smem<CH>(H.at<disc_loop_launch>(i), use_slots));
  cudaError_t e = set_smem(kernel, smem, kGroupSmemThreshold);
  if (e != cudaSuccess) return e;
  const int64_t cap = static_cast<int64_t>(sm_count()) * resident_ctas(reinterpret_cast<const void*>(kernel), kLoopThreads, smem);
  int64_t units[DISC_MAX_GROUP];
  for (int i = 0; i < H.n; ++i) units[i] = loop_blocks_wanted<CH>(H.at<disc_loop_launch>(i));
  group_blocks(units, H.n, cap, G.block_off);
  const int64_t off = G.block_off[H.n];
  if (off == 0) return cudaSuccess;
  e = launch_k(kernel, dim3(static_cast<unsigned>(off)), dim3(kLoopThreads), smem, s, G);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int CH = kCH, typename K>
inline cudaError_t launch_row_group(K kernel, const HostGroup& H, cudaStream_t s, bool use_slots) {
  disc_group G;
  H.fill(G);
  size_t smem = 0;
  for (int i = 0; i < H.n; ++i) smem = std::max(smem, row_smem<CH>(H.at<disc_reduce_launch>(i), use_slots));
  const int block = row_block(H.at<disc_reduce_launch>(0));
  cudaError_t e = set_smem(kernel, smem, kGroupSmemThreshold);
  if (e != cudaSuccess) return e;
  const int64_t cap = static_cast<int64_t>(sm_count()) * resident_ctas(reinterpret_cast<const void*>(kernel), block, smem);
  int64_t units[DISC_MAX_GROUP];
  for (int i = 0; i < H.n; ++i) {
    const disc_reduce_launch& L = H.at<disc_reduce_launch>(i);
    units[i] = L.K > 0 ? (L.K + block / L.group - 1) / (block / L.group) : 0;
  }
  group_blocks(units, H.n, cap, G.block_off);
  const int64_t off = G.block_off[H.n];
  if (off == 0) return cudaSuccess;
  e = launch_k(kernel, dim3(static_cast<unsigned>(off)), dim3(block), smem, s, G);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int CH = kCH, typename K>
inline cudaError_t launch_col_group(K kernel, const HostGroup& H, cudaStream_t s, bool use_slots) {
  disc_group G;
  H.fill(G);
  size_t smem = 0;
  int64_t off = 0;
  for (int i = 0; i < H.n; ++i) {
    const disc_reduce_launch& L = H.at<disc_reduce_launch>(i);
    smem = std::max(smem, use_slots ? static_cast<size_t>(L.pre.n_slots) * CH * kColThreads * (L.vec == 4 ? 16 : 4) : 0);
    G.block_off[i] = static_cast<int32_t>(off);
    const int64_t span = static_cast<int64_t>(L.group) * L.vec;
    if (L.K * L.C > 0) off += L.K * ((L.C + span - 1) / span) * L.splits;
  }
  G.block_off[H.n] = static_cast<int32_t>(off);
  if (off == 0) return cudaSuccess;
  cudaError_t e = set_smem(kernel, smem, kGroupSmemThreshold);
  if (e != cudaSuccess) return e;
  e = launch_k(kernel, dim3(static_cast<unsigned>(off)), dim3(kColThreads), smem, s, G);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// Scalar (VEC=1) instantiations keep as many bytes in flight per thread as the float4
// ones: DISC_VEC1_CH_SCALE x the chunks (capped at 8).
#ifndef DISC_VEC1_CH_SCALE
#define DISC_VEC1_CH_SCALE 1  // A/B: 4 (CH 8 at VEC=1) is 1.4-2.8x slower on odd-width softmax rows
#endif
constexpr int vec1_ch(int ch) { return ch * DISC_VEC1_CH_SCALE < 8 ? ch * DISC_VEC1_CH_SCALE : (ch > 8 ? ch : 8); }

template <typename Prog, int CH = kCH, bool ALLOW_WIDE = true>
inline cudaError_t loop_pass(const disc_loop_launch& L, cudaStream_t s, bool use_slots, const HostGroup* g) {
  constexpr int C1 = vec1_ch(CH);
  if (g) {
    if constexpr (ALLOW_WIDE)
      if (L.wide) return L.vec == 4 ? launch_loop_group<CH>(k_loop_g<4, true, Prog, CH>, *g, s, use_slots)
                                    : launch_loop_group<C1>(k_loop_g<1, true, Prog, C1>, *g, s, use_slots);
    return L.vec == 4 ? launch_loop_group<CH>(k_loop_g<4, false, Prog, CH>, *g, s, use_slots)
                      : launch_loop_group<C1>(k_loop_g<1, false, Prog, C1>, *g, s, use_slots);
  }
  if constexpr (ALLOW_WIDE)
    if (L.wide) return L.vec == 4 ? launch_loop_with<CH>(k_loop<4, true, Prog, CH>, L, s, use_slots)
                                  : launch_loop_with<C1>(k_loop<1, true, Prog, C1>, L, s, use_slots);
  return L.vec == 4 ? launch_loop_with<CH>(k_loop<4, false, Prog, CH>, L, s, use_slots)
                    : launch_loop_with<C1>(k_loop<1, false, Prog, C1>, L, s, use_slots);
}

bool col_mb();  // DISC_COL_MB (fused.cu)

template <int V, bool W, typename Pre, typename Post, int C, bool ST, bool U>
inline void (*sum_row_kernel(const disc_reduce_launch& L))(disc_reduce_launch) {
  if (L.regcap && row_block(L) <= 256) return k_row_smb<V, W, Pre, Post, C, ST, U>;
  return k_row<V, W, DISC_REDUCE_SUM, Pre, Post, C, ST, U>;
}
template <int V, bool W, typename Pre, typename Post, int C, bool ST, bool U>
inline void (*sum_row_group_kernel(const HostGroup& H))(disc_group) {
  const disc_reduce_launch& L = H.at<disc_reduce_launch>(0);  // the group key includes regcap
  if (L.regcap && row_block(L) <= 256) return k_row_g_smb<V, W, Pre, Post, C, ST, U>;
  return k_row_g<V, W, DISC_REDUCE_SUM, Pre, Post, C, ST, U>;
}

// Max-reduce row kernel for a launch (k_row_mb when the pattern asks for it and the
// launch's block is <= 256 threads).
template <int V, bool W, typename Pre, typename Post, int C, bool ST, bool U>
inline void (*max_row_kernel(const disc_reduce_launch& L))(disc_reduce_launch) {
  if constexpr (Pre::kMaxRowMinBlocks > 0)
    if (row_block(L) <= 256) return k_row_mb<V, W, Pre, Post, C, ST, U>;
  return k_row<V, W, DISC_REDUCE_MAX, Pre, Post, C, ST, U>;
}
template <int V, bool W, typename Pre, typename Post, int C, bool ST, bool U>
inline void (*max_row_group_kernel(const HostGroup& H))(disc_group) {
  if constexpr (Pre::kMaxRowMinBlocks > 0)
    if (row_block(H.at<disc_reduce_launch>(0)) <= 256) return k_row_g_mb<V, W, Pre, Post, C, ST, U>;
  return k_row_g<V, W, DISC_REDUCE_MAX, Pre, Post, C, ST, U>;
}

// Dispatch on (vec, wide, reduce kind) for a given program functor pair.
// ALLOW_WIDE = false (generated programs, used only on !wide launches) instantiates no
// 64-bit-index kernels.
template <typename Pre, typename Post, int CH = kCH, bool ALLOW_WIDE = true>
inline cudaError_t row_pass(const disc_reduce_launch& L, cudaStream_t s, bool use_slots, const HostGroup* g = nullptr) {
  const bool sum = L.kind == DISC_REDUCE_SUM;
  constexpr int C1 = vec1_ch(CH);
#define DISC_ROW_U(V, W, ST, C, U)                                                                           \
  (g ? (sum ? launch_row_group<C>(sum_row_group_kernel<V, W, Pre, Post, C, ST, U>(*g), *g, s, use_slots)     \
            : launch_row_group<C>(max_row_group_kernel<V, W, Pre, Post, C, ST, U>(*g), *g, s, use_slots))    \
     : (sum ? launch_row_with<C>(sum_row_kernel<V, W, Pre, Post, C, ST, U>(L), L, s, use_slots)         \
            : launch_row_with<C>(max_row_kernel<V, W, Pre, Post, C, ST, U>(L), L, s, use_slots)))
#define DISC_ROW(V, W, ST, C) DISC_ROW_U(V, W, ST, C, false)
  if constexpr (ALLOW_WIDE)
    if (L.wide) return L.vec == 4 ? (L.unaligned ? DISC_ROW_U(4, true, false, CH, true) : DISC_ROW(4, true, false, CH))
                                  : DISC_ROW(1, true, false, C1);
  if constexpr (!std::is_same<Pre, Interp>::value) {  // register-resident short rows (generated programs)
    if (L.short_rows) {
#define DISC_ROWS(M, ST)                                                                                          \
  (g ? (sum ? launch_row_group<1>(k_row_short_g<DISC_REDUCE_SUM, Pre, Post, M, ST>, *g, s, false)                 \
            : launch_row_group<1>(k_row_short_g<DISC_REDUCE_MAX, Pre, Post, M, ST>, *g, s, false))                \
     : (sum ? launch_row_with<1>(k_row_short<DISC_REDUCE_SUM, Pre, Post, M, ST>, L, s, false)                     \
            : launch_row_with<1>(k_row_short<DISC_REDUCE_MAX, Pre, Post, M, ST>, L, s, false)))
      if (L.stage == 3) return L.short_rows <= 8 ? DISC_ROWS(8, true) : DISC_ROWS(32, true);
      return L.short_rows <= 8 ? DISC_ROWS(8, false) : DISC_ROWS(32, false);
#undef DISC_ROWS
    }
  }
  if (L.stage) return L.vec == 4 ? DISC_ROW(4, false, true, CH) : DISC_ROW(1, false, true, CH);
  if (L.vec == 4) return L.unaligned ? DISC_ROW_U(4, false, false, CH, true) : DISC_ROW(4, false, false, CH);
  return DISC_ROW(1, false, false, C1);
#undef DISC_ROW
#undef DISC_ROW_U
}

template <typename Pre, int CH = kCH, bool ALLOW_WIDE = true>
inline cudaError_t col_pass_t(const disc_reduce_launch& L, cudaStream_t s, bool use_slots, const HostGroup* g = nullptr) {
  const bool sum = L.kind == DISC_REDUCE_SUM;
  if (g) {
#define DISC_COLG(V, W)                                                                                   \
  (sum ? launch_col_group<CH>(col_mb() ? k_col_g_mb<V, W, DISC_REDUCE_SUM, Pre, CH> : k_col_g<V, W, DISC_REDUCE_SUM, Pre, CH>, \
                              *g, s, use_slots)                                                           \
       : launch_col_group<CH>(col_mb() ? k_col_g_mb<V, W, DISC_REDUCE_MAX, Pre, CH> : k_col_g<V, W, DISC_REDUCE_MAX, Pre, CH>, \
                              *g, s, use_slots))
    if constexpr (ALLOW_WIDE)
      if (L.wide) return L.vec == 4 ? DISC_COLG(4, true) : DISC_COLG(1, true);
    return L.vec == 4 ? DISC_COLG(4, false) : DISC_COLG(1, false);
#undef DISC_COLG
  }
  if constexpr (ALLOW_WIDE) if (L.wide) {
    if (L.vec == 4) return sum ? launch_col_with<CH>(k_col<4, true, DISC_REDUCE_SUM, Pre, CH>, L, s, use_slots)
                               : launch_col_with<CH>(k_col<4, true, DISC_REDUCE_MAX, Pre, CH>, L, s, use_slots);
    return sum ? launch_col_with<CH>(k_col<1, true, DISC_REDUCE_SUM, Pre, CH>, L, s, use_slots)
               : launch_col_with<CH>(k_col<1, true, DISC_REDUCE_MAX, Pre, CH>, L, s, use_slots);
  }
  if (L.vec == 4) return sum ? launch_col_with<CH>(k_col<4, false, DISC_REDUCE_SUM, Pre, CH>, L, s, use_slots)
                             : launch_col_with<CH>(k_col<4, false, DISC_REDUCE_MAX, Pre, CH>, L, s, use_slots);
  return sum ? launch_col_with<CH>(k_col<1, false, DISC_REDUCE_SUM, Pre, CH>, L, s, use_slots)
             : launch_col_with<CH>(k_col<1, false, DISC_REDUCE_MAX, Pre, CH>, L, s, use_slots);
}

}  // namespace disc_dev
