// Device interpreter for lowered fusion tapes (disc_program), v2.
//
// One dispatch evaluates an instruction on a TILE of CH chunks x VEC elements of one row
// of the launch's [rows, W] view (f = row*W + col): the opcode (operand modes folded in)
// is decoded once per tile through a single jump table, then applied to CH*VEC elements
// held in registers.  The accumulator lives in registers; values used out of order live
// in per-thread shared-memory slots.  Loads are mostly 2D-affine in (row, col), so no
// per-element division is needed; scalar constants are hoisted into shared memory once
// per block.  Instruction words and load descriptors are read from __grid_constant__
// parameter space (warp-uniform).
#pragma once

#include <cstdint>

#include "disc_cuda.h"

namespace disc_dev {

template <int VEC>
struct Vec;
template <>
struct Vec<1> {
  using T = float;
};
template <>
struct Vec<4> {
  using T = float4;
};

__device__ __forceinline__ float op_max(float a, float b) { return (a < b) ? b : a; }  // std::max(a,b)

__device__ __forceinline__ float rcp_approx(float b) {
  float r;
  asm("rcp.approx.f32 %0, %1;" : "=f"(r) : "f"(b));  // rel. error 2^-23; 1/0 = inf, 1/inf = 0
  return r;
}

template <int OP>
__device__ __forceinline__ float bin1(float a, float b) {
  if constexpr (OP == 0) return __fadd_rn(a, b);
  if constexpr (OP == 1) return __fsub_rn(a, b);
  if constexpr (OP == 2) return __fmul_rn(a, b);
  if constexpr (OP == 3) return __fdiv_rn(a, b);  // IEEE: unfused plans are bit-exact
  if constexpr (OP == 5) return __fmul_rn(a, rcp_approx(b));  // DISC_OP_FDIV (fused groups)
  return op_max(a, b);
}
#ifndef DISC_FAST_TANH
#define DISC_FAST_TANH 1
#endif
// tanh in two ranges, both <= 1 ulp-ish relative (north star: 1e-5 relative, not floored):
//  * |x| < 0.5: odd minimax polynomial x + x^3 P(x^2), P of degree 3 on the FMA pipe
//    (<= 0.84 ulp over every f32 in [2^-12, 0.5], coefficients fitted by Lawson-weighted
//    least squares on the relative error by tools/fit_tanh.py);
//  * |x| >= 0.5: sign(x) (1 - 2 / (2^(2 log2(e) |x|) + 1)) on the MUFU ex2/rcp units: absolute
//    error <= 3e-7 and tanh >= 0.46, so relative error <= 7e-7.  (The exp form alone was
//    only absolute-accurate: ~1e-3 relative just above 2^-12.)
//  * |x| < 2^-12: tanh(x) rounds to x; returned exactly, sign included.
// The two branches cost about the same (7-8 instructions); libdevice tanhf is ~18.
#ifndef DISC_TANH_NEWTON
#define DISC_TANH_NEWTON 0  // A/B on B200: -6% on the tanh column reduce, -1..3% elsewhere
#endif
#ifndef DISC_TANH_BRANCHFREE
#define DISC_TANH_BRANCHFREE 0
#endif
__device__ __forceinline__ float tanh_fast(float x) {
  const float ax = fabsf(x);
#if DISC_TANH_BRANCHFREE
  {  // both ranges evaluated, one select: no reconvergence per element, chains interleave
    const float s = __fmul_rn(x, x);
    float p = __fmaf_rn(0.01724148355424404f, s, -0.05304549261927605f);
    p = __fmaf_rn(p, s, 0.13325878977775574f);
    p = __fmaf_rn(p, s, -0.333331435918808f);
    const float y = __fmaf_rn(__fmul_rn(s, x), p, x);
    float t, r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(__fmul_rn(ax, 2.8853900817779268f)));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(__fadd_rn(t, 1.0f)));
    const float e = copysignf(__fmaf_rn(-2.0f, r, 1.0f), x);
    return ax < 0.5f ? (ax < 2.44140625e-4f ? x : y) : e;
  }
#endif
  if (ax < 0.5f) {
    const float s = __fmul_rn(x, x);
    float p = __fmaf_rn(0.01724148355424404f, s, -0.05304549261927605f);
    p = __fmaf_rn(p, s, 0.13325878977775574f);
    p = __fmaf_rn(p, s, -0.333331435918808f);
    const float y = __fmaf_rn(__fmul_rn(s, x), p, x);
    return ax < 2.44140625e-4f ? x : y;
  }
  float t, r;
#if DISC_TANH_NEWTON
  // one MUFU op (ex2) instead of two: 1 / (t + 1) by Newton iterations on the FMA pipe from
  // a bit-trick seed (|x| clamped at 9.5, where tanh rounds to 1 in f32)
  const float p = __fmul_rn(fminf(ax, 9.5f), 2.8853900817779268f);
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(p));
  const float d = __fadd_rn(t, 1.0f);
  r = __int_as_float(0x7EF311C3 - __float_as_int(d));
  r = __fmul_rn(r, __fmaf_rn(-d, r, 2.0f));
  r = __fmul_rn(r, __fmaf_rn(-d, r, 2.0f));
  r = __fmul_rn(r, __fmaf_rn(-d, r, 2.0f));
#else
  const float p = __fmul_rn(ax, 2.8853900817779268f);  // 2 log2(e)
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(p));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(__fadd_rn(t, 1.0f)));  // t = inf -> r = 0 -> 1
#endif
  return copysignf(__fmaf_rn(-2.0f, r, 1.0f), x);  // NaN: ax < 0.5 false -> NaN propagates
}

// tanh's two ranges as separate straight-line paths (same arithmetic as tanh_fast).
__device__ __forceinline__ float tanh_poly(float x) {  // |x| < 0.5
  const float s = __fmul_rn(x, x);
  float p = __fmaf_rn(0.01724148355424404f, s, -0.05304549261927605f);
  p = __fmaf_rn(p, s, 0.13325878977775574f);
  p = __fmaf_rn(p, s, -0.333331435918808f);
  const float y = __fmaf_rn(__fmul_rn(s, x), p, x);
  return fabsf(x) < 2.44140625e-4f ? x : y;
}
// 2^p on the FMA pipe for p in [0, 30] (DISC_TANH_EXP_POLY): p = n + f with n the nearest
// integer (magic-number rounding, no F2I), 2^f by its degree-7 Taylor polynomial on
// |f| <= 0.5 (relative error ~1e-9), n added to the exponent field.
#ifndef DISC_TANH_EXP_POLY
#define DISC_TANH_EXP_POLY 0
#endif
__device__ __forceinline__ float exp2_fma(float p) {
  const float j = __fadd_rn(p, 12582912.0f);  // 1.5 * 2^23
  const float f = __fsub_rn(p, __fsub_rn(j, 12582912.0f));
  float q = 1.5252734e-5f;
  q = __fmaf_rn(q, f, 1.5403530e-4f);
  q = __fmaf_rn(q, f, 1.3333558e-3f);
  q = __fmaf_rn(q, f, 9.6181291e-3f);
  q = __fmaf_rn(q, f, 5.5504109e-2f);
  q = __fmaf_rn(q, f, 2.4022651e-1f);
  q = __fmaf_rn(q, f, 6.9314718e-1f);
  q = __fmaf_rn(q, f, 1.0f);
  return __int_as_float(__float_as_int(q) + ((__float_as_int(j) - 0x4B400000) << 23));
}
__device__ __forceinline__ float tanh_exp(float x) {  // |x| >= 0.5 (and NaN)
  float t, r;
#if DISC_TANH_EXP_POLY
  const float p = __fmul_rn(fabsf(x), 2.8853900817779268f);
  t = exp2_fma(p < 30.0f ? p : 30.0f);  // tanh rounds to 1 from 2^30 on; NaN -> handled below
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(__fadd_rn(t, 1.0f)));
  const float y = copysignf(__fmaf_rn(-2.0f, r, 1.0f), x);
  return x != x ? x : y;
#else
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(__fmul_rn(fabsf(x), 2.8853900817779268f)));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(__fadd_rn(t, 1.0f)));
  return copysignf(__fmaf_rn(-2.0f, r, 1.0f), x);
#endif
}
// Warp-uniform range dispatch (DISC_TANH_VOTE): when no active lane has an argument below
// 0.5 (the column reduce's x + b) only the exp path runs; otherwise (GELU on normalised
// activations, where tanh_fast's per-element branch diverged) both paths run and one is
// selected, without per-element reconvergence.  Results are identical to tanh_fast.
// A/B s5/s6 on B200 vs tanh_fast: column reduce 3863 -> 4175 GB/s, LN+GELU K2 5393 -> 5496,
// BERT flat, sweep 4332 -> 4428; both paths always (DISC_TANH_BRANCHFREE): LN K2 5734 but
// the column reduce 2906.
#ifndef DISC_TANH_VOTE
#define DISC_TANH_VOTE 1
#endif
#ifndef DISC_TANH_TILE_VOTE
#define DISC_TANH_TILE_VOTE 1  // generated programs: one vote per tile (un_tile), not per float4
#endif
__device__ __forceinline__ float tanh_vote(float x) {
  const bool small = fabsf(x) < 0.5f;
  const unsigned m = __activemask();
  if (!__any_sync(m, small)) return tanh_exp(x);
  const float y = tanh_poly(x), e = tanh_exp(x);
  return small ? y : e;
}
__device__ __forceinline__ float4 tanh_vote(float4 a) {
  const bool sx = fabsf(a.x) < 0.5f, sy = fabsf(a.y) < 0.5f, sz = fabsf(a.z) < 0.5f, sw = fabsf(a.w) < 0.5f;
  const unsigned m = __activemask();
  if (!__any_sync(m, sx || sy || sz || sw)) return make_float4(tanh_exp(a.x), tanh_exp(a.y), tanh_exp(a.z), tanh_exp(a.w));
  const float4 y = make_float4(tanh_poly(a.x), tanh_poly(a.y), tanh_poly(a.z), tanh_poly(a.w));
  const float4 e = make_float4(tanh_exp(a.x), tanh_exp(a.y), tanh_exp(a.z), tanh_exp(a.w));
  return make_float4(sx ? y.x : e.x, sy ? y.y : e.y, sz ? y.z : e.z, sw ? y.w : e.w);
}

// A unary op over a tile's CH chunks (generated programs).  tanh: ONE warp vote for the
// whole tile, so the exp-only path of every chunk is straight-line code the compiler can
// interleave (per-float4 votes left 4 branch-separated chains per step).
__device__ __forceinline__ bool tanh_small(float x) { return fabsf(x) < 0.5f; }
__device__ __forceinline__ bool tanh_small(float4 a) {
  return tanh_small(a.x) || tanh_small(a.y) || tanh_small(a.z) || tanh_small(a.w);
}
__device__ __forceinline__ float tanh_exp_v(float x) { return tanh_exp(x); }
__device__ __forceinline__ float4 tanh_exp_v(float4 a) {
  return make_float4(tanh_exp(a.x), tanh_exp(a.y), tanh_exp(a.z), tanh_exp(a.w));
}
__device__ __forceinline__ float tanh_both(float x) {
  const float y = tanh_poly(x), e = tanh_exp(x);
  return fabsf(x) < 0.5f ? y : e;
}
__device__ __forceinline__ float4 tanh_both(float4 a) {
  return make_float4(tanh_both(a.x), tanh_both(a.y), tanh_both(a.z), tanh_both(a.w));
}

template <int OP>
__device__ __forceinline__ float un1(float a) {
  if constexpr (OP == 0) return expf(a);
  if constexpr (OP == 1) {
#if DISC_FAST_TANH && DISC_TANH_VOTE
    return tanh_vote(a);
#elif DISC_FAST_TANH
    return tanh_fast(a);
#else
    return tanhf(a);
#endif
  }
  return -a;
}
template <int OP>
__device__ __forceinline__ float bin(float a, float b) { return bin1<OP>(a, b); }
template <int OP>
__device__ __forceinline__ float4 bin(float4 a, float4 b) {
  return make_float4(bin1<OP>(a.x, b.x), bin1<OP>(a.y, b.y), bin1<OP>(a.z, b.z), bin1<OP>(a.w, b.w));
}
template <int OP>
__device__ __forceinline__ float un(float a) { return un1<OP>(a); }
template <int OP>
__device__ __forceinline__ float4 un(float4 a) {
#if DISC_FAST_TANH && DISC_TANH_VOTE
  if constexpr (OP == 1) return tanh_vote(a);
#endif
  return make_float4(un1<OP>(a.x), un1<OP>(a.y), un1<OP>(a.z), un1<OP>(a.w));
}
template <int OP, typename T, int CH>
__device__ __forceinline__ void un_tile(const T (&a)[CH], T (&o)[CH]) {
#if DISC_FAST_TANH && DISC_TANH_VOTE && DISC_TANH_TILE_VOTE
  if constexpr (OP == 1) {
    bool sm = false;
#pragma unroll
    for (int c = 0; c < CH; ++c) sm |= tanh_small(a[c]);
    if (!__any_sync(__activemask(), sm)) {
#pragma unroll
      for (int c = 0; c < CH; ++c) o[c] = tanh_exp_v(a[c]);
    } else {
#pragma unroll
      for (int c = 0; c < CH; ++c) o[c] = tanh_both(a[c]);
    }
    return;
  }
#endif
#pragma unroll
  for (int c = 0; c < CH; ++c) o[c] = un<OP>(a[c]);
}

__device__ __forceinline__ float splat(float v, float) { return v; }
__device__ __forceinline__ float4 splat(float v, float4) { return make_float4(v, v, v, v); }

// u32 fast division (n < 2^31): q = umulhi(n, magic) >> shift; magic 0 means d == 1.
__device__ __forceinline__ uint32_t fdiv(uint32_t n, uint32_t magic, uint32_t shift) {
  return magic ? (__umulhi(n, magic) >> shift) : n;
}

template <bool WIDE>
__device__ __forceinline__ int64_t gather_index(const disc_load& L, int64_t f) {
  int64_t src = L.offset;
  if (WIDE) {
    int64_t rem = f;
    for (int d = L.rank - 1; d > 0; --d) {
      const int64_t dim = L.dims[d];
      const int64_t q = rem / dim;
      src += (rem - q * dim) * L.strides[d];
      rem = q;
    }
    src += rem * L.strides[0];
  } else {
    uint32_t rem = static_cast<uint32_t>(f);
    for (int d = L.rank - 1; d > 0; --d) {
      const uint32_t q = fdiv(rem, L.magic[d], L.shift[d]);
      src += static_cast<int64_t>(rem - q * static_cast<uint32_t>(L.dims[d])) * L.strides[d];
      rem = q;
    }
    src += static_cast<int64_t>(rem) * L.strides[0];
  }
  return src;
}

__device__ __forceinline__ float ldg(const float* p) { return __ldg(p); }

// Stores (and cache reads) the compiler cannot see as memory writes (asm volatile, no
// memory clobber).  Grouped kernels read their launch descriptor from shared memory; a
// plain store through a generic pointer may alias it, so every descriptor field used in
// a loop was re-read (LDS) after each output / row-cache store -- ~10 extra instructions
// per element in short-row kernels.  These accesses never touch the descriptor (outputs
// are global, caches are the dynamic shared-memory slots), and volatile asm keeps their
// order among themselves; __syncthreads() orders them against everything else.
#ifndef DISC_NC_STORES
#define DISC_NC_STORES 0  // A/B r2x on the sweep: 1 = 4311, 0 = 4376 GB/s (volatile asm costs the row kernels more)
#endif
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void st_out(float* p, float v) {
  if constexpr (DISC_NC_STORES) asm volatile("st.global.f32 [%0], %1;" ::"l"(p), "f"(v));
  else *p = v;
}
__device__ __forceinline__ void st_out(float* p, float4 v) {
  if constexpr (DISC_NC_STORES)
    asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w));
  else *reinterpret_cast<float4*>(p) = v;
}
__device__ __forceinline__ void st_cache(float* p, float v) {
  if constexpr (DISC_NC_STORES) asm volatile("st.shared.f32 [%0], %1;" ::"r"(smem_addr(p)), "f"(v));
  else *p = v;
}
__device__ __forceinline__ void st_cache(float* p, float4 v) {
  if constexpr (DISC_NC_STORES)
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(smem_addr(p)), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w));
  else *reinterpret_cast<float4*>(p) = v;
}
__device__ __forceinline__ void ld_cache(const float* p, float& v) {
  if constexpr (DISC_NC_STORES) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(smem_addr(p)));
  else v = *p;
}
__device__ __forceinline__ void ld_cache(const float* p, float4& v) {
  if constexpr (DISC_NC_STORES)
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(smem_addr(p)));
  else v = *reinterpret_cast<const float4*>(p);
}

// A tile: CH chunks of VEC elements.  Column tiles (ROWS = false): chunk c at
// (row, col0 + c*cstride) -- cstride = warp/group width * VEC keeps every access
// coalesced.  Row tiles (ROWS = true, column reductions): chunk c at (row + c*cstride,
// col0), so a thread keeps CH rows of loads in flight for the same VEC columns.
// I is the index type: int32_t for launches whose every address fits in 31 bits (!wide),
// int64_t otherwise; FULL tiles have all CH chunks valid (no per-chunk guard).
template <typename I, bool FULL, bool ROWS = false, bool STAGED = false>
struct Tile {
  using Index = I;
  static constexpr bool kRows = ROWS;
  static constexpr bool kStaged = STAGED;  // outputs with an out_slot go to shared memory
  I row;
  I col0;
  I W;
  I cstride;
  int nvalid;              // leading valid chunks (== CH when FULL)
  float* cache = nullptr;  // row cache: this row in slot 0 (slot k at cache + k*slot_stride), or null
  I slot_stride = 0;
  __device__ __forceinline__ bool has(int c) const { return FULL || c < nvalid; }
  // Flat-index distance between consecutive chunks.
  __device__ __forceinline__ I step() const { return ROWS ? cstride * W : cstride; }
};
using TileCtx = Tile<int64_t, false>;

// Row cache: fill on the reduce pass, read on the epilogue (see disc_cache_mode).
template <int VEC, int CH, typename Ctx>
__device__ __forceinline__ bool cached_load(const disc_program& P, const Ctx& t, int l,
                                            typename Vec<VEC>::T (&v)[CH]) {
  if (P.cache_mode != DISC_CACHE_READ || P.cache_slot[l] < 0 || !t.cache) return false;
  const float* c0 = t.cache + P.cache_slot[l] * t.slot_stride + t.col0;
#pragma unroll
  for (int c = 0; c < CH; ++c)
    if (t.has(c)) ld_cache(c0 + c * t.cstride, v[c]);
  return true;
}

template <int VEC, int CH, typename Ctx>
__device__ __forceinline__ void cache_fill(const disc_program& P, const Ctx& t, int l,
                                           const typename Vec<VEC>::T (&v)[CH]) {
  if (P.cache_mode != DISC_CACHE_FILL || P.cache_slot[l] < 0 || !t.cache) return;
  float* c0 = t.cache + P.cache_slot[l] * t.slot_stride + t.col0;
#pragma unroll
  for (int c = 0; c < CH; ++c)
    if (t.has(c)) st_cache(c0 + c * t.cstride, v[c]);
}

template <int VEC>
__device__ __forceinline__ typename Vec<VEC>::T load_row(const disc_load& L, const float* base, int64_t col) {
  // base already includes offset + row*rs (affine) or row*W (identity)
  if constexpr (VEC == 1) {
    return ldg(base + col * L.cs);
  } else {
    if (L.vec_ok == 1) return __ldg(reinterpret_cast<const float4*>(base + col));
    if (L.vec_ok == 2) {
      const float v = ldg(base);
      return make_float4(v, v, v, v);
    }
    const int64_t cs = L.cs;
    const float* p = base + col * cs;
    return make_float4(ldg(p), ldg(p + cs), ldg(p + 2 * cs), ldg(p + 3 * cs));
  }
}

template <int VEC, bool WIDE>
__device__ __forceinline__ typename Vec<VEC>::T load_gather(const disc_load& L, int64_t f) {
  if constexpr (VEC == 1) {
    return ldg(L.ptr + gather_index<WIDE>(L, f));
  } else {
    const int64_t s = gather_index<WIDE>(L, f);
    if (L.vec_ok == 1) return __ldg(reinterpret_cast<const float4*>(L.ptr + s));
    if (L.vec_ok == 2) {
      const float v = ldg(L.ptr + s);
      return make_float4(v, v, v, v);
    }
    const int64_t st = L.strides[L.rank - 1];
    return make_float4(ldg(L.ptr + s), ldg(L.ptr + s + st), ldg(L.ptr + s + 2 * st), ldg(L.ptr + s + 3 * st));
  }
}

// Hoists CONST loads of `P` into consts[load index] (call from every thread, then sync).
__device__ __forceinline__ void hoist_consts(const disc_program& P, float* consts) {
  for (int l = threadIdx.x + threadIdx.y * blockDim.x; l < P.n_loads; l += blockDim.x * blockDim.y)
    if (P.loads[l].mode == DISC_LOAD_CONST) consts[l] = ldg(P.loads[l].ptr + P.loads[l].offset);
}

// --- building blocks for generated (straight-line) programs --------------------------

// Load classes (structural: part of a generated pattern's key).  Contiguous row loads
// split on whether the launch's vector width can load them whole (vec_ok == 1).
enum LoadClass {
  kLcIdentity = 0, kLcConst = 1, kLcSplat = 2, kLcContig = 3, kLcStrided = 4, kLcGather = 5, kLcContigU = 6
};

__host__ __device__ inline int load_class(const disc_load& L) {
  switch (L.mode) {
    case DISC_LOAD_IDENTITY: return kLcIdentity;
    case DISC_LOAD_CONST: return kLcConst;
    case DISC_LOAD_AFFINE:
      return L.cs == 0 ? kLcSplat : (L.cs == 1 ? (L.vec_ok == 1 ? kLcContig : kLcContigU) : kLcStrided);
    default: return kLcGather;
  }
}

#ifndef DISC_COL_BCAST1
#define DISC_COL_BCAST1 1  // column tiles load a row-broadcast operand once, not once per row chunk
#endif

// One load of a tile with its binding class known at compile time.  Index math in the
// tile's index type (32-bit for !wide launches: one wide multiply-add per pointer).
template <int VEC, int CH, bool WIDE, int CLS, typename Ctx>
__device__ __forceinline__ void load_cls(const disc_program& P, const Ctx& t, const float* consts, int l,
                                         typename Vec<VEC>::T (&v)[CH]) {
  using I = typename Ctx::Index;
  constexpr bool ROWS = Ctx::kRows;
  const disc_load& L = P.loads[l];
  if constexpr (CLS == kLcIdentity) {
    if constexpr (!ROWS)
      if (cached_load<VEC, CH>(P, t, l, v)) return;
    const float* base = L.ptr + (t.row * t.W + t.col0);
    const I step = t.step();
#pragma unroll
    for (int c = 0; c < CH; ++c)
      if (t.has(c)) {
        if constexpr (VEC == 1) v[c] = ldg(base + c * step);
        else v[c] = __ldg(reinterpret_cast<const float4*>(base + c * step));
      }
    if constexpr (!ROWS) cache_fill<VEC, CH>(P, t, l, v);
  } else if constexpr (CLS == kLcConst) {
    const float x = consts[l];
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = splat(x, v[c]);
  } else if constexpr (CLS == kLcSplat) {  // value depends on the row only
    const I rs = static_cast<I>(L.rs);
    const float* base = L.ptr + (static_cast<I>(L.offset) + t.row * rs);
    if constexpr (ROWS) {
#pragma unroll
      for (int c = 0; c < CH; ++c)
        if (t.has(c)) v[c] = splat(ldg(base + c * t.cstride * rs), v[c]);
    } else {
      const float x = ldg(base);
#pragma unroll
      for (int c = 0; c < CH; ++c) v[c] = splat(x, v[c]);
    }
  } else if constexpr (CLS == kLcContig || CLS == kLcContigU) {
    const I rs = static_cast<I>(L.rs);
    const float* base = L.ptr + (static_cast<I>(L.offset) + t.row * rs + t.col0);
    if constexpr (ROWS && DISC_COL_BCAST1) {
      if (rs == 0) {  // column tile of a row-broadcast operand (C3's bias): one load for all chunks
        typename Vec<VEC>::T x;
        if constexpr (VEC == 1) x = ldg(base);
        else if constexpr (CLS == kLcContig) x = __ldg(reinterpret_cast<const float4*>(base));
        else x = make_float4(ldg(base), ldg(base + 1), ldg(base + 2), ldg(base + 3));
#pragma unroll
        for (int c = 0; c < CH; ++c) v[c] = x;
        return;
      }
    }
    const I step = ROWS ? t.cstride * rs : t.cstride;
#pragma unroll
    for (int c = 0; c < CH; ++c)
      if (t.has(c)) {
        const float* p = base + c * step;
        if constexpr (VEC == 1) v[c] = ldg(p);
        else if constexpr (CLS == kLcContig) v[c] = __ldg(reinterpret_cast<const float4*>(p));
        else v[c] = make_float4(ldg(p), ldg(p + 1), ldg(p + 2), ldg(p + 3));
      }
  } else if constexpr (CLS == kLcStrided) {  // cs not in {0, 1}: element loads
    const I cs = static_cast<I>(L.cs), rs = static_cast<I>(L.rs);
    const float* base = L.ptr + (static_cast<I>(L.offset) + t.row * rs);
#pragma unroll
    for (int c = 0; c < CH; ++c)
      if (t.has(c)) {
        const float* p = ROWS ? base + c * t.cstride * rs + t.col0 * cs : base + (t.col0 + c * t.cstride) * cs;
        if constexpr (VEC == 1) v[c] = ldg(p);
        else v[c] = make_float4(ldg(p), ldg(p + cs), ldg(p + 2 * cs), ldg(p + 3 * cs));
      }
  } else {
    const int64_t f0 = static_cast<int64_t>(t.row) * t.W + t.col0;
    const int64_t step = t.step();
#pragma unroll
    for (int c = 0; c < CH; ++c)
      if (t.has(c)) v[c] = load_gather<VEC, WIDE>(L, f0 + c * step);
  }
}

// Per-row scalar of a splat-class load (value depends on the row only): one register
// per chunk (column tiles: the same row, loaded once).
template <int CH, typename Ctx>
__device__ __forceinline__ void load_splat(const disc_program& P, const Ctx& t, int l, float (&s)[CH]) {
  using I = typename Ctx::Index;
  const disc_load& L = P.loads[l];
  const I rs = static_cast<I>(L.rs);
  const float* base = L.ptr + (static_cast<I>(L.offset) + t.row * rs);
  if constexpr (Ctx::kRows) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      if (t.has(c)) s[c] = ldg(base + c * t.cstride * rs);
  } else {
    const float x = ldg(base);
#pragma unroll
    for (int c = 0; c < CH; ++c) s[c] = x;
  }
}

// L2 prefetch of a tile's chunks of load l (streaming identity operands: the next
// grid-stride tile is requested while the current one computes; no registers held).
template <int VEC, int CH, int CLS, typename Ctx>
__device__ __forceinline__ void prefetch_cls(const disc_program& P, const Ctx& t, int l) {
  if constexpr (CLS == kLcIdentity) {
    const float* p = P.loads[l].ptr + (t.row * t.W + t.col0);
    const auto step = t.step();
#pragma unroll
    for (int c = 0; c < CH; ++c)
      if (t.has(c)) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + c * step));
  }
}

template <int VEC, int CH, typename Ctx>
__device__ __forceinline__ void store_tile(float* out, const Ctx& t, const typename Vec<VEC>::T (&v)[CH]) {
  float* o = out + (t.row * t.W + t.col0);
  const auto step = t.step();
#pragma unroll
  for (int c = 0; c < CH; ++c)
    if (t.has(c)) st_out(o + c * step, v[c]);
}

// Output o of a tile: its shared-memory slot in a staged launch, else global memory.
template <int VEC, int CH, typename Ctx>
__device__ __forceinline__ void store_out(const disc_program& P, int o, const Ctx& t,
                                          const typename Vec<VEC>::T (&v)[CH]) {
  if constexpr (Ctx::kStaged) {
    if (P.out_slot[o] >= 0) {
      float* s0 = t.cache + P.out_slot[o] * t.slot_stride + t.col0;
#pragma unroll
      for (int c = 0; c < CH; ++c)
        if (t.has(c)) st_cache(s0 + c * t.cstride, v[c]);
      return;
    }
  }
  store_tile<VEC, CH>(P.outs[o], t, v);
}

// Evaluates program P on one tile.  slots: this thread's slot base; slot k, chunk c lives
// at slots[(k * CH + c) * stride].  Returns with acc[] = the last instruction's value.
template <int VEC, int CH, bool WIDE, typename Ctx = TileCtx>
__device__ __forceinline__ void run_tile(const disc_program& P, const Ctx& t,
                                         typename Vec<VEC>::T (&acc)[CH], typename Vec<VEC>::T* slots, int stride,
                                         const float* consts, float red) {
  using T = typename Vec<VEC>::T;
  const int n = P.n_instr;
  const int64_t f0 = t.row * t.W + t.col0;
#define DISC_S(k, c) slots[((k) * CH + (c)) * stride]
#define DISC_FOR_C _Pragma("unroll") for (int c = 0; c < CH; ++c)
#define DISC_BIN_CASES(OPI)                                                                       \
  case DISC_I_BIN + 4 * OPI + 0: DISC_FOR_C acc[c] = bin<OPI>(acc[c], acc[c]); break;            \
  case DISC_I_BIN + 4 * OPI + 1: DISC_FOR_C acc[c] = bin<OPI>(acc[c], DISC_S(in.b, c)); break;   \
  case DISC_I_BIN + 4 * OPI + 2: DISC_FOR_C acc[c] = bin<OPI>(DISC_S(in.a, c), acc[c]); break;   \
  case DISC_I_BIN + 4 * OPI + 3: DISC_FOR_C acc[c] = bin<OPI>(DISC_S(in.a, c), DISC_S(in.b, c)); break;
#define DISC_UN_CASES(OPI)                                                              \
  case DISC_I_UN + 2 * OPI + 0: DISC_FOR_C acc[c] = un<OPI>(acc[c]); break;             \
  case DISC_I_UN + 2 * OPI + 1: DISC_FOR_C acc[c] = un<OPI>(DISC_S(in.a, c)); break;
  for (int pc = 0; pc < n; ++pc) {
    const disc_instr in = P.code[pc];
    switch (in.op) {
      case DISC_I_LOAD_ID: {
        if (cached_load<VEC, CH>(P, t, in.load, acc)) break;
        const float* base = P.loads[in.load].ptr + f0;
        DISC_FOR_C if (c < t.nvalid) {
          if constexpr (VEC == 1) acc[c] = ldg(base + c * t.cstride);
          else acc[c] = __ldg(reinterpret_cast<const float4*>(base + c * t.cstride));
        }
        cache_fill<VEC, CH>(P, t, in.load, acc);
        break;
      }
      case DISC_I_LOAD_AFF: {
        const disc_load& L = P.loads[in.load];
        const float* base = L.ptr + L.offset + t.row * L.rs;
        DISC_FOR_C if (c < t.nvalid) acc[c] = load_row<VEC>(L, base, t.col0 + c * t.cstride);
        break;
      }
      case DISC_I_LOAD_GATHER: {
        const disc_load& L = P.loads[in.load];
        DISC_FOR_C if (c < t.nvalid) acc[c] = load_gather<VEC, WIDE>(L, f0 + c * t.cstride);
        break;
      }
      case DISC_I_LOAD_CONST: {
        const float v = consts[in.load];
        DISC_FOR_C acc[c] = splat(v, acc[c]);
        break;
      }
      case DISC_I_REDVAL:
        DISC_FOR_C acc[c] = splat(red, acc[c]);
        break;
      case DISC_I_RCPVAL: {
        const float r = __frcp_rn(red);
        DISC_FOR_C acc[c] = splat(r, acc[c]);
        break;
      }
      case DISC_I_COPY:
        DISC_FOR_C acc[c] = DISC_S(in.a, c);
        break;
      DISC_BIN_CASES(0)
      DISC_BIN_CASES(1)
      DISC_BIN_CASES(2)
      DISC_BIN_CASES(3)
      DISC_BIN_CASES(4)
      DISC_UN_CASES(0)
      DISC_UN_CASES(1)
      DISC_UN_CASES(2)
      case DISC_I_FDIV + 0: DISC_FOR_C acc[c] = bin<5>(acc[c], acc[c]); break;
      case DISC_I_FDIV + 1: DISC_FOR_C acc[c] = bin<5>(acc[c], DISC_S(in.b, c)); break;
      case DISC_I_FDIV + 2: DISC_FOR_C acc[c] = bin<5>(DISC_S(in.a, c), acc[c]); break;
      case DISC_I_FDIV + 3: DISC_FOR_C acc[c] = bin<5>(DISC_S(in.a, c), DISC_S(in.b, c)); break;
      default:
        break;
    }
    if (in.flags & DISC_F_SLOT) {
      DISC_FOR_C DISC_S(in.dst, c) = acc[c];
    }
    if (in.flags & DISC_F_OUT) store_out<VEC, CH>(P, in.out, t, acc);
  }
#undef DISC_S
#undef DISC_FOR_C
#undef DISC_BIN_CASES
#undef DISC_UN_CASES
}

}  // namespace disc_dev
