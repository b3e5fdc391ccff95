// Device-side interpreter for lowered fusion tapes (disc_program).
//
// A thread evaluates the program at one flat index f (VEC=1) or at four consecutive
// flat indices f..f+3 (VEC=4, float4 lanes).  Values flow through an accumulator
// register; values needed later live in per-thread shared-memory slots.  Instruction
// words and gather maps are read from __grid_constant__ parameter space (uniform).
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

__device__ __forceinline__ float apply_bin(int op, float a, float b) {
  switch (op) {
    case DISC_OP_ADD: return __fadd_rn(a, b);
    case DISC_OP_SUB: return __fsub_rn(a, b);
    case DISC_OP_MUL: return __fmul_rn(a, b);
    case DISC_OP_DIV: return __fdiv_rn(a, b);
    default: return op_max(a, b);
  }
}

__device__ __forceinline__ float apply_un(int op, float a) {
  switch (op) {
    case DISC_OP_EXP: return expf(a);
    case DISC_OP_TANH: return tanhf(a);
    default: return -a;
  }
}

__device__ __forceinline__ float4 apply_bin(int op, float4 a, float4 b) {
  return make_float4(apply_bin(op, a.x, b.x), apply_bin(op, a.y, b.y), apply_bin(op, a.z, b.z),
                     apply_bin(op, a.w, b.w));
}
__device__ __forceinline__ float4 apply_un(int op, float4 a) {
  return make_float4(apply_un(op, a.x), apply_un(op, a.y), apply_un(op, a.z), apply_un(op, a.w));
}

__device__ __forceinline__ float splat(float v, float) { return v; }
__device__ __forceinline__ float4 splat(float v, float4) { return make_float4(v, v, v, v); }

// u32 fast division (n < 2^31): q = umulhi(n, magic) >> shift, magic == 0 means d == 1.
__device__ __forceinline__ uint32_t fdiv(uint32_t n, uint32_t magic, uint32_t shift) {
  return magic ? (__umulhi(n, magic) >> shift) : n;
}

template <bool WIDE>
__device__ __forceinline__ int64_t map_index(const disc_load& L, int64_t f) {
  if (L.rank == 0) return f;
  int64_t src = L.offset;
  if (WIDE) {
    int64_t rem = f;
    for (int d = L.rank - 1; d > 0; --d) {
      int64_t dim = L.dims[d];
      int64_t q = rem / dim;
      src += (rem - q * dim) * L.strides[d];
      rem = q;
    }
    src += rem * L.strides[0];
  } else {
    uint32_t rem = static_cast<uint32_t>(f);
    for (int d = L.rank - 1; d > 0; --d) {
      uint32_t q = fdiv(rem, L.magic[d], L.shift[d]);
      src += static_cast<int64_t>(rem - q * static_cast<uint32_t>(L.dims[d])) * L.strides[d];
      rem = q;
    }
    src += static_cast<int64_t>(rem) * L.strides[0];
  }
  return src;
}

__device__ __forceinline__ float ldg(const float* p) { return __ldg(p); }

template <int VEC, bool WIDE>
__device__ __forceinline__ typename Vec<VEC>::T do_load(const disc_load& L, int64_t f) {
  if constexpr (VEC == 1) {
    return ldg(L.ptr + map_index<WIDE>(L, f));
  } else {
    if (L.mode == DISC_LOAD_IDENTITY) return __ldg(reinterpret_cast<const float4*>(L.ptr + f));
    int64_t s = map_index<WIDE>(L, f);
    if (L.vec_ok == 1) return __ldg(reinterpret_cast<const float4*>(L.ptr + s));
    if (L.vec_ok == 2) {
      float v = ldg(L.ptr + s);
      return make_float4(v, v, v, v);
    }
    // Four consecutive f share the outer coordinates (innermost extent % 4 == 0).
    int64_t st = L.strides[L.rank - 1];
    return make_float4(ldg(L.ptr + s), ldg(L.ptr + s + st), ldg(L.ptr + s + 2 * st), ldg(L.ptr + s + 3 * st));
  }
}

template <int VEC>
__device__ __forceinline__ void do_store(float* out, int64_t f, typename Vec<VEC>::T v) {
  if constexpr (VEC == 1) {
    out[f] = v;
  } else {
    *reinterpret_cast<float4*>(out + f) = v;
  }
}

// Evaluates `P` at flat index f.  `slots` points at this thread's slot 0; slot k is at
// slots[k * stride].  `red` is the row's reduce value for DISC_OP_REDVAL.  Returns acc.
template <int VEC, bool WIDE>
__device__ __forceinline__ typename Vec<VEC>::T run_program(const disc_program& P, int64_t f,
                                                            typename Vec<VEC>::T* slots, int stride,
                                                            float red) {
  using T = typename Vec<VEC>::T;
  T acc{};
  const int n = P.n_instr;
  for (int pc = 0; pc < n; ++pc) {
    const disc_instr in = P.code[pc];
    const int op = in.op;
    if (op == DISC_OP_LOAD) {
      acc = do_load<VEC, WIDE>(P.loads[in.load], f);
    } else if (op == DISC_OP_REDVAL) {
      acc = splat(red, acc);
    } else {
      T a = in.a == DISC_SRC_ACC ? acc : slots[in.a * stride];
      if (op >= DISC_OP_EXP) {
        acc = op == DISC_OP_COPY ? a : apply_un(op, a);
      } else {
        T b = in.b == DISC_SRC_ACC ? acc : slots[in.b * stride];
        acc = apply_bin(op, a, b);
      }
    }
    if (in.dst != DISC_SRC_NONE) slots[in.dst * stride] = acc;
    if (in.out >= 0) do_store<VEC>(P.outs[in.out], f, acc);
  }
  return acc;
}

}  // namespace disc_dev
