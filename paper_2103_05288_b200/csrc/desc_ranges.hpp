// Byte ranges of a launch descriptor that are ever read (by the host scheduler or a
// kernel): a program's header, its first n_instr instructions, its first n_loads load
// bindings and its output pointers, plus the launch's geometry tail.  Copies of
// descriptors on the hot host path (recipe replay, the request queue, grouped-launch
// tables) move only these ranges: a disc_reduce_launch is ~9.3 KB, its used part
// typically 1-3 KB.
#pragma once

#include <cstddef>
#include <cstring>

#include "disc_cuda.h"

namespace disc_desc {

struct Range {
  size_t off, len;
};
constexpr int kMaxRanges = 8;

inline int program_ranges(const disc_program& P, size_t base, Range* r) {
  r[0] = {base, offsetof(disc_program, code) + static_cast<size_t>(P.n_instr) * sizeof(disc_instr)};
  r[1] = {base + offsetof(disc_program, loads), static_cast<size_t>(P.n_loads) * sizeof(disc_load)};
  r[2] = {base + offsetof(disc_program, outs), sizeof(disc_program) - offsetof(disc_program, outs)};
  return 3;
}

inline int ranges(const disc_loop_launch& L, Range* r) {
  int n = program_ranges(L.prog, offsetof(disc_loop_launch, prog), r);
  const size_t tail = offsetof(disc_loop_launch, prog) + sizeof(disc_program);
  r[n++] = {tail, sizeof(disc_loop_launch) - tail};
  return n;
}

inline int ranges(const disc_reduce_launch& R, Range* r) {
  int n = program_ranges(R.pre, offsetof(disc_reduce_launch, pre), r);
  n += program_ranges(R.post, offsetof(disc_reduce_launch, post), r + n);
  const size_t tail = offsetof(disc_reduce_launch, post) + sizeof(disc_program);
  r[n++] = {tail, sizeof(disc_reduce_launch) - tail};
  return n;
}

// Copies the used ranges of `src` into `dst` (same type; bytes outside stay untouched).
template <typename Launch>
inline void copy_used(Launch* dst, const Launch& src) {
  Range r[kMaxRanges];
  const int n = ranges(src, r);
  for (int i = 0; i < n; ++i)
    if (r[i].len) std::memcpy(reinterpret_cast<char*>(dst) + r[i].off, reinterpret_cast<const char*>(&src) + r[i].off, r[i].len);
}

}  // namespace disc_desc
