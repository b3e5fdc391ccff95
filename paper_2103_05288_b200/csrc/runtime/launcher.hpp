// Per-launch binding of a KernelArtifact to device kernels: the B200 replacement for the
// reference's run_kernel (executor.cpp:137-219).  Shapes are validated on the host with
// the reference's runtime error messages, then the tape is lowered to one fused program
// (or, for exotic member-to-member gathers, materialised member by member) and launched
// through the disc_cuda.h device ABI.  Nothing is compiled per shape.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../host/compiler.hpp"
#include "disc_cuda.h"

namespace disc::rt {

struct DevTensor {
  const float* ptr = nullptr;
  std::vector<int64_t> dims;
};

struct OutBuf {
  float* ptr = nullptr;
  int64_t capacity_bytes = 0;
};

// Stream-ordered bump allocator for per-launch device scratch (reduce results feeding a
// separate epilogue pass, f64 split-R partials, materialised members).  Chunks are
// recycled only at reset(), i.e. between launches on the same stream.
// A device-memory source for large chunks (the executor's DeviceArena); without one,
// chunks come from the stream-ordered pool.
struct ChunkSource {
  virtual void* get_chunk(int64_t bytes) = 0;
  virtual void put_chunk(void* p) = 0;
  virtual ~ChunkSource() = default;
};

class Scratch {
 public:
  explicit Scratch(void* stream, ChunkSource* src = nullptr) : stream_(stream), src_(src) {}
  ~Scratch();
  void set_stream(void* s) { stream_ = s; }
  void* alloc(int64_t bytes);
  void reset();

 private:
  struct Chunk {
    char* base;
    int64_t size;
  };
  void* stream_;
  ChunkSource* src_;
  std::vector<Chunk> chunks_;
  size_t cur_ = 0;
  int64_t used_ = 0;
};

enum class SchedulePref { kAuto, kMaterialize, kFusedOnly, kTwoPass, kAtomic };

struct LaunchReport {
  int device_kernels = 0;       // device kernels issued for this kLaunch
  bool materialized = false;    // per-member fallback used
  std::string schedule;         // "loop", "row", "col_twopass", ... (diagnostics)
  int64_t algorithmic_bytes = 0;  // boundary bytes (SURVEY §8d formula)
};

// Shape-keyed cache of recorded fused launches (owned by an executor).
struct LaunchCache;
LaunchCache* new_launch_cache();
void free_launch_cache(LaunchCache* c);

// Runs one kLaunch.  `ext` are the external inputs bound at the artifact's
// external_input_dims; `outs` are the planned output buffers.  With a cache and a
// nonzero plan serial, fused lowerings are recorded once per (plan, kernel, version,
// register file, operand dims, pointer alignment/aliasing) and replayed afterwards.
LaunchReport launch_kernel(const KernelArtifact& art, const VersionArtifact& ver, const std::vector<DevTensor>& ext,
                           const std::vector<int64_t>& regs, const std::vector<OutBuf>& outs, Scratch& scratch,
                           void* stream, SchedulePref pref, LaunchCache* cache = nullptr, uint64_t plan_serial = 0);

// Library call (eval_matmul semantics, f64 accumulation).
void launch_gemm(int64_t m, int64_t k, int64_t n, const DevTensor& a, const DevTensor& b, const OutBuf& c,
                 Scratch& scratch, void* stream);

// Host-side shape simulation of a tape (exposed for tests): dims of every member.
std::vector<std::vector<int64_t>> simulate_tape(const KernelArtifact& art, const VersionArtifact& ver,
                                                const std::vector<std::vector<int64_t>>& ext_dims,
                                                const std::vector<int64_t>& regs);

// Algorithmic boundary bytes of one kLaunch at the given shapes, host only.
int64_t launch_bytes_estimate(const KernelArtifact& art, const VersionArtifact& ver,
                              const std::vector<std::vector<int64_t>>& ext_dims, const std::vector<int64_t>& regs);

// u32 fast-division constants (exposed for tests).
void fast_div_magic(uint32_t d, uint32_t* magic, uint32_t* shift);

}  // namespace disc::rt
