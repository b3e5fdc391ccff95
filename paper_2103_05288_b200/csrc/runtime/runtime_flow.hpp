// The runtime flow on the device: executes a CompiledPlan's host instruction list with
// stream launches and a stream-ordered device caching allocator.  Instruction semantics,
// ExecStats and BufferEvents follow the reference Executor::run (executor.cpp:221-465).
#pragma once

#include <algorithm>
#include <chrono>
#include <map>
#include <mutex>
#include <set>
#include <unordered_map>
#include <memory>
#include <string>
#include <vector>

#include "../host/compiler.hpp"
#include "launcher.hpp"

namespace disc::rt {

struct ExecStats {
  int64_t launch_count = 0;
  int64_t library_calls = 0;
  int64_t host_instruction_count = 0;
  int64_t peak_bytes = 0;
  int64_t alloc_calls = 0;
  int64_t allocator_cache_hits = 0;
  int64_t aliased_allocs = 0;
  double host_ms = 0.0;
  double kernel_ms = 0.0;
};

struct BufferEvent {
  int logical = -1, physical = -1, alloc_instr = -1, dealloc_instr = -1;
};

// Large-block device memory shared by an executor and its host-thread sub-executors:
// address-ordered best fit with coalescing over big regions taken from the stream-ordered
// pool, so a stream of fresh shapes allocates without a driver call per buffer.  Every
// user issues on the same stream, so a freed range can be handed out again at once: the
// new owner's work is ordered after the old owner's on that stream.
class DeviceArena : public ChunkSource {
 public:
  static constexpr int64_t kRegion = int64_t{2} << 30;
  explicit DeviceArena(void* stream) : stream_(stream) {}
  ~DeviceArena() override;
  void* alloc(int64_t bytes);  // 256-byte multiples
  void free(void* p);
  void* get_chunk(int64_t bytes) override { return alloc((bytes + 255) / 256 * 256); }
  void put_chunk(void* p) override { free(p); }
  // Returns wholly free regions to the pool while more than `keep` bytes sit idle
  // (reserved regions are kept).
  void release_idle(int64_t keep);
  // Grows the arena to at least `bytes` now, as one region that is never released.
  void reserve(int64_t bytes);
  int64_t idle_bytes();
  int64_t region_bytes();
  void set_stream(void* s) { stream_ = s; }

 private:
  void insert_free(char* p, int64_t n);
  void erase_free(std::map<char*, int64_t>::iterator it);
  char* region_of(char* p) const;
  std::mutex mu_;
  void* stream_;
  std::map<char*, int64_t> regions_;                 // base -> bytes
  std::set<char*> reserved_;                         // bases never released
  std::map<char*, int64_t> free_by_addr_;            // start -> bytes
  std::set<std::pair<int64_t, char*>> free_by_size_;  // (bytes, start)
  std::unordered_map<char*, int64_t> used_;          // start -> bytes
  int64_t region_total_ = 0, used_total_ = 0;
};

// Physical device memory under the logical allocator.  Blocks up to kSlabMax are rounded up
// to size classes (four per power of two, <= 25% slack), carved from kSlab slabs and
// recycled per class across different exact sizes; larger blocks come from the shared
// DeviceArena.  Nothing here calls the driver per buffer once warm.
class PhysicalPool {
 public:
  static constexpr int64_t kSlab = int64_t{64} << 20;
  static constexpr int64_t kSlabMax = int64_t{1} << 20;
  PhysicalPool(void* stream, std::shared_ptr<DeviceArena> arena) : stream_(stream), arena_(std::move(arena)) {}
  ~PhysicalPool();
  static int64_t class_of(int64_t bytes);
  void* get(int64_t cls);
  void put(void* p, int64_t cls);
  int64_t free_bytes() const { return free_bytes_; }
  void set_stream(void* s) { stream_ = s; }
  void set_arena(std::shared_ptr<DeviceArena> a) { arena_ = std::move(a); }
  DeviceArena& arena() { return *arena_; }

 private:
  void* stream_;
  std::shared_ptr<DeviceArena> arena_;
  std::map<int64_t, std::vector<void*>> free_;  // small class bytes -> free blocks
  std::vector<char*> slabs_;
  int64_t slab_used_ = kSlab;                   // bytes used in slabs_.back()
  int64_t free_bytes_ = 0;
};

// Exact-byte-size free-list allocator over device memory (reference CachedAllocator,
// executor.cpp:53-76, same hit/miss accounting).  Physical memory comes from the size-class
// PhysicalPool; an optional byte budget moves cached free blocks back to it and bounds the
// pool (never hit by parity workloads, bounds memory across >=10k distinct shapes).
class DeviceCachingAllocator {
 public:
  DeviceCachingAllocator(void* stream, std::shared_ptr<DeviceArena> arena)
      : stream_(stream), pool_(stream, std::move(arena)) {}
  ~DeviceCachingAllocator();
  int alloc(int64_t bytes, ExecStats& stats);
  void free(int block);
  float* data(int block) const { return blocks_[block].ptr; }
  int64_t bytes(int block) const { return blocks_[block].bytes; }
  void set_stream(void* s) {
    stream_ = s;
    pool_.set_stream(s);
  }
  PhysicalPool& pool() { return pool_; }
  // The budget is enforced at the start of the next run (enforce_budget): blocks returned
  // at the end of a run back its outputs, which stay readable until then.
  void set_budget(int64_t b) { budget_ = b; }
  void enforce_budget();
  // Grouped execution: frees are held back until release_deferred() (work queued for
  // later issue may still use the blocks), so no block is reused inside one group.
  void set_defer(bool on);
  void trim();
  int64_t cached_bytes() const { return cached_; }

 private:
  struct Block {
    float* ptr = nullptr;
    int64_t bytes = 0;
    int64_t cls = 0;  // physical size class
  };
  void* stream_;
  PhysicalPool pool_;
  std::vector<Block> blocks_;
  std::vector<int> retired_;
  std::map<int64_t, std::vector<int>> free_;
  int64_t cached_ = 0;
  int64_t budget_ = 0;
  bool defer_ = false;
  std::vector<int> deferred_;
  void release(int block);
};

struct LaunchRecord {
  int instr = -1;         // plan instruction index
  int kernel = -1;        // artifact id (-1: library call)
  std::string schedule;   // schedule the selector picked
  int64_t bytes = 0;      // algorithmic boundary bytes
  double ms = 0.0;        // device time (timing mode only, after finish_timing)
  int device_kernels = 0;
  int ev = -1;            // event pair index (timing mode)
};

struct OutputView {
  const float* ptr = nullptr;
  std::vector<int64_t> dims;
};

struct InputBinding {
  std::string name;
  const float* ptr = nullptr;  // device pointer
  std::vector<int64_t> dims;
};

class DeviceExecutor {
 public:
  // `arena`: the large-block arena to share (host-thread sub-executors get their parent's).
  DeviceExecutor(int device, void* stream, std::shared_ptr<DeviceArena> arena = nullptr);
  ~DeviceExecutor();
  void set_stream(void* s);
  void* stream() const { return stream_; }
  // Runs the plan; outputs remain valid until the next run.
  // append_records: keep the launch records of earlier runs (batched sweeps).
  // plan_serial: stable id of `plan` (enables the launch recipe cache; 0 disables).
  void run(const CompiledPlan& plan, const std::vector<InputBinding>& inputs, bool append_records = false,
           uint64_t plan_serial = 0);
  // Static plans (no shape program) run as CUDA graphs: a run whose queued device work
  // hashes like the previous run's is captured once and replayed afterwards
  // (SURVEY 8(f) rank 2).  On by default; DISC_GRAPHS=0 or set_graphs(false) disables.
  void set_graphs(bool on) { graphs_ = on; }
  int64_t graph_replays() const { return graph_replays_; }
  // Grouped execution of independent requests (disc_executor_run_grouped), over raw
  // C-ABI arrays (request r: plans[r], inputs offs[r] .. offs[r+1]-1).  Each request's
  // runtime flow runs on the host (shapes, buffers, versions, schedules) while its device
  // work is queued (begin_grouped / begin_request / run); the queues are flushed level by
  // level with the same plan kernel of all requests fused into grouped launches.  With
  // host threads > 1 and enough requests, contiguous request ranges run on worker threads
  // (each with its own sub-executor: allocator, scratch, recipe cache, queue) and their
  // queues are merged into one flush; calls of >= 128 requests flush in two phases (the
  // largest eighth first).  Request outputs stay valid until the next run.
  void run_grouped_batch(int n, const CompiledPlan* const* plans, const uint64_t* serials, const int* offs,
                         const char* const* names, const void* const* data, const int64_t* const* dims,
                         const int* ranks, bool on_host);
  void set_host_threads(int n);
  int host_threads() const { return host_threads_; }
  // Asynchronous flush (grouped calls on device inputs): a call's flows return once queued
  // and its flushes are issued by a background thread in call order, so the host flows of
  // the next phase / call overlap the flush of this one.  Stream order = call order, so
  // every host-side memory reuse stays safe.  Anything that touches the stream from the
  // caller's thread first waits until all queued flushes are issued (wait_issued).
  void set_async_flush(bool on);
  void wait_issued();
  bool grouped() const { return grouped_; }
  const std::vector<std::vector<OutputView>>& request_outputs() const { return req_outputs_; }
  const std::vector<ExecStats>& request_stats() const { return req_stats_; }
  // Timing mode: waits for the recorded events and fills record/stat device times.
  void finish_timing();
  const std::vector<OutputView>& outputs() const { return outputs_; }
  const ExecStats& stats() const { return stats_; }
  const std::vector<BufferEvent>& events() const { return events_; }
  int64_t device_launches() const { return device_launches_; }
  int64_t algorithmic_bytes() const { return algorithmic_bytes_; }
  const std::vector<LaunchRecord>& launch_records() const { return records_; }
  void set_timing(bool on) { timing_ = on; }
  void set_schedule(SchedulePref p) {
    pref_ = p;
    for (auto& x : subs_) x->set_schedule(p);
  }
  // The byte budget bounds the idle device memory the executor and its host-thread
  // sub-executors keep between runs: a quarter for the exact-size caches (an equal share
  // each; a stream of fresh shapes fills every cache with sizes that never recur), the
  // rest for idle arena regions (reused across sizes).  Enforced at run start.
  void reserve(int64_t bytes) { arena_->reserve(bytes); }
  void set_cache_budget(int64_t b) {
    budget_total_ = b;
    const int64_t share = b > 0 ? std::max<int64_t>(1, b / 4 / static_cast<int64_t>(1 + subs_.size())) : 0;
    alloc_.set_budget(share);
    for (auto& x : subs_) x->alloc_.set_budget(share);
  }
  // Host-staging helper: device copy of host data owned by the executor (not counted in
  // plan allocator stats).
  const float* stage_input(int slot, const void* host, int64_t bytes);
  // run_kernel equivalent on device externals.
  void run_kernel(const KernelArtifact& art, const VersionArtifact& ver, const std::vector<DevTensor>& ext,
                  const std::vector<int64_t>& regs);
  Scratch& scratch() { return scratch_; }

 private:
  int device_;
  void* stream_;
  std::shared_ptr<DeviceArena> arena_;
  DeviceCachingAllocator alloc_;
  int64_t budget_total_ = 0;
  Scratch scratch_;
  std::vector<OutputView> outputs_;
  std::vector<float*> passthrough_;  // owned copies for input pass-through outputs
  std::vector<int64_t> passthrough_bytes_;
  std::vector<std::pair<void*, int64_t>> staging_;
  ExecStats stats_;
  std::vector<BufferEvent> events_;
  int64_t device_launches_ = 0;
  int64_t algorithmic_bytes_ = 0;
  std::vector<LaunchRecord> records_;
  bool timing_ = false;
  SchedulePref pref_ = SchedulePref::kAuto;
  LaunchCache* cache_ = nullptr;
  std::vector<std::pair<void*, void*>> ev_pool_;
  size_t ev_next_ = 0;
  bool timing_pending_ = false;
  bool grouped_ = false;
  bool group_timing_ = false;
  bool records_grouped_ = false;  // records_ describe grouped launches
  void begin_grouped();
  void begin_request();
  void run_impl(const CompiledPlan& plan, const std::vector<InputBinding>& inputs, bool append_records,
                uint64_t plan_serial);
  struct GraphEntry {
    std::vector<std::string> seen;                      // recent work signatures (capture on a repeat)
    std::vector<std::pair<std::string, void*>> graphs;  // captured graphs by exact signature (<= 4)
    uint64_t last_use = 0;
  };
  static constexpr size_t kMaxGraphPlans = 64;  // plans with cached graphs per executor (LRU)
  std::map<uint64_t, GraphEntry> graph_cache_;
  uint64_t graph_clock_ = 0;
  bool graphs_ = true;
  int64_t graph_replays_ = 0;
  // multi-threaded host flow (run_grouped_batch)
  int host_threads_ = 1;
  struct Flusher;
  std::unique_ptr<Flusher> flusher_;
  bool async_flush_ = false;
  bool flush_idle() const;
  struct Pool;
  std::unique_ptr<Pool> pool_;
  std::vector<std::unique_ptr<DeviceExecutor>> subs_;
  void run_requests(const int* ids, int count, const CompiledPlan* const* plans, const uint64_t* serials,
                    const int* offs, const char* const* names, const void* const* data, const int64_t* const* dims,
                    const int* ranks, bool on_host);
  void begin_phase();
  void append_group_records();
  std::vector<int> req_ids_;  // request id of each req_outputs_ entry (grouped calls)
  void* detach_grouped();      // worker: issue packed small inputs, hand the queue over
  void finish_detached();      // after the merged flush
  int issue_small_inputs();
  std::chrono::steady_clock::time_point t_group_;
  // grouped calls: small host inputs packed into one pinned arena (one H2D per group)
  static constexpr int64_t kSmallInput = 64 << 10;
  struct SmallChunk {
    void* host = nullptr;   // pinned
    void* dev = nullptr;
    int64_t cap = 0, used = 0;
    void* event = nullptr;  // after the chunk's H2D copy
    bool pending = false;
  };
  std::vector<SmallChunk> small_;
  size_t small_cur_ = 0;
  int request_ = -1;
  std::vector<std::vector<OutputView>> req_outputs_;
  std::vector<ExecStats> req_stats_;
  int take_event_pair();
};

}  // namespace disc::rt
