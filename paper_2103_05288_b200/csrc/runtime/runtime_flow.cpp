// Device runtime flow (see runtime_flow.hpp).
#include "runtime_flow.hpp"

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <exception>
#include <functional>
#include <mutex>
#include <numeric>
#include <thread>

#include <pthread.h>
#include <sched.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <set>

#include "disc_cuda.h"
#include "shape_eval.hpp"

namespace disc::rt {

namespace {

void cuda_ok(int rc, const char* what) {
  if (rc != 0) throw RuntimeError(std::string(what) + ": " + disc_cuda_last_error());
}

int64_t numel(const std::vector<int64_t>& d) {
  int64_t n = 1;
  for (int64_t x : d) n *= x;
  return n;
}

using Clock = std::chrono::steady_clock;

}  // namespace

// ---------------------------------------------------------------------------

DeviceArena::~DeviceArena() {
  for (auto& [base, n] : regions_) disc_cuda_free(base, stream_);
}

char* DeviceArena::region_of(char* p) const {
  auto it = regions_.upper_bound(p);
  return it == regions_.begin() ? nullptr : std::prev(it)->first;
}

void DeviceArena::insert_free(char* p, int64_t n) {
  free_by_addr_.emplace(p, n);
  free_by_size_.emplace(n, p);
}

void DeviceArena::erase_free(std::map<char*, int64_t>::iterator it) {
  free_by_size_.erase({it->second, it->first});
  free_by_addr_.erase(it);
}

void* DeviceArena::alloc(int64_t bytes) {
  std::lock_guard<std::mutex> lock(mu_);
  auto fit = free_by_size_.lower_bound({bytes, nullptr});
  if (fit == free_by_size_.end()) {
    const int64_t n = std::max(bytes, kRegion);
    void* q = nullptr;
    cuda_ok(disc_cuda_malloc(static_cast<size_t>(n), stream_, &q), "device allocation");
    regions_.emplace(static_cast<char*>(q), n);
    region_total_ += n;
    insert_free(static_cast<char*>(q), n);
    fit = free_by_size_.lower_bound({bytes, nullptr});
  }
  const auto [n, p] = *fit;
  erase_free(free_by_addr_.find(p));
  if (n > bytes) insert_free(p + bytes, n - bytes);
  used_.emplace(p, bytes);
  used_total_ += bytes;
  return p;
}

void DeviceArena::free(void* q) {
  std::lock_guard<std::mutex> lock(mu_);
  char* p = static_cast<char*>(q);
  auto u = used_.find(p);
  if (u == used_.end()) throw InternalError("arena free of an unknown block");
  int64_t n = u->second;
  used_.erase(u);
  used_total_ -= n;
  char* reg = region_of(p);
  auto next = free_by_addr_.lower_bound(p);
  if (next != free_by_addr_.end() && next->first == p + n && region_of(next->first) == reg) {
    n += next->second;
    auto after = std::next(next);
    erase_free(next);
    next = after;
  }
  if (next != free_by_addr_.begin()) {
    auto prev = std::prev(next);
    if (prev->first + prev->second == p && region_of(prev->first) == reg) {
      p = prev->first;
      n += prev->second;
      erase_free(prev);
    }
  }
  insert_free(p, n);
}

void DeviceArena::release_idle(int64_t keep) {
  std::lock_guard<std::mutex> lock(mu_);
  for (auto it = regions_.begin(); it != regions_.end() && region_total_ - used_total_ > keep;) {
    auto f = free_by_addr_.find(it->first);
    if (f != free_by_addr_.end() && f->second == it->second && !reserved_.count(it->first)) {  // wholly free
      erase_free(f);
      disc_cuda_free(it->first, stream_);
      region_total_ -= it->second;
      it = regions_.erase(it);
    } else {
      ++it;
    }
  }
}

void DeviceArena::reserve(int64_t bytes) {
  std::lock_guard<std::mutex> lock(mu_);
  if (region_total_ >= bytes) return;
  const int64_t n = (bytes - region_total_ + 255) / 256 * 256;
  void* q = nullptr;
  cuda_ok(disc_cuda_malloc(static_cast<size_t>(n), stream_, &q), "device reservation");
  regions_.emplace(static_cast<char*>(q), n);
  reserved_.insert(static_cast<char*>(q));
  region_total_ += n;
  insert_free(static_cast<char*>(q), n);
}

int64_t DeviceArena::idle_bytes() {
  std::lock_guard<std::mutex> lock(mu_);
  return region_total_ - used_total_;
}

int64_t DeviceArena::region_bytes() {
  std::lock_guard<std::mutex> lock(mu_);
  return region_total_;
}

PhysicalPool::~PhysicalPool() {
  for (char* p : slabs_) arena_->free(p);
}

int64_t PhysicalPool::class_of(int64_t bytes) {
  const int64_t b = std::max<int64_t>(bytes, 256);
  if (b > kSlabMax) return (b + 255) / 256 * 256;  // arena blocks: 256-byte granularity
  int e = 63 - __builtin_clzll(static_cast<unsigned long long>(b - 1));  // 2^e < b <= 2^(e+1)
  const int64_t step = std::max<int64_t>(256, int64_t{1} << std::max(0, e - 2));  // 4 classes per octave
  return (b + step - 1) / step * step;
}

void* PhysicalPool::get(int64_t cls) {
  if (cls > kSlabMax) return arena_->alloc(cls);
  auto it = free_.find(cls);
  if (it != free_.end()) {
    void* p = it->second.back();
    it->second.pop_back();
    if (it->second.empty()) free_.erase(it);
    free_bytes_ -= cls;
    return p;
  }
  if (slab_used_ + cls > kSlab) {  // slabs come from the arena too (reserved memory, no driver call)
    slabs_.push_back(static_cast<char*>(arena_->alloc(kSlab)));
    slab_used_ = 0;
  }
  void* p = slabs_.back() + slab_used_;
  slab_used_ += cls;
  return p;
}

void PhysicalPool::put(void* p, int64_t cls) {
  if (cls > kSlabMax) {
    arena_->free(p);
    return;
  }
  free_[cls].push_back(p);
  free_bytes_ += cls;
}

DeviceCachingAllocator::~DeviceCachingAllocator() = default;  // the pool owns the memory

int DeviceCachingAllocator::alloc(int64_t bytes, ExecStats& stats) {
  auto it = free_.find(bytes);
  if (it != free_.end() && !it->second.empty()) {
    int id = it->second.back();
    it->second.pop_back();
    if (it->second.empty()) free_.erase(it);
    cached_ -= bytes;
    stats.allocator_cache_hits++;
    return id;
  }
  stats.alloc_calls++;
  // 16-byte granularity like the reference; physical blocks are 256-byte aligned classes.
  const int64_t cls = PhysicalPool::class_of((std::max<int64_t>(bytes, 1) + 15) / 16 * 16);
  void* p = pool_.get(cls);
  if (!retired_.empty()) {  // ids released by trim() are recycled: blocks_ stays bounded
    const int id = retired_.back();
    retired_.pop_back();
    blocks_[id] = {static_cast<float*>(p), bytes, cls};
    return id;
  }
  blocks_.push_back({static_cast<float*>(p), bytes, cls});
  return static_cast<int>(blocks_.size()) - 1;
}

void DeviceCachingAllocator::free(int block) {
  if (defer_) {
    deferred_.push_back(block);
    return;
  }
  release(block);
}

void DeviceCachingAllocator::set_defer(bool on) {
  defer_ = on;
  if (!on) {
    for (int b : deferred_) release(b);
    deferred_.clear();
  }
}

void DeviceCachingAllocator::release(int block) {
  free_[blocks_[block].bytes].push_back(block);
  cached_ += blocks_[block].bytes;
}

void DeviceCachingAllocator::enforce_budget() {
  if (budget_ > 0 && cached_ > budget_) trim();
}

void DeviceCachingAllocator::trim() {
  // Release cached free blocks (largest sizes first) until under half the budget.  Released
  // ids are retired (reused by later misses), so hit/miss accounting stays exact-size and
  // neither blocks_ nor free_ grows without bound under a stream of fresh shapes.
  while (!free_.empty() && cached_ > budget_ / 2) {
    auto it = std::prev(free_.end());
    for (int id : it->second) {
      pool_.put(blocks_[id].ptr, blocks_[id].cls);
      blocks_[id].ptr = nullptr;
      cached_ -= blocks_[id].bytes;
      retired_.push_back(id);
    }
    free_.erase(it);
  }
}

// ---------------------------------------------------------------------------

DeviceExecutor::DeviceExecutor(int device, void* stream, std::shared_ptr<DeviceArena> arena)
    : device_(device),
      stream_(stream),
      arena_(arena ? std::move(arena) : std::make_shared<DeviceArena>(stream)),
      alloc_(stream, arena_),
      scratch_(stream, arena_.get()),
      cache_(new_launch_cache()) {
  cuda_ok(disc_cuda_set_device(device), "set device");
}

int DeviceExecutor::take_event_pair() {
  if (ev_next_ == ev_pool_.size()) {
    void *a = nullptr, *b = nullptr;
    cuda_ok(disc_cuda_event_create(&a), "event");
    cuda_ok(disc_cuda_event_create(&b), "event");
    ev_pool_.push_back({a, b});
  }
  return static_cast<int>(ev_next_++);
}

void DeviceExecutor::begin_grouped() {
  if (grouped_) throw InternalError("grouped execution already in progress");
  if (timing_pending_) cuda_ok(disc_cuda_stream_synchronize(stream_), "stream sync");
  timing_pending_ = false;
  records_.clear();
  ev_next_ = 0;
  device_launches_ = 0;
  algorithmic_bytes_ = 0;
  req_outputs_.clear();
  req_stats_.clear();
  scratch_.reset();
  records_grouped_ = false;
  t_group_ = Clock::now();
  cuda_ok(disc_cuda_queue_begin(stream_), "queue begin");
  alloc_.set_defer(true);
  grouped_ = true;
  group_timing_ = timing_;
  request_ = -1;
}

// Next phase of the same grouped call: a new queue, nothing reset (outputs, scratch and
// deferred frees of earlier phases stay).
void DeviceExecutor::begin_phase() {
  if (grouped_) throw InternalError("grouped execution already in progress");
  cuda_ok(disc_cuda_queue_begin(stream_), "queue begin");
  grouped_ = true;
}

void DeviceExecutor::begin_request() {
  if (!grouped_) throw InternalError("begin_request outside grouped execution");
  cuda_ok(disc_cuda_queue_request(), "queue request");
  ++request_;
}

int DeviceExecutor::issue_small_inputs() {
  int rc = 0;
  for (auto& c : small_) {  // packed small inputs: one H2D per chunk ahead of every queued op
    if (c.used == 0) continue;
    if (rc == 0) rc = disc_cuda_memcpy(c.dev, c.host, static_cast<size_t>(c.used), 0 | DISC_MEMCPY_NOW, stream_);
    if (rc == 0) rc = disc_cuda_event_record(c.event, stream_);
    c.pending = true;
    c.used = 0;
  }
  small_cur_ = 0;
  return rc;
}

void* DeviceExecutor::detach_grouped() {
  grouped_ = false;
  const int rc = issue_small_inputs();
  void* q = disc_cuda_queue_detach();
  cuda_ok(rc, "small-input copy");
  return q;
}

void DeviceExecutor::finish_detached() { alloc_.set_defer(false); }

// Persistent worker threads for run_grouped_batch.
struct DeviceExecutor::Pool {
  std::vector<std::thread> threads;
  std::mutex mu;
  std::condition_variable cv, done;
  std::function<void(int)> job;
  uint64_t gen = 0;
  int pending = 0;
  bool stop = false;
  std::vector<Clock::time_point> wake_at = std::vector<Clock::time_point>(64);
  Pool(int n, int device) {
    // Workers are pinned one per CPU of the creating thread's affinity set (worker w on the
    // (w+1)-th CPU; the caller keeps the first).  Unpinned, a wake-up of many short jobs
    // lands the woken threads on the waker's CPU and they run one after another until the
    // load balancer spreads them (measured: 7 x 4 ms jobs took 58 ms unpinned, 11 pinned).
    // DISC_PIN_THREADS=0 disables; a rank's CPU slice is its process affinity mask.
    std::vector<int> cpus;
    static const bool pin = [] {
      const char* e = std::getenv("DISC_PIN_THREADS");
      return !e || std::atoi(e) != 0;
    }();
    cpu_set_t allowed;
    CPU_ZERO(&allowed);
    if (pin && sched_getaffinity(0, sizeof allowed, &allowed) == 0)
      for (int c = 0; c < CPU_SETSIZE; ++c)
        if (CPU_ISSET(c, &allowed)) cpus.push_back(c);
    for (int w = 0; w < n; ++w)
      threads.emplace_back([this, w, device, cpus] {
        if (cpus.size() > 1) {
          cpu_set_t one;
          CPU_ZERO(&one);
          CPU_SET(cpus[(w + 1) % cpus.size()], &one);
          pthread_setaffinity_np(pthread_self(), sizeof one, &one);
        }
        disc_cuda_set_device(device);
        uint64_t seen = 0;
        for (;;) {
          std::function<void(int)> f;
          {
            std::unique_lock<std::mutex> l(mu);
            cv.wait(l, [&] { return stop || gen != seen; });
            if (stop) return;
            seen = gen;
            f = job;
          }
          wake_at[w] = Clock::now();
          f(w);
          std::lock_guard<std::mutex> l(mu);
          if (--pending == 0) done.notify_all();
        }
      });
  }
  void start(const std::function<void(int)>& f) {  // f(w) on every worker, asynchronously
    const int capture = disc_cuda_capture_mode();  // workers run in the caller's capture mode
    std::lock_guard<std::mutex> l(mu);
    job = [f, capture](int w) {
      disc_cuda_set_capture_local(capture);
      f(w);
    };
    pending = static_cast<int>(threads.size());
    ++gen;
    cv.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> l(mu);
    done.wait(l, [&] { return pending == 0; });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> l(mu);
      stop = true;
    }
    cv.notify_all();
    for (auto& t : threads) t.join();
  }
};

// Background issuer of grouped flushes (set_async_flush): jobs run in submission order.
struct DeviceExecutor::Flusher {
  std::thread th;
  std::mutex mu;
  std::condition_variable cv, idle;
  std::deque<std::function<void()>> jobs;
  int pending = 0;
  bool stop = false;
  std::exception_ptr err;
  explicit Flusher(int device) {
    th = std::thread([this, device] {
      disc_cuda_set_device(device);
      for (;;) {
        std::function<void()> f;
        {
          std::unique_lock<std::mutex> l(mu);
          cv.wait(l, [&] { return stop || !jobs.empty(); });
          if (jobs.empty()) return;
          f = std::move(jobs.front());
          jobs.pop_front();
        }
        try {
          f();
        } catch (...) {
          std::lock_guard<std::mutex> l(mu);
          if (!err) err = std::current_exception();
        }
        std::lock_guard<std::mutex> l(mu);
        if (--pending == 0) idle.notify_all();
      }
    });
  }
  void submit(std::function<void()> f) {
    std::lock_guard<std::mutex> l(mu);
    jobs.push_back(std::move(f));
    ++pending;
    cv.notify_one();
  }
  void wait() {
    std::unique_lock<std::mutex> l(mu);
    idle.wait(l, [&] { return pending == 0; });
    if (err) {
      std::exception_ptr e = err;
      err = nullptr;
      std::rethrow_exception(e);
    }
  }
  bool is_idle() {
    std::lock_guard<std::mutex> l(mu);
    return pending == 0;
  }
  ~Flusher() {
    {
      std::lock_guard<std::mutex> l(mu);
      stop = true;
    }
    cv.notify_all();
    th.join();
  }
};

void DeviceExecutor::set_async_flush(bool on) {
  wait_issued();
  async_flush_ = on;
  if (on && !flusher_) flusher_ = std::make_unique<Flusher>(device_);
}

void DeviceExecutor::wait_issued() {
  if (flusher_) flusher_->wait();
}

bool DeviceExecutor::flush_idle() const { return !flusher_ || flusher_->is_idle(); }

void DeviceExecutor::set_host_threads(int n) {
  n = std::max(1, std::min(n, 64));
  if (n == host_threads_) return;
  pool_.reset();
  subs_.clear();
  host_threads_ = n;
  if (n > 1) {
    for (int w = 1; w < n; ++w) {
      subs_.push_back(std::make_unique<DeviceExecutor>(device_, stream_, arena_));
      subs_.back()->set_schedule(pref_);
    }
    pool_ = std::make_unique<Pool>(n - 1, device_);
  }
  set_cache_budget(budget_total_);
}

void DeviceExecutor::run_requests(const int* ids, int count, const CompiledPlan* const* plans, const uint64_t* serials,
                                  const int* offs, const char* const* names, const void* const* data,
                                  const int64_t* const* dims, const int* ranks, bool on_host) {
  std::vector<InputBinding> in;
  for (int j = 0; j < count; ++j) {
    const int r = ids[j];
    begin_request();
    const int i0 = offs[r], n = offs[r + 1] - i0;
    in.resize(n);
    for (int i = 0; i < n; ++i) {
      const int k = i0 + i;
      in[i].name = names[k];
      in[i].dims.assign(dims[k], dims[k] + ranks[k]);
      int64_t bytes = 4;
      for (int64_t d : in[i].dims) bytes *= d;
      // one staging buffer per (request, input): all of a group's copies are in flight together
      in[i].ptr = on_host ? stage_input(k, data[k], bytes) : static_cast<const float*>(data[k]);
    }
    req_ids_.push_back(r);
    run(*plans[r], in, true, serials[r]);
  }
}

// Reads the records of the flush just issued (non-timing: metadata only) into records_.
void DeviceExecutor::append_group_records() {
  const int nrec = disc_cuda_queue_num_records();
  for (int i = 0; i < nrec; ++i) {
    int level = 0, members = 0, kernel = -1;
    int64_t bytes = 0;
    const char* sched = nullptr;
    float ms = 0.f;
    if (group_timing_) {
      records_.push_back({i, -1, "", 0, 0.0, 1, -1});  // device times read in finish_timing
    } else {
      cuda_ok(disc_cuda_queue_record(i, &level, &members, &bytes, &kernel, &sched, &ms), "group record");
      records_.push_back({level, kernel, std::string("group:") + (sched ? sched : ""), bytes, 0.0, members, -1});
    }
    device_launches_ += 1;
  }
}

static bool prof_host() {
  static const bool on = std::getenv("DISC_HOST_PROFILE") != nullptr;
  return on;
}

void DeviceExecutor::run_grouped_batch(int n, const CompiledPlan* const* plans, const uint64_t* serials,
                                       const int* offs, const char* const* names, const void* const* data,
                                       const int64_t* const* dims, const int* ranks, bool on_host) {
  constexpr int kMinPerThread = 8;
  // Phases: with enough requests, the largest eighth (by input size) is flushed first, so
  // the device starts on the long kernels while the host runs the other flows
  // (DISC_GROUP_PHASES=1: one flush).  Timing mode keeps one flush (per-launch events).
  static const int max_phases = [] {
    const char* e = std::getenv("DISC_GROUP_PHASES");
    return e ? std::max(1, std::atoi(e)) : 2;
  }();
  std::vector<std::vector<int>> phases;
  if (!timing_ && max_phases >= 2 && n >= 128) {
    std::vector<std::pair<int64_t, int>> w(n);
    for (int r = 0; r < n; ++r) {
      int64_t e = 0;
      for (int k = offs[r]; k < offs[r + 1]; ++k) {
        int64_t m = 1;
        for (int d = 0; d < ranks[k]; ++d) m *= dims[k][d];
        e += m;
      }
      w[r] = {-e, r};
    }
    const int k = std::max(1, n / 8);
    std::nth_element(w.begin(), w.begin() + k, w.end());
    std::vector<char> first(n, 0);
    for (int i = 0; i < k; ++i) first[w[i].second] = 1;
    // the other requests: max_phases - 1 contiguous index ranges of equal count
    phases.resize(max_phases);
    const int rest = n - k, per = (rest + max_phases - 2) / (max_phases - 1);
    int seen = 0;
    for (int r = 0; r < n; ++r) {
      if (first[r]) {
        phases[0].push_back(r);
      } else {
        phases[1 + std::min(max_phases - 2, seen / std::max(1, per))].push_back(r);
        ++seen;
      }
    }
    while (phases.size() > 1 && phases.back().empty()) phases.pop_back();
  } else {
    phases.emplace_back(n);
    std::iota(phases[0].begin(), phases[0].end(), 0);
  }
  // the previous call's outputs are dead: idle memory beyond the budget goes back first
  if (budget_total_ > 0) {
    alloc_.enforce_budget();
    for (auto& x : subs_) x->alloc_.enforce_budget();
    // returning whole regions frees device memory on the stream now: only when no queued
    // flush (whose kernels may still use them) is pending
    if (flush_idle()) arena_->release_idle(budget_total_ - budget_total_ / 4);
  }
  // async flush: device inputs only (host inputs stage through the executor's pinned
  // chunks, which the next call's flows would overwrite) and never in timing mode
  const bool async = async_flush_ && !on_host && !timing_;
  if (!async) wait_issued();
  // session
  begin_grouped();  // resets outputs, records, scratch; defers frees
  req_ids_.clear();
  std::vector<char> sub_used(subs_.size(), 0);
  std::vector<std::exception_ptr> errs;
  int rc = 0;
  const auto t_start = Clock::now();
  double flush_ms = 0;
  for (size_t ph = 0; ph < phases.size(); ++ph) {
    const std::vector<int>& P = phases[ph];
    const int m = static_cast<int>(P.size());
    const int T = std::max(1, std::min(host_threads_, m / kMinPerThread));
    std::vector<int> bounds(T + 1);
    for (int w = 0; w <= T; ++w) bounds[w] = static_cast<int>(int64_t{m} * w / T);
    std::vector<void*> handles(T, nullptr);
    std::vector<std::exception_ptr> perr(T);
    std::vector<double> wt(T, 0.0), wl(T, 0.0), ws(T, 0.0);
    const auto t_phase = Clock::now();
    if (ph > 0) begin_phase();
    if (T > 1) {
      pool_->start([&](int w) {
        if (w + 1 >= T) return;
        const auto tl = Clock::now();
        DeviceExecutor& ex = *subs_[w];
        try {
          if (!sub_used[w]) {
            ex.set_timing(false);
            ex.begin_grouped();
            ex.req_ids_.clear();
            sub_used[w] = 1;
          } else {
            ex.begin_phase();
          }
          const auto tw = Clock::now();
          ex.run_requests(P.data() + bounds[w + 1], bounds[w + 2] - bounds[w + 1], plans, serials, offs, names, data,
                          dims, ranks, on_host);
          wt[w + 1] = std::chrono::duration<double, std::milli>(Clock::now() - tw).count();
        } catch (...) {
          perr[w + 1] = std::current_exception();
        }
        try {
          if (ex.grouped()) handles[w + 1] = ex.detach_grouped();
        } catch (...) {
          if (!perr[w + 1]) perr[w + 1] = std::current_exception();
        }
        wl[w + 1] = std::chrono::duration<double, std::milli>(Clock::now() - tl).count();
        ws[w + 1] = std::chrono::duration<double, std::milli>(tl - t_phase).count();
      });
    }
    try {  // this thread's range, concurrently with the workers
      const auto tw = Clock::now();
      run_requests(P.data() + bounds[0], bounds[1] - bounds[0], plans, serials, offs, names, data, dims, ranks, on_host);
      wt[0] = std::chrono::duration<double, std::milli>(Clock::now() - tw).count();
    } catch (...) {
      perr[0] = std::current_exception();
    }
    if (T > 1) pool_->wait();
    if (prof_host()) {
      std::fprintf(stderr, "[disc host]   phase %zu: %d requests on %d threads, flows %.3f ms wall; per thread:", ph, m, T,
                   std::chrono::duration<double, std::milli>(Clock::now() - t_phase).count());
      for (double x : wt) std::fprintf(stderr, " %.2f", x);
      std::fprintf(stderr, "; worker lambda:");
      for (double x : wl) std::fprintf(stderr, " %.2f", x);
      std::fprintf(stderr, "; start offset:");
      for (double x : ws) std::fprintf(stderr, " %.2f", x);
      std::fprintf(stderr, "; wake offset:");
      for (int w = 0; w + 1 < T; ++w)
        std::fprintf(stderr, " %.2f", std::chrono::duration<double, std::milli>(pool_->wake_at[w] - t_phase).count());
      std::fprintf(stderr, "\n");
    }
    // merged flush of this phase: this thread's queue + the workers' detached ones
    grouped_ = false;
    const auto t_flush = Clock::now();
    std::vector<void*> hs;
    for (int w = 1; w < T; ++w)
      if (handles[w]) hs.push_back(handles[w]);
    if (async) {
      // issued in the background, in call order; this thread's queue (the first requests)
      // goes first, as in the synchronous merge
      if (void* mine = disc_cuda_queue_detach()) hs.insert(hs.begin(), mine);
      flusher_->submit([hs, capture = disc_cuda_capture_mode()] {
        disc_cuda_set_capture_local(capture);  // a dry run's flush stays a dry run
        if (disc_cuda_queue_flush_detached(hs.data(), static_cast<int>(hs.size()), 0) != 0)
          throw RuntimeError(std::string("grouped launch: ") + disc_cuda_last_error());
      });
      flush_ms += std::chrono::duration<double, std::milli>(Clock::now() - t_flush).count();
    } else {
      const int src = issue_small_inputs();
      const int frc = disc_cuda_queue_flush_detached(hs.data(), static_cast<int>(hs.size()), group_timing_ ? 1 : 0);
      flush_ms += std::chrono::duration<double, std::milli>(Clock::now() - t_flush).count();
      if (rc == 0) rc = src ? src : frc;
      if (rc == 0) append_group_records();
    }
    for (auto& e : perr)
      if (e) errs.push_back(e);
    if (!errs.empty() || rc) break;
  }
  static const bool prof = std::getenv("DISC_HOST_PROFILE") != nullptr;
  if (prof)
    std::fprintf(stderr, "[disc host] grouped call: %d requests, %zu phases, host %.3f ms (flush %.3f ms)\n", n,
                 phases.size(), std::chrono::duration<double, std::milli>(Clock::now() - t_start).count(), flush_ms);
  // end of session: frees released, outputs / stats in request order
  alloc_.set_defer(false);
  std::vector<std::vector<OutputView>> outs(n);
  std::vector<ExecStats> sts(n);
  auto gather = [&](DeviceExecutor& ex) {
    for (size_t j = 0; j < ex.req_ids_.size() && j < ex.req_outputs_.size(); ++j) {
      outs[ex.req_ids_[j]] = ex.req_outputs_[j];
      sts[ex.req_ids_[j]] = ex.req_stats_[j];
    }
  };
  gather(*this);
  for (size_t w = 0; w < subs_.size(); ++w)
    if (sub_used[w]) {
      subs_[w]->finish_detached();
      gather(*subs_[w]);
      algorithmic_bytes_ += subs_[w]->algorithmic_bytes();
    }
  req_outputs_.swap(outs);
  req_stats_.swap(sts);
  for (const auto& e : errs) std::rethrow_exception(e);
  cuda_ok(rc, "grouped launch");
  records_grouped_ = true;
  timing_pending_ = group_timing_;
}

void DeviceExecutor::finish_timing() {
  wait_issued();
  if (!timing_pending_) return;
  timing_pending_ = false;
  if (records_grouped_) {
    double total = 0;
    for (size_t i = 0; i < records_.size(); ++i) {
      int level = 0, members = 0, kernel = -1;
      int64_t bytes = 0;
      const char* sched = nullptr;
      float ms = 0.f;
      cuda_ok(disc_cuda_queue_record(static_cast<int>(i), &level, &members, &bytes, &kernel, &sched, &ms),
              "group record");
      records_[i] = {level, kernel, std::string("group:") + (sched ? sched : ""), bytes, ms, members, -1};
      total += ms;
    }
    stats_.kernel_ms = total;
    return;
  }
  cuda_ok(disc_cuda_stream_synchronize(stream_), "stream sync");
  double total = 0;
  for (auto& r : records_) {
    if (r.ev < 0) continue;
    float ms = 0;
    cuda_ok(disc_cuda_event_elapsed_ms(ev_pool_[r.ev].first, ev_pool_[r.ev].second, &ms), "event elapsed");
    r.ms = ms;
    total += ms;
  }
  stats_.kernel_ms = total;
}

DeviceExecutor::~DeviceExecutor() {
  try {
    wait_issued();
  } catch (...) {
  }
  flusher_.reset();
  disc_cuda_stream_synchronize(stream_);
  for (auto& [_, g] : graph_cache_)
    for (auto& [h, exec] : g.graphs) disc_cuda_graph_destroy(exec);
  for (auto& c : small_) {
    disc_cuda_host_free(c.host);
    disc_cuda_free(c.dev, stream_);
    disc_cuda_event_destroy(c.event);
  }
  free_launch_cache(cache_);
  for (float* p : passthrough_)
    if (p) disc_cuda_free(p, stream_);
  for (auto& s : staging_)
    if (s.first) disc_cuda_free(s.first, stream_);
  for (auto& e : ev_pool_) {
    disc_cuda_event_destroy(e.first);
    disc_cuda_event_destroy(e.second);
  }
}

void DeviceExecutor::set_stream(void* s) {
  wait_issued();
  // Cached blocks and arena ranges are reused in stream order: work of the old stream must
  // be done before the new stream may touch them.
  if (stream_ && s != stream_) disc_cuda_stream_synchronize(stream_);
  stream_ = s;
  alloc_.set_stream(s);
  scratch_.set_stream(s);
  arena_->set_stream(s);
  for (auto& x : subs_) x->set_stream(s);
}

const float* DeviceExecutor::stage_input(int slot, const void* host, int64_t bytes) {
  if (grouped_ && bytes <= kSmallInput) {
    // Small host inputs of a grouped call are packed into pinned arena chunks that go H2D
    // as one copy per chunk ahead of the group's flush, not one PCIe transfer each.
    for (;;) {
      if (small_cur_ == small_.size()) {
        SmallChunk c;
        c.cap = int64_t{8} << 20;
        cuda_ok(disc_cuda_host_alloc(static_cast<size_t>(c.cap), &c.host), "small-input arena");
        cuda_ok(disc_cuda_malloc(static_cast<size_t>(c.cap), stream_, &c.dev), "small-input arena");
        cuda_ok(disc_cuda_event_create(&c.event), "small-input arena");
        small_.push_back(c);
      }
      SmallChunk& c = small_[small_cur_];
      if (c.used == 0 && c.pending) {  // the previous group's copy from this chunk
        cuda_ok(disc_cuda_event_synchronize(c.event), "small-input arena");
        c.pending = false;
      }
      const int64_t off = (c.used + 255) / 256 * 256;
      if (off + bytes <= c.cap) {
        std::memcpy(static_cast<char*>(c.host) + off, host, static_cast<size_t>(bytes));
        c.used = off + bytes;
        return reinterpret_cast<const float*>(static_cast<char*>(c.dev) + off);
      }
      ++small_cur_;
    }
  }
  if (static_cast<int>(staging_.size()) <= slot) staging_.resize(slot + 1, {nullptr, 0});
  auto& s = staging_[slot];
  if (s.second < bytes) {
    if (s.first) disc_cuda_free(s.first, stream_);
    s.first = nullptr;
    cuda_ok(disc_cuda_malloc(static_cast<size_t>(std::max<int64_t>(bytes, 16)), stream_, &s.first), "input staging");
    s.second = bytes;
  }
  if (bytes) cuda_ok(disc_cuda_memcpy(s.first, host, static_cast<size_t>(bytes), 0, stream_), "input H2D");
  return static_cast<const float*>(s.first);
}

void DeviceExecutor::run_kernel(const KernelArtifact& art, const VersionArtifact& ver, const std::vector<DevTensor>& ext,
                                const std::vector<int64_t>& regs) {
  wait_issued();
  std::vector<std::vector<int64_t>> ed;
  for (const auto& e : ext) ed.push_back(e.dims);
  auto dims = simulate_tape(art, ver, ed, regs);
  std::vector<OutBuf> outs;
  outputs_.clear();
  scratch_.reset();
  for (int t : art.output_tape_indices) {
    int64_t bytes = numel(dims[t]) * 4;
    float* p = static_cast<float*>(scratch_.alloc(bytes));
    outs.push_back({p, bytes});
    outputs_.push_back({p, dims[t]});
  }
  LaunchReport rep = launch_kernel(art, ver, ext, regs, outs, scratch_, stream_, pref_);
  device_launches_ = rep.device_kernels;
  records_ = {{-1, -1, rep.schedule, rep.algorithmic_bytes, 0.0, rep.device_kernels, -1}};
}

void DeviceExecutor::run(const CompiledPlan& plan, const std::vector<InputBinding>& inputs, bool append_records,
                         uint64_t plan_serial) {
  if (!grouped_) wait_issued();  // direct launches go behind every queued flush
  static const bool env_on = [] {
    const char* e = std::getenv("DISC_GRAPHS");
    return !e || std::atoi(e) != 0;
  }();
  const bool graph = env_on && graphs_ && !grouped_ && !timing_ && plan_serial != 0 && plan.shape_program.empty() &&
                     stream_ != nullptr && !disc_cuda_queue_active();
  if (!graph) return run_impl(plan, inputs, append_records, plan_serial);
  cuda_ok(disc_cuda_queue_begin(stream_), "queue begin");
  cuda_ok(disc_cuda_queue_request(), "queue request");
  try {
    run_impl(plan, inputs, append_records, plan_serial);
  } catch (...) {
    if (void* q = disc_cuda_queue_detach()) disc_cuda_queue_issue_graph(q, nullptr);  // valid work before the error
    throw;
  }
  void* q = disc_cuda_queue_detach();
  if (!q) return;
  const void* sig_data = nullptr;
  size_t sig_n = 0;
  cuda_ok(disc_cuda_queue_signature(q, &sig_data, &sig_n), "queue signature");
  std::string h(static_cast<const char*>(sig_data), sig_n);  // empty: not capturable
  if (!graph_cache_.count(plan_serial) && graph_cache_.size() >= kMaxGraphPlans) {
    // evict the least recently used plan's graphs (a server compiling many static plans)
    auto lru = graph_cache_.begin();
    for (auto it = graph_cache_.begin(); it != graph_cache_.end(); ++it)
      if (it->second.last_use < lru->second.last_use) lru = it;
    for (auto& [_, exec] : lru->second.graphs) disc_cuda_graph_destroy(exec);
    graph_cache_.erase(lru);
  }
  GraphEntry& g = graph_cache_[plan_serial];
  g.last_use = ++graph_clock_;
  for (auto& [gh, exec] : g.graphs)
    if (!h.empty() && gh == h) {  // same launches, same pointers (full compare): replay
      disc_cuda_queue_discard(q);
      cuda_ok(disc_cuda_graph_launch(exec, stream_), "graph replay");
      ++graph_replays_;
      device_launches_ = 1;
      return;
    }
  // capture work seen before (buffer placement can cycle between a few states)
  const bool repeat = !h.empty() && std::find(g.seen.begin(), g.seen.end(), h) != g.seen.end();
  if (repeat) {
    void* exec = nullptr;
    cuda_ok(disc_cuda_queue_issue_graph(q, &exec), "graph capture");
    if (exec) {
      if (g.graphs.size() >= 4) {
        disc_cuda_graph_destroy(g.graphs.front().second);
        g.graphs.erase(g.graphs.begin());
      }
      g.graphs.emplace_back(std::move(h), exec);
    }
  } else {
    cuda_ok(disc_cuda_queue_issue_graph(q, nullptr), "issue");
    if (!h.empty()) {
      if (g.seen.size() >= 8) g.seen.erase(g.seen.begin());
      g.seen.push_back(std::move(h));
    }
  }
}

void DeviceExecutor::run_impl(const CompiledPlan& plan, const std::vector<InputBinding>& inputs, bool append_records,
                              uint64_t plan_serial) {
  ExecStats stats;
  stats.host_instruction_count = plan.host_instruction_count();
  const auto t_run = Clock::now();
  // The previous run's outputs (returned to the cache at its end) are dead from here on:
  // only now may the budget release cached blocks.
  alloc_.enforce_budget();
  if (budget_total_ > 0 && !grouped_) arena_->release_idle(budget_total_ - budget_total_ / 4);
  if (!append_records && !grouped_) {
    if (timing_pending_) cuda_ok(disc_cuda_stream_synchronize(stream_), "stream sync");
    timing_pending_ = false;
    records_.clear();
    records_grouped_ = false;
    ev_next_ = 0;
    device_launches_ = 0;
    algorithmic_bytes_ = 0;
  }
  if (!grouped_) scratch_.reset();  // grouped: scratch of every request stays live until the flush
  if (grouped_) cuda_ok(disc_cuda_queue_mark(0, -1, "h2d"), "queue mark");  // input staging copies

  std::vector<int64_t> regs(plan.shape_program.num_regs, 0);
  struct Slot {
    const InputBinding* input = nullptr;
    int block = -1;
    int64_t bytes = 0;
  };
  std::vector<Slot> slots(plan.num_buffers);
  std::map<int, int> version_of;
  int64_t live = 0;
  std::map<int, BufferEvent> events;
  std::vector<const std::vector<int64_t>*> input_dims(plan.inputs.size(), nullptr);

  auto input_asserts = [&] {
    for (size_t i = 0; i < plan.inputs.size(); ++i) {
      const auto& pi = plan.inputs[i];
      const auto& d = slots[i].input->dims;
      for (size_t k = 0; k < pi.dims.size(); ++k) {
        int64_t want = resolve(pi.dims[k], regs);
        if (d[k] != want)
          throw RuntimeError("input " + pi.id + " dim " + std::to_string(k) + " violates a shape constraint: expected " +
                             std::to_string(want) + ", got " + std::to_string(d[k]));
      }
    }
  };

  auto view = [&](int buf, const std::vector<int64_t>& dims) -> DevTensor {
    const Slot& s = slots[buf];
    if (s.input) {
      if (numel(dims) > numel(s.input->dims))
        throw RuntimeError("input " + s.input->name + " is smaller than its planned extent");
      return {s.input->ptr, dims};
    }
    if (numel(dims) * 4 > s.bytes) throw InternalError("read exceeds planned buffer size");
    return {alloc_.data(s.block), dims};
  };
  auto out_buf = [&](int buf) -> OutBuf {
    const Slot& s = slots[buf];
    if (s.input) throw InternalError("write into an input buffer");
    return {alloc_.data(s.block), s.bytes};
  };

  bool shapes_ready = plan.shape_program.empty();
  outputs_.assign(plan.outputs.size(), {});

  for (size_t pc = 0; pc < plan.instrs.size(); ++pc) {
    const Instr& in = plan.instrs[pc];
    switch (in.kind) {
      case InstrKind::kBindInput: {
        const auto& pi = plan.inputs[in.a];
        const InputBinding* b = nullptr;
        for (const auto& x : inputs)
          if (x.name == pi.id) b = &x;
        if (!b) throw RuntimeError("missing input " + pi.id);
        if (b->dims.size() != pi.dims.size()) throw RuntimeError("input " + pi.id + " rank mismatch");
        slots[in.b].input = b;
        input_dims[in.a] = &b->dims;
        break;
      }
      case InstrKind::kEvalShape:
        for (size_t i = 0; i < input_dims.size(); ++i)
          if (!input_dims[i]) throw InternalError("shape evaluation before inputs are bound");
        eval_shape_range(plan, in.a, in.b, input_dims, regs);
        shapes_ready = true;
        input_asserts();
        break;
      case InstrKind::kAlloc: {
        int64_t elems = in.size.const_elems;
        for (int r : in.size.regs) elems *= regs[r];
        const int64_t bytes = elems * 4;
        Slot& s = slots[in.b];
        s.block = alloc_.alloc(bytes, stats);
        s.bytes = bytes;
        live += bytes;
        stats.peak_bytes = std::max(stats.peak_bytes, live);
        events[in.b] = {in.b, s.block, static_cast<int>(pc), -1};
        break;
      }
      case InstrKind::kDealloc: {
        Slot& s = slots[in.b];
        if (!in.reserve) {  // reserved blocks pass straight to a later alias
          alloc_.free(s.block);
          live -= s.bytes;
        }
        events[in.b].dealloc_instr = static_cast<int>(pc);
        break;
      }
      case InstrKind::kAlias: {
        Slot& s = slots[in.b];
        s.block = slots[in.a].block;
        s.bytes = slots[in.a].bytes;
        stats.aliased_allocs++;
        events[in.b] = {in.b, s.block, static_cast<int>(pc), -1};
        break;
      }
      case InstrKind::kSelectVersion: {
        const KernelArtifact& art = plan.kernels[in.a];
        int chosen = -1;
        for (const auto& v : art.versions) {
          bool pass = true;
          for (const auto& g : v.guards) {
            if (g.kind == GuardTest::Kind::kNever) pass = false;
            else if (g.kind == GuardTest::Kind::kRefEqual) pass = pass && resolve(g.a, regs) == resolve(g.b, regs);
            else if (g.kind == GuardTest::Kind::kTotalDivisibleBy4) {
              int64_t total = 1;
              for (const auto& d : art.space_dims) total *= resolve(d, regs);
              pass = pass && total % 4 == 0;
            }
            if (!pass) break;
          }
          if (pass) {
            chosen = v.id;
            break;
          }
        }
        if (chosen < 0) throw RuntimeError("no kernel version guard matched");
        version_of[in.a] = chosen;
        break;
      }
      case InstrKind::kComputeLaunch:
        break;  // the reference tile rule (256/1024) is superseded by the schedule selector
      case InstrKind::kLaunch: {
        if (!shapes_ready && !plan.shape_program.empty()) throw InternalError("launch before shape evaluation");
        const KernelArtifact& art = plan.kernels[in.a];
        const int vid = in.fixed_version >= 0 ? in.fixed_version : version_of.at(in.a);
        const VersionArtifact* ver = nullptr;
        for (const auto& v : art.versions)
          if (v.id == vid) ver = &v;
        if (!ver) throw InternalError("unknown kernel version selected");
        std::vector<DevTensor> ext;
        for (size_t a = 0; a < in.arg_bufs.size(); ++a)
          ext.push_back(view(in.arg_bufs[a], resolve_all(art.external_input_dims[a], regs)));
        std::vector<OutBuf> outs;
        for (int b : in.out_bufs) outs.push_back(out_buf(b));
        const int ev = timing_ && !grouped_ ? take_event_pair() : -1;
        if (ev >= 0) cuda_ok(disc_cuda_event_record(ev_pool_[ev].first, stream_), "event");
        LaunchReport rep = launch_kernel(art, *ver, ext, regs, outs, scratch_, stream_, pref_, cache_, plan_serial);
        if (ev >= 0) cuda_ok(disc_cuda_event_record(ev_pool_[ev].second, stream_), "event");
        stats.launch_count++;
        algorithmic_bytes_ += rep.algorithmic_bytes;
        if (grouped_) {  // the queued ops of this kLaunch carry its bytes / artifact / schedule
          cuda_ok(disc_cuda_queue_mark(rep.algorithmic_bytes, in.a, rep.schedule.c_str()), "queue mark");
          break;
        }
        device_launches_ += rep.device_kernels;
        records_.push_back({static_cast<int>(pc), in.a, rep.schedule, rep.algorithmic_bytes, 0.0, rep.device_kernels, ev});
        break;
      }
      case InstrKind::kLibraryCall: {
        const int64_t m = resolve(in.lib_dims[0], regs), k = resolve(in.lib_dims[1], regs),
                      n = resolve(in.lib_dims[2], regs);
        DevTensor a = view(in.arg_bufs[0], {m, k}), b = view(in.arg_bufs[1], {k, n});
        const int ev = timing_ && !grouped_ ? take_event_pair() : -1;
        if (ev >= 0) cuda_ok(disc_cuda_event_record(ev_pool_[ev].first, stream_), "event");
        launch_gemm(m, k, n, a, b, out_buf(in.out_bufs[0]), scratch_, stream_);
        if (ev >= 0) cuda_ok(disc_cuda_event_record(ev_pool_[ev].second, stream_), "event");
        stats.library_calls++;
        if (grouped_) {
          cuda_ok(disc_cuda_queue_mark(4 * (m * k + k * n + m * n), -1, "gemm"), "queue mark");
          algorithmic_bytes_ += 4 * (m * k + k * n + m * n);
          break;
        }
        device_launches_ += (m && n) ? 1 : 0;
        records_.push_back({static_cast<int>(pc), -1, "gemm", 4 * (m * k + k * n + m * n), 0.0, (m && n) ? 1 : 0, ev});
        break;
      }
      case InstrKind::kBindOutput: {
        const auto& po = plan.outputs[in.a];
        std::vector<int64_t> dims = resolve_all(po.dims, regs);
        DevTensor t = view(in.b, dims);
        if (slots[in.b].input && grouped_) {
          // Pass-through in a group: a per-request copy (scratch lives until the next run).
          const int64_t bytes = numel(dims) * 4;
          float* p = static_cast<float*>(scratch_.alloc(bytes));
          if (bytes) cuda_ok(disc_cuda_memcpy(p, t.ptr, static_cast<size_t>(bytes), 2, stream_), "output copy");
          outputs_[in.a] = {p, dims};
        } else if (slots[in.b].input) {
          // Pass-through of a caller input: copy so the output outlives the binding.
          if (passthrough_.size() <= static_cast<size_t>(in.a)) {
            passthrough_.resize(in.a + 1, nullptr);
            passthrough_bytes_.resize(in.a + 1, 0);
          }
          const int64_t bytes = numel(dims) * 4;
          float*& p = passthrough_[in.a];
          if (passthrough_bytes_[in.a] < bytes) {
            if (p) disc_cuda_free(p, stream_);
            void* q = nullptr;
            cuda_ok(disc_cuda_malloc(static_cast<size_t>(std::max<int64_t>(bytes, 16)), stream_, &q), "output copy");
            p = static_cast<float*>(q);
            passthrough_bytes_[in.a] = bytes;
          }
          if (bytes) cuda_ok(disc_cuda_memcpy(p, t.ptr, static_cast<size_t>(bytes), 2, stream_), "output copy");
          outputs_[in.a] = {p, dims};
        } else {
          outputs_[in.a] = {t.ptr, dims};
        }
        break;
      }
    }
  }
  if (plan.shape_program.empty()) input_asserts();
  if (grouped_) cuda_ok(disc_cuda_queue_mark(0, -1, "copy"), "queue mark");  // pass-through output copies

  // Every block still held returns to the cache for the next run (outputs stay readable
  // until then: the next run's work is ordered after them on the stream).
  std::set<int> returned;
  for (const auto& [logical, ev] : events)
    if (ev.dealloc_instr < 0 && returned.insert(ev.physical).second) alloc_.free(ev.physical);

  stats.host_ms = std::chrono::duration<double, std::milli>(Clock::now() - t_run).count();
  stats_ = stats;
  if (grouped_) {
    req_outputs_.push_back(outputs_);
    req_stats_.push_back(stats);
  } else {
    timing_pending_ = timing_pending_ || timing_;
  }
  events_.clear();
  for (const auto& [_, ev] : events) events_.push_back(ev);
}

}  // namespace disc::rt
