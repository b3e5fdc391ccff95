// Multi-GPU request dispatcher, native: independent variable-shape requests
// are sharded across device workers with no collective on the data path -- a request (plan
// + inputs) is self-contained and the path has no cross-request reduction.
//
// One worker thread per entry of `devices` (a device may repeat: several workers share a
// GPU, each with its own stream), each owning a DeviceExecutor (caching allocator, buffer
// arena, host-flow threads) and pinned to its own contiguous slice of the process's CPUs,
// so the workers' host flows never compete for cores.  A batch is partitioned by greedy
// LPT on the requests' algorithmic bytes (largest first, to the least-loaded worker, lowest
// index on ties -- the rule of dispatch.shard, so a one-process-per-GPU deployment and
// this in-process form assign identically) and every worker runs its share as ONE grouped
// call (disc_executor_run_grouped semantics: per-request flows, grouped launches).  The
// reference runs the same requests one Executor::run at a time (executor.cpp:221-465).
#include <pthread.h>
#include <sched.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <exception>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "capi_common.hpp"
#include "disc_cuda.h"
#include "runtime/runtime_flow.hpp"

using namespace disc;
using disc_capi::guard;

namespace {

std::vector<std::vector<int>> cpu_slices(int n) {
  std::vector<int> cpus;
  cpu_set_t allowed;
  CPU_ZERO(&allowed);
  if (sched_getaffinity(0, sizeof allowed, &allowed) == 0)
    for (int c = 0; c < CPU_SETSIZE; ++c)
      if (CPU_ISSET(c, &allowed)) cpus.push_back(c);
  std::vector<std::vector<int>> out(n);
  if (cpus.empty()) return out;
  for (int w = 0; w < n; ++w) {
    const size_t a = cpus.size() * w / n, b = std::max(a + 1, cpus.size() * (w + 1) / n);
    for (size_t i = a; i < b && i < cpus.size(); ++i) out[w].push_back(cpus[i]);
    if (out[w].empty()) out[w].push_back(cpus[w % cpus.size()]);
  }
  return out;
}

struct Worker {
  int device = 0;
  std::vector<int> cpus;
  std::thread th;
  std::mutex mu;
  std::condition_variable cv;
  std::function<void()> job;
  bool stop = false, busy = false;
  std::exception_ptr err;
  void* stream = nullptr;
  std::unique_ptr<rt::DeviceExecutor> ex;
  std::vector<int> reqs;  // global request ids of the last batch, in order
  int64_t bytes = 0;
  double ms = 0.0;
};

}  // namespace

struct disc_dispatcher_s {
  std::vector<std::unique_ptr<Worker>> workers;
  std::vector<std::pair<int, int>> where;  // request -> (worker, index in the worker's batch)
  std::mutex done_mu;
  std::condition_variable done_cv;
  int pending = 0;

  void loop(Worker& w, int host_threads, std::exception_ptr* init_err, std::mutex* init_mu,
            std::condition_variable* init_cv, int* init_left) {
    if (!w.cpus.empty()) {
      cpu_set_t set;
      CPU_ZERO(&set);
      for (int c : w.cpus) CPU_SET(c, &set);
      pthread_setaffinity_np(pthread_self(), sizeof set, &set);  // the executor's pool inherits the slice
    }
    try {
      if (disc_cuda_set_device(w.device) != 0) throw RuntimeError(std::string("set device: ") + disc_cuda_last_error());
      if (disc_cuda_stream_create(&w.stream) != 0) throw RuntimeError(std::string("stream: ") + disc_cuda_last_error());
      w.ex = std::make_unique<rt::DeviceExecutor>(w.device, w.stream);
      w.ex->set_host_threads(std::max(1, host_threads));
    } catch (...) {
      *init_err = std::current_exception();
    }
    {
      std::lock_guard<std::mutex> l(*init_mu);  // notify under the lock: the waiter owns these
      --*init_left;
      init_cv->notify_all();
    }
    for (;;) {
      std::function<void()> f;
      {
        std::unique_lock<std::mutex> l(w.mu);
        w.cv.wait(l, [&] { return w.stop || w.job; });
        if (w.stop && !w.job) break;
        f = std::move(w.job);
        w.job = nullptr;
      }
      f();
      std::lock_guard<std::mutex> l(done_mu);
      if (--pending == 0) done_cv.notify_all();
    }
    w.ex.reset();
    if (w.stream) disc_cuda_stream_destroy(w.stream);
  }

  ~disc_dispatcher_s() {
    for (auto& w : workers) {
      {
        std::lock_guard<std::mutex> l(w->mu);
        w->stop = true;
      }
      w->cv.notify_all();
    }
    for (auto& w : workers)
      if (w->th.joinable()) w->th.join();
  }
};

extern "C" {

int disc_dispatcher_create(int n_workers, const int* devices, int host_threads, disc_dispatcher* out) {
  return guard([&] {
    if (n_workers < 1) throw Error(ErrorClass::kUsage, "dispatcher needs at least one worker");
    auto d = std::make_unique<disc_dispatcher_s>();
    const auto slices = cpu_slices(n_workers);
    std::exception_ptr init_err;
    std::mutex init_mu;
    std::condition_variable init_cv;
    int left = n_workers;
    for (int w = 0; w < n_workers; ++w) {
      d->workers.push_back(std::make_unique<Worker>());
      Worker& wk = *d->workers.back();
      wk.device = devices ? devices[w] : w;
      wk.cpus = slices[w];
      // host-flow threads per worker: its CPU slice unless the caller says otherwise
      const int ht = host_threads > 0 ? host_threads : static_cast<int>(std::max<size_t>(1, wk.cpus.size()));
      disc_dispatcher_s* self = d.get();
      wk.th = std::thread([self, &wk, ht, &init_err, &init_mu, &init_cv, &left] {
        self->loop(wk, ht, &init_err, &init_mu, &init_cv, &left);
      });
    }
    {
      std::unique_lock<std::mutex> l(init_mu);
      init_cv.wait(l, [&] { return left == 0; });
    }
    if (init_err) std::rethrow_exception(init_err);  // ~disc_dispatcher_s joins the workers
    *out = d.release();
  });
}

void disc_dispatcher_destroy(disc_dispatcher d) { delete d; }

int disc_dispatcher_num_workers(disc_dispatcher d) { return static_cast<int>(d->workers.size()); }

int disc_dispatcher_worker_device(disc_dispatcher d, int w) {
  return w >= 0 && w < static_cast<int>(d->workers.size()) ? d->workers[w]->device : -1;
}

// LPT assignment of a batch (host only): worker_of[r] for every request.
int disc_dispatcher_assign(disc_dispatcher d, int n, const disc_plan* plans, const int* offs, const char* const* names,
                           const int64_t* const* dims, const int* ranks, int* worker_of) {
  return guard([&] {
    std::vector<std::pair<int64_t, int>> cost(n);
    for (int r = 0; r < n; ++r) {
      int64_t b = 0;
      const int i0 = offs[r];
      if (int rc = disc_plan_algorithmic_bytes(plans[r], offs[r + 1] - i0, names + i0, dims + i0, ranks + i0, &b))
        throw RuntimeError(std::string("request ") + std::to_string(r) + ": " + disc_last_error());
      cost[r] = {b, r};
    }
    std::sort(cost.begin(), cost.end(), [](const auto& a, const auto& b) {
      return a.first != b.first ? a.first > b.first : a.second < b.second;
    });
    const int W = static_cast<int>(d->workers.size());
    std::vector<int64_t> load(W, 0);
    for (const auto& [b, r] : cost) {
      int best = 0;
      for (int w = 1; w < W; ++w)
        if (load[w] < load[best]) best = w;
      worker_of[r] = best;
      load[best] += b;
    }
  });
}

// Runs a batch: each worker's share (LPT, or `worker_of` when given) as one grouped call on
// its executor; returns when all are done.  Inputs: host pointers (on_host = 1), or device
// pointers on the device of the worker each request is assigned to (on_host = 0; use
// disc_dispatcher_assign first to place them).
int disc_dispatcher_run_grouped(disc_dispatcher d, int n, const disc_plan* plans, const int* offs,
                                const char* const* names, const void* const* data, const int64_t* const* dims,
                                const int* ranks, int on_host, const int* worker_of) {
  return guard([&] {
    const int W = static_cast<int>(d->workers.size());
    std::vector<int> assign(n);
    if (worker_of) {
      for (int r = 0; r < n; ++r) {
        if (worker_of[r] < 0 || worker_of[r] >= W) throw Error(ErrorClass::kUsage, "worker index out of range");
        assign[r] = worker_of[r];
      }
    } else if (int rc = disc_dispatcher_assign(d, n, plans, offs, names, dims, ranks, assign.data())) {
      throw RuntimeError(disc_last_error());
    }
    d->where.assign(n, {-1, -1});
    struct Share {
      std::vector<const CompiledPlan*> plans;
      std::vector<uint64_t> serials;
      std::vector<int> offs{0};
      std::vector<const char*> names;
      std::vector<const void*> data;
      std::vector<const int64_t*> dims;
      std::vector<int> ranks;
    };
    std::vector<Share> share(W);
    for (auto& w : d->workers) {
      w->reqs.clear();
      w->err = nullptr;
      w->bytes = 0;
    }
    for (int r = 0; r < n; ++r) {
      const int w = assign[r];
      Worker& wk = *d->workers[w];
      Share& s = share[w];
      d->where[r] = {w, static_cast<int>(wk.reqs.size())};
      wk.reqs.push_back(r);
      s.plans.push_back(plans[r]->plan.get());
      s.serials.push_back(plans[r]->serial);
      for (int k = offs[r]; k < offs[r + 1]; ++k) {
        s.names.push_back(names[k]);
        s.data.push_back(data[k]);
        s.dims.push_back(dims[k]);
        s.ranks.push_back(ranks[k]);
      }
      s.offs.push_back(static_cast<int>(s.names.size()));
    }
    {
      std::lock_guard<std::mutex> l(d->done_mu);
      d->pending = 0;
      for (int w = 0; w < W; ++w) d->pending += !d->workers[w]->reqs.empty();
    }
    for (int w = 0; w < W; ++w) {
      Worker& wk = *d->workers[w];
      if (wk.reqs.empty()) continue;
      Share* s = &share[w];
      {
        std::lock_guard<std::mutex> l(wk.mu);
        wk.job = [&wk, s, on_host] {
          const auto t0 = std::chrono::steady_clock::now();
          try {
            wk.ex->run_grouped_batch(static_cast<int>(s->plans.size()), s->plans.data(), s->serials.data(),
                                     s->offs.data(), s->names.data(), s->data.data(), s->dims.data(), s->ranks.data(),
                                     on_host != 0);
            wk.bytes = wk.ex->algorithmic_bytes();
            if (disc_cuda_stream_synchronize(wk.stream) != 0)
              throw RuntimeError(std::string("stream sync: ") + disc_cuda_last_error());
          } catch (...) {
            wk.err = std::current_exception();
          }
          wk.ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        };
      }
      wk.cv.notify_all();
    }
    {
      std::unique_lock<std::mutex> l(d->done_mu);
      d->done_cv.wait(l, [&] { return d->pending == 0; });
    }
    for (auto& w : d->workers)
      if (w->err) std::rethrow_exception(w->err);
  });
}

int disc_dispatcher_request_worker(disc_dispatcher d, int r) {
  return r >= 0 && r < static_cast<int>(d->where.size()) ? d->where[r].first : -1;
}

int disc_dispatcher_num_request_outputs(disc_dispatcher d, int r) {
  if (r < 0 || r >= static_cast<int>(d->where.size()) || d->where[r].first < 0) return -1;
  const auto& ro = d->workers[d->where[r].first]->ex->request_outputs();
  const int j = d->where[r].second;
  return j < static_cast<int>(ro.size()) ? static_cast<int>(ro[j].size()) : -1;
}

int disc_dispatcher_request_output(disc_dispatcher d, int r, int i, const float** dptr, const int64_t** dims,
                                   int* rank, int* device) {
  return guard([&] {
    const auto [w, j] = d->where.at(r);
    if (w < 0) throw Error(ErrorClass::kUsage, "request was not run");
    const auto& o = d->workers[w]->ex->request_outputs().at(j).at(i);
    *dptr = o.ptr;
    *dims = o.dims.data();
    *rank = static_cast<int>(o.dims.size());
    if (device) *device = d->workers[w]->device;
  });
}

int disc_dispatcher_copy_request_output(disc_dispatcher d, int r, int i, void* dst, int dst_on_host) {
  return guard([&] {
    const auto [w, j] = d->where.at(r);
    if (w < 0) throw Error(ErrorClass::kUsage, "request was not run");
    Worker& wk = *d->workers[w];
    const auto& o = wk.ex->request_outputs().at(j).at(i);
    int64_t n = 1;
    for (int64_t x : o.dims) n *= x;
    if (n == 0) return;
    if (disc_cuda_set_device(wk.device) != 0) throw RuntimeError(std::string("set device: ") + disc_cuda_last_error());
    if (disc_cuda_memcpy(dst, o.ptr, static_cast<size_t>(n * 4), dst_on_host ? 1 : 2, wk.stream) != 0)
      throw RuntimeError(std::string("output copy: ") + disc_cuda_last_error());
    if (dst_on_host == 1 && disc_cuda_stream_synchronize(wk.stream) != 0)
      throw RuntimeError(std::string("stream sync: ") + disc_cuda_last_error());
  });
}

int disc_dispatcher_worker_stats(disc_dispatcher d, int w, int64_t* requests, int64_t* bytes, double* ms) {
  return guard([&] {
    const Worker& wk = *d->workers.at(w);
    if (requests) *requests = static_cast<int64_t>(wk.reqs.size());
    if (bytes) *bytes = wk.bytes;
    if (ms) *ms = wk.ms;
  });
}

}  // extern "C"
