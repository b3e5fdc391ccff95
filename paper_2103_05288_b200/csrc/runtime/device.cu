// C ABI of the device layer (include/disc_cuda.h): streams, stream-ordered memory,
// events and the kernel launches the runtime flow issues.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <type_traits>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <unordered_map>
#include <vector>

#include <cuda_profiler_api.h>

#include "disc_cuda.h"
#include "../kernels/kernels.cuh"
#include "../desc_ranges.hpp"

using disc_dev::HostGroup;

namespace disc_launch {
cudaError_t loop(const disc_loop_launch& L, cudaStream_t s, const HostGroup* g = nullptr);
cudaError_t reduce(const disc_reduce_launch& L, cudaStream_t s, const HostGroup* g = nullptr);
cudaError_t col_pass(const disc_reduce_launch& L, cudaStream_t s, const HostGroup* g = nullptr);
cudaError_t finalize_columns(const disc_reduce_launch& L, cudaStream_t s, const HostGroup* g = nullptr);
cudaError_t pad(const disc_pad_launch& P, cudaStream_t s);
cudaError_t concat(const disc_concat_launch& C, cudaStream_t s);
cudaError_t copy2d_group(const HostGroup& H, cudaStream_t s);
cudaError_t gemm(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c, double* ws, cudaStream_t s);
cudaError_t fill_uniform(float* dst, int64_t n, uint64_t seed, float lo, float hi, cudaStream_t s);
cudaError_t flush(void* p, size_t bytes, cudaStream_t s);
cudaError_t spin(uint64_t ns, cudaStream_t s);
void set_pdl(int mode);
int pdl_mode();
}  // namespace disc_launch

// Generated fast paths (patterns_gen.cu): straight-line kernels for known program
// structures, keyed by (schedule kind, structural hash of the lowered program).
namespace disc_spec {
struct Entry {
  int kind;        // 0 loop, 1 row (pre+post), 2 column pass (pre)
  uint64_t key;
  cudaError_t (*launch)(const void* launch, int vec, cudaStream_t s, const HostGroup* g);
};
const Entry* lookup(int kind, uint64_t key);
int count();
}  // namespace disc_spec

namespace {
thread_local std::string t_err;
std::atomic<int64_t> g_launches{0};
std::atomic<int64_t> g_mallocs{0}, g_frees{0}, g_oom_retries{0};  // driver-pool calls (diagnostics)
std::atomic<int64_t> g_spec_launches{0};
std::atomic<int64_t> g_fused_launches{0};  // fused launches (grouped: per member), generated or not
bool g_spec_enabled = true;

// Capture mode (host-only dry run used by the pattern generator): device calls become
// no-ops, allocations return fake aligned addresses, launches are recorded.  The mode is
// per host thread (a dry run must not turn another thread's real executor into a no-op);
// the executor's host-flow workers inherit their caller's mode for each job
// (disc_cuda_set_capture_local).
thread_local bool g_capture = false;
thread_local bool g_capture_record = true;  // capture mode 2: dry run without recording (host timing)
std::atomic<uint64_t> g_fake_next{uint64_t{1} << 36};
std::mutex g_records_mu;
std::vector<std::string> g_records;

uint64_t mix(uint64_t h, uint64_t v) {
  for (int i = 0; i < 8; ++i) {
    h ^= (v >> (8 * i)) & 0xff;
    h *= 1099511628211ull;
  }
  return h;
}

// Structure of a program: everything except pointers and load bindings.
uint64_t program_hash(const disc_program& P) {
  uint64_t h = 14695981039346656037ull;
  h = mix(h, P.n_instr);
  h = mix(h, P.n_slots);
  h = mix(h, P.n_loads);
  h = mix(h, P.n_outs);
  for (int i = 0; i < P.n_instr; ++i) {
    const disc_instr& I = P.code[i];
    const int op = I.op <= DISC_I_LOAD_CONST ? 0 : I.op;
    h = mix(h, (uint64_t)op | ((uint64_t)I.a << 8) | ((uint64_t)I.b << 16) | ((uint64_t)I.flags << 24) |
                   ((uint64_t)I.dst << 32) | ((uint64_t)I.load << 40) | ((uint64_t)I.out << 48));
  }
  for (int l = 0; l < P.n_loads; ++l) h = mix(h, 0x100 + disc_dev::load_class(P.loads[l]));
  return h;
}

std::string program_text(const disc_program& P) {
  std::string s = "{\"slots\":" + std::to_string(P.n_slots) + ",\"loads\":" + std::to_string(P.n_loads) +
                  ",\"outs\":" + std::to_string(P.n_outs) + ",\"code\":[";
  for (int i = 0; i < P.n_instr; ++i) {
    const disc_instr& I = P.code[i];
    const int op = I.op <= DISC_I_LOAD_CONST ? 0 : I.op;
    s += (i ? ",[" : "[") + std::to_string(op) + "," + std::to_string(I.a) + "," + std::to_string(I.b) + "," +
         std::to_string(I.flags) + "," + std::to_string(I.dst) + "," + std::to_string(I.load) + "," +
         std::to_string(I.out) + "]";
  }
  s += "],\"lclass\":[";
  for (int l = 0; l < P.n_loads; ++l) s += (l ? "," : "") + std::to_string(disc_dev::load_class(P.loads[l]));
  return s + "]}";
}

uint64_t launch_key(int kind, const disc_program& a, const disc_program* b) {
  uint64_t h = mix(1469598103934665603ull, kind);
  h = mix(h, program_hash(a));
  if (b) h = mix(h, program_hash(*b));
  return h;
}

void record(const std::string& kind, uint64_t key, const std::string& body) {
  if (!g_capture_record) return;
  char hex[32];
  std::snprintf(hex, sizeof hex, "%016llx", static_cast<unsigned long long>(key));
  std::lock_guard<std::mutex> lock(g_records_mu);
  g_records.push_back("{\"kind\":\"" + kind + "\",\"key\":\"" + hex + "\"," + body + "}");
}

int check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return 0;
  t_err = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return 4;
}
cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

int counted(cudaError_t e, const char* what, int n = 1) {
  if (e == cudaSuccess) g_launches.fetch_add(n, std::memory_order_relaxed);
  return check(e, what);
}

// ---------------------------------------------------------------------------
// Descriptor upload for grouped launches: a pinned host ring mirrored by a device ring
// per stream.  A region stays reserved until the event recorded after the kernel that
// reads it; reuse waits for that event (in practice the ring is large enough that the
// host never waits).
struct Ring {
  unsigned char* host = nullptr;
  unsigned char* dev = nullptr;
  size_t cap = 0, head = 0;
  std::deque<std::tuple<size_t, size_t, cudaEvent_t>> inflight;  // [begin, end) until event
  std::vector<cudaEvent_t> spare;
  // outgrown buffers, freed once the last event recorded while they were current is done
  std::vector<std::tuple<unsigned char*, unsigned char*, cudaEvent_t>> retired;
};
constexpr size_t kRingMax = size_t{1} << 30;

// Outgrown ring buffers are released without blocking the host: the device part
// stream-ordered (cudaFreeAsync), the pinned host part only once its last user is done
// and then kept for the process (cudaFreeHost would synchronise the device); growth is
// geometric (x4 from 64 MB), so this happens a handful of times at most.
void ring_collect(Ring& r, cudaStream_t st) {
  for (size_t i = 0; i < r.retired.size();) {
    auto& [h, d, ev] = r.retired[i];
    if (d) {
      cudaFreeAsync(d, st);
      d = nullptr;
    }
    if (cudaEventQuery(ev) == cudaSuccess) {
      r.spare.push_back(ev);
      r.retired[i] = r.retired.back();
      r.retired.pop_back();
    } else {
      ++i;
    }
  }
}
std::mutex g_ring_mu;
int64_t g_copy_ns = 0, g_copy_bytes = 0;  // host profile (DISC_HOST_PROFILE)
std::unordered_map<cudaStream_t, Ring> g_rings;

cudaError_t ring_reserve(Ring& r, size_t n, cudaStream_t st, size_t* off) {
  n = (n + 255) / 256 * 256;
  ring_collect(r, st);
  {
    // Would the next region have to wait for work still in flight?  Then grow instead
    // (up to kRingMax): the host keeps running ahead of the device.
    size_t b = r.head, e = r.head + n;
    if (e > r.cap) {
      b = 0;
      e = n;
    }
    bool busy = false;
    for (auto& f : r.inflight)
      if (std::get<0>(f) < e && b < std::get<1>(f) && cudaEventQuery(std::get<2>(f)) != cudaSuccess) busy = true;
    if (busy && r.cap < kRingMax && !r.inflight.empty()) {
      cudaEvent_t last = std::get<2>(r.inflight.back());
      r.retired.emplace_back(r.host, r.dev, last);  // 'last' is recorded after every user
      r.inflight.pop_back();
      for (auto& f : r.inflight) r.spare.push_back(std::get<2>(f));
      r.inflight.clear();
      const size_t nc = std::min(kRingMax, std::max(4 * r.cap, n));
      r.host = r.dev = nullptr;
      r.cap = 0;
      r.head = 0;
      if (cudaError_t x = cudaMallocHost(reinterpret_cast<void**>(&r.host), nc)) return x;
      if (cudaError_t x = cudaMallocAsync(reinterpret_cast<void**>(&r.dev), nc, st)) return x;
      r.cap = nc;
    }
  }
  if (n > r.cap) {  // grow: drain everything in flight, then reallocate
    for (auto& f : r.inflight) {
      cudaEventSynchronize(std::get<2>(f));
      r.spare.push_back(std::get<2>(f));
    }
    r.inflight.clear();
    if (r.host) cudaFreeHost(r.host);
    if (r.dev) cudaFree(r.dev);
    r.host = r.dev = nullptr;
    r.cap = std::max<size_t>({n, 4 * r.cap, size_t{64} << 20});
    r.head = 0;
    if (cudaError_t e = cudaMallocHost(reinterpret_cast<void**>(&r.host), r.cap)) return e;
    if (cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&r.dev), r.cap)) return e;
  }
  if (r.head + n > r.cap) r.head = 0;
  const size_t b = r.head, e = r.head + n;
  auto overlaps = [&] {
    for (auto& f : r.inflight)
      if (std::get<0>(f) < e && b < std::get<1>(f)) return true;
    return false;
  };
  while (!r.inflight.empty() && overlaps()) {
    cudaEventSynchronize(std::get<2>(r.inflight.front()));
    r.spare.push_back(std::get<2>(r.inflight.front()));
    r.inflight.pop_front();
  }
  r.head = e;
  *off = b;
  (void)st;
  return cudaSuccess;
}

cudaError_t ring_release(Ring& r, size_t off, size_t n, cudaStream_t st) {
  cudaEvent_t ev;
  if (r.spare.empty()) {
    if (cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) return e;
  } else {
    ev = r.spare.back();
    r.spare.pop_back();
  }
  r.inflight.emplace_back(off, off + (n + 255) / 256 * 256, ev);
  return cudaEventRecord(ev, st);
}

// Kernel instantiation key of a fused launch (members of one grouped launch share it).
struct GroupKey {
  int kind = 0;  // 0 loop, 1 row, 2 column pass
  const disc_spec::Entry* entry = nullptr;
  int vec = 0, wide = 0, red = 0, stage = 0, block = 0, unaligned = 0, regcap = 0, short_rows = 0;
  bool operator<(const GroupKey& o) const {
    return std::tie(kind, entry, vec, wide, red, stage, block, unaligned, regcap, short_rows) <
           std::tie(o.kind, o.entry, o.vec, o.wide, o.red, o.stage, o.block, o.unaligned, o.regcap, o.short_rows);
  }
};

bool regcap_in_key() {  // DISC_REGCAP_KEY=1: separate groups per register-cap choice
  static const bool on = [] {
    const char* e = std::getenv("DISC_REGCAP_KEY");
    return e && std::atoi(e) != 0;
  }();
  return on;
}

bool is_col(int sched) {
  return sched == DISC_SCHED_COL_SINGLE || sched == DISC_SCHED_COL_TWOPASS || sched == DISC_SCHED_COL_ATOMIC;
}

// Grouping key, or false if the launch is issued alone (generic reduce).
bool group_key(int kind, const void* l, GroupKey* k) {
  if (kind == 0) {
    const auto& L = *static_cast<const disc_loop_launch*>(l);
    k->kind = 0;
    k->vec = L.vec;
    k->wide = L.wide;
    k->entry = (g_spec_enabled && !L.wide) ? disc_spec::lookup(0, launch_key(0, L.prog, nullptr)) : nullptr;
    return true;
  }
  const auto& R = *static_cast<const disc_reduce_launch*>(l);
  const bool row = R.schedule == DISC_SCHED_ROW;
  if (!row && !is_col(R.schedule)) return false;
  k->kind = row ? 1 : 2;
  k->vec = R.vec;
  k->wide = R.wide;
  k->red = R.kind;
  k->stage = row ? R.stage : 0;
  k->block = row ? (R.group > 256 ? R.group : 256) : 256;
  k->unaligned = row ? R.unaligned : 0;  // a separate kernel instantiation
  // regcap (k_row_smb) is NOT part of the key: a group runs its largest member's choice
  // (members are issued largest first), so mixed widths never split a group
  k->regcap = (row && regcap_in_key()) ? R.regcap : 0;
  k->short_rows = row ? R.short_rows : 0;  // another kernel (k_row_short)
  const uint64_t key = row ? launch_key(1, R.pre, &R.post) : launch_key(2, R.pre, nullptr);
  k->entry = (g_spec_enabled && !R.wide) ? disc_spec::lookup(row ? 1 : 2, key) : nullptr;
  return true;
}

int64_t launch_weight(int kind, const void* l) {
  if (kind == 0) return static_cast<const disc_loop_launch*>(l)->total;
  const auto& R = *static_cast<const disc_reduce_launch*>(l);
  return R.K * R.R * (R.C > 0 ? R.C : 1);
}

// Grouped launch of one homogeneous group (<= DISC_MAX_GROUP members, same key) in three
// steps: plan (compact record layout), pack (records into a pinned table), launch.
void plan_group(const GroupKey& k, HostGroup& H) {
  // generated groups share one program structure: the first member's ranges cover all
  const int n = k.entry ? 1 : H.n;
  if (k.kind == 0)
    disc_dev::group_segments<disc_loop_launch>(H.members, n, &H.nseg, H.seg, &H.stride);
  else
    disc_dev::group_segments<disc_reduce_launch>(H.members, n, &H.nseg, H.seg, &H.stride);
}

void pack_group(const HostGroup& H, unsigned char* dst) {  // compact records: only the ranges kernels read
  const auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < H.n; ++i) {
    unsigned char* rec = dst + static_cast<size_t>(i) * H.stride;
    const unsigned char* src = static_cast<const unsigned char*>(H.members[i]);
    for (int s = 0; s < H.nseg; ++s) std::memcpy(rec + H.seg[s][2] * 16, src + H.seg[s][0] * 16, H.seg[s][1] * 16);
  }
  g_copy_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
  g_copy_bytes += static_cast<int64_t>(H.stride) * H.n;
}

int launch_group(const GroupKey& k, const HostGroup& H, cudaStream_t st) {
  const void* first = H.members[0];
  int rc = 0;
  if (k.kind == 0) {
    const auto& L = *static_cast<const disc_loop_launch*>(first);
    rc = counted(k.entry ? k.entry->launch(first, L.vec, st, &H) : disc_launch::loop(L, st, &H), "grouped loop");
  } else if (k.kind == 1) {
    const auto& R = *static_cast<const disc_reduce_launch*>(first);
    rc = counted(k.entry ? k.entry->launch(first, R.vec, st, &H) : disc_launch::reduce(R, st, &H), "grouped row reduce");
  } else {
    bool finalize = false;
    for (int i = 0; i < H.n; ++i) {
      const auto& R = *static_cast<const disc_reduce_launch*>(H.members[i]);
      if (R.K * R.C <= 0) continue;
      if (R.schedule == DISC_SCHED_COL_ATOMIC)
        if ((rc = check(cudaMemsetAsync(R.workspace, 0, sizeof(double) * R.K * R.C, st), "workspace memset"))) return rc;
      finalize = finalize || R.schedule != DISC_SCHED_COL_SINGLE;
    }
    const auto& R = *static_cast<const disc_reduce_launch*>(first);
    rc = counted(k.entry ? k.entry->launch(first, R.vec, st, &H) : disc_launch::col_pass(R, st, &H), "grouped column pass");
    if (!rc && finalize) rc = counted(disc_launch::finalize_columns(R, st, &H), "grouped column finalize");
  }
  if (rc) return rc;
  g_spec_launches.fetch_add(k.entry ? H.n : 0, std::memory_order_relaxed);
  g_fused_launches.fetch_add(H.n, std::memory_order_relaxed);
  return 0;
}

// Stand-alone grouped launch (disc_cuda_launch_*_group): its own table upload.
int issue_group(const GroupKey& k, const std::vector<const void*>& members, cudaStream_t st) {
  HostGroup H{};
  H.members = members.data();
  H.n = static_cast<int>(members.size());
  plan_group(k, H);
  const size_t bytes = static_cast<size_t>(H.stride) * H.n;
  std::lock_guard<std::mutex> lock(g_ring_mu);
  Ring& r = g_rings[st];
  size_t off = 0;
  if (int rc = check(ring_reserve(r, bytes, st, &off), "group table")) return rc;
  pack_group(H, r.host + off);
  if (int rc = check(cudaMemcpyAsync(r.dev + off, r.host + off, bytes, cudaMemcpyHostToDevice, st), "group table upload"))
    return rc;
  H.dev_table = r.dev + off;
  if (int rc = launch_group(k, H, st)) return rc;
  return check(ring_release(r, off, bytes, st), "group table release");
}

// Grouped copy kernel over a table of disc_copy2d items already on the device.
int launch_copies(const disc_dev::disc_copy2d* host_items, const unsigned char* dev_items, int n, cudaStream_t st) {
  std::vector<const void*> ptrs(n);
  for (int i = 0; i < n; ++i) ptrs[i] = host_items + i;
  HostGroup H{};
  H.members = ptrs.data();
  H.n = n;
  H.dev_table = dev_items;
  H.stride = static_cast<int32_t>(sizeof(disc_dev::disc_copy2d));
  return counted(disc_launch::copy2d_group(H, st), "grouped copy");
}

// Concat (eval_concat) as one 2-D copy per part.
void concat_items(const disc_concat_launch& C, std::vector<disc_dev::disc_copy2d>& out) {
  int64_t a = C.axis_offset;
  for (int p = 0; p < C.n_parts; ++p) {
    const int64_t cols = C.part_axis[p] * C.inner;
    if (C.outer > 0 && cols > 0)
      out.push_back({C.parts[p], C.out + a * C.inner, C.outer, cols, cols, C.axis_total * C.inner});
    a += C.part_axis[p];
  }
}

// Splits n launches of one kind into homogeneous groups and issues each (largest first).
int issue_grouped(int kind, const void* const* ls, int n, cudaStream_t st, int* issued = nullptr) {
  std::map<GroupKey, std::vector<const void*>> groups;
  std::vector<GroupKey> order;
  for (int i = 0; i < n; ++i) {
    GroupKey k;
    if (!group_key(kind, ls[i], &k)) {  // issued alone
      if (int rc = kind == 0 ? disc_cuda_launch_loop(static_cast<const disc_loop_launch*>(ls[i]), st)
                             : disc_cuda_launch_reduce(static_cast<const disc_reduce_launch*>(ls[i]), st))
        return rc;
      continue;
    }
    auto it = groups.find(k);
    if (it == groups.end()) {
      order.push_back(k);
      it = groups.emplace(k, std::vector<const void*>()).first;
    }
    it->second.push_back(ls[i]);
  }
  for (const GroupKey& k : order) {
    auto& m = groups[k];
    std::stable_sort(m.begin(), m.end(),
                     [&](const void* a, const void* b) { return launch_weight(kind, a) > launch_weight(kind, b); });
    for (size_t i = 0; i < m.size(); i += DISC_MAX_GROUP) {
      std::vector<const void*> chunk(m.begin() + i, m.begin() + std::min(m.size(), i + DISC_MAX_GROUP));
      if (int rc = issue_group(k, chunk, st)) return rc;
      if (issued) ++*issued;
    }
  }
  return 0;
}

// ---------------------------------------------------------------------------
// Per-thread request queue (disc_cuda_queue_*).
enum QKind { kQLoop = 0, kQReduce, kQPad, kQConcat, kQGemm, kQMemcpy, kQMemset };
struct QMemcpy {
  void* dst;
  const void* src;
  size_t bytes;
  int kind;
};
struct QMemset {
  void* dst;
  int value;
  size_t bytes;
};
struct QGemm {
  int64_t m, k, n;
  const float *a, *b;
  float* c;
  double* ws;
};
struct QOp {
  int kind;
  size_t off;  // payload offset in the arena
  int64_t bytes = 0;
  int kernel = -1;
  int sched = -1;  // index into Queue::names
  int grouped = 0;  // fused launch: 1 = groupable (gk valid), 0 = issued alone
  GroupKey gk;      // computed when queued (on the thread that runs the request's flow)
};
struct QRecord {
  int level, members, kernel, sched;
  int64_t bytes;
  cudaEvent_t a = nullptr, b = nullptr;
  float ms = 0.f;
};
// Growable byte arena without zero-fill (descriptors are copied in by used ranges).
struct Arena {
  std::unique_ptr<unsigned char[]> buf;
  size_t cap = 0, used = 0;
  unsigned char* data() const { return buf.get(); }
  void clear() { used = 0; }
  size_t take(size_t n) {  // 16 B aligned offset of n fresh bytes (16 B granules: readable in whole granules)
    n = (n + 15) / 16 * 16;
    const size_t off = (used + 15) / 16 * 16;
    if (off + n > cap) {
      const size_t nc = std::max(off + n, 2 * cap + (size_t{1} << 20));
      std::unique_ptr<unsigned char[]> nb(new unsigned char[nc]);
      if (used) std::memcpy(nb.get(), buf.get(), used);
      buf = std::move(nb);
      cap = nc;
    }
    used = off + n;
    return off;
  }
};

struct Queue {
  bool active = false;
  cudaStream_t stream = nullptr;
  Arena arena;
  std::vector<std::vector<QOp>> reqs;
  size_t mark_from = 0;
  std::vector<void*> frees;
  std::vector<std::string> names;
  std::vector<QRecord> records;
  std::vector<cudaEvent_t> events;  // pool for timing
  size_t next_event = 0;
  std::string sig;                  // disc_cuda_queue_signature
};
thread_local Queue t_q;

bool queued(void* stream) { return t_q.active && S(stream) == t_q.stream; }

template <typename T>
void enqueue(int kind, const T& payload) {
  if (t_q.reqs.empty()) t_q.reqs.emplace_back();
  const size_t off = t_q.arena.take(sizeof(T));
  QOp op{kind, off};
  if constexpr (std::is_same<T, disc_loop_launch>::value || std::is_same<T, disc_reduce_launch>::value) {
    disc_desc::copy_used(reinterpret_cast<T*>(t_q.arena.data() + off), payload);
    op.grouped = group_key(kind == kQLoop ? 0 : 1, &payload, &op.gk) ? 1 : 0;
  } else {
    std::memcpy(t_q.arena.data() + off, &payload, sizeof(T));
  }
  t_q.reqs.back().push_back(op);
}

cudaEvent_t queue_event() {
  if (t_q.next_event == t_q.events.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    t_q.events.push_back(e);
  }
  return t_q.events[t_q.next_event++];
}

}  // namespace

extern "C" {

const char* disc_cuda_last_error(void) { return t_err.c_str(); }

int disc_cuda_device_count(int* n) {
  if (g_capture) {
    *n = 1;
    return 0;
  }
  return check(cudaGetDeviceCount(n), "cudaGetDeviceCount");
}
int disc_cuda_get_device(int* device) {
  if (g_capture) {
    *device = 0;
    return 0;
  }
  return check(cudaGetDevice(device), "cudaGetDevice");
}
int disc_cuda_set_device(int device) {
  if (g_capture) return 0;
  if (int rc = check(cudaSetDevice(device), "cudaSetDevice")) return rc;
  // The stream-ordered pool keeps freed memory (release threshold = max) instead of
  // returning it to the driver at every synchronisation: a stream of fresh shapes misses
  // the exact-size cache on every allocation, and cudaMallocAsync from a warm pool is
  // ~1 us instead of a driver mapping call.
  static std::mutex mu;
  static std::vector<char> done;
  std::lock_guard<std::mutex> lock(mu);
  if (device >= 0 && static_cast<size_t>(device) >= done.size()) done.resize(device + 1, 0);
  if (device >= 0 && !done[device]) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = ~uint64_t{0};
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done[device] = 1;
  }
  return 0;
}

int disc_cuda_device_info(int device, int* sm_count, int64_t* l2_bytes, int64_t* hbm_bytes) {
  if (g_capture) {
    *sm_count = 148;
    *l2_bytes = 126 << 20;
    *hbm_bytes = int64_t{180} << 30;
    return 0;
  }
  cudaDeviceProp p;
  if (int rc = check(cudaGetDeviceProperties(&p, device), "cudaGetDeviceProperties")) return rc;
  *sm_count = p.multiProcessorCount;
  *l2_bytes = p.l2CacheSize;
  *hbm_bytes = static_cast<int64_t>(p.totalGlobalMem);
  return 0;
}

int disc_cuda_stream_create(void** stream) {
  if (g_capture) {  // host-only runs: a distinct fake handle
    *stream = reinterpret_cast<void*>(g_fake_next.fetch_add(4096));
    return 0;
  }
  cudaStream_t s;
  int rc = check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
  *stream = s;
  return rc;
}
int disc_cuda_stream_destroy(void* stream) {
  if (g_capture) return 0;
  return check(cudaStreamDestroy(S(stream)), "cudaStreamDestroy"); }
int disc_cuda_stream_synchronize(void* stream) {
  if (g_capture) return 0;
  return check(cudaStreamSynchronize(S(stream)), "cudaStreamSynchronize");
}
int disc_cuda_device_synchronize(void) {
  if (g_capture) return 0;
  return check(cudaDeviceSynchronize(), "cudaDeviceSynchronize"); }

int disc_cuda_malloc(size_t bytes, void* stream, void** dptr) {
  if (g_capture) {
    *dptr = reinterpret_cast<void*>(g_fake_next.fetch_add((bytes + 4095) / 4096 * 4096 + 4096));
    return 0;
  }
  g_mallocs.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaMallocAsync(dptr, bytes ? bytes : 16, S(stream));
  if (e == cudaErrorMemoryAllocation) {
    g_oom_retries.fetch_add(1, std::memory_order_relaxed);
    // The pool keeps freed memory (release threshold = max): on exhaustion wait for the
    // stream's pending frees, return the pool's unused memory to the driver and retry once.
    (void)cudaGetLastError();
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(S(stream), &cs);
    if (cs == cudaStreamCaptureStatusNone) {
      int dev = 0;
      cudaMemPool_t pool;
      cudaStreamSynchronize(S(stream));
      if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
        cudaMemPoolTrimTo(pool, 0);
      e = cudaMallocAsync(dptr, bytes ? bytes : 16, S(stream));
    }
  }
  return check(e, "cudaMallocAsync");
}
int disc_cuda_free(void* dptr, void* stream) {
  if (g_capture) return 0;
  if (queued(stream)) {  // queued work may still read it: free after the flush
    t_q.frees.push_back(dptr);
    return 0;
  }
  g_frees.fetch_add(1, std::memory_order_relaxed);
  return check(cudaFreeAsync(dptr, S(stream)), "cudaFreeAsync");
}
int disc_cuda_host_alloc(size_t bytes, void** hptr) {
  if (g_capture) {  // host-only runs: pageable memory stands in for pinned
    *hptr = std::malloc(bytes ? bytes : 16);
    return *hptr ? 0 : 4;
  }
  return check(cudaMallocHost(hptr, bytes ? bytes : 16), "cudaMallocHost");
}
int disc_cuda_host_free(void* hptr) {
  if (g_capture) {
    std::free(hptr);
    return 0;
  }
  return check(cudaFreeHost(hptr), "cudaFreeHost");
}

int disc_cuda_memcpy(void* dst, const void* src, size_t bytes, int kind, void* stream) {
  if (!bytes) return 0;
  if (queued(stream) && !(kind & DISC_MEMCPY_NOW)) {
    enqueue(kQMemcpy, QMemcpy{dst, src, bytes, kind});
    return 0;
  }
  if (g_capture) return 0;
  static const cudaMemcpyKind kinds[] = {cudaMemcpyHostToDevice, cudaMemcpyDeviceToHost, cudaMemcpyDeviceToDevice,
                                         cudaMemcpyDefault};
  return check(cudaMemcpyAsync(dst, src, bytes, kinds[kind & 3], S(stream)), "cudaMemcpyAsync");
}
int disc_cuda_memset(void* dst, int value, size_t bytes, void* stream) {
  if (queued(stream)) {
    if (bytes) enqueue(kQMemset, QMemset{dst, value, bytes});
    return 0;
  }
  if (g_capture) return 0;
  return check(cudaMemsetAsync(dst, value, bytes, S(stream)), "cudaMemsetAsync");
}

int disc_cuda_event_create(void** ev) {
  if (g_capture) {
    *ev = reinterpret_cast<void*>(g_fake_next.fetch_add(16));
    return 0;
  }
  cudaEvent_t e;
  int rc = check(cudaEventCreate(&e), "cudaEventCreate");
  *ev = e;
  return rc;
}
int disc_cuda_event_destroy(void* ev) {
  if (g_capture) return 0;
  return check(cudaEventDestroy(static_cast<cudaEvent_t>(ev)), "cudaEventDestroy"); }
int disc_cuda_event_record(void* ev, void* stream) {
  if (g_capture) return 0;
  return check(cudaEventRecord(static_cast<cudaEvent_t>(ev), S(stream)), "cudaEventRecord");
}
int disc_cuda_stream_wait_event(void* stream, void* ev) {
  if (g_capture) return 0;
  return check(cudaStreamWaitEvent(S(stream), static_cast<cudaEvent_t>(ev), 0), "cudaStreamWaitEvent");
}
int disc_cuda_event_synchronize(void* ev) {
  if (g_capture) return 0;
  return check(cudaEventSynchronize(static_cast<cudaEvent_t>(ev)), "cudaEventSynchronize");
}
int disc_cuda_event_elapsed_ms(void* a, void* b, float* ms) {
  if (g_capture) {
    *ms = 0.f;
    return 0;
  }
  return check(cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(a), static_cast<cudaEvent_t>(b)), "cudaEventElapsedTime");
}

int disc_cuda_launch_loop(const disc_loop_launch* l, void* stream) {
  if (l->total <= 0) return 0;
  if (queued(stream)) {  // (capture mode too: the grouping dry run)
    enqueue(kQLoop, *l);
    return 0;
  }
  const uint64_t key = launch_key(0, l->prog, nullptr);
  if (g_capture) {
    if (g_capture_record) record("loop", key, "\"vec\":" + std::to_string(l->vec) + ",\"pre\":" + program_text(l->prog));
    else if (g_spec_enabled && !l->wide) (void)disc_spec::lookup(0, key);
    return 0;
  }
  g_fused_launches.fetch_add(1, std::memory_order_relaxed);
  if (g_spec_enabled && !l->wide)
    if (const disc_spec::Entry* e = disc_spec::lookup(0, key)) {
      g_spec_launches.fetch_add(1, std::memory_order_relaxed);
      return counted(e->launch(l, l->vec, S(stream), nullptr), "launch loop (generated)");
    }
  return counted(disc_launch::loop(*l, S(stream)), "launch loop");
}

int disc_cuda_launch_reduce(const disc_reduce_launch* l, void* stream) {
  if (queued(stream)) {
    enqueue(kQReduce, *l);
    return 0;
  }
  const bool row = l->schedule == DISC_SCHED_ROW;
  const bool col = l->schedule == DISC_SCHED_COL_SINGLE || l->schedule == DISC_SCHED_COL_TWOPASS ||
                   l->schedule == DISC_SCHED_COL_ATOMIC;
  const uint64_t key = row ? launch_key(1, l->pre, &l->post) : launch_key(2, l->pre, nullptr);
  if (g_capture) {
    if (!g_capture_record) {
      if (g_spec_enabled && (row || col)) (void)disc_spec::lookup(row ? 1 : 2, key);
      return 0;
    }
    if (row || col)
      record(row ? "row" : "col", key,
             "\"vec\":" + std::to_string(l->vec) + ",\"stage\":" + std::to_string(row ? l->stage : 0) +
                 ",\"short\":" + std::to_string(row ? l->short_rows : 0) + ",\"regcap\":" + std::to_string(row ? l->regcap : 0) + ",\"pre\":" + program_text(l->pre) +
                 (row ? ",\"post\":" + program_text(l->post) : std::string()));
    return 0;
  }
  const disc_spec::Entry* e = (g_spec_enabled && !l->wide && (row || col)) ? disc_spec::lookup(row ? 1 : 2, key) : nullptr;
  if (e) g_spec_launches.fetch_add(1, std::memory_order_relaxed);
  g_fused_launches.fetch_add(1, std::memory_order_relaxed);
  if (!col) return counted(e ? e->launch(l, l->vec, S(stream), nullptr) : disc_launch::reduce(*l, S(stream)), "launch reduce");
  if (l->K * l->C <= 0) return 0;
  if (l->schedule == DISC_SCHED_COL_ATOMIC) {
    if (int rc = check(cudaMemsetAsync(l->workspace, 0, sizeof(double) * l->K * l->C, S(stream)), "workspace memset"))
      return rc;
  }
  if (int rc = counted(e ? e->launch(l, l->vec, S(stream), nullptr) : disc_launch::col_pass(*l, S(stream)), "launch column pass"))
    return rc;
  if (l->schedule == DISC_SCHED_COL_SINGLE) return 0;
  return counted(disc_launch::finalize_columns(*l, S(stream)), "launch column finalize");
}

int disc_cuda_launch_pad(const disc_pad_launch* l, void* stream) {
  if (l->total <= 0) return 0;
  if (queued(stream)) {
    enqueue(kQPad, *l);
    return 0;
  }
  if (g_capture) return 0;
  return counted(disc_launch::pad(*l, S(stream)), "launch pad");
}
int disc_cuda_launch_concat(const disc_concat_launch* l, void* stream) {
  if (queued(stream)) {
    enqueue(kQConcat, *l);
    return 0;
  }
  if (g_capture) return 0;
  return counted(disc_launch::concat(*l, S(stream)), "launch concat");
}
int disc_cuda_gemm_ws(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c, double* ws,
                      void* stream) {
  if (queued(stream)) {
    enqueue(kQGemm, QGemm{m, k, n, a, b, c, ws});
    return 0;
  }
  if (g_capture) return 0;
  return counted(disc_launch::gemm(m, k, n, a, b, c, ws, S(stream)), "launch gemm");
}
int disc_cuda_gemm(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c, void* stream) {
  return disc_cuda_gemm_ws(m, k, n, a, b, c, nullptr, stream);
}
int disc_cuda_fill_uniform(float* dst, int64_t n, uint64_t seed, float lo, float hi, void* stream) {
  if (g_capture) return 0;
  return counted(disc_launch::fill_uniform(dst, n, seed, lo, hi, S(stream)), "launch fill");
}
int disc_cuda_flush_l2(void* scratch, size_t bytes, void* stream) {
  if (g_capture) return 0;
  return counted(disc_launch::flush(scratch, bytes, S(stream)), "launch flush");
}
int disc_cuda_spin(uint64_t microseconds, void* stream) {
  if (g_capture) return 0;
  return counted(disc_launch::spin(microseconds * 1000ull, S(stream)), "launch spin");
}
int64_t disc_cuda_kernel_launches(void) { return g_launches.load(); }
int64_t disc_cuda_alloc_stats(int64_t* mallocs, int64_t* frees, int64_t* oom_retries) {
  if (mallocs) *mallocs = g_mallocs.load();
  if (frees) *frees = g_frees.load();
  if (oom_retries) *oom_retries = g_oom_retries.load();
  return 0;
}

int disc_cuda_set_pdl(int mode) {
  disc_launch::set_pdl(mode < 0 ? 0 : (mode > 2 ? 2 : mode));
  return 0;
}
int disc_cuda_pdl_mode(void) { return disc_launch::pdl_mode(); }

int disc_cuda_set_specialization(int enabled) {
  g_spec_enabled = enabled != 0;
  return 0;
}
int64_t disc_cuda_specialized_launches(void) { return g_spec_launches.load(); }
int64_t disc_cuda_fused_launches(void) { return g_fused_launches.load(); }
int disc_cuda_profiler(int on) {
  if (g_capture) return 0;
  return check(on ? cudaProfilerStart() : cudaProfilerStop(), "cudaProfiler");
}
int disc_cuda_num_specializations(void) { return disc_spec::count(); }

int disc_cuda_launch_loop_group(const disc_loop_launch* const* launches, int n, void* stream) {
  if (g_capture || n <= 0) return 0;
  return issue_grouped(0, reinterpret_cast<const void* const*>(launches), n, S(stream));
}
int disc_cuda_launch_reduce_group(const disc_reduce_launch* const* launches, int n, void* stream) {
  if (g_capture || n <= 0) return 0;
  return issue_grouped(1, reinterpret_cast<const void* const*>(launches), n, S(stream));
}

int disc_cuda_queue_begin(void* stream) {
  if (t_q.active) {
    t_err = "disc_cuda_queue_begin: a queue is already active on this thread";
    return 5;
  }
  t_q.active = true;
  t_q.stream = S(stream);
  t_q.arena.clear();
  t_q.reqs.clear();
  t_q.frees.clear();
  t_q.mark_from = 0;
  return 0;
}
int disc_cuda_queue_active(void) { return t_q.active ? 1 : 0; }
int disc_cuda_queue_request(void) {
  if (!t_q.active) return 0;
  if (t_q.reqs.empty() || !t_q.reqs.back().empty()) t_q.reqs.emplace_back();
  t_q.mark_from = 0;
  return 0;
}
int disc_cuda_queue_mark(int64_t bytes, int kernel, const char* schedule) {
  if (!t_q.active || t_q.reqs.empty()) return 0;
  auto& ops = t_q.reqs.back();
  if (t_q.mark_from < ops.size()) {
    int name = -1;
    const std::string sched = schedule ? schedule : "";
    for (size_t i = 0; i < t_q.names.size(); ++i)
      if (t_q.names[i] == sched) name = static_cast<int>(i);
    if (name < 0) {
      t_q.names.push_back(sched);
      name = static_cast<int>(t_q.names.size()) - 1;
    }
    ops[t_q.mark_from].bytes = bytes;
    for (size_t i = t_q.mark_from; i < ops.size(); ++i) {
      ops[i].kernel = kernel;
      ops[i].sched = name;
    }
  }
  t_q.mark_from = ops.size();
  return 0;
}

}  // extern "C"

namespace {

// Issues the queued work of `qs` (the calling thread's queue and/or detached ones) level
// by level on qs[0]'s stream; records go to the calling thread.  Three phases: plan every
// level's actions (groups keyed by kernel instantiation, grouped copies, single ops) and
// the size of every group's record table; pack all tables into ONE pinned ring region and
// upload it with one copy; issue the actions -- so consecutive grouped kernels follow each
// other directly (programmatic dependent launch chains them) instead of each waiting
// behind its own table copy.
int flush_queues(const std::vector<Queue*>& qs, int timing) {
  const auto t_start = std::chrono::steady_clock::now();
  const cudaStream_t st = qs[0]->stream;
  t_q.records.clear();
  t_q.next_event = 0;
  std::vector<std::vector<int>> remap(qs.size());
  auto intern = [&](const std::string& n) {
    for (size_t i = 0; i < t_q.names.size(); ++i)
      if (t_q.names[i] == n) return static_cast<int>(i);
    t_q.names.push_back(n);
    return static_cast<int>(t_q.names.size()) - 1;
  };
  for (size_t k = 0; k < qs.size(); ++k)
    for (const auto& n : qs[k]->names) remap[k].push_back(intern(n));
  auto name_of = [&](size_t k, int sched) { return sched >= 0 ? remap[k][sched] : -1; };
  const int copy_name = intern("copy");
  struct ReqRef {
    size_t q;
    const std::vector<QOp>* ops;
  };
  std::vector<ReqRef> reqs;
  size_t levels = 0;
  for (size_t k = 0; k < qs.size(); ++k)
    for (const auto& r : qs[k]->reqs) {
      reqs.push_back({k, &r});
      levels = std::max(levels, r.size());
    }
  struct FOp {
    const QOp* op;
    const unsigned char* p;
    size_t q;
  };
  // ---- phase 1: plan ----
  enum AKind { kSingle, kAlone, kGroup, kCopies };
  struct Action {
    AKind kind;
    int level, members = 1, kernel = -1, sched = -1;
    int64_t bytes = 0;
    FOp f{};                                   // kSingle / kAlone
    int fkind = 0;                             // kAlone: 0 loop, 1 reduce
    GroupKey gk;                               // kGroup
    std::vector<const void*> ptrs;             // kGroup members
    HostGroup H{};                             // kGroup (members/n set when issued)
    std::vector<disc_dev::disc_copy2d> items;  // kCopies
    size_t table = 0, table_bytes = 0;         // offset in the uploaded region
  };
  std::vector<Action> acts;
  size_t total = 0;
  auto place = [&](Action& a, size_t bytes) {
    a.table = total;
    a.table_bytes = bytes;
    total += (bytes + 255) / 256 * 256;
  };
  auto plan_level = [&](size_t lv, std::vector<Action>& acts) {
    // few distinct kernel instantiations per level: a linear key table beats a map
    std::vector<std::pair<GroupKey, std::vector<FOp>>> groups[2];
    std::vector<FOp> alone[2];
    Action copies{kCopies, static_cast<int>(lv)};
    copies.sched = copy_name;
    for (const ReqRef& rr : reqs) {
      if (lv >= rr.ops->size()) continue;
      const QOp& op = (*rr.ops)[lv];
      const unsigned char* p = qs[rr.q]->arena.data() + op.off;
      if (op.kind == kQLoop || op.kind == kQReduce) {
        const int kind = op.kind == kQLoop ? 0 : 1;
        if (!op.grouped) {
          alone[kind].push_back({&op, p, rr.q});
          continue;
        }
        auto& gs = groups[kind];
        size_t gi = 0;
        auto same = [](const GroupKey& a, const GroupKey& b) { return !(a < b) && !(b < a); };
        while (gi < gs.size() && !same(gs[gi].first, op.gk)) ++gi;
        if (gi == gs.size()) gs.emplace_back(op.gk, std::vector<FOp>());
        gs[gi].second.push_back({&op, p, rr.q});
        continue;
      }
      if (op.kind == kQConcat ||
          (op.kind == kQMemcpy && (reinterpret_cast<const QMemcpy*>(p)->kind & 3) == 2 &&
           reinterpret_cast<const QMemcpy*>(p)->bytes % 4 == 0)) {
        if (op.kind == kQConcat) {
          concat_items(*reinterpret_cast<const disc_concat_launch*>(p), copies.items);
        } else {
          const auto& c = *reinterpret_cast<const QMemcpy*>(p);
          const int64_t n = static_cast<int64_t>(c.bytes / 4);
          copies.items.push_back({static_cast<const float*>(c.src), static_cast<float*>(c.dst), 1, n, n, n});
        }
        copies.bytes += op.bytes;
        continue;
      }
      Action a{kSingle, static_cast<int>(lv)};
      a.f = {&op, p, rr.q};
      a.bytes = op.bytes;
      a.kernel = op.kernel;
      a.sched = name_of(rr.q, op.sched);
      acts.push_back(std::move(a));
    }
    for (size_t i0 = 0; i0 < copies.items.size(); i0 += DISC_MAX_GROUP) {
      Action c{kCopies, static_cast<int>(lv)};
      c.sched = copy_name;
      c.bytes = i0 == 0 ? copies.bytes : 0;
      c.items.assign(copies.items.begin() + i0,
                     copies.items.begin() + std::min(copies.items.size(), i0 + DISC_MAX_GROUP));
      c.members = static_cast<int>(c.items.size());
      c.table_bytes = sizeof(disc_dev::disc_copy2d) * c.items.size();
      acts.push_back(std::move(c));
    }
    for (int kind = 0; kind < 2; ++kind) {
      for (const FOp& f : alone[kind]) {
        Action a{kAlone, static_cast<int>(lv)};
        a.f = f;
        a.fkind = kind;
        a.bytes = f.op->bytes;
        a.kernel = f.op->kernel;
        a.sched = name_of(f.q, f.op->sched);
        acts.push_back(std::move(a));
      }
      for (auto& [k, m] : groups[kind]) {
        {  // larger members first (weights computed once)
          std::vector<std::pair<int64_t, size_t>> w(m.size());
          for (size_t i = 0; i < m.size(); ++i) w[i] = {-launch_weight(kind, m[i].p), i};
          std::stable_sort(w.begin(), w.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
          std::vector<FOp> sorted(m.size());
          for (size_t i = 0; i < m.size(); ++i) sorted[i] = m[w[i].second];
          m.swap(sorted);
        }
        for (size_t i = 0; i < m.size(); i += DISC_MAX_GROUP) {
          const size_t e = std::min(m.size(), i + DISC_MAX_GROUP);
          Action g{kGroup, static_cast<int>(lv)};
          g.gk = k;
          g.kernel = m[i].op->kernel;
          g.sched = name_of(m[i].q, m[i].op->sched);
          for (size_t j = i; j < e; ++j) {
            g.ptrs.push_back(m[j].p);
            g.bytes += m[j].op->bytes;
            if (m[j].op->kernel != g.kernel) g.kernel = -1;
            if (name_of(m[j].q, m[j].op->sched) != g.sched) g.sched = -1;
          }
          g.members = static_cast<int>(g.ptrs.size());
          g.H.members = g.ptrs.data();
          g.H.n = g.members;
          plan_group(k, g.H);
          g.table_bytes = static_cast<size_t>(g.H.stride) * g.H.n;
          acts.push_back(std::move(g));
        }
      }
    }
  };
  // levels are planned independently (in parallel for large flushes), then concatenated
  std::vector<std::vector<Action>> per(levels);
  {
    size_t ops = 0;
    for (const ReqRef& rr : reqs) ops += rr.ops->size();
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const size_t nt = ops >= 8192 ? std::min<size_t>(hw, levels) : 1;
    if (nt <= 1) {
      for (size_t lv = 0; lv < levels; ++lv) plan_level(lv, per[lv]);
    } else {
      std::atomic<size_t> next{0};
      auto worker = [&] {
        for (size_t lv; (lv = next.fetch_add(1)) < levels;) plan_level(lv, per[lv]);
      };
      std::vector<std::thread> th;
      for (size_t w = 1; w < nt; ++w) th.emplace_back(worker);
      worker();
      for (auto& t : th) t.join();
    }
  }
  for (auto& v : per)
    for (Action& x : v) {
      if (x.kind == kGroup || x.kind == kCopies) place(x, x.table_bytes);
      acts.push_back(std::move(x));
    }
  if (g_capture) {  // grouping dry run (host only): describe the actions, issue nothing
    static const char* kinds[] = {"single", "alone", "group", "copies"};
    for (const Action& a : acts) {
      std::string sched = a.sched >= 0 ? t_q.names[a.sched] : "mixed";
      std::string j = "{\"level\":" + std::to_string(a.level) + ",\"action\":\"" + kinds[a.kind] +
                      "\",\"members\":" + std::to_string(a.members) + ",\"bytes\":" + std::to_string(a.bytes) +
                      ",\"kernel\":" + std::to_string(a.kernel) + ",\"schedule\":\"" + sched + "\"";
      if (a.kind == kGroup) {
        j += ",\"table_bytes\":" + std::to_string(a.table_bytes) + ",\"generated\":" + (a.gk.entry ? "true" : "false") +
             ",\"order\":[";
        for (size_t i = 0; i < a.ptrs.size(); ++i)
          j += (i ? "," : "") + std::to_string(launch_weight(a.gk.kind == 0 ? 0 : 1, a.ptrs[i]));
        j += "]";
      }
      std::lock_guard<std::mutex> lock(g_records_mu);
      g_records.push_back(j + "}");
    }
    for (Queue* q : qs) {
      q->frees.clear();
      q->reqs.clear();
      q->arena.clear();
    }
    return 0;
  }
  // ---- phase 2: pack every table into one ring region, one upload ----
  const auto t_plan = std::chrono::steady_clock::now();
  std::unique_lock<std::mutex> lock(g_ring_mu);
  Ring& ring = g_rings[st];
  size_t base = 0;
  int rc = 0;
  if (total > 0) {
    rc = check(ring_reserve(ring, total, st, &base), "group tables");
    if (!rc) {
      // pack the member records; large flushes split the packing over threads
      struct Task {
        Action* a;
        int i0, i1;
      };
      std::vector<Task> tasks;
      size_t members = 0;
      for (Action& a : acts) {
        if (a.kind == kGroup) {
          a.H.members = a.ptrs.data();  // (vector moved into acts)
          for (int i = 0; i < a.H.n; i += 256) tasks.push_back({&a, i, std::min(a.H.n, i + 256)});
          members += a.H.n;
        } else if (a.kind == kCopies) {
          std::memcpy(ring.host + base + a.table, a.items.data(), a.table_bytes);
        }
      }
      auto pack_range = [&](size_t t0, size_t t1) {
        for (size_t t = t0; t < t1; ++t) {
          const HostGroup& H = tasks[t].a->H;
          unsigned char* dst = ring.host + base + tasks[t].a->table;
          for (int i = tasks[t].i0; i < tasks[t].i1; ++i) {
            unsigned char* rec = dst + static_cast<size_t>(i) * H.stride;
            const unsigned char* src = static_cast<const unsigned char*>(H.members[i]);
            for (int sg = 0; sg < H.nseg; ++sg)
              std::memcpy(rec + H.seg[sg][2] * 16, src + H.seg[sg][0] * 16, H.seg[sg][1] * 16);
          }
        }
      };
      const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
      const size_t nt = members >= 4096 ? std::min<size_t>(hw, tasks.size()) : 1;
      if (nt <= 1) {
        pack_range(0, tasks.size());
      } else {
        std::vector<std::thread> th;
        for (size_t w = 1; w < nt; ++w)
          th.emplace_back(pack_range, tasks.size() * w / nt, tasks.size() * (w + 1) / nt);
        pack_range(0, tasks.size() / nt);
        for (auto& t : th) t.join();
      }
      rc = check(cudaMemcpyAsync(ring.dev + base, ring.host + base, total, cudaMemcpyHostToDevice, st),
                 "group tables upload");
    }
  }
  lock.unlock();
  const auto t_pack = std::chrono::steady_clock::now();
  // ---- phase 3: issue ----
  auto begin_rec = [&](const Action& a) {
    QRecord rec{a.level, a.members, a.kernel, a.sched, a.bytes};
    if (timing) {
      rec.a = queue_event();
      rec.b = queue_event();
      cudaEventRecord(rec.a, st);
    }
    t_q.records.push_back(rec);
  };
  auto end_rec = [&] {
    if (timing) cudaEventRecord(t_q.records.back().b, st);
  };
  static const bool prof_issue = std::getenv("DISC_HOST_PROFILE") != nullptr;
  double kind_ms[4] = {0, 0, 0, 0};
  int kind_n[4] = {0, 0, 0, 0};
  for (Action& a : acts) {
    if (rc) break;
    const auto t_a = prof_issue ? std::chrono::steady_clock::now() : std::chrono::steady_clock::time_point{};
    begin_rec(a);
    switch (a.kind) {
      case kGroup:
        a.H.members = a.ptrs.data();
        a.H.dev_table = ring.dev + base + a.table;
        rc = launch_group(a.gk, a.H, st);
        break;
      case kCopies:
        rc = launch_copies(a.items.data(), ring.dev + base + a.table, a.members, st);
        break;
      case kAlone:
        rc = a.fkind == 0 ? disc_cuda_launch_loop(reinterpret_cast<const disc_loop_launch*>(a.f.p), st)
                          : disc_cuda_launch_reduce(reinterpret_cast<const disc_reduce_launch*>(a.f.p), st);
        break;
      case kSingle: {
        const unsigned char* p = a.f.p;
        switch (a.f.op->kind) {
          case kQPad: rc = counted(disc_launch::pad(*reinterpret_cast<const disc_pad_launch*>(p), st), "launch pad"); break;
          case kQGemm: {
            const auto& g = *reinterpret_cast<const QGemm*>(p);
            rc = counted(disc_launch::gemm(g.m, g.k, g.n, g.a, g.b, g.c, g.ws, st), "launch gemm");
            break;
          }
          case kQMemcpy: {
            static const cudaMemcpyKind kinds[] = {cudaMemcpyHostToDevice, cudaMemcpyDeviceToHost,
                                                   cudaMemcpyDeviceToDevice, cudaMemcpyDefault};
            const auto& c = *reinterpret_cast<const QMemcpy*>(p);
            rc = check(cudaMemcpyAsync(c.dst, c.src, c.bytes, kinds[c.kind & 3], st), "cudaMemcpyAsync");
            break;
          }
          case kQMemset: {
            const auto& m = *reinterpret_cast<const QMemset*>(p);
            rc = check(cudaMemsetAsync(m.dst, m.value, m.bytes, st), "cudaMemsetAsync");
            break;
          }
        }
        break;
      }
    }
    end_rec();
    if (prof_issue) {
      const int k = static_cast<int>(a.kind) & 3;
      kind_ms[k] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_a).count();
      ++kind_n[k];
    }
  }
  if (prof_issue)
    std::fprintf(stderr, "[disc issue] by action kind (n, ms): 0:%d/%.3f 1:%d/%.3f 2:%d/%.3f 3:%d/%.3f\n", kind_n[0],
                 kind_ms[0], kind_n[1], kind_ms[1], kind_n[2], kind_ms[2], kind_n[3], kind_ms[3]);
  if (total > 0) {
    std::lock_guard<std::mutex> l2(g_ring_mu);
    if (!rc) rc = check(ring_release(ring, base, total, st), "group tables release");
  }
  static const bool prof = std::getenv("DISC_HOST_PROFILE") != nullptr;
  if (prof) {
    const auto t_end = std::chrono::steady_clock::now();
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "[disc flush] %zu actions: plan %.3f ms, pack+upload %.3f ms, issue %.3f ms\n", acts.size(),
                 ms(t_start, t_plan), ms(t_plan, t_pack), ms(t_pack, t_end));
  }
  for (Queue* q : qs) {
    g_frees.fetch_add(static_cast<int64_t>(q->frees.size()), std::memory_order_relaxed);
    for (void* p : q->frees)
      if (!rc) rc = check(cudaFreeAsync(p, st), "cudaFreeAsync");
    q->frees.clear();
    q->reqs.clear();
    q->arena.clear();
  }
  return rc;
}

}  // namespace

extern "C" {

int disc_cuda_queue_flush(int timing) {
  if (!t_q.active) return 0;
  t_q.active = false;  // everything below issues for real
  return flush_queues({&t_q}, timing);
}

void* disc_cuda_queue_detach(void) {
  if (!t_q.active) return nullptr;
  Queue* q = new Queue();
  q->active = false;
  q->stream = t_q.stream;
  std::swap(q->arena, t_q.arena);
  std::swap(q->reqs, t_q.reqs);
  std::swap(q->frees, t_q.frees);
  std::swap(q->names, t_q.names);
  t_q.active = false;
  t_q.reqs.clear();
  t_q.arena.clear();
  t_q.frees.clear();
  return q;
}

// ---- static plans as CUDA graphs ------------------------
// Canonical bytes of a queue's work: per op its kind and the bytes a replay depends on --
// the used descriptor ranges of fused launches (descriptors are zero-filled when built),
// the fields (never padding) of copies, memsets and GEMMs.  Empty: not capturable (frees
// inside the run).  A cached graph is replayed only on an exact match of these bytes.
int disc_cuda_queue_signature(void* queue, const void** data, size_t* n) {
  Queue* q = static_cast<Queue*>(queue);
  std::string& s = q->sig;
  s.clear();
  auto put = [&](const void* p, size_t k) { s.append(static_cast<const char*>(p), k); };
  auto put64 = [&](uint64_t v) { put(&v, sizeof v); };
  if (q->frees.empty()) {
    s.push_back('G');  // capturable (also with no ops: an empty graph)
    for (const auto& r : q->reqs)
      for (const QOp& op : r) {
        put64(static_cast<uint64_t>(op.kind));
        const unsigned char* p = q->arena.data() + op.off;
        if (op.kind == kQLoop || op.kind == kQReduce) {
          disc_desc::Range rg[disc_desc::kMaxRanges];
          const int k = op.kind == kQLoop ? disc_desc::ranges(*reinterpret_cast<const disc_loop_launch*>(p), rg)
                                          : disc_desc::ranges(*reinterpret_cast<const disc_reduce_launch*>(p), rg);
          for (int i = 0; i < k; ++i) put(p + rg[i].off, rg[i].len);
        } else if (op.kind == kQMemcpy) {
          const auto& m = *reinterpret_cast<const QMemcpy*>(p);
          put64(reinterpret_cast<uintptr_t>(m.dst));
          put64(reinterpret_cast<uintptr_t>(m.src));
          put64(m.bytes);
          put64(static_cast<uint64_t>(m.kind));
        } else if (op.kind == kQMemset) {
          const auto& m = *reinterpret_cast<const QMemset*>(p);
          put64(reinterpret_cast<uintptr_t>(m.dst));
          put64(static_cast<uint64_t>(m.value));
          put64(m.bytes);
        } else if (op.kind == kQGemm) {
          const auto& g = *reinterpret_cast<const QGemm*>(p);
          put64(g.m), put64(g.k), put64(g.n);
          put64(reinterpret_cast<uintptr_t>(g.a)), put64(reinterpret_cast<uintptr_t>(g.b));
          put64(reinterpret_cast<uintptr_t>(g.c));
          put64(reinterpret_cast<uintptr_t>(g.ws));
        } else {  // pad / concat descriptors: zero-filled when built (launcher.cpp)
          put(p, op.kind == kQPad ? sizeof(disc_pad_launch) : sizeof(disc_concat_launch));
        }
      }
  }
  *data = s.data();
  *n = s.size();
  return 0;
}

uint64_t disc_cuda_queue_hash(void* queue) {
  const void* d = nullptr;
  size_t n = 0;
  disc_cuda_queue_signature(queue, &d, &n);
  if (!n) return 0;  // not capturable
  uint64_t h = 1469598103934665603ull;
  const unsigned char* b = static_cast<const unsigned char*>(d);
  for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  return h ? h : 1;
}

void disc_cuda_queue_discard(void* queue) { delete static_cast<Queue*>(queue); }

// Issues a detached queue's ops in order (no grouping) inside a stream capture, then
// instantiates and launches the graph; *graph_exec receives it (nullptr if the queue could
// not be captured, in which case the ops were issued directly).  Consumes the queue.
int disc_cuda_queue_issue_graph(void* queue, void** graph_exec) {
  Queue* q = static_cast<Queue*>(queue);
  const bool want = graph_exec != nullptr;
  if (want) *graph_exec = nullptr;
  const cudaStream_t st = q->stream;
  auto issue_all = [&]() -> int {
    for (const auto& r : q->reqs)
      for (const QOp& op : r) {
        const unsigned char* p = q->arena.data() + op.off;
        int rc = 0;
        switch (op.kind) {
          case kQLoop: rc = disc_cuda_launch_loop(reinterpret_cast<const disc_loop_launch*>(p), st); break;
          case kQReduce: rc = disc_cuda_launch_reduce(reinterpret_cast<const disc_reduce_launch*>(p), st); break;
          case kQPad: rc = disc_cuda_launch_pad(reinterpret_cast<const disc_pad_launch*>(p), st); break;
          case kQConcat: rc = disc_cuda_launch_concat(reinterpret_cast<const disc_concat_launch*>(p), st); break;
          case kQGemm: {
            const auto& g = *reinterpret_cast<const QGemm*>(p);
            rc = disc_cuda_gemm_ws(g.m, g.k, g.n, g.a, g.b, g.c, g.ws, st);
            break;
          }
          case kQMemcpy: {
            const auto& c = *reinterpret_cast<const QMemcpy*>(p);
            rc = disc_cuda_memcpy(c.dst, c.src, c.bytes, c.kind & 3, st);
            break;
          }
          case kQMemset: {
            const auto& m = *reinterpret_cast<const QMemset*>(p);
            rc = disc_cuda_memset(m.dst, m.value, m.bytes, st);
            break;
          }
        }
        if (rc) {
          if (std::getenv("DISC_GRAPH_DEBUG"))
            std::fprintf(stderr, "[disc graph] op kind %d failed: %s\n", op.kind, t_err.c_str());
          return rc;
        }
      }
    return 0;
  };
  int rc = 0;
  bool done = false;
  // (the legacy default stream cannot be captured; a failed begin leaves its error to clear)
  bool capturing = false;
  if (want && q->frees.empty() && st != nullptr) {
    capturing = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (!capturing) cudaGetLastError();
  }
  if (capturing) {
    disc_dev::set_capturing(true);
    const int irc = issue_all();
    disc_dev::set_capturing(false);
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(st, &g);
    cudaGraphExec_t ex = nullptr;
    if (irc == 0 && e == cudaSuccess && g && cudaGraphInstantiate(&ex, g, 0) == cudaSuccess) {
      rc = check(cudaGraphLaunch(ex, st), "cudaGraphLaunch");
      if (!rc) {
        g_launches.fetch_add(1, std::memory_order_relaxed);
        *graph_exec = ex;
      } else {
        cudaGraphExecDestroy(ex);
      }
      done = true;
    }
    if (g) cudaGraphDestroy(g);
    if (!done) {  // capture not possible: issue directly below
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
        cudaGraph_t junk = nullptr;
        cudaStreamEndCapture(st, &junk);
        if (junk) cudaGraphDestroy(junk);
      }
      cudaGetLastError();
    }
  }
  if (!done) {
    rc = issue_all();
    g_frees.fetch_add(static_cast<int64_t>(q->frees.size()), std::memory_order_relaxed);
    for (void* f : q->frees)
      if (!rc) rc = check(cudaFreeAsync(f, st), "cudaFreeAsync");
  }
  delete q;
  return rc;
}

int disc_cuda_graph_launch(void* graph_exec, void* stream) {
  const int rc = check(cudaGraphLaunch(static_cast<cudaGraphExec_t>(graph_exec), S(stream)), "cudaGraphLaunch");
  if (!rc) g_launches.fetch_add(1, std::memory_order_relaxed);
  return rc;
}
int disc_cuda_graph_destroy(void* graph_exec) {
  return check(cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(graph_exec)), "cudaGraphExecDestroy");
}

int64_t disc_cuda_host_profile(int64_t* table_bytes) {
  if (table_bytes) *table_bytes = g_copy_bytes;
  const int64_t ns = g_copy_ns;
  g_copy_ns = g_copy_bytes = 0;
  return ns;
}

int disc_cuda_queue_flush_detached(void* const* queues, int n, int timing) {
  std::vector<Queue*> qs;
  if (t_q.active) {
    t_q.active = false;
    qs.push_back(&t_q);
  }
  for (int i = 0; i < n; ++i)
    if (queues[i]) qs.push_back(static_cast<Queue*>(queues[i]));
  int rc = 0;
  if (!qs.empty()) rc = flush_queues(qs, timing);
  for (int i = 0; i < n; ++i) delete static_cast<Queue*>(queues[i]);
  return rc;
}

int disc_cuda_queue_num_records(void) { return static_cast<int>(t_q.records.size()); }
int disc_cuda_queue_record(int i, int* level, int* members, int64_t* bytes, int* kernel, const char** schedule,
                           float* ms) {
  if (i < 0 || i >= static_cast<int>(t_q.records.size())) {
    t_err = "disc_cuda_queue_record: index out of range";
    return 5;
  }
  QRecord& r = t_q.records[i];
  if (r.a && r.b && r.ms == 0.f) {
    if (int rc = check(cudaEventSynchronize(r.b), "cudaEventSynchronize")) return rc;
    if (int rc = check(cudaEventElapsedTime(&r.ms, r.a, r.b), "cudaEventElapsedTime")) return rc;
  }
  *level = r.level;
  *members = r.members;
  *bytes = r.bytes;
  *kernel = r.kernel;
  *schedule = r.sched >= 0 ? t_q.names[r.sched].c_str() : "mixed";
  *ms = r.ms;
  return 0;
}

int disc_cuda_set_capture(int enabled) {
  g_capture = enabled != 0;
  g_capture_record = enabled == 1;
  if (g_capture) {
    std::lock_guard<std::mutex> lock(g_records_mu);
    g_records.clear();
  }
  return 0;
}
int disc_cuda_set_capture_local(int mode) {
  g_capture = mode != 0;
  g_capture_record = mode == 1;
  return 0;
}
int disc_cuda_capture_mode(void) { return g_capture ? (g_capture_record ? 1 : 2) : 0; }
int disc_cuda_capturing(void) { return g_capture ? 1 : 0; }

int disc_cuda_capture_records(char** json) {
  std::lock_guard<std::mutex> lock(g_records_mu);
  std::string s = "[";
  for (size_t i = 0; i < g_records.size(); ++i) s += (i ? ",\n" : "\n") + g_records[i];
  s += "\n]";
  *json = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(*json, s.c_str(), s.size() + 1);
  return 0;
}

}  // extern "C"
