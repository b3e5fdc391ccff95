// Tape -> device program binding and schedule selection (see launcher.hpp).
#include "launcher.hpp"

#include "../desc_ranges.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>
#include <mutex>
#include <unordered_set>
#include <tuple>
#include <unordered_map>

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

std::vector<int64_t> row_major(const std::vector<int64_t>& dims) {
  std::vector<int64_t> s(dims.size(), 1);
  for (int i = static_cast<int>(dims.size()) - 2; i >= 0; --i) s[i] = s[i + 1] * dims[i + 1];
  return s;
}

// ---------------------------------------------------------------------------
// Gather maps: consumer flat index f -> source flat index.

struct Map {
  std::vector<int64_t> dims, strides;  // consumer dims (row-major), source stride per dim
  int64_t offset = 0;
  bool operator==(const Map& o) const { return dims == o.dims && strides == o.strides && offset == o.offset; }
};

// Drops extent-1 dims and merges contiguous neighbours; the result is a canonical form
// (equal canonical forms => equal functions).
Map canonical(const Map& m) {
  Map c;
  c.offset = m.offset;
  for (size_t i = 0; i < m.dims.size(); ++i) {
    if (m.dims[i] == 1) continue;
    if (!c.dims.empty() && c.strides.back() == m.strides[i] * m.dims[i]) {
      c.dims.back() *= m.dims[i];
      c.strides.back() = m.strides[i];
      continue;
    }
    c.dims.push_back(m.dims[i]);
    c.strides.push_back(m.strides[i]);
  }
  if (c.dims.empty()) {
    c.dims = {1};
    c.strides = {0};
  }
  return c;
}

bool is_identity(const Map& c) {  // c canonical
  if (c.offset != 0) return false;
  return c.dims.size() == 1 && (c.strides[0] == 1 || c.dims[0] == 1);
}

Map identity_map(int64_t n) { return canonical(Map{{n}, {1}, 0}); }

Map broadcast_map(const std::vector<int64_t>& in, const std::vector<int64_t>& out, const std::vector<int64_t>& bdims) {
  Map m;
  m.dims = out;
  m.strides.assign(out.size(), 0);
  auto st = row_major(in);
  for (size_t i = 0; i < bdims.size(); ++i)
    if (in[i] != 1) m.strides[bdims[i]] = st[i];
  return canonical(m);
}

Map slice_map(const std::vector<int64_t>& in, const std::vector<int64_t>& starts, const std::vector<int64_t>& steps,
              const std::vector<int64_t>& out) {
  Map m;
  m.dims = out;
  auto st = row_major(in);
  for (size_t i = 0; i < in.size(); ++i) {
    m.offset += starts[i] * st[i];
    m.strides.push_back(steps[i] * st[i]);
  }
  return canonical(m);
}

Map transpose_map(const std::vector<int64_t>& in, const std::vector<int64_t>& perm) {
  Map m;
  auto st = row_major(in);
  for (int64_t p : perm) {
    m.dims.push_back(in[p]);
    m.strides.push_back(st[p]);
  }
  return canonical(m);
}

bool is_const_map(const Map& c) {  // c canonical
  for (int64_t st : c.strides)
    if (st != 0) return false;
  return true;
}

// ---------------------------------------------------------------------------
// Program assembly: SSA values (one per instruction) -> accumulator + slots; loads are
// bound to the launch's [rows, W] view afterwards (bind_view).

struct NotFusible {
  const char* why;
};

struct Built {
  disc_program prog;
  std::vector<Map> maps;       // per load (canonical, over the consumer's flat index)
  std::vector<int> load_pc;    // LOAD instruction of each load
};

class ProgramBuilder {
 public:
  int load(const float* ptr, const Map& c) {
    auto key = std::make_tuple(ptr, c.dims, c.strides, c.offset);
    auto it = cse_.find(key);
    if (it != cse_.end()) return it->second;
    if (maps_.size() >= DISC_MAX_LOADS) throw NotFusible{"too many loads"};
    ptrs_.push_back(ptr);
    maps_.push_back(c);
    int v = push({DISC_OP_LOAD, -1, -1, static_cast<int>(maps_.size()) - 1});
    cse_[key] = v;
    return v;
  }
  int op(int code, int a, int b = -1) {
    // Fused row epilogue: x / REDVAL -> x * (1 / REDVAL), the reciprocal once per row
    // (softmax normalisation; within 1.5 ulp of the IEEE quotient).  Unfused plans never
    // see REDVAL, so their IEEE division stays bit-exact.
    if (code == DISC_OP_DIV && b >= 0 && b == red_ && rcp_enabled()) {
      if (rcp_ < 0) rcp_ = push({DISC_OP_RCPVAL, -1, -1, -1});
      return push({DISC_OP_MUL, a, rcp_, -1});
    }
    if (code == DISC_OP_DIV && fast_div_) return push({DISC_OP_FDIV, a, b, -1});
    return push({code, a, b, -1});
  }
  // Programs of multi-member (fused) groups divide with a * rcp.approx(b) (<= 2 ulp;
  // the north-star tolerance is 1e-5); single-op plans keep IEEE division (bit-exact
  // against the reference, test_executor.cpp:317-332).  DISC_FAST_DIV=0 disables.
  void set_fast_div(bool on) {
    static const bool enabled = [] {
      const char* e = std::getenv("DISC_FAST_DIV");
      return !e || std::atoi(e) != 0;
    }();
    fast_div_ = on && enabled;
  }
  int redval() {
    if (red_ < 0) red_ = push({DISC_OP_REDVAL, -1, -1, -1});
    return red_;
  }
  static bool rcp_enabled() {
    static const bool on = [] {
      const char* e = std::getenv("DISC_RCP_REDVAL");
      return !e || std::atoi(e) != 0;
    }();
    return on;
  }
  void output(int v, float* ptr) { outs_.emplace_back(v, ptr); }

  // result >= 0: the program must end with that value in the accumulator.
  Built finish(int result) {
    std::vector<int> out_of(ins_.size(), -1);
    std::vector<float*> out_ptrs;
    for (auto [v, ptr] : outs_) {
      int o = static_cast<int>(out_ptrs.size());
      if (o >= DISC_MAX_OUTS) throw NotFusible{"too many outputs"};
      out_ptrs.push_back(ptr);
      if (out_of[v] < 0) {
        out_of[v] = o;
      } else {
        push({DISC_OP_COPY, v, -1, -1});
        out_of.push_back(o);
      }
    }
    if (result >= 0 && result != static_cast<int>(ins_.size()) - 1) {
      push({DISC_OP_COPY, result, -1, -1});
      out_of.push_back(-1);
    }
    out_of.resize(ins_.size(), -1);
    const int n = static_cast<int>(ins_.size());
    if (n > DISC_MAX_INSTR) throw NotFusible{"program too long"};

    // Operands not produced by the immediately preceding instruction (and every COPY
    // operand) are read from a slot.
    std::vector<int> last_use(n, -1);
    std::vector<char> slotted(n, 0);
    auto from_slot = [&](int i, int v) { return v >= 0 && (v != i - 1 || ins_[i].code == DISC_OP_COPY); };
    for (int i = 0; i < n; ++i)
      for (int v : {ins_[i].a, ins_[i].b})
        if (from_slot(i, v)) {
          slotted[v] = 1;
          last_use[v] = std::max(last_use[v], i);
        }
    std::vector<int> slot_of(n, -1);
    std::vector<int> holder(DISC_MAX_SLOTS, -1);
    int nslots = 0;
    Built B;
    std::memset(&B.prog, 0, sizeof B.prog);
    disc_program& P = B.prog;
    B.load_pc.assign(maps_.size(), -1);
    for (int i = 0; i < n; ++i) {
      for (int s = 0; s < DISC_MAX_SLOTS; ++s)
        if (holder[s] >= 0 && last_use[holder[s]] <= i) holder[s] = -1;
      const Ins& x = ins_[i];
      disc_instr& I = P.code[i];
      const bool sa = from_slot(i, x.a), sb = from_slot(i, x.b);
      I.a = sa ? static_cast<uint8_t>(slot_of[x.a]) : 0;
      I.b = sb ? static_cast<uint8_t>(slot_of[x.b]) : 0;
      switch (x.code) {
        case DISC_OP_LOAD:
          I.op = DISC_I_LOAD_ID;  // patched by bind_view
          I.load = static_cast<uint8_t>(x.load);
          B.load_pc[x.load] = i;
          break;
        case DISC_OP_REDVAL:
          I.op = DISC_I_REDVAL;
          break;
        case DISC_OP_RCPVAL:
          I.op = DISC_I_RCPVAL;
          break;
        case DISC_OP_COPY:
          I.op = DISC_I_COPY;
          break;
        case DISC_OP_EXP: case DISC_OP_TANH: case DISC_OP_NEG:
          I.op = static_cast<uint8_t>(DISC_I_UN + 2 * (x.code - DISC_OP_EXP) + (sa ? 1 : 0));
          break;
        case DISC_OP_FDIV:
          I.op = static_cast<uint8_t>(DISC_I_FDIV + (sa ? 2 : 0) + (sb ? 1 : 0));
          break;
        default:
          I.op = static_cast<uint8_t>(DISC_I_BIN + 4 * (x.code - DISC_OP_ADD) + (sa ? 2 : 0) + (sb ? 1 : 0));
          break;
      }
      if (out_of[i] >= 0) {
        I.flags |= DISC_F_OUT;
        I.out = static_cast<uint8_t>(out_of[i]);
      }
      if (slotted[i]) {
        int s = 0;
        while (s < DISC_MAX_SLOTS && holder[s] >= 0) ++s;
        if (s == DISC_MAX_SLOTS) throw NotFusible{"too many live values"};
        holder[s] = i;
        slot_of[i] = s;
        I.flags |= DISC_F_SLOT;
        I.dst = static_cast<uint8_t>(s);
        nslots = std::max(nslots, s + 1);
      }
    }
    P.n_instr = n;
    P.n_slots = nslots;
    P.cache_mode = DISC_CACHE_NONE;
    P.flags = disc_cuda_pdl_mode() == 2 ? DISC_PROG_PDL_EARLY : 0;
    for (int l = 0; l < DISC_MAX_LOADS; ++l) P.cache_slot[l] = -1;
    for (int o = 0; o < DISC_MAX_OUTS; ++o) P.out_slot[o] = -1;
    P.n_loads = static_cast<int32_t>(maps_.size());
    for (size_t l = 0; l < maps_.size(); ++l) P.loads[l].ptr = ptrs_[l];
    B.maps = maps_;
    P.n_outs = static_cast<int32_t>(out_ptrs.size());
    for (size_t o = 0; o < out_ptrs.size(); ++o) P.outs[o] = out_ptrs[o];
    return B;
  }

 private:
  struct Ins {
    int code, a, b, load;
  };
  std::vector<Ins> ins_;
  std::vector<const float*> ptrs_;
  std::vector<Map> maps_;
  std::map<std::tuple<const float*, std::vector<int64_t>, std::vector<int64_t>, int64_t>, int> cse_;
  std::vector<std::pair<int, float*>> outs_;
  int red_ = -1;
  int rcp_ = -1;
  bool fast_div_ = false;
  int push(Ins i) {
    ins_.push_back(i);
    return static_cast<int>(ins_.size()) - 1;
  }
};

// Binds every load of `b` to the [rows, W] view (f = row*W + col).
void bind_view(Built& b, int64_t W) {
  disc_program& P = b.prog;
  for (size_t l = 0; l < b.maps.size(); ++l) {
    const Map& c = b.maps[l];
    disc_load& L = P.loads[l];
    const float* ptr = L.ptr;
    std::memset(&L, 0, sizeof L);
    L.ptr = ptr;
    int op;
    if (is_identity(c)) {
      L.mode = DISC_LOAD_IDENTITY;
      op = DISC_I_LOAD_ID;
    } else if (is_const_map(c)) {
      L.mode = DISC_LOAD_CONST;
      L.offset = c.offset;
      op = DISC_I_LOAD_CONST;
    } else if (c.dims.size() == 1) {  // src = off + f*s = off + row*(W*s) + col*s
      L.mode = DISC_LOAD_AFFINE;
      L.offset = c.offset;
      L.rs = W * c.strides[0];
      L.cs = c.strides[0];
      op = DISC_I_LOAD_AFF;
    } else if (c.dims.size() == 2 && c.dims[1] == W) {
      L.mode = DISC_LOAD_AFFINE;
      L.offset = c.offset;
      L.rs = c.strides[0];
      L.cs = c.strides[1];
      op = DISC_I_LOAD_AFF;
    } else {
      if (c.dims.size() > DISC_MAX_RANK) throw NotFusible{"gather rank too large"};
      L.mode = DISC_LOAD_GATHER;
      L.rank = static_cast<int32_t>(c.dims.size());
      L.offset = c.offset;
      for (size_t d = 0; d < c.dims.size(); ++d) {
        L.dims[d] = c.dims[d];
        L.strides[d] = c.strides[d];
        if (c.dims[d] < (int64_t{1} << 31)) fast_div_magic(static_cast<uint32_t>(c.dims[d]), &L.magic[d], &L.shift[d]);
      }
      op = DISC_I_LOAD_GATHER;
    }
    P.code[b.load_pc[l]].op = static_cast<uint8_t>(op);
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// VEC=4 feasibility for every load/output of the programs on a [*, W] view; sets vec_ok
// (whether each load can be fetched whole at the chosen vector width).
int choose_vec(const std::vector<Built*>& progs, int64_t W) {
  bool v4 = W % 4 == 0;
  for (Built* b : progs) {
    disc_program& P = b->prog;
    for (int o = 0; o < P.n_outs && v4; ++o)
      if (!aligned16(P.outs[o])) v4 = false;
    for (int l = 0; l < P.n_loads && v4; ++l) {
      const disc_load& L = P.loads[l];
      if (L.mode == DISC_LOAD_IDENTITY && !aligned16(L.ptr)) v4 = false;
      if (L.mode == DISC_LOAD_GATHER && L.dims[L.rank - 1] % 4 != 0) v4 = false;
    }
  }
  for (Built* b : progs) {
    disc_program& P = b->prog;
    for (int l = 0; l < P.n_loads; ++l) {
      disc_load& L = P.loads[l];
      if (L.mode == DISC_LOAD_AFFINE) {
        const bool ok = !v4 || (aligned16(L.ptr) && L.offset % 4 == 0 && L.rs % 4 == 0);
        L.vec_ok = L.cs == 0 ? 2 : (L.cs == 1 && ok) ? 1 : 0;
      } else if (L.mode == DISC_LOAD_GATHER) {
        const int r = L.rank;
        const int64_t inner = L.strides[r - 1];
        bool ok = inner == 1 && (!v4 || (aligned16(L.ptr) && L.offset % 4 == 0));
        for (int d = 0; d < r - 1 && ok && v4; ++d) ok = L.strides[d] % 4 == 0;
        L.vec_ok = inner == 0 ? 2 : (ok ? 1 : 0);
      }
    }
  }
  return v4 ? 4 : 1;
}

// Largest element index any load of P can touch on a [rows, W] view: kernels index in 32
// bits unless this (or the view itself) reaches 2^31 (the launch's `wide` flag).
int64_t max_reach(const disc_program& P, int64_t rows, int64_t W) {
  int64_t m = rows * W;
  for (int l = 0; l < P.n_loads; ++l) {
    const disc_load& L = P.loads[l];
    int64_t r = L.offset;
    if (L.mode == DISC_LOAD_AFFINE) {
      r += std::max<int64_t>(rows - 1, 0) * std::abs(L.rs) + std::max<int64_t>(W - 1, 0) * std::abs(L.cs) + 3;
    } else if (L.mode == DISC_LOAD_GATHER) {
      for (int d = 0; d < L.rank; ++d) r += std::max<int64_t>(L.dims[d] - 1, 0) * std::abs(L.strides[d]);
      r += 3;
    }
    m = std::max(m, r);
  }
  return m;
}

// Row width for an elementwise launch: the innermost extent that makes the most loads
// 2D-affine (no per-element division); the whole space as one row when all loads are
// contiguous or constant.
int64_t choose_width(const Built& b, int64_t total) {
  std::vector<int64_t> cands;
  for (const Map& c : b.maps)
    if (!is_identity(c) && !is_const_map(c) && c.dims.size() >= 2) cands.push_back(c.dims.back());
  int64_t best = total;
  int best_score = -1;
  for (int64_t W : cands) {
    if (W <= 0 || total % W != 0) continue;
    int score = 0;
    for (const Map& c : b.maps)
      score += is_identity(c) || is_const_map(c) || c.dims.size() == 1 || (c.dims.size() == 2 && c.dims[1] == W);
    score = score * 2 + (W % 4 == 0);
    if (score > best_score) {
      best_score = score;
      best = W;
    }
  }
  return best > 0 ? best : 1;
}

int lanes_per_row(int64_t W, int vec) {
  const int64_t per = (W / vec + 1) / 2;  // CH = 2 chunks per lane
  int l = 1;
  while (l < per && l < 32) l <<= 1;
  return l;
}

constexpr int64_t kWideLimitView = (int64_t{1} << 31) - 64;

// Placeholder pointer of the reduce-argument cache load (16 B aligned, never dereferenced:
// the load is always served from shared memory, see disc_reduce_launch.arg_slot).
const float* const kArgCachePtr = reinterpret_cast<const float*>(uintptr_t{0xA5C0} << 4);

// DISC_UNALIGNED_ROWS=0 keeps odd-width rows on the scalar (vec 1) row kernel (A/B).
bool unaligned_rows_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("DISC_UNALIGNED_ROWS");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

// Narrowest odd row width that takes the float4-body row kernel (DISC_UNALIGNED_MIN, A/B).
int64_t unaligned_min_width() {
  static const int64_t w = [] {
    const char* e = std::getenv("DISC_UNALIGNED_MIN");
    return int64_t{e ? std::atoi(e) : 16};  // A/B: 16 beats the staged kernel on R = 17, 31 (C1 3897 -> 4122)
  }();
  return w;
}

// DISC_SINGLE_ROWS=0 keeps single-element rows on the row schedule (A/B).
bool single_rows_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("DISC_SINGLE_ROWS");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

// A device float holding -inf (the MAX identity as a hoisted constant load), one per
// device layer (capture mode: a fake address that is never read).
const float* neg_inf_ptr() {
  if (disc_cuda_capturing()) return reinterpret_cast<const float*>(uintptr_t{0xA5D0} << 4);  // dry runs: never read
  static std::mutex mu;
  static std::map<int, const float*> per_device;
  int dev = 0;
  disc_cuda_get_device(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = per_device.find(dev);
  if (it != per_device.end()) return it->second;
  void* d = nullptr;
  const float v = -INFINITY;
  if (disc_cuda_malloc(sizeof(float), nullptr, &d) != 0 ||
      disc_cuda_memcpy(d, &v, sizeof v, 0 | DISC_MEMCPY_NOW, nullptr) != 0 || disc_cuda_stream_synchronize(nullptr) != 0)
    throw RuntimeError(std::string("constant allocation: ") + disc_cuda_last_error());
  return per_device[dev] = static_cast<const float*>(d);
}

// DISC_ARG_CACHE=0 disables the reduce-argument cache (A/B).
// Shortest rows whose fused epilogue reads the cached reduce argument (DISC_SHORT_ARG_MIN;
// 32 restores round 1's behaviour: recompute below a warp-width of floats).
int64_t short_arg_min() {
  static const int64_t v = [] {
    const char* e = std::getenv("DISC_SHORT_ARG_MIN");
    return e ? std::max<int64_t>(2, std::atoll(e)) : int64_t{2};
  }();
  return v;
}

// Row passes per column-reduce split (DISC_COL_MIN_PASSES; round 1: 8).
int64_t col_min_passes() {
  static const int64_t v = [] {
    const char* e = std::getenv("DISC_COL_MIN_PASSES");
    return e ? std::max<int64_t>(1, std::atoll(e)) : int64_t{128};  // A/B r2r: 8/32 -> 128: +10% large
  }();
  return v;
}

// Short rows staged through shared memory from this width (DISC_STAGE_MIN; round 1: 16).
// Default 32 = off: on B200 the staged kernel lost at every width (grouped, 4 GB per
// shape: S=2 2864 -> 1759, S=7 3072 -> 2426, S=20 vs S=24 unstaged 2677 vs 4968 GB/s).
// Scalar rows of even width too when on (DISC_STAGE_EVEN=0: odd widths only).
int64_t stage_min() {
  static const int64_t v = [] {
    const char* e = std::getenv("DISC_STAGE_MIN");
    return e ? std::max<int64_t>(2, std::atoll(e)) : int64_t{32};  // A/B r2s: staging loses at every width
  }();
  return v;
}
bool stage_even() {
  static const bool on = [] {
    const char* e = std::getenv("DISC_STAGE_EVEN");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

int short_rows_g() {  // DISC_SHORT_G: minimum lanes per row for rows of < 32 floats (1 = off)
  static const int v = [] {
    const char* e = std::getenv("DISC_SHORT_G");
    return e ? std::max(1, std::atoi(e)) : 1;
  }();
  return v;
}

bool short_vec4() {  // DISC_SHORT_VEC4=1: rows of 4k floats (< 32) take the short kernel too
  static const bool on = [] {
    const char* e = std::getenv("DISC_SHORT_VEC4");
    return e && std::atoi(e) != 0;
  }();
  return on;
}

bool short_rows_enabled() {  // DISC_SHORT_ROWS=0: the looped row kernel for short rows too
  static const bool on = [] {
    const char* e = std::getenv("DISC_SHORT_ROWS");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

int row_pad_mode() {  // DISC_ROW_PAD: 0 row-cache rows at pitch R, 1 padded within budget, 2 padded (A/B)
  static const int v = [] {
    const char* e = std::getenv("DISC_ROW_PAD");
    return e ? std::atoi(e) : 1;
  }();
  return v;
}
bool row_pad_enabled() { return row_pad_mode() != 0; }

int short_rows_max() {  // rows narrower than this run one thread per row (DISC_SHORT_MAX)
  static const int v = [] {
    const char* e = std::getenv("DISC_SHORT_MAX");
    return e ? std::max(2, std::min(32, std::atoi(e))) : 8;
  }();
  return v;
}

// Scalar rows narrower than this run the warp-staged short-row kernel (stage 3) when
// their operands are 16 B aligned (DISC_WARP_STAGE_MAX; <= 2 = off, max 32).  Off: A/B s3
// on B200 (grouped softmax, 2 GB per width): S=2 2457 -> 995, S=7 5170 -> 2497, S=17
// 2917 -> 1487, S=31 3032 -> 2208 GB/s -- 64-128 registers (the staging copies, MAXR
// unrolled) and ~1 KB per warp in flight per round trip.
int warp_stage_max() {
  static const int v = [] {
    const char* e = std::getenv("DISC_WARP_STAGE_MAX");
    return e ? std::min(32, std::atoi(e)) : 2;
  }();
  return v;
}

int sum_row_mb_force() {  // 0 off (default), 1 every fused sum row, 2 the width rule, 3 argument-only epilogues
  static const int v = [] {
    const char* e = std::getenv("DISC_SUM_ROW_MB");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

bool col_pow2() {
  static const bool on = [] {
    const char* e = std::getenv("DISC_COL_POW2");
    return e && std::atoi(e) != 0;
  }();
  return on;
}

// Row launches staged by TMA bulk copies (DISC_TMA_ROWS, DISC_TMA_MIN_R / _MAX_R, and the
// double buffer's shared-memory budget DISC_TMA_SMEM_KB).
bool tma_rows_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("DISC_TMA_ROWS");
    return e && std::atoi(e) != 0;
  }();
  return on;
}
int64_t tma_min_r() {
  static const int64_t v = [] {
    const char* e = std::getenv("DISC_TMA_MIN_R");
    return e ? std::atoll(e) : int64_t{2};
  }();
  return v;
}
int64_t tma_max_r() {
  static const int64_t v = [] {
    const char* e = std::getenv("DISC_TMA_MAX_R");
    return e ? std::atoll(e) : int64_t{4096};
  }();
  return v;
}
int64_t tma_smem_budget() {
  static const int64_t v = [] {
    const char* e = std::getenv("DISC_TMA_SMEM_KB");
    return int64_t{e ? std::atoi(e) : 96} * 1024;
  }();
  return v;
}

// Column reduces with C % 4 != 0 fold rows into float4-wide super rows (DISC_COL_FOLD=0: off).
bool fold_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("DISC_COL_FOLD");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

// Few long rows without a fused epilogue run on the column machinery (DISC_SPLIT_ROWS=0: off).
bool split_rows_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("DISC_SPLIT_ROWS");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

bool arg_cache_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("DISC_ARG_CACHE");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

int sm_count();

// Threads per row (power of two) for the row schedule over K rows of R elements:
//  * ~32 chunks per thread, so long rows keep a warp (no block barrier) when rows abound;
//  * widened while that improves machine fill and wave balance: a one-wave grid of
//    sm x (1024 / block) CTAs walks groups of 256/G rows, so the score is
//    min(1, waves) x waves/ceil(waves); wider groups must win by > 3%.
// Row-schedule policy (DISC_ROW_POLICY, read once; for A/B measurement):
//   0  ~32 chunks per thread, widened only to fill the machine
//   1  0 + wave-balance widening
//   2  1 + staged short rows (16 <= R < 32) (default)
int row_policy() {
  static const int p = [] {
    const char* e = std::getenv("DISC_ROW_POLICY");
    return e ? std::atoi(e) : 2;
  }();
  return p;
}

int choose_row_group(int64_t K, int64_t R, int vec) {
  const int64_t chunks = R / vec;
  if (K <= 0 || chunks <= 0) return 1;
  auto np2 = [](int64_t x) {
    int g = 1;
    while (g < x && g < 1024) g <<= 1;
    return g;
  };
  static const int cpt = [] {  // target chunks per thread (DISC_ROW_CPT, A/B)
    const char* e = std::getenv("DISC_ROW_CPT");
    return e ? std::max(1, std::atoi(e)) : 32;
  }();
  int g = np2((chunks + cpt - 1) / cpt);
  if (row_policy() == 0) {
    const int64_t need = (int64_t{sm_count()} * 1024 + K - 1) / K;
    while (g < need && g < 1024 && int64_t{g} * 4 <= chunks) g <<= 1;
    return g;
  }
  auto score = [&](int gg) {
    const int block = std::max(gg, 256);
    const int64_t groups = (K + block / gg - 1) / (block / gg);
    const double slots = double(sm_count()) * std::max(1, 1024 / block);
    const double waves = double(groups) / slots;
    return waves < 1 ? waves : waves / std::ceil(waves);
  };
  double best = score(g);
  for (int gg = g * 2; gg <= 1024 && int64_t{gg} * 4 <= chunks; gg <<= 1) {
    const double sc = score(gg);
    if (sc > best * 1.03) {
      best = sc;
      g = gg;
    }
  }
  return g;
}

disc_loop_launch make_loop(Built& b, int64_t total) {
  disc_loop_launch L;
  std::memset(&L, 0, sizeof L);
  const int64_t W = choose_width(b, total);
  bind_view(b, W);
  L.vec = choose_vec({&b}, W);
  L.prog = b.prog;
  L.total = total;
  L.W = W;
  L.rows = total / W;
  L.wide = total > kWideLimitView || max_reach(L.prog, L.rows, W) > kWideLimitView;
  L.lpr = lanes_per_row(W, L.vec);
  static const int pf = [] {
    const char* e = std::getenv("DISC_PREFETCH");
    return e ? std::atoi(e) : 1;
  }();
  L.prefetch = pf;
  return L;
}

int dhlo_to_op(DhloOpKind k) {
  switch (k) {
    case DhloOpKind::kAdd: return DISC_OP_ADD;
    case DhloOpKind::kSub: return DISC_OP_SUB;
    case DhloOpKind::kMul: return DISC_OP_MUL;
    case DhloOpKind::kDiv: return DISC_OP_DIV;
    case DhloOpKind::kMaximum: return DISC_OP_MAX;
    case DhloOpKind::kExp: return DISC_OP_EXP;
    case DhloOpKind::kTanh: return DISC_OP_TANH;
    case DhloOpKind::kNeg: return DISC_OP_NEG;
    default: throw InternalError("not an elementwise op");
  }
}

// ---------------------------------------------------------------------------
// Binding context for one launch.

struct Binding {
  const KernelArtifact& art;
  const VersionArtifact& ver;
  const std::vector<DevTensor>& ext;
  const std::vector<int64_t>& regs;
  std::vector<std::vector<int64_t>> dims;  // per member
  int red = -1;                            // reduce member
  std::vector<char> post;                  // reachable from the reduce
};

// The map through which member t reads its data argument (broadcast/slice only).
Map arg_map(const Binding& B, int t, const std::vector<int64_t>& arg_dims) {
  const TapeInstr& ti = B.art.tape[t];
  const auto& out = B.dims[t];
  if (ti.kind == DhloOpKind::kDynamicBroadcastInDim)
    return B.ver.implicit_broadcast ? broadcast_map(arg_dims, out, ti.dims) : identity_map(numel(out));
  if (ti.kind == DhloOpKind::kDynamicSlice)
    return slice_map(arg_dims, resolve_all(ti.slice_starts, B.regs), resolve_all(ti.slice_strides, B.regs), out);
  return identity_map(numel(out));
}

const std::vector<int64_t>& ref_dims(const Binding& B, const TapeRef& r) {
  return r.kind == TapeRef::Kind::kExternal ? B.ext.at(r.index).dims : B.dims.at(r.index);
}

// Lowers members into one program.  `red_ptr`/`row_fused` describe how post members
// see the reduce result: REDVAL when row-aligned in a fused row kernel, else a load.
class Lowering {
 public:
  Lowering(const Binding& B, ProgramBuilder& pb, const float* red_ptr, const Map* row_map)
      : B_(B), pb_(pb), red_ptr_(red_ptr), row_map_(row_map) {}

  // Member t is read through an identity load of `ptr` instead of being recomputed
  // (the reduce-argument cache of a fused row epilogue).
  void substitute(int t, const float* ptr) { subst_[t] = ptr; }
  // Rows of one element: the reduce member is the SSA value v (see launch_fused).
  void set_reduce_value(int v) {
    red_value_ = v;
    memo_[B_.red] = v;
  }

  int value(int t) {
    auto it = memo_.find(t);
    if (it != memo_.end()) return it->second;
    auto sb = subst_.find(t);
    if (sb != subst_.end()) return memo_[t] = pb_.load(sb->second, identity_map(numel(B_.dims[t])));
    const TapeInstr& ti = B_.art.tape[t];
    int v;
    if (t == B_.red) {
      v = reduce_at(identity_map(numel(B_.dims[t])));
    } else if (is_elementwise_binary(ti.kind)) {
      int a = at_identity(ti.args[0]);
      int b = at_identity(ti.args[1]);
      v = pb_.op(dhlo_to_op(ti.kind), a, b);
    } else if (is_elementwise_unary(ti.kind)) {
      v = pb_.op(dhlo_to_op(ti.kind), at_identity(ti.args[0]));
    } else if (ti.kind == DhloOpKind::kDynamicBroadcastInDim || ti.kind == DhloOpKind::kDynamicSlice) {
      const TapeRef& a = ti.args[0];
      Map m = arg_map(B_, t, ref_dims(B_, a));
      if (a.kind == TapeRef::Kind::kExternal) v = pb_.load(B_.ext[a.index].ptr, m);
      else if (is_identity(m)) v = value(a.index);
      else if (a.index == B_.red) v = reduce_at(m);
      else throw NotFusible{"member consumed through a gather"};
    } else {
      throw NotFusible{"op kind not fusible"};
    }
    memo_[t] = v;
    return v;
  }

  int at_identity(const TapeRef& r) {
    if (r.kind == TapeRef::Kind::kExternal) return pb_.load(B_.ext[r.index].ptr, identity_map(numel(B_.ext[r.index].dims)));
    return value(r.index);
  }

 private:
  const Binding& B_;
  ProgramBuilder& pb_;
  const float* red_ptr_;
  const Map* row_map_;
  std::map<int, int> memo_;
  std::map<int, const float*> subst_;
  int red_value_ = -1;

  int reduce_at(const Map& m) {
    if (red_value_ >= 0) {  // single-element rows: the reduce is an elementwise value
      if (m == identity_map(numel(B_.dims[B_.red]))) return red_value_;
      throw NotFusible{"reduce read off-row"};
    }
    if (row_map_) {
      if (m == *row_map_) return pb_.redval();
      throw NotFusible{"reduce read off-row"};
    }
    if (!red_ptr_) throw NotFusible{"reduce value unavailable in this phase"};
    return pb_.load(red_ptr_, m);
  }
};

std::vector<int64_t> reduce_out_dims(const std::vector<int64_t>& in, const std::vector<int64_t>& axes) {
  std::vector<int64_t> out;
  for (int i = 0; i < static_cast<int>(in.size()); ++i)
    if (std::find(axes.begin(), axes.end(), i) == axes.end()) out.push_back(in[i]);
  return out;
}

// Reduce geometry over the reduce argument's dims.
struct Geometry {
  int schedule = DISC_SCHED_ROW;
  int64_t K = 1, R = 1, C = 1;
  int rank = 0, mask = 0;
  std::vector<int64_t> gdims;
};

Geometry reduce_geometry(const std::vector<int64_t>& dims, const std::vector<int64_t>& axes) {
  Geometry g;
  int64_t kept = 1, red = 1;
  for (int i = 0; i < static_cast<int>(dims.size()); ++i) {
    bool r = std::find(axes.begin(), axes.end(), i) != axes.end();
    (r ? red : kept) *= dims[i];
  }
  if (kept == 0 || red == 0) {  // empty: identities only (or nothing at all)
    g.K = kept;
    g.R = red;
    return g;
  }
  std::vector<std::pair<int64_t, bool>> seg;
  for (int i = 0; i < static_cast<int>(dims.size()); ++i) {
    if (dims[i] == 1) continue;
    bool r = std::find(axes.begin(), axes.end(), i) != axes.end();
    if (!seg.empty() && seg.back().second == r) seg.back().first *= dims[i];
    else seg.emplace_back(dims[i], r);
  }
  auto pattern = [&](std::initializer_list<bool> p) {
    if (seg.size() != p.size()) return false;
    size_t i = 0;
    for (bool b : p)
      if (seg[i++].second != b) return false;
    return true;
  };
  if (seg.empty()) return g;
  if (pattern({true})) {
    g.R = seg[0].first;
  } else if (pattern({false})) {
    g.K = seg[0].first;
  } else if (pattern({false, true})) {
    g.K = seg[0].first;
    g.R = seg[1].first;
  } else if (pattern({true, false})) {
    g.schedule = DISC_SCHED_COL_SINGLE;
    g.R = seg[0].first;
    g.C = seg[1].first;
  } else if (pattern({false, true, false})) {
    g.schedule = DISC_SCHED_COL_SINGLE;
    g.K = seg[0].first;
    g.R = seg[1].first;
    g.C = seg[2].first;
  } else {
    g.schedule = DISC_SCHED_GENERIC;
    g.K = kept;
    g.R = red;
    g.rank = static_cast<int>(dims.size());
    if (g.rank > DISC_MAX_RANK) throw NotFusible{"rank too large for generic reduce"};
    g.gdims = dims;
    for (int64_t a : axes) g.mask |= 1 << a;
  }
  return g;
}

int next_pow2(int64_t v) {
  int p = 1;
  while (p < v && p < 1024) p <<= 1;
  return p;
}

int sm_count() {
  static int n = [] {
    int sm = 148;
    int64_t l2 = 0, hbm = 0;
    if (disc_cuda_device_info(0, &sm, &l2, &hbm) != 0) sm = 148;
    return sm;
  }();
  return n;
}

constexpr int64_t kWideLimit = (int64_t{1} << 31) - 64;

// ---------------------------------------------------------------------------

struct Plan {
  bool is_reduce = false;
  disc_loop_launch loop;
  disc_reduce_launch red;
  bool has_post_pass = false;
  disc_loop_launch post_pass;
};

}  // namespace

// ---------------------------------------------------------------------------

void fast_div_magic(uint32_t d, uint32_t* magic, uint32_t* shift) {
  if (d <= 1) {
    *magic = 0;
    *shift = 0;
    return;
  }
  uint32_t l = 0;
  while ((uint64_t{1} << l) < d) ++l;  // ceil(log2 d)
  const uint64_t p = 31 + l;
  *magic = static_cast<uint32_t>(((uint64_t{1} << p) + d - 1) / d);
  *shift = static_cast<uint32_t>(p - 32);
}

Scratch::~Scratch() {
  for (auto& c : chunks_) {
    if (src_)
      src_->put_chunk(c.base);
    else
      disc_cuda_free(c.base, stream_);
  }
}

void* Scratch::alloc(int64_t bytes) {
  bytes = (std::max<int64_t>(bytes, 16) + 255) / 256 * 256;
  while (cur_ < chunks_.size() && used_ + bytes > chunks_[cur_].size) {
    ++cur_;
    used_ = 0;
  }
  if (cur_ == chunks_.size()) {
    int64_t size = std::max<int64_t>(bytes, int64_t{64} << 20);
    void* p = nullptr;
    if (src_)
      p = src_->get_chunk(size);
    else
      cuda_ok(disc_cuda_malloc(static_cast<size_t>(size), stream_, &p), "scratch allocation");
    chunks_.push_back({static_cast<char*>(p), size});
    used_ = 0;
  }
  void* p = chunks_[cur_].base + used_;
  used_ += bytes;
  return p;
}

void Scratch::reset() {
  cur_ = 0;
  used_ = 0;
}

std::vector<std::vector<int64_t>> simulate_tape(const KernelArtifact& art, const VersionArtifact& ver,
                                                const std::vector<std::vector<int64_t>>& ext_dims,
                                                const std::vector<int64_t>& regs) {
  std::vector<std::vector<int64_t>> dims(art.tape.size());
  auto arg = [&](const TapeRef& r) -> const std::vector<int64_t>& {
    return r.kind == TapeRef::Kind::kExternal ? ext_dims.at(r.index) : dims.at(r.index);
  };
  for (size_t t = 0; t < art.tape.size(); ++t) {
    const TapeInstr& ti = art.tape[t];
    std::vector<int64_t> out = resolve_all(ti.out_dims, regs);
    const int64_t n = numel(out);
    switch (ti.kind) {
      case DhloOpKind::kAdd: case DhloOpKind::kSub: case DhloOpKind::kMul: case DhloOpKind::kDiv:
      case DhloOpKind::kMaximum: case DhloOpKind::kExp: case DhloOpKind::kTanh: case DhloOpKind::kNeg:
        for (const auto& a : ti.args)
          if (numel(arg(a)) != n) throw RuntimeError("fused elementwise operand size mismatch");
        if (ver.vectorized4 && n % 4 != 0) throw InternalError("vectorized kernel launched with ragged extent");
        dims[t] = out;
        break;
      case DhloOpKind::kReduceSum: case DhloOpKind::kReduceMax:
        dims[t] = reduce_out_dims(arg(ti.args[0]), ti.dims);
        break;
      case DhloOpKind::kDynamicBroadcastInDim: {
        const auto& in = arg(ti.args[0]);
        if (ver.implicit_broadcast) {
          for (size_t i = 0; i < ti.dims.size(); ++i)
            if (in[i] != 1 && in[i] != out[ti.dims[i]]) throw RuntimeError("broadcast dim incompatible at runtime");
        } else if (numel(in) != n) {
          throw InternalError("no-broadcast version launched with non-identity shape");
        }
        dims[t] = out;
        break;
      }
      case DhloOpKind::kDynamicSlice: {
        const auto& in = arg(ti.args[0]);
        auto starts = resolve_all(ti.slice_starts, regs), steps = resolve_all(ti.slice_strides, regs);
        for (size_t i = 0; i < in.size(); ++i) {
          if (steps[i] <= 0) throw RuntimeError("slice stride <= 0");
          if (starts[i] < 0) throw RuntimeError("slice index out of range");
          if (out[i] > 0 && starts[i] + (out[i] - 1) * steps[i] >= in[i]) throw RuntimeError("slice index out of range");
        }
        dims[t] = out;
        break;
      }
      case DhloOpKind::kTranspose: {
        const auto& in = arg(ti.args[0]);
        for (int64_t p : ti.dims) dims[t].push_back(in[p]);
        break;
      }
      case DhloOpKind::kDynamicReshape:
        if (n != numel(arg(ti.args[0]))) throw RuntimeError("reshape element count mismatch at runtime");
        dims[t] = out;
        break;
      case DhloOpKind::kDynamicPad: {
        const auto& in = arg(ti.args[0]);
        auto lo = resolve_all(ti.pad_low, regs), hi = resolve_all(ti.pad_high, regs),
             it = resolve_all(ti.pad_interior, regs);
        for (size_t i = 0; i < in.size(); ++i) {
          if (lo[i] < 0 || hi[i] < 0 || it[i] < 0) throw RuntimeError("negative padding");
          dims[t].push_back(lo[i] + hi[i] + in[i] + (in[i] > 0 ? (in[i] - 1) * it[i] : 0));
        }
        break;
      }
      case DhloOpKind::kConcat: {
        if (ti.args.empty()) throw RuntimeError("concat with no operands");
        std::vector<int64_t> d = arg(ti.args[0]);
        int64_t along = 0;
        for (const auto& a : ti.args) {
          const auto& p = arg(a);
          for (size_t i = 0; i < d.size(); ++i)
            if (static_cast<int64_t>(i) != ti.axis && p[i] != d[i])
              throw RuntimeError("concat non-axis dim mismatch at runtime");
          along += p[ti.axis];
        }
        d[ti.axis] = along;
        dims[t] = d;
        break;
      }
      default:
        throw InternalError("unexpected op in kernel tape");
    }
  }
  return dims;
}

namespace {

void check_capacity(const std::vector<int64_t>& d, const OutBuf& o) {
  if (numel(d) * 4 > o.capacity_bytes) throw InternalError("kernel output exceeds planned buffer size");
}

int64_t algorithmic_bytes(const KernelArtifact& art, const std::vector<DevTensor>& ext,
                          const std::vector<std::vector<int64_t>>& dims) {
  int64_t bytes = 0;
  for (size_t e = 0; e < ext.size(); ++e) {
    int64_t whole = numel(ext[e].dims), sliced = 0;
    bool only_slices = true;
    for (size_t t = 0; t < art.tape.size(); ++t)
      for (const auto& a : art.tape[t].args)
        if (a.kind == TapeRef::Kind::kExternal && a.index == static_cast<int>(e)) {
          if (art.tape[t].kind == DhloOpKind::kDynamicSlice) sliced += numel(dims[t]);
          else only_slices = false;
        }
    bytes += 4 * (only_slices ? std::min(sliced, whole) : whole);
  }
  for (int o : art.output_tape_indices) bytes += 4 * numel(dims[o]);
  return bytes;
}

}  // namespace

int64_t launch_bytes_estimate(const KernelArtifact& art, const VersionArtifact& ver,
                              const std::vector<std::vector<int64_t>>& ext_dims, const std::vector<int64_t>& regs) {
  std::vector<DevTensor> ext(ext_dims.size());
  for (size_t e = 0; e < ext_dims.size(); ++e) ext[e].dims = ext_dims[e];
  return algorithmic_bytes(art, ext, simulate_tape(art, ver, ext_dims, regs));
}

namespace {

// Where the fused lowering sends its work: straight to the device, or into a recipe
// (cached and replayed with real pointers patched in).
class Issuer {
 public:
  virtual ~Issuer() = default;
  virtual void* scratch(int64_t bytes) = 0;
  virtual void loop(const disc_loop_launch& L) = 0;
  virtual void reduce(const disc_reduce_launch& R) = 0;
};

// Issues the fused lowering; throws NotFusible when the tape needs materialisation.
// Host-cost profile of launch_kernel (DISC_FLOW_PROFILE=1: totals printed at exit).
namespace {
struct FlowProf {
  std::atomic<int64_t> calls{0}, hits{0}, ns_total{0}, ns_key{0}, ns_sim{0}, ns_lower{0}, ns_pre{0}, ns_post{0}, ns_bind{0}, ns_sched{0}, ns_issue{0};
  ~FlowProf() {
    if (!std::getenv("DISC_FLOW_PROFILE") || !calls) return;
    std::fprintf(stderr, "[disc flow] launch_kernel: %lld calls, %lld recipe hits; us/call: total %.2f, key %.2f, "
                 "simulate %.2f, lower+issue %.2f\n", (long long)calls.load(), (long long)hits.load(),
                 ns_total / 1e3 / calls, ns_key / 1e3 / calls, ns_sim / 1e3 / calls, ns_lower / 1e3 / calls);
    std::fprintf(stderr, "[disc flow] reduce lowering us/call: pre %.2f, post %.2f, bind %.2f, schedule %.2f, issue %.2f\n",
                 ns_pre / 1e3 / calls, ns_post / 1e3 / calls, ns_bind / 1e3 / calls, ns_sched / 1e3 / calls,
                 ns_issue / 1e3 / calls);
  }
};
FlowProf g_flow_prof;
bool flow_prof_on() {
  static const bool on = std::getenv("DISC_FLOW_PROFILE") != nullptr;
  return on;
}
int64_t now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

LaunchReport launch_fused(Binding& B, const std::vector<OutBuf>& outs, Issuer& issue, SchedulePref pref) {
  const KernelArtifact& art = B.art;
  const int n = static_cast<int>(art.tape.size());
  LaunchReport rep;

  if (B.red < 0) {
    // kLoop: all members identity-aligned over N elements.
    const int64_t N = numel(B.dims[art.output_tape_indices.at(0)]);
    for (int t = 0; t < n; ++t)
      if (numel(B.dims[t]) != N) throw NotFusible{"member size differs from the space"};
    ProgramBuilder pb;
    pb.set_fast_div(B.art.tape.size() > 1);
    Lowering lw(B, pb, nullptr, nullptr);
    for (size_t o = 0; o < art.output_tape_indices.size(); ++o)
      pb.output(lw.value(art.output_tape_indices[o]), outs[o].ptr);
    Built b = pb.finish(-1);
    disc_loop_launch L = make_loop(b, N);
    if (N > 0) {
      issue.loop(L);
      rep.device_kernels = 1;
    }
    rep.schedule = L.vec == 4 ? "loop_v4" : "loop";
    return rep;
  }

  // kInput: reduce-rooted.
  const bool prof = flow_prof_on();
  int64_t tp = prof ? now_ns() : 0;
  auto lap = [&](std::atomic<int64_t>& acc) {
    if (!prof) return;
    const int64_t t = now_ns();
    acc += t - tp;
    tp = t;
  };
  const TapeInstr& rt = art.tape[B.red];
  const TapeRef& rarg = rt.args[0];
  const std::vector<int64_t>& adims = ref_dims(B, rarg);
  const int64_t N = numel(adims);
  for (int t = 0; t < n; ++t)
    if (t != B.red && numel(B.dims[t]) != N) throw NotFusible{"member size differs from the space"};
  Geometry geo = reduce_geometry(adims, rt.dims);
  const int64_t nout = numel(B.dims[B.red]);

  // Reduce result destination: its output buffer, else scratch when an epilogue needs it.
  int red_out_idx = -1;
  for (size_t o = 0; o < art.output_tape_indices.size(); ++o)
    if (art.output_tape_indices[o] == B.red && red_out_idx < 0) red_out_idx = static_cast<int>(o);
  bool has_post = false;
  for (int o : art.output_tape_indices)
    if (B.post[o]) has_post = true;
  float* red_ptr = red_out_idx >= 0 ? outs[red_out_idx].ptr : nullptr;
  if (!red_ptr && has_post) red_ptr = static_cast<float*>(issue.scratch(nout * 4));

  disc_reduce_launch R;
  std::memset(&R, 0, sizeof R);
  R.arg_slot = -1;
  R.kind = rt.kind == DhloOpKind::kReduceSum ? DISC_REDUCE_SUM : DISC_REDUCE_MAX;
  R.red_out = red_ptr;
  R.wide = N > kWideLimit || nout > kWideLimit;

  // Pre program: pre-member outputs, then the reduce argument (left in acc).
  Built pre;
  {
    ProgramBuilder pb;
    pb.set_fast_div(B.art.tape.size() > 1);
    Lowering lw(B, pb, nullptr, nullptr);
    for (size_t o = 0; o < art.output_tape_indices.size(); ++o) {
      int t = art.output_tape_indices[o];
      if (t == B.red || B.post[t]) continue;
      pb.output(lw.value(t), outs[o].ptr);
    }
    int arg = lw.at_identity(rarg);
    pre = pb.finish(arg);
  }

  R.K = geo.K;
  R.R = geo.R;
  R.C = geo.C;
  R.schedule = geo.schedule;
  const bool empty = geo.K == 0 || geo.R == 0 || N == 0;
  if (empty) {
    R.schedule = DISC_SCHED_ROW;  // identities for every (possibly) non-empty output
    R.K = nout;
    R.R = 0;
    R.C = 1;
  }

  // Rows of a single element (softmax over S = 1, ...): the reduce is elementwise -- SUM
  // gives the value itself (exact through the f64 accumulator), MAX gives std::max(-inf, v)
  // (v, or -inf for NaN, as the reference's reduce_step) -- so the whole group runs as ONE
  // vectorised elementwise program instead of a thread-per-row reduction.
  if (R.schedule == DISC_SCHED_ROW && !empty && R.R == 1 && single_rows_enabled()) {
    ProgramBuilder pb;
    pb.set_fast_div(B.art.tape.size() > 1);
    Lowering lw(B, pb, nullptr, nullptr);
    int v = lw.at_identity(rarg);
    if (R.kind == DISC_REDUCE_MAX) v = pb.op(DISC_OP_MAX, pb.load(neg_inf_ptr(), canonical(Map{{geo.K}, {0}, 0})), v);
    lw.set_reduce_value(v);
    for (size_t o = 0; o < art.output_tape_indices.size(); ++o) pb.output(lw.value(art.output_tape_indices[o]), outs[o].ptr);
    Built b = pb.finish(-1);
    disc_loop_launch L = make_loop(b, geo.K);
    issue.loop(L);
    rep.device_kernels = 1;
    rep.schedule = "row1_loop";
    return rep;
  }

  lap(g_flow_prof.ns_pre);
  // Post program: fused into the row kernel when every reduce read is row-aligned.
  Built post;
  std::memset(&post.prog, 0, sizeof post.prog);
  bool post_fused = false, post_pass = false;
  disc_loop_launch PL;
  std::memset(&PL, 0, sizeof PL);
  if (has_post) {
    if (R.schedule == DISC_SCHED_ROW && !empty) {
      Map row = canonical(Map{{R.K, R.R}, {1, 0}, 0});
      try {
        ProgramBuilder pb;
    pb.set_fast_div(B.art.tape.size() > 1);
        Lowering lw(B, pb, nullptr, &row);
        // The epilogue reads the reduce argument back from shared memory (written by the
        // reduce pass) instead of recomputing it (softmax: exp once per element); rows up
        // to 4096 keep every cache slot within 64 KB.  Short rows too (thread per row:
        // 256 rows x R < 32 floats per slot), where the recompute made the epilogue
        // issue-bound; such launches are never staged.
        if (arg_cache_enabled() && rarg.kind == TapeRef::Kind::kMember && R.R >= short_arg_min() && R.R <= 4096)
          lw.substitute(rarg.index, kArgCachePtr);
        for (size_t o = 0; o < art.output_tape_indices.size(); ++o) {
          int t = art.output_tape_indices[o];
          if (B.post[t]) pb.output(lw.value(t), outs[o].ptr);
        }
        post = pb.finish(-1);
        post_fused = true;
      } catch (const NotFusible&) {
      }
    }
    if (!post_fused) {
      if (!red_ptr) throw NotFusible{"no reduce buffer"};
      ProgramBuilder pb;
    pb.set_fast_div(B.art.tape.size() > 1);
      Lowering lw(B, pb, red_ptr, nullptr);
      int64_t Npost = 0;
      for (size_t o = 0; o < art.output_tape_indices.size(); ++o) {
        int t = art.output_tape_indices[o];
        if (!B.post[t]) continue;
        pb.output(lw.value(t), outs[o].ptr);
        Npost = numel(B.dims[t]);
      }
      Built pp = pb.finish(-1);
      PL = make_loop(pp, Npost);
      post_pass = Npost > 0;
    }
  }

  // Few long rows and no fused epilogue (a full reduction [N] -> [1], column sums of
  // [N, 1], ...): one row per thread group would leave most SMs idle (K CTAs), so the rows
  // run on the column machinery with C = 1 -- each row's R split across CTAs, f64 partials
  // joined in a fixed order.
  if (R.schedule == DISC_SCHED_ROW && !empty && !post_fused && split_rows_enabled() && R.K < sm_count() &&
      R.R >= 8192) {
    R.schedule = DISC_SCHED_COL_SINGLE;
    R.C = 1;
  }

  lap(g_flow_prof.ns_post);
  // Bind loads to the schedule's [rows, W] view and pick the vector width.
  if (empty) {
    bind_view(pre, 1);
    R.vec = 1;
  } else if (R.schedule == DISC_SCHED_ROW) {
    bind_view(pre, R.R);
    if (post_fused) bind_view(post, R.R);
    R.vec = choose_vec({&pre, &post}, R.R);
    // Odd-width rows: float4 body from each row's first 16 B-aligned column + scalar
    // head/tail, when every operand is a 16 B-aligned identity, a row splat or a constant.
    // Short rows (R < 32) run the register-resident thread-per-row kernel (see below):
    // scalar, never the unaligned float4 body; rows of 4k floats too with DISC_SHORT_VEC4.
    const bool short_row = short_rows_enabled() && !R.wide && R.R >= 2 &&
                           (R.R < short_rows_max() || (R.vec == 1 && R.R < warp_stage_max())) && (R.vec == 1 || short_vec4());
    if (short_row) {
      R.vec = 1;
      R.short_rows = 1;  // pending: confirmed (or dropped) with the row group below
    }
    if (!short_row && R.vec == 1 && R.R % 4 != 0 && R.R >= unaligned_min_width() && unaligned_rows_enabled()) {
      bool ok = true;
      for (const Built* b : {&pre, &post}) {
        const disc_program& P = b->prog;
        for (int l = 0; l < P.n_loads && ok; ++l) {
          const disc_load& Ld = P.loads[l];
          ok = (Ld.mode == DISC_LOAD_IDENTITY && aligned16(Ld.ptr)) || Ld.mode == DISC_LOAD_CONST ||
               (Ld.mode == DISC_LOAD_AFFINE && Ld.cs == 0);
        }
        for (int o = 0; o < P.n_outs && ok; ++o) ok = aligned16(P.outs[o]);
      }
      if (ok) {
        R.vec = 4;
        R.unaligned = 1;
      }
    }
  } else if (R.schedule == DISC_SCHED_GENERIC) {
    bind_view(pre, 1);
    R.vec = 1;
    R.wide = 1;
    R.g_rank = geo.rank;
    R.g_mask = geo.mask;
    for (int d = 0; d < geo.rank; ++d) R.g_dims[d] = geo.gdims[d];
  } else {
    // Column reduce of [N, C] with C % 4 != 0: fold f = 4 / gcd(C, 4) rows into super rows
    // of f*C floats (a multiple of 4), so the column kernel runs 128-bit loads instead of
    // scalar ones; the finalize sums super-columns c, c + C, ... per output.  Operands must
    // be identity (flat index preserved) or constants, or column broadcasts [N, C] with
    // row stride 0, which read a tiled copy (f repeats of the C values, built by a small
    // loop launch).  The last N mod f rows form a partial super row (kernel tail).
    int64_t fold = 1;
    std::vector<int> tiled;
    if (fold_enabled() && R.K == 1 && R.C % 4 != 0 && R.R >= 64 && !empty) {
      const int64_t f = 4 / std::gcd<int64_t>(R.C, 4);
      bool ok = true;
      for (size_t l = 0; l < pre.maps.size() && ok; ++l) {
        const Map& c = pre.maps[l];
        if (is_identity(c) || is_const_map(c)) continue;
        if (c.dims.size() == 2 && c.dims[1] == R.C && c.strides[0] == 0) {
          tiled.push_back(static_cast<int>(l));
          continue;
        }
        ok = false;
      }
      if (ok) fold = f;
    }
    if (fold > 1) {
      const int64_t C0 = R.C, N0 = R.R;
      R.fold = static_cast<int32_t>(fold);
      R.fold_cout = C0;
      R.fold_tail = static_cast<int32_t>(N0 % fold);
      R.R = N0 / fold;
      R.C = fold * C0;
      std::vector<float*> tiles;
      for (int l : tiled) {  // tile[j*C + c] = src(c), j < f
        ProgramBuilder tb;
        const Map& c = pre.maps[l];
        float* t = static_cast<float*>(issue.scratch(4 * R.C));
        tb.output(tb.load(pre.prog.loads[l].ptr, canonical(Map{{fold, C0}, {0, c.strides[1]}, c.offset})), t);
        Built tbb = tb.finish(-1);
        issue.loop(make_loop(tbb, R.C));
        rep.device_kernels += 1;
        tiles.push_back(t);
      }
      bind_view(pre, R.C);
      for (size_t i = 0; i < tiled.size(); ++i) {  // the tiled copy, affine over the folded view
        disc_load& Ld = pre.prog.loads[tiled[i]];
        std::memset(&Ld, 0, sizeof Ld);
        Ld.ptr = tiles[i];
        Ld.mode = DISC_LOAD_AFFINE;
        Ld.rs = 0;
        Ld.cs = 1;
        pre.prog.code[pre.load_pc[tiled[i]]].op = DISC_I_LOAD_AFF;
      }
      R.vec = choose_vec({&pre}, R.C);
    } else {
      bind_view(pre, R.C);
      R.vec = choose_vec({&pre}, R.C);
    }
  }
  R.pre = pre.prog;
  R.post = post.prog;
  lap(g_flow_prof.ns_bind);
  if (!empty && R.schedule != DISC_SCHED_GENERIC) {
    const bool row_view = R.schedule == DISC_SCHED_ROW;
    const int64_t vrows = row_view ? R.K : R.K * R.R, vW = row_view ? R.R : R.C;
    if (max_reach(R.pre, vrows, vW) > kWideLimit || (post_fused && max_reach(R.post, vrows, vW) > kWideLimit))
      R.wide = 1;
  }

  if (R.schedule == DISC_SCHED_ROW) {
    int g = choose_row_group(R.K, R.R, R.vec);
    if (R.short_rows) g = 1;  // thread per row
    if (short_rows_g() > 1 && R.R < 32) {  // A/B: several lanes per short row (coalesced, fewer iterations)
      const int64_t chunks = (R.R + R.vec - 1) / R.vec;
      int cap = 1;
      while (cap < chunks && cap < 32) cap <<= 1;
      g = std::max(g, std::min(short_rows_g(), cap));
    }
    // Staged short rows (R < 32 floats: even a whole row is under one 128 B line): the
    // block copies its contiguous span of every identity operand through shared memory,
    // one thread per row.  Only when that layout is bank-conflict-free (odd R for scalar
    // rows, odd R/4 for float4 rows); otherwise rows pack 32/G per warp as usual.
    // Staged short rows (stage_min() <= R < 32): scalar rows of any width (odd R is
    // bank-conflict-free, even R 2-way), float4 rows when R/4 is odd.  The cached reduce
    // argument is one more slot.
    bool warp_stage = false;
    // Warp-staged short rows (stage 3, generated programs): every identity operand and
    // output of a warp's 32 rows goes through shared memory with 128-bit coalesced copies
    // (kernels.cuh row_short_body); slots as below, 16 B-aligned operands only.
    if (!empty && R.short_rows && g == 1 && !R.wide && warp_stage_max() > 2) {
      bool ok = true;
      for (const disc_program* P : {&R.pre, &R.post}) {
        for (int l = 0; l < P->n_loads && ok; ++l)
          if (P->loads[l].mode == DISC_LOAD_IDENTITY && P->loads[l].ptr != kArgCachePtr) ok = aligned16(P->loads[l].ptr);
        for (int o = 0; o < P->n_outs && ok; ++o) ok = aligned16(P->outs[o]);
      }
      if (ok) warp_stage = true;
    }
    if (!empty && !R.wide && !R.unaligned && row_policy() >= 2 && R.R < 32 &&
        (warp_stage || (R.R >= stage_min() && (R.vec == 1 ? ((R.R & 1) || stage_even()) : ((R.R / 4) & 1))))) {
      int n = 0;
      auto slot_of_ptr = [&](const float* ptr, const disc_program& P) -> int {
        for (int l = 0; l < P.n_loads; ++l)
          if (P.loads[l].mode == DISC_LOAD_IDENTITY && P.loads[l].ptr == ptr && P.cache_slot[l] >= 0)
            return P.cache_slot[l];
        return -1;
      };
      for (int l = 0; l < R.pre.n_loads; ++l)
        if (R.pre.loads[l].mode == DISC_LOAD_IDENTITY) {
          const int k = slot_of_ptr(R.pre.loads[l].ptr, R.pre);
          R.pre.cache_slot[l] = static_cast<int8_t>(k >= 0 ? k : n++);
        }
      if (post_fused)
        for (int l = 0; l < R.post.n_loads; ++l)
          if (R.post.loads[l].mode == DISC_LOAD_IDENTITY) {
            int k = slot_of_ptr(R.post.loads[l].ptr, R.pre);
            if (k < 0) k = slot_of_ptr(R.post.loads[l].ptr, R.post);
            R.post.cache_slot[l] = static_cast<int8_t>(k >= 0 ? k : n++);
          }
      for (int o = 0; o < R.pre.n_outs; ++o) R.pre.out_slot[o] = static_cast<int8_t>(n++);
      if (post_fused)
        for (int o = 0; o < R.post.n_outs; ++o) R.post.out_slot[o] = static_cast<int8_t>(n++);
      int arg = -1;
      for (int q = 0; post_fused && q < R.post.n_loads; ++q)
        if (R.post.loads[q].ptr == kArgCachePtr) arg = R.post.cache_slot[q];
      const int64_t slot_bytes = (256 * R.R + 3) / 4 * 4 * 4;
      if (n > 0 && n <= 8 && n * slot_bytes <= 112 * 1024) {
        R.stage = warp_stage ? 3 : 1;
        R.arg_slot = arg;  // the reduce pass writes it, the epilogue reads it (never copied in)
        R.cache_loads = n;
        R.pre.cache_mode = DISC_CACHE_READ;
        R.post.cache_mode = DISC_CACHE_READ;
        g = 1;
      } else {
        for (int l = 0; l < DISC_MAX_LOADS; ++l) R.pre.cache_slot[l] = R.post.cache_slot[l] = -1;
        for (int o = 0; o < DISC_MAX_OUTS; ++o) R.pre.out_slot[o] = R.post.out_slot[o] = -1;
      }
    }
    // TMA staging (stage 2): every identity operand of the block's rows arrives by bulk
    // copy into a double-buffered shared-memory span (prefetched one block-iteration
    // ahead), the programs read it from there (and the cached reduce argument), outputs go
    // straight to global memory.  Rows of any width (R % 4 != 0: scalar reads from shared
    // memory, bank-conflict-free across the G lanes of a row).
    if (!empty && !R.wide && !R.stage && tma_rows_enabled() && R.R >= tma_min_r() && R.R <= tma_max_r()) {
      int n = 0, arg = -1;
      auto slot_of = [&](const float* ptr, const disc_program& P) -> int {
        for (int l = 0; l < P.n_loads; ++l)
          if (P.loads[l].mode == DISC_LOAD_IDENTITY && P.loads[l].ptr == ptr && P.cache_slot[l] >= 0)
            return P.cache_slot[l];
        return -1;
      };
      for (int l = 0; l < DISC_MAX_LOADS; ++l) R.pre.cache_slot[l] = R.post.cache_slot[l] = -1;
      for (int l = 0; l < R.pre.n_loads; ++l)
        if (R.pre.loads[l].mode == DISC_LOAD_IDENTITY) {
          const int k = slot_of(R.pre.loads[l].ptr, R.pre);
          R.pre.cache_slot[l] = static_cast<int8_t>(k >= 0 ? k : n++);
        }
      for (int l = 0; post_fused && l < R.post.n_loads; ++l)
        if (R.post.loads[l].mode == DISC_LOAD_IDENTITY) {
          if (R.post.loads[l].ptr == kArgCachePtr) {
            if (arg < 0) arg = n++;
            R.post.cache_slot[l] = static_cast<int8_t>(arg);
            continue;
          }
          int k = slot_of(R.post.loads[l].ptr, R.pre);
          if (k < 0) k = slot_of(R.post.loads[l].ptr, R.post);
          R.post.cache_slot[l] = static_cast<int8_t>(k >= 0 ? k : n++);
        }
      if (R.R % 4 != 0) {  // scalar reads from shared memory
        R.vec = 1;
        R.unaligned = 0;
      }
      int gt = std::max(g, 1);
      auto stage_bytes = [&](int gg) { return int64_t{std::max(gg, 256) / gg} * (R.R + 3) / 4 * 4 * n * 4 * 2; };
      while (stage_bytes(gt) > tma_smem_budget() && gt < 1024) gt <<= 1;
      if (n > 0 && n <= 8 && stage_bytes(gt) <= tma_smem_budget()) {
        g = gt;
        R.stage = 2;
        R.cache_loads = n;
        R.arg_slot = arg;
        R.pre.cache_mode = DISC_CACHE_READ;
        R.post.cache_mode = DISC_CACHE_READ;
        for (int o = 0; o < DISC_MAX_OUTS; ++o) R.pre.out_slot[o] = R.post.out_slot[o] = -1;
      } else {
        for (int l = 0; l < DISC_MAX_LOADS; ++l) R.pre.cache_slot[l] = R.post.cache_slot[l] = -1;
      }
    }
    // Row cache: contiguous loads the epilogue re-reads come from shared memory instead
    // of a second pass over HBM/L2 (softmax: x is read once).
    if (post_fused && !R.stage) {
      int nc = 0;
      for (int q = 0; q < R.post.n_loads; ++q)
        if (R.post.loads[q].ptr == kArgCachePtr) {
          R.arg_slot = nc;
          R.post.cache_slot[q] = static_cast<int8_t>(nc++);
        }
      for (int q = 0; q < R.post.n_loads && nc < 2 + (R.arg_slot >= 0); ++q) {
        if (R.post.loads[q].mode != DISC_LOAD_IDENTITY || R.post.loads[q].ptr == kArgCachePtr) continue;
        for (int p = 0; p < R.pre.n_loads; ++p)
          if (R.pre.loads[p].mode == DISC_LOAD_IDENTITY && R.pre.loads[p].ptr == R.post.loads[q].ptr) {
            if (R.pre.cache_slot[p] < 0) R.pre.cache_slot[p] = static_cast<int8_t>(nc++);
            R.post.cache_slot[q] = R.pre.cache_slot[p];
            break;
          }
      }
      static const int64_t budget = [] {  // row-cache bytes per block (DISC_ROW_CACHE_KB, A/B)
        const char* e = std::getenv("DISC_ROW_CACHE_KB");
        return int64_t{e ? std::atoi(e) : 32} * 1024;  // A/B: 48 -> 32 KB: BERT 5336 -> 5572 GB/s, C1/C2 flat
      }();
      const int64_t rrow = R.unaligned ? (R.R + 6) / 4 * 4 : R.R;  // padded rows (kernels.cuh row_body)
      // Row pitch: the 8 (float4) or 32 (scalar) threads of one shared-memory wavefront
      // are 8/G or 32/G rows x G lanes; with a pitch of G x an odd number of bank units
      // they hit distinct banks (thread-per-row float4 rows of 16 or 32 floats were 4- and
      // 8-way conflicted).
      auto pitch = [&](int gg) -> int64_t {
        const int unit = R.vec == 4 ? 4 : 1, phase = R.vec == 4 ? 8 : 32;
        if (!row_pad_enabled() || R.short_rows || gg >= phase) return rrow;
        int64_t p = (rrow + unit - 1) / unit;
        while (p % gg != 0 || (p / gg) % 2 == 0) ++p;
        return p * unit;
      };
      // The pitch never changes the lane count nor exceeds the budget (DISC_ROW_PAD=2: it
      // may, A/B): grouped launches share the largest member's shared memory.
      auto bytes_at = [&](int gg, int64_t p) { return int64_t{std::max(gg, 256) / gg} * nc * p * 4; };
      auto bytes = [&](int gg) { return bytes_at(gg, row_pad_mode() == 2 ? pitch(gg) : rrow); };
      // the epilogue of an argument-cached launch reads the cache: it must fit (one row of
      // up to 3 slots of 4100 floats), so such launches may exceed the budget up to 64 KB;
      // short rows stay one thread per row within that limit
      const int64_t limit = R.arg_slot >= 0 ? std::max<int64_t>(budget, 64 * 1024) : budget;
      while (nc && bytes(g) > (R.short_rows ? limit : budget) && g < 1024) g <<= 1;
      if (nc && bytes(g) <= limit) {
        R.cache_loads = nc;
        if (pitch(g) != rrow && bytes_at(g, pitch(g)) <= std::max(bytes(g), R.short_rows ? limit : budget))
          R.row_pitch = static_cast<int32_t>(pitch(g));
        R.pre.cache_mode = DISC_CACHE_FILL;
        R.post.cache_mode = DISC_CACHE_READ;
      } else {
        if (R.arg_slot >= 0) throw InternalError("reduce-argument cache over budget");
        for (int l = 0; l < DISC_MAX_LOADS; ++l) R.pre.cache_slot[l] = R.post.cache_slot[l] = -1;
      }
    }
    R.group = g;
    // Short scalar rows, one thread per row: the register-resident kernel (whole row at
    // once, one sequential accumulator) when the programs are generated ones.
    if (R.short_rows)
      R.short_rows = (g == 1 && (!R.stage || R.stage == 3) && !R.unaligned) ? (R.R <= 8 ? 8 : 32) : 0;
    if (R.stage == 3 && !R.short_rows) throw InternalError("warp-staged rows without the short-row kernel");
    // Register cap (6 resident blocks, <= 40 registers) for sum rows with a fused epilogue
    // at <= 256 threads, on long rows and row widths that are multiples of 64 (A/B r3a/r3c
    // on the softmax epilogue, grouped: S = 64 4627 -> 5138, 128 5036 -> 5646, 256 4985 ->
    // 5586, 1024 4480 -> 5143, BERT S = 128 4111 -> 4513 GB/s; but S = 24 4553 -> 3739,
    // 48 4656 -> 3944, 200 4621 -> 4349, and the plain LN sums lose 8%).  On the headline
    // sweep, whose grouped launches mix widths, neither the width rule (4336: it splits the
    // groups) nor capping every fused sum row (4365-4371) beats none (4388 GB/s, A/B r3d/r3e):
    // off by default; DISC_SUM_ROW_MB = 1 caps every fused sum row, 2 applies the width rule.
    if (R.kind == DISC_REDUCE_SUM && post_fused && std::max(g, 256) <= 256) {
      const int mode = sum_row_mb_force();
      // mode 3: epilogues that only read the cached reduce argument (softmax-like: y =
      // arg * 1/sum) -- the pattern that gains -- not LN-like ones that re-read operands
      bool arg_only = R.arg_slot >= 0 && R.post.n_loads >= 1;
      for (int q = 0; q < R.post.n_loads && arg_only; ++q) arg_only = R.post.loads[q].ptr == kArgCachePtr;
      R.regcap = mode == 1 ? 1
                 : (mode == 2 && (R.R >= 256 || (R.R >= 64 && R.R % 64 == 0))) ? 1
                 : (mode == 3 && arg_only && R.R >= 32) ? 1 : 0;
    }
    rep.schedule = R.short_rows ? (R.stage == 3 ? (post_fused ? "row_fused_short_ws" : "row_short_ws")
                                             : (post_fused ? "row_fused_short" : "row_short"))
                   : R.stage == 2 ? (post_fused ? "row_fused_tma" : "row_tma")
                   : R.stage ? (post_fused ? "row_fused_staged" : "row_staged")
                           : post_fused ? (R.cache_loads ? "row_fused_cached" : "row_fused") : "row";
  } else if (R.schedule != DISC_SCHED_GENERIC) {
    if (!R.red_out) R.red_out = static_cast<float*>(issue.scratch(nout * 4));
    // Q lanes per row segment, one VEC-wide column chunk each (each thread keeps its
    // columns and walks rows): the whole row when it has <= 256 chunks (256/Q rows per
    // pass, consecutive threads on consecutive chunks across rows), else equal tiles of
    // <= 256 chunks.  Round 1 used a power of two <= 32 (C = 33 floats: a second tile with
    // one busy lane of 32).  DISC_COL_POW2=1 restores it.
    const int64_t cchunks = (R.C + R.vec - 1) / R.vec;
    int Q = 1;
    while (Q < cchunks && Q < 32) Q <<= 1;
    // pow2 tiles of 32 chunks stay when they waste < 10% (A/B r2v: C = 1000, 4096 3.99-4.14
    // vs 3.80-3.85 TB/s with one 250-chunk row per pass); narrow and badly tiled rows use
    // Q = their chunk count (C = 12: 3197 -> 4062, C = 33 folded: 2265 -> 3701 GB/s)
    const double pow2_eff = double(cchunks) / double(((cchunks + Q - 1) / Q) * Q);
    if (!col_pow2() && (cchunks < 32 || pow2_eff < 0.9)) {
      const int64_t ntile = (cchunks + 255) / 256;
      Q = static_cast<int>(std::max<int64_t>(1, (cchunks + ntile - 1) / ntile));
    }
    R.group = Q;
    const int64_t span = int64_t{Q} * R.vec;
    const int64_t tiles = (R.C + span - 1) / span;
    const int64_t ctas = R.K * tiles;
    const int64_t rows_per_pass = 256 / Q;
    const int64_t want = (int64_t{sm_count()} * 8 + ctas - 1) / ctas;
    // each split covers >= col_min_passes() row passes: a CTA's fixed cost (descriptor
    // staging, the per-column join through shared memory, the partial store) is amortised
    // over enough rows (grouped launches of many members otherwise run 10^5 tiny CTAs)
    const int64_t max_split = std::max<int64_t>(1, R.R / (rows_per_pass * col_min_passes()));
    int64_t splits = std::min(want, max_split);
    if (pref == SchedulePref::kTwoPass || pref == SchedulePref::kAtomic) splits = std::max<int64_t>(splits, 2);
    splits = std::min<int64_t>(std::max<int64_t>(splits, 1), 65535);
    R.splits = static_cast<int32_t>(splits);
    const int64_t nws = R.K * R.C;  // workspace columns (folded: f per output)
    if (splits == 1 && R.fold <= 1) {
      R.schedule = DISC_SCHED_COL_SINGLE;
      rep.schedule = "col_single";
    } else if (pref == SchedulePref::kAtomic && R.kind == DISC_REDUCE_SUM) {
      R.schedule = DISC_SCHED_COL_ATOMIC;
      R.workspace = static_cast<double*>(issue.scratch(8 * nws));
      rep.schedule = "col_atomic";
    } else {
      R.schedule = DISC_SCHED_COL_TWOPASS;  // folded launches always finalize (the fold)
      R.workspace = static_cast<double*>(issue.scratch(8 * nws * splits));
      rep.schedule = "col_twopass";
    }
    if (R.fold > 1) rep.schedule += "_fold";
  } else {
    if (!R.red_out) R.red_out = static_cast<float*>(issue.scratch(nout * 4));
    rep.schedule = "generic";
  }

  lap(g_flow_prof.ns_sched);
  issue.reduce(R);
  lap(g_flow_prof.ns_issue);
  rep.device_kernels += (R.schedule == DISC_SCHED_COL_TWOPASS || R.schedule == DISC_SCHED_COL_ATOMIC) ? 2 : 1;
  if (post_pass) {
    issue.loop(PL);
    rep.device_kernels += 1;
    rep.schedule += "+post";
  }
  return rep;
}

// Single-load program helper for materialisation and standalone artifacts.
void run_copy(const float* src, const Map& m, float* dst, int64_t n, void* stream) {
  if (n <= 0) return;
  ProgramBuilder pb;
  pb.output(pb.load(src, m), dst);
  Built b = pb.finish(-1);
  disc_loop_launch L = make_loop(b, n);
  cuda_ok(disc_cuda_launch_loop(&L, stream), "gather");
}

// Reference semantics member by member: every member is materialised in device
// scratch at its own dims, exactly like run_kernel's scratch tensors.
LaunchReport launch_materialized(Binding& B, const std::vector<OutBuf>& outs, Scratch& scratch, void* stream) {
  const KernelArtifact& art = B.art;
  const int n = static_cast<int>(art.tape.size());
  LaunchReport rep;
  rep.materialized = true;
  rep.schedule = "materialized";
  std::vector<float*> buf(n, nullptr);
  auto tensor = [&](const TapeRef& r) -> DevTensor {
    if (r.kind == TapeRef::Kind::kExternal) return B.ext[r.index];
    return DevTensor{buf[r.index], B.dims[r.index]};
  };
  for (int t = 0; t < n; ++t) {
    const TapeInstr& ti = art.tape[t];
    const int64_t cnt = numel(B.dims[t]);
    buf[t] = static_cast<float*>(scratch.alloc(cnt * 4));
    if (is_elementwise_binary(ti.kind) || is_elementwise_unary(ti.kind)) {
      if (cnt == 0) continue;
      ProgramBuilder pb;
      std::vector<int> vals;
      for (const auto& a : ti.args) {
        DevTensor x = tensor(a);
        vals.push_back(pb.load(x.ptr, identity_map(numel(x.dims))));
      }
      int v = vals.size() == 2 ? pb.op(dhlo_to_op(ti.kind), vals[0], vals[1]) : pb.op(dhlo_to_op(ti.kind), vals[0]);
      pb.output(v, buf[t]);
      Built b = pb.finish(-1);
      disc_loop_launch L = make_loop(b, cnt);
      cuda_ok(disc_cuda_launch_loop(&L, stream), "materialized elementwise");
      rep.device_kernels++;
    } else if (ti.kind == DhloOpKind::kDynamicBroadcastInDim || ti.kind == DhloOpKind::kDynamicSlice) {
      DevTensor x = tensor(ti.args[0]);
      if (cnt == 0) continue;
      run_copy(x.ptr, arg_map(B, t, x.dims), buf[t], cnt, stream);
      rep.device_kernels++;
    } else if (is_reduce(ti.kind)) {
      DevTensor x = tensor(ti.args[0]);
      if (cnt == 0) continue;
      disc_reduce_launch R;
      std::memset(&R, 0, sizeof R);
      R.arg_slot = -1;
      ProgramBuilder pb;
      int v = pb.load(x.ptr, identity_map(numel(x.dims)));
      Built b = pb.finish(v);
      bind_view(b, 1);
      R.pre = b.prog;
      R.kind = ti.kind == DhloOpKind::kReduceSum ? DISC_REDUCE_SUM : DISC_REDUCE_MAX;
      R.red_out = buf[t];
      R.vec = 1;
      R.wide = 1;
      R.group = 1;
      R.K = cnt;
      if (numel(x.dims) == 0) {  // empty reduced extent: identities
        R.schedule = DISC_SCHED_ROW;
        R.R = 0;
        R.C = 1;
      } else {
        R.schedule = DISC_SCHED_GENERIC;
        R.R = numel(x.dims) / cnt;
        R.g_rank = static_cast<int>(x.dims.size());
        if (R.g_rank > DISC_MAX_RANK) throw InternalError("rank too large");
        for (int d = 0; d < R.g_rank; ++d) R.g_dims[d] = x.dims[d];
        for (int64_t a : ti.dims) R.g_mask |= 1 << a;
      }
      cuda_ok(disc_cuda_launch_reduce(&R, stream), "materialized reduce");
      rep.device_kernels++;
    } else {
      throw InternalError("unexpected op in kernel tape");
    }
  }
  for (size_t o = 0; o < art.output_tape_indices.size(); ++o) {
    int t = art.output_tape_indices[o];
    const int64_t bytes = numel(B.dims[t]) * 4;
    if (bytes) cuda_ok(disc_cuda_memcpy(outs[o].ptr, buf[t], static_cast<size_t>(bytes), 2, stream), "output copy");
  }
  return rep;
}

LaunchReport launch_standalone(Binding& B, const std::vector<OutBuf>& outs, void* stream) {
  const TapeInstr& ti = B.art.tape.at(0);
  LaunchReport rep;
  const auto& od = B.dims[0];
  const int64_t cnt = numel(od);
  float* dst = outs.at(0).ptr;
  switch (ti.kind) {
    case DhloOpKind::kTranspose: {
      const DevTensor& x = B.ext.at(ti.args[0].index);
      rep.schedule = "transpose";
      if (cnt) {
        run_copy(x.ptr, transpose_map(x.dims, ti.dims), dst, cnt, stream);
        rep.device_kernels = 1;
      }
      return rep;
    }
    case DhloOpKind::kDynamicReshape: {
      const DevTensor& x = B.ext.at(ti.args[0].index);
      rep.schedule = "reshape";
      if (cnt) {
        cuda_ok(disc_cuda_memcpy(dst, x.ptr, static_cast<size_t>(cnt * 4), 2, stream), "reshape copy");
        rep.device_kernels = 1;
      }
      return rep;
    }
    case DhloOpKind::kDynamicPad: {
      const DevTensor& x = B.ext.at(ti.args[0].index);
      disc_pad_launch P;
      std::memset(&P, 0, sizeof P);
      P.in = x.ptr;
      P.out = dst;
      P.rank = static_cast<int32_t>(x.dims.size());
      if (P.rank > DISC_MAX_RANK) throw InternalError("pad rank exceeds DISC_MAX_RANK");
      P.value = ti.pad_value;
      P.total = cnt;
      auto lo = resolve_all(ti.pad_low, B.regs), it = resolve_all(ti.pad_interior, B.regs);
      for (int d = 0; d < P.rank; ++d) {
        P.out_dims[d] = od[d];
        P.in_dims[d] = x.dims[d];
        P.low[d] = lo[d];
        P.step[d] = 1 + it[d];
      }
      rep.schedule = "pad";
      if (cnt) {
        cuda_ok(disc_cuda_launch_pad(&P, stream), "pad");
        rep.device_kernels = 1;
      }
      return rep;
    }
    case DhloOpKind::kConcat: {
      const int ax = static_cast<int>(ti.axis);
      int64_t outer = 1, inner = 1;
      for (int d = 0; d < ax; ++d) outer *= od[d];
      for (size_t d = ax + 1; d < od.size(); ++d) inner *= od[d];
      rep.schedule = "concat";
      int64_t offset = 0;
      for (size_t p0 = 0; p0 < ti.args.size(); p0 += DISC_MAX_CONCAT) {
        disc_concat_launch C;
        std::memset(&C, 0, sizeof C);
        C.out = dst;
        C.outer = outer;
        C.inner = inner;
        C.axis_total = od[ax];
        C.axis_offset = offset;
        for (size_t p = p0; p < ti.args.size() && p < p0 + DISC_MAX_CONCAT; ++p) {
          const DevTensor x = ti.args[p].kind == TapeRef::Kind::kExternal ? B.ext.at(ti.args[p].index) : DevTensor{};
          C.parts[C.n_parts] = x.ptr;
          C.part_axis[C.n_parts] = x.dims[ax];
          offset += x.dims[ax];
          C.n_parts++;
        }
        if (cnt) {
          cuda_ok(disc_cuda_launch_concat(&C, stream), "concat");
          rep.device_kernels++;
        }
      }
      return rep;
    }
    default:
      throw InternalError("unexpected standalone kernel kind");
  }
}

}  // namespace

namespace {

class DirectIssuer final : public Issuer {
 public:
  DirectIssuer(Scratch& s, void* stream) : scratch_(s), stream_(stream) {}
  void* scratch(int64_t bytes) override { return scratch_.alloc(bytes); }
  void loop(const disc_loop_launch& L) override { cuda_ok(disc_cuda_launch_loop(&L, stream_), "fused loop"); }
  void reduce(const disc_reduce_launch& R) override { cuda_ok(disc_cuda_launch_reduce(&R, stream_), "fused reduce"); }

 private:
  Scratch& scratch_;
  void* stream_;
};

// Tagged pointers: [63:60] kind (1 external, 2 output, 3 scratch), [59:32] index,
// [3:0] the real pointer's low bits (alignment decisions see the same value).
constexpr uint64_t kTagExt = 1, kTagOut = 2, kTagScratch = 3;
inline const void* tag(uint64_t kind, uint64_t index, uintptr_t low) {
  return reinterpret_cast<const void*>((kind << 60) | (index << 32) | (low & 15));
}

struct Recipe {
  std::vector<int64_t> scratch_bytes;
  std::vector<std::pair<int, std::unique_ptr<disc_loop_launch>>> loops;     // (order, launch)
  std::vector<std::pair<int, std::unique_ptr<disc_reduce_launch>>> reduces;
  int steps = 0;
  LaunchReport rep;
};

class RecordingIssuer final : public Issuer {
 public:
  explicit RecordingIssuer(Recipe& r) : r_(r) {}
  void* scratch(int64_t bytes) override {
    r_.scratch_bytes.push_back(bytes);
    return const_cast<void*>(tag(kTagScratch, r_.scratch_bytes.size() - 1, 0));
  }
  void loop(const disc_loop_launch& L) override {
    r_.loops.emplace_back(r_.steps++, std::make_unique<disc_loop_launch>(L));
  }
  void reduce(const disc_reduce_launch& R) override {
    r_.reduces.emplace_back(r_.steps++, std::make_unique<disc_reduce_launch>(R));
  }

 private:
  Recipe& r_;
};

struct Patch {
  const std::vector<DevTensor>& ext;
  const std::vector<OutBuf>& outs;
  const std::vector<void*>& scratch;
  template <typename T>
  void operator()(T*& p) const {
    const uint64_t v = reinterpret_cast<uint64_t>(p);
    const uint64_t kind = v >> 60, idx = (v >> 32) & 0x0fffffff;
    if (kind == kTagExt) p = const_cast<T*>(reinterpret_cast<const T*>(ext.at(idx).ptr));
    else if (kind == kTagOut) p = reinterpret_cast<T*>(outs.at(idx).ptr);
    else if (kind == kTagScratch) p = reinterpret_cast<T*>(scratch.at(idx));
    else if (v && reinterpret_cast<const float*>(p) != kArgCachePtr && reinterpret_cast<const float*>(p) != neg_inf_ptr())
      throw InternalError("untagged pointer in a launch recipe");  // (device constants stay as they are)
  }
  void program(disc_program& P) const {
    for (int l = 0; l < P.n_loads; ++l) (*this)(P.loads[l].ptr);
    for (int o = 0; o < P.n_outs; ++o) (*this)(P.outs[o]);
  }
};

void replay(const Recipe& r, const std::vector<DevTensor>& ext, const std::vector<OutBuf>& outs, Scratch& scratch,
            void* stream) {
  std::vector<void*> sp;
  sp.reserve(r.scratch_bytes.size());
  for (int64_t b : r.scratch_bytes) sp.push_back(scratch.alloc(b));
  const Patch patch{ext, outs, sp};
  size_t li = 0, ri = 0;
  for (int step = 0; step < r.steps; ++step) {
    if (li < r.loops.size() && r.loops[li].first == step) {
      disc_loop_launch L;  // only the used byte ranges are copied (desc_ranges.hpp)
      disc_desc::copy_used(&L, *r.loops[li++].second);
      patch.program(L.prog);
      cuda_ok(disc_cuda_launch_loop(&L, stream), "fused loop");
    } else {
      disc_reduce_launch R;
      disc_desc::copy_used(&R, *r.reduces[ri++].second);
      patch.program(R.pre);
      patch.program(R.post);
      patch(R.red_out);
      patch(R.workspace);
      cuda_ok(disc_cuda_launch_reduce(&R, stream), "fused reduce");
    }
  }
}

uint64_t hmix(uint64_t h, uint64_t v) { return (h ^ v) * 0x100000001b3ull + (h >> 29); }

}  // namespace

// Shape-keyed cache of fused launch recipes (one per executor).
struct LaunchCache {
  struct Entry {
    std::vector<int64_t> key;  // full key, compared on hit
    std::shared_ptr<Recipe> recipe;  // null: the tape needs materialisation
  };
  std::unordered_map<uint64_t, std::vector<Entry>> map;
  size_t entries = 0;
  // Keys seen once (hash only): a recipe is recorded on a key's SECOND launch, so a stream
  // of fresh shapes lowers each launch once, directly, instead of recording a recipe that
  // is never replayed.  Both tables are bounded (cleared when full: a new generation).
  std::unordered_set<uint64_t> seen_once;
  static constexpr size_t kMaxEntries = 16384, kMaxSeen = 1 << 16;
};

namespace {
// True on the first sighting of key hash h (a hash collision only costs one recording).
bool it_seen_first(LaunchCache* c, uint64_t h) {
  if (c->seen_once.size() >= LaunchCache::kMaxSeen) c->seen_once.clear();
  return c->seen_once.insert(h).second;
}
}  // namespace

LaunchCache* new_launch_cache() { return new LaunchCache(); }
void free_launch_cache(LaunchCache* c) { delete c; }

LaunchReport launch_kernel_impl(const KernelArtifact& art, const VersionArtifact& ver, const std::vector<DevTensor>& ext,
                                const std::vector<int64_t>& regs, const std::vector<OutBuf>& outs, Scratch& scratch,
                                void* stream, SchedulePref pref, LaunchCache* cache, uint64_t plan_serial);

LaunchReport launch_kernel(const KernelArtifact& art, const VersionArtifact& ver, const std::vector<DevTensor>& ext,
                           const std::vector<int64_t>& regs, const std::vector<OutBuf>& outs, Scratch& scratch,
                           void* stream, SchedulePref pref, LaunchCache* cache, uint64_t plan_serial) {
  if (!flow_prof_on()) return launch_kernel_impl(art, ver, ext, regs, outs, scratch, stream, pref, cache, plan_serial);
  const int64_t t0 = now_ns();
  LaunchReport r = launch_kernel_impl(art, ver, ext, regs, outs, scratch, stream, pref, cache, plan_serial);
  g_flow_prof.ns_total += now_ns() - t0;
  g_flow_prof.calls++;
  return r;
}

LaunchReport launch_kernel_impl(const KernelArtifact& art, const VersionArtifact& ver, const std::vector<DevTensor>& ext,
                                const std::vector<int64_t>& regs, const std::vector<OutBuf>& outs, Scratch& scratch,
                                void* stream, SchedulePref pref, LaunchCache* cache, uint64_t plan_serial) {
  const bool prof = flow_prof_on();
  int64_t tp = prof ? now_ns() : 0;
  // Recipe cache: everything the lowering depends on is in the key.
  std::vector<int64_t> key;
  uint64_t h = 0;
  const bool cacheable = cache && plan_serial && !art.standalone && pref != SchedulePref::kMaterialize;
  if (cacheable) {
    key.reserve(8 + regs.size() + 4 * ext.size());
    key.push_back(static_cast<int64_t>(plan_serial));
    key.push_back(art.kernel_id);
    key.push_back(ver.id);
    key.push_back(static_cast<int64_t>(pref));
    key.insert(key.end(), regs.begin(), regs.end());
    for (size_t i = 0; i < ext.size(); ++i) {
      key.push_back(static_cast<int64_t>(ext[i].dims.size()));
      key.insert(key.end(), ext[i].dims.begin(), ext[i].dims.end());
      int64_t same = -1;  // aliasing pattern among externals
      for (size_t j = 0; j < i; ++j)
        if (ext[j].ptr == ext[i].ptr) same = static_cast<int64_t>(j);
      key.push_back((reinterpret_cast<uintptr_t>(ext[i].ptr) & 15) | (same << 8));
    }
    for (const auto& o : outs) key.push_back((reinterpret_cast<uintptr_t>(o.ptr) & 15) | (o.capacity_bytes << 4));
    for (int64_t v : key) h = hmix(h, static_cast<uint64_t>(v));
    auto it = cache->map.find(h);
    if (it != cache->map.end())
      for (const auto& e : it->second)
        if (e.key == key) {
          if (!e.recipe) break;  // known to need the materialised path
          replay(*e.recipe, ext, outs, scratch, stream);
          if (prof) g_flow_prof.hits++;
          return e.recipe->rep;
        }
  }
  if (prof) {
    const int64_t t = now_ns();
    g_flow_prof.ns_key += t - tp;
    tp = t;
  }
  bool record = cacheable;
  if (record && it_seen_first(cache, h)) record = false;  // first sighting: lower directly

  std::vector<std::vector<int64_t>> ext_dims;
  for (const auto& e : ext) ext_dims.push_back(e.dims);
  Binding B{art, ver, ext, regs, simulate_tape(art, ver, ext_dims, regs), -1, {}};
  for (size_t o = 0; o < art.output_tape_indices.size(); ++o)
    check_capacity(B.dims.at(art.output_tape_indices[o]), outs.at(o));
  if (prof) {
    const int64_t t = now_ns();
    g_flow_prof.ns_sim += t - tp;
    tp = t;
  }
  struct LowerTimer {
    bool on;
    int64_t t0;
    ~LowerTimer() {
      if (on) g_flow_prof.ns_lower += now_ns() - t0;
    }
  } lower_timer{prof, tp};

  LaunchReport rep;
  if (art.standalone) {
    rep = launch_standalone(B, outs, stream);
  } else {
    const int n = static_cast<int>(art.tape.size());
    for (int t = 0; t < n; ++t)
      if (is_reduce(art.tape[t].kind)) B.red = t;
    B.post.assign(n, 0);
    if (B.red >= 0)
      for (int t = B.red + 1; t < n; ++t)
        for (const auto& a : art.tape[t].args)
          if (a.kind == TapeRef::Kind::kMember && (a.index == B.red || B.post[a.index])) B.post[t] = 1;
    bool done = false;
    if (pref != SchedulePref::kMaterialize) {
      try {
        if (record) {
          // Record with tagged pointers, cache, then replay with the real ones.
          std::vector<DevTensor> text(ext.size());
          for (size_t i = 0; i < ext.size(); ++i) {
            size_t first = i;
            for (size_t j = 0; j < i; ++j)
              if (ext[j].ptr == ext[i].ptr) {
                first = j;
                break;
              }
            text[i] = {static_cast<const float*>(tag(kTagExt, first, reinterpret_cast<uintptr_t>(ext[i].ptr))), ext[i].dims};
          }
          std::vector<OutBuf> touts(outs.size());
          for (size_t o = 0; o < outs.size(); ++o)
            touts[o] = {static_cast<float*>(const_cast<void*>(tag(kTagOut, o, reinterpret_cast<uintptr_t>(outs[o].ptr)))),
                        outs[o].capacity_bytes};
          Binding TB{art, ver, text, regs, B.dims, B.red, B.post};
          auto recipe = std::make_shared<Recipe>();
          RecordingIssuer rec(*recipe);
          recipe->rep = launch_fused(TB, touts, rec, pref);
          recipe->rep.algorithmic_bytes = algorithmic_bytes(art, ext, B.dims);
          if (cache->entries >= LaunchCache::kMaxEntries) {
            cache->map.clear();
            cache->entries = 0;
          }
          cache->map[h].push_back({key, recipe});
          cache->entries++;
          replay(*recipe, ext, outs, scratch, stream);
          return recipe->rep;
        }
        DirectIssuer direct(scratch, stream);
        rep = launch_fused(B, outs, direct, pref);
        done = true;
      } catch (const NotFusible& nf) {
        if (pref == SchedulePref::kFusedOnly) throw InternalError(std::string("not fusible: ") + nf.why);
        if (cacheable) {
          if (cache->entries >= LaunchCache::kMaxEntries) {
            cache->map.clear();
            cache->entries = 0;
          }
          cache->map[h].push_back({key, nullptr});
          cache->entries++;
        }
      }
    }
    if (!done) rep = launch_materialized(B, outs, scratch, stream);
  }
  rep.algorithmic_bytes = algorithmic_bytes(art, ext, B.dims);
  return rep;
}

void launch_gemm(int64_t m, int64_t k, int64_t n, const DevTensor& a, const DevTensor& b, const OutBuf& c,
                 Scratch& scratch, void* stream) {
  if (a.dims.size() != 2 || b.dims.size() != 2) throw RuntimeError("matmul operands must be rank-2");
  if (a.dims[1] != b.dims[0]) throw RuntimeError("matmul inner dim mismatch at runtime");
  if (m * n * 4 > c.capacity_bytes) throw InternalError("kernel output exceeds planned buffer size");
  if (m == 0 || n == 0) return;
  if (k == 0) {
    cuda_ok(disc_cuda_memset(c.ptr, 0, static_cast<size_t>(m * n * 4), stream), "gemm zero");
    return;
  }
  // f64 widening workspace from the executor's scratch (arena memory, no per-call allocation)
  double* ws = static_cast<double*>(scratch.alloc(8 * (m * k + k * n + m * n)));
  cuda_ok(disc_cuda_gemm_ws(m, k, n, a.ptr, b.ptr, c.ptr, ws, stream), "gemm");
}

}  // namespace disc::rt
