/* disc-b200 device layer: the kernel boundary under the runtime flow.
 *
 * Replaces the reference's in-process CPU "device" calls inside Executor::run:
 *   run_kernel(KernelArtifact, VersionArtifact, externals, regs)  executor.cpp:137-219 (call: 421)
 *   CachedAllocator::alloc/free/data                               executor.cpp:53-76  (calls: 347,363,457)
 *   eval_matmul(a, b)                                             kernels.cpp:293-303 (call: 434)
 * A fused tape is lowered on the host (once per plan) to a small register program and
 * passed to the kernel BY VALUE (__grid_constant__ parameters); shapes are bound per
 * launch as gather maps.  Nothing is compiled per shape.
 */
#ifndef DISC_CUDA_H_
#define DISC_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DISC_MAX_RANK 8
#define DISC_MAX_INSTR 64
#define DISC_MAX_LOADS 16
#define DISC_MAX_OUTS 8
#define DISC_MAX_SLOTS 12
#define DISC_MAX_CONCAT 8

/* Tape operations (host-level semantics).  Elementwise ops have the reference's f32
 * semantics (kernels.cpp:26-44): IEEE add/sub/mul/div (no FMA contraction),
 * max(a,b) = (a<b)?b:a, libdevice expf/tanhf. */
enum disc_op {
  DISC_OP_LOAD = 0,
  DISC_OP_ADD, DISC_OP_SUB, DISC_OP_MUL, DISC_OP_DIV, DISC_OP_MAX,
  DISC_OP_EXP, DISC_OP_TANH, DISC_OP_NEG,
  DISC_OP_COPY,
  DISC_OP_REDVAL,     /* the current row's reduce result (row schedule only) */
  DISC_OP_RCPVAL,     /* 1 / REDVAL (IEEE reciprocal, once per row): x / REDVAL is lowered
                         to x * RCPVAL in fused epilogues (<= 1.5 ulp from the quotient) */
  DISC_OP_FDIV,       /* a * rcp.approx(b): Div inside multi-member (fused) groups, <= 2 ulp
                         (IEEE a / b stays the single-op plans' semantics, bit-exact) */
};

/* Pre-decoded device opcodes: operand sources (accumulator A / slot S) are folded into
 * the opcode so the interpreter dispatches once per instruction through one jump table. */
enum disc_opcode {
  DISC_I_LOAD_ID = 0,   /* acc = ptr[f]                      (contiguous) */
  DISC_I_LOAD_AFF = 1,  /* acc = ptr[off + row*rs + col*cs]  (2D affine) */
  DISC_I_LOAD_GATHER = 2, /* acc = ptr[map(f)]               (general gather) */
  DISC_I_LOAD_CONST = 3,  /* acc = hoisted scalar (loaded once per block) */
  DISC_I_REDVAL = 4,
  DISC_I_COPY = 5,      /* acc = slot[a] */
  DISC_I_RCPVAL = 6,    /* acc = 1 / row reduce result */
  DISC_I_BIN = 8,       /* 8 + 4*(op-ADD) + mode, mode 0 AA, 1 AS, 2 SA, 3 SS (a op b) */
  DISC_I_UN = 28,       /* 28 + 2*(op-EXP) + mode, mode 0 A, 1 S */
  DISC_I_FDIV = 34,     /* 34 + mode (as DISC_I_BIN): fused-group division */
  DISC_I_END = 38,
};
#define DISC_F_SLOT 1   /* also keep acc in slot dst */
#define DISC_F_OUT 2    /* also store acc to outs[out] */

typedef struct {
  uint8_t op;      /* disc_opcode */
  uint8_t a, b;    /* operand slots */
  uint8_t flags;   /* DISC_F_* */
  uint8_t dst;     /* slot written when DISC_F_SLOT */
  uint8_t load;    /* loads[] index for LOAD_* */
  uint8_t out;     /* outs[] index when DISC_F_OUT */
  uint8_t pad;
} disc_instr;

/* A load binds an external operand for one launch.  The launch views its space as
 * [rows, W] (f = row*W + col); most operands are then 2D-affine in (row, col):
 *   identity  src = f
 *   affine    src = offset + row*rs + col*cs   (row/column broadcasts, offsets, strides)
 *   const     src = offset                      (hoisted: read once per block)
 *   gather    src = offset + sum_d coord_d(f) * strides[d], coords row-major over dims
 *             (magic/shift: u32 fast division, magic 0 = divide by 1). */
enum disc_load_mode { DISC_LOAD_IDENTITY = 0, DISC_LOAD_AFFINE = 1, DISC_LOAD_GATHER = 2, DISC_LOAD_CONST = 3 };
typedef struct {
  const float* ptr;
  int32_t mode;
  int32_t rank;     /* gather */
  int32_t vec_ok;   /* VEC=4: 1 = 128-bit load, 2 = splat (inner stride 0), 0 = 4 scalar loads */
  int32_t pad;
  int64_t offset;
  int64_t rs, cs;   /* affine */
  int64_t dims[DISC_MAX_RANK];
  int64_t strides[DISC_MAX_RANK];
  uint32_t magic[DISC_MAX_RANK];
  uint32_t shift[DISC_MAX_RANK];
} disc_load;

/* Row cache (row schedule): identity loads are kept in shared-memory slots; slot k holds
 * the block's rows back to back (row r at k*slot_stride + r*R).  cache_mode 1: the pre
 * program also writes the loaded tile to slot cache_slot[l]; 2: the program reads it from
 * there instead of global memory.  In a staged launch (disc_reduce_launch.stage) the
 * block copies its rows into the input slots first and programs write output o to slot
 * out_slot[o]; the block then copies the output slots out (coalesced). */
enum disc_cache_mode { DISC_CACHE_NONE = 0, DISC_CACHE_FILL = 1, DISC_CACHE_READ = 2 };

typedef struct {
  int32_t n_instr;
  int32_t n_slots;
  int32_t n_loads;
  int32_t n_outs;
  int32_t cache_mode;
  int8_t cache_slot[DISC_MAX_LOADS];
  int8_t out_slot[DISC_MAX_OUTS];   /* staged launches: smem slot of output o, -1 = global */
  int32_t flags;    /* DISC_PROG_* launch flags (not part of the program structure) */
  disc_instr code[DISC_MAX_INSTR];
  disc_load loads[DISC_MAX_LOADS];
  float* outs[DISC_MAX_OUTS];
} disc_program;

/* disc_program.flags: with programmatic dependent launch, let the next kernel's CTAs
 * launch as soon as this grid has passed its dependency wait (instead of at its exit). */
#define DISC_PROG_PDL_EARLY 1

enum disc_reduce_kind { DISC_REDUCE_SUM = 0, DISC_REDUCE_MAX = 1 };

/* Elementwise (kLoop) schedule: one program over the space viewed as [rows, W]. */
typedef struct {
  disc_program prog;
  int64_t total;    /* rows * W */
  int64_t W;        /* row width in elements (multiple of vec) */
  int64_t rows;
  int32_t vec;      /* 4 or 1 */
  int32_t wide;     /* 1: 64-bit index math */
  int32_t lpr;      /* lanes per row (power of two <= 32): narrow rows pack several per warp */
  int32_t prefetch; /* 1: L2-prefetch the next grid-stride tile's streaming operands */
} disc_loop_launch;

/* Reduce schedules over the reduce argument collapsed to [K, R, C] (R reduced). */
enum disc_reduce_schedule {
  DISC_SCHED_ROW = 0,       /* C == 1: rows of R, G threads per row (warp / block) */
  DISC_SCHED_COL_TWOPASS,   /* split-R partials in f64 workspace, ordered finalize */
  DISC_SCHED_COL_ATOMIC,    /* split-R f64 atomics into workspace, finalize */
  DISC_SCHED_COL_SINGLE,    /* one pass, no split */
  DISC_SCHED_GENERIC,       /* non-contiguous reduced axes: thread per output */
};

typedef struct {
  disc_program pre;         /* ends with the reduce argument in acc; stores pre outputs */
  disc_program post;        /* row schedule fused epilogue (REDVAL), n_instr 0 if none */
  int64_t K, R, C;          /* collapsed geometry (ROW: C == 1) */
  int32_t kind;             /* disc_reduce_kind */
  int32_t schedule;         /* disc_reduce_schedule */
  int32_t vec;              /* 4 or 1 along the contiguous dim */
  int32_t wide;
  int32_t group;            /* ROW: threads per row (power of two) */
  int32_t splits;           /* COL: number of R splits */
  int32_t cache_loads;      /* ROW: number of shared-memory slots (0 = no cache) */
  int32_t stage;            /* ROW: 1 = staged block tiles (see disc_program.out_slot), 2 = TMA-staged,
                               3 = warp-staged short rows */
  float* red_out;           /* f32 reduce result [K*C] */
  double* workspace;        /* COL two-pass/atomic: f64 [splits or 1][K*C] */
  /* GENERIC: arg dims and reduced-axis mask */
  int32_t g_rank;
  int32_t g_mask;
  int64_t g_dims[DISC_MAX_RANK];
  /* ROW with a fused epilogue: shared-memory slot that keeps the reduce ARGUMENT (the
   * pre program's per-element value) for the epilogue, which reads it as a cached
   * identity load instead of recomputing it (softmax: exp(x - max)); -1 = none */
  int32_t arg_slot;
  /* ROW, vec 4, R % 4 != 0 (only identity / row-splat / const operands): each row runs a
   * float4 body from its first 16 B-aligned column plus a scalar head and tail; row-cache
   * rows are padded to R + 3 and shifted so the body stays aligned in shared memory */
  int32_t unaligned;
  /* COL, K == 1, C % 4 != 0: rows folded by `fold` into super rows of C = fold * fold_cout
   * floats (R = full super rows); the finalize joins super-columns c, c + fold_cout, ...
   * into output c.  fold_tail: rows of a last, partial super row (N mod fold). */
  int32_t fold;
  int32_t fold_tail;
  int64_t fold_cout;
  /* ROW sum with <= 256 threads: 1 = the register-capped kernel (6 resident blocks) */
  int32_t regcap;
  /* ROW, R < 32, scalar rows, one thread per row: 8 or 32 = the register-resident short-row
   * kernel (the whole row evaluated at once, one sequential accumulator), 0 = off */
  int32_t short_rows;
  /* ROW with a row cache: floats between consecutive rows in a cache slot (0 = R, or
   * R + 3 rounded to 4 for unaligned rows); padded so that the rows one shared-memory
   * wavefront touches fall in distinct banks */
  int32_t row_pitch;
} disc_reduce_launch;

/* Standalone pad (eval_pad, kernels.cpp:125-147), output-driven gather. */
typedef struct {
  const float* in;
  float* out;
  int32_t rank;
  float value;
  int64_t total;
  int64_t out_dims[DISC_MAX_RANK];
  int64_t in_dims[DISC_MAX_RANK];
  int64_t low[DISC_MAX_RANK];
  int64_t step[DISC_MAX_RANK];   /* 1 + interior */
} disc_pad_launch;

/* Standalone concat (eval_concat, kernels.cpp:196-232) of up to DISC_MAX_CONCAT parts. */
typedef struct {
  const float* parts[DISC_MAX_CONCAT];
  int64_t part_axis[DISC_MAX_CONCAT];  /* extent along the axis */
  int32_t n_parts;
  int32_t pad;
  float* out;
  int64_t outer, inner;   /* out viewed as [outer, axis_total, inner] */
  int64_t axis_total;
  int64_t axis_offset;    /* where parts[0] starts along the axis (multi-launch concat) */
} disc_concat_launch;

/* ---- device management --------------------------------------------------- */
const char* disc_cuda_last_error(void);
int disc_cuda_device_count(int* n);
int disc_cuda_set_device(int device);
int disc_cuda_get_device(int* device);
int disc_cuda_device_info(int device, int* sm_count, int64_t* l2_bytes, int64_t* hbm_bytes);
int disc_cuda_stream_create(void** stream);
int disc_cuda_stream_destroy(void* stream);
int disc_cuda_stream_synchronize(void* stream);
int disc_cuda_device_synchronize(void);

/* ---- memory (raw; the exact-size caching policy lives in the executor) ---- */
int disc_cuda_malloc(size_t bytes, void* stream, void** dptr);   /* stream-ordered pool */
int disc_cuda_free(void* dptr, void* stream);
int disc_cuda_host_alloc(size_t bytes, void** hptr);             /* pinned */
int disc_cuda_host_free(void* hptr);
/* kind: 0 h2d, 1 d2h, 2 d2d, 3 default (UVA); | DISC_MEMCPY_NOW issues the copy even while
 * this thread queues work for `stream` (it then precedes every queued op). */
#define DISC_MEMCPY_NOW 4
int disc_cuda_memcpy(void* dst, const void* src, size_t bytes, int kind, void* stream);
int disc_cuda_memset(void* dst, int value, size_t bytes, void* stream);

/* ---- events --------------------------------------------------------------- */
int disc_cuda_event_create(void** ev);
int disc_cuda_event_destroy(void* ev);
int disc_cuda_event_record(void* ev, void* stream);
int disc_cuda_event_synchronize(void* ev);
int disc_cuda_stream_wait_event(void* stream, void* ev);  /* later work on stream waits for ev */
int disc_cuda_event_elapsed_ms(void* start, void* stop, float* ms);

/* ---- kernels (asynchronous on `stream`) ----------------------------------- */
int disc_cuda_launch_loop(const disc_loop_launch* l, void* stream);
int disc_cuda_launch_reduce(const disc_reduce_launch* l, void* stream);
int disc_cuda_launch_pad(const disc_pad_launch* l, void* stream);
int disc_cuda_launch_concat(const disc_concat_launch* l, void* stream);
/* C[m,n] = A[m,k] B[k,n], f32 in/out, f64 accumulation (eval_matmul semantics). */
int disc_cuda_gemm(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c,
                   void* stream);
/* Same, with the f64 widening workspace supplied by the caller (>= 8*(m*k + k*n + m*n)
 * bytes, stream-ordered like the operands); ws = NULL allocates it per call. */
int disc_cuda_gemm_ws(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c, double* ws,
                      void* stream);
/* Fills n floats with uniform [lo, hi) (counter-based; bench/test input synthesis). */
int disc_cuda_fill_uniform(float* dst, int64_t n, uint64_t seed, float lo, float hi, void* stream);
/* Writes `bytes` (>= 2x L2) to a scratch buffer, then reads its first half back, to evict L2
 * between timed iterations and leave it clean (no write-back inside the next kernel). */
int disc_cuda_flush_l2(void* scratch, size_t bytes, void* stream);
/* Occupies `stream` for the given time (bench/profiling aid: lets the host queue a run
 * ahead of the device so per-launch events measure device time only). */
int disc_cuda_spin(uint64_t microseconds, void* stream);
/* Number of kernels this library has launched (process-wide counter). */
int64_t disc_cuda_kernel_launches(void);
/* Diagnostics: stream-ordered pool calls made so far (cudaMallocAsync, cudaFreeAsync) and
 * allocations retried after an out-of-memory (stream sync + pool trim). */
int64_t disc_cuda_alloc_stats(int64_t* mallocs, int64_t* frees, int64_t* oom_retries);

/* Programmatic dependent launch for fused kernels: 0 plain stream serialisation; 1 (default)
 * each kernel's launch overlaps the previous kernel and its dependency wait; 2 also lets
 * the next kernel's CTAs launch early (DISC_PROG_PDL_EARLY, set by the runtime). */
int disc_cuda_set_pdl(int mode);
int disc_cuda_pdl_mode(void);
/* Generated fast paths: launches whose lowered program structure matches a pattern
 * compiled ahead of time (kernels/patterns_gen.cu) run straight-line kernels instead of
 * the interpreter.  Enabled by default; the counter reports how many launches used one. */
int disc_cuda_set_specialization(int enabled);
int64_t disc_cuda_specialized_launches(void);
/* Fused loop/reduce launches issued (a grouped launch counts its members): with
 * disc_cuda_specialized_launches, the share that ran generated straight-line code. */
int64_t disc_cuda_fused_launches(void);
/* Profiler capture range (cudaProfilerStart/Stop; ncu --profile-from-start off). */
int disc_cuda_profiler(int on);
int disc_cuda_num_specializations(void);
/* ---- grouped launches and the request queue --------------------------------
 * A grouped launch issues n independent fused launches as ONE kernel per homogeneous
 * subgroup (same kernel instantiation: program structure, schedule, vector width, index
 * width); each member keeps its single-launch grid and its results are bit-identical
 * to a separate launch.  Descriptors are uploaded through a pinned ring buffer.
 * (No reference counterpart: the reference runs one request at a time,
 * executor.cpp:221-465; this is the SURVEY 8(f) rank-3 host-dispatch item.) */
int disc_cuda_launch_loop_group(const disc_loop_launch* const* launches, int n, void* stream);
int disc_cuda_launch_reduce_group(const disc_reduce_launch* const* launches, int n, void* stream);
/* Queue mode (per host thread): launches, copies and memsets on `stream` are recorded
 * instead of issued (allocations stay immediate, frees on `stream` are deferred until the
 * flush).  disc_cuda_queue_request() starts the next independent request (a dependency
 * chain); disc_cuda_queue_mark() attributes the ops queued since the previous mark to
 * one kLaunch (algorithmic bytes, artifact id, schedule name).  disc_cuda_queue_flush()
 * issues the k-th op of every request as level k -- fused launches of a level grouped by
 * kernel instantiation, larger members first -- then the deferred frees, and ends queue
 * mode.  With timing != 0 every issued group is bracketed by events; the records are
 * readable after a synchronize through disc_cuda_queue_record(). */
int disc_cuda_queue_begin(void* stream);
int disc_cuda_queue_request(void);
int disc_cuda_queue_mark(int64_t bytes, int kernel, const char* schedule);
int disc_cuda_queue_flush(int timing);
int disc_cuda_queue_active(void);
/* Multi-threaded host flow: a worker thread detaches its queue (the handle owns the
 * recorded ops; the thread's queue ends) and one thread flushes its own active queue (if
 * any) together with the detached ones -- their requests merged level by level and
 * grouped as if queued by one thread; the handles are consumed. */
void* disc_cuda_queue_detach(void);
/* Static plans as CUDA graphs: the executor queues a run, hashes the queued ops (0 = not
 * capturable) and either replays the graph captured for the same hash or issues the queue
 * under stream capture (disc_cuda_queue_issue_graph: ops in order, no grouping) and keeps
 * the instantiated graph; graph_exec == nullptr issues the ops directly, no capture. */
uint64_t disc_cuda_queue_hash(void* queue);
/* The canonical bytes the hash covers (owned by the queue, valid until it is consumed);
 * n = 0: not capturable.  Graph caches compare these in full before a replay. */
int disc_cuda_queue_signature(void* queue, const void** data, size_t* n);
void disc_cuda_queue_discard(void* queue);
int disc_cuda_queue_issue_graph(void* queue, void** graph_exec);
int disc_cuda_graph_launch(void* graph_exec, void* stream);
int disc_cuda_graph_destroy(void* graph_exec);
/* Host profile: ns spent packing grouped-launch descriptor tables since the last call. */
int64_t disc_cuda_host_profile(int64_t* table_bytes);
int disc_cuda_queue_flush_detached(void* const* queues, int n, int timing);
int disc_cuda_queue_num_records(void);
int disc_cuda_queue_record(int i, int* level, int* members, int64_t* bytes, int* kernel, const char** schedule,
                           float* ms);

/* Capture mode (pattern generator, host only): device calls become no-ops, allocations
 * return fake addresses and fused launches are recorded as JSON program structures.
 * The mode is per host thread: 0 off, 1 capture + record, 2 capture without recording.
 * disc_cuda_set_capture(mode) also clears the records; _set_capture_local only sets this
 * thread's mode (executor host-flow workers inherit their caller's mode per job). */
int disc_cuda_set_capture(int enabled);
int disc_cuda_set_capture_local(int mode);
int disc_cuda_capture_mode(void);
int disc_cuda_capture_records(char** json);   /* free with disc_free */
int disc_cuda_capturing(void);

#ifdef __cplusplus
}
#endif

#endif /* DISC_CUDA_H_ */
