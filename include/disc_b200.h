/* disc-b200: B200-native backend for the DISC dynamic-shape compiler's fused-kernel path.
 *
 * C ABI (extern "C", plain pointers and sizes, no C++ or torch types).  The reference
 * artifact (/root/reference/proj) has no FFI -- its boundary is the C++ API -- so each
 * entry point below cites the reference C++ call it stands in for.  Status codes follow
 * the reference CLI exit codes (tools/disc_main.cpp:353-366): 0 ok, 2 usage,
 * 3 parse/validation/compile error, 4 runtime/internal error.  On failure
 * disc_last_error() holds "error[<class>]: <message>" with the reference's message text.
 */
#ifndef DISC_B200_H_
#define DISC_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct disc_compiler_s* disc_compiler;
typedef struct disc_plan_s* disc_plan;          /* immutable, shareable across threads */
typedef struct disc_executor_s* disc_executor;  /* one per (host thread, device, stream) */

/* ---- errors / memory --------------------------------------------------- */
const char* disc_last_error(void);       /* thread-local; error.hpp:25-63 classes */
int disc_last_error_class(void);         /* ErrorClass enum value, -1 if none */
void disc_free(void* p);                 /* frees strings returned through char** */
const char* disc_version(void);

/* ---- compile side (host) ----------------------------------------------- */
/* parse_graph + compile_graph (framework.cpp:350, codegen.cpp:688) */
int disc_compile_graph(const char* graph_json, int inject_constraints, int enable_fusion,
                       int static_fallback, disc_plan* out);
/* static_specialize (codegen.cpp:698) */
int disc_static_specialize(const char* graph_json, disc_plan* out);
/* Compiler: shape-agnostic plan cache with coalescing (codegen.cpp:762-802) */
int disc_compiler_create(int inject_constraints, int enable_fusion, int static_fallback,
                         disc_compiler* out);
void disc_compiler_destroy(disc_compiler c);
int disc_compiler_compile(disc_compiler c, const char* graph_json, disc_plan* out);
void disc_compiler_stats(disc_compiler c, int64_t* compile_count, int64_t* cache_hits);
/* cache_key (codegen.cpp:703), dump-ir stages (codegen.cpp:624-684), lower_to_dhlo+to_json */
int disc_cache_key(const char* graph_json, int inject_constraints, int enable_fusion,
                   int static_fallback, char** out);
int disc_dump_stage(const char* graph_json, int inject_constraints, int enable_fusion,
                    const char* stage, char** out);
int disc_lower_dhlo_json(const char* graph_json, char** out);
int disc_dhlo_roundtrip(const char* dhlo_json, char** out); /* dhlo_from_json -> to_json */

/* ---- plans ------------------------------------------------------------- */
/* plan_from_json / plan_to_json / check_plan (runtime_program.cpp:182-575) */
int disc_plan_from_json(const char* plan_json, disc_plan* out);
int disc_plan_to_json(disc_plan p, char** out);
int disc_plan_check(disc_plan p, char** diagnostics_json);
void disc_plan_retain(disc_plan p);
/* Identity of the underlying CompiledPlan: equal for handles the Compiler's cache shared
 * (codegen.hpp:65-83 returns one shared_ptr per signature). */
const void* disc_plan_identity(disc_plan p);
void disc_plan_release(disc_plan p);
int disc_plan_num_inputs(disc_plan p);
const char* disc_plan_input_name(disc_plan p, int i);
int disc_plan_input_rank(disc_plan p, int i);
int disc_plan_num_outputs(disc_plan p);
const char* disc_plan_output_name(disc_plan p, int i);
int disc_plan_num_kernels(disc_plan p);
int64_t disc_plan_eager_op_count(disc_plan p);
int64_t disc_plan_host_instruction_count(disc_plan p);
/* PlanInput.declared[d] (runtime_program.hpp:28-160): the graph's declared dim, a
 * symbol name or a decimal constant (drives the CLI's synthetic inputs, disc_main.cpp:113-136). */
const char* disc_plan_input_declared(disc_plan p, int i, int d);
const char* disc_plan_signature(disc_plan p);  /* CompiledPlan.signature_digest */
/* Evaluate the host shape program for concrete input dims (EvalShape, executor.cpp:303-341):
 * writes the register file (up to cap entries) and each output's dims. */
int disc_plan_eval_shapes(disc_plan p, int n_inputs, const int64_t* const* dims, const int* ranks,
                          int64_t* regs, int regs_cap, int* n_regs);

/* ---- runtime flow on the device ---------------------------------------- */
/* Executor (executor.hpp:74-83): owns a stream-ordered device caching allocator that
 * persists across runs.  `cuda_stream` may be NULL (legacy default stream). */
int disc_executor_create(int device, void* cuda_stream, disc_executor* out);
void disc_executor_destroy(disc_executor e);
int disc_executor_set_stream(disc_executor e, void* cuda_stream);
/* Executor::run (executor.cpp:221-465).  Inputs are f32, row-major, bound by name; data
 * pointers are device pointers, or host pointers when inputs_on_host != 0 (copied H2D
 * inside the call).  Launches are asynchronous on the executor's stream; outputs stay
 * valid (device-resident) until the next run on this executor. */
int disc_executor_run(disc_executor e, disc_plan p, int n_inputs, const char* const* names,
                      const void* const* data, const int64_t* const* dims, const int* ranks,
                      int inputs_on_host);
/* Runs n_requests requests of one plan back to back (asynchronously); request r binds
 * data/dims/ranks[r*n_inputs + i] to names[i].  Launch records accumulate over the
 * batch; outputs/stats/events are those of the last request. */
int disc_executor_run_batch(disc_executor e, disc_plan p, int n_requests, int n_inputs,
                            const char* const* names, const void* const* data,
                            const int64_t* const* dims, const int* ranks, int inputs_on_host);
/* Runs a heterogeneous stream of requests back to back (asynchronously): request r runs
 * plans[r] on inputs input_offsets[r] .. input_offsets[r+1]-1 of the flat arrays. */
int disc_executor_run_stream(disc_executor e, int n_requests, const disc_plan* plans, const int* input_offsets,
                             const char* const* names, const void* const* data, const int64_t* const* dims,
                             const int* ranks, int inputs_on_host);
/* Grouped execution of independent requests (same arguments as run_stream).  Every
 * request's runtime flow -- shape program, buffer plan, version guards, schedule
 * selection, the reference's runtime checks -- runs on the host exactly as in
 * disc_executor_run, but its device work is queued; the queue is then issued level by
 * level with the same fused kernel of ALL requests merged into one grouped launch per
 * kernel instantiation (disc_cuda_queue_*).  Outputs are bit-identical to running the
 * requests one by one; no buffer is reused across requests inside the call.  Request r's
 * outputs: disc_executor_request_output / _copy_request_output, valid until the next run.
 * Launch records (timing mode) are one per grouped launch.  Replaces a loop of
 * Executor::run calls (executor.cpp:221-465) for a batch of requests. */
int disc_executor_run_grouped(disc_executor e, int n_requests, const disc_plan* plans, const int* input_offsets,
                              const char* const* names, const void* const* data, const int64_t* const* dims,
                              const int* ranks, int inputs_on_host);
/* Host threads for disc_executor_run_grouped (default 1): calls with >= 64 requests per
 * thread run contiguous request ranges' runtime flows on worker threads (own sub-executor
 * each: allocator, scratch, recipe cache) and merge their queues into one grouped flush. */
int disc_executor_set_host_threads(disc_executor e, int n);
/* Static plans (no shape program, e.g. disc_static_specialize) run as CUDA graphs: a run
 * whose device work (launch parameters and pointers included) hashes like the previous
 * run's is captured, later identical runs replay it.  Default on. */
int disc_executor_set_graphs(disc_executor e, int on);
int64_t disc_executor_graph_replays(disc_executor e);
int disc_executor_num_requests(disc_executor e);
int disc_executor_num_request_outputs(disc_executor e, int request);  /* -1: no such request */
int disc_executor_request_output(disc_executor e, int request, int i, const float** dptr, const int64_t** dims,
                                 int* rank);
int disc_executor_copy_request_output(disc_executor e, int request, int i, void* dst, int dst_on_host);
int disc_executor_request_stats(disc_executor e, int request, int64_t* stats7);
/* Interleaves a request stream over several executors (each with its own stream and
 * allocator, typically on one device): request r runs on exs[which[r]].  Independent
 * requests on different streams overlap on the device (small and mid-size requests are
 * latency-bound per kernel).  Launch records accumulate per executor over the call. */
int disc_executors_run_interleaved(const disc_executor* exs, int n_exec, int n_requests, const int* which,
                                   const disc_plan* plans, const int* input_offsets, const char* const* names,
                                   const void* const* data, const int64_t* const* dims, const int* ranks,
                                   int inputs_on_host);
int disc_executor_num_outputs(disc_executor e);
/* Device pointer + dims of output i of the last run. */
int disc_executor_output(disc_executor e, int i, const float** dptr, const int64_t** dims,
                         int* rank);
/* Copies output i (stream-ordered) to dst: dst_on_host 0 device, 1 host (synchronizes the
 * stream), 2 pinned host, asynchronous (valid after disc_executor_synchronize; lets
 * requests on several executors overlap H2D, compute and D2H). */
int disc_executor_copy_output(disc_executor e, int i, void* dst, int dst_on_host);
int disc_executor_synchronize(disc_executor e);
/* ExecStats (executor.hpp:30-40): launch_count, library_calls, host_instruction_count,
 * peak_bytes, alloc_calls, allocator_cache_hits, aliased_allocs; ms2 = host_ms, kernel_ms.
 * kernel_ms is device time (CUDA events) when timing is enabled, else 0. */
int disc_executor_stats(disc_executor e, int64_t* s7, double* ms2);
/* BufferEvent list (executor.hpp:44-49): 4 ints per event (logical, physical, alloc_instr,
 * dealloc_instr). */
int disc_executor_num_events(disc_executor e);
int disc_executor_event(disc_executor e, int i, int* four);
/* Device kernels launched by the last run (CUDA launches, not plan kLaunch count). */
int64_t disc_executor_device_launches(disc_executor e);
/* Per-launch records of the last run: plan instruction, artifact id (-1 = library call),
 * schedule name, algorithmic boundary bytes, device ms (timing mode). */
int disc_executor_num_records(disc_executor e);
int disc_executor_record(disc_executor e, int i, int* instr, int* kernel, int64_t* bytes, double* ms,
                         int* device_kernels, const char** schedule);
/* Sum of algorithmic boundary bytes over the last run's launches. */
int64_t disc_executor_algorithmic_bytes(disc_executor e);
/* 1: time every kLaunch/kLibraryCall with CUDA events (asynchronous; read back when
 * stats/records are queried). */
int disc_executor_set_timing(disc_executor e, int enabled);
/* Schedule override for testing: "auto" (default), "materialize" (per-member tape),
 * "fused" (forbid the per-member fallback), "twopass"/"atomic" column reductions. */
int disc_executor_set_schedule(disc_executor e, const char* schedule);
/* Allocator byte budget for cached free blocks (0 = unlimited). */
int disc_executor_set_cache_budget(disc_executor e, int64_t bytes);
/* Reserves `bytes` of device memory for the executor's buffer arena now (kept for the
 * executor's lifetime), so a stream of fresh shapes never grows it mid-stream. */
int disc_executor_reserve(disc_executor e, int64_t bytes);
/* Asynchronous grouped flush (device inputs, non-timing): disc_executor_run_grouped returns
 * once the requests' host flows are queued; their grouped launches are issued by a
 * background thread in call order, so the next call's flows overlap this call's issue.
 * Outputs (pointers, stats) are known on return; copies, synchronize and other stream work
 * of the executor wait first.  Call disc_executor_wait_issued before recording your own
 * events or launching your own work on the executor's stream. */
int disc_executor_set_async_flush(disc_executor e, int on);
int disc_executor_wait_issued(disc_executor e);

/* ---- single-kernel entry (run_kernel, executor.cpp:137-219) ------------- */
/* Runs artifact `kernel` at version `version` on device externals with the given
 * register file; outputs are device buffers owned by the executor until the next call. */
int disc_executor_run_kernel(disc_executor e, disc_plan p, int kernel, int version, int n_ext,
                             const float* const* ext, const int64_t* const* ext_dims,
                             const int* ext_ranks, const int64_t* regs, int n_regs);
/* Host-only dry run of the runtime flow for the given input shapes: returns the lowered
 * device programs of every fused launch as JSON (used by tools/gen_patterns.py). */
int disc_plan_capture_programs(disc_plan p, int n_inputs, const char* const* names,
                               const int64_t* const* dims, const int* ranks, char** json);
/* Grouping dry run (host only, no device): runs disc_executor_run_grouped's host flow for
 * the requests (device-resident inputs of the given dims) in capture mode and returns the
 * flush plan as JSON: one entry per issued action {level, action: group|copies|single|alone,
 * members, bytes, kernel, schedule[, table_bytes, generated, order]}.  Free with disc_free. */
int disc_plan_group_dry_run(int n_requests, const disc_plan* plans, const int* input_offsets, const char* const* names,
                            const int64_t* const* dims, const int* ranks, int host_threads, char** json);
/* Host-side cost of one run (capture mode: no device work), microseconds per run. */
int disc_plan_host_overhead(disc_plan p, int n_inputs, const char* const* names,
                            const int64_t* const* dims, const int* ranks, int iters, double* us_per_run);
/* Algorithmic boundary bytes (external inputs read + outputs written, per
 * kLaunch) of one run at the given input shapes -- host only, no device work.  The
 * multi-GPU dispatcher balances requests by this. */
int disc_plan_algorithmic_bytes(disc_plan p, int n_inputs, const char* const* names,
                                const int64_t* const* dims, const int* ranks, int64_t* bytes);
/* guard_passes (executor.cpp:78-98) */
int disc_guard_passes(disc_plan p, int kernel, int version, const int64_t* regs, int n_regs);

/* ---- multi-GPU request dispatcher -------------------------- */
/* One worker thread per entry of `devices` (a device may repeat), each with its own
 * executor, stream and host-flow threads (host_threads <= 0: its CPU slice), pinned to a
 * contiguous slice of the process's CPUs.  A batch is split by greedy LPT on algorithmic
 * bytes (the rule of dispatch.shard) and each worker runs its share as one grouped call;
 * no collective touches the data path.  Replaces one Executor::run per request
 * (executor.cpp:221-465) spread over threads by the caller. */
typedef struct disc_dispatcher_s* disc_dispatcher;
int disc_dispatcher_create(int n_workers, const int* devices, int host_threads, disc_dispatcher* out);
void disc_dispatcher_destroy(disc_dispatcher d);
int disc_dispatcher_num_workers(disc_dispatcher d);
int disc_dispatcher_worker_device(disc_dispatcher d, int worker);
/* Host-only LPT assignment: worker_of[r] for each request (place device inputs with it). */
int disc_dispatcher_assign(disc_dispatcher d, int n_requests, const disc_plan* plans, const int* input_offsets,
                           const char* const* names, const int64_t* const* dims, const int* ranks, int* worker_of);
/* Runs the batch (worker_of = NULL: LPT) and returns when every worker is done.  Inputs are
 * host pointers (inputs_on_host = 1) or device pointers on the assigned worker's device. */
int disc_dispatcher_run_grouped(disc_dispatcher d, int n_requests, const disc_plan* plans, const int* input_offsets,
                                const char* const* names, const void* const* data, const int64_t* const* dims,
                                const int* ranks, int inputs_on_host, const int* worker_of);
int disc_dispatcher_request_worker(disc_dispatcher d, int request);
int disc_dispatcher_num_request_outputs(disc_dispatcher d, int request);
int disc_dispatcher_request_output(disc_dispatcher d, int request, int i, const float** dptr, const int64_t** dims,
                                   int* rank, int* device);
int disc_dispatcher_copy_request_output(disc_dispatcher d, int request, int i, void* dst, int dst_on_host);
/* Last batch, worker w: requests run, algorithmic bytes, wall ms of its grouped call. */
int disc_dispatcher_worker_stats(disc_dispatcher d, int worker, int64_t* requests, int64_t* bytes, double* ms);

#ifdef __cplusplus
}
#endif

#endif /* DISC_B200_H_ */
