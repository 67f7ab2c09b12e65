/*
 * mapfuse_b200.h -- the C-ABI boundary of the B200 fused-sequence engine.
 *
 * This is the drop-in replacement for the reference's execution boundary
 *
 *     LaunchResult vm::launch(const kernel::KernelIR&, const DeviceConfig&,
 *                             const LaunchArgs&)
 *         /root/reference/proj/include/mapfuse/vm.hpp:94  (interpreter:
 *         proj/src/vm.cpp:450-479)
 *
 * and of the compile pipeline that feeds it (the
 * reference's pipeline.cpp is listed in proj/CMakeLists.txt:48 but absent).
 * Plain C: opaque handles, plain pointers and sizes, no C++ or torch types.
 *
 * Error model (mirrors the reference's exceptions):
 *   MF_OK            0
 *   MF_ERR_FAULT     1  vm::VmFault (proj/include/mapfuse/vm.hpp:21): bad or
 *                       missing binding, shape mismatch, CUDA failure
 *   MF_ERR_INVALID   2  ir::ParseError / invalid argument
 *                       (proj/include/mapfuse/ir.hpp:35-43) and library /
 *                       script validation diagnostics
 * The message of the last failure on the calling thread: mf_last_error().
 *
 * Buffers are row-major fp32, padded so both dimensions are multiples of 32
 * (proj/include/mapfuse/blas.hpp:29-30).  Unlike vm::launch, reduction
 * outputs need NOT be pre-zeroed (vm.hpp:91-93): every output is fully
 * overwritten, deterministically.  Intermediates of a multi-kernel plan that
 * the caller does not bind are allocated in the plan's device workspace.
 */
#ifndef MAPFUSE_B200_H
#define MAPFUSE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MF_OK 0
#define MF_ERR_FAULT 1
#define MF_ERR_INVALID 2

/* Planner modes for mf_compile. */
#define MF_MODE_FUSED 0   /* planner-selected fusion partition (reference mode) */
#define MF_MODE_UNFUSED 1 /* one kernel per elementary call (the baseline chain) */
#define MF_MODE_B200 2    /* fused + row-resident chains (ATAX in one pass; beyond the paper) */

typedef struct mf_plan mf_plan;

/* Replaces vm::GlobalBuffer{rows, cols, std::vector<float>*}
 * (proj/include/mapfuse/vm.hpp:25-28).  `data` is a DEVICE pointer for
 * mf_launch / mf_launch_kernel and a HOST pointer for mf_launch_host. */
typedef struct {
  const char* name;
  int rows;
  int cols;
  float* data;
} mf_buffer;

/* Replaces LaunchArgs::scalars (vm.hpp:32). */
typedef struct {
  const char* name;
  float value;
} mf_scalar;

/* Replaces ExecutionStats' traffic counters (vm.hpp:41-56): algorithmic bytes
 * of the launched kernels (each distinct input read once, each output written
 * once -- SURVEY.md 8d), kernel count, and device time when measured. */
typedef struct {
  uint64_t bytes_loaded;
  uint64_t bytes_stored;
  double ms; /* filled by mf_launch_host (synchronous); 0 for async launches */
  int kernels;
} mf_stats;

/* Script text -> parse, dependency graph, fusion planning, combination
 * selection, code generation (KernelIR per kernel) and lowering onto the
 * sm_100a kernel families.  rows/cols are the logical problem size (padded
 * to 32 internally, as blas::make_problem does, proj/src/blas.cpp:109-110).
 * manifest == NULL uses the built-in elementary-function library. */
int mf_compile(const char* script_text, const char* manifest, int rows, int cols, int mode,
               mf_plan** out);

/* Convenience: compile one of the shipped Table-1 sequences by name
 * (blas::build_sequence, proj/include/mapfuse/blas.hpp:27). */
int mf_compile_sequence(const char* sequence, int rows, int cols, int mode, mf_plan** out);

/* Empirical search support: the rank-th best combination
 * (0 = the selector's choice) and the number of combinations. */
int mf_compile_ranked(const char* script_text, const char* manifest, int rows, int cols, int mode,
                      int rank, mf_plan** out);
int64_t mf_count_combinations(const char* script_text, const char* manifest, int rows, int cols);
/* The shipped script text of a Table-1 sequence (blas::build_sequence). */
int mf_sequence_script(const char* name, char* buf, int cap);
/* Cost-model prediction of the plan's time in microseconds. */
double mf_plan_predicted_us(const mf_plan* plan);
/* Plan files: compile once, run many.  save: size convention as
 * mf_plan_describe; load re-lowers every KernelIR in the file. */
int mf_plan_save(const mf_plan* plan, char* buf, int cap);
int mf_plan_load(const char* text, mf_plan** out);

/* One kernel given as KernelIR text (kernel::emit_pseudo_source format,
 * proj/src/kernel.cpp:33-65) -> single-kernel plan.  This is the exact
 * vm::launch(KernelIR, ...) boundary.  rows/cols: the padded domain. */
int mf_plan_create(const char* kernel_ir_text, int rows, int cols, mf_plan** out);

/* The device description of the SURVEY's boundary: the
 * reference's DeviceConfig (proj/include/mapfuse/device.hpp, device.cfg text)
 * plus the B200 facts a plan sizes itself by. */
typedef struct {
  const char* device_config; /* DeviceConfig text (device.cfg format); NULL = the shipped one */
  int sm_count;              /* SMs the plan's persistent kernels (matrix, row-resident) may occupy;
                                0 = all of the device's (capped by option max_sms) */
  int rows, cols;            /* padded domain of the kernel (the VM derives the grid from it) */
} mf_device_desc;

/* mf_plan_create with a device description: the kernel is checked against
 * the DeviceConfig's static limits as vm::launch checks them (threads per
 * block, shared bytes per block: MF_ERR_FAULT, proj/src/vm.cpp:457-460; a
 * malformed config: MF_ERR_INVALID), and every launch of the plan sizes its
 * co-resident grids for at most desc->sm_count SMs (the caller keeps the
 * rest, e.g. for concurrent work). */
int mf_plan_create_desc(const char* kernel_ir_text, const mf_device_desc* desc, mf_plan** out);

void mf_plan_destroy(mf_plan* plan);

int mf_plan_num_kernels(const mf_plan* plan);
/* JSON description of the plan (kernels, fused calls, buffers, roles,
 * algorithmic bytes).  Returns the needed size (including NUL); copies if
 * cap is large enough. */
int mf_plan_describe(const mf_plan* plan, char* buf, int cap);
/* Emitted KernelIR text of kernel k (same size convention). */
int mf_plan_kernel_text(const mf_plan* plan, int k, char* buf, int cap);
/* Comma-separated names that kernel k leaves as per-rank PARTIAL sums under
 * row sharding and that must be all-reduced before use:
 * column (cross-row) reductions, and dots over split vectors.  A dot over
 * vectors a matrix plan replicates (column-indexed) is whole on every rank
 * and is not listed. */
int mf_plan_kernel_column_outputs(const mf_plan* plan, int k, char* buf, int cap);

/* Launches every kernel of the plan on `stream` (a cudaStream_t; NULL = the
 * legacy default stream).  Asynchronous.  Buffers: device pointers.
 * A plan may be launched concurrently on several streams and from several
 * threads: it keeps one device workspace (cross-CTA partials, barrier
 * counters, unbound intermediates) per stream, so launches on different
 * streams never share scratch; launches on one stream are ordered by it. */
int mf_launch(const mf_plan* plan, const mf_buffer* buffers, int nbuf, const mf_scalar* scalars,
              int nscalars, void* stream, mf_stats* stats);

/* Launches kernel k only (sharded execution interleaves collectives). */
int mf_launch_kernel(const mf_plan* plan, int k, const mf_buffer* buffers, int nbuf,
                     const mf_scalar* scalars, int nscalars, void* stream, mf_stats* stats);

/* CUDA C++ source of kernel k when it runs on the generic path (the code
 * generator's output for KernelIRs no hand-written family covers); "" for
 * hand-written kernels.  Size convention as mf_plan_describe. */
int mf_plan_kernel_source(const mf_plan* plan, int k, char* buf, int cap);
/* Compiles every generic kernel of the plan for sm_100a now (NVRTC; needs no
 * GPU), so the first launch does not pay for it.  Returns MF_OK or the
 * compiler's diagnostics via mf_last_error(). */
int mf_plan_prepare(const mf_plan* plan);

/* vm::launch itself (proj/include/mapfuse/vm.hpp:94) over host buffers:
 * KernelIR text + device config text (NULL = the shipped device.cfg) ->
 * buffers updated in place, ExecutionStats (and, with MF_VM_TRACE, the
 * race-report size) as JSON in `json` (size convention as
 * mf_plan_describe; a negative return is -status on failure).  Kernels no
 * hand-written family covers -- and all kernels under MF_VM_TRACE or the
 * "vm_exact" option -- run the generic kernel with the VM's counters. */
#define MF_VM_TRACE 1     /* LaunchArgs::trace: device-side trace + detect_races */
#define MF_VM_NO_POISON 2 /* LaunchArgs::poison_onchip = false */
int mf_vm_launch(const char* kernel_ir_text, const char* device_config, const mf_buffer* host_buffers,
                 int nbuf, const mf_scalar* scalars, int nscalars, int flags, char* json, int cap);

/* vm::measure_routine (proj/include/mapfuse/vm.hpp:108): modeled cycles of
 * one routine ("load_A", "compute", ... = Routine::id()) of `function` in the
 * simulated fusion environment, counted on the GPU by the generic kernel's
 * VM instrumentation.  manifest NULL = the shipped library; device_config
 * NULL = the shipped device.cfg.  *cycles = -1 when infeasible. */
int mf_measure_routine(const char* manifest, const char* function, const char* routine,
                       int instances, int iterations, int extra_shared_bytes,
                       const char* device_config, int64_t* cycles);

/* Bound plans: the plan's kernels prepared once for fixed device buffers and
 * scalars (validation, scalar coefficients, grids, workspace), so a launch
 * costs only the kernel launches -- or, with mf_bound_graph_launch, one
 * CUDA-graph launch of the whole plan (captured on the first call; `stream`
 * must not be the legacy default stream).  The bound plan owns its own
 * workspace; its plan must outlive it.  Not for peer (sharded) launches. */
typedef struct mf_bound mf_bound;
int mf_plan_bind(const mf_plan* plan, const mf_buffer* buffers, int nbuf, const mf_scalar* scalars,
                 int nscalars, mf_bound** out);
int mf_bound_launch(mf_bound* bound, void* stream);
int mf_bound_graph_launch(mf_bound* bound, void* stream);
void mf_bound_destroy(mf_bound* bound);

/* Implementation generator: kernel k of a compiled plan
 * has mf_plan_count_implementations(plan, k) implementations -- routine
 * orderings x block shapes x instances x serial iterations x memory plans,
 * feasible, deduplicated, pruned.  mf_plan_implementation describes one as
 * JSON; mf_plan_set_implementation switches kernel k to it (generic kernels
 * change; kernels a hand-written family covers lower to the same kernel).
 * Returns -status when the plan carries no script (KernelIR / plan file). */
int64_t mf_plan_count_implementations(const mf_plan* plan, int k);
/* Size of the whole search space of a script: exact covers x implementation
 * choices of every kernel (the paper's Table 4 "Impl. count"). */
int64_t mf_count_implementation_space(const char* script_text, const char* manifest, int rows,
                                      int cols);
int mf_plan_implementation(const mf_plan* plan, int k, int index, char* json, int cap);
int mf_plan_set_implementation(mf_plan* plan, int k, int index);

/* Synchronizes `stream` and reports (MF_ERR_FAULT) the first device fault a
 * generic kernel of this plan recorded since the last check: out-of-bounds
 * global or on-chip index, poisoned on-chip read, division by zero -- the
 * VM's faults (proj/src/vm.cpp:77-81, :102-109, :184-185).  Hand-written
 * kernels validate everything before launch and never record faults.
 * mf_launch_host checks by itself. */
int mf_plan_check(const mf_plan* plan, void* stream);

/* vm::launch's exact contract with host memory: copies inputs host->device,
 * runs the plan, copies every bound output back, synchronizes.  stats->ms is
 * the device time of the kernels alone -- except for element-wise plans over
 * PINNED host buffers, which run as a chunked 3-stream pipeline (H2D, kernels
 * and D2H of different chunks overlap); there stats->ms covers the whole
 * pipeline. */
int mf_launch_host(const mf_plan* plan, const mf_buffer* host_buffers, int nbuf,
                   const mf_scalar* scalars, int nscalars, mf_stats* stats);

/* Row-sharded runs with the column reduction fused into the kernel: every
 * rank (one process per GPU) creates a peer group sized for n columns,
 * exports its IPC handle bytes, opens every peer's handle, then launches
 * kernels through mf_launch_kernel_peers.  Kernels with column outputs
 * (A^T r, B^T y) then finish with an in-kernel reduce-scatter + all-gather
 * over NVLink peer memory instead of a separate collective.  Ranks must
 * issue the same launch sequence.  mf_peer_group_connect_local links groups
 * living in one process (virtual ranks sharing a GPU; tests). */
typedef struct mf_peer_group mf_peer_group;
int mf_peer_group_create(int nranks, int rank, int64_t n_capacity, mf_peer_group** out);
int mf_peer_group_handle(const mf_peer_group* g, void* out, int cap); /* returns bytes needed */
int mf_peer_group_open(mf_peer_group* g, int peer, const void* handle, int len);
int mf_peer_group_connect_local(mf_peer_group* g, int peer, const mf_peer_group* other);
void mf_peer_group_destroy(mf_peer_group* g);
/* Synchronizes `stream` and reports (MF_ERR_FAULT) whether an in-kernel peer
 * barrier of this rank gave up waiting: a peer did not arrive within
 * MF_PEER_TIMEOUT_MS (default 10000) ms -- a rank crashed, or the ranks
 * issued different launch sequences.  The kernel then finished without the
 * cross-rank sum (outputs are invalid) instead of hanging the GPU; recreate
 * the group.  Clears the flag. */
int mf_peer_group_check(mf_peer_group* g, void* stream);
int mf_launch_kernel_peers(const mf_plan* plan, int k, mf_peer_group* g, const mf_buffer* buffers,
                           int nbuf, const mf_scalar* scalars, int nscalars, void* stream,
                           mf_stats* stats);
/* The whole plan on this rank's row panel with every cross-rank reduction
 * (matrix column outputs, stream-kernel dots) finished in-kernel -- the
 * sharded launch of SURVEY.md 8(b) for one-process-per-GPU C / C++ hosts,
 * no NCCL call.  Plans with generic kernels that reduce across rows need a
 * host collective (mf_launch_kernel + all-reduce) and are rejected. */
int mf_launch_peers(const mf_plan* plan, mf_peer_group* g, const mf_buffer* buffers, int nbuf,
                    const mf_scalar* scalars, int nscalars, void* stream, mf_stats* stats);

/* Counter-based synthetic data on the device, identical to the CPU checker's
 * generator: out[r*ld + c] = U(seed, (row0 + r) * ncols_global + c). */
/* Single-process, multi-GPU row-sharded launch: the mf_launch_sharded of
 * SURVEY.md 8(b).  GPU g (CUDA device devices[g]) runs plans[g] -- the plan
 * for its row panel, used with that device only -- on its buffers
 * per_gpu[g][0 .. nbuf[g]) and stream streams[g] (a cudaStream_t).  After
 * each kernel, the kernel's column reductions and dots
 * (mf_plan_kernel_column_outputs) are summed in place over the GPUs with
 * ncclAllReduce(ncclFloat, ncclSum) on comms[g] (the caller's ncclComm_t, one
 * per GPU, e.g. from ncclCommInitAll), inside one ncclGroupStart/End.  NCCL
 * is resolved at run time from the copy the process has loaded (with one GPU
 * and comms[0] == NULL no collective is issued).  Async on the
 * streams; stats are summed over the GPUs.  Replaces a host loop over
 * vm::launch per shard plus the host all-reduce the reference would need. */
int mf_launch_sharded(const mf_plan* const* plans, int ngpus, const int* devices,
                      const mf_buffer* const* per_gpu, const int* nbuf, const mf_scalar* scalars,
                      int nscalars, void* const* comms, void* const* streams, mf_stats* stats);

int mf_generate(float* dev, int64_t rows, int64_t cols, int64_t ld, uint64_t seed, int64_t row0,
                int64_t ncols_global, void* stream);

/* Engine options: "matrix_k" (2|4 float4 slots per thread), "f64acc" (0|1:
 * accumulate matrix reductions in fp64), "occupancy" (CTAs per SM),
 * "generic" (0|1: run every kernel on the generic NVRTC-emitted path, even
 * where a hand-written family applies), "generic_poison" (0|1: generic
 * kernels poison on-chip memory and fault on uninitialised reads),
 * "generic_iterations" (0 = per size, else the serial iterations of generic
 * kernels), "generic_by" (0 = default, else block rows of depth-2 generic
 * kernels), "generic_prefetch" (0 = auto, else how many iterations ahead
 * generic kernels issue their loads), "generic_rewrite" (mask, default 55:
 * 1 warp row reduction, 2 deferred on-chip accumulators, 4 prologue vectors
 * read from global, 8 row-reduction stores folded, 16 barrier pruning, 32
 * late tile prefetch, 64 warp vectors; 0 = the paper's literal tile
 * algorithm), "generic_checked" (0|1: keep per-access
 * index checks even when the bounds are proved at launch), "vm_exact" (0|1:
 * vm::launch always counts like the VM), "nvtx" (0|1: NVTX ranges per
 * kernel), "codegen_barriers" (test hook, 0 = codegen omits barriers),
 * "tma" (-1 auto | 0 register-fed | 1 TMA ring matrix kernels),
 * "tma_consumers" (0 auto | 256 | 512), "rowres_variant" (row-resident chain
 * with n <= 16384: 0 auto | 1 stage-held | 2 register-held rows),
 * "rowres_cluster" (wide-row chain:
 * 0 auto | 1 .. 7, see mf_rowres.cu), "matrix_tile_finalize" (matrix
 * outputs finished on tile-completion counters instead of after a grid
 * barrier: 0 none | 1 row outputs | 2 row and column outputs),
 * "max_sms" (0 = all SMs, else cap the
 * matrix grid), "matrix_l2_normal" (-1 auto: evict-normal for kernels that
 * store a matrix, evict-first otherwise | 0 | 1), "stream_unroll" (0 = 2 |
 * 2 | 4 | 8 float4 per thread per stream), "stream_ctas_per_sm" (0 = one CTA
 * per block, else a capped grid striding over blocks), "matrix_waves" (row
 * bands per co-resident CTA of the register-fed matrix kernel, 1 .. 16) and
 * "matrix_dynamic" (0 | 1: tiles after a CTA's first from a counter),
 * "finalize_group" (0 = 8 | 8 | 16 | 32 lanes per slot in the cross-CTA
 * finalize), "rowres_force_cluster" (0 | 1: rows of n <= 16384 over a CTA
 * cluster), "rowres_l2_ahead" (-1 auto = 0 .. 8 rows prefetched into L2
 * beyond the row-resident ring), "stream_ld_hint" (0 | 1: .L2::256B hint on
 * element-wise loads).  Round-2 experiments; their defaults are the measured
 * best (profiles/r02_*). */
int mf_set_option(const char* key, int value);
int mf_get_option(const char* key);

const char* mf_last_error(void);
const char* mf_version(void);

#ifdef __cplusplus
}
#endif

#endif /* MAPFUSE_B200_H */
