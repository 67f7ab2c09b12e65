// mf_exec.hpp -- binds a NativePlan to device buffers and launches it.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "mf_jit.hpp"
#include "mf_native.hpp"

namespace mapfuse::b200 {

// vm::VmFault analogue (proj/include/mapfuse/vm.hpp:21-23).
struct Fault : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// ir::ParseError / invalid-argument analogue.
struct Invalid : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct DevBuf {
  float* ptr = nullptr;
  int64_t rows = 0, cols = 0;
  int64_t size() const { return rows * cols; }
};
using BufMap = std::map<std::string, DevBuf>;
using ScalarMap = std::map<std::string, double>;

struct EngineOptions {
  int matrix_k = 2;
  int f64acc = 0;
  int occupancy = 2;
  int stream_unroll = 0;       // 0 = default (2), else 2 / 4 / 8 float4 per thread per stream
  int stream_ctas_per_sm = 0;  // 0 = one CTA per block (non-persistent), else capped grid
  int tma = -1;  // matrix kernels: -1 auto (by shape), 1 = TMA ring, 0 = register-fed
  int max_sms = 0;  // > 0: cap the SMs a matrix kernel's grid is sized for
  int tma_consumers = 0;  // TMA matrix variant: 0 auto (by shape), 256 or 512 consumer threads
  int matrix_tile_finalize = 0;  // matrix outputs finished on tile counters: 0 none, 1 rows, 2 rows + columns
  int rowres_variant = 0;  // row-resident chain, n <= 16384: 0 auto, 1 stage-held, 2 register-held
  int rowres_cluster = 0;  // wide-row chain variant: 0 auto, 1 stage-held, 2 register-held, 3 8192-col slices
  // matrix operand loads: 0 evict-first L2 policy, 1 evict-normal, -1 auto =
  // evict-normal when the kernel also stores a matrix (GEMVER stage 1: 2036 ->
  // 1996 us, fewer dirty lines of B left for the next kernel to write back),
  // evict-first for read-only kernels (BiCGK 159.7 -> 157.7 us)
  int matrix_l2_normal = -1;
  int tma_bulk_store = 1;  // TMA store shapes: 1 = E leaves through cp.async.bulk S2G, 0 = st.global
  // register-fed matrix kernels: row bands per co-resident CTA (1 = one tile
  // per CTA) and whether CTAs past their first tile take the next one from a
  // counter (1) or round-robin (0)
  int matrix_waves = 1;
  int matrix_reverse = -1;  // register-fed matrix kernels: row batches bottom-up within each band:
                            // -1 auto (after an earlier kernel stored the matrix) | 0 never | 1 always
  int stream_ld_hint = 0;  // element-wise kernels' loads: 0 plain, 1 .L2::256B prefetch-size hint
  int rowres_force_cluster = 0;
  int rowres_l2_ahead = -1;  // row-resident chains: rows prefetched into L2 beyond the ring (-1 auto)  // 1: rows of n <= 16384 also split over a CTA cluster (variant 7 by default)
  int finalize_group = 0;  // cross-CTA finalize lanes per float4 slot: 0 (= 8) | 8 | 16 | 32
  int matrix_dynamic = 0;
  int generic_poison = 0;
  int nvtx = 0;
  int generic_checked = 0;  // 1: generic kernels keep per-access checks even when proved in bounds  // 1: an NVTX range around every kernel launch (named after the plan kernel)  // 1: generic kernels poison on-chip memory (VM fault on uninitialised reads)
};

// A row-sharding group's in-kernel exchange buffers (see PeerLinks).
struct PeerGroup {
  int nranks = 1, rank = 0;
  int64_t n_cap = 0;
  float* inbox = nullptr;     // local: [2][P][n_cap]
  float* outbox = nullptr;    // local: [2][n_cap]
  unsigned* flags = nullptr;  // local: 64 counters, zeroed
  float* peer_inbox[8] = {};
  float* peer_outbox[8] = {};
  unsigned* peer_flags[8] = {};
  std::vector<void*> opened;  // IPC mappings to close
  unsigned epoch = 0;
  ~PeerGroup();
};
EngineOptions& options();

// SMs a persistent kernel's grid may use: the device's, capped by option
// max_sms and by the launching plan's device description (PlanSmsScope,
// thread-local for the duration of one launch / bind call).
int effective_sms();
struct PlanSmsScope {
  explicit PlanSmsScope(int cap);
  ~PlanSmsScope();
  PlanSmsScope(const PlanSmsScope&) = delete;
  PlanSmsScope& operator=(const PlanSmsScope&) = delete;
  int saved;
};

// Device scratch owned by one plan: cross-CTA partials, barrier / ticket
// counters, unbound intermediates, and (for host launches) device mirrors of
// host buffers.  Launches of one plan on one stream are serialized by the
// stream; the mutex guards the allocation tables.
class Workspace {
 public:
  ~Workspace();
  void* scratch(size_t bytes, cudaStream_t s);   // grows on demand
  unsigned* counters(cudaStream_t s);            // zeroed once, self-resetting
  unsigned* tile_counters(size_t words, cudaStream_t s);  // matrix tile counters, zeroed, self-resetting
  float* named(const std::string& key, int64_t words);  // persistent per key
  unsigned* jit_fault(cudaStream_t s);           // generic kernels' fault word pair, zeroed once
  bool jit_used() const { return jit_fault_ != nullptr; }
  std::mutex mu;

 private:
  void* scratch_ = nullptr;
  size_t scratch_bytes_ = 0;
  unsigned* counters_ = nullptr;
  unsigned* tile_ = nullptr;
  size_t tile_words_ = 0;
  unsigned* jit_fault_ = nullptr;
  std::map<std::string, std::pair<float*, int64_t>> named_;
  std::vector<void*> retired_;  // outgrown buffers, freed with the workspace
};

// A prepared launch: replays one kernel (all host-side work done) on a stream.
using Recorder = std::vector<std::function<cudaError_t(cudaStream_t)>>;

// Launches plan.kernels[k]; throws Fault / Invalid.
void run_kernel(const NativePlan& plan, int k, const BufMap& bufs, const ScalarMap& scalars,
                cudaStream_t stream, Workspace& ws, PeerGroup* peers = nullptr);
// Synchronizes `stream` and turns a fault recorded by a generic kernel of
// this workspace (host/cudagen.cpp: bounds, poisoned read, division by zero)
// into a Fault -- the VM's VmFault (proj/src/vm.cpp:77-81).  Resets it.
void check_jit_faults(Workspace& ws, cudaStream_t stream);
// The reference VM's instrumentation on a generic kernel (host/cudagen.cpp
// MFJ_STATS / MFJ_TRACE): runs it once, synchronously, and returns the
// counters (mf_jit.hpp MfjStat layout), the access trace if `trace` (up to
// trace_cap records) and the block count.  Returns the number of trace
// records the kernel produced (> trace_cap: rerun with a larger buffer).
// cost = DeviceConfig cycles per global word, shared word, arith op,
// barrier, atomic, and the warp size.
int64_t run_generic_counted(const NativeKernel& k, const BufMap& bufs, const ScalarMap& sc,
                            const int cost[6], bool trace, int64_t trace_cap, cudaStream_t s,
                            Workspace& ws, std::vector<uint64_t>* stats,
                            std::vector<MfjRec>* recs, int64_t* blocks);
// Prepares plan.kernels[k] for the given bindings (validation, coefficients,
// grid, workspace) and appends its launch to `rec` instead of launching.
// Peer (in-kernel collective) launches are not recordable.
void record_kernel(const NativePlan& plan, int k, const BufMap& bufs, const ScalarMap& scalars,
                   cudaStream_t stream, Workspace& ws, Recorder& rec);
// Binds any plan intermediates the caller left unbound (workspace-backed).
BufMap complete_bindings(const NativePlan& plan, const BufMap& bufs, Workspace& ws);

int device_sm_count();
void check_cuda(cudaError_t e, const char* what);

}  // namespace mapfuse::b200

namespace mapfuse::vm {
// Engine option "vm_exact" (env MF_VM_EXACT): vm::launch always runs the
// generic kernel with the VM's counters, even where a hand-written family
// applies (exact ExecutionStats at the cost of speed).
void set_exact(bool on);
bool exact();
}  // namespace mapfuse::vm
