// mapfuse/planner.hpp -- the optimizer: fusion planner, code generator,
// B200 cost model, combination selector and the compile pipeline.
//
// The reference declares these modules in its build (proj/CMakeLists.txt:40-48:
// planner.cpp, implgen.cpp, costmodel.cpp, selector.cpp, codegen.cpp,
// pipeline.cpp) but ships none of their sources; their contract is SPEC.md
// :181-533.  This is a new implementation of that contract, retargeted to
// B200: every kernel the selector chooses is lowered onto a hand-written
// sm_100a kernel family, and the cost model predicts HBM time from
// algorithmic bytes and measured per-family efficiency.
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "mapfuse/device.hpp"
#include "mapfuse/kernel.hpp"
#include "mapfuse/library.hpp"
#include "mapfuse/script.hpp"
#include "mf_native.hpp"

namespace mapfuse::plan {

struct Sizes {
  int64_t rows = 0, cols = 0;  // padded problem size
};

// ---------------------------------------------------------------- planner
struct Fusion {
  std::vector<int> calls;              // sorted call ids (size >= 2)
  std::vector<script::Edge> internal;  // dataflow kept on chip
  std::vector<std::string> shared;     // read-only inputs read by several members
  int64_t saved_words = 0;
};

// Rule ids: nesting-mismatch | global-barrier-required |
// no-savings | block-capacity.  A non-convex set (a path leaves the set and
// re-enters it) also needs a global barrier and reports that rule.
struct ConstraintViolation {
  std::string rule;
  std::vector<int> nodes;
  std::string explanation;
};

// Planner rule set.  reference: SPEC.md's rules (+ convexity).  row_resident
// (mode "b200"): additionally a row reduction may feed a column reduction of
// the SAME matrix inside one kernel when a whole row fits one CTA's ring
// (cols <= row_resident_max_cols): the CTA -- or, for rows wider than one
// CTA's shared memory, a cluster of up to 8 CTAs over distributed shared
// memory -- completes t_i itself, no global barrier is needed (mf_rowres.cu).
// Beyond the paper; off by default.
struct PlannerOptions {
  bool row_resident = false;
  int64_t row_resident_max_cols = 131072;
  int64_t cols = 0;  // padded problem cols (row-resident feasibility)
  // block-capacity rule: the fusion's smallest Algorithm 1/2
  // kernel (BY = 2, one instance, one iteration, first-fit shared plan) must
  // fit one CTA.  B200: 227 KB opt-in shared memory, 1024 threads.
  int64_t block_shared_bytes = 227 * 1024;
  int max_threads_per_block = 1024;
};

std::optional<ConstraintViolation> fusibility(const std::vector<int>& nodes,
                                              const script::Script& s,
                                              const script::DataDependencyGraph& g,
                                              const lib::Library& L,
                                              const PlannerOptions& opt = {});
inline bool is_fusible(const std::vector<int>& nodes, const script::Script& s,
                       const script::DataDependencyGraph& g, const lib::Library& L,
                       const PlannerOptions& opt = {}) {
  return !fusibility(nodes, s, g, L, opt).has_value();
}

// Words each script name occupies at the padded size (tiles m*n, vectors m
// or n by role, scalars 1).
std::map<std::string, int64_t> element_words(const script::Script& s, const lib::Library& L,
                                             Sizes sz);

// (words moved by the members unfused) - (words moved fused).
int64_t transfer_savings(const Fusion& f, const script::Script& s,
                         const script::DataDependencyGraph& g, const lib::Library& L, Sizes sz);

// All connected (edges + shared inputs), fusible subsets of size 2..max_size
// with positive savings, sorted by call ids.
std::vector<Fusion> enumerate_fusions(const script::Script& s, const script::DataDependencyGraph& g,
                                      const lib::Library& L, Sizes sz, int max_size = 6,
                                      const PlannerOptions& opt = {});

// ---------------------------------------------------------------- codegen
struct CodegenParams {
  int by = 8;          // block rows for depth-2 kernels (BY macro)
  int instances = 4;   // instances per block for depth-1 kernels (IPB)
  int iterations = 1;  // serial iterations (ITERS)
  bool barriers = true;  // test hook: suppress barrier insertion
  // Routine-call order of the loop body (SPEC.md:262 enumerate_orderings):
  // a permutation of the default order's loop items, consistent with the
  // routine dependencies; empty = the default (script order per member).
  std::vector<int> order;
  // Shared-memory plan (SPEC.md:263-268 plan_memory): false = one region per
  // element; true = greedy first-fit over live ranges, regions of elements
  // with disjoint live ranges overlap (barrier condition 2 guards reuse).
  bool overlap = false;
};

// Algorithm 1 / 2 kernel for a set of calls (one call = unfused kernel).
kernel::KernelIR generate_kernel(const std::vector<int>& calls, const script::Script& s,
                                 const script::DataDependencyGraph& g, const lib::Library& L,
                                 const CodegenParams& p = {});

// ---------------------------------------------------------------- implementation generator
// (SPEC.md:248-334).  All topological orders of the loop body's routine calls
// (loads before the computes reading them, computes before their stores,
// producer computes before consumer computes), at most `cap`.
std::vector<std::vector<int>> enumerate_orderings(const std::vector<int>& calls, const script::Script& s,
                                                  const script::DataDependencyGraph& g,
                                                  const lib::Library& L, int cap = 64);

struct SearchSpace {
  std::vector<int> block_rows{2, 4, 8, 16};  // BY, depth 2
  std::vector<int> instances{1, 2, 4};       // depth 1 (capped by the functions' max_instances)
  std::vector<int> iterations{1, 2, 4, 8, 16};
  bool overlap_plans = true;                 // also the first-fit overlapping memory plan
  int max_orderings = 64;
};

struct FusionImplementation {
  std::vector<int> calls;
  CodegenParams params;   // order, block shape, instances, iterations, memory plan
  kernel::KernelIR kir;
  int shared_bytes = 0;   // per block
};

// Cross product orderings x block shapes x instances x iterations x memory
// plans, feasible under the device limits, with iterations that divide the
// iterated grid extent at `sz` (Sizes{0,0}: no size filter), deduplicated by
// kernel text and pruned (prune_implementations).  Deterministic order.
std::vector<FusionImplementation> enumerate_implementations(const std::vector<int>& calls,
                                                            const script::Script& s,
                                                            const script::DataDependencyGraph& g,
                                                            const lib::Library& L, Sizes sz,
                                                            const SearchSpace& space = {},
                                                            const vm::DeviceConfig& dev = {});
// Drops implementations strictly dominated by another with the same block
// shape, instances and iterations but fewer shared bytes.
std::vector<FusionImplementation> prune_implementations(std::vector<FusionImplementation> list);
// The implementations of kernel k of a compiled plan (from its script and
// library, at the plan's size); throws if the plan does not carry its script.
std::vector<FusionImplementation> kernel_implementations(const b200::NativePlan& p, int k);
// Covers x implementation choices of a script at a size (Table 4 "Impl. count").
int64_t count_implementation_space(const std::string& script_text, const lib::Library& L, int rows,
                                   int cols);
// Replaces kernel k by the given implementation (of kernel_implementations).
void set_kernel_implementation(b200::NativePlan& p, int k, const FusionImplementation& impl);

// ---------------------------------------------------------------- lowering
// KernelIR -> the sm_100a kernel family and its operand roles.  Throws
// std::invalid_argument when no hand-written template covers the kernel.
b200::NativeKernel lower_kernel(const kernel::KernelIR& k);
// Generic path: KernelIR -> CUDA C++ that executes it with
// the reference VM's semantics (proj/src/vm.cpp:357-445), one CTA per VM
// block.  Throws std::invalid_argument for a KernelIR the VM would reject
// statically (unexpanded macro, barrier inside a body, unknown region).
b200::NativeKernel generic_kernel(const kernel::KernelIR& k);
// lower_kernel when a hand-written family covers the kernel, else the
// generic kernel (or always generic with engine option "generic" = 1).
b200::NativeKernel lower_or_generic(const kernel::KernelIR& k);
// Engine option "generic" (env MF_GENERIC): route every kernel to the
// generic path (tests, and the measured cost of the generic emitter).
void set_force_generic(bool on);
bool force_generic();
// Engine option "generic_iterations": 0 = chosen per problem size
// (generic_params), >= 1 = fixed serial iterations for generic kernels.
void set_generic_iterations(int n);
int generic_iterations();
// Engine option "generic_by": 0 = default, else the block rows (BY) of
// depth-2 generic kernels (2 | 4 | 8 | 16).
void set_generic_by(int by);
int generic_by();
// Engine option "generic_prefetch": loads of the loop body are issued this
// many iterations ahead (0 = auto: 4, 2 or 1 within 32 registers per thread).
void set_generic_prefetch(int d);
int generic_prefetch();
// Engine option "generic_rewrite": which rewrites of the paper's literal
// tile algorithm uninstrumented generic kernels use (host/cudagen.cpp); the
// instrumented variants always run the literal algorithm.
//   kRwRowReduce  a forwarded tile's rows summed by a warp reduce-scatter
//                 (no transposed shared read, no shared atomics)
//   kRwDefer      loop-body on-chip accumulators kept in registers until
//                 after the serial iterations
//   kRwGlobal     prologue copies of read-only vectors read from global
//   kRwStore      a row reduction's store routine folded into its lanes
//   kRwPrune      barriers the rewritten kernel no longer needs compiled out
enum : int {
  kRwRowReduce = 1,
  kRwDefer = 2,
  kRwGlobal = 4,
  kRwStore = 8,
  kRwPrune = 16,
  kRwLatePrefetch = 32,  // depth 2: next tile's loads issued after the current tile's last use
  kRwWarpVector = 64,    // body copies of a warp-width vector slice held in registers, read by shuffle
  kRwAll = 127,
  // store folding measured slower (generic BiCGK 220 -> 720 us): the
  // lanes' scattered row atomics replace one contiguous warp atomic per tile
  kRwDefault = kRwRowReduce | kRwDefer | kRwGlobal | kRwPrune | kRwLatePrefetch,
};
void set_generic_rewrite(int mask);
int generic_rewrite();
// Default implementation parameters of a generic kernel whose domain buffer
// is dom_rows x dom_cols (a vector: 1 x length).
CodegenParams generic_params(const kernel::KernelIR& k, int64_t dom_rows, int64_t dom_cols);
// Shape of the kernel's domain buffer in the script at the padded size.
std::pair<int64_t, int64_t> domain_shape(const kernel::KernelIR& k, const script::Script& s,
                                         const lib::Library& L, Sizes sz);
// Test hook "codegen_barriers" = 0: codegen omits every barrier (the SPEC's
// mutation check) -- the reference VM's race detector and
// compute-sanitizer racecheck on the generic kernel must both flag it.
void set_codegen_barriers(bool on);
bool codegen_barriers();
bool stream_template_exists(int nin, int nout, bool dot);
bool matrix_template_exists(int nmat, int nrank, int store, int nrow, int ncol);

// ---------------------------------------------------------------- cost model
// t = max(bytes / (eta * BW), flops / F) + launch.  eta per kernel family
// and variant comes from the benchmark table (measured on B200; overridable
// with MF_COST_DB=<file of "key eta" lines>).
struct CostModel {
  vm::B200Device dev;
  std::map<std::string, double> eta;

  static CostModel defaults();
  // Picks the best variant for the kernel, stores it in k.variant, returns us.
  double predict_us(b200::NativeKernel& k, int64_t m, int64_t n) const;
};

// ---------------------------------------------------------------- selector
struct Item {
  std::vector<int> calls;
  kernel::KernelIR kir;
  b200::NativeKernel native;
  double predicted_us = 0;
};

struct Combination {
  std::vector<Item> kernels;  // launch order (topological over the condensed DAG)
  double predicted_us = 0;
};

// k best exact covers of the script's calls by lowerable fusions and single
// calls, ascending predicted time (ties: fewer kernels, then call ids).
std::vector<Combination> enumerate_combinations(const script::Script& s,
                                                const script::DataDependencyGraph& g,
                                                const lib::Library& L, Sizes sz,
                                                const CostModel& cm, int k,
                                                bool allow_fusion = true,
                                                const PlannerOptions& opt = {});
uint64_t count_combinations(const script::Script& s, const script::DataDependencyGraph& g,
                            const lib::Library& L, Sizes sz);

// ---------------------------------------------------------------- pipeline
// parse -> graph -> validate -> plan -> select -> codegen -> lower.
// mode: 0 fused (the paper's rules), 1 unfused (one kernel per call),
//       2 b200 (fused + row-resident chains, beyond the paper).
b200::NativePlan compile(const std::string& script_text, const lib::Library& L, int rows, int cols,
                         int mode);
// The rank-th best combination (0 = the selector's choice) -- empirical
// top-k search (SPEC.md:677-693 cmd_search) times these on the device.
b200::NativePlan compile_ranked(const std::string& script_text, const lib::Library& L, int rows,
                                int cols, int mode, int rank);
int64_t count_covers(const std::string& script_text, const lib::Library& L, int rows, int cols);

// Plan files: a compiled plan as re-runnable text -- header,
// buffer table, and each kernel's KernelIR (re-lowered on load).
std::string save_plan(const b200::NativePlan& p);
b200::NativePlan load_plan(const std::string& text);

}  // namespace mapfuse::plan
