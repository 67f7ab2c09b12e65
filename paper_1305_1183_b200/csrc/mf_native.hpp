// mf_native.hpp -- the "native plan": what one planner-selected kernel does,
// in terms the hand-written sm_100a templates understand.
//
// The reference executes a fused kernel by interpreting its KernelIR on a
// virtual SIMT device (proj/src/vm.cpp:450-479).  Here the same KernelIR is
// lowered (mf_lower.cpp) into one of two kernel families:
//
//   StreamOp  depth-1 map chains (add / scal / waxpby / axpydot_stage and
//             their fusions) = up to 2 stored linear combinations of up to 4
//             input streams, plus an optional dot reduction (dot, AXPYDOT).
//   MatrixOp  depth-2 single pass over one or two row-major matrices:
//             optional rank-2 update (ger2) with optional store, row
//             reductions y = a*E x (sgemv / sgemvs) and column reductions
//             y = a*E^T x (sgemtv), all from ONE read of each matrix.
//
// Scalars enter as coefficient polynomials (products of script scalars and
// literals) evaluated in fp64 at launch time.
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <vector>

namespace mapfuse::b200 {

// sum_k c_k * prod(syms_k); syms name script scalars.
struct Coef {
  struct Term {
    double c = 1.0;
    std::vector<std::string> syms;
  };
  std::vector<Term> terms;

  static Coef constant(double v) { return Coef{{Term{v, {}}}}; }
  static Coef symbol(const std::string& s) { return Coef{{Term{1.0, {s}}}}; }
  bool is_zero() const { return terms.empty(); }
  Coef operator*(const Coef& o) const;
  Coef operator+(const Coef& o) const;
  double eval(const std::map<std::string, double>& scalars) const;  // throws on unbound
  std::string str() const;
};

struct StreamOp {
  std::vector<std::string> inputs;  // <= 4 global vectors (or flattened matrices)
  struct Out {
    std::string name;
    std::vector<Coef> coef;  // one per input
  };
  std::vector<Out> outs;    // <= 2 stored outputs
  bool has_dot = false;
  std::vector<Coef> dot_a, dot_b;  // r = sum (dot_a . in)(dot_b . in)
  std::string dot_out;             // 1x1 buffer
};

struct MatrixOp {
  std::vector<std::string> mats;  // 1 or 2 row-major matrices (m x n)
  // rank update applied to mats[0]: E = M0 + sum_q u_q v_q^T (ger2)
  std::vector<std::pair<std::string, std::string>> rank;  // (u: length m, v: length n)
  std::string store;  // E written here (ger2 output), "" if not stored
  struct Red {
    int mat = 0;      // which matrix (E for mat 0 when rank is non-empty)
    std::string x;    // row reduction: x length n ; column reduction: x length m
    std::string y;    // output
    Coef coef;        // y = coef * (E x)  or  coef * (E^T x)
  };
  std::vector<Red> rows;  // y[i] = coef * sum_j E[i][j] x[j]     (<= 2)
  std::vector<Red> cols;  // y[j] = coef * sum_i E[i][j] x[i]     (<= 2)
  // row-resident chain (planner mode "b200"): cols[0].x is rows[0]'s result,
  // computed in the same pass; rows[0].y may be "" (t never stored)
  bool chain = false;
};

// An index expression a generic kernel evaluates, as an affine form over
// symbols with known ranges -- proved in bounds at launch (then the kernel
// runs without per-access checks, in 32-bit index arithmetic when safe).
struct GenericBound {
  enum Kind : int { Const = 0, FullX = 1, FullY = 2, NElems = 3, LaunchX = 4, LaunchY = 5 };
  struct Term {
    int64_t coef = 0;
    int lo_kind = Const, hi_kind = Const;  // bound = value of kind (0 for Const) + offset
    int64_t lo = 0, hi = 0;
  };
  int buffer = -1;       // >= 0 global buffer; -1 on-chip (words); -2 range only (conditions)
  int64_t words = 0;     // on-chip: valid words [0, words)
  bool two = false;      // global 2-D (row, col) index
  bool affine = true;    // false: not provable (div / mod / min, unbounded loop variable)
  int64_t c0[2] = {0, 0};
  std::vector<Term> terms[2];
};

// Generic kernel: any KernelIR, emitted as CUDA C++ by
// host/cudagen.cpp following the reference VM's execution semantics
// (proj/src/vm.cpp:357-445) and JIT-compiled for sm_100a with NVRTC
// (mf_jit.cpp).  Covers every kernel the hand-written families do not.
struct GenericOp {
  std::string source;                // CUDA C++ translation unit (NVRTC input)
  std::vector<std::string> buffers;  // MfjArgs::buf[i] order
  std::vector<char> extent;          // per buffer: 't' m x n, 'm', 'n', '1' (traffic accounting)
  std::vector<std::string> scalars;  // MfjArgs::scal[j] order
  std::vector<std::string> inputs, outputs;  // global loads / stores (+ atomics)
  std::vector<std::string> accumulated;      // targets of global atomic adds
  int depth = 1, block_x = 32, block_y = 1, instances = 1, iterations = 1;
  char iter_dim = 'x';
  std::string domain;
  int shared_words_total = 0;
  std::vector<GenericBound> bounds;  // every index expression (launch-time proof)
};

struct NativeKernel {
  enum class Kind { Stream, Matrix, Generic } kind = Kind::Stream;
  std::string name;  // e.g. "bicgk_k0[sgemv+sgemtv]"
  std::vector<int> calls;  // script call ids covered
  StreamOp stream;
  MatrixOp matrix;
  GenericOp generic;
  // Generic kernels only: true = the reference VM's contract (global atomic
  // outputs accumulate onto what the caller stored, vm.hpp:91-93); false =
  // this engine's contract (outputs are overwritten: zeroed before launch).
  bool vm_semantics = false;
  int generic_poison = -1;  // generic kernels: -1 engine option, 0 / 1 explicit (LaunchArgs::poison_onchip)
  // implementation variant chosen by the cost model (matrix kernels):
  // tma -1 = engine default, 0 register-fed, 1 TMA ring; k = float4 slots/thread
  int variant_tma = -1;
  int variant_k = 0;

  // Algorithmic traffic: every distinct input read once, every
  // output written once.  Evaluated for a concrete m x n.
  uint64_t bytes_loaded(int64_t m, int64_t n) const;
  uint64_t bytes_stored(int64_t m, int64_t n) const;
  // Names produced by a column (cross-row-band) reduction: under row sharding
  // these need an all-reduce.
  std::vector<std::string> column_outputs() const;
  std::vector<std::string> inputs() const;
  std::vector<std::string> outputs() const;
};

enum class Role { Input, Output, Intermediate };

struct BufferSpec {
  std::string name;
  int rows = 1, cols = 1;  // padded shape for the plan's m x n
  Role role = Role::Input;
  bool scalar = false;     // 1x1 reduction output
  bool row_indexed = false;  // vector indexed by matrix rows (length m); sharded by rows
};

struct NativePlan {
  std::string sequence;   // informational
  int rows = 0, cols = 0;  // padded problem size
  std::vector<NativeKernel> kernels;  // launch order
  std::vector<BufferSpec> buffers;
  std::vector<std::string> scalars;   // script scalar names the plan needs
  std::vector<std::string> kernel_ir;  // emitted KernelIR text per kernel (may be empty)
  double predicted_us = 0.0;           // cost-model prediction (0 if not planned)
  // what the plan was compiled from (implementation search re-generates
  // kernels from it); empty for plans made from KernelIR text / plan files
  std::string script_text, manifest;
  const BufferSpec* find(const std::string& n) const {
    for (const auto& b : buffers)
      if (b.name == n) return &b;
    return nullptr;
  }
  uint64_t bytes_loaded() const;
  uint64_t bytes_stored() const;
  std::string describe_json() const;
  // Row-sharded execution (sharding.py, mf_launch_peers, mf_launch_sharded):
  // plans with a matrix split A into row panels and split row-indexed
  // vectors, replicating column-indexed ones; depth-1 plans split every
  // vector.  The outputs of kernel k that are then per-rank PARTIAL sums and
  // must be summed over the ranks: column reductions always; a dot only when
  // its vectors are split (a dot over replicated vectors is already whole).
  bool row_sharded_matrix() const;
  std::vector<std::string> rank_reductions(int k) const;
};

}  // namespace mapfuse::b200
