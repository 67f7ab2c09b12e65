// mf_jit.hpp -- NVRTC-compiled generic kernels (host/cudagen.cpp emits them).
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

namespace mapfuse::b200 {

// Host mirror of the emitted `struct MfjArgs` (host/cudagen.cpp kPrelude):
// same member types and order, so the layouts agree.
constexpr int kMfjMaxBuffers = 64;
constexpr int kMfjMaxScalars = 32;
struct MfjRec {  // vm::TraceRecord as the kernel writes it
  int block;
  int epoch;
  unsigned char space;  // 0 shared, 1 register, 2 global (vm::Space order)
  int region;
  long long addr;
  int thread;
  unsigned char kinds;
};
struct MfjArgs {
  float* buf[kMfjMaxBuffers];
  long long rows[kMfjMaxBuffers];
  long long cols[kMfjMaxBuffers];
  float scal[kMfjMaxScalars];
  long long full_x, full_y, n_elems;
  unsigned int* fault;
  unsigned long long* stats;  // kMfjStatWords counters (layout in host/cudagen.cpp)
  MfjRec* trace;
  long long trace_cap;
  int cost[6];  // DeviceConfig cycles: global word, shared word, arith, barrier, atomic; warp size
};
constexpr int kMfjStatWords = 134;
enum MfjStat : int {
  kStatLoaded = 0, kStatStored = 64, kStatShared = 128, kStatAtomics = 129, kStatBarriers = 130,
  kStatArith = 131, kStatBlockCycles = 132, kStatTraceCursor = 133,
};
// Instrumentation variants of a generic kernel (compile-time in the source).
struct JitFlags {
  bool poison = false;
  bool stats = false;  // the VM's ExecutionStats counters
  bool trace = false;  // the VM's access trace (implies stats)
  bool unchecked = false;  // every index proved in bounds at launch: no per-access checks
  bool idx32 = false;      // ... and every index value fits 32 bits: int index arithmetic
  bool exact = false;      // ... and the grid's serial iterations cover the domain exactly:
                           // no iteration of any block falls outside it
};

// Device fault codes written by generic kernels (first fault wins).
enum JitFault : unsigned {
  kJitOk = 0,
  kJitGlobalBounds = 1,
  kJitOnchipBounds = 2,
  kJitPoisonRead = 3,
  kJitDivZero = 4,
  kJitBadStep = 5,
};

// Compiles (once per process, cached) and launches on `stream`.
void jit_launch(const std::string& src, JitFlags flags, dim3 grid, dim3 block, size_t smem,
                const MfjArgs& args, cudaStream_t stream);
// NVRTC compile only (no GPU needed): returns the sm_100a cubin; log optional.
std::vector<char> jit_compile_only(const std::string& src, JitFlags flags, std::string* log);
// Compiles into the process cache (no GPU needed); later launches reuse it.
void jit_prepare(const std::string& src, JitFlags flags);
// Compiles and loads the module on the current device (before a graph capture).
void jit_load(const std::string& src, JitFlags flags);
bool jit_available(std::string* why);
size_t jit_cache_size();

}  // namespace mapfuse::b200
