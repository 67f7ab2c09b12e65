// mf_kernels.cuh -- launch-side view of the sm_100a kernel families.
//
// Argument blocks are plain structs passed by value; the host side
// (mf_exec.cpp) fills them from a NativeKernel + bound device buffers.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace mapfuse::b200 {

constexpr int kStreamMaxIn = 4;
constexpr int kStreamMaxOut = 2;

// Depth-1 streaming kernel: out_o = sum_i coef[o][i] * in_i  (fp64 arithmetic,
// one rounding to fp32 per stored value -- bit-identical to the reference's
// fp64 formulas, proj/src/blas.cpp:185-265), plus optional
// r = sum (da . in)(db . in) in fp64 with a deterministic two-level reduce.
// In-kernel cross-GPU reduction of column outputs (row-sharded runs).
// Every rank owns a group-allocated inbox [2][P][n], outbox [2][n] and two
// arrival counters; peers' copies are mapped into this process (CUDA IPC over
// NVLink, or plain pointers for virtual ranks sharing one GPU).
constexpr int kMaxRanks = 8;
// flags[rank][kPeerErrorWord]: set by a peer barrier that timed out (a peer
// never arrived); mf_peer_group_check reports and clears it.
constexpr int kPeerErrorWord = 62;
struct PeerLinks {
  int nranks = 1, rank = 0;
  float* inbox[kMaxRanks] = {};
  float* outbox[kMaxRanks] = {};
  unsigned* flags[kMaxRanks] = {};
  unsigned epoch = 0;               // launches so far in this group (1-based)
  long long n_cap = 0;              // inbox / outbox row capacity (floats)
  long long timeout_ns = 0;         // peer barrier wait bound (globaltimer ns); 0 = unbounded
};

struct StreamArgs {
  long long n4 = 0;                       // float4 slots per stream
  const float4* in[kStreamMaxIn] = {};
  float4* out[kStreamMaxOut] = {};
  double coef[kStreamMaxOut][kStreamMaxIn] = {};
  double da[kStreamMaxIn] = {}, db[kStreamMaxIn] = {};
  float* r = nullptr;                     // 1x1 dot output
  double* part = nullptr;                 // [gridDim.x] per-CTA partials
  unsigned* ticket = nullptr;             // last-CTA-done counter (self-resetting)
  PeerLinks peer;                         // row-/element-sharded runs: the dot finishes across ranks
  int ld_hint = 0;                        // element-wise loads: 0 plain ld.global.nc, 1 .L2::256B prefetch size
};

// Depth-2 single-pass matrix kernel (see mf_kernels.cu for the mapping).
struct MatrixArgs {
  long long m = 0, n = 0, ld = 0;   // rows, cols, row stride (floats)
  const float* M[2] = {};
  const float* u[2] = {};
  const float* v[2] = {};
  float* E = nullptr;               // stored rank-updated matrix (ger2 output)
  const float* xr[2] = {};          // row-reduction vectors (length n)
  float* yr[2] = {};                // row outputs (length m)
  double ar[2] = {1.0, 1.0};
  const float* xc[2] = {};          // column-reduction vectors (length m)
  float* yc[2] = {};                // column outputs (length n)
  double ac[2] = {1.0, 1.0};
  void* colpart = nullptr;          // [NCOL][RB][n] accumulator type
  void* rowpart = nullptr;          // [NROW][CB][m] accumulator type
  unsigned* bar = nullptr;          // grid barrier {count, generation} (peer path)
  unsigned* tilecnt = nullptr;      // tile-completion counters (local path; zeroed, self-resetting)
  int G = 1, NG = 1;                // column finalize: row bands per group, groups
  long long slice = 0;              // row-resident cluster: columns per CTA (0 = the kernel's chunk)
  int tile_fin = 0;                 // finish on tile counters: 0 none, 1 row outputs, 2 rows + columns
  int CB = 1, RB = 1, tiles = 1;    // column chunks, row bands, CB*RB
  PeerLinks peer;                   // nranks > 1: fused cross-GPU column reduction
  int l2_normal = 0;                // matrix loads: 0 evict-first L2 policy, 1 evict-normal
  int l2_ahead = 0;                 // row-resident chains: rows prefetched into L2 beyond the ring
  int rev = 0;                      // register-fed matrix kernel: each band's row batches bottom-up
  int fin_g = 0;                    // cross-CTA finalize lanes per slot: 0 = 8, or 16 | 32
  int dyn = 0;                      // tiles after blockIdx.x from counter bar[4] (bar[5] counts
                                    // exhausted CTAs; the last one resets both)
};

// Shape of a matrix-kernel instantiation.
struct MatrixShape {
  int nmat = 1, nrank = 0, store = 0, nrow = 0, ncol = 0;
  bool operator==(const MatrixShape&) const = default;
};

struct MatrixTuning {
  int K = 2;           // float4 column slots per thread (chunk width 1024*K columns)
  int R = 8;           // rows per reduction batch
  bool f64acc = false; // accumulate reductions in fp64
  int occupancy = 2;   // CTAs per SM targeted (register-fed variant)
  bool tma = true;     // TMA/mbarrier shared-memory ring (mf_matrix_tma.cu)
  int consumers = 256; // TMA variant: consumer threads per CTA (256 | 512)
  bool bulk_store = false;  // TMA variant, store shapes: E leaves through cp.async.bulk S2G
  int waves = 1;        // register-fed variant: tiles per co-resident CTA
  bool dynamic = false; // ... tiles after the first taken from a counter
};

// Launchers; return cudaSuccess or the launch error.  `sms` = SM count.
cudaError_t launch_stream(int nin, int nout, bool dot, const StreamArgs& a, int grid, int unroll,
                          cudaStream_t s);
// Stream grid.  Maps: ctas_per_sm = 0 (default) launches one CTA per block
// of 256*U float4, > 0 caps the grid at sms * ctas_per_sm (CTAs stride over
// blocks).  Dot kernels: persistent, sms * (ctas_per_sm or 4) CTAs.
int stream_grid(long long n4, int sms, int ctas_per_sm, int nin, int unroll, bool dot);
int stream_unroll_for(int nin, bool dot, int unroll);

// Fills CB/RB/tiles and returns the grid size (co-resident for the barrier).
cudaError_t matrix_config(const MatrixShape& sh, const MatrixTuning& t, long long m, long long n,
                          int sms, MatrixArgs* a, int* grid);
cudaError_t launch_matrix(const MatrixShape& sh, const MatrixTuning& t, const MatrixArgs& a,
                          int grid, cudaStream_t s);
bool matrix_shape_supported(const MatrixShape& sh);

// TMA-fed variant (mf_matrix_tma.cu).
cudaError_t matrix_tma_config(const MatrixShape& sh, const MatrixTuning& t, long long m,
                              long long n, int sms, MatrixArgs* a, int* grid);
cudaError_t launch_matrix_tma(const MatrixShape& sh, const MatrixTuning& t, const MatrixArgs& a,
                              int grid, cudaStream_t s);
int tma_stages(const MatrixShape& sh, const MatrixTuning& t);

// Row-resident chained reduction t = a*A x ; y = b*A^T t, one pass (mf_rowres.cu).
long long rowres_max_cols();
// variant: 1 stage-held rows, 2 register-held rows; rowres_variant maps 0 (auto)
int rowres_variant(int requested, long long n);
cudaError_t rowres_config(long long m, long long n, int sms, int variant, MatrixArgs* a, int* grid);
cudaError_t launch_rowres(const MatrixArgs& a, int grid, int variant, cudaStream_t s);
// Wide rows (16384 < n <= 131072): a cluster of ceil(n/16384) CTAs shares each
// row over distributed shared memory, then a cooperative finalize kernel
// combines the cluster bands' column partials (colpart [bands][n]).
// variant: 1 stage-held 16384-column slices, 2 register-held 16384-column
// slices, 3 register-held 8192-column slices (clusters up to 16);
// rowres_cluster_variant maps 0 (auto) to the default.
long long rowres_cluster_max_cols();
int rowres_cluster_variant(int requested, long long n);
int rowres_cluster_bands(long long m, long long n, int sms, int variant);  // co-resident clusters (0: unsupported)
cudaError_t launch_rowres_cluster(MatrixArgs a, int variant, int finalize_grid, cudaStream_t s);
bool tma_supported(const MatrixShape& sh, const MatrixTuning& t);  // fits a >= 2-stage ring
size_t matrix_acc_bytes(const MatrixTuning& t);

// Counter-based synthetic data (identical to oracle/mf_oracle.c
// mfo_hash_uniform): out[r*ld + c] = U(seed, (row0 + r) * ncols_global + c).
cudaError_t launch_generate(float* out, long long rows, long long cols, long long ld,
                            unsigned long long seed, long long row0, long long ncols_global,
                            cudaStream_t s);

}  // namespace mapfuse::b200
