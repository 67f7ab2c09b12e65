// mf_kernels.cu -- hand-written sm_100a kernels for fused map/reduce BLAS-1/2.
//
// Everything here is HBM-bound (<= 1 flop/byte): no tensor cores, no GEMM
// reshaping.  The design levers are the ones the roofline rewards:
//   * every matrix element is read from HBM exactly once per fused kernel
//     (128-bit, evict-first loads), every output written once;
//   * persistent grids sized to the SM count (148 on B200) x occupancy;
//   * intermediates stay in registers (the paper's register rule, section
//     3.2.3): a thread owns fixed column slots of the matrix for the whole
//     pass, so column reductions (sgemtv, A^T r) need no transpose through
//     shared memory -- the reference's stride-33 tile transpose
//     (proj/data/blas_library.mf:325-335) disappears;
//   * row reductions (sgemv, A p) are batched R rows at a time:
//     register partials -> warp butterfly (log2 R shuffles per value) ->
//     one shared-memory combine per batch;
//   * cross-CTA combination is deterministic: per-CTA partials land in L2,
//     one grid barrier (cooperative launch), then every CTA finalizes a
//     slice -- no float atomics, results are run-to-run reproducible
//     (the reference's VM is deterministic too, proj/include/mapfuse/vm.hpp:15).
#include "mf_kernels.cuh"
#include "mf_device.cuh"

#include <algorithm>
#include <cstdio>

namespace mapfuse::b200 {
namespace {

using namespace dev;

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// ---------------------------------------------------------------------------
// Depth-1 stream kernel.

template <int NIN, int NOUT, bool DOT>
struct StreamBody {
  __device__ __forceinline__ static void apply(const StreamArgs& a, const float4 (&v)[NIN],
                                               long long idx, double& acc) {
    float4 o[NOUT > 0 ? NOUT : 1];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double x[NIN];
#pragma unroll
      for (int k = 0; k < NIN; ++k) x[k] = (double)comp(v[k], c);
#pragma unroll
      for (int q = 0; q < NOUT; ++q) {
        // left-to-right, no contraction: sum_k coef_k * x_k as the reference
        // evaluates its fp64 formulas (blas.cpp:190, :258, :264)
        double s = __dmul_rn(a.coef[q][0], x[0]);
#pragma unroll
        for (int k = 1; k < NIN; ++k) s = __dadd_rn(s, __dmul_rn(a.coef[q][k], x[k]));
        set_comp(o[q], c, (float)s);
      }
      if constexpr (DOT) {
        double p = __dmul_rn(a.da[0], x[0]);
        double q2 = __dmul_rn(a.db[0], x[0]);
#pragma unroll
        for (int k = 1; k < NIN; ++k) {
          p = __dadd_rn(p, __dmul_rn(a.da[k], x[k]));
          q2 = __dadd_rn(q2, __dmul_rn(a.db[k], x[k]));
        }
        acc = fma(p, q2, acc);
      }
    }
#pragma unroll
    for (int q = 0; q < NOUT; ++q) st_stream(a.out[q] + idx, o[q]);
  }
};

// read-only 128-bit load; hint 1 asks L2 to fetch the whole 256 B sector group
__device__ __forceinline__ float4 ld_stream_in(const float4* p, int hint) {
  if (hint == 1) {
    float4 v;
    asm("ld.global.nc.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
        : "l"(p));
    return v;
  }
  return __ldg(p);
}

template <int NIN, int NOUT, bool DOT, int U>
__global__ void __launch_bounds__(kThreads) stream_kernel(StreamArgs a) {
  // Block-contiguous layout: block b = float4 [b*256*U, (b+1)*256*U) of every
  // stream; thread t loads b*256*U + u*256 + t, so a warp's U loads per input
  // are U contiguous 512 B runs and the CTA's footprint one contiguous
  // 4*U KB run per stream.  Default launch: one CTA per block (non-persistent,
  // the block scheduler issues blocks in address order, so the whole GPU
  // sweeps a compact, ordered wavefront); a capped grid strides over blocks.
  // Measured on B200 (tools/copy_probe.cu, y = f(x1..xk), 1 GiB per stream):
  // 1/2/3 inputs reach 6.9/7.0/7.2 TB/s this way against 6.0/6.3-6.7/6.7-7.0
  // for a persistent grid-stride sweep; plain ld.global.nc beats an
  // evict-first L2 policy by 2-5%.
  // With a dot, every CTA ends in a block reduction and a ticket on one
  // counter, so dot kernels keep a persistent grid (4 CTAs/SM) sweeping
  // grid-strided float4 slots with evict-first loads: AXPYDOT 2^24 runs
  // 41 us this way against 45-47 us block-contiguous (tools/sweep.py).
  double acc = 0.0;
  if constexpr (DOT) {
    const long long stride = (long long)gridDim.x * kThreads;
    long long i = (long long)blockIdx.x * kThreads + threadIdx.x;
    for (; i + (U - 1) * stride < a.n4; i += U * stride) {
      float4 v[U][NIN];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int k = 0; k < NIN; ++k) v[u][k] = ld_stream(a.in[k] + i + u * stride);
#pragma unroll
      for (int u = 0; u < U; ++u) StreamBody<NIN, NOUT, DOT>::apply(a, v[u], i + u * stride, acc);
    }
    for (; i < a.n4; i += stride) {
      float4 v[NIN];
#pragma unroll
      for (int k = 0; k < NIN; ++k) v[k] = ld_stream(a.in[k] + i);
      StreamBody<NIN, NOUT, DOT>::apply(a, v, i, acc);
    }
  } else {
    constexpr long long BLK = (long long)U * kThreads;
    const long long nblk = (a.n4 + BLK - 1) / BLK;
    for (long long b = blockIdx.x; b < nblk; b += gridDim.x) {
      const long long base = b * BLK + threadIdx.x;
      if (base + (U - 1) * kThreads < a.n4) {
        float4 v[U][NIN];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int k = 0; k < NIN; ++k) v[u][k] = ld_stream_in(a.in[k] + base + u * kThreads, a.ld_hint);
#pragma unroll
        for (int u = 0; u < U; ++u)
          StreamBody<NIN, NOUT, DOT>::apply(a, v[u], base + u * kThreads, acc);
      } else {
        for (long long i = base; i < a.n4; i += kThreads) {
          float4 v[NIN];
#pragma unroll
          for (int k = 0; k < NIN; ++k) v[k] = ld_stream_in(a.in[k] + i, a.ld_hint);
          StreamBody<NIN, NOUT, DOT>::apply(a, v, i, acc);
        }
      }
    }
  }
  if constexpr (DOT) {
    __shared__ double wsum[kWarps];
    __shared__ bool last;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < kWarps; ++w) s += wsum[w];
      a.part[blockIdx.x] = s;
      unsigned prev;  // acq_rel RMW chain: publishes this partial, acquires all earlier ones
      asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(prev) : "l"(a.ticket) : "memory");
      last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (last) {  // deterministic: fixed assignment of partials + fixed tree
      double s = 0.0;
#pragma unroll 8
      for (int b = threadIdx.x; b < (int)gridDim.x; b += kThreads) s += __ldcg(a.part + b);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = s;
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kWarps; ++w) t += wsum[w];
        if (a.peer.nranks > 1) {
          // Fused cross-rank reduction of the dot (sharded runs): every rank
          // puts its fp64 partial into slot `rank` of every peer's inbox over
          // NVLink, one system-scope arrival barrier, then each rank sums the
          // P partials in fixed rank order (deterministic, identical on all
          // ranks); a second barrier frees the inboxes for the next launch.
          const PeerLinks& pl = a.peer;
          for (int q = 0; q < pl.nranks; ++q) reinterpret_cast<double*>(pl.inbox[q])[pl.rank] = t;
          peer_signal_wait(pl, 0);
          const volatile double* mine = reinterpret_cast<const volatile double*>(pl.inbox[pl.rank]);
          t = 0.0;
          for (int q = 0; q < pl.nranks; ++q) t += mine[q];
          peer_signal_wait(pl, 1);
        }
        *a.r = (float)t;
        *a.ticket = 0u;  // ready for the next launch
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Depth-2 matrix kernel.
//
// Mapping: a CTA owns a tile = (column chunk cb) x (row band rb).  Thread t
// owns the K float4 column slots c_k = cb*4*T*K + 4*(t + T*k) for the whole
// band: the matching slices of the row-reduction vectors x (and of the rank
// vectors v1, v2) and the column-reduction accumulators live in registers.
// Rows stream through in batches of R: all R*K (x NMAT) 128-bit loads of a
// batch are issued before any arithmetic.

#ifdef MF_TIMELINE
// Diagnostic build only (tools/matrix_timeline.py): per-CTA %globaltimer
// stamps at kernel entry, end of the streaming loop, after the grid barrier
// and at exit; slot 4 holds the CTA's %smid.
__device__ unsigned long long g_mf_timeline[5][4096];
#define MF_STAMP(slot)                                                              \
  do {                                                                              \
    if (threadIdx.x == 0 && blockIdx.x < 4096) {                                    \
      unsigned long long t_;                                                        \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                        \
      g_mf_timeline[slot][blockIdx.x] = t_;                                         \
      if (slot == 0) {                                                              \
        unsigned sm_;                                                               \
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_));                            \
        g_mf_timeline[4][blockIdx.x] = sm_;                                         \
      }                                                                             \
    }                                                                               \
  } while (0)
#else
#define MF_STAMP(slot) \
  do {                 \
  } while (0)
#endif

template <int NMAT, int NRANK, bool STORE, int NROW, int NCOL, int K, int R, typename ACC>
__global__ void __launch_bounds__(kThreads, 2) matrix_kernel(MatrixArgs a) {
  MF_STAMP(0);
  constexpr int NV = (NROW > 0 ? NROW : 1) * R;
  constexpr long long C = 4LL * kThreads * K;
  __shared__ ACC red[2][kWarps][NV];
  __shared__ unsigned s_flag;
  __shared__ int s_next;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  ACC* colpart = static_cast<ACC*>(a.colpart);
  ACC* rowpart = static_cast<ACC*>(a.rowpart);
  int buf = 0;
  const unsigned long long pol = matrix_policy(a.l2_normal);

  // Tile schedule: the first tile is blockIdx.x; later ones round-robin, or
  // (a.dyn) from a counter -- the CTA that finishes first takes the next, so
  // the last wave is balanced.  A tile's partials depend only on the tile,
  // never on which CTA computed it, so results stay deterministic.  The next
  // index is fetched at the start of a tile and read at its end.
  int tile = blockIdx.x;
  if (a.dyn && tid == 0) s_next = (int)gridDim.x + (int)atomicAdd(a.bar + 4, 1u);
  for (; tile < a.tiles;) {
    const int cb = tile % a.CB, rb = tile / a.CB;
    const long long r0 = (long long)rb * a.m / a.RB, r1 = (long long)(rb + 1) * a.m / a.RB;
    long long col[K];
    bool ok[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      col[k] = (long long)cb * C + 4LL * (tid + kThreads * k);
      ok[k] = col[k] < a.n;
    }
    const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 xs[NROW > 0 ? NROW : 1][K];
    double vd[NRANK > 0 ? NRANK : 1][K][4];  // rank vectors, widened once per tile
#pragma unroll
    for (int k = 0; k < K; ++k) {
#pragma unroll
      for (int o = 0; o < NROW; ++o)
        xs[o][k] = ok[k] ? __ldg(reinterpret_cast<const float4*>(a.xr[o] + col[k])) : zero4;
#pragma unroll
      for (int q = 0; q < NRANK; ++q) {
        const float4 v4 = ok[k] ? __ldg(reinterpret_cast<const float4*>(a.v[q] + col[k])) : zero4;
#pragma unroll
        for (int e = 0; e < 4; ++e) vd[q][k][e] = (double)comp(v4, e);
      }
    }
    ACC cacc[NCOL > 0 ? NCOL : 1][K][4];
#pragma unroll
    for (int c = 0; c < NCOL; ++c)
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int e = 0; e < 4; ++e) cacc[c][k][e] = ACC(0);

    // a.rev: the band's batches bottom-up (the last rows a preceding kernel
    // stored are the ones still in L2)
    const long long nbatch = (r1 - r0 + R - 1) / R;
    for (long long bi = 0; bi < nbatch; ++bi) {
      const long long i0 = r0 + (a.rev ? nbatch - 1 - bi : bi) * R;
      double us[NRANK > 0 ? NRANK : 1][R];
      float xcs[NCOL > 0 ? NCOL : 1][R];
      float4 av[R][NMAT][K];
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        const long long i = i0 + rr;
        const bool rv = i < r1;
#pragma unroll
        for (int q = 0; q < NRANK; ++q) us[q][rr] = rv ? (double)__ldg(a.u[q] + i) : 0.0;
#pragma unroll
        for (int c = 0; c < NCOL; ++c) xcs[c][rr] = rv ? __ldg(a.xc[c] + i) : 0.f;
#pragma unroll
        for (int mt = 0; mt < NMAT; ++mt)
#pragma unroll
          for (int k = 0; k < K; ++k)
            av[rr][mt][k] = (rv && ok[k])
                                ? ld_policy(reinterpret_cast<const float4*>(a.M[mt] + i * a.ld + col[k]), pol)
                                : zero4;
      }
      ACC rp[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) rp[j] = ACC(0);
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
          float4 st;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            ACC ev[NMAT];
#pragma unroll
            for (int mt = 0; mt < NMAT; ++mt) ev[mt] = (ACC)comp(av[rr][mt][k], e);
            if constexpr (NRANK > 0) {
              // ger2 in fp64, rounded once: bit-identical to the reference's
              // B = A + u1 v1^T + u2 v2^T (blas.cpp:230-233)
              // u*v is exact in fp64, so fma(u, v, d) == d + u*v rounded once:
              // the same two fp64 roundings as the reference's expression.
              double d = (double)comp(av[rr][0][k], e);
#pragma unroll
              for (int q = 0; q < NRANK; ++q) d = fma(us[q][rr], vd[q][k][e], d);
              const float df = (float)d;
              if constexpr (STORE) set_comp(st, e, df);
              if constexpr (sizeof(ACC) == 4) ev[0] = df;
              else ev[0] = (ACC)d;
            }
#pragma unroll
            for (int o = 0; o < NROW; ++o) {
              const int mt = (NMAT == 2) ? o : 0;
              rp[o * R + rr] = fmacc<ACC>(ev[mt], (ACC)comp(xs[o][k], e), rp[o * R + rr]);
            }
#pragma unroll
            for (int c = 0; c < NCOL; ++c) {
              const int mt = (NMAT == 2) ? c : 0;
              cacc[c][k][e] = fmacc<ACC>(ev[mt], (ACC)xcs[c][rr], cacc[c][k][e]);
            }
          }
          if constexpr (STORE) {
            const long long i = i0 + rr;
            if (i < r1 && ok[k]) st_stream(reinterpret_cast<float4*>(a.E + i * a.ld + col[k]), st);
          }
        }
      }
      if constexpr (NROW > 0) {
        ACC wsum = butterfly<ACC, NV>(rp, lane);
        constexpr int group = 32 / NV;  // lanes holding the same value index
        if ((lane & (group - 1)) == 0) red[buf][warp][lane / group] = wsum;
        __syncthreads();
        if (tid < NV) {
          ACC s = red[buf][0][tid];
#pragma unroll
          for (int w = 1; w < kWarps; ++w) s += red[buf][w][tid];
          const int o = tid / R, rr = tid % R;
          const long long i = i0 + rr;
          if (i < r1) {
            if (a.CB == 1) a.yr[o][i] = (float)(a.ar[o] * (double)s);
            else rowpart[((long long)o * a.CB + cb) * a.m + i] = s;
          }
        }
        buf ^= 1;
      }
    }
    // column partials of this tile
#pragma unroll
    for (int c = 0; c < NCOL; ++c)
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (ok[k]) {
          ACC* dst = colpart + ((long long)c * a.RB + rb) * a.n + col[k];
#pragma unroll
          for (int e = 0; e < 4; ++e) dst[e] = cacc[c][k][e];
        }
    if (a.peer.nranks <= 1 && a.tile_fin > 0)  // single GPU: finish what this tile completes
      tile_done<NROW, NCOL, ACC>(a, cb, rb, C, r0, r1, tid, kThreads, &s_flag, [] { __syncthreads(); });
    if (a.dyn) {
      __syncthreads();  // s_next was written a whole tile ago
      tile = s_next;
      __syncthreads();
      if (tid == 0 && tile < a.tiles) s_next = (int)gridDim.x + (int)atomicAdd(a.bar + 4, 1u);
    } else {
      tile += gridDim.x;
    }
  }
  if (a.dyn && tid == 0) {  // the last CTA to run out of tiles resets the counters
    __threadfence();
    if (atomicAdd(a.bar + 5, 1u) == gridDim.x - 1) {
      atomicExch(a.bar + 4, 0u);
      atomicExch(a.bar + 5, 0u);
    }
  }

  if constexpr (NCOL > 0 || NROW > 0) {
    const bool need_rows = (NROW > 0) && a.CB > 1;
    MF_STAMP(1);
    if (NCOL == 0 && !need_rows) return;
    if (a.peer.nranks <= 1) {
      const bool rows_left = need_rows && a.tile_fin < 1, cols_left = NCOL > 0 && a.tile_fin < 2;
      if (!rows_left && !cols_left) return;  // everything finished on tile counters
      grid_barrier(a.bar);  // grid-wide fixed-order finalize
      finalize<NROW, NCOL, ACC>(a, tid, kThreads, rows_left, cols_left);
      return;
    }
    // row-sharded over several GPUs: cooperative grid, cross-rank finalize
    grid_barrier(a.bar);
    MF_STAMP(2);
    finalize_any<NROW, NCOL, ACC>(a, tid, kThreads);
    MF_STAMP(3);
  }
}

// ---------------------------------------------------------------------------
// Synthetic data (counter-based, matches oracle/mf_oracle.c).

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__global__ void generate_kernel(float* out, long long rows, long long cols, long long ld,
                                unsigned long long seed, long long row0, long long ncg) {
  const unsigned long long hs = splitmix64(seed);
  const long long total = rows * cols;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long r = t / cols, c = t % cols;
    const unsigned long long idx = (unsigned long long)(row0 + r) * (unsigned long long)ncg + c;
    const unsigned long long h = splitmix64(idx ^ hs);
    const unsigned k = (unsigned)(h >> 40);
    out[r * ld + c] = (float)k * (1.0f / 8388608.0f) - 1.0f;
  }
}

// ---------------------------------------------------------------------------
// Dispatch tables.

using MatrixFn = void (*)(MatrixArgs);

template <int NMAT, int NRANK, bool STORE, int NROW, int NCOL>
MatrixFn pick(const MatrixTuning& t) {
  // Register budget (<= 128 at 2 CTAs/SM): shapes carrying a second matrix
  // or the rank-2 update halve the rows per batch.
  // Rows per batch R is cut for the shapes carrying the rank-2 update (fp64
  // element math + the store path) or a second matrix.
  constexpr int R2 = (NRANK > 0) ? 2 : (NMAT == 2 ? 4 : 8);
  if (t.f64acc) return matrix_kernel<NMAT, NRANK, STORE, NROW, NCOL, 2, (R2 > 4 ? 4 : 2), double>;
  if (t.K == 4) return matrix_kernel<NMAT, NRANK, STORE, NROW, NCOL, 4, (R2 / 2), float>;
  return matrix_kernel<NMAT, NRANK, STORE, NROW, NCOL, 2, R2, float>;
}

MatrixFn matrix_fn(const MatrixShape& s, const MatrixTuning& t) {
  // The instantiations the planner can emit (SURVEY.md 2.2 kernel family T1).
  if (s == MatrixShape{1, 0, 0, 1, 0}) return pick<1, 0, false, 1, 0>(t);  // sgemv(s)
  if (s == MatrixShape{1, 0, 0, 0, 1}) return pick<1, 0, false, 0, 1>(t);  // sgemtv
  if (s == MatrixShape{1, 0, 0, 1, 1}) return pick<1, 0, false, 1, 1>(t);  // BiCGK
  if (s == MatrixShape{1, 0, 0, 2, 0}) return pick<1, 0, false, 2, 0>(t);  // 2x sgemv on A
  if (s == MatrixShape{1, 0, 0, 0, 2}) return pick<1, 0, false, 0, 2>(t);  // 2x sgemtv on A
  if (s == MatrixShape{1, 2, 1, 0, 1}) return pick<1, 2, true, 0, 1>(t);   // ger2+sgemtv
  if (s == MatrixShape{1, 2, 1, 0, 0}) return pick<1, 2, true, 0, 0>(t);   // ger2
  if (s == MatrixShape{2, 0, 0, 2, 0}) return pick<2, 0, false, 2, 0>(t);  // GESUMMV
  return nullptr;
}

template <int NIN, int NOUT, bool DOT>
cudaError_t go_stream(const StreamArgs& a, int grid, int unroll, cudaStream_t s) {
  unroll = stream_unroll_for(NIN, DOT, unroll);
  if (unroll >= 8) stream_kernel<NIN, NOUT, DOT, 8><<<grid, kThreads, 0, s>>>(a);
  else if (unroll >= 4) stream_kernel<NIN, NOUT, DOT, 4><<<grid, kThreads, 0, s>>>(a);
  else stream_kernel<NIN, NOUT, DOT, 2><<<grid, kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

// ---------------------------------------------------------------------------
int stream_unroll_for(int nin, bool dot, int unroll) {
  if (unroll > 0) return unroll;
  // block-contiguous maps: 2 float4 per thread per stream (tools/copy_probe.cu
  // B2 vs B4); grid-strided dot kernels: ~8 loads in flight per thread
  if (!dot) return 2;
  return nin <= 2 ? 8 : 2;
}

int stream_grid(long long n4, int sms, int ctas_per_sm, int nin, int unroll, bool dot) {
  if (dot) {
    const long long want = (long long)sms * (ctas_per_sm > 0 ? ctas_per_sm : 4);
    return (int)std::max(1LL, std::min(want, (n4 + kThreads - 1) / kThreads));
  }
  const long long blk = (long long)kThreads * stream_unroll_for(nin, dot, unroll);
  const long long nblk = std::max(1LL, (n4 + blk - 1) / blk);
  if (ctas_per_sm <= 0) return (int)std::min<long long>(nblk, 0x7fffffffLL);  // one CTA per block
  return (int)std::max(1LL, std::min(nblk, (long long)sms * ctas_per_sm));
}

cudaError_t launch_stream(int nin, int nout, bool dot, const StreamArgs& a, int grid, int unroll,
                          cudaStream_t s) {
#define MF_STREAM_CASE(I, O, D) \
  if (nin == I && nout == O && dot == D) return go_stream<I, O, D>(a, grid, unroll, s);
  MF_STREAM_CASE(1, 0, true)
  MF_STREAM_CASE(1, 1, false)
  MF_STREAM_CASE(1, 1, true)
  MF_STREAM_CASE(1, 2, false)
  MF_STREAM_CASE(1, 2, true)
  MF_STREAM_CASE(2, 0, true)
  MF_STREAM_CASE(2, 1, false)
  MF_STREAM_CASE(2, 1, true)
  MF_STREAM_CASE(2, 2, false)
  MF_STREAM_CASE(2, 2, true)
  MF_STREAM_CASE(3, 0, true)
  MF_STREAM_CASE(3, 1, false)
  MF_STREAM_CASE(3, 1, true)
  MF_STREAM_CASE(3, 2, false)
  MF_STREAM_CASE(3, 2, true)
  MF_STREAM_CASE(4, 0, true)
  MF_STREAM_CASE(4, 1, false)
  MF_STREAM_CASE(4, 1, true)
  MF_STREAM_CASE(4, 2, false)
  MF_STREAM_CASE(4, 2, true)
#undef MF_STREAM_CASE
  return cudaErrorNotSupported;
}

bool matrix_shape_supported(const MatrixShape& sh) {
  return matrix_fn(sh, MatrixTuning{}) != nullptr;
}

size_t matrix_acc_bytes(const MatrixTuning& t) { return t.f64acc ? 8 : 4; }

cudaError_t matrix_config(const MatrixShape& sh, const MatrixTuning& t, long long m, long long n,
                          int sms, MatrixArgs* a, int* grid) {
  MatrixFn fn = matrix_fn(sh, t);
  if (!fn) return cudaErrorNotSupported;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, 0);
  if (e != cudaSuccess) return e;
  per_sm = std::max(1, std::min(per_sm, t.occupancy));
  const int K = t.f64acc ? 2 : t.K;
  const long long C = 4LL * kThreads * K;
  const int CB = (int)((n + C - 1) / C);
  const long long G = (long long)sms * per_sm;  // co-resident CTAs
  // Row bands: the tile count (CB * RB) should be a whole multiple of the
  // grid (no tail wave) with at least ~8 rows per band.  Search grids from G
  // down to G/2 for one whose lcm with CB gives such a band count.
  long long RB = 0, g = 0;
  for (long long cand = G; cand >= std::max(1LL, G / 2) && RB == 0; --cand) {
    long long a0 = cand, b0 = CB;
    while (b0) { long long t0 = a0 % b0; a0 = b0; b0 = t0; }
    const long long l = cand / a0 * CB;  // lcm(cand, CB)
    const long long rb = l / CB;
    if (rb <= std::max(1LL, m / 8)) { RB = rb; g = cand; }
  }
  if (RB == 0) {  // small problems: fewer CTAs than SMs is fine
    RB = std::max(1LL, std::min(m / 4, std::max(1LL, G / CB)));
    g = std::min<long long>(G, (long long)CB * RB);
  }
  if (t.waves > 1) RB = std::min(RB * t.waves, std::max(RB, m / 8));
  const long long tiles = (long long)CB * RB;
  a->dyn = t.dynamic && tiles > g ? 1 : 0;
  a->CB = CB;
  a->RB = (int)RB;
  a->tiles = (int)tiles;
  *grid = (int)g;
  return cudaSuccess;
}

cudaError_t launch_matrix(const MatrixShape& sh, const MatrixTuning& t, const MatrixArgs& a,
                          int grid, cudaStream_t s) {
  MatrixFn fn = matrix_fn(sh, t);
  if (!fn) return cudaErrorNotSupported;
  // only the cross-GPU finalize needs a co-resident grid (grid barrier)
  const bool needs_barrier = a.peer.nranks > 1 ? (sh.ncol > 0 || (sh.nrow > 0 && a.CB > 1))
                                                : ((sh.ncol > 0 && a.tile_fin < 2) ||
                                                   (sh.nrow > 0 && a.CB > 1 && a.tile_fin < 1));
  MatrixArgs copy = a;
  void* args[] = {&copy};
  if (needs_barrier)
    return cudaLaunchCooperativeKernel((const void*)fn, dim3(grid), dim3(kThreads), args, 0, s);
  fn<<<grid, kThreads, 0, s>>>(copy);
  return cudaGetLastError();
}

#ifdef MF_TIMELINE
extern "C" int mf_debug_timeline(unsigned long long* host) {  // host: 5 x 4096; read + clear
  cudaError_t e = cudaMemcpyFromSymbol(host, g_mf_timeline, sizeof(g_mf_timeline));
  void* p = nullptr;
  if (e == cudaSuccess) e = cudaGetSymbolAddress(&p, g_mf_timeline);
  if (e == cudaSuccess) e = cudaMemset(p, 0, sizeof(g_mf_timeline));
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  return (int)e;
}
#endif

cudaError_t launch_generate(float* out, long long rows, long long cols, long long ld,
                            unsigned long long seed, long long row0, long long ncols_global,
                            cudaStream_t s) {
  long long total = rows * cols;
  int grid = (int)std::max(1LL, std::min<long long>((total + 255) / 256, 148LL * 16));
  generate_kernel<<<grid, 256, 0, s>>>(out, rows, cols, ld, seed, row0, ncols_global);
  return cudaGetLastError();
}

}  // namespace mapfuse::b200
