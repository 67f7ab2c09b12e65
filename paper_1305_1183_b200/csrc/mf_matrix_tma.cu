// mf_matrix_tma.cu -- the depth-2 matrix kernel with a TMA-fed shared-memory
// ring (the default matrix path).
//
// Same math and thread->column ownership as the register-fed variant in
// mf_kernels.cu, but the matrix rows never pass through registers on their
// way on-chip: one producer warp streams each row segment of the CTA's column
// chunk into an S-stage shared-memory ring with cp.async.bulk (the TMA bulk
// engine, SASS UBLKCP), completion tracked by mbarrier transaction counts.
// Eight consumer warps read their float4 column slots out of the ring,
// update the column accumulators held in registers, and reduce row partials.
// Bytes in flight per SM are set by the ring depth (up to ~190 KB), not by
// register pressure -- which is what the rank-2-update shape (GEMVER's
// ger2 + sgemtv, which also streams B back out) needs to reach HBM roofline.
//
// Per stage: R rows x NMAT matrices x C = 4*256*K floats, plus the R-float
// slices of the column-reduction vectors and rank vectors u_q (bulk-copied
// too; R >= 4 keeps every copy a multiple of 16 bytes).
#include <algorithm>

#include "mf_device.cuh"
#include "mf_kernels.cuh"

namespace mapfuse::b200 {
namespace {

using namespace dev;

// consumer threads per CTA: 256 (8 warps) or 512 (16 warps) + 1 producer warp

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "MF_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra MF_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar, unsigned long long policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
template <int NC>
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(NC) : "memory");
}

// Bands start on multiples of R so every per-row vector slice is 16-byte
// aligned for the bulk engine.
__device__ __forceinline__ void band(const MatrixArgs& a, int rb, int R, long long* r0,
                                     long long* r1) {
  const long long units = a.m / R;
  *r0 = (long long)rb * units / a.RB * R;
  *r1 = (long long)(rb + 1) * units / a.RB * R;
}

// BULK (store shapes): the updated matrix E is written back into the stage it
// was read from and leaves through the bulk engine (cp.async.bulk S2G, one
// copy per row segment) instead of per-thread st.global; the stage returns to
// the producer once its store has read shared memory.
template <int NMAT, int NRANK, bool STORE, int NROW, int NCOL, int K, int R, typename ACC, int NC,
          bool BULK = false>
__global__ void __launch_bounds__(NC + 32, 1) matrix_tma_kernel(MatrixArgs a, int S) {
  static_assert(!BULK || STORE, "bulk stores need a stored matrix");
  constexpr int kConsumers = NC;
  constexpr int kConsumerWarps = NC / 32;
  constexpr int kTmaThreads = NC + 32;
  static_assert(R >= 4, "bulk copies of per-row slices need R >= 4");
  constexpr int NV = (NROW > 0 ? NROW : 1) * R;
  constexpr int C = 4 * kConsumers * K;
  constexpr long long kMatStage = (long long)NMAT * R * C;  // floats
  extern __shared__ __align__(128) unsigned char smem[];
  float* sm_mat = reinterpret_cast<float*>(smem);
  float* sm_xc = sm_mat + S * kMatStage;
  float* sm_u = sm_xc + S * NCOL * R;
  unsigned long long* full =
      reinterpret_cast<unsigned long long*>(sm_u + ((S * NRANK * R + 1) & ~1));
  unsigned long long* empty = full + S;
  __shared__ ACC red[2][kConsumerWarps][NV];
  __shared__ unsigned s_flag;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], BULK ? 1 : kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ---------------- producer warp: one elected lane drives the bulk engine
    if (lane == 0) {
      const unsigned long long pol = matrix_policy(a.l2_normal);
      unsigned long long keep;  // per-row vector slices are re-read by every column chunk
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
      int stage = 0;
      unsigned phase = 0;
      for (int tile = blockIdx.x; tile < a.tiles; tile += gridDim.x) {
        const int cb = tile % a.CB, rb = tile / a.CB;
        const long long c0 = (long long)cb * C;
        const unsigned row_bytes = (unsigned)(min((long long)C, a.n - c0) * 4);
        long long r0, r1;
        band(a, rb, R, &r0, &r1);
        for (long long i0 = r0; i0 < r1; i0 += R) {
          mbar_wait(&empty[stage], phase ^ 1u);
          const unsigned tx = R * NMAT * row_bytes + (NCOL + NRANK) * R * 4;
          mbar_expect_tx(&full[stage], tx);
          float* dst = sm_mat + stage * kMatStage;
#pragma unroll
          for (int mt = 0; mt < NMAT; ++mt)
#pragma unroll
            for (int rr = 0; rr < R; ++rr)
              bulk_g2s(dst + (mt * R + rr) * C, a.M[mt] + (i0 + rr) * a.ld + c0, row_bytes,
                       &full[stage], pol);
#pragma unroll
          for (int c = 0; c < NCOL; ++c)
            bulk_g2s(sm_xc + (stage * NCOL + c) * R, a.xc[c] + i0, R * 4, &full[stage], keep);
#pragma unroll
          for (int q = 0; q < NRANK; ++q)
            bulk_g2s(sm_u + (stage * NRANK + q) * R, a.u[q] + i0, R * 4, &full[stage], keep);
          if (++stage == S) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------- consumer warps
    ACC* colpart = static_cast<ACC*>(a.colpart);
    ACC* rowpart = static_cast<ACC*>(a.rowpart);
    int stage = 0;
    unsigned phase = 0;
    int buf = 0;
    int prev_stage = -1;  // BULK: stage whose store may still be reading shared memory
    for (int tile = blockIdx.x; tile < a.tiles; tile += gridDim.x) {
      const int cb = tile % a.CB, rb = tile / a.CB;
      long long r0, r1;
      band(a, rb, R, &r0, &r1);
      const unsigned row_bytes = (unsigned)(min((long long)C, a.n - (long long)cb * C) * 4);
      int lcol[K];
      long long col[K];
      bool ok[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        lcol[k] = 4 * (tid + kConsumers * k);
        col[k] = (long long)cb * C + lcol[k];
        ok[k] = col[k] < a.n;
      }
      const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
      float4 xs[NROW > 0 ? NROW : 1][K];
      double vd[NRANK > 0 ? NRANK : 1][K][4];
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

      for (long long i0 = r0; i0 < r1; i0 += R) {
        mbar_wait(&full[stage], phase);
        float* st_mat = sm_mat + stage * kMatStage;
        ACC rp[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) rp[j] = ACC(0);
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          float xcs[NCOL > 0 ? NCOL : 1];
          double us[NRANK > 0 ? NRANK : 1];
#pragma unroll
          for (int c = 0; c < NCOL; ++c) xcs[c] = sm_xc[(stage * NCOL + c) * R + rr];
#pragma unroll
          for (int q = 0; q < NRANK; ++q) us[q] = (double)sm_u[(stage * NRANK + q) * R + rr];
#pragma unroll
          for (int k = 0; k < K; ++k) {
            if (!ok[k]) continue;
            float4 av[NMAT];
#pragma unroll
            for (int mt = 0; mt < NMAT; ++mt)
              av[mt] = *reinterpret_cast<const float4*>(st_mat + (mt * R + rr) * C + lcol[k]);
            float4 st;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              ACC ev[NMAT];
#pragma unroll
              for (int mt = 0; mt < NMAT; ++mt) ev[mt] = (ACC)comp(av[mt], e);
              if constexpr (NRANK > 0) {
                double d = (double)comp(av[0], e);
#pragma unroll
                for (int q = 0; q < NRANK; ++q) d = fma(us[q], vd[q][k][e], d);
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
                cacc[c][k][e] = fmacc<ACC>(ev[mt], (ACC)xcs[c], cacc[c][k][e]);
              }
            }
            if constexpr (BULK)
              *reinterpret_cast<float4*>(st_mat + rr * C + lcol[k]) = st;  // in place: own slots
            else if constexpr (STORE)
              st_stream(reinterpret_cast<float4*>(a.E + (i0 + rr) * a.ld + col[k]), st);
          }
        }
        if constexpr (BULK) {
          // every consumer's E values are in the stage: make them visible to
          // the async proxy, then one thread sends the R row segments out and
          // returns the PREVIOUS stage once its store has read shared memory
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          consumers_sync<NC>();
          if (tid == 0) {
#pragma unroll
            for (int rr = 0; rr < R; ++rr)
              bulk_s2g(a.E + (i0 + rr) * a.ld + (long long)cb * C, st_mat + rr * C, row_bytes);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            if (prev_stage >= 0) {
              asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
              mbar_arrive(&empty[prev_stage]);
            }
            prev_stage = stage;
          }
        } else {
          // stage fully consumed by this warp -> release it to the producer
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[stage]);
        }
        if (++stage == S) {
          stage = 0;
          phase ^= 1u;
        }
        if constexpr (NROW > 0) {
          ACC wsum = butterfly<ACC, NV>(rp, lane);
          constexpr int group = 32 / NV;
          if ((lane & (group - 1)) == 0) red[buf][warp][lane / group] = wsum;
          consumers_sync<NC>();
          if (tid < NV) {
            ACC s = red[buf][0][tid];
#pragma unroll
            for (int w = 1; w < kConsumerWarps; ++w) s += red[buf][w][tid];
            const int o = tid / R, rr = tid % R;
            const long long i = i0 + rr;
            if (a.CB == 1) a.yr[o][i] = (float)(a.ar[o] * (double)s);
            else rowpart[((long long)o * a.CB + cb) * a.m + i] = s;
          }
          buf ^= 1;
        }
      }
#pragma unroll
      for (int c = 0; c < NCOL; ++c)
#pragma unroll
        for (int k = 0; k < K; ++k)
          if (ok[k]) {
            ACC* dst = colpart + ((long long)c * a.RB + rb) * a.n + col[k];
#pragma unroll
            for (int e = 0; e < 4; ++e) dst[e] = cacc[c][k][e];
          }
      if (a.peer.nranks <= 1 && a.tile_fin > 0)  // single GPU: consumers finish what this tile completes
        tile_done<NROW, NCOL, ACC>(a, cb, rb, C, r0, r1, tid, kConsumers, &s_flag,
                                   [] { consumers_sync<NC>(); });
    }
    if constexpr (BULK) {
      // E must be in global memory before the grid barrier / kernel end
      if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  }

  if constexpr (NCOL > 0 || NROW > 0) {
    const bool need_rows = (NROW > 0) && a.CB > 1;
    if (NCOL == 0 && !need_rows) return;
    if (a.peer.nranks <= 1) {
      const bool rows_left = need_rows && a.tile_fin < 1, cols_left = NCOL > 0 && a.tile_fin < 2;
      if (!rows_left && !cols_left) return;  // everything finished on tile counters
      grid_barrier(a.bar);  // grid-wide fixed-order finalize
      finalize<NROW, NCOL, ACC>(a, tid, kTmaThreads, rows_left, cols_left);
      return;
    }
    // row-sharded over several GPUs: cooperative grid, cross-rank finalize
    grid_barrier(a.bar);
    finalize_any<NROW, NCOL, ACC>(a, tid, kTmaThreads);
  }
}

using TmaFn = void (*)(MatrixArgs, int);

template <int NMAT, int NRANK, bool STORE, int NROW, int NCOL>
TmaFn pick_tma(const MatrixTuning& t) {
  if (t.f64acc) return matrix_tma_kernel<NMAT, NRANK, STORE, NROW, NCOL, 2, 4, double, 256>;
  if constexpr (STORE) {
    if (t.bulk_store && t.consumers == 512)
      return matrix_tma_kernel<NMAT, NRANK, STORE, NROW, NCOL, 2, 4, float, 512, true>;
    if (t.bulk_store && t.K != 4)
      return matrix_tma_kernel<NMAT, NRANK, STORE, NROW, NCOL, 2, 4, float, 256, true>;
  }
  if (t.consumers == 512) return matrix_tma_kernel<NMAT, NRANK, STORE, NROW, NCOL, 2, 4, float, 512>;
  if (t.K == 4) return matrix_tma_kernel<NMAT, NRANK, STORE, NROW, NCOL, 4, 4, float, 256>;
  return matrix_tma_kernel<NMAT, NRANK, STORE, NROW, NCOL, 2, 4, float, 256>;
}

TmaFn tma_fn(const MatrixShape& s, const MatrixTuning& t) {
  if (s == MatrixShape{1, 0, 0, 1, 0}) return pick_tma<1, 0, false, 1, 0>(t);
  if (s == MatrixShape{1, 0, 0, 0, 1}) return pick_tma<1, 0, false, 0, 1>(t);
  if (s == MatrixShape{1, 0, 0, 1, 1}) return pick_tma<1, 0, false, 1, 1>(t);
  if (s == MatrixShape{1, 0, 0, 2, 0}) return pick_tma<1, 0, false, 2, 0>(t);
  if (s == MatrixShape{1, 0, 0, 0, 2}) return pick_tma<1, 0, false, 0, 2>(t);
  if (s == MatrixShape{1, 2, 1, 0, 1}) return pick_tma<1, 2, true, 0, 1>(t);
  if (s == MatrixShape{1, 2, 1, 0, 0}) return pick_tma<1, 2, true, 0, 0>(t);
  if (s == MatrixShape{2, 0, 0, 2, 0}) return pick_tma<2, 0, false, 2, 0>(t);
  return nullptr;
}

// columns one CTA covers (the chunk width) and threads per CTA
long long tma_chunk(const MatrixTuning& t) {
  if (t.f64acc) return 4LL * 256 * 2;
  if (t.consumers == 512) return 4LL * 512 * 2;
  return 4LL * 256 * (t.K == 4 ? 4 : 2);
}
int tma_threads(const MatrixTuning& t) { return (!t.f64acc && t.consumers == 512 ? 512 : 256) + 32; }

size_t tma_stage_bytes(const MatrixShape& s, const MatrixTuning& t) {
  const size_t R = 4, C = (size_t)tma_chunk(t);
  return (size_t)s.nmat * R * C * 4 + (size_t)(s.ncol + s.nrank) * R * 4;
}

}  // namespace

int tma_stages(const MatrixShape& sh, const MatrixTuning& t) {
  const size_t budget = 200 * 1024;
  return (int)std::max<size_t>(2, std::min<size_t>(8, budget / tma_stage_bytes(sh, t)));
}

bool tma_supported(const MatrixShape& sh, const MatrixTuning& t) {
  return tma_fn(sh, t) != nullptr && 2 * tma_stage_bytes(sh, t) <= 200 * 1024;
}

size_t tma_smem_bytes(const MatrixShape& sh, const MatrixTuning& t) {
  const int S = tma_stages(sh, t);
  return (size_t)S * tma_stage_bytes(sh, t) + 16 + 2 * (size_t)S * 8 + 128;
}

cudaError_t matrix_tma_config(const MatrixShape& sh, const MatrixTuning& t, long long m,
                              long long n, int sms, MatrixArgs* a, int* grid) {
  TmaFn fn = tma_fn(sh, t);
  if (!fn) return cudaErrorNotSupported;
  const size_t smem = tma_smem_bytes(sh, t);
  cudaError_t e = cudaFuncSetAttribute((const void*)fn,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, tma_threads(t), smem);
  if (e != cudaSuccess) return e;
  per_sm = std::max(1, per_sm);
  const long long C = tma_chunk(t);
  const int CB = (int)((n + C - 1) / C);
  const long long G = (long long)sms * per_sm;
  const long long units = m / 4;  // R = 4 row units
  long long RB = 0, g = 0;
  for (long long cand = G; cand >= std::max(1LL, G / 2) && RB == 0; --cand) {
    long long a0 = cand, b0 = CB;
    while (b0) {
      long long t0 = a0 % b0;
      a0 = b0;
      b0 = t0;
    }
    const long long rb = cand / a0;  // lcm(cand, CB) / CB
    if (rb <= std::max(1LL, units / 2)) {
      RB = rb;
      g = cand;
    }
  }
  if (RB == 0) {
    RB = std::max(1LL, std::min(units, std::max(1LL, G / CB)));
    g = std::min<long long>(G, (long long)CB * RB);
  }
  a->CB = CB;
  a->RB = (int)RB;
  a->tiles = (int)(CB * RB);
  *grid = (int)g;
  return cudaSuccess;
}

cudaError_t launch_matrix_tma(const MatrixShape& sh, const MatrixTuning& t, const MatrixArgs& a,
                              int grid, cudaStream_t s) {
  TmaFn fn = tma_fn(sh, t);
  if (!fn) return cudaErrorNotSupported;
  const size_t smem = tma_smem_bytes(sh, t);
  int S = tma_stages(sh, t);
  const bool needs_barrier = a.peer.nranks > 1 ? (sh.ncol > 0 || (sh.nrow > 0 && a.CB > 1))
                                                : ((sh.ncol > 0 && a.tile_fin < 2) ||
                                                   (sh.nrow > 0 && a.CB > 1 && a.tile_fin < 1));
  MatrixArgs copy = a;
  void* args[] = {&copy, &S};
  if (needs_barrier)
    return cudaLaunchCooperativeKernel((const void*)fn, dim3(grid), dim3(tma_threads(t)), args,
                                       smem, s);
  fn<<<grid, tma_threads(t), smem, s>>>(copy, S);
  return cudaGetLastError();
}

}  // namespace mapfuse::b200
