// mf_rowres.cu -- row-resident chained reduction: t = a*A x ; y = b*A^T t
// in ONE pass over A (ATAX in a single read).
//
// The paper (and SPEC.md:190) forbid fusing a reduction with the consumer of
// its result: on the paper's 32x32-tile kernels t_i is only complete after a
// global barrier, so ATAX reads A twice.  On B200 a whole row
// of a matrix with n <= 16384 fp32 columns (64 KB) fits in one stage of a
// shared-memory ring, so a CTA that owns entire rows completes t_i itself:
//   producer warp: cp.async.bulk of row i (up to 64 KB) into a 3-stage ring;
//   16 consumer warps: each thread owns K float4 column slots; pass 1 reads
//     them from the staged row and reduces A_i . x across the CTA (warp
//     shuffles + 16-way shared-memory combine, fixed order); pass 2 re-reads
//     the same slots and accumulates A_i^T t_i into register column
//     accumulators, then releases the stage;
//   column partials of every CTA's row band are combined after one grid
//   barrier (or across GPUs in-kernel, see mf_device.cuh finalize_any).
// Traffic: mn + 2n words instead of 2mn + m + 2n.  Planner mode "b200" only.
#include <algorithm>
#include <map>
#include <mutex>

#include "mf_device.cuh"
#include "mf_kernels.cuh"

namespace mapfuse::b200 {
namespace {

using namespace dev;

constexpr int kRrConsumers = 512;
constexpr int kRrWarps = kRrConsumers / 32;
constexpr int kRrThreads = kRrConsumers + 32;
constexpr int kRrStages = 3;

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void rr_mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count));
}
__device__ __forceinline__ void rr_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void rr_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void rr_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nRR_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra RR_WAIT_%=;\n}\n" ::"r"(smem_addr(b)),
      "r"(parity)
      : "memory");
}
// L2 prefetch of a global range (the bulk-copy engine, no shared memory):
// rows beyond the ring are on their way from DRAM while the ring's stages
// are still being consumed, so a stage refill reads L2
__device__ __forceinline__ void rr_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void rr_bulk(void* dst, const void* src, unsigned bytes,
                                        unsigned long long* bar, unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}

// The CTA total of one row's 16 warp partials, in every thread: lane l reads
// warp (l & 15)'s partial (one shared-memory wavefront per warp instead of 16
// broadcast reads), then a 16-lane xor butterfly.  Every warp computes the
// same fixed tree, so t_i is identical across the CTA (and across the
// stage-held and register-held variants).
template <int R>
__device__ __forceinline__ float combine_warps(const float (&red)[kRrWarps][R], int rr, int lane) {
  static_assert(kRrWarps == 16, "16-lane butterfly");
  float s = red[lane & 15][rr];
#pragma unroll
  for (int off = 8; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  return s;
}

template <int K, int R>
__global__ void __launch_bounds__(kRrThreads, 1) rowres_kernel(MatrixArgs a) {
  constexpr int C = 4 * kRrConsumers * K;  // columns covered by one CTA
  extern __shared__ __align__(128) unsigned char smem[];
  float* ring = reinterpret_cast<float*>(smem);  // stage = R rows of n floats (<= R*C)
  unsigned long long* full = reinterpret_cast<unsigned long long*>(ring + (size_t)kRrStages * R * C);
  unsigned long long* empty = full + kRrStages;
  __shared__ float red[2][kRrWarps][R];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long r0 = (long long)blockIdx.x * a.m / gridDim.x;
  const long long r1 = (long long)(blockIdx.x + 1) * a.m / gridDim.x;
  if (tid == 0) {
    for (int s = 0; s < kRrStages; ++s) {
      rr_mbar_init(&full[s], 1);
      rr_mbar_init(&empty[s], kRrWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kRrWarps) {
    if (lane == 0) {  // producer: R consecutive rows (contiguous) per stage
      const unsigned long long pol = evict_first_policy();
      int stage = 0;
      unsigned phase = 0;
      for (long long i = r0; i < r1; i += R) {
        const long long rows = (r1 - i) < R ? (r1 - i) : R;
        const long long bytes = rows * a.n * 4;
        // rows i + (stages + d) R, d < l2_ahead: into L2 now (the first
        // pass also covers the ring's own first stages' successors)
        for (int d = (i == r0 ? 0 : a.l2_ahead - 1); d >= 0 && d < a.l2_ahead; ++d) {
          const long long j = i + (long long)(kRrStages + d) * R;
          if (j < r1) {
            const long long pb = ((r1 - j) < R ? (r1 - j) : R) * a.n * 4;
            const char* ps = reinterpret_cast<const char*>(a.M[0] + j * a.ld);
            for (long long off = 0; off < pb; off += 16384)
              rr_prefetch_l2(ps + off, (unsigned)((pb - off) < 16384 ? (pb - off) : 16384));
          }
        }
        rr_wait(&empty[stage], phase ^ 1u);
        rr_expect_tx(&full[stage], (unsigned)bytes);
        // 16 KB pieces keep several bulk transfers in flight per stage
        const char* src = reinterpret_cast<const char*>(a.M[0] + i * a.ld);
        char* dst = reinterpret_cast<char*>(ring + (size_t)stage * R * C);
        for (long long off = 0; off < bytes; off += 16384) {
          const long long piece = (bytes - off) < 16384 ? (bytes - off) : 16384;
          rr_bulk(dst + off, src + off, (unsigned)piece, &full[stage], pol);
        }
        if (++stage == kRrStages) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
    __syncwarp();
  } else {
    int lcol[K];
    bool ok[K];
    float4 xs[K];
    float cacc[K][4];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      lcol[k] = 4 * (tid + kRrConsumers * k);
      ok[k] = lcol[k] < a.n;
      xs[k] = ok[k] ? __ldg(reinterpret_cast<const float4*>(a.xr[0] + lcol[k]))
                    : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int e = 0; e < 4; ++e) cacc[k][e] = 0.f;
    }
    int stage = 0, buf = 0;
    unsigned phase = 0;
    for (long long i0 = r0; i0 < r1; i0 += R) {
      rr_wait(&full[stage], phase);
      const float* rows = ring + (size_t)stage * R * C;
      const int nr = (r1 - i0) < R ? (int)(r1 - i0) : R;
      // pass 1: A_i . x for the stage's rows (rows stay in shared memory)
      float part[R];
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        part[rr] = 0.f;
        if (rr >= nr) continue;
        const float* row = rows + (size_t)rr * a.n;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          if (!ok[k]) continue;
          const float4 v = *reinterpret_cast<const float4*>(row + lcol[k]);
          part[rr] = fmaf(v.x, xs[k].x, part[rr]);
          part[rr] = fmaf(v.y, xs[k].y, part[rr]);
          part[rr] = fmaf(v.z, xs[k].z, part[rr]);
          part[rr] = fmaf(v.w, xs[k].w, part[rr]);
        }
      }
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) part[rr] += __shfl_xor_sync(0xffffffffu, part[rr], off);
        if (lane == 0) red[buf][warp][rr] = part[rr];
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kRrConsumers) : "memory");
      float ti[R];
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        const float s = combine_warps(red[buf], rr, lane);
        // t_i rounded to fp32 exactly as the unfused plan stores it
        ti[rr] = (float)(a.ar[0] * (double)s);
        if (tid == 0 && a.yr[0] && rr < nr) a.yr[0][i0 + rr] = ti[rr];
      }
      buf ^= 1;
      // pass 2: accumulate A_i^T t_i into the register column accumulators
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        if (rr >= nr) continue;
        const float* row = rows + (size_t)rr * a.n;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          if (!ok[k]) continue;
          const float4 v = *reinterpret_cast<const float4*>(row + lcol[k]);
          cacc[k][0] = fmaf(v.x, ti[rr], cacc[k][0]);
          cacc[k][1] = fmaf(v.y, ti[rr], cacc[k][1]);
          cacc[k][2] = fmaf(v.z, ti[rr], cacc[k][2]);
          cacc[k][3] = fmaf(v.w, ti[rr], cacc[k][3]);
        }
      }
      __syncwarp();
      if (lane == 0) rr_arrive(&empty[stage]);  // this warp is done with the stage
      if (++stage == kRrStages) {
        stage = 0;
        phase ^= 1u;
      }
    }
    float* colpart = static_cast<float*>(a.colpart);
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (ok[k]) {
        float* dst = colpart + (long long)blockIdx.x * a.n + lcol[k];
        *reinterpret_cast<float4*>(dst) = make_float4(cacc[k][0], cacc[k][1], cacc[k][2], cacc[k][3]);
      }
  }
  grid_barrier(a.bar);
  finalize_any<0, 1, float>(a, tid, kRrThreads);
}

// Register-held variant of rowres_kernel (option "rowres_variant" 2): 512
// threads, no producer warp (16 warps = 4 per SM sub-partition, so 128
// registers per thread).  Each thread loads its R x K float4 slots of the
// stage into registers once; after the CTA reduction's barrier (every warp
// has its copy) thread 0 refills that stage with the rows S stages ahead, so
// all S stages stream from HBM while the CTA finishes the rows, and pass 2
// runs from registers -- one shared-memory read per row instead of two.
template <int K, int R>
__global__ void __launch_bounds__(kRrConsumers, 1) rowres_reg_kernel(MatrixArgs a) {
  constexpr int C = 4 * kRrConsumers * K;
  constexpr int S = kRrStages;
  extern __shared__ __align__(128) unsigned char smem[];
  float* ring = reinterpret_cast<float*>(smem);  // stage = R rows of n floats (<= R*C)
  unsigned long long* full = reinterpret_cast<unsigned long long*>(ring + (size_t)S * R * C);
  __shared__ float red[2][kRrWarps][R];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long r0 = (long long)blockIdx.x * a.m / gridDim.x;
  const long long r1 = (long long)(blockIdx.x + 1) * a.m / gridDim.x;
  const long long ngroups = (r1 - r0 + R - 1) / R;
  const unsigned long long pol = evict_first_policy();
  auto refill = [&](long long g) {  // thread 0: rows [r0 + g R, +R) -> stage g % S
    const long long i = r0 + g * R;
    const long long rows = (r1 - i) < R ? (r1 - i) : R;
    const long long bytes = rows * a.n * 4;
    const int stage = (int)(g % S);
    rr_expect_tx(&full[stage], (unsigned)bytes);
    const char* src = reinterpret_cast<const char*>(a.M[0] + i * a.ld);
    char* dst = reinterpret_cast<char*>(ring + (size_t)stage * R * C);
    for (long long off = 0; off < bytes; off += 16384) {
      const long long piece = (bytes - off) < 16384 ? (bytes - off) : 16384;
      rr_bulk(dst + off, src + off, (unsigned)piece, &full[stage], pol);
    }
  };
  if (tid == 0) {
    for (int st = 0; st < S; ++st) rr_mbar_init(&full[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (long long g = 0; g < S && g < ngroups; ++g) refill(g);
  }
  __syncthreads();
  int lcol[K];
  bool ok[K];
  float4 xs[K];
  float cacc[K][4];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    lcol[k] = 4 * (tid + kRrConsumers * k);
    ok[k] = lcol[k] < a.n;
    xs[k] = ok[k] ? __ldg(reinterpret_cast<const float4*>(a.xr[0] + lcol[k])) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int e = 0; e < 4; ++e) cacc[k][e] = 0.f;
  }
  int buf = 0;
  for (long long g = 0; g < ngroups; ++g) {
    const int stage = (int)(g % S);
    const long long i0 = r0 + g * R;
    const int nr = (r1 - i0) < R ? (int)(r1 - i0) : R;
    rr_wait(&full[stage], (unsigned)((g / S) & 1));
    const float* rows = ring + (size_t)stage * R * C;
    float4 v[R][K];
    float part[R];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      part[rr] = 0.f;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        v[rr][k] = (rr < nr && ok[k]) ? *reinterpret_cast<const float4*>(rows + (size_t)rr * a.n + lcol[k])
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
        part[rr] = fmaf(v[rr][k].x, xs[k].x, part[rr]);
        part[rr] = fmaf(v[rr][k].y, xs[k].y, part[rr]);
        part[rr] = fmaf(v[rr][k].z, xs[k].z, part[rr]);
        part[rr] = fmaf(v[rr][k].w, xs[k].w, part[rr]);
      }
    }
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) part[rr] += __shfl_xor_sync(0xffffffffu, part[rr], off);
      if (lane == 0) red[buf][warp][rr] = part[rr];
    }
    __syncthreads();  // every warp holds the stage in registers: it is free
    if (tid == 0 && g + S < ngroups) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      refill(g + S);
    }
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const float s = combine_warps(red[buf], rr, lane);
      // t_i rounded to fp32 exactly as the unfused plan stores it
      const float ti = (float)(a.ar[0] * (double)s);
      if (tid == 0 && a.yr[0] && rr < nr) a.yr[0][i0 + rr] = ti;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        cacc[k][0] = fmaf(v[rr][k].x, ti, cacc[k][0]);
        cacc[k][1] = fmaf(v[rr][k].y, ti, cacc[k][1]);
        cacc[k][2] = fmaf(v[rr][k].z, ti, cacc[k][2]);
        cacc[k][3] = fmaf(v[rr][k].w, ti, cacc[k][3]);
      }
    }
    buf ^= 1;
  }
  float* colpart = static_cast<float*>(a.colpart);
#pragma unroll
  for (int k = 0; k < K; ++k)
    if (ok[k]) {
      float* dst = colpart + (long long)blockIdx.x * a.n + lcol[k];
      *reinterpret_cast<float4*>(dst) = make_float4(cacc[k][0], cacc[k][1], cacc[k][2], cacc[k][3]);
    }
  grid_barrier(a.bar);
  finalize_any<0, 1, float>(a, tid, kRrConsumers);
}

// ---------------------------------------------------------------------------
// Wide rows (n > 16384): a thread-block CLUSTER of CL CTAs holds one row
// between them -- CTA `crank` streams columns [crank*C, (crank+1)*C) of every
// row of the cluster's band through its own 3-stage TMA ring.  Per row:
//   pass 1: each CTA reduces its slice's A_i . x (warps -> shared combine)
//           and publishes the partial: a store into slot `crank` of every
//           cluster CTA's exchange buffer over distributed shared memory and
//           a remote mbarrier arrive (release.cluster) -- one row AHEAD of
//           its pass 2 (software pipelining), so waiting overlaps the next
//           row's reduction;
//   wait:   the local slot mbarrier (CL arrivals, acquire.cluster); every CTA
//           sums the CL partials in rank order -> t_i, bit-identical in the
//           whole cluster;
//   pass 2: A_i^T t_i into the register column accumulators of the slice.
// No cluster-wide barrier per row: CTAs run loosely coupled.  A CTA publishes
// row j+A (A = kRcAhead) only after it consumed row j-1, which needed every
// peer's row-(j-1) partial -- published only after all of that peer's
// threads finished row j-1-A-1 (named barrier inside the reduction) -- so the
// live slots span at most 2A+3 rows: kRcDepth = 8 slots never collide.  Column partials
// per cluster band go to colpart[cluster][n]; rowres_finalize_kernel sums them
// in fixed order (locally or across GPUs).  ATAX at 131072 columns: one read
// of A instead of two.
__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_id() {
  unsigned r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_count() {
  unsigned r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire;" ::: "memory"); }
__device__ __forceinline__ void cl_store(float* local_addr, unsigned target, float v) {
  unsigned remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_addr(local_addr)), "r"(target));
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(remote), "f"(v) : "memory");
}

template <int K>
__device__ __forceinline__ float rr_slice_dot(const float* row, const int (&lcol)[K], const bool (&ok)[K],
                                              const float4 (&xs)[K]) {
  float part = 0.f;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (!ok[k]) continue;
    const float4 v = *reinterpret_cast<const float4*>(row + lcol[k]);
    part = fmaf(v.x, xs[k].x, part);
    part = fmaf(v.y, xs[k].y, part);
    part = fmaf(v.z, xs[k].z, part);
    part = fmaf(v.w, xs[k].w, part);
  }
  return part;
}

__device__ __forceinline__ void cl_arrive_remote(unsigned long long* local_bar, unsigned target) {
  unsigned remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_addr(local_bar)), "r"(target));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
// One message instead of two: the value lands in the target CTA's slot and
// completes 4 transaction bytes on its slot mbarrier (st.async), so no
// release fence has to wait for the store's round trip before the arrive.
__device__ __forceinline__ void cl_store_async(float* local_addr, unsigned long long* local_bar,
                                               unsigned target, float v) {
  unsigned ra, rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_addr(local_addr)), "r"(target));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_addr(local_bar)), "r"(target));
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(ra),
               "r"(__float_as_uint(v)), "r"(rb)
               : "memory");
}

__device__ __forceinline__ void cl_wait_bar(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nCL_WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra CL_WAIT_%=;\n}\n" ::"r"(smem_addr(b)),
      "r"(parity)
      : "memory");
}

// Rows a CTA publishes ahead of the one it finishes.  1: the next row's
// slice was requested a whole row earlier, so its reduction rarely waits on
// memory (2 measured 1.55x slower: the slice two rows ahead was only just
// requested from HBM when its reduction needs it).
constexpr int kRcAhead = 1;
constexpr int kRcDepth = 8;  // exchange slots: > the largest lead (kRcAhead + 3 rows) of a CTA

template <int K, int CL, int S, bool XA>
__global__ void __launch_bounds__(kRrThreads, 1) rowres_cluster_kernel(MatrixArgs a) {
  constexpr int C = 4 * kRrConsumers * K;  // columns per CTA slice
  constexpr int kRrStages = S;
  extern __shared__ __align__(128) unsigned char smem[];
  float* ring = reinterpret_cast<float*>(smem);  // stage = one row slice (C floats)
  unsigned long long* full = reinterpret_cast<unsigned long long*>(ring + (size_t)kRrStages * C);
  unsigned long long* empty = full + kRrStages;
  __shared__ float red[2][kRrWarps];
  __shared__ float xch[kRcDepth][CL];                 // the cluster's partial dots, per row slot
  __shared__ __align__(8) unsigned long long xbar[kRcDepth];  // CL remote arrivals per slot
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned crank = cl_rank(), cid = cl_id(), ncl = cl_count();
  const long long W = a.slice > 0 ? a.slice : C;  // this CTA's column slice (<= C)
  const long long c0 = (long long)crank * W;
  const long long width = a.n - c0 < W ? (a.n - c0 > 0 ? a.n - c0 : 0) : W;
  const long long r0 = (long long)cid * a.m / ncl, r1 = (long long)(cid + 1) * a.m / ncl;
  const long long nrows = r1 - r0;
  if (tid == 0) {
    for (int s = 0; s < kRrStages; ++s) {
      rr_mbar_init(&full[s], 1);
      rr_mbar_init(&empty[s], kRrWarps);
    }
    for (int d = 0; d < kRcDepth; ++d) rr_mbar_init(&xbar[d], XA ? 1 : CL);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if constexpr (XA)  // arm every slot's first phase: CL partials of 4 bytes
      for (int d = 0; d < kRcDepth; ++d) rr_expect_tx(&xbar[d], CL * 4);
  }
  __syncthreads();
  cl_arrive();  // every CTA's barriers initialised before any remote arrive
  cl_wait();
  if (warp == kRrWarps) {
    if (lane == 0 && width > 0) {  // producer: row slices through a 3-stage TMA ring
      const unsigned long long pol = evict_first_policy();
      for (long long j = 0; j < nrows; ++j) {
        const int stage = (int)(j % kRrStages);
        rr_wait(&empty[stage], (unsigned)(((j / kRrStages) & 1) ^ 1u));
        const long long bytes = width * 4;
        rr_expect_tx(&full[stage], (unsigned)bytes);
        const char* src = reinterpret_cast<const char*>(a.M[0] + (r0 + j) * a.ld + c0);
        char* dst = reinterpret_cast<char*>(ring + (size_t)stage * C);
        for (long long off = 0; off < bytes; off += 16384) {
          const long long piece = (bytes - off) < 16384 ? (bytes - off) : 16384;
          rr_bulk(dst + off, src + off, (unsigned)piece, &full[stage], pol);
        }
      }
    }
    __syncwarp();
  } else {
    int lcol[K];
    bool ok[K];
    float4 xs[K];
    float cacc[K][4];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      lcol[k] = 4 * (tid + kRrConsumers * k);
      ok[k] = lcol[k] < width;
      xs[k] = ok[k] ? __ldg(reinterpret_cast<const float4*>(a.xr[0] + c0 + lcol[k]))
                    : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int e = 0; e < 4; ++e) cacc[k][e] = 0.f;
    }
    int rbuf = 0;
    auto cta_sum = [&](float part) {  // consumers only: named barrier 1
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
      if (lane == 0) red[rbuf][warp] = part;
      asm volatile("bar.sync 1, %0;" ::"n"(kRrConsumers) : "memory");
      float sum = red[rbuf][0];
#pragma unroll
      for (int w = 1; w < kRrWarps; ++w) sum += red[rbuf][w];
      rbuf ^= 1;
      return sum;
    };
    auto slice_partial = [&](long long j) {
      if (width <= 0) return cta_sum(0.f);
      rr_wait(&full[j % kRrStages], (unsigned)((j / kRrStages) & 1));
      return cta_sum(rr_slice_dot<K>(ring + (size_t)(j % kRrStages) * C, lcol, ok, xs));
    };
    auto publish = [&](long long j, float p) {  // my partial -> slot j of every cluster CTA
      if (tid < CL) {
        if constexpr (XA) {
          cl_store_async(&xch[j % kRcDepth][crank], &xbar[j % kRcDepth], (unsigned)tid, p);
        } else {
          cl_store(&xch[j % kRcDepth][crank], (unsigned)tid, p);
          cl_arrive_remote(&xbar[j % kRcDepth], (unsigned)tid);
        }
      }
    };
    for (long long j = 0; j < kRcAhead && j < nrows; ++j) publish(j, slice_partial(j));
    for (long long j = 0; j < nrows; ++j) {
      // software pipelining: the partials of the next kRcAhead rows go out
      // before waiting on this one (their slices are already in the ring)
      if (j + kRcAhead < nrows) publish(j + kRcAhead, slice_partial(j + kRcAhead));
      cl_wait_bar(&xbar[j % kRcDepth], (unsigned)((j / kRcDepth) & 1));
      float s32 = 0.f;  // slices combined in cluster rank order: identical in every CTA
#pragma unroll
      for (int q = 0; q < CL; ++q) s32 += xch[j % kRcDepth][q];
      if (XA && tid == 0) rr_expect_tx(&xbar[j % kRcDepth], CL * 4);  // arm the slot for row j + kRcDepth
      const float ti = (float)(a.ar[0] * (double)s32);  // t_i rounded to fp32 as the unfused plan stores it
      if (crank == 0 && tid == kRrConsumers - 1 && a.yr[0]) a.yr[0][r0 + j] = ti;  // not a publisher: its release must not wait on this store
      if (width > 0) {
        const float* row = ring + (size_t)(j % kRrStages) * C;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          if (!ok[k]) continue;
          const float4 v = *reinterpret_cast<const float4*>(row + lcol[k]);
          cacc[k][0] = fmaf(v.x, ti, cacc[k][0]);
          cacc[k][1] = fmaf(v.y, ti, cacc[k][1]);
          cacc[k][2] = fmaf(v.z, ti, cacc[k][2]);
          cacc[k][3] = fmaf(v.w, ti, cacc[k][3]);
        }
        __syncwarp();
        if (lane == 0) rr_arrive(&empty[j % kRrStages]);
      }
    }
    float* colpart = static_cast<float*>(a.colpart);
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (ok[k]) {
        float* dst = colpart + (long long)cid * a.n + c0 + lcol[k];
        *reinterpret_cast<float4*>(dst) = make_float4(cacc[k][0], cacc[k][1], cacc[k][2], cacc[k][3]);
      }
  }
  cl_arrive();  // no CTA leaves while a peer may still address its shared memory
  cl_wait();
}

// Register-held variant (no producer warp, 16 warps = 4 per SM sub-partition,
// so 128 registers per thread): every consumer loads its K float4 slots of
// row j from the stage into registers ONCE; after the CTA reduction of row j
// (whose named barrier proves every warp has its copy) thread 0 refills that
// stage with row j+S.  All S stages stream from HBM while row j waits for the
// cluster's t_j, and pass 2 runs from registers: one shared-memory read per
// row instead of two, no stage held across the exchange.  The exchange of
// row j is not overlapped with row j+1's reduction -- the ring keeps HBM busy
// instead.  Exchange slots: a CTA publishes row j only after it consumed row
// j-1 (all peers' row j-1 partials), so live slots span <= 3 rows.
constexpr int kRgThreads = kRrConsumers;

template <int K, int CL, int S, bool XA>
__global__ void __launch_bounds__(kRgThreads, 1) rowres_cluster_reg_kernel(MatrixArgs a) {
  constexpr int C = 4 * kRgThreads * K;  // columns per CTA slice
  extern __shared__ __align__(128) unsigned char smem[];
  float* ring = reinterpret_cast<float*>(smem);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(ring + (size_t)S * C);
  __shared__ float red[2][kRrWarps];
  __shared__ float xch[kRcDepth][CL];
  __shared__ __align__(8) unsigned long long xbar[kRcDepth];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned crank = cl_rank(), cid = cl_id(), ncl = cl_count();
  const long long c0 = (long long)crank * C;
  const long long width = a.n - c0 < C ? (a.n - c0 > 0 ? a.n - c0 : 0) : C;
  const long long r0 = (long long)cid * a.m / ncl, r1 = (long long)(cid + 1) * a.m / ncl;
  const long long nrows = r1 - r0;
  const unsigned long long pol = evict_first_policy();
  auto refill = [&](long long j) {  // thread 0: row j's slice -> stage j % S
    const int stage = (int)(j % S);
    const long long bytes = width * 4;
    rr_expect_tx(&full[stage], (unsigned)bytes);
    const char* src = reinterpret_cast<const char*>(a.M[0] + (r0 + j) * a.ld + c0);
    char* dst = reinterpret_cast<char*>(ring + (size_t)stage * C);
    for (long long off = 0; off < bytes; off += 16384) {
      const long long piece = (bytes - off) < 16384 ? (bytes - off) : 16384;
      rr_bulk(dst + off, src + off, (unsigned)piece, &full[stage], pol);
    }
  };
  if (tid == 0) {
    for (int s = 0; s < S; ++s) rr_mbar_init(&full[s], 1);
    for (int d = 0; d < kRcDepth; ++d) rr_mbar_init(&xbar[d], XA ? 1 : CL);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if constexpr (XA)  // arm every slot's first phase: CL partials of 4 bytes
      for (int d = 0; d < kRcDepth; ++d) rr_expect_tx(&xbar[d], CL * 4);
    if (width > 0)
      for (long long j = 0; j < S && j < nrows; ++j) refill(j);
  }
  __syncthreads();
  cl_arrive();  // every CTA's barriers initialised before any remote arrive
  cl_wait();
  const float* xp = a.xr[0] + c0 + 4 * tid;
  const float* sp = ring + 4 * tid;
  float4 xs[K];
  float cacc[K][4];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    xs[k] = (4 * tid + 4 * kRgThreads * k < width) ? __ldg(reinterpret_cast<const float4*>(xp + 4 * kRgThreads * k))
                                                  : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int e = 0; e < 4; ++e) cacc[k][e] = 0.f;
  }
  int rbuf = 0;
  for (long long j = 0; j < nrows; ++j) {
    float4 v[K];
    float part = 0.f;
    if (width > 0) {
      const int stage = (int)(j % S);
      rr_wait(&full[stage], (unsigned)((j / S) & 1));
      const float* row = sp + (size_t)stage * C;
#pragma unroll
      for (int k = 0; k < K; ++k)
        v[k] = (4 * tid + 4 * kRgThreads * k < width) ? *reinterpret_cast<const float4*>(row + 4 * kRgThreads * k)
                                                     : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        part = fmaf(v[k].x, xs[k].x, part);
        part = fmaf(v[k].y, xs[k].y, part);
        part = fmaf(v[k].z, xs[k].z, part);
        part = fmaf(v[k].w, xs[k].w, part);
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
    if (lane == 0) red[rbuf][warp] = part;
    __syncthreads();  // every warp holds row j in registers: its stage is free
    if (tid == 0 && width > 0 && j + S < nrows) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      refill(j + S);
    }
    if (tid < CL) {  // my partial -> slot j of every cluster CTA
      float sum = red[rbuf][0];
#pragma unroll
      for (int w = 1; w < kRrWarps; ++w) sum += red[rbuf][w];
      if constexpr (XA) {
        cl_store_async(&xch[j % kRcDepth][crank], &xbar[j % kRcDepth], (unsigned)tid, sum);
      } else {
        cl_store(&xch[j % kRcDepth][crank], (unsigned)tid, sum);
        cl_arrive_remote(&xbar[j % kRcDepth], (unsigned)tid);
      }
    }
    rbuf ^= 1;
    cl_wait_bar(&xbar[j % kRcDepth], (unsigned)((j / kRcDepth) & 1));
    float s32 = 0.f;  // slices combined in cluster rank order: identical in every CTA
#pragma unroll
    for (int q = 0; q < CL; ++q) s32 += xch[j % kRcDepth][q];
    if (XA && tid == 0) rr_expect_tx(&xbar[j % kRcDepth], CL * 4);  // arm the slot for row j + kRcDepth
    const float ti = (float)(a.ar[0] * (double)s32);  // t_i rounded to fp32 as the unfused plan stores it
    if (crank == 0 && tid == kRrConsumers - 1 && a.yr[0]) a.yr[0][r0 + j] = ti;  // not a publisher: its release must not wait on this store
    if (width > 0) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        cacc[k][0] = fmaf(v[k].x, ti, cacc[k][0]);
        cacc[k][1] = fmaf(v[k].y, ti, cacc[k][1]);
        cacc[k][2] = fmaf(v[k].z, ti, cacc[k][2]);
        cacc[k][3] = fmaf(v[k].w, ti, cacc[k][3]);
      }
    }
  }
  float* colpart = static_cast<float*>(a.colpart) + (long long)cid * a.n + c0 + 4 * tid;
#pragma unroll
  for (int k = 0; k < K; ++k)
    if (4 * tid + 4 * kRgThreads * k < width)
      *reinterpret_cast<float4*>(colpart + 4 * kRgThreads * k) =
          make_float4(cacc[k][0], cacc[k][1], cacc[k][2], cacc[k][3]);
  cl_arrive();  // no CTA leaves while a peer may still address its shared memory
  cl_wait();
}

// colpart[RB][n] -> y (fixed band order; across GPUs when a.peer is set).
__global__ void __launch_bounds__(256) rowres_finalize_kernel(MatrixArgs a) {
  finalize_any<0, 1, float>(a, threadIdx.x, 256);
}

using RrFn = void (*)(MatrixArgs);

// stage ~64 KB: R rows of the CTA's column span
// variant 1: stage-held rows (producer warp, two shared-memory reads per row);
// 2: register-held rows (rowres_reg_kernel)
RrFn rowres_fn(long long n, int variant) {
  const bool reg = variant == 2;
  if (n <= 4LL * kRrConsumers * 2) return reg ? rowres_reg_kernel<2, 4> : rowres_kernel<2, 4>;
  if (n <= 4LL * kRrConsumers * 4) return reg ? rowres_reg_kernel<4, 2> : rowres_kernel<4, 2>;
  if (n <= 4LL * kRrConsumers * 8) return reg ? rowres_reg_kernel<8, 1> : rowres_kernel<8, 1>;
  return nullptr;
}
int rowres_threads(int variant) { return variant == 2 ? kRrConsumers : kRrThreads; }

size_t rowres_smem(long long n) {
  (void)n;
  return (size_t)kRrStages * 16384 * 4 + 2 * kRrStages * 8 + 128;  // R*C = 16384 floats
}

using RcFn = void (*)(MatrixArgs);

// Cluster variants (option "rowres_cluster"):
//   1: 16384-column slices (K = 8), clusters of ceil(n/16384) <= 8, 3 x 64 KB
//      stages, row j+1 reduced ahead of row j's exchange (stage-held);
//   2: the same slices, register-held rows with early stage release;
//   3: 8192-column slices (K = 4), clusters of ceil(n/8192) <= 16
//      (non-portable above 8), 6 x 32 KB stages, register-held rows;
//   4, 5, 6: variants 1, 2, 3 with the exchange sent as st.async messages;
//   7: variant 4 with the cluster size that keeps the most SMs streaming
//      (slices of ceil(n / CL) columns, up to 16384; n = 131072: 9 CTAs of
//      14592 columns, 135 SMs, instead of 8 of 16384 on 120).
struct RcVariant {
  int K, stages;
  bool reg;
  long long slice() const { return 4LL * kRrConsumers * K; }
  size_t smem() const { return (size_t)stages * slice() * 4 + 2 * (size_t)stages * 8 + 128; }
  int threads() const { return reg ? kRgThreads : kRrThreads; }
};

RcVariant rc_variant(int v) {
  switch (v) {
    case 1:
    case 4:
    case 7: return {8, 3, false};
    case 3:
    case 6: return {4, 6, true};
    default: return {8, 3, true};
  }
}

template <int CL>
RcFn rc_fn_cl(int variant) {
  switch (variant) {
    case 1:
    case 4:
      if constexpr (CL <= 8)
        return variant == 1 ? rowres_cluster_kernel<8, CL, 3, false> : rowres_cluster_kernel<8, CL, 3, true>;
      return nullptr;
    case 7: return rowres_cluster_kernel<8, CL, 3, true>;
    case 3: return rowres_cluster_reg_kernel<4, CL, 6, false>;
    case 6: return rowres_cluster_reg_kernel<4, CL, 6, true>;
    case 5:
      if constexpr (CL <= 8) return rowres_cluster_reg_kernel<8, CL, 3, true>;
      return nullptr;
    default:
      if constexpr (CL <= 8) return rowres_cluster_reg_kernel<8, CL, 3, false>;
      return nullptr;
  }
}

RcFn rowres_cluster_fn(int variant, int cl) {
  switch (cl) {
    case 1: return rc_fn_cl<1>(variant);  // rows of n <= 16384 on the cluster kernels' code path
    case 2: return rc_fn_cl<2>(variant);
    case 3: return rc_fn_cl<3>(variant);
    case 4: return rc_fn_cl<4>(variant);
    case 5: return rc_fn_cl<5>(variant);
    case 6: return rc_fn_cl<6>(variant);
    case 7: return rc_fn_cl<7>(variant);
    case 8: return rc_fn_cl<8>(variant);
    case 9: return rc_fn_cl<9>(variant);
    case 10: return rc_fn_cl<10>(variant);
    case 11: return rc_fn_cl<11>(variant);
    case 12: return rc_fn_cl<12>(variant);
    case 13: return rc_fn_cl<13>(variant);
    case 14: return rc_fn_cl<14>(variant);
    case 15: return rc_fn_cl<15>(variant);
    case 16: return rc_fn_cl<16>(variant);
    default: return nullptr;
  }
}

bool rc_attrs(RcFn fn, const RcVariant& var, int cl) {
  if (cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)var.smem()) !=
      cudaSuccess)
    return false;
  return cl <= 8 ||
         cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
}

// variant 7: the cluster size in [ceil(n / 16384), 16] with the most
// co-resident CTAs (ties: the smaller cluster), per device and n
int rc_best_cluster(long long n, long long* slice) {
  static std::mutex mu;
  static std::map<std::pair<int, long long>, std::pair<int, long long>> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({dev, n});
  if (it != cache.end()) {
    *slice = it->second.second;
    return it->second.first;
  }
  const RcVariant var = rc_variant(7);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int best = 0, best_cov = 0;
  long long best_w = 0;
  for (int cl = (int)((n + var.slice() - 1) / var.slice()); cl <= 16; ++cl) {
    const long long w = ((n + cl - 1) / cl + 31) / 32 * 32;
    if (w > var.slice() || (long long)(cl - 1) * w >= n) continue;  // every CTA gets columns
    RcFn fn = rowres_cluster_fn(7, cl);
    if (!fn || !rc_attrs(fn, var, cl)) continue;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(var.threads());
    cfg.dynamicSmemBytes = var.smem();
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(cl * std::max(1, sms / cl));
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, (const void*)fn, &cfg) != cudaSuccess) continue;
    if (nc * cl > best_cov) {
      best_cov = nc * cl;
      best = cl;
      best_w = w;
    }
  }
  cudaGetLastError();
  cache[{dev, n}] = {best, best_w};
  *slice = best_w;
  return best;
}

// fills cfg (grid left to the caller) for variant v at n columns; nullptr if
// unsupported.  *slice_out: columns per CTA (0 = the variant's full slice).
RcFn rc_setup(int v, long long n, cudaLaunchConfig_t* cfg, cudaLaunchAttribute* attr, int* cl_out,
              long long* slice_out = nullptr) {
  const RcVariant var = rc_variant(v);
  long long slice = 0;
  const int cl = v == 7 ? rc_best_cluster(n, &slice) : (int)((n + var.slice() - 1) / var.slice());
  if (slice_out) *slice_out = slice;
  RcFn fn = rowres_cluster_fn(v, cl);
  if (!fn) return nullptr;
  if (cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)var.smem()) !=
      cudaSuccess)
    return nullptr;
  if (cl > 8 &&
      cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
    return nullptr;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg->blockDim = dim3(var.threads());
  cfg->dynamicSmemBytes = var.smem();
  cfg->attrs = attr;
  cfg->numAttrs = 1;
  *cl_out = cl;
  return fn;
}

}  // namespace

long long rowres_max_cols() { return 4LL * kRrConsumers * 8; }
long long rowres_cluster_max_cols() { return 16 * 8192; }

// auto (tools/rowres_sweep.py on B200, profiles/r02_rowres_variants.txt):
// the st.async exchange (variants 4 / 5; 1 / 2 / 3 took 13.8 / 20.5 / 31.7 ms
// at 131072^2).  Register-held rows (5) against stage-held (4), by cluster
// size: 2 CTAs 669 vs 607 us (32768^2), 3: -2.4%, 4: -6.5% (65536^2 2.33 vs
// 2.49 ms), 5: -6.3%, 6: +2%, 7: -3.9%, 8: -3% to +0.5% -- so 5 from clusters
// of 3 up, 4 for clusters of 2.  Both sum in the same order (bit-identical).
int rowres_cluster_variant(int requested, long long n) {
  if (requested >= 1 && requested <= 7) return requested;
  return (n + rowres_max_cols() - 1) / rowres_max_cols() >= 3 ? 5 : 4;
}

cudaError_t launch_rowres_cluster(MatrixArgs a, int variant, int finalize_grid, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  int cl = 0;
  RcFn fn = rc_setup(variant, a.n, &cfg, attr, &cl, &a.slice);
  if (!fn) return cudaErrorNotSupported;
  cfg.stream = s;
  cfg.gridDim = dim3(cl * a.RB);  // a.RB = rowres_cluster_bands(m, n, sms): colpart is [RB][n]
  cudaError_t e = cudaLaunchKernelEx(&cfg, fn, a);
  if (e != cudaSuccess) return e;
  void* args[] = {&a};
  return cudaLaunchCooperativeKernel((const void*)rowres_finalize_kernel, dim3(finalize_grid), dim3(256),
                                     args, 0, s);
}

int rowres_cluster_bands(long long m, long long n, int sms, int variant) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  int cl = 0;
  RcFn fn = rc_setup(variant, n, &cfg, attr, &cl);
  if (!fn) return 0;
  cfg.gridDim = dim3(cl * std::max(1, sms / cl));
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, (const void*)fn, &cfg) != cudaSuccess) return 0;
  nclusters = std::min(nclusters, std::max(1, sms / cl));  // the SM budget (option max_sms)
  return std::max(1, std::min<int>(nclusters, (int)std::min<long long>(m, 1 << 20)));
}

// auto: register-held rows only for n <= 4096 (R = 4 rows per stage), where
// they measured faster (tools/rowres_sweep.py, profiles/r02_rowres_variants.txt:
// ATAX 131072x4096 330.8 vs 340.0 us); from 8192 columns up the stage-held
// kernel's one-row lookahead wins (16384^2: 169.1 vs 174.1 us)
int rowres_variant(int requested, long long n) {
  if (requested == 1 || requested == 2) return requested;
  return n <= 4LL * kRrConsumers * 2 ? 2 : 1;
}

cudaError_t rowres_config(long long m, long long n, int sms, int variant, MatrixArgs* a, int* grid) {
  RrFn fn = rowres_fn(n, variant);
  if (!fn) return cudaErrorNotSupported;
  const size_t smem = rowres_smem(n);
  cudaError_t e = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const long long g = std::max(1LL, std::min<long long>(sms, m));
  a->CB = 1;
  a->RB = (int)g;  // one row band per CTA: colpart is [grid][n]
  a->tiles = (int)g;
  *grid = (int)g;
  return cudaSuccess;
}

cudaError_t launch_rowres(const MatrixArgs& a, int grid, int variant, cudaStream_t s) {
  RrFn fn = rowres_fn(a.n, variant);
  if (!fn) return cudaErrorNotSupported;
  MatrixArgs copy = a;
  void* args[] = {&copy};
  return cudaLaunchCooperativeKernel((const void*)fn, dim3(grid), dim3(rowres_threads(variant)), args,
                                     rowres_smem(a.n), s);
}

}  // namespace mapfuse::b200
