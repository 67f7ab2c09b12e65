// mf_device.cuh -- device helpers shared by the sm_100a kernel families.
#pragma once

#include <cuda_runtime.h>

#include "mf_kernels.cuh"

namespace mapfuse::b200 {
namespace dev {

// Streaming 128-bit load: bypass L1 allocation and mark the L2 line
// evict-first -- matrix and stream operands are touched exactly once.
__device__ __forceinline__ unsigned long long evict_first_policy() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Matrix-operand L2 policy: evict-first (default) or evict-normal, chosen per
// launch (MatrixArgs::l2_normal; option "matrix_l2_normal").
__device__ __forceinline__ unsigned long long matrix_policy(int normal) {
  unsigned long long p;
  if (normal) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ float4 ld_policy(const float4* p, unsigned long long pol) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(evict_first_policy()));
  return v;
}

__device__ __forceinline__ void st_stream(float4* p, float4 v) {
  asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

__device__ __forceinline__ float comp(const float4& v, int c) {
  return c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w));
}
__device__ __forceinline__ void set_comp(float4& v, int c, float x) {
  if (c == 0) v.x = x;
  else if (c == 1) v.y = x;
  else if (c == 2) v.z = x;
  else v.w = x;
}

// ---------------------------------------------------------------------------
// Grid barrier for co-resident (cooperatively launched) grids.  bar[0] counts
// arrivals, bar[1] is a generation number; self-resetting across launches.
// One acq_rel RMW per CTA (publishes the CTA's writes -- ordered before it by
// bar.sync -- and, for the last arriver, acquires everyone's), one release
// increment of the generation, acquire polling: two L2 round trips on the
// critical path instead of the four a fence-based barrier takes.
__device__ __forceinline__ void grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned g, arrived;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(arrived) : "l"(bar) : "memory");
    if (arrived == gridDim.x - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(bar) : "memory");
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 1) : "memory");
    } else {
      unsigned cur;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar + 1) : "memory");
        if (cur != g) break;
        __nanosleep(32);
      }
    }
  }
  __syncthreads();
}

// Butterfly reduce-scatter: NV values per lane (NV power of two <= 32) ->
// lane l ends up holding the warp total of value index (l >> (5 - log2 NV)).
template <typename T, int NV>
__device__ __forceinline__ T butterfly(T (&v)[NV], int lane) {
  static_assert((NV & (NV - 1)) == 0 && NV <= 32, "NV must be a power of two <= 32");
  int width = NV;
  int mask = 16;
#pragma unroll
  for (int step = 0; (NV >> step) > 1; ++step) {
    const int half = (NV >> step) >> 1;
    const bool hi = (lane & mask) != 0;
#pragma unroll
    for (int j = 0; j < half; ++j) {
      T send = hi ? v[j] : v[j + half];
      T keep = hi ? v[j + half] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, mask);
    }
    mask >>= 1;
    width >>= 1;
  }
  T r = v[0];
  for (; mask > 0; mask >>= 1) r += __shfl_xor_sync(0xffffffffu, r, mask);
  return r;
}

template <typename ACC>
__device__ __forceinline__ ACC fmacc(ACC a, ACC b, ACC c);
template <>
__device__ __forceinline__ float fmacc<float>(float a, float b, float c) {
  return fmaf(a, b, c);
}
template <>
__device__ __forceinline__ double fmacc<double>(double a, double b, double c) {
  return fma(a, b, c);
}

// Cross-CTA partial sums, parallel and deterministic: G lanes cooperate on
// one float4 slot (lane g of the group sums partials g, g+G, g+2G, ... in
// order; a fixed xor butterfly combines the G), so a slot with 148 partials
// costs ~19 dependent L2 loads per lane at G = 8 instead of 148.  G is 8;
// option "finalize_group" fixes 16 or 32 (measured equal or slower on every
// shape, profiles/r02_finalize_group.txt: the finalize is not bound by that
// chain).  A launch-constant G keeps the summation order, and the result, the
// same on every launch.  Loop trip counts are warp-uniform so every shuffle
// has all 32 lanes.
constexpr int kFinGroup = 8;

__device__ __forceinline__ int fin_group(int fixed) {
  return (fixed == 16 || fixed == 32) ? fixed : kFinGroup;
}

template <typename ACC>
__device__ __forceinline__ void group_sum4(const ACC* base, long long stride, int count, bool valid,
                                           int glane, int G, ACC (&t)[4]) {
  t[0] = t[1] = t[2] = t[3] = ACC(0);
  if (valid)
#pragma unroll 4
    for (int b = glane; b < count; b += G) {
      const ACC* q = base + (long long)b * stride;
#pragma unroll
      for (int e = 0; e < 4; ++e) t[e] += __ldcg(q + e);
    }
  for (int off = G / 2; off > 0; off >>= 1)
#pragma unroll
    for (int e = 0; e < 4; ++e) t[e] += __shfl_xor_sync(0xffffffffu, t[e], off);
}

// Visits slots [0, total) in warp-uniform rounds, G lanes per slot;
// f(slot, valid, glane, lead).
template <typename F>
__device__ __forceinline__ void for_each_slot_grouped(long long total, int tid, int nthreads, int G, F&& f) {
  const int lane = tid & 31;
  const int glane = lane % G;
  const long long warps_total = (long long)gridDim.x * (nthreads / 32);
  const long long gwarp = (long long)blockIdx.x * (nthreads / 32) + tid / 32;
  const int per_warp = 32 / G;
  for (long long first = gwarp * per_warp; first < total; first += warps_total * per_warp) {
    const long long slot = first + lane / G;
    f(slot, slot < total, glane, glane == 0 && slot < total);
  }
}

// Cross-CTA finalize after the grid barrier: column outputs sum the RB band
// partials, row outputs (when the row was split over CB column chunks) sum
// the CB chunk partials -- fixed order, so results are reproducible.
template <int NROW, int NCOL, typename ACC>
__device__ __forceinline__ void finalize(const MatrixArgs& a, int tid, int nthreads, bool do_rows = true,
                                         bool do_cols = true) {
  const ACC* colpart = static_cast<const ACC*>(a.colpart);
  const ACC* rowpart = static_cast<const ACC*>(a.rowpart);
  const bool need_rows = (NROW > 0) && a.CB > 1 && do_rows;
  const long long n4 = a.n / 4, m4 = a.m / 4;
  const long long col_slots = do_cols ? (long long)NCOL * n4 : 0;
  const long long total = col_slots + (need_rows ? (long long)NROW * m4 : 0);
  const int G = fin_group(a.fin_g);
  for_each_slot_grouped(total, tid, nthreads, G, [&](long long s, bool valid, int glane, bool lead) {
    ACC t[4];
    // invalid lanes only occur past the last slot: follow that region's branch
    // so each warp's shuffles stay convergent (col_slots is a multiple of 8,
    // a warp holds 32 / G <= 4 slots)
    const bool col_branch = valid ? (s < col_slots) : !need_rows;
    if (col_branch) {
      const int c = valid ? (int)(s / n4) : 0;
      const long long j = valid ? (s % n4) * 4 : 0;
      group_sum4<ACC>(colpart + (long long)c * a.RB * a.n + j, a.n, a.RB, valid && NCOL > 0, glane, G, t);
      if (lead && NCOL > 0) {
        float4 o = make_float4((float)(a.ac[c] * (double)t[0]), (float)(a.ac[c] * (double)t[1]),
                               (float)(a.ac[c] * (double)t[2]), (float)(a.ac[c] * (double)t[3]));
        *reinterpret_cast<float4*>(a.yc[c] + j) = o;
      }
    } else {
      const long long q = valid ? s - col_slots : 0;
      const int o = (int)(q / m4);
      const long long i = (q % m4) * 4;
      group_sum4<ACC>(rowpart + (long long)o * a.CB * a.m + i, a.m, a.CB, valid, glane, G, t);
      if (lead) {
        float4 r = make_float4((float)(a.ar[o] * (double)t[0]), (float)(a.ar[o] * (double)t[1]),
                               (float)(a.ar[o] * (double)t[2]), (float)(a.ar[o] * (double)t[3]));
        *reinterpret_cast<float4*>(a.yr[o] + i) = r;
      }
    }
  });
}

// ---------------------------------------------------------------------------
// Tile-completion finalize (single GPU, option "matrix_tile_finalize": 1 row
// outputs, 2 row and column outputs; 0, the default, finishes both after the
// grid barrier).  When a CTA has written the partials of tile (cb, rb) it
// counts the tile on arrival counters (MatrixArgs::tilecnt; acq_rel RMW after
// a CTA barrier, so the whole CTA's partials are published with it); the LAST
// arriver of a group finishes that group's sum in a fixed order, so results
// do not depend on arrival order:
//   [cb*NG + g]        tiles of column chunk cb in row-band group g (G bands):
//                      last arriver sums the group's column partials into the
//                      group's first slot (or straight into y when NG == 1);
//   [CB*NG + cb]       finished groups of chunk cb: last sums the NG group
//                      partials into y;
//   [CB*NG + CB + rb]  finished column chunks of row band rb (row outputs
//                      split over CB > 1 chunks): last sums the CB row partials.
// Counters reset themselves (the last arriver stores 0).  Measured on B200
// (DESIGN.md 5): in one-wave grids every chunk completes at the same moment,
// and the grid barrier plus the grid-wide 8-lane finalize is as fast or
// faster -- the last-arriver sums run on one CTA per chunk or band.
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

template <typename ACC>
__device__ __forceinline__ void add4_cg(ACC (&t)[4], const ACC* q) {
  if constexpr (sizeof(ACC) == 4) {
    const float4 v = __ldcg(reinterpret_cast<const float4*>(q));
    t[0] += v.x;
    t[1] += v.y;
    t[2] += v.z;
    t[3] += v.w;
  } else {
    const double2 v0 = __ldcg(reinterpret_cast<const double2*>(q));
    const double2 v1 = __ldcg(reinterpret_cast<const double2*>(q) + 1);
    t[0] += v0.x;
    t[1] += v0.y;
    t[2] += v1.x;
    t[3] += v1.y;
  }
}

template <typename ACC>
__device__ __forceinline__ void store4(ACC* q, const ACC (&t)[4]) {
  if constexpr (sizeof(ACC) == 4) {
    *reinterpret_cast<float4*>(q) = make_float4(t[0], t[1], t[2], t[3]);
  } else {
    reinterpret_cast<double2*>(q)[0] = make_double2(t[0], t[1]);
    reinterpret_cast<double2*>(q)[1] = make_double2(t[2], t[3]);
  }
}

// Column slots of chunk [c0, c0 + w): sum partial slots first, first + step,
// ... (count of them) in that order; to_y: scale by ac and write y, else
// write the sum back into slot `first`.
template <int NCOL, typename ACC>
__device__ __forceinline__ void sum_column_slots(const MatrixArgs& a, long long c0, long long w, int first,
                                                 int step, int count, bool to_y, int tid, int nthr) {
  ACC* colpart = static_cast<ACC*>(a.colpart);
  const long long nslot = w / 4;
#pragma unroll
  for (int c = 0; c < NCOL; ++c) {
    for (long long sl = tid; sl < nslot; sl += nthr) {
      const long long j = c0 + 4 * sl;
      ACC t[4] = {ACC(0), ACC(0), ACC(0), ACC(0)};
      const ACC* q = colpart + ((long long)c * a.RB + first) * a.n + j;
      const long long stride = (long long)step * a.n;
#pragma unroll 8
      for (int p = 0; p < count; ++p) add4_cg<ACC>(t, q + p * stride);
      if (to_y) {
        *reinterpret_cast<float4*>(a.yc[c] + j) =
            make_float4((float)(a.ac[c] * (double)t[0]), (float)(a.ac[c] * (double)t[1]),
                        (float)(a.ac[c] * (double)t[2]), (float)(a.ac[c] * (double)t[3]));
      } else {
        store4<ACC>(colpart + ((long long)c * a.RB + first) * a.n + j, t);
      }
    }
  }
}

// Called by the nthr threads that wrote tile (cb, rb) (the whole CTA, or the
// TMA kernel's consumer warps), right after its column partials; [r0, r1) are
// the band's rows, C the chunk width.  sync() is a barrier over those threads.
template <int NROW, int NCOL, typename ACC, typename Sync>
__device__ __forceinline__ void tile_done(const MatrixArgs& a, int cb, int rb, long long C, long long r0,
                                          long long r1, int tid, int nthr, unsigned* s_flag, Sync sync) {
  const bool need_rows = (NROW > 0) && a.CB > 1 && a.tile_fin >= 1;
  const bool cols = NCOL > 0 && a.tile_fin >= 2;
  if (!cols && !need_rows) return;
  unsigned* tc = a.tilecnt;
  const int G = a.G, NG = a.NG, g = rb / G;
  sync();  // every partial of this tile is written
  if (tid == 0) {
    unsigned f = 0;
    if (cols) {
      const unsigned gsize = (unsigned)min(G, a.RB - g * G);
      unsigned* cnt = tc + (long long)cb * NG + g;
      if (atom_add_acq_rel(cnt, 1u) == gsize - 1) {
        *reinterpret_cast<volatile unsigned*>(cnt) = 0u;
        f |= 1u;
      }
    }
    if (need_rows) {
      unsigned* cnt = tc + (long long)a.CB * NG + a.CB + rb;
      if (atom_add_acq_rel(cnt, 1u) == (unsigned)a.CB - 1) {
        *reinterpret_cast<volatile unsigned*>(cnt) = 0u;
        f |= 2u;
      }
    }
    *s_flag = f;
  }
  sync();
  const unsigned f = *s_flag;
  if (NCOL > 0 && (f & 1u)) {
    const long long c0 = (long long)cb * C;
    const long long w = min(C, a.n - c0);
    const int gsize = min(G, a.RB - g * G);
    sum_column_slots<NCOL, ACC>(a, c0, w, g * G, 1, gsize, NG == 1, tid, nthr);
    if (NG > 1) {
      sync();  // this group's sum is written
      if (tid == 0) {
        unsigned* cnt = tc + (long long)a.CB * NG + cb;
        unsigned f2 = 0;
        if (atom_add_acq_rel(cnt, 1u) == (unsigned)NG - 1) {
          *reinterpret_cast<volatile unsigned*>(cnt) = 0u;
          f2 = 1u;
        }
        *s_flag = f2;
      }
      sync();
      if (*s_flag) sum_column_slots<NCOL, ACC>(a, c0, w, 0, G, NG, true, tid, nthr);
    }
  }
  if (NROW > 0 && need_rows && (f & 2u)) {
    const ACC* rowpart = static_cast<const ACC*>(a.rowpart);
    const long long nr = r1 - r0;
    for (long long q = tid; q < (long long)NROW * nr; q += nthr) {
      const int o = (int)(q / nr);
      const long long i = r0 + q % nr;
      ACC t = ACC(0);
      const ACC* p = rowpart + (long long)o * a.CB * a.m + i;
#pragma unroll 8
      for (int c = 0; c < a.CB; ++c) t += __ldcg(p + (long long)c * a.m);
      a.yr[o][i] = (float)(a.ar[o] * (double)t);
    }
  }
  sync();  // s_flag is reused by the next tile
}

// ---------------------------------------------------------------------------
// Fused cross-rank finalize for column outputs (after the local grid barrier).
// Phase A: every rank sums its band partials and writes the local column sums
//          of slice s straight into rank s's inbox (remote stores over NVLink).
// Phase B: after a system-scope arrival barrier, rank s reduces its slice over
//          the P sources in fixed rank order (deterministic, identical on every
//          rank), scales, writes its own y and its outbox.
// Phase C: after a second barrier, every rank pulls the other slices from the
//          owners' outboxes into its y.  Traffic per rank = 2(P-1)/P * n
//          floats, the ring all-reduce volume, with no extra kernel launch.
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Bounded wait: a peer that never arrives (a rank that crashed or launched a
// different kernel) makes the barrier give up after timeout_ns of wall time,
// raise the group's error word and let the kernel finish -- the host gets a
// clear error from mf_peer_group_check instead of a hung GPU or a trap that
// poisons the context.
__device__ __forceinline__ void peer_signal_wait(const PeerLinks& pl, int which) {
  // one thread of block 0, after a grid barrier: all CTAs' writes are done
  __threadfence_system();
  for (int s = 0; s < pl.nranks; ++s) atomicAdd_system(pl.flags[s] + which, 1u);
  const unsigned target = pl.epoch * (unsigned)pl.nranks;
  const unsigned long long t0 = global_ns();
  volatile unsigned* mine = pl.flags[pl.rank] + which;
  while (*mine < target) {
    __nanosleep(128);
    if (pl.timeout_ns > 0 && (long long)(global_ns() - t0) > pl.timeout_ns) {
      atomicExch_system(pl.flags[pl.rank] + kPeerErrorWord, 1u + (unsigned)which);
      break;
    }
  }
  __threadfence_system();
}

template <int NCOL, typename ACC>
__device__ __forceinline__ void finalize_columns_peers(const MatrixArgs& a, int tid, int nthreads) {
  const PeerLinks& pl = a.peer;
  const ACC* colpart = static_cast<const ACC*>(a.colpart);
  const long long n4 = a.n / 4, gstride = (long long)gridDim.x * nthreads;
  const long long slice4 = n4 / pl.nranks;  // n / P is a multiple of 4 (n % 32 == 0, P <= 8)
  const long long P = pl.nranks;
  // Phase A: local sums -> owner's inbox[c][rank][j]
  const int G = fin_group(a.fin_g);
  for_each_slot_grouped((long long)NCOL * n4, tid, nthreads, G,
                        [&](long long s, bool valid, int glane, bool lead) {
    const int c = valid ? (int)(s / n4) : 0;
    const long long j4 = valid ? s % n4 : 0, j = j4 * 4;
    ACC t[4];
    group_sum4<ACC>(colpart + (long long)c * a.RB * a.n + j, a.n, a.RB, valid, glane, G, t);
    if (!lead) return;
    const int owner = (int)min(j4 / slice4, P - 1);
    float4 v = make_float4((float)t[0], (float)t[1], (float)t[2], (float)t[3]);
    float* dst = pl.inbox[owner] + ((long long)c * P + pl.rank) * pl.n_cap + j;
    *reinterpret_cast<float4*>(dst) = v;
  });
  grid_barrier(a.bar);
  if (blockIdx.x == 0 && tid == 0) peer_signal_wait(pl, 0);
  grid_barrier(a.bar);
  // Phase B: reduce my slice in fixed source order
  const long long lo4 = slice4 * pl.rank, hi4 = (pl.rank == P - 1) ? n4 : lo4 + slice4;
  const float* inbox = pl.inbox[pl.rank];
  float* outbox = pl.outbox[pl.rank];
  for (long long s = (long long)blockIdx.x * nthreads + tid; s < (long long)NCOL * (hi4 - lo4);
       s += gstride) {
    const int c = (int)(s / (hi4 - lo4));
    const long long j = (lo4 + s % (hi4 - lo4)) * 4;
    double t[4] = {0, 0, 0, 0};
    for (long long r = 0; r < P; ++r) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(inbox + ((long long)c * P + r) * pl.n_cap + j));
      t[0] += v.x;
      t[1] += v.y;
      t[2] += v.z;
      t[3] += v.w;
    }
    float4 o = make_float4((float)(a.ac[c] * t[0]), (float)(a.ac[c] * t[1]), (float)(a.ac[c] * t[2]),
                           (float)(a.ac[c] * t[3]));
    *reinterpret_cast<float4*>(a.yc[c] + j) = o;
    *reinterpret_cast<float4*>(outbox + (long long)c * pl.n_cap + j) = o;
  }
  grid_barrier(a.bar);
  if (blockIdx.x == 0 && tid == 0) peer_signal_wait(pl, 1);
  grid_barrier(a.bar);
  // Phase C: gather the other slices from their owners
  for (long long s = (long long)blockIdx.x * nthreads + tid; s < (long long)NCOL * n4; s += gstride) {
    const int c = (int)(s / n4);
    const long long j4 = s % n4;
    const int owner = (int)min(j4 / slice4, P - 1);
    if (owner == pl.rank) continue;
    const float4 v = __ldcg(reinterpret_cast<const float4*>(pl.outbox[owner] + (long long)c * pl.n_cap + j4 * 4));
    *reinterpret_cast<float4*>(a.yc[c] + j4 * 4) = v;
  }
}

// Row partials (when a row spans several column chunks) are local to a rank.
template <int NROW, typename ACC>
__device__ __forceinline__ void finalize_rows(const MatrixArgs& a, int tid, int nthreads) {
  if (NROW == 0 || a.CB <= 1) return;
  const ACC* rowpart = static_cast<const ACC*>(a.rowpart);
  const long long m4 = a.m / 4;
  const int G = fin_group(a.fin_g);
  for_each_slot_grouped((long long)NROW * m4, tid, nthreads, G,
                        [&](long long q, bool valid, int glane, bool lead) {
    const int o = valid ? (int)(q / m4) : 0;
    const long long i = valid ? (q % m4) * 4 : 0;
    ACC t[4];
    group_sum4<ACC>(rowpart + (long long)o * a.CB * a.m + i, a.m, a.CB, valid, glane, G, t);
    if (!lead) return;
    float4 r = make_float4((float)(a.ar[o] * (double)t[0]), (float)(a.ar[o] * (double)t[1]),
                           (float)(a.ar[o] * (double)t[2]), (float)(a.ar[o] * (double)t[3]));
    *reinterpret_cast<float4*>(a.yr[o] + i) = r;
  });
}

template <int NROW, int NCOL, typename ACC>
__device__ __forceinline__ void finalize_any(const MatrixArgs& a, int tid, int nthreads) {
  if (NCOL > 0 && a.peer.nranks > 1) {
    finalize_rows<NROW, ACC>(a, tid, nthreads);
    finalize_columns_peers<NCOL, ACC>(a, tid, nthreads);
  } else {
    finalize<NROW, NCOL, ACC>(a, tid, nthreads);
  }
}

}  // namespace dev
}  // namespace mapfuse::b200
