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
__device__ __forceinline__ void grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    unsigned g = *gen;
    __threadfence();
    unsigned arrived = atomicAdd(bar, 1u);
    if (arrived == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) __nanosleep(64);
    }
    __threadfence();
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

// Cross-CTA finalize after the grid barrier: column outputs sum the RB band
// partials, row outputs (when the row was split over CB column chunks) sum
// the CB chunk partials -- fixed order, so results are reproducible.
template <int NROW, int NCOL, typename ACC>
__device__ __forceinline__ void finalize(const MatrixArgs& a, int tid, int nthreads) {
  ACC* colpart = static_cast<ACC*>(a.colpart);
  ACC* rowpart = static_cast<ACC*>(a.rowpart);
  const bool need_rows = (NROW > 0) && a.CB > 1;
  const long long n4 = a.n / 4, m4 = a.m / 4;
  const long long col_slots = (long long)NCOL * n4;
  const long long total = col_slots + (need_rows ? (long long)NROW * m4 : 0);
  for (long long s = (long long)blockIdx.x * nthreads + tid; s < total;
       s += (long long)gridDim.x * nthreads) {
    if (s < col_slots) {
      const int c = (int)(s / n4);
      const long long j = (s % n4) * 4;
      ACC t[4] = {ACC(0), ACC(0), ACC(0), ACC(0)};
      for (int b = 0; b < a.RB; ++b) {
        const ACC* p = colpart + ((long long)c * a.RB + b) * a.n + j;
#pragma unroll
        for (int e = 0; e < 4; ++e) t[e] += __ldcg(p + e);
      }
      float4 o;
      o.x = (float)(a.ac[c] * (double)t[0]);
      o.y = (float)(a.ac[c] * (double)t[1]);
      o.z = (float)(a.ac[c] * (double)t[2]);
      o.w = (float)(a.ac[c] * (double)t[3]);
      *reinterpret_cast<float4*>(a.yc[c] + j) = o;
    } else {
      const long long q = s - col_slots;
      const int o = (int)(q / m4);
      const long long i = (q % m4) * 4;
      ACC t[4] = {ACC(0), ACC(0), ACC(0), ACC(0)};
      for (int b = 0; b < a.CB; ++b) {
        const ACC* p = rowpart + ((long long)o * a.CB + b) * a.m + i;
#pragma unroll
        for (int e = 0; e < 4; ++e) t[e] += __ldcg(p + e);
      }
      float4 r;
      r.x = (float)(a.ar[o] * (double)t[0]);
      r.y = (float)(a.ar[o] * (double)t[1]);
      r.z = (float)(a.ar[o] * (double)t[2]);
      r.w = (float)(a.ar[o] * (double)t[3]);
      *reinterpret_cast<float4*>(a.yr[o] + i) = r;
    }
  }
}

}  // namespace dev
}  // namespace mapfuse::b200
