// ger_probe.cu -- access-pattern experiment for the rank-update + column
// reduction shape (GEMVER k0: B = A + u v^T, t = B^T y; A read once, B
// written once, t reduced over rows) on an m x n fp32 matrix.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ger_probe tools/ger_probe.cu
//   ./ger_probe [m] [n]
// Layouts (L2 flushed before every timed launch, median of 9, GB/s counts
// A + B only):
//   T  band tiles: 2 CTAs/SM persistent, CTA = (2048-col chunk, row band),
//      R rows per batch (the register-fed matrix kernel's mapping)
//   O<U,c> column owner: c CTAs/SM, CTA owns a contiguous column slice for ALL
//      rows (t completes inside the CTA: no partials, no grid barrier); 8 row
//      groups x slice/4 threads; U rows per thread in flight
//   M  the map alone, one CTA per 512-float4 block (the stream kernel's
//      layout): the ceiling without the column reduction
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)

struct Args {
  const float* A;
  float* B;
  const float* u;
  const float* v;
  const float* y;
  float* t;
  float* part;
  long long m, n;
};

__device__ __forceinline__ float4 upd(float4 a, float u, float4 v) {
  return make_float4(fmaf(u, v.x, a.x), fmaf(u, v.y, a.y), fmaf(u, v.z, a.z), fmaf(u, v.w, a.w));
}

// T: band tiles (K = 2 float4 per thread, chunk 2048 columns)
// IL: rows of band rb are rb, rb + RB, rb + 2 RB, ... (interleaved bands: the
// CTAs of a column chunk sweep the matrix together, a compact window)
template <int R, bool IL>
__global__ void __launch_bounds__(256, 2) band_tiles(Args a, int CB, int RB) {
  const int tid = threadIdx.x;
  for (int tile = blockIdx.x; tile < CB * RB; tile += gridDim.x) {
    const int cb = tile % CB, rb = tile / CB;
    const long long r0 = (long long)rb * a.m / RB, r1 = (long long)(rb + 1) * a.m / RB;
    long long col[2];
    float4 vv[2], acc[2];
    for (int k = 0; k < 2; ++k) {
      col[k] = (long long)cb * 2048 + 4 * (tid + 256 * k);
      vv[k] = *reinterpret_cast<const float4*>(a.v + col[k]);
      acc[k] = make_float4(0, 0, 0, 0);
    }
    // band rows: contiguous [r0, r1) or interleaved rb + RB * q
    const long long cnt = IL ? (a.m - rb + RB - 1) / RB : r1 - r0;
    for (long long q0 = 0; q0 < cnt; q0 += R) {
      float4 av[R][2];
      float us[R], ys[R];
      long long row[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const long long q = min(q0 + r, cnt - 1);
        row[r] = IL ? rb + q * RB : r0 + q;
        const long long i = row[r];
        us[r] = __ldg(a.u + i);
        ys[r] = (q0 + r < cnt) ? __ldg(a.y + i) : 0.f;
#pragma unroll
        for (int k = 0; k < 2; ++k) av[r][k] = __ldg(reinterpret_cast<const float4*>(a.A + i * a.n + col[k]));
      }
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const float4 b = upd(av[r][k], us[r], vv[k]);
          if (q0 + r < cnt) *reinterpret_cast<float4*>(a.B + row[r] * a.n + col[k]) = b;
          acc[k].x = fmaf(b.x, ys[r], acc[k].x);
          acc[k].y = fmaf(b.y, ys[r], acc[k].y);
          acc[k].z = fmaf(b.z, ys[r], acc[k].z);
          acc[k].w = fmaf(b.w, ys[r], acc[k].w);
        }
    }
    for (int k = 0; k < 2; ++k)
      *reinterpret_cast<float4*>(a.part + (long long)rb * a.n + col[k]) = acc[k];
  }
}

// N: non-persistent tiles, one CTA per (RT-row band, 2048-col chunk), launched
// band-major (address order); each tile writes its column partial.
template <int RT, int R>
__global__ void __launch_bounds__(256) np_tiles(Args a, int CB) {
  const int tid = threadIdx.x;
  const int cb = blockIdx.x % CB, rb = blockIdx.x / CB;
  const long long r0 = (long long)rb * RT, r1 = min(a.m, r0 + RT);
  long long col[2];
  float4 vv[2], acc[2];
  for (int k = 0; k < 2; ++k) {
    col[k] = (long long)cb * 2048 + 4 * (tid + 256 * k);
    vv[k] = *reinterpret_cast<const float4*>(a.v + col[k]);
    acc[k] = make_float4(0, 0, 0, 0);
  }
  for (long long i0 = r0; i0 < r1; i0 += R) {
    float4 av[R][2];
    float us[R], ys[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const long long i = i0 + r;
      us[r] = __ldg(a.u + i);
      ys[r] = __ldg(a.y + i);
#pragma unroll
      for (int k = 0; k < 2; ++k) av[r][k] = __ldg(reinterpret_cast<const float4*>(a.A + i * a.n + col[k]));
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const float4 b = upd(av[r][k], us[r], vv[k]);
        *reinterpret_cast<float4*>(a.B + (i0 + r) * a.n + col[k]) = b;
        acc[k].x = fmaf(b.x, ys[r], acc[k].x);
        acc[k].y = fmaf(b.y, ys[r], acc[k].y);
        acc[k].z = fmaf(b.z, ys[r], acc[k].z);
        acc[k].w = fmaf(b.w, ys[r], acc[k].w);
      }
  }
  for (int k = 0; k < 2; ++k)
    *reinterpret_cast<float4*>(a.part + (long long)(rb % 512) * a.n + col[k]) = acc[k];
}

// O: column owner.  Slice = S4 float4 columns per CTA; 8 row groups.
template <int U>
__global__ void __launch_bounds__(1024) column_owner(Args a, int S4) {
  extern __shared__ float4 red[];
  const int tid = threadIdx.x;
  const int j = tid % S4, rg = tid / S4;  // rg in [0, 8)
  const long long n4 = a.n / 4;
  const long long c4 = (long long)blockIdx.x * S4 + j;
  const bool ok = c4 < n4 && rg < 8;
  float4 acc = make_float4(0, 0, 0, 0);
  if (ok) {
    const float4 vv = *reinterpret_cast<const float4*>(a.v + 4 * c4);
    const float4* Ap = reinterpret_cast<const float4*>(a.A) + c4;
    float4* Bp = reinterpret_cast<float4*>(a.B) + c4;
    long long i0 = rg;
    for (; i0 + 8 * (U - 1) < a.m; i0 += 8 * U) {
      float4 av[U];
      float us[U], ys[U];
#pragma unroll
      for (int r = 0; r < U; ++r) {
        av[r] = __ldg(Ap + (i0 + 8 * r) * n4);
        us[r] = __ldg(a.u + i0 + 8 * r);
        ys[r] = __ldg(a.y + i0 + 8 * r);
      }
#pragma unroll
      for (int r = 0; r < U; ++r) {
        const float4 b = upd(av[r], us[r], vv);
        Bp[(i0 + 8 * r) * n4] = b;
        acc.x = fmaf(b.x, ys[r], acc.x);
        acc.y = fmaf(b.y, ys[r], acc.y);
        acc.z = fmaf(b.z, ys[r], acc.z);
        acc.w = fmaf(b.w, ys[r], acc.w);
      }
    }
    for (; i0 < a.m; i0 += 8) {
      const float4 b = upd(__ldg(Ap + i0 * n4), __ldg(a.u + i0), vv);
      Bp[i0 * n4] = b;
      const float ys = __ldg(a.y + i0);
      acc.x = fmaf(b.x, ys, acc.x);
      acc.y = fmaf(b.y, ys, acc.y);
      acc.z = fmaf(b.z, ys, acc.z);
      acc.w = fmaf(b.w, ys, acc.w);
    }
  }
  if (rg < 8) red[rg * S4 + j] = acc;
  __syncthreads();
  if (rg == 0 && ok) {
    float4 s = red[j];
    for (int g = 1; g < 8; ++g) {
      s.x += red[g * S4 + j].x;
      s.y += red[g * S4 + j].y;
      s.z += red[g * S4 + j].z;
      s.w += red[g * S4 + j].w;
    }
    *reinterpret_cast<float4*>(a.t + 4 * c4) = s;
  }
}

// M: the map alone, stream-kernel layout (2 float4 per thread, one CTA per block)
__global__ void __launch_bounds__(256) map_only(Args a) {
  const long long n4 = a.n / 4;
  const long long base = (long long)blockIdx.x * 512 + threadIdx.x;
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const long long q = base + 256 * u;
    if (q < a.m * n4) {
      const long long i = q / n4, c4 = q % n4;
      const float4 vv = __ldg(reinterpret_cast<const float4*>(a.v) + c4);
      reinterpret_cast<float4*>(a.B)[q] = upd(__ldg(reinterpret_cast<const float4*>(a.A) + q), __ldg(a.u + i), vv);
    }
  }
}

int main(int argc, char** argv) {
  const long long m = argc > 1 ? atoll(argv[1]) : 32768, n = argc > 2 ? atoll(argv[2]) : 32768;
  Args a{};
  a.m = m;
  a.n = n;
  float *A, *B, *u, *v, *y, *t, *part, *fa, *fb;
  CK(cudaMalloc(&A, m * n * 4));
  CK(cudaMalloc(&B, m * n * 4));
  CK(cudaMalloc(&u, m * 4));
  CK(cudaMalloc(&y, m * 4));
  CK(cudaMalloc(&v, n * 4));
  CK(cudaMalloc(&t, n * 4));
  CK(cudaMalloc(&part, 512 * n * 4));
  CK(cudaMalloc(&fa, 1LL << 30));
  CK(cudaMalloc(&fb, 1LL << 30));
  CK(cudaMemset(A, 0, m * n * 4));
  CK(cudaMemset(u, 0, m * 4));
  CK(cudaMemset(y, 0, m * 4));
  CK(cudaMemset(v, 0, n * 4));
  CK(cudaMemset(fb, 0, 1LL << 30));
  a.A = A;
  a.B = B;
  a.u = u;
  a.v = v;
  a.y = y;
  a.t = t;
  a.part = part;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto run = [&](const char* name, auto launch) {
    std::vector<float> ts;
    for (int r = 0; r < 11; ++r) {
      CK(cudaMemsetAsync(fa, 1, 1LL << 30));
      CK(cudaMemcpyAsync(fa, fb, 512LL << 20, cudaMemcpyDeviceToDevice));
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (r >= 2) ts.push_back(ms);
    }
    std::sort(ts.begin(), ts.end());
    const float ms = ts[ts.size() / 2];
    printf("%-28s %9.1f us  %7.0f GB/s\n", name, ms * 1e3, 8.0 * m * n / ms / 1e6);
    fflush(stdout);
  };
  char nm[96];
  {
    const int CB = (int)(n / 2048), G = 2 * sms;
    const int RB = G / CB > 0 ? (G * 2) / CB : 1;  // 2 tiles per CTA, as lcm(296, 16)/16
    snprintf(nm, sizeof nm, "T R=8 CB=%d RB=%d", CB, RB);
    run(nm, [&] { band_tiles<8, false><<<G, 256>>>(a, CB, RB); });
    snprintf(nm, sizeof nm, "T R=4 CB=%d RB=%d", CB, RB);
    run(nm, [&] { band_tiles<4, false><<<G, 256>>>(a, CB, RB); });
    snprintf(nm, sizeof nm, "TI R=8 CB=%d RB=%d", CB, RB);
    run(nm, [&] { band_tiles<8, true><<<G, 256>>>(a, CB, RB); });
    snprintf(nm, sizeof nm, "TI R=4 CB=%d RB=%d", CB, RB);
    run(nm, [&] { band_tiles<4, true><<<G, 256>>>(a, CB, RB); });
    // one tile per CTA: all 16 chunks x RB/2 bands resident
    snprintf(nm, sizeof nm, "TI R=8 CB=%d RB=%d (1 tile/CTA)", CB, RB / 2 + 0);
    run(nm, [&] { band_tiles<8, true><<<CB * (G / CB), 256>>>(a, CB, G / CB); });
  }
  {
    const int CB = (int)(n / 2048);
    run("N RT=16 R=4", [&] { np_tiles<16, 4><<<(unsigned)(CB * (m / 16)), 256>>>(a, CB); });
    run("N RT=32 R=4", [&] { np_tiles<32, 4><<<(unsigned)(CB * (m / 32)), 256>>>(a, CB); });
    run("N RT=64 R=4", [&] { np_tiles<64, 4><<<(unsigned)(CB * (m / 64)), 256>>>(a, CB); });
    run("N RT=64 R=8", [&] { np_tiles<64, 8><<<(unsigned)(CB * (m / 64)), 256>>>(a, CB); });
    run("N RT=128 R=8", [&] { np_tiles<128, 8><<<(unsigned)(CB * (m / 128)), 256>>>(a, CB); });
    run("N RT=8 R=4", [&] { np_tiles<8, 4><<<(unsigned)(CB * (m / 8)), 256>>>(a, CB); });
    const int G8 = 8 * sms, RB8 = G8 / CB;
    snprintf(nm, sizeof nm, "T R=2 8/SM CB=%d RB=%d", CB, RB8);
    run(nm, [&] { band_tiles<2, false><<<CB * RB8, 256>>>(a, CB, RB8); });
  }
  const long long n4 = n / 4;
  if (getenv("GER_OWNER"))
  for (int c : {1, 2, 3, 4}) {
    const int ctas = sms * c;
    const int S4 = (int)((n4 + ctas - 1) / ctas);
    const int threads = S4 * 8;
    if (threads > 1024) continue;
    const size_t smem = (size_t)threads * 16;
    CK(cudaFuncSetAttribute(column_owner<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(column_owner<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(column_owner<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int grid = (int)((n4 + S4 - 1) / S4);
    snprintf(nm, sizeof nm, "O U=4 c=%d S4=%d", c, S4);
    run(nm, [&] { column_owner<4><<<grid, threads, smem>>>(a, S4); });
    snprintf(nm, sizeof nm, "O U=8 c=%d S4=%d", c, S4);
    run(nm, [&] { column_owner<8><<<grid, threads, smem>>>(a, S4); });
    snprintf(nm, sizeof nm, "O U=16 c=%d S4=%d", c, S4);
    run(nm, [&] { column_owner<16><<<grid, threads, smem>>>(a, S4); });
  }
  {
    const long long blocks = (m * n4 + 511) / 512;
    run("M map only", [&] { map_only<<<(unsigned)blocks, 256>>>(a); });
  }
  return 0;
}
