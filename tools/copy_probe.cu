// copy_probe.cu -- which 1:1 read/write access pattern reaches the HBM copy
// ceiling on B200 (experiment behind the stream/matrix kernel layouts).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o copy_probe tools/copy_probe.cu

//   ./copy_probe [n_floats] [max inputs]
// Variants (y = 2*x1 + x2 + ... over n floats, 1-3 inputs, L2 flushed before
// each timed launch, median of 9); l/s = evict-first/no-allocate cache hints
// on loads/stores (the stream kernel's ld_stream/st_stream) or plain ld/st:
//   P<U>  persistent grid-stride, U float4 per thread in flight, grid ctas*148
//   Q<U>  persistent, CTA b takes blocks b, b+G, ... of 256*U contiguous float4
//   B<U>  non-persistent: one CTA per 256*U float4 block, launched in address order
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

__device__ __forceinline__ float4 ld_h(const float4* p) {
  float4 v;
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_h(float4* p, float4 v) {
  asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ float4 ld_p(const float4* p) { return __ldg(p); }
__device__ __forceinline__ void st_p(float4* p, float4 v) { *p = v; }
__device__ __forceinline__ float4 twice(float4 v) {
  return make_float4(2.f * v.x, 2.f * v.y, 2.f * v.z, 2.f * v.w);
}

// LH/SH: cache hints on loads / stores.  NIN inputs summed into one output.
template <bool LH>
__device__ __forceinline__ float4 ld(const float4* p) {
  return LH ? ld_h(p) : ld_p(p);
}
template <bool SH>
__device__ __forceinline__ void st(float4* p, float4 v) {
  if (SH) st_h(p, v);
  else st_p(p, v);
}
template <int NIN>
__device__ __forceinline__ float4 combine(const float4 (&v)[NIN]) {
  float4 o = twice(v[0]);
#pragma unroll
  for (int k = 1; k < NIN; ++k) {
    o.x += v[k].x;
    o.y += v[k].y;
    o.z += v[k].z;
    o.w += v[k].w;
  }
  return o;
}
struct Ptrs {
  const float4* x[3];
  float4* y;
};

// persistent grid-stride (the stream kernel's current layout)
template <int NIN, int U, bool LH, bool SH>
__global__ void __launch_bounds__(256) persist(Ptrs p, long long n4) {
  const long long stride = (long long)gridDim.x * 256;
  long long i = (long long)blockIdx.x * 256 + threadIdx.x;
  for (; i + (U - 1) * stride < n4; i += U * stride) {
    float4 v[U][NIN];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < NIN; ++k) v[u][k] = ld<LH>(p.x[k] + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) st<SH>(p.y + i + u * stride, combine<NIN>(v[u]));
  }
  for (; i < n4; i += stride) {
    float4 v[NIN];
#pragma unroll
    for (int k = 0; k < NIN; ++k) v[k] = p.x[k][i];
    p.y[i] = combine<NIN>(v);
  }
}

// persistent, block-strided: CTA b takes blocks b, b+G, ... of 256*U
// contiguous float4 (compact address-ordered wavefront, contiguous blocks)
template <int NIN, int U, bool LH, bool SH>
__global__ void __launch_bounds__(256) pblock(Ptrs p, long long n4) {
  const long long nblk = (n4 + 256LL * U - 1) / (256LL * U);
  for (long long b = blockIdx.x; b < nblk; b += gridDim.x) {
    const long long base = b * 256 * U + threadIdx.x;
    float4 v[U][NIN];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < NIN; ++k)
        if (base + u * 256 < n4) v[u][k] = ld<LH>(p.x[k] + base + u * 256);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (base + u * 256 < n4) st<SH>(p.y + base + u * 256, combine<NIN>(v[u]));
  }
}

// non-persistent: one CTA per block
template <int NIN, int U, bool LH, bool SH>
__global__ void __launch_bounds__(256) blocked(Ptrs p, long long n4) {
  const long long base = (long long)blockIdx.x * 256 * U + threadIdx.x;
  float4 v[U][NIN];
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int k = 0; k < NIN; ++k)
      if (base + u * 256 < n4) v[u][k] = ld<LH>(p.x[k] + base + u * 256);
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (base + u * 256 < n4) st<SH>(p.y + base + u * 256, combine<NIN>(v[u]));
}

// D: bulk-engine copy, persistent, one CTA (one elected thread) per SM: CTA b
// moves blocks b, b+G, ... of BLK bytes global -> shared (cp.async.bulk,
// mbarrier complete_tx) -> global (cp.async.bulk bulk_group), S-stage ring.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
template <int S>
__global__ void __launch_bounds__(32) dma_copy(const char* x, char* y, long long nbytes, int BLK) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long full[S];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const long long nblk = nbytes / BLK;
  unsigned phase[S] = {};
  int k = 0;
  // prologue: S loads in flight
  long long b = blockIdx.x;
  long long inflight[S];
  for (int s = 0; s < S; ++s) inflight[s] = -1;
  for (int s = 0; s < S && b < nblk; ++s, b += gridDim.x) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(BLK) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(sm + (size_t)s * BLK)), "l"(x + b * BLK), "r"(BLK), "r"(smem_u32(&full[s])) : "memory");
    inflight[s] = b;
  }
  for (;; ++k) {
    const int s = k % S;
    if (inflight[s] < 0) break;
    // wait for the load of stage s, store it out
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                 ::"r"(smem_u32(&full[s])), "r"(phase[s]) : "memory");
    phase[s] ^= 1u;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(y + inflight[s] * BLK),
                 "r"(smem_u32(sm + (size_t)s * BLK)), "r"(BLK) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (k > 0) {
      // refill the previous stage once its store (one group older) has read it
      const int q = (k - 1) % S;
      if (b < nblk) {
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[q])), "r"(BLK) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_u32(sm + (size_t)q * BLK)), "l"(x + b * BLK), "r"(BLK), "r"(smem_u32(&full[q])) : "memory");
        inflight[q] = b;
        b += gridDim.x;
      } else {
        inflight[q] = -1;
      }
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// B with T threads per CTA
template <int NIN, int U, int T>
__global__ void __launch_bounds__(T) blocked_t(Ptrs p, long long n4) {
  const long long base = (long long)blockIdx.x * T * U + threadIdx.x;
  float4 v[U][NIN];
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int k = 0; k < NIN; ++k)
      if (base + u * T < n4) v[u][k] = ld<false>(p.x[k] + base + u * T);
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (base + u * T < n4) st<false>(p.y + base + u * T, combine<NIN>(v[u]));
}

static double bytes_per_elem = 8.0;

int main(int argc, char** argv) {
  const long long n = argc > 1 ? atoll(argv[1]) : (1LL << 30);
  const long long n4 = n / 4;
  float *x, *y, *fa, *fb;
  CK(cudaMalloc(&x, n * 4));
  CK(cudaMalloc(&y, n * 4));
  CK(cudaMalloc(&fa, 1LL << 30));
  CK(cudaMalloc(&fb, 1LL << 30));
  CK(cudaMemset(x, 0, n * 4));
  CK(cudaMemset(fb, 0, 1LL << 30));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto flush = [&] {
    CK(cudaMemsetAsync(fa, 1, 1LL << 30));
    // read fb through a copy into fa's second half-sized view: touches 1 GiB clean
    CK(cudaMemcpyAsync(fa, fb, 512LL << 20, cudaMemcpyDeviceToDevice));
  };
  auto run = [&](const char* name, auto launch) {
    std::vector<float> ts;
    for (int r = 0; r < 11; ++r) {
      flush();
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (r >= 2) ts.push_back(ms);
    }
    std::sort(ts.begin(), ts.end());
    const float ms = ts[ts.size() / 2];
    printf("%-28s %9.1f us  %7.0f GB/s\n", name, ms * 1e3, bytes_per_elem * n / ms / 1e6);
    fflush(stdout);
  };
  char nm[96];
  const int nin_max = argc > 2 ? atoi(argv[2]) : 3;
  float* x2;
  float* x3;
  CK(cudaMalloc(&x2, n * 4));
  CK(cudaMalloc(&x3, n * 4));
  CK(cudaMemset(x2, 0, n * 4));
  CK(cudaMemset(x3, 0, n * 4));
  Ptrs P{{(const float4*)x, (const float4*)x2, (const float4*)x3}, (float4*)y};
  bytes_per_elem = 0;
#define VARS(NIN, U, LH, SH)                                                                   \
  {                                                                                            \
    bytes_per_elem = 4.0 * (NIN + 1);                                                          \
    const long long nb = (n4 + 256LL * U - 1) / (256LL * U);                                   \
    for (int c : {2, 4}) {                                                                     \
      snprintf(nm, sizeof nm, "in%d P%d l%d s%d ctas=%d", NIN, U, LH, SH, c);                  \
      run(nm, [&] { persist<NIN, U, LH, SH><<<sms * c, 256>>>(P, n4); });                      \
      snprintf(nm, sizeof nm, "in%d Q%d l%d s%d ctas=%d", NIN, U, LH, SH, c);                  \
      run(nm, [&] { pblock<NIN, U, LH, SH><<<(unsigned)std::min<long long>(nb, sms * c), 256>>>(P, n4); }); \
    }                                                                                          \
    snprintf(nm, sizeof nm, "in%d B%d l%d s%d", NIN, U, LH, SH);                               \
    run(nm, [&] { blocked<NIN, U, LH, SH><<<(unsigned)nb, 256>>>(P, n4); });                   \
  }
#define HINTS(NIN, U) VARS(NIN, U, false, false) VARS(NIN, U, true, false) VARS(NIN, U, false, true) VARS(NIN, U, true, true)
  if (getenv("PROBE_THREADS")) {
#define BT(NIN, U, T)                                                                   \
  {                                                                                     \
    bytes_per_elem = 4.0 * (NIN + 1);                                                   \
    const long long nb = (n4 + (long long)T * U - 1) / ((long long)T * U);              \
    snprintf(nm, sizeof nm, "in%d B%d T=%d", NIN, U, T);                                \
    run(nm, [&] { blocked_t<NIN, U, T><<<(unsigned)nb, T>>>(P, n4); });                 \
  }
    BT(3, 2, 128) BT(3, 2, 256) BT(3, 2, 512) BT(3, 4, 128) BT(3, 1, 512) BT(3, 1, 1024)
    BT(2, 2, 128) BT(2, 2, 256) BT(2, 2, 512) BT(2, 4, 128) BT(2, 1, 512)
    BT(1, 2, 128) BT(1, 2, 256) BT(1, 2, 512) BT(1, 4, 128) BT(1, 1, 512)
    return 0;
  }
  if (getenv("PROBE_DMA")) {
    bytes_per_elem = 8.0;
    for (int blk : {8192, 16384, 32768}) {
      for (int per_sm : {1, 2}) {
        const int S = 8;
        const size_t smem = (size_t)S * blk;
        if (smem * per_sm > 200 * 1024) continue;
        CK(cudaFuncSetAttribute(dma_copy<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        snprintf(nm, sizeof nm, "DMA blk=%d S=8 ctas=%d", blk, per_sm);
        run(nm, [&] { dma_copy<8><<<sms * per_sm, 32, smem>>>((const char*)x, (char*)y, n * 4, blk); });
      }
    }
    for (int blk : {4096, 8192}) {
      const int S = 8;
      const size_t smem = (size_t)S * blk;
      CK(cudaFuncSetAttribute(dma_copy<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      snprintf(nm, sizeof nm, "DMA blk=%d S=8 ctas=3", blk);
      run(nm, [&] { dma_copy<8><<<sms * 3, 32, smem>>>((const char*)x, (char*)y, n * 4, blk); });
    }
    return 0;
  }
  if (nin_max >= 1) { HINTS(1, 2) HINTS(1, 4) }
  if (nin_max >= 2) { HINTS(2, 2) HINTS(2, 4) }
  if (nin_max >= 3) { HINTS(3, 2) HINTS(3, 4) }
  return 0;
}
