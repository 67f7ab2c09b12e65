/* A plain-C, single-process multi-GPU client of mf_launch_sharded (the
 * sharded launch of SURVEY.md 8(b)): BiCGK q = A p, s = A^T r row-sharded
 * over every visible GPU, one ncclComm_t per GPU from ncclCommInitAll, the
 * partial s all-reduced by NCCL between kernels.  Checked against an fp64
 * host evaluation with the parity tolerance |got - ref| <= 2^-17 S + ulp. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime.h>
#include <nccl.h>

#include "mapfuse_b200.h"

#define MAXG 8

static float urand(unsigned* s) {
  *s = *s * 1664525u + 1013904223u;
  return (float)((*s >> 8) & 0xffff) / 32768.0f - 1.0f;
}

static int close_enough(float got, double ref, double S) {
  return fabs((double)got - ref) <= ldexp(S, -17) + nextafterf(fabsf((float)ref), INFINITY) - fabsf((float)ref);
}

int main(void) {
  const int m = 2048, n = 1536;
  int ngpus = 0;
  if (cudaGetDeviceCount(&ngpus) != cudaSuccess || ngpus < 1) return 2;
  if (ngpus > MAXG) ngpus = MAXG;
  int devs[MAXG];
  for (int g = 0; g < ngpus; ++g) devs[g] = g;
  ncclComm_t comms[MAXG];
  if (ncclCommInitAll(comms, ngpus, devs) != ncclSuccess) {
    fprintf(stderr, "ncclCommInitAll failed\n");
    return 1;
  }
  float* A = malloc(sizeof(float) * m * n);
  float *p = malloc(sizeof(float) * n), *r = malloc(sizeof(float) * m);
  unsigned seed = 12345u;
  for (long i = 0; i < (long)m * n; ++i) A[i] = urand(&seed);
  for (int j = 0; j < n; ++j) p[j] = urand(&seed);
  for (int i = 0; i < m; ++i) r[i] = urand(&seed);

  mf_plan* plans[MAXG];
  mf_buffer bufs[MAXG][5];
  const mf_buffer* per_gpu[MAXG];
  int nbuf[MAXG], row0[MAXG], rows[MAXG];
  void* streams[MAXG];
  void* cm[MAXG];
  float* dq[MAXG];
  float* ds[MAXG];
  for (int g = 0; g < ngpus; ++g) {
    /* contiguous row panels, multiples of 32 rows */
    row0[g] = (m / 32) * g / ngpus * 32;
    rows[g] = (m / 32) * (g + 1) / ngpus * 32 - row0[g];
    cudaSetDevice(g);
    cudaStream_t st;
    cudaStreamCreate(&st);
    streams[g] = st;
    cm[g] = comms[g];
    if (mf_compile_sequence("BICGK", rows[g], n, MF_MODE_FUSED, &plans[g]) != MF_OK) {
      fprintf(stderr, "compile: %s\n", mf_last_error());
      return 1;
    }
    float *dA, *dp, *dr;
    cudaMalloc((void**)&dA, sizeof(float) * rows[g] * n);
    cudaMalloc((void**)&dp, sizeof(float) * n);
    cudaMalloc((void**)&dr, sizeof(float) * rows[g]);
    cudaMalloc((void**)&dq[g], sizeof(float) * rows[g]);
    cudaMalloc((void**)&ds[g], sizeof(float) * n);
    cudaMemcpy(dA, A + (long)row0[g] * n, sizeof(float) * rows[g] * n, cudaMemcpyHostToDevice);
    cudaMemcpy(dp, p, sizeof(float) * n, cudaMemcpyHostToDevice);
    cudaMemcpy(dr, r + row0[g], sizeof(float) * rows[g], cudaMemcpyHostToDevice);
    mf_buffer b[5] = {{"A", rows[g], n, dA}, {"p", 1, n, dp}, {"r", 1, rows[g], dr},
                      {"q", 1, rows[g], dq[g]}, {"s", 1, n, ds[g]}};
    for (int i = 0; i < 5; ++i) bufs[g][i] = b[i];
    per_gpu[g] = bufs[g];
    nbuf[g] = 5;
  }
  mf_stats stats;
  if (mf_launch_sharded((const mf_plan* const*)plans, ngpus, devs, per_gpu, nbuf, NULL, 0, cm, streams,
                        &stats) != MF_OK) {
    fprintf(stderr, "mf_launch_sharded: %s\n", mf_last_error());
    return 1;
  }
  float* q = malloc(sizeof(float) * m);
  float* s = malloc(sizeof(float) * n * ngpus);
  for (int g = 0; g < ngpus; ++g) {
    cudaSetDevice(g);
    cudaStreamSynchronize((cudaStream_t)streams[g]);
    cudaMemcpy(q + row0[g], dq[g], sizeof(float) * rows[g], cudaMemcpyDeviceToHost);
    cudaMemcpy(s + (long)g * n, ds[g], sizeof(float) * n, cudaMemcpyDeviceToHost);
  }
  for (int i = 0; i < m; ++i) {
    double ref = 0, S = 0;
    for (int j = 0; j < n; ++j) {
      ref += (double)A[(long)i * n + j] * p[j];
      S += fabs((double)A[(long)i * n + j] * p[j]);
    }
    if (!close_enough(q[i], ref, S)) {
      fprintf(stderr, "q[%d] %g vs %g\n", i, q[i], ref);
      return 1;
    }
  }
  for (int j = 0; j < n; ++j) {
    double ref = 0, S = 0;
    for (int i = 0; i < m; ++i) {
      ref += (double)A[(long)i * n + j] * r[i];
      S += fabs((double)A[(long)i * n + j] * r[i]);
    }
    for (int g = 0; g < ngpus; ++g)
      if (!close_enough(s[(long)g * n + j], ref, S) || s[(long)g * n + j] != s[j]) {
        fprintf(stderr, "s[%d] on GPU %d %g vs %g\n", j, g, s[(long)g * n + j], ref);
        return 1;
      }
  }
  if (stats.kernels != ngpus) {
    fprintf(stderr, "stats.kernels %d\n", stats.kernels);
    return 1;
  }
  /* a missing buffer is an argument error, reported as a status code */
  int bad_n[MAXG];
  for (int g = 0; g < ngpus; ++g) bad_n[g] = 3;
  if (mf_launch_sharded((const mf_plan* const*)plans, ngpus, devs, per_gpu, bad_n, NULL, 0, cm, streams,
                        NULL) == MF_OK)
    return 1;
  for (int g = 0; g < ngpus; ++g) {
    mf_plan_destroy(plans[g]);
    ncclCommDestroy(comms[g]);
  }
  printf("c sharded client ok (%d GPU(s), NCCL all-reduce of s)\n", ngpus);
  return 0;
}
