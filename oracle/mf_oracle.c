/*
 * mf_oracle.c -- CPU restatement of the reference's oracle for the fused
 * BLAS-1/BLAS-2 sequence path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1305_1183_b200/)
 * links, loads or calls this file.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs use it, and only as the
 * checker (or as the timed CPU baseline), never as the thing measured.
 *
 * What it restates (all citations relative to /root/reference/):
 *   - input generation: proj/src/blas.cpp:107-139 (make_problem) -- a
 *     std::mt19937(seed) stream fed through
 *     std::uniform_real_distribution<float>(-1, 1); scalars are
 *     0.25f + 0.5f*|U| (blas.cpp:120).  mt19937 is restated from its published
 *     definition (Matsumoto & Nishimura 1998); the float conversion follows
 *     libstdc++'s generate_canonical<float, 24> (one 32-bit draw, converted
 *     to float, divided by 2^32, clamped below 1).
 *   - sequence formulas: proj/src/blas.cpp:178-270 (reference_execute), fp64
 *     arithmetic, narrowed to float once at the end (blas.cpp:150-154).
 *     matvec / matvec_t follow blas.cpp:156-174 loop for loop (same summation
 *     order) so results are bit-identical to the reference built with the
 *     same (non-contracting) floating-point flags.
 *   - per-call semantics: proj/src/blas.cpp:275-342 (reference_call), each
 *     call narrowed to float after it runs (blas.cpp:281).
 *
 * Parity pinning: tests/test_oracle.py checks this file against golden
 * vectors produced by the reference itself (oracle/_ref, built from
 * /root/reference/proj/src by oracle/Makefile; fixtures committed under
 * tests/golden/ with the generating script oracle/gen_golden.py).
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared (see oracle/Makefile).
 * -ffp-contract=off matters: an FMA-contracted build would not reproduce the
 * reference's double rounding sequence.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* MT19937 (32-bit), published algorithm.                                    */

typedef struct {
  uint32_t s[624];
  int i;
} mfo_rng;

static void mt_seed(mfo_rng* g, uint32_t seed) {
  g->s[0] = seed;
  for (int k = 1; k < 624; ++k)
    g->s[k] = 1812433253u * (g->s[k - 1] ^ (g->s[k - 1] >> 30)) + (uint32_t)k;
  g->i = 624;
}

static void mt_twist(mfo_rng* g) {
  for (int k = 0; k < 624; ++k) {
    uint32_t y = (g->s[k] & 0x80000000u) | (g->s[(k + 1) % 624] & 0x7fffffffu);
    uint32_t v = g->s[(k + 397) % 624] ^ (y >> 1);
    if (y & 1u) v ^= 0x9908b0dfu;
    g->s[k] = v;
  }
  g->i = 0;
}

static uint32_t mt_next(mfo_rng* g) {
  if (g->i >= 624) mt_twist(g);
  uint32_t y = g->s[g->i++];
  y ^= y >> 11;
  y ^= (y << 7) & 0x9d2c5680u;
  y ^= (y << 15) & 0xefc60000u;
  y ^= y >> 18;
  return y;
}

/* libstdc++ uniform_real_distribution<float>(a=-1, b=1):
 *   u = generate_canonical<float,24>(g) = float(g()) / 2^32 (clamped < 1)
 *   return u * (b - a) + a            (all in float)                       */
static float mt_uniform_m1p1(mfo_rng* g) {
  float u = (float)mt_next(g) / 4294967296.0f;
  if (u >= 1.0f) u = nextafterf(1.0f, 0.0f);
  return u * 2.0f + -1.0f;
}

void* mfo_rng_new(uint32_t seed) {
  mfo_rng* g = (mfo_rng*)malloc(sizeof(mfo_rng));
  if (g) mt_seed(g, seed);
  return g;
}
void mfo_rng_free(void* g) { free(g); }

/* Fills n floats with U(-1,1), continuing the stream. */
void mfo_rng_fill(void* g, float* out, size_t n) {
  for (size_t k = 0; k < n; ++k) out[k] = mt_uniform_m1p1((mfo_rng*)g);
}

/* One scalar input: 0.25f + 0.5f * |U(-1,1)|  (blas.cpp:120). */
float mfo_rng_scalar(void* g) {
  float u = mt_uniform_m1p1((mfo_rng*)g);
  return 0.25f + 0.5f * fabsf(u);
}

uint32_t mfo_rng_raw(void* g) { return mt_next((mfo_rng*)g); }

/* ------------------------------------------------------------------------ */
/* Counter-based generator for sizes the mt19937 stream cannot reach in     */
/* reasonable time (the 131072^2 sharded configs).      */
/* The product's device generator (csrc/mf_gen.cu) implements the same       */
/* function; values are k * 2^-23 - 1 with k < 2^24, exact in float.         */

static uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

float mfo_hash_uniform(uint64_t seed, uint64_t index) {
  uint64_t h = splitmix64(index ^ splitmix64(seed));
  uint32_t k = (uint32_t)(h >> 40); /* 24 bits */
  return (float)k * (1.0f / 8388608.0f) - 1.0f;
}

void mfo_hash_fill(uint64_t seed, uint64_t base, float* out, size_t n) {
  for (size_t k = 0; k < n; ++k) out[k] = mfo_hash_uniform(seed, base + k);
}

/* ------------------------------------------------------------------------ */
/* fp64 helpers mirroring blas.cpp:156-174.                                  */

static double* widen(const float* v, size_t n) {
  double* d = (double*)malloc(n * sizeof(double));
  for (size_t k = 0; k < n; ++k) d[k] = (double)v[k];
  return d;
}

static void narrow(const double* d, float* out, size_t n) {
  for (size_t k = 0; k < n; ++k) out[k] = (float)d[k];
}

/* y[i] = sum_j a[i*cols+j] * x[j], j ascending (blas.cpp:156-164). */
static void matvec(const double* a, int rows, int cols, const double* x, double* y) {
  for (int i = 0; i < rows; ++i) {
    double acc = 0.0;
    const double* row = a + (size_t)i * (size_t)cols;
    for (int j = 0; j < cols; ++j) acc += row[j] * x[j];
    y[i] = acc;
  }
}

/* y[j] = sum_i a[i*cols+j] * x[i], i ascending per j (blas.cpp:166-174).
 * Evaluated row-wise with one accumulator per column: the per-column
 * summation order (i ascending) and therefore every rounding step is the
 * same as the reference's column-strided loop, only cache-friendlier.      */
static void matvec_t(const double* a, int rows, int cols, const double* x, double* y) {
  for (int j = 0; j < cols; ++j) y[j] = 0.0;
  for (int i = 0; i < rows; ++i) {
    const double* row = a + (size_t)i * (size_t)cols;
    double xi = x[i];
    for (int j = 0; j < cols; ++j) y[j] += row[j] * xi;
  }
}

/* ------------------------------------------------------------------------ */
/* reference_execute restatement, one entry per Table-1 sequence             */
/* (blas.cpp:185-265).  Matrices row-major rows x cols; vectors as sized by  */
/* the caller.                                                               */

void mfo_axpydot(int n, const float* w, const float* v, const float* u, float alpha,
                 float* z_out, float* r_out) {
  double a = alpha, r = 0.0;
  double* z = (double*)malloc((size_t)n * sizeof(double));
  for (int i = 0; i < n; ++i) z[i] = (double)w[i] - a * (double)v[i];
  for (int i = 0; i < n; ++i) r += z[i] * (double)u[i];
  narrow(z, z_out, (size_t)n);
  *r_out = (float)r;
  free(z);
}

void mfo_vadd(int n, const float* w, const float* y, const float* z, float* x_out) {
  for (int i = 0; i < n; ++i) x_out[i] = (float)((double)w[i] + (double)y[i] + (double)z[i]);
}

void mfo_waxpby(int n, const float* x, const float* y, float alpha, float beta, float* w_out) {
  double a = alpha, b = beta;
  for (int i = 0; i < n; ++i) w_out[i] = (float)(a * (double)x[i] + b * (double)y[i]);
}

void mfo_sscal(int n, const float* x, float alpha, float* y_out) {
  double a = alpha;
  for (int i = 0; i < n; ++i) y_out[i] = (float)(a * (double)x[i]);
}

void mfo_madd(int m, int n, const float* A, const float* B, float* C_out) {
  size_t mn = (size_t)m * (size_t)n;
  for (size_t k = 0; k < mn; ++k) C_out[k] = (float)((double)A[k] + (double)B[k]);
}

void mfo_bicgk(int m, int n, const float* A, const float* p, const float* r, float* q_out,
               float* s_out) {
  size_t mn = (size_t)m * (size_t)n;
  double* a = widen(A, mn);
  double* pd = widen(p, (size_t)n);
  double* rd = widen(r, (size_t)m);
  double* q = (double*)malloc((size_t)m * sizeof(double));
  double* s = (double*)malloc((size_t)n * sizeof(double));
  matvec(a, m, n, pd, q);
  matvec_t(a, m, n, rd, s);
  narrow(q, q_out, (size_t)m);
  narrow(s, s_out, (size_t)n);
  free(a); free(pd); free(rd); free(q); free(s);
}

void mfo_atax(int m, int n, const float* A, const float* x, float* y_out) {
  size_t mn = (size_t)m * (size_t)n;
  double* a = widen(A, mn);
  double* xd = widen(x, (size_t)n);
  double* t = (double*)malloc((size_t)m * sizeof(double));
  double* y = (double*)malloc((size_t)n * sizeof(double));
  matvec(a, m, n, xd, t);
  matvec_t(a, m, n, t, y);
  narrow(y, y_out, (size_t)n);
  free(a); free(xd); free(t); free(y);
}

void mfo_sgemv(int m, int n, const float* A, const float* x, const float* y, float alpha,
               float beta, float* z_out) {
  size_t mn = (size_t)m * (size_t)n;
  double* a = widen(A, mn);
  double* xd = widen(x, (size_t)n);
  double* t = (double*)malloc((size_t)m * sizeof(double));
  matvec(a, m, n, xd, t);
  double al = alpha, be = beta;
  for (int i = 0; i < m; ++i) z_out[i] = (float)(al * t[i] + be * (double)y[i]);
  free(a); free(xd); free(t);
}

void mfo_sgemvt(int m, int n, const float* A, const float* y, const float* z, float alpha,
                float beta, float* x_out, float* w_out) {
  size_t mn = (size_t)m * (size_t)n;
  double* a = widen(A, mn);
  double* yd = widen(y, (size_t)m);
  double* t = (double*)malloc((size_t)n * sizeof(double));
  double* x = (double*)malloc((size_t)n * sizeof(double));
  double* u = (double*)malloc((size_t)m * sizeof(double));
  double al = alpha, be = beta;
  matvec_t(a, m, n, yd, t);
  for (int j = 0; j < n; ++j) x[j] = be * t[j] + (double)z[j];
  matvec(a, m, n, x, u);
  for (int i = 0; i < m; ++i) w_out[i] = (float)(al * u[i]);
  narrow(x, x_out, (size_t)n);
  free(a); free(yd); free(t); free(x); free(u);
}

void mfo_gemver(int m, int n, const float* A, const float* u1, const float* v1,
                const float* u2, const float* v2, const float* y, const float* z, float alpha,
                float beta, float* B_out, float* x_out, float* w_out) {
  size_t mn = (size_t)m * (size_t)n;
  double* b = (double*)malloc(mn * sizeof(double));
  for (int i = 0; i < m; ++i) {
    double a1 = u1[i], a2 = u2[i];
    for (int j = 0; j < n; ++j) {
      size_t k = (size_t)i * (size_t)n + (size_t)j;
      b[k] = (double)A[k] + a1 * (double)v1[j] + a2 * (double)v2[j];
    }
  }
  double* yd = widen(y, (size_t)m);
  double* t = (double*)malloc((size_t)n * sizeof(double));
  double* x = (double*)malloc((size_t)n * sizeof(double));
  double* w0 = (double*)malloc((size_t)m * sizeof(double));
  double al = alpha, be = beta;
  matvec_t(b, m, n, yd, t);
  for (int j = 0; j < n; ++j) x[j] = be * t[j] + (double)z[j];
  matvec(b, m, n, x, w0);
  narrow(b, B_out, mn);
  narrow(x, x_out, (size_t)n);
  for (int i = 0; i < m; ++i) w_out[i] = (float)(al * w0[i]);
  free(b); free(yd); free(t); free(x); free(w0);
}

void mfo_gesummv(int m, int n, const float* A, const float* B, const float* x, float alpha,
                 float beta, float* y_out) {
  size_t mn = (size_t)m * (size_t)n;
  double* xd = widen(x, (size_t)n);
  double* a = widen(A, mn);
  double* t1 = (double*)malloc((size_t)m * sizeof(double));
  matvec(a, m, n, xd, t1);
  free(a);
  double* bb = widen(B, mn);
  double* t2 = (double*)malloc((size_t)m * sizeof(double));
  matvec(bb, m, n, xd, t2);
  free(bb);
  double al = alpha, be = beta;
  for (int i = 0; i < m; ++i) y_out[i] = (float)(al * t1[i] + be * t2[i]);
  free(xd); free(t1); free(t2);
}

/* ------------------------------------------------------------------------ */
/* reference_call restatement (blas.cpp:287-338): one library call, fp64,    */
/* narrowed to float afterwards.  Used to pin the unfused (one kernel per    */
/* call) GPU chain, whose kernels round at every call boundary.              */

void mfo_call_add(int n, const float* a, const float* b, float* c) {
  for (int i = 0; i < n; ++i) c[i] = (float)((double)a[i] + (double)b[i]);
}
void mfo_call_scal(int n, float alpha, const float* v, float* x) {
  double a = alpha;
  for (int i = 0; i < n; ++i) x[i] = (float)(a * (double)v[i]);
}
void mfo_call_waxpby(int n, float alpha, const float* x, float beta, const float* y, float* w) {
  double a = alpha, b = beta;
  for (int i = 0; i < n; ++i) w[i] = (float)(a * (double)x[i] + b * (double)y[i]);
}
void mfo_call_axpydot_stage(int n, const float* w, float alpha, const float* v, float* z) {
  double a = alpha;
  for (int i = 0; i < n; ++i) z[i] = (float)((double)w[i] - a * (double)v[i]);
}
void mfo_call_dot(int n, const float* x, const float* y, float* r) {
  double acc = 0.0;
  for (int i = 0; i < n; ++i) acc += (double)x[i] * (double)y[i];
  *r = (float)acc;
}
void mfo_call_ger2(int m, int n, const float* A, const float* u1, const float* v1,
                   const float* u2, const float* v2, float* B) {
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) {
      size_t k = (size_t)i * (size_t)n + (size_t)j;
      B[k] = (float)((double)A[k] + (double)u1[i] * (double)v1[j] +
                     (double)u2[i] * (double)v2[j]);
    }
}
/* sgemv (scaled=0) / sgemvs (scaled=1): y = [alpha *] A x */
void mfo_call_sgemv(int m, int n, int scaled, float alpha, const float* A, const float* x,
                    float* y) {
  size_t mn = (size_t)m * (size_t)n;
  double* a = widen(A, mn);
  double* xd = widen(x, (size_t)n);
  double* t = (double*)malloc((size_t)m * sizeof(double));
  matvec(a, m, n, xd, t);
  if (scaled) {
    double al = alpha;
    for (int i = 0; i < m; ++i) t[i] *= al;
  }
  narrow(t, y, (size_t)m);
  free(a); free(xd); free(t);
}
void mfo_call_sgemtv(int m, int n, const float* A, const float* x, float* y) {
  size_t mn = (size_t)m * (size_t)n;
  double* a = widen(A, mn);
  double* xd = widen(x, (size_t)m);
  double* t = (double*)malloc((size_t)n * sizeof(double));
  matvec_t(a, m, n, xd, t);
  narrow(t, y, (size_t)n);
  free(a); free(xd); free(t);
}

/* ------------------------------------------------------------------------ */
/* Sampled fp64 checks for the generated (hash) matrices at sizes that do    */
/* not fit host memory: A[i][j] = hash(seed, i*n+j).   */

/* q_i = sum_j A[i][j] * x[j] and |A||x| for the listed rows. */
void mfo_hash_rows(uint64_t seed, int64_t n, const int64_t* rows, int nrows, const float* x,
                   double* out, double* absout) {
  for (int k = 0; k < nrows; ++k) {
    double acc = 0.0, aacc = 0.0;
    uint64_t base = (uint64_t)rows[k] * (uint64_t)n;
    for (int64_t j = 0; j < n; ++j) {
      double a = (double)mfo_hash_uniform(seed, base + (uint64_t)j);
      acc += a * (double)x[j];
      aacc += fabs(a) * fabs((double)x[j]);
    }
    out[k] = acc;
    absout[k] = aacc;
  }
}

/* s_j = sum_i A[i][j] * r[i] for the listed columns, i over [row0, row1). */
void mfo_hash_cols(uint64_t seed, int64_t n, int64_t row0, int64_t row1, const int64_t* cols,
                   int ncols, const float* r, double* out, double* absout) {
  for (int k = 0; k < ncols; ++k) { out[k] = 0.0; absout[k] = 0.0; }
  for (int64_t i = row0; i < row1; ++i) {
    double ri = (double)r[i - row0];
    uint64_t base = (uint64_t)i * (uint64_t)n;
    for (int k = 0; k < ncols; ++k) {
      double a = (double)mfo_hash_uniform(seed, base + (uint64_t)cols[k]);
      out[k] += a * ri;
      absout[k] += fabs(a) * fabs(ri);
    }
  }
}

/* Multi-threaded helpers (pthreads; the image has no libgomp).             */
#include <pthread.h>

typedef struct {
  void (*fn)(void* ctx, int64_t i);
  void* ctx;
  int64_t lo, hi, step;
} mfo_range;

static void* mfo_range_run(void* p) {
  mfo_range* r = (mfo_range*)p;
  for (int64_t i = r->lo; i < r->hi; i += r->step) r->fn(r->ctx, i);
  return NULL;
}

/* fn(ctx, i) for i in [0, count), index i on thread i % nthreads. */
static void mfo_parallel_for(int64_t count, int nthreads, void (*fn)(void*, int64_t), void* ctx) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  mfo_range rg[256];
  for (int t = 0; t < nthreads; ++t) {
    rg[t].fn = fn;
    rg[t].ctx = ctx;
    rg[t].lo = t;
    rg[t].hi = count;
    rg[t].step = nthreads;
    if (t > 0) pthread_create(&th[t], NULL, mfo_range_run, &rg[t]);
  }
  mfo_range_run(&rg[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
}

static double mfo_hash_value(uint64_t hs, uint64_t index) {
  const uint64_t h = splitmix64(index ^ hs);
  return (double)((float)(uint32_t)(h >> 40) * (1.0f / 8388608.0f) - 1.0f);
}

/* y = A x and |A||x| for EVERY row of a hash-generated m x n matrix, fp64,   */
/* rows interleaved over `nthreads` threads (the chained ATAX check at        */
/* 131072^2 needs the whole intermediate t = A x).  Each */
/* row's sum runs in column order, like mfo_hash_rows.                        */
typedef struct {
  uint64_t hs;
  int64_t n;
  const float* x;
  double *out, *absout;
} mfo_matvec_ctx;

static void mfo_matvec_row(void* p, int64_t i) {
  const mfo_matvec_ctx* c = (const mfo_matvec_ctx*)p;
  double acc = 0.0, aacc = 0.0;
  const uint64_t base = (uint64_t)i * (uint64_t)c->n;
  for (int64_t j = 0; j < c->n; ++j) {
    const double a = mfo_hash_value(c->hs, base + (uint64_t)j);
    acc += a * (double)c->x[j];
    aacc += fabs(a) * fabs((double)c->x[j]);
  }
  c->out[i] = acc;
  c->absout[i] = aacc;
}

void mfo_hash_matvec_all(uint64_t seed, int64_t m, int64_t n, const float* x, double* out,
                         double* absout, int nthreads) {
  mfo_matvec_ctx c = {splitmix64(seed), n, x, out, absout};
  mfo_parallel_for(m, nthreads, mfo_matvec_row, &c);
}

/* y_j = sum_i A[i][j] t_i and sum_i |A[i][j]| tabs_i for the listed columns, */
/* i over [0, m), with fp64 row weights (t = the fp64 intermediate of a       */
/* chained reduction, tabs its |.|-formula); columns split over threads.     */
typedef struct {
  uint64_t hs;
  int64_t n, m;
  const int64_t* cols;
  const double *t, *tabs;
  double *out, *absout;
} mfo_cols_ctx;

static void mfo_cols_one(void* p, int64_t k) {
  const mfo_cols_ctx* c = (const mfo_cols_ctx*)p;
  double acc = 0.0, aacc = 0.0;
  for (int64_t i = 0; i < c->m; ++i) {
    const double a = mfo_hash_value(c->hs, (uint64_t)i * (uint64_t)c->n + (uint64_t)c->cols[k]);
    acc += a * c->t[i];
    aacc += fabs(a) * c->tabs[i];
  }
  c->out[k] = acc;
  c->absout[k] = aacc;
}

void mfo_hash_cols_f64(uint64_t seed, int64_t n, int64_t m, const int64_t* cols, int ncols,
                       const double* t, const double* tabs, double* out, double* absout,
                       int nthreads) {
  mfo_cols_ctx c = {splitmix64(seed), n, m, cols, t, tabs, out, absout};
  mfo_parallel_for(ncols, nthreads, mfo_cols_one, &c);
}
