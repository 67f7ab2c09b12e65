/* A plain-C client of the C-ABI (include/mapfuse_b200.h): what a non-C++
 * caller of the reference's execution path links against.  Compiles the
 * shipped VADD sequence, runs it on host buffers, checks x = w + y + z. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "mapfuse_b200.h"

int main(void) {
  const int n = 1 << 20;
  float *w = malloc(sizeof(float) * n), *y = malloc(sizeof(float) * n);
  float *z = malloc(sizeof(float) * n), *x = malloc(sizeof(float) * n);
  for (int i = 0; i < n; ++i) {
    w[i] = (float)i * 0.5f;
    y[i] = 1.0f;
    z[i] = -0.25f;
    x[i] = 0.0f;
  }
  mf_plan* plan = NULL;
  if (mf_compile_sequence("VADD", 1, n, MF_MODE_FUSED, &plan) != MF_OK) {
    fprintf(stderr, "compile: %s\n", mf_last_error());
    return 1;
  }
  mf_buffer bufs[4] = {{"w", 1, n, w}, {"y", 1, n, y}, {"z", 1, n, z}, {"x", 1, n, x}};
  mf_stats st;
  if (mf_launch_host(plan, bufs, 4, NULL, 0, &st) != MF_OK) {
    fprintf(stderr, "launch: %s\n", mf_last_error());
    return 1;
  }
  for (int i = 0; i < n; ++i)
    if (x[i] != (float)((double)w[i] + (double)y[i] + (double)z[i])) {
      fprintf(stderr, "mismatch at %d\n", i);
      return 1;
    }
  if (st.kernels != 1 || st.bytes_loaded != 12ull * n || st.bytes_stored != 4ull * n) {
    fprintf(stderr, "unexpected stats\n");
    return 1;
  }
  /* errors come back as status codes + message */
  mf_buffer bad[1] = {{"w", 1, n, w}};
  int rc = mf_launch_host(plan, bad, 1, NULL, 0, &st);
  if (rc != MF_ERR_FAULT) return 1;
  printf("c-abi client ok (%.3f ms, %s)\n", st.ms, mf_version());
  mf_plan_destroy(plan);
  free(w); free(y); free(z); free(x);
  return 0;
}
