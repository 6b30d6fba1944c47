/* A plain-C caller of the runtime's C ABI (include/iterbatch_b200.h): one Hotspot2D run in graph
 * mode, the same thing the reference's `run_batched(hotspot_program(), state, K, I)` does
 * (pkg/src/iterbatch/workloads.py:453-471), with the T_C / T_E split the paper measures.
 *
 *   gcc -O2 -I include -o /tmp/hotspot_c examples/hotspot_c.c \
 *       -L paper_2501_09398_b200 -literbatch_b200 -Wl,-rpath,$PWD/paper_2501_09398_b200
 *   /tmp/hotspot_c 1024 10000 80
 */
#include <stdio.h>
#include <stdlib.h>

#include "iterbatch_b200.h"

int main(int argc, char **argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 1024;
  const int64_t iters = argc > 2 ? atoll(argv[2]) : 10000;
  const int64_t k = argc > 3 ? atoll(argv[3]) : 80;
  if (k < 1 || iters % k) {
    fprintf(stderr, "batch size %lld must divide %lld\n", (long long)k, (long long)iters);
    return 2;
  }
  const int64_t dims[2] = {n, n};
  const double diffusion = 0.1;
  float *t = malloc((size_t)(n * n) * sizeof(float)), *p = malloc((size_t)(n * n) * sizeof(float));
  unsigned s = 20240817u;
  for (int64_t i = 0; i < n * n; ++i) {  /* any inputs; parity is tested from Python */
    s = s * 1664525u + 1013904223u;
    t[i] = (float)(s >> 8) / 16777216.0f;
    p[i] = t[i] * 1e-3f;
  }
  ib_ctx *ctx = NULL;
  if (ib_create(&ctx, IB_SOLVER_HOTSPOT2D, IB_F32, dims, 2, &diffusion, 1, NULL, 0) != IB_OK) {
    fprintf(stderr, "ib_create: %s\n", ib_last_error());
    return 1;
  }
  const size_t bytes = (size_t)(n * n) * sizeof(float);
  ib_times tc = {0}, te = {0};
  if (ib_upload(ctx, 0, t, bytes) || ib_upload(ctx, 1, p, bytes) ||
      ib_graph_build(ctx, k, IB_BUILD_MANUAL, IB_FLAG_PDL, &tc) ||
      ib_graph_run(ctx, iters / k, &te) || ib_download(ctx, 0, t, bytes)) {
    fprintf(stderr, "run: %s\n", ib_last_error());
    ib_destroy(ctx);
    return 1;
  }
  printf("hotspot2d %lldx%lld, N=%lld, K=%lld: T_C %.1f us (%lld nodes), T_E %.3f ms device, "
         "%.3f us/iteration, T[0]=%.6f\n", (long long)n, (long long)n, (long long)iters, (long long)k,
         1e6 * tc.build_s, (long long)tc.nodes, 1e3 * te.gpu_s, 1e6 * te.gpu_s / (double)iters, t[0]);
  ib_destroy(ctx);
  free(t);
  free(p);
  return 0;
}
