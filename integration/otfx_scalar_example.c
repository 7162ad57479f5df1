/* A C caller of the engine, no Python anywhere: the reference's Dirac-pair
 * fixture (T/test_solver.py:70-77, `solve_scalar` of two unit point masses on
 * a 33 x 33 grid, tau = 3, default SolverConfig) through the C ABI of
 * include/otfx.h -- what a cgo / JNI / N-API binding of otflux would call.
 *
 *   gcc -std=c99 -I include integration/otfx_scalar_example.c \
 *       -L paper_1712_10279_b200 -l:libotfx.so -Wl,-rpath,$PWD/paper_1712_10279_b200
 *
 * Prints: iterations converged W1 (the reference's value is 0.5 +- 2 %). */
#include <stdio.h>
#include <stdlib.h>

#include "otfx.h"

#define CHECK(call)                                                       \
  do {                                                                    \
    if ((call) != OTFX_OK) {                                              \
      fprintf(stderr, "%s failed: %s\n", #call, otfx_last_error());       \
      return 1;                                                           \
    }                                                                     \
  } while (0)

int main(void) {
  const int n = 33;
  const double tau = 3.0;
  /* step sizes exactly as the reference computes them (S/solver.py:71-74,
   * dx = 1 / (n - 1), inv_dx = 1 / dx) */
  const double dx = 1.0 / (n - 1);
  otfx_engine_desc d = {0};
  d.kind = OTFX_KIND_SCALAR;
  d.dtype = OTFX_F64;
  d.n = n;
  d.k = 1;
  d.ell = 0;
  d.norm_u = OTFX_NORM_L2;
  d.norm_w = OTFX_NORM_L1;
  d.device = 0;
  d.row_begin = 0;
  d.row_end = n;
  d.tau = tau;
  d.mu = 1.0 / (16.0 * tau * (double)(n - 1) * (double)(n - 1));
  d.nu = 0.0;
  d.alpha = 1.0;
  d.eps_reg = 0.0;
  d.inv_dx = 1.0 / dx;

  double* l0 = calloc((size_t)n * n, sizeof(double));
  double* l1 = calloc((size_t)n * n, sizeof(double));
  if (!l0 || !l1) return 1;
  l0[8 * n + 16] = 1.0; /* dirac_pair(GridSpec(33), (8, 16), (24, 16)) */
  l1[24 * n + 16] = 1.0;

  otfx_engine* e = NULL;
  CHECK(otfx_engine_create(&d, &e));
  double masses[2];
  CHECK(otfx_engine_set_marginals(e, l0, l1, masses));
  otfx_run_config cfg = {1e-3, 1e-5, 200000, 100}; /* SolverConfig defaults */
  int64_t nh = 0, iters = 0;
  int converged = 0;
  double wall = 0.0;
  CHECK(otfx_engine_run(e, &cfg, NULL, 0, &nh, &iters, &converged, &wall));
  otfx_history_point* h = malloc((size_t)nh * sizeof(otfx_history_point));
  if (!h) return 1;
  CHECK(otfx_engine_history(e, h, nh, &nh));
  printf("%lld %d %.17g\n", (long long)iters, converged, h[nh - 1].primal);
  CHECK(otfx_engine_destroy(e));
  free(h);
  free(l0);
  free(l1);
  return 0;
}
