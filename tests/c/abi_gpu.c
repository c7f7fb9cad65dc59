/* Plain-C consumer of include/ripple_fv.h on the GPU (no Python, no torch):
 * create -> set_state -> fill_padding -> advance -> max_wavespeed -> get_state ->
 * destroy, plus a deferred numerical-domain error.  Built and run by
 * tests/test_abi_gpu_c.py.  Prints "ok" and exits 0 on success. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "ripple_fv.h"

#define CHECK(cond)                                                          \
  do {                                                                       \
    if (!(cond)) {                                                           \
      fprintf(stderr, "FAILED %s:%d: %s (%s)\n", __FILE__, __LINE__, #cond,  \
              rpl_last_error());                                             \
      return 1;                                                              \
    }                                                                        \
  } while (0)

int main(void) {
  const int nx = 130, ny = 70, C = 4;
  const size_t n = (size_t)nx * ny;
  rpl_config c;
  rpl_config_init(&c);
  c.ndim = 2;
  c.size[0] = nx;
  c.size[1] = ny;
  c.dx[0] = c.dx[1] = 1.0 / nx;
  c.parts[1] = 2; /* two partitions on this rank: halos written by the step kernel */
  rpl_domain* d = NULL;
  CHECK(rpl_create(&c, &d) == RPL_OK && d);

  /* uniform state, dense SoA [C][ny][nx]: a fixed point of the scheme (bitwise) */
  const double rho = 0.9, u = 0.4, v = -0.3, p = 1.2, g = 1.4;
  const double E = p / (g - 1.0) + 0.5 * rho * (u * u + v * v);
  double* U = malloc(sizeof(double) * C * n);
  double* V = malloc(sizeof(double) * C * n);
  for (size_t i = 0; i < n; ++i) {
    U[0 * n + i] = rho;
    U[1 * n + i] = rho * u;
    U[2 * n + i] = rho * v;
    U[3 * n + i] = E;
  }
  CHECK(rpl_set_state(d, U) == RPL_OK);
  CHECK(rpl_fill_padding(d) == RPL_OK);
  double S = 0.0;
  CHECK(rpl_max_wavespeed(d, &S) == RPL_OK);
  const double S_exact = sqrt((rho * u / rho) * (rho * u / rho) + (rho * v / rho) * (rho * v / rho)) +
                         sqrt(g * ((g - 1.0) * (E - 0.5 * (rho * u * rho * u + rho * v * rho * v) / rho)) / rho);
  CHECK(fabs(S - S_exact) <= 1e-14 * S_exact);
  CHECK(rpl_advance(d, 0.4 * c.dx[0] / S, 5) == RPL_OK);
  CHECK(rpl_get_state(d, V) == RPL_OK);
  CHECK(memcmp(U, V, sizeof(double) * C * n) == 0);

  /* negative total energy in one cell: reported at the next synchronising call */
  U[3 * n + 1000] = -1.0;
  CHECK(rpl_set_state(d, U) == RPL_OK);
  CHECK(rpl_advance(d, 1e-4, 1) == RPL_OK); /* enqueued, no host sync */
  CHECK(rpl_synchronize(d) == RPL_E_DOMAIN);
  CHECK(strstr(rpl_last_error(), "domain") != NULL);
  rpl_destroy(d);
  free(U);
  free(V);
  printf("ok\n");
  return 0;
}
