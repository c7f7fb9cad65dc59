/* Plain-C consumer of include/ripple_fv.h on the GPU (no Python, no torch):
 * create -> set_state -> fill_padding -> advance -> max_wavespeed -> get_state ->
 * destroy, plus a deferred numerical-domain error; and a non-trivial run (a random
 * positive state, 3 partitions, periodic x / reflective y, 30 steps) checked against
 * the CPU oracle's C API (oracle/ripple_oracle.h, test infrastructure) at <= 1e-10
 * with the S15 metric, and against the split kernel bitwise.  Built and run by
 * tests/test_abi_gpu_c.py.  Prints "ok" and exits 0 on success. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "ripple_fv.h"
#include "ripple_oracle.h"

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

  /* random positive state (a 64-bit LCG; the oracle gets the same numbers):
   * GPU (3 partitions in y, fused) vs GPU (split kernel) bitwise, vs oracle S15 */
  {
    const int mx = 97, my = 66;
    const size_t m = (size_t)mx * my;
    double* W = malloc(sizeof(double) * C * m);   /* dense SoA for the ABI */
    double* A = malloc(sizeof(double) * C * m);   /* dense AoS for the oracle */
    double* G1 = malloc(sizeof(double) * C * m);
    double* G2 = malloc(sizeof(double) * C * m);
    unsigned long long st = 20210418ull;
    for (size_t i = 0; i < m; ++i) {
      double r[4];
      for (int k = 0; k < 4; ++k) {
        st = st * 6364136223846793005ull + 1442695040888963407ull;
        r[k] = (double)(st >> 11) * (1.0 / 9007199254740992.0);  /* [0, 1) */
      }
      const double rr = 0.5 + r[0], uu = r[1] - 0.5, vv = r[2] - 0.5, pp = 0.5 + r[3];
      const double q[4] = {rr, rr * uu, rr * vv, pp / (g - 1.0) + 0.5 * rr * (uu * uu + vv * vv)};
      for (int k = 0; k < C; ++k) {
        W[k * m + i] = q[k];
        A[i * C + k] = q[k];
      }
    }
    const double dxm = 1.0 / mx, dtm = 0.3 * dxm / 3.0;
    for (int kern = 0; kern < 2; ++kern) {
      rpl_config e;
      rpl_config_init(&e);
      e.ndim = 2;
      e.size[0] = mx;
      e.size[1] = my;
      e.dx[0] = e.dx[1] = dxm;
      e.parts[1] = kern == 0 ? 3 : 1;
      e.kernel = kern == 0 ? RPL_KERNEL_FUSED : RPL_KERNEL_SPLIT;
      e.bc_lo[0] = e.bc_hi[0] = RPL_BC_PERIODIC;
      e.bc_lo[1] = e.bc_hi[1] = RPL_BC_REFLECTIVE;
      rpl_domain* h = NULL;
      CHECK(rpl_create(&e, &h) == RPL_OK && h);
      CHECK(rpl_set_state(h, W) == RPL_OK);
      CHECK(rpl_advance(h, dtm, 30) == RPL_OK);
      CHECK(rpl_get_state(h, kern == 0 ? G1 : G2) == RPL_OK);
      rpl_destroy(h);
    }
    CHECK(memcmp(G1, G2, sizeof(double) * C * m) == 0);
    orc_grid og;
    memset(&og, 0, sizeof(og));
    og.ndim = 2;
    og.n[0] = mx;
    og.n[1] = my;
    og.n[2] = 1;
    og.pad = 2;
    og.dx[0] = og.dx[1] = dxm;
    og.gamma = g;
    og.bc_lo[0] = og.bc_hi[0] = ORC_BC_PERIODIC;
    og.bc_lo[1] = og.bc_hi[1] = ORC_BC_REFLECTIVE;
    og.order = 1;
    CHECK(orc_step_f64(&og, A, dtm, 30) == ORC_OK);
    /* S15: per component max|g - o| / max|o|, momenta sharing one scale */
    double scale[4] = {0, 0, 0, 0}, err[4] = {0, 0, 0, 0};
    for (size_t i = 0; i < m; ++i)
      for (int k = 0; k < C; ++k) {
        const double o = A[i * C + k], gg = G1[k * m + i];
        if (fabs(o) > scale[k]) scale[k] = fabs(o);
        if (fabs(gg - o) > err[k]) err[k] = fabs(gg - o);
      }
    const double mom = scale[1] > scale[2] ? scale[1] : scale[2];
    scale[1] = scale[2] = mom;
    for (int k = 0; k < C; ++k) CHECK(err[k] <= 1e-10 * scale[k]);
    free(W);
    free(A);
    free(G1);
    free(G2);
  }
  printf("ok\n");
  return 0;
}
