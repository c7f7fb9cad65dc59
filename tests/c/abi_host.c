/* Plain-C consumer of include/ripple_fv.h (no Python, no torch): the host-only
 * entry points -- config defaults and validation, arena sizing, halo plan -- and
 * their error behaviour.  Built and run by tests/test_abi_host.py::test_plain_c_consumer.
 * Prints "ok" and exits 0 on success. */
#include <stdio.h>
#include <string.h>

#include "ripple_fv.h"

#define CHECK(cond)                                                      \
  do {                                                                   \
    if (!(cond)) {                                                       \
      fprintf(stderr, "FAILED %s:%d: %s (%s)\n", __FILE__, __LINE__, #cond, \
              rpl_last_error());                                         \
      return 1;                                                          \
    }                                                                    \
  } while (0)

int main(void) {
  rpl_config c;
  rpl_config_init(&c);
  CHECK(c.ndim == 1 && c.pad == 2 && c.dtype == RPL_F64 && c.layout == RPL_SOA);
  CHECK(c.gamma == 1.4 && c.nranks == 1 && c.order == 1);
  CHECK(strcmp(rpl_kernel_name(NULL, 0), "") == 0);

  /* BASELINE configs[1]: 2-D 1024^2, pad 2, fp64 */
  c.ndim = 2;
  c.size[0] = c.size[1] = 1024;
  c.dx[0] = c.dx[1] = 1.0 / 1024;
  CHECK(rpl_config_check(&c) == RPL_OK);
  size_t bytes = 0;
  CHECK(rpl_arena_bytes(&c, &bytes) == RPL_OK);
  /* two padded buffers of 4 components x 1028 rows x pitch >= 1028 doubles */
  CHECK(bytes >= 2ull * 4 * 1028 * 1028 * 8 && bytes < 2ull * 4 * 1028 * 1200 * 8);

  /* divisibility and pad errors */
  c.parts[1] = 3;
  CHECK(rpl_config_check(&c) == RPL_E_NOT_DIVISIBLE);
  CHECK(strlen(rpl_last_error()) > 0);
  c.parts[1] = 4;
  CHECK(rpl_config_check(&c) == RPL_OK);
  c.order = 2;
  c.pad = 1;
  CHECK(rpl_config_check(&c) == RPL_E_PAD_TOO_SMALL);
  c.pad = 2;
  CHECK(rpl_config_check(&c) == RPL_OK);

  /* halo plan of a 2 x 2 partition grid, periodic in x: every partition receives
   * its ghost boxes from the neighbouring partitions and from itself (BCs) */
  c.order = 1;
  c.parts[0] = 2;
  c.parts[1] = 2;
  c.bc_lo[0] = c.bc_hi[0] = RPL_BC_PERIODIC;
  int32_t n = 0;
  CHECK(rpl_halo_plan(&c, NULL, 0, &n) == RPL_OK && n > 0);
  rpl_halo_edge edges[512];
  CHECK(n <= 512);
  CHECK(rpl_halo_plan(&c, edges, 512, &n) == RPL_OK);
  int64_t ghost_cells = 0;
  for (int i = 0; i < n; ++i) {
    int64_t v = 1;
    for (int d = 0; d < 2; ++d) v *= edges[i].dst_hi[d] - edges[i].dst_lo[d];
    CHECK(v > 0);
    ghost_cells += v;
  }
  /* every ghost cell of every partition has exactly one source:
   * 4 partitions x ((512 + 4)^2 - 512^2) ghost cells */
  CHECK(ghost_cells == 4ll * ((516ll * 516) - 512ll * 512));
  printf("ok\n");
  return 0;
}
