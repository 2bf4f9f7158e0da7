/* Plain-C consumer of include/liecl_b200.h (no C++, no Python): the su(2)
 * closure of i*X and i*Z through liecl_b200_closure_dense. Build:
 *   gcc -std=c11 -Iinclude examples/c_abi_demo.c -Lpaper_2506_01120_b200/lib \
 *       -lliecl_b200 -Wl,-rpath,paper_2506_01120_b200/lib -o c_abi_demo        */
#include <stdio.h>
#include <string.h>

#include "liecl_b200.h"

int main(void) {
  liecl_b200_ctx* ctx = NULL;
  if (liecl_b200_ctx_create(0, &ctx) != LIECL_B200_OK) {
    fprintf(stderr, "no device: %s\n", liecl_b200_last_error());
    return 2;
  }
  /* column-major 2x2 complex (re, im interleaved): i*X and i*Z */
  const double gens[2][8] = {{0, 0, 0, 1, 0, 1, 0, 0}, {0, 1, 0, 0, 0, 0, 0, -1}};
  double basis[4][8];
  liecl_b200_config cfg;
  memset(&cfg, 0, sizeof cfg);
  cfg.tolerance = 1e-10;
  liecl_b200_stats st;
  char warnings[256];
  const int s = liecl_b200_closure_dense(ctx, &gens[0][0], 2, 2, LIECL_B200_METHOD_ORTHONORM_DIMONLY, &cfg,
                                         &basis[0][0], NULL, 4, &st, warnings, sizeof warnings, NULL, 0, NULL);
  if (s != LIECL_B200_OK) {
    fprintf(stderr, "closure failed (%d): %s\n", s, liecl_b200_last_error());
    return 1;
  }
  printf("dimension %llu, brackets %llu\n", (unsigned long long)st.dimension,
         (unsigned long long)st.commutators_evaluated);
  liecl_b200_ctx_destroy(ctx);
  return st.dimension == 3 ? 0 : 1;
}
