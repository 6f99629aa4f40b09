/* A plain-C client of include/zk_b200.h: what a maintainer binding the
 * library from C (or any FFI) writes. Exit code 0 = all checks passed,
 * 77 = no CUDA device (the library must then fail loudly, which is checked). */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "zk_b200.h"

#define CHECK(x)                                                            \
  do {                                                                      \
    int rc_ = (x);                                                          \
    if (rc_ != ZK_OK) {                                                     \
      fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, zk_last_error());    \
      return 1;                                                             \
    }                                                                       \
  } while (0)

int main(void) {
  /* host-only planner: dedup + counters of (4,2),(4,-2),(2,0),(4,2) */
  int32_t n[4] = {4, 4, 2, 4}, m[4] = {2, -2, 0, 2}, un[4], um[4], sc[4];
  int64_t U = 0, steps = 0, chains = 0;
  CHECK(zk_plan_describe(n, m, 4, un, um, sc, &U));
  if (U != 2 || sc[0] != 0 || sc[1] != 0 || sc[2] != 1 || sc[3] != 0) return 2;
  CHECK(zk_step_counters(n, m, 4, 0, 1, &steps, &chains));
  if (chains != 2) return 3;
  int32_t bad_n = 3, bad_m = 2;
  if (zk_plan_describe(&bad_n, &bad_m, 1, un, um, sc, &U) != ZK_EINVAL) return 4;

  zk_ctx* ctx = NULL;
  int rc = zk_ctx_create(0, &ctx);
  if (rc == ZK_ENODEV || rc == ZK_ECUDA) {
    printf("no device: %s\n", zk_last_error());
    return 77;
  }
  CHECK(rc);
  zk_plan* plan = NULL;
  CHECK(zk_plan_create(ctx, n, m, 4, 3, &plan));
  enum { P = 5 };
  double rho[P] = {0.0, 0.25, 0.5, 0.75, 1.0}, out[P * 4];
  CHECK(zk_radial_eval(ctx, plan, rho, P, 0, 0, out, P, 0, ZK_HOST_INPUT | ZK_HOST_OUTPUT));
  /* R_4^2 = 4 rho^4 - 3 rho^2, R_2^0 = 2 rho^2 - 1 */
  for (int p = 0; p < P; ++p) {
    const double r = rho[p];
    if (fabs(out[0 * P + p] - (4 * r * r * r * r - 3 * r * r)) > 1e-15) return 5;
    if (out[1 * P + p] != out[0 * P + p] || out[3 * P + p] != out[0 * P + p]) return 6;
    if (fabs(out[2 * P + p] - (2 * r * r - 1)) > 1e-15) return 7;
  }
  if (zk_radial_eval(ctx, plan, rho, P, 4, 0, out, P, 0, ZK_HOST_INPUT | ZK_HOST_OUTPUT) !=
      ZK_EINVAL)
    return 8;
  int64_t launches = 0;
  CHECK(zk_ctx_launch_count(ctx, &launches));
  if (launches < 1) return 9;
  CHECK(zk_plan_destroy(plan));
  CHECK(zk_ctx_destroy(ctx));
  printf("capi_demo ok\n");
  return 0;
}
