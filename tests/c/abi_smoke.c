/* Plain-C consumer of the sgm C ABI (include/sgm.h): no Python, no torch.  Creates a host-only
   plan (device = -1: queries only), checks the form lengths against a = n+p-2, b = n+p-1
   (N_e = 3 a^2 b, N_h = 3 a b^2 for a cube), reads one 1D table and checks that a
   compute call on a host-only plan is refused with SGM_E_INVALID_ARG.  Exit code 0 on success. */
#include <stdio.h>
#include <stdlib.h>

#include "sgm.h"

int main(void) {
  sgm_plan_desc desc = {{10, 10, 10}, 3, NULL, 0, -1};
  sgm_plan plan = NULL;
  if (sgm_plan_create(&desc, &plan) != SGM_OK) { printf("create: %s\n", sgm_last_error()); return 1; }
  size_t ne = 0, nh = 0;
  sgm_plan_len(plan, SGM_FORM_E, &ne);
  sgm_plan_len(plan, SGM_FORM_H, &nh);
  const size_t a = 11, b = 12;
  if (ne != 3 * a * a * b || nh != 3 * a * b * b) { printf("lengths %zu %zu\n", ne, nh); return 2; }
  int L = 0;
  sgm_plan_table(plan, SGM_TAB_G, 0, NULL, &L);
  double* G = (double*)malloc(sizeof(double) * (size_t)L * (size_t)L);
  if (sgm_plan_table(plan, SGM_TAB_G, 0, G, &L) != SGM_OK || L != (int)a) { printf("table\n"); return 3; }
  double colsum = 0.0; /* Hat G = int D''_k B_c: every entry of a CS-by-B-spline pairing is >= 0 */
  for (int i = 0; i < L * L; ++i) { if (G[i] < 0.0) return 4; colsum += G[i]; }
  double dummy = 0.0;
  if (sgm_curl(plan, SGM_CURL_PRIMAL, &dummy, &dummy, NULL) != SGM_E_INVALID_ARG) { printf("host-only plan ran a compute call\n"); return 5; }
  free(G);
  sgm_plan_destroy(plan);
  printf("abi_smoke ok (%s)\n", sgm_version());
  return 0;
}
