/* rd_demo.c — the C-ABI of librd.so used from plain C (no Python, no torch).
 *
 *   gcc -O2 -I include examples/rd_demo.c -L paper_2409_17658_b200 -lrd \
 *       -Wl,-rpath,$PWD/paper_2409_17658_b200 -o rd_demo
 *   ./rd_demo host        # host-only calls (no GPU needed)
 *   ./rd_demo 7 100       # gamma_R(P_7 [] C_100) and the recurrence for m = 7 (GPU)
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "rd.h"

static int host_only(void) {
  int64_t N = 0;
  if (rd_build_states(5, NULL, &N) != RD_OK) return 1;
  char *w = (char *)malloc((size_t)N * 5);
  rd_build_states(5, w, &N);
  int16_t *A = (int16_t *)malloc((size_t)(N * N) * sizeof(int16_t));
  rd_build_matrix(5, A, &N);
  int64_t nnz = 0;
  for (int64_t e = 0; e < N * N; ++e) nnz += A[e] < RD_INF;
  printf("m=5: N=%lld first=%.5s last=%.5s nnz=%lld\n", (long long)N, w, w + (N - 1) * 5, (long long)nnz);
  /* the closed form from a recurrence (host logic only): gamma(n) = ceil(2n/3) for m = 1 */
  int32_t diag[10] = {INT32_MAX, 0, 2, 2, 3, 4, 4, 5, 6, 6};
  rd_period_t per = {1, 6, 3, 2, 9};
  rd_formula_t f;
  if (rd_closed_form_from(&per, diag, &f, NULL) != RD_OK) return 1;
  printf("m=1 closed form: alpha=%d beta=%d d=(%d,%d,%d) n_valid=%d\n", f.alpha, f.beta, f.d[0], f.d[1], f.d[2],
         f.n_valid);
  /* errors come back as statuses with a message */
  int rc = rd_build_matrix(0, NULL, &N);
  printf("rd_build_matrix(0): %d \"%s\"\n", rc, rd_last_error());
  free(w);
  free(A);
  return 0;
}

int main(int argc, char **argv) {
  if (argc > 1 && strcmp(argv[1], "host") == 0) return host_only();
  const int m = argc > 1 ? atoi(argv[1]) : 7;
  const int64_t n = argc > 2 ? atoll(argv[2]) : 100;
  rd_period_t per;
  int32_t diag[51];
  int rc = rd_power_sequence(m, 50, &per, diag);
  if (rc < 0) { fprintf(stderr, "rd_power_sequence: %s\n", rd_last_error()); return 1; }
  printf("m=%d: n0=%d alpha=%d beta=%d (k_stop=%d)\n", m, per.n0, per.alpha, per.beta, per.k_stop);
  int64_t g = 0;
  if (rd_roman_cylinder(m, n, &g) != RD_OK) { fprintf(stderr, "%s\n", rd_last_error()); return 1; }
  printf("gamma_R(P_%d [] C_%lld) = %lld\n", m, (long long)n, (long long)g);
  return 0;
}
