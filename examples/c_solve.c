/* Plain-C use of the drop-in boundary (include/spcg_b200.h): no Python, no
 * torch.  Builds a 2-D 5-point Poisson system on the host as CSR, solves it
 * through spcg_cg_solve_host (host b -> host x) in full CSR and in
 * symmetric-half storage (both accumulation modes), and checks the true
 * residual on the host.  Exit status 0 = all solves converged and agree.
 *
 *   gcc -O2 -Iinclude examples/c_solve.c -Lpaper_1010_4639_b200/_lib \
 *       -lspcg_b200 -Wl,-rpath,$PWD/paper_1010_4639_b200/_lib -lm -o c_solve
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "spcg_b200.h"

static int check(int rc, const char* what) {
  if (rc != SPCG_OK) fprintf(stderr, "%s failed (%d): %s\n", what, rc, spcg_last_error());
  return rc;
}

/* y = A x for host CSR */
static void host_spmv(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                      const double* x, double* y) {
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) acc += v[k] * x[ci[k]];
    y[i] = acc;
  }
}

int main(int argc, char** argv) {
  const int64_t m = argc > 1 ? atoll(argv[1]) : 96, n = m * m;
  /* full CSR and its lower half (L+D, diagonal last) */
  int64_t* rp = malloc(sizeof(int64_t) * (n + 1));
  int64_t* ci = malloc(sizeof(int64_t) * 5 * n);
  double* v = malloc(sizeof(double) * 5 * n);
  int64_t* lrp = malloc(sizeof(int64_t) * (n + 1));
  int64_t* lci = malloc(sizeof(int64_t) * 3 * n);
  double* lv = malloc(sizeof(double) * 3 * n);
  int64_t k = 0, lk = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t r = i / m, c = i % m;
    rp[i] = k;
    lrp[i] = lk;
    const int64_t nb[5] = {r > 0 ? i - m : -1, c > 0 ? i - 1 : -1, i, c < m - 1 ? i + 1 : -1,
                           r < m - 1 ? i + m : -1};
    for (int t = 0; t < 5; ++t) {
      if (nb[t] < 0) continue;
      ci[k] = nb[t];
      v[k++] = nb[t] == i ? 4.0 : -1.0;
      if (nb[t] < i) {
        lci[lk] = nb[t];
        lv[lk++] = -1.0;
      }
    }
    lci[lk] = i;  /* diagonal last */
    lv[lk++] = 4.0;
  }
  rp[n] = k;
  lrp[n] = lk;
  double* xg = malloc(sizeof(double) * n);
  double* b = malloc(sizeof(double) * n);
  double* x = malloc(sizeof(double) * n);
  double* y = malloc(sizeof(double) * n);
  srand(1);
  for (int64_t i = 0; i < n; ++i) xg[i] = (double)rand() / RAND_MAX - 0.5;
  host_spmv(n, rp, ci, v, xg, b);

  int sms = 0, grid = 0, ma = 0, mi = 0;
  if (check(spcg_device_info(&sms, &grid, &ma, &mi), "spcg_device_info")) return 1;
  printf("device: %d SMs, sm_%d%d, ABI %d\n", sms, ma, mi, spcg_abi_version());

  spcg_matrix_t full = NULL, half = NULL;
  if (check(spcg_matrix_create_host(SPCG_FMT_CSR, n, rp[n], rp, ci, v, &full), "create CSR") ||
      check(spcg_matrix_create_host(SPCG_FMT_SCSR, n, lrp[n], lrp, lci, lv, &half), "create SCSR"))
    return 1;
  const struct { spcg_matrix_t h; int acc; const char* name; } runs[3] = {
      {full, SPCG_ACC_PRIVATIZED, "full CSR"},
      {half, SPCG_ACC_PRIVATIZED, "symmetric half, privatized"},
      {half, SPCG_ACC_ATOMIC, "symmetric half, atomic"}};
  int64_t its0 = -1;
  int bad = 0;
  for (int r = 0; r < 3; ++r) {
    spcg_cg_options o = {0};
    o.tol = 1e-10;
    o.max_iter = 0; /* n */
    o.recompute_final_residual = 1;
    o.accumulation = runs[r].acc;
    spcg_cg_result res = {0};
    if (check(spcg_cg_solve_host(runs[r].h, b, NULL, x, NULL, &o, &res, NULL), "solve")) return 1;
    host_spmv(n, rp, ci, v, x, y);
    double rr = 0.0, bb = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      rr += (b[i] - y[i]) * (b[i] - y[i]);
      bb += b[i] * b[i];
    }
    const double rel = sqrt(rr / bb);
    printf("%-28s iterations %lld converged %d rel %.3e (host check %.3e) %.3f ms\n", runs[r].name,
           (long long)res.iterations, res.converged, res.final_relative_residual, rel,
           res.device_ms);
    if (!res.converged || rel > 1e-9) bad = 1;
    if (its0 < 0) its0 = res.iterations;
    if (llabs(res.iterations - its0) > 1 + its0 / 100) bad = 1;
  }
  spcg_matrix_destroy(full);
  spcg_matrix_destroy(half);
  printf(bad ? "FAILED\n" : "OK\n");
  return bad;
}
