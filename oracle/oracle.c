/*
 * oracle.c — TEST INFRASTRUCTURE ONLY.  CPU restatement of the reference's
 * solve path (arxiv/paper_1010_4639, package `spcg`), used as the parity
 * checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.
 * Never linked into or called by the product (paper_1010_4639_b200/).
 *
 * Each function cites the reference code it restates.  Built with
 * -O3 -fopenmp -ffp-contract=off (the reference's setup.py:5-16 builds with
 * -O3 -fopenmp and no -ffast-math; on x86-64 without -mfma that means
 * separately rounded multiply and add, which -ffp-contract=off pins down).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef int64_t idx_t;

/* config.py:37-40 */
static idx_t resolve_chunk(idx_t items, int workers, idx_t chunk) {
  if (chunk > 0) return chunk;
  idx_t c = (items + 8 * (idx_t)workers - 1) / (8 * (idx_t)workers);
  return c < 1 ? 1 : c;
}

/* _ckernels.pyx:31-47 csr_gather: one sequential sum per row. */
void orc_csr_gather(idx_t n, const idx_t* row_start, const idx_t* col_idx, const double* values,
                    const double* x, double* y, int workers) {
  idx_t i;
#pragma omp parallel for num_threads(workers) schedule(static)
  for (i = 0; i < n; ++i) {
    double acc = 0.0;
    for (idx_t k = row_start[i]; k < row_start[i + 1]; ++k) acc = acc + values[k] * x[col_idx[k]];
    y[i] = acc;
  }
}

/* _ckernels.pyx:50-62 scatter_atomic: y[cols[k]] += vals[k]*x[rows[k]].
 * Sequential here (one valid order of the unspecified atomic order). */
void orc_scatter_seq(idx_t m, const idx_t* rows, const idx_t* cols, const double* vals,
                     const double* x, double* y) {
  for (idx_t k = 0; k < m; ++k) y[cols[k]] += vals[k] * x[rows[k]];
}

/* _ckernels.pyx:65-91 scatter_privatized: chunk c -> worker c mod W, private
 * outputs merged in worker order.  priv must hold workers*n zeros. */
void orc_scatter_privatized(idx_t m, idx_t n, const idx_t* rows, const idx_t* cols,
                            const double* vals, const double* x, double* y, double* priv,
                            int workers, idx_t chunk) {
  idx_t nchunks = m > 0 ? (m + chunk - 1) / chunk : 0;
  int w;
#pragma omp parallel for num_threads(workers) schedule(static)
  for (w = 0; w < workers; ++w) {
    double* pw = priv + (size_t)w * (size_t)n;
    for (idx_t c = w; c < nchunks; c += workers) {
      idx_t lo = c * chunk, hi = lo + chunk;
      if (hi > m) hi = m;
      for (idx_t k = lo; k < hi; ++k) pw[cols[k]] += vals[k] * x[rows[k]];
    }
  }
  for (w = 0; w < workers; ++w)
    for (idx_t j = 0; j < n; ++j) y[j] += priv[(size_t)w * (size_t)n + j];
}

/* config.py:43-56 pairwise_merge: fixed-order pairwise tree (in place). */
double orc_pairwise_merge(double* a, idx_t size) {
  if (size == 0) return 0.0;
  while (size > 1) {
    idx_t half = size / 2, out = 0;
    for (idx_t k = 0; k < half; ++k) a[out++] = a[2 * k] + a[2 * k + 1];
    if (size % 2) a[out++] = a[size - 1];
    size = out;
  }
  return a[0];
}

/* _ckernels.pyx:94-108 dot_partials + _compiled.py:38-46 dot. */
double orc_dot(idx_t n, const double* u, const double* v, int workers, idx_t chunk_cfg) {
  if (n == 0) return 0.0;
  idx_t chunk = resolve_chunk(n, workers, chunk_cfg);
  idx_t nchunks = (n + chunk - 1) / chunk;
  double* part = (double*)malloc(sizeof(double) * (size_t)nchunks);
  idx_t c;
#pragma omp parallel for num_threads(workers) schedule(static)
  for (c = 0; c < nchunks; ++c) {
    double acc = 0.0;
    idx_t hi = (c + 1) * chunk;
    if (hi > n) hi = n;
    for (idx_t k = c * chunk; k < hi; ++k) acc = acc + u[k] * v[k];
    part[c] = acc;
  }
  double r = orc_pairwise_merge(part, nchunks);
  free(part);
  return r;
}

/* _ckernels.pyx:111-117 axpy_kernel + _compiled.py:49-57 (alpha==0 copies v). */
void orc_axpy(idx_t n, double alpha, const double* u, const double* v, double* out, int workers) {
  if (alpha == 0.0) {
    memmove(out, v, sizeof(double) * (size_t)n);
    return;
  }
  idx_t i;
#pragma omp parallel for num_threads(workers) schedule(static)
  for (i = 0; i < n; ++i) out[i] = v[i] + alpha * u[i];
}

/* Matrix passed to the CG restatement.  kind 0: full CSR (spmv_full);
 * kind 1: symmetric half L+D with its strictly-lower COO (spmv_sym,
 * _compiled.py:22-35; acc 0 = atomic (sequential scatter), 1 = privatized). */
typedef struct {
  int kind;
  int acc;
  idx_t n;
  const idx_t* row_start;
  const idx_t* col_idx;
  const double* values;
  idx_t m_strict;
  const idx_t* s_rows;
  const idx_t* s_cols;
  const double* s_vals;
} orc_matrix;

static void spmv(const orc_matrix* A, const double* x, double* y, int workers, idx_t chunk_cfg,
                 double* priv) {
  orc_csr_gather(A->n, A->row_start, A->col_idx, A->values, x, y, workers);
  if (A->kind == 1) {
    if (A->acc == 0) {
      orc_scatter_seq(A->m_strict, A->s_rows, A->s_cols, A->s_vals, x, y);
    } else {
      idx_t chunk = resolve_chunk(A->m_strict, workers, chunk_cfg);
      memset(priv, 0, sizeof(double) * (size_t)workers * (size_t)A->n);
      orc_scatter_privatized(A->m_strict, A->n, A->s_rows, A->s_cols, A->s_vals, x, y, priv,
                             workers, chunk);
    }
  }
}

/* Status codes shared with include/spcg_b200.h. */
enum { ORC_OK = 0, ORC_NOT_SPD = 3, ORC_NF_ALPHA = 4, ORC_NF_RES = 5, ORC_NF_BETA = 6 };

typedef struct {
  idx_t iterations;
  int converged;
  int status;
  idx_t fail_iteration;
  double final_rel;
  double b_norm;
} orc_result;

/* solver.py:65-172 cg_solve, operation for operation.  hist may be NULL;
 * x0 may be NULL.  max_iter <= 0 means max(1, n). */
int orc_cg_solve(const orc_matrix* A, const double* b, const double* x0, double* x, double tol,
                 idx_t max_iter, int recompute, double* hist, int workers, idx_t chunk_cfg,
                 orc_result* res) {
  const idx_t n = A->n;
  if (max_iter <= 0) max_iter = n > 1 ? n : 1;
  double* r = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* p = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* q = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* t = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* priv = A->kind == 1 && A->acc == 1
                     ? (double*)malloc(sizeof(double) * (size_t)workers * (size_t)(n + 1))
                     : NULL;
  memset(res, 0, sizeof(*res));
  double b_norm = sqrt(orc_dot(n, b, b, workers, chunk_cfg));
  res->b_norm = b_norm;
  if (b_norm == 0.0) { /* solver.py:109-118 */
    memset(x, 0, sizeof(double) * (size_t)n);
    res->converged = 1;
    goto done;
  }
  if (x0) memcpy(x, x0, sizeof(double) * (size_t)n);
  else memset(x, 0, sizeof(double) * (size_t)n);
  spmv(A, x, q, workers, chunk_cfg, priv);          /* q0 = A x */
  orc_axpy(n, -1.0, q, b, r, workers);               /* r = b - q0 */
  memcpy(p, r, sizeof(double) * (size_t)n);
  double rr = orc_dot(n, r, r, workers, chunk_cfg);
  double rel = sqrt(rr) / b_norm;
  idx_t iterations = 0;
  int converged = 0;
  if (sqrt(rr) <= tol * b_norm) {
    converged = 1;
    max_iter = 0;
  }
  for (idx_t k = 1; k <= max_iter; ++k) {
    spmv(A, p, q, workers, chunk_cfg, priv);
    double pq = orc_dot(n, p, q, workers, chunk_cfg);
    if (pq <= 0.0) {
      res->status = ORC_NOT_SPD;
      res->fail_iteration = k;
      goto done;
    }
    double alpha = rr / pq;
    if (!isfinite(alpha)) {
      res->status = ORC_NF_ALPHA;
      res->fail_iteration = k;
      goto done;
    }
    orc_axpy(n, alpha, p, x, t, workers);
    memcpy(x, t, sizeof(double) * (size_t)n);
    orc_axpy(n, -alpha, q, r, t, workers);
    memcpy(r, t, sizeof(double) * (size_t)n);
    double rr_new = orc_dot(n, r, r, workers, chunk_cfg);
    rel = sqrt(rr_new) / b_norm;
    if (!isfinite(rel)) {
      res->status = ORC_NF_RES;
      res->fail_iteration = k;
      goto done;
    }
    if (hist) hist[k - 1] = rel;
    iterations = k;
    if (sqrt(rr_new) <= tol * b_norm) {
      converged = 1;
      rr = rr_new;
      break;
    }
    double beta = rr_new / rr;
    if (!isfinite(beta)) {
      res->status = ORC_NF_BETA;
      res->fail_iteration = k;
      goto done;
    }
    orc_axpy(n, beta, p, r, t, workers); /* p = r + beta p */
    memcpy(p, t, sizeof(double) * (size_t)n);
    rr = rr_new;
  }
  if (recompute) {
    spmv(A, x, q, workers, chunk_cfg, priv);
    orc_axpy(n, -1.0, q, b, t, workers);
    rel = sqrt(orc_dot(n, t, t, workers, chunk_cfg)) / b_norm;
  }
  res->iterations = iterations;
  res->converged = converged;
  res->final_rel = rel;
done:
  free(r);
  free(p);
  free(q);
  free(t);
  free(priv);
  return res->status;
}

/* 7/5/27-point stencils in the reference's sorted-CSR order (genprob.py:50-93
 * for 5/7-point; 27-point is the survey's new generator), int64 arrays, for
 * the CPU baseline at full size without numpy temporaries.  part: 0 full,
 * 1 L+D.  Returns nnz; pass NULL arrays to count only. */
idx_t orc_stencil(int kind, int part, idx_t nx, idx_t ny, idx_t nz, idx_t* row_start,
                  idx_t* col_idx, double* values) {
  const idx_t nxy = nx * ny, n = nxy * nz;
  const double diag = kind == 0 ? 4.0 : (kind == 1 ? 6.0 : 26.0);
  idx_t k = 0;
  if (row_start) row_start[0] = 0;
  for (idx_t i = 0; i < n; ++i) {
    const idx_t ix = i % nx, iy = (i / nx) % ny, iz = i / nxy;
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const int nzc = (dx != 0) + (dy != 0) + (dz != 0);
          if (kind == 0 && (dz != 0 || nzc > 1)) continue;
          if (kind == 1 && nzc > 1) continue;
          const idx_t jx = ix + dx, jy = iy + dy, jz = iz + dz;
          if (jx < 0 || jx >= nx || jy < 0 || jy >= ny || jz < 0 || jz >= nz) continue;
          const idx_t j = i + dz * nxy + dy * nx + dx;
          if (part == 1 && j > i) continue;
          if (col_idx) {
            col_idx[k] = j;
            values[k] = j == i ? diag : -1.0;
          }
          ++k;
        }
    if (row_start) row_start[i + 1] = k;
  }
  return k;
}
