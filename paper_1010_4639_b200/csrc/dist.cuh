// dist.cuh — per-pass CG kernels for the row-sharded multi-GPU solve.
//
// Each rank owns lines [row0,row1) of A (a "local" handle whose column
// indices are localized: owned columns -> [0,nloc), halo columns ->
// [nloc, nloc+nhalo)).  The gathered vectors are stored extended:
//   r_ext[0..nloc)       own residual
//   r_ext[nloc..)        halo: the neighbours' p_k values for this iteration
//   p_ext[*][nloc..)     always 0
// so the fold r_j + beta*p_j gives own p_k for owned j and exactly the
// received p_k for halo j — the same tile kernels serve both cases.
// Scalars live in a device StepState; the two per-iteration dot products
// are reduced in fixed order on each rank (last-CTA-done) and summed across
// ranks by ncclAllReduce on StepState::red, so every rank computes bitwise
// identical alpha/beta/flags and stops at the same iteration.
#pragma once
#include "lines.cuh"

namespace spcg {

struct StepState {
  double rr, alpha, beta, b_norm, rel, tol;
  double red;  // local partial sum; NCCL all-reduces it in place
  double pad0;
  long long k, max_it, fail_iter;
  int status, converged, done, x0_given;
  unsigned int counter;  // last-CTA-done ticket
  int record;
};

// Fixed-order grid reduction without a grid barrier: every CTA writes its
// block sum to part[], the last CTA to arrive sums part[] in index order.
struct RedSmem {
  double red[32];
  double bcast;
};

template <class SM>
__device__ __forceinline__ void last_block_sum(double v, SM& sm, double* part, StepState* S) {
  const double bs = block_sum(v, sm);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = bs;
    __threadfence();
    const unsigned int t = atomicAdd(&S->counter, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double s = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) s += __ldcg(part + i);
  s = block_sum(s, sm);
  if (threadIdx.x == 0) {
    S->red = s;
    S->counter = 0;
  }
}

// pass A: p_k = fold, q = A p_k, x += alpha_{k-1} p_{k-1}, red = p.q partial
#ifndef SPCG_DIST_MINB
#define SPCG_DIST_MINB 2
#endif
template <int FMT>
__global__ void __launch_bounds__(kBlock, SPCG_DIST_MINB)
    dist_pass_a(const MatView M, StepState* S, const double* r_ext, const double* p_old,
                double* p_new, double* x, double* q, double* part) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  if (S->done) return;
  constexpr bool TWO = (FMT == K_SCSR_PRIV);
  const bool first = S->k == 0;
  const double beta = S->beta, alpha = S->alpha;
  smem_init(sm);
  Pipe P;
  pipe_start<TWO>(P, sm, M);
  double pq = 0.0;
  for (int j = 0; j < P.m; ++j) {
    const int s = pipe_acquire(P, sm, j);
    bool active = false;
    int i = -1;
    LineOut o;
    if (first) {
      SrcFirst src{r_ext};
      o = tile_line<FMT, false>(sm, s, M, src, q, active, i, sm.val[s]);
    } else {
      SrcFold src{r_ext, p_old, beta};
      o = tile_line<FMT, false>(sm, s, M, src, q, active, i, sm.val[s], x);
    }
    if (active) {
      if (!first) x[i] = mul_add_rn(o.xo, alpha, p_old[i]);
      p_new[i] = o.xi;
      q[i] = o.q;
      pq += line_pq<FMT>(o);
    }
    pipe_release<TWO>(P, sm, M, s);
  }
  pipe_drain(P, sm);
  last_block_sum(pq, sm, part, S);
}

// y = A x_ext (plain gather; initial / true residual)
template <int FMT>
__global__ void __launch_bounds__(kBlock, 2)
    dist_spmv(const MatView M, const double* x_ext, double* y) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  constexpr bool TWO = (FMT == K_SCSR_PRIV);
  smem_init(sm);
  Pipe P;
  pipe_start<TWO>(P, sm, M);
  SrcPlain src{x_ext};
  for (int j = 0; j < P.m; ++j) {
    const int s = pipe_acquire(P, sm, j);
    bool active = false;
    int i = -1;
    const LineOut o = tile_line<FMT, false>(sm, s, M, src, y, active, i, sm.val[s]);
    if (active) y[i] = o.q;
    pipe_release<TWO>(P, sm, M, s);
  }
  pipe_drain(P, sm);
}

// Elementwise kernels over the nloc own lines (grid-stride, fixed order).
// mode 0: red = b.b               mode 1: r = b - q (or b), red = r.r
// mode 2: r -= alpha q, red = r.r mode 3: red = |b - q|^2 (true residual)
__global__ void __launch_bounds__(kBlock) dist_elem(int mode, long long nloc, StepState* S,
                                                   const double* b, const double* q, double* r,
                                                   double* part) {
  __shared__ RedSmem sm;
  if (mode == 2 && S->done) return;
  const double alpha = S->alpha;
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long G = (long long)gridDim.x * blockDim.x;
  double acc = 0.0;
  for (long long i = g; i < nloc; i += G) {
    double v;
    if (mode == 0) {
      v = b[i];
    } else if (mode == 1) {
      v = q ? mul_add_rn(b[i], -1.0, q[i]) : b[i];
      r[i] = v;
    } else if (mode == 2) {
      v = mul_add_rn(r[i], -alpha, q[i]);
      r[i] = v;
    } else {
      v = mul_add_rn(b[i], -1.0, q[i]);
    }
    acc = fma(v, v, acc);
  }
  last_block_sum(acc, sm, part, S);
}

// Scalar steps (one thread), operating on the all-reduced S->red.
// op 0: after ||b||^2          op 1: after r0.r0 (start)
// op 2: after p.q (alpha)      op 3: after r.r (convergence, beta)
// op 4: after the true residual
__global__ void dist_scalar(int op, StepState* S, double* hist) {
  if (op == 0) {
    S->b_norm = sqrt(S->red);
    S->k = 0;
    S->status = 0;
    S->converged = 0;
    S->fail_iter = 0;
    S->alpha = 0.0;
    S->beta = 0.0;
    if (S->b_norm == 0.0) {
      S->done = 1;
      S->converged = 1;
      S->rel = 0.0;
    } else {
      S->done = 0;
    }
    return;
  }
  if (op == 1) {
    if (S->b_norm == 0.0) return;
    S->rr = S->red;
    S->rel = sqrt(S->rr) / S->b_norm;
    if (sqrt(S->rr) <= S->tol * S->b_norm) {
      S->converged = 1;
      S->done = 1;
    } else if (S->max_it <= 0) {
      S->done = 1;
    }
    return;
  }
  if (S->done) return;
  if (op == 2) {
    const double pq = S->red;
    if (pq <= 0.0) {
      S->status = 3;
      S->fail_iter = S->k + 1;
      S->done = 1;
      return;
    }
    S->alpha = S->rr / pq;
    if (!isfinite(S->alpha)) {
      S->status = 4;
      S->fail_iter = S->k + 1;
      S->done = 1;
    }
    return;
  }
  if (op == 3) {
    const double rr_new = S->red;
    const long long k = S->k + 1;
    S->rel = sqrt(rr_new) / S->b_norm;
    if (!isfinite(S->rel)) {
      S->status = 5;
      S->fail_iter = k;
      S->done = 1;
      return;
    }
    if (S->record && hist) hist[k - 1] = S->rel;
    S->k = k;
    if (sqrt(rr_new) <= S->tol * S->b_norm) {
      S->converged = 1;
      S->rr = rr_new;
      S->done = 1;
      return;
    }
    const double beta = rr_new / S->rr;
    if (!isfinite(beta)) {
      S->status = 6;
      S->fail_iter = k;
      S->done = 1;
      return;
    }
    S->beta = beta;
    S->rr = rr_new;
    if (k >= S->max_it) S->done = 1;
    return;
  }
}

__global__ void dist_true_rel(StepState* S) { S->rel = sqrt(S->red) / S->b_norm; }

// Halo values to send: mode 0 plain v[idx]; mode 1 next direction
// p_k = r + beta p_{k-1} (first iteration: r), skipped once done.
__global__ void dist_pack(int mode, StepState* S, long long cnt, const int* idx, const double* r,
                          const double* p, double* out) {
  if (mode == 1 && S->done) return;
  const bool first = S->k == 0;
  const double beta = S->beta;
  const long long G = (long long)gridDim.x * blockDim.x;
  for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < cnt; s += G) {
    const int i = idx[s];
    out[s] = (mode == 0 || first) ? r[i] : __dadd_rn(r[i], __dmul_rn(beta, p[i]));
  }
}

// x = x0 (or 0); final x += alpha_K p_K
__global__ void dist_x(int mode, long long nloc, StepState* S, const double* src, double* x) {
  const long long G = (long long)gridDim.x * blockDim.x;
  const double alpha = S->alpha;
  const bool upd = S->k > 0 && S->status == 0;
  const bool zero_b = S->b_norm == 0.0;  // solver.py:109-118: x = 0 even for x0 != 0
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nloc; i += G) {
    if (mode == 0) x[i] = (src && !zero_b) ? src[i] : 0.0;
    else if (upd) x[i] = mul_add_rn(x[i], alpha, src[i]);
  }
}

}  // namespace spcg
