// dist.cuh — per-pass CG kernels: the row-sharded multi-GPU solve and the
// single-GPU streaming engine (the same engine with no peers).
//
// Each rank owns lines [row0,row1) of A (a "local" handle whose column
// indices are localized: owned columns -> [0,nloc), halo columns ->
// [nloc, nloc+nhalo)).  The search direction is stored extended,
// p_ext = [own p | neighbours' p], so pass A is a plain SpMV over p_ext.
// One iteration (unfolded CG: every pass streams at full speed, and each
// kernel keeps the whole register budget for its own loop):
//   A  q = A p_ext, partial p.q              -> ncclAllReduce -> alpha
//   B  r -= alpha q, partial r.r             -> ncclAllReduce -> beta, flags
//   C  x += alpha p, p = r + beta p          -> pack p halo -> ncclSend/Recv
// Scalars live in a device StepState; dot products are reduced in fixed
// order on each rank (last-CTA-done) and summed across ranks by
// ncclAllReduce on StepState::red, so every rank computes bitwise identical
// alpha/beta/flags and stops at the same iteration.
#pragma once
#include "lines.cuh"

namespace spcg {

// Block size of the elementwise passes (B, C, x): independent of the tile
// kernels' kBlock so their grid-stride parallelism does not shrink with it.
constexpr int kElemBlock = 512;

struct StepState {
  double rr, alpha, beta, b_norm, rel, tol;
  double red;  // local partial sum; NCCL all-reduces it in place
  double pad0;
  long long k, max_it, fail_iter;
  long long kc;  // iterations whose pass C ran
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

// pass A: q = A p_ext, red = p.q partial (skipped once done).  WIDE: the
// view carries wide tiles (short-row CSR); a separate instantiation so the
// other kernels do not pay the two-line body's registers.
template <int FMT, bool WIDE = false>
__global__ void __launch_bounds__(kBlock, kStreamMinBlocks)
    dist_spmv_pq(const MatView M, StepState* S, const double* p_ext, double* q, double* part) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  if (S->done) return;
  constexpr bool TWO = (FMT == K_SCSR_PRIV);
  smem_init(sm);
  Pipe P;
  pipe_start<TWO>(P, sm, M);
  SrcPlain src{p_ext};
  double pq = 0.0;
  for (int j = 0; j < P.m; ++j) {
    const int s = pipe_acquire(P, sm, j);
    if (WIDE && wide_tile<FMT>(sm, s)) {
      LineOut o2[2];
      bool act[2];
      int li[2];
      csr_line_pair(sm, s, src, o2, act, li, nullptr);
#pragma unroll
      for (int t = 0; t < 2; ++t)
        if (act[t]) {
          q[li[t]] = o2[t].q;
          pq += o2[t].xi * o2[t].q;
        }
    } else {
      bool active = false;
      int i = -1;
      // atomic formats (single GPU): transposed scatter into q (zeroed by
      // pass B), p.Ap from the line's own gather (line_pq)
      const LineOut o = tile_line<FMT, true>(sm, s, M, src, q, active, i, sm.val[s]);
      if (active) {
        finish_plain<FMT>(o, i, q);
        pq += line_pq<FMT>(o);
      }
    }
    pipe_release<TWO>(P, sm, M, s);
  }
  pipe_drain(P, sm);
  last_block_sum(pq, sm, part, S);
}

// Reverse halo of the single-pass symmetric SpMV: partial sums of the
// transposed scatters that landed in this rank's ghost slots (halo columns
// owned by lower ranks) arrive in buf, aligned with the send list; add them
// into q at those rows.  Atomic adds: a row can be in several peers' halos,
// and this format's summation order is unspecified anyway.
__global__ void __launch_bounds__(256) dist_unpack_add(long long total, const int* idx,
                                                       const double* buf, double* q) {
  const long long G = (long long)gridDim.x * blockDim.x;
  for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < total; s += G)
    red_add_f64(q + idx[s], buf[s]);
}

// y = A x_ext (plain gather; initial / true residual)
template <int FMT, bool WIDE = false>
__global__ void __launch_bounds__(kBlock, kStreamMinBlocks)
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
    if (WIDE && wide_tile<FMT>(sm, s)) {
      LineOut o2[2];
      bool act[2];
      int li[2];
      csr_line_pair(sm, s, src, o2, act, li, nullptr);
#pragma unroll
      for (int t = 0; t < 2; ++t)
        if (act[t]) y[li[t]] = o2[t].q;
    } else {
      bool active = false;
      int i = -1;
      const LineOut o = tile_line<FMT, false>(sm, s, M, src, y, active, i, sm.val[s]);
      if (active) finish_plain<FMT>(o, i, y);
    }
    pipe_release<TWO>(P, sm, M, s);
  }
  pipe_drain(P, sm);
}

// Elementwise kernels over the nloc own lines (grid-stride, fixed order).
// mode 0: red = b.b               mode 1: r = b - q (or b), red = r.r, p = r
// mode 2: r -= alpha q, red = r.r mode 3: red = |b - q|^2 (true residual)
// Mode 2 moves 16-byte pairs, two in flight per thread (r, q 16-B aligned).
__global__ void __launch_bounds__(kElemBlock) dist_elem(int mode, long long nloc, StepState* S,
                                                   const double* b, double* q, double* r,
                                                   double* p, double* part, int zq, int rev = 0) {
  __shared__ RedSmem sm;
  if (mode == 2 && S->done) return;
  const double alpha = S->alpha;
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long G = (long long)gridDim.x * blockDim.x;
  double acc = 0.0;
  if (mode == 2) {
    const double na = -alpha;
    const long long np = nloc >> 1;
    const double2* q2 = reinterpret_cast<const double2*>(q);
    double2* r2 = reinterpret_cast<double2*>(r);
    long long i = g;
    for (; i + G < np; i += 2 * G) {
      const long long ia = rev ? np - 1 - i : i, ib = rev ? np - 1 - (i + G) : i + G;
      const double2 qa = q2[ia], qb = q2[ib], ra = r2[ia], rb = r2[ib];
      const double2 oa = make_double2(mul_add_rn(ra.x, na, qa.x), mul_add_rn(ra.y, na, qa.y));
      const double2 ob = make_double2(mul_add_rn(rb.x, na, qb.x), mul_add_rn(rb.y, na, qb.y));
      r2[ia] = oa;
      r2[ib] = ob;
      if (zq) {
        reinterpret_cast<double2*>(q)[ia] = make_double2(0.0, 0.0);
        reinterpret_cast<double2*>(q)[ib] = make_double2(0.0, 0.0);
      }
      acc = fma(oa.x, oa.x, acc);
      acc = fma(oa.y, oa.y, acc);
      acc = fma(ob.x, ob.x, acc);
      acc = fma(ob.y, ob.y, acc);
    }
    if (i < np) {
      const long long ia = rev ? np - 1 - i : i;
      const double2 qa = q2[ia], ra = r2[ia];
      const double2 oa = make_double2(mul_add_rn(ra.x, na, qa.x), mul_add_rn(ra.y, na, qa.y));
      r2[ia] = oa;
      if (zq) reinterpret_cast<double2*>(q)[ia] = make_double2(0.0, 0.0);
      acc = fma(oa.x, oa.x, acc);
      acc = fma(oa.y, oa.y, acc);
    }
    if ((nloc & 1) && g == 0) {
      const double v = mul_add_rn(r[nloc - 1], na, q[nloc - 1]);
      if (zq) q[nloc - 1] = 0.0;
      r[nloc - 1] = v;
      acc = fma(v, v, acc);
    }
  } else {
    for (long long i = g; i < nloc; i += G) {
      double v;
      if (mode == 0) {
        v = b[i];
      } else if (mode == 1) {
        v = q ? mul_add_rn(b[i], -1.0, q[i]) : b[i];
        if (q && zq) q[i] = 0.0;
        r[i] = v;
        p[i] = v;
      } else {
        v = mul_add_rn(b[i], -1.0, q[i]);
      }
      acc = fma(v, v, acc);
    }
  }
  last_block_sum(acc, sm, part, S);
}

// pass C: x += alpha p, p = r + beta p, for an iteration that neither
// converged nor failed (a converged solve applies its last x update at the
// end; an exhausted max_iter runs its pass C).  xv: x is 16-byte aligned.
__global__ void __launch_bounds__(kElemBlock) dist_update(long long nloc, StepState* S, const double* r,
                                                     double* p, double* x, int xv, int rev = 0) {
  if (S->status != 0 || S->converged || S->kc >= S->k) return;
  const double alpha = S->alpha, beta = S->beta;
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long G = (long long)gridDim.x * blockDim.x;
  const long long np = nloc >> 1;
  const double2* r2 = reinterpret_cast<const double2*>(r);
  double2* p2 = reinterpret_cast<double2*>(p);
  for (long long j = g; j < np; j += G) {
    const long long i = rev ? np - 1 - j : j;
    const double2 pv = p2[i], rv = r2[i];
    if (xv) {
      double2* x2 = reinterpret_cast<double2*>(x);
      const double2 xo = x2[i];
      x2[i] = make_double2(mul_add_rn(xo.x, alpha, pv.x), mul_add_rn(xo.y, alpha, pv.y));
    } else {
      x[2 * i] = mul_add_rn(x[2 * i], alpha, pv.x);
      x[2 * i + 1] = mul_add_rn(x[2 * i + 1], alpha, pv.y);
    }
    p2[i] = make_double2(mul_add_rn(rv.x, beta, pv.x), mul_add_rn(rv.y, beta, pv.y));
  }
  if ((nloc & 1) && g == 0) {
    const long long i = nloc - 1;
    const double pv = p[i];
    x[i] = mul_add_rn(x[i], alpha, pv);
    p[i] = mul_add_rn(r[i], beta, pv);
  }
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
  if (op == 2) S->kc = S->k;  // pass C of iteration k (if any) has run
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

// Halo values to send: v[idx] for every send row.
__global__ void dist_pack(long long cnt, const int* idx, const double* v, double* out) {
  const long long G = (long long)gridDim.x * blockDim.x;
  for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < cnt; s += G)
    out[s] = v[idx[s]];
}

// x = x0 (or 0); final x += alpha_K p_K of a converged solve (its pass C
// was skipped)
__global__ void dist_x(int mode, long long nloc, StepState* S, const double* src, double* x) {
  const long long G = (long long)gridDim.x * blockDim.x;
  const double alpha = S->alpha;
  const bool upd = S->k > 0 && S->status == 0 && S->converged;
  const bool zero_b = S->b_norm == 0.0;  // solver.py:109-118: x = 0 even for x0 != 0
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nloc; i += G) {
    if (mode == 0) x[i] = (src && !zero_b) ? src[i] : 0.0;
    else if (upd) x[i] = mul_add_rn(x[i], alpha, src[i]);
  }
}

}  // namespace spcg
