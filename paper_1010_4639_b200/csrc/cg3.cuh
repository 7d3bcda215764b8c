// cg3.cuh — streaming persistent CG, three passes per iteration.
//
// For systems that stream from HBM (P2 / P3 / Q27 class) the folded gather
// of cg_kernel (r_j + beta p_j: two gathered vectors per entry) is bound by
// gather latency at the 64-register budget, and that pass ran at ~1.8x the
// time of a plain SpMV.  Unfolding the p-update costs 8n more bytes per
// iteration but every pass then runs at streaming speed:
//   pass A (tiles)   q = A p, partial p.q                 -> all-reduce (alpha)
//   pass B           r -= alpha q, partial r.r             -> all-reduce (beta)
//   pass C           x += alpha p, p = r + beta p          -> barrier
// Bytes: 12 nnz + 4n + (16 + 24 + 40) n.  Operation order and rounding are
// the reference's (solver.py:133-156): x and r use the iteration's alpha,
// then p = r + beta p.  Elementwise passes move 16-byte pairs with two pairs
// in flight per thread.
#pragma once
#include "cg.cuh"

namespace spcg {

template <int FMT>
__global__ void __launch_bounds__(kBlock, kStreamMinBlocks) cg3_kernel(const CgArgs A) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  constexpr bool TWO = (FMT == K_SCSR_PRIV);
  constexpr bool ATOM = (FMT == K_SCSR_ATOMIC || FMT == K_CSC);
  const MatView& M = A.M;
  const int n = M.n;
  const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long gstride = (long long)gridDim.x * blockDim.x;
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
  double* p = A.p0;

  smem_init(sm);
  Pipe P;
  pipe_start<TWO>(P, sm, M, /*allow_resident=*/false);  // stream body writes in place
  uint32_t epoch = 0;

  double part = 0.0;
  for (long long i = gtid; i < n; i += gstride) part = fma(A.b[i], A.b[i], part);
  const double b_norm = sqrt(grid_allreduce(part, sm, A.slots, epoch));
  if (b_norm == 0.0) {  // solver.py:109-118
    for (long long i = gtid; i < n; i += gstride) A.x[i] = 0.0;
    if (leader) {
      A.res->iterations = 0;
      A.res->fail_iter = 0;
      A.res->converged = 1;
      A.res->status = ST_OK;
      A.res->final_rel = 0.0;
      A.res->b_norm = 0.0;
    }
    pipe_drain(P, sm);
    return;
  }
  // x = x0, r = b - A x0, p = r (solver.py:120-124)
  if (A.x0 != nullptr) {
    for (long long i = gtid; i < n; i += gstride) A.x[i] = A.x0[i];
    SrcPlain sx{A.x0};
    run_tiles<FMT, false, TWO, false>(P, sm, M, sx, A.q, [&](int, int i, const LineOut& o) {
      finish_plain<FMT>(o, i, A.q);
    });
    grid_allreduce(0.0, sm, A.slots, epoch);
    part = 0.0;
    for (long long i = gtid; i < n; i += gstride) {
      const double qi = A.q[i];
      if (ATOM) A.q[i] = 0.0;
      const double ri = mul_add_rn(A.b[i], -1.0, qi);
      A.r[i] = ri;
      p[i] = ri;
      part = fma(ri, ri, part);
    }
  } else {
    part = 0.0;
    for (long long i = gtid; i < n; i += gstride) {
      const double bi = A.b[i];
      A.x[i] = 0.0;
      A.r[i] = bi;
      p[i] = bi;
      part = fma(bi, bi, part);
    }
  }
  double rr = grid_allreduce(part, sm, A.slots, epoch);  // also publishes p

  const double tol_b = A.tol * b_norm;
  long long max_it = A.max_iter;
  double rel = sqrt(rr) / b_norm;
  int converged = 0, status = ST_OK;
  long long iterations = 0, fail_iter = 0;
  if (sqrt(rr) <= tol_b) {
    converged = 1;
    max_it = 0;
  }
  double alpha = 0.0, beta = 0.0;
  const long long np = (long long)n >> 1;
  double2* r2 = reinterpret_cast<double2*>(A.r);
  double2* p2 = reinterpret_cast<double2*>(p);
  const double2* q2 = reinterpret_cast<const double2*>(A.q);
  double2* z2 = reinterpret_cast<double2*>(A.q);

#if SPCG_TRACE
  unsigned long long tr[4] = {0, 0, 0, 0};
  unsigned long long tlast = A.trace ? globaltimer_ns() : 0;
  auto mark = [&](int ph) {
    if (A.trace && threadIdx.x == 0) {
      const unsigned long long t = globaltimer_ns();
      tr[ph] += t - tlast;
      tlast = t;
    }
  };
#else
  auto mark = [](int) {};
#endif
  for (long long k = 1; k <= max_it; ++k) {
    // pass A: q = A p, p.q
    double pq = 0.0;
    SrcPlain sp{p};
    run_tiles<FMT, true, TWO, false>(P, sm, M, sp, A.q, [&](int, int i, const LineOut& o) {
      if (!ATOM) A.q[i] = o.q;
      if (FMT == K_SCSR_ATOMIC) red_add_f64(A.q + i, o.q);
      pq += line_pq<FMT>(o);
    });
    mark(0);
    pq = grid_allreduce(pq, sm, A.slots, epoch);
    mark(1);
    if (pq <= 0.0) {
      status = ST_NOT_SPD;
      fail_iter = k;
      break;
    }
    alpha = rr / pq;
    if (!isfinite(alpha)) {
      status = ST_NF_ALPHA;
      fail_iter = k;
      break;
    }
    // pass B: r -= alpha q, r.r   (16-byte pairs, two in flight)
    part = 0.0;
    const double na = -alpha;
    {
      long long pi = gtid;
      for (; pi + gstride < np; pi += 2 * gstride) {
        const double2 qa = q2[pi], qb = q2[pi + gstride];
        const double2 ra = r2[pi], rb = r2[pi + gstride];
        double2 oa, ob;
        oa.x = mul_add_rn(ra.x, na, qa.x);
        oa.y = mul_add_rn(ra.y, na, qa.y);
        ob.x = mul_add_rn(rb.x, na, qb.x);
        ob.y = mul_add_rn(rb.y, na, qb.y);
        r2[pi] = oa;
        r2[pi + gstride] = ob;
        if (ATOM) {
          z2[pi] = make_double2(0.0, 0.0);
          z2[pi + gstride] = make_double2(0.0, 0.0);
        }
        part = fma(oa.x, oa.x, part);
        part = fma(oa.y, oa.y, part);
        part = fma(ob.x, ob.x, part);
        part = fma(ob.y, ob.y, part);
      }
      if (pi < np) {
        const double2 qa = q2[pi], ra = r2[pi];
        double2 oa;
        oa.x = mul_add_rn(ra.x, na, qa.x);
        oa.y = mul_add_rn(ra.y, na, qa.y);
        r2[pi] = oa;
        if (ATOM) z2[pi] = make_double2(0.0, 0.0);
        part = fma(oa.x, oa.x, part);
        part = fma(oa.y, oa.y, part);
      }
      if ((n & 1) && gtid == 0) {
        const long long i = n - 1;
        const double qi = A.q[i];
        if (ATOM) A.q[i] = 0.0;
        const double ri = mul_add_rn(A.r[i], na, qi);
        A.r[i] = ri;
        part = fma(ri, ri, part);
      }
    }
    mark(2);
    const double rr_new = grid_allreduce(part, sm, A.slots, epoch);
    mark(1);
    rel = sqrt(rr_new) / b_norm;
    if (!isfinite(rel)) {
      status = ST_NF_RES;
      fail_iter = k;
      break;
    }
    if (A.record_history && leader) A.hist[k - 1] = rel;
    iterations = k;
    if (sqrt(rr_new) <= tol_b) {
      converged = 1;
      rr = rr_new;
      break;
    }
    beta = rr_new / rr;
    if (!isfinite(beta)) {
      status = ST_NF_BETA;
      fail_iter = k;
      break;
    }
    rr = rr_new;
    // pass C: x += alpha p, p = r + beta p   (x is the caller's array: scalar)
    for (long long i = gtid; i < np; i += gstride) {
      const double2 pv = p2[i], rv = r2[i];
      A.x[2 * i] = mul_add_rn(A.x[2 * i], alpha, pv.x);
      A.x[2 * i + 1] = mul_add_rn(A.x[2 * i + 1], alpha, pv.y);
      p2[i] = make_double2(mul_add_rn(rv.x, beta, pv.x), mul_add_rn(rv.y, beta, pv.y));
    }
    if ((n & 1) && gtid == 0) {
      const long long i = n - 1;
      const double pv = p[i];
      A.x[i] = mul_add_rn(A.x[i], alpha, pv);
      p[i] = mul_add_rn(A.r[i], beta, pv);
    }
    mark(3);
    grid_allreduce(0.0, sm, A.slots, epoch);  // p complete before the next gather
    mark(1);
  }
#if SPCG_TRACE
  if (A.trace && threadIdx.x == 0) {
#pragma unroll
    for (int ph = 0; ph < 4; ++ph) A.trace[blockIdx.x * 5 + ph] = tr[ph];
  }
#endif

  if (status != ST_OK) {
    if (leader) {
      A.res->iterations = iterations;
      A.res->fail_iter = fail_iter;
      A.res->converged = 0;
      A.res->status = status;
      A.res->final_rel = rel;
      A.res->b_norm = b_norm;
    }
    pipe_drain(P, sm);
    return;
  }
  // a converged solve broke out before its pass C: apply its x += alpha p
  // (an exhausted max_iter ran pass C, so x is already complete)
  if (converged && iterations > 0)
    for (long long i = gtid; i < n; i += gstride) A.x[i] = mul_add_rn(A.x[i], alpha, p[i]);
  if (A.recompute) {
    grid_allreduce(0.0, sm, A.slots, epoch);
    SrcPlain sx{A.x};
    run_tiles<FMT, false, TWO, false>(P, sm, M, sx, A.q, [&](int, int i, const LineOut& o) {
      finish_plain<FMT>(o, i, A.q);
    });
    grid_allreduce(0.0, sm, A.slots, epoch);
    part = 0.0;
    for (long long i = gtid; i < n; i += gstride) {
      const double tr = mul_add_rn(A.b[i], -1.0, A.q[i]);
      part = fma(tr, tr, part);
    }
    rel = sqrt(grid_allreduce(part, sm, A.slots, epoch)) / b_norm;
  }
  if (leader) {
    A.res->iterations = iterations;
    A.res->fail_iter = 0;
    A.res->converged = converged;
    A.res->status = ST_OK;
    A.res->final_rel = rel;
    A.res->b_norm = b_norm;
  }
  pipe_drain(P, sm);
}

}  // namespace spcg
