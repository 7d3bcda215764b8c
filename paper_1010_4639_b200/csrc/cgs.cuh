// cgs.cuh — streaming persistent CG for systems that do not fit on chip
// (P2 / P3 / Q27 class): two-reduction CG exactly as cg_kernel, but with the
// residual and the search direction stored interleaved as 16-byte pairs
//   RP[a][j] = (r_k,j , p_{k-1},j)
// so the folded gather r_j + beta p_j is ONE 128-bit load with one address
// per entry (half the gather instructions and address registers — pass A is
// bound by gather latency at the 64-register budget of 2 CTAs/SM).  Pass B
// reads the pair and q, recomputes p_k = r_k + beta p_{k-1} (bitwise the
// value pass A gathered) and writes the full pair (r_{k+1}, p_k) into RP[b],
// so no partial-sector writes reach HBM.
#pragma once
#include "cg.cuh"

namespace spcg {

struct SrcPairFirst {  // iteration 1: p_1 = r_0
  const double2* rp;
  __device__ __forceinline__ double get(int j) const { return rp[j].x; }
};
struct SrcPairFold {  // p_k = r_k + beta p_{k-1}
  const double2* rp;
  double beta;
  __device__ __forceinline__ double get(int j) const {
    const double2 t = rp[j];
    return __dadd_rn(t.x, __dmul_rn(beta, t.y));
  }
};

struct CgsArgs {
  CgArgs base;   // b, x0, x, q, hist, slots, res, tol, max_iter, flags, M
  double2* RP[2];
};

template <int FMT>
__global__ void __launch_bounds__(kBlock, kStreamMinBlocks) cgs_kernel(const CgsArgs G) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  constexpr bool TWO = (FMT == K_SCSR_PRIV);
  constexpr bool ATOM = (FMT == K_SCSR_ATOMIC || FMT == K_CSC);
  const CgArgs& A = G.base;
  const MatView& M = A.M;
  const int n = M.n;
  const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long gstride = (long long)gridDim.x * blockDim.x;
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;

  smem_init(sm);
  Pipe P;
  pipe_start<TWO>(P, sm, M, /*allow_resident=*/false);
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
  // x = x0, r0 = b - A x0  ->  RP[0] = (r0, 0)
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
      G.RP[0][i] = make_double2(ri, 0.0);
      part = fma(ri, ri, part);
    }
  } else {
    part = 0.0;
    for (long long i = gtid; i < n; i += gstride) {
      const double bi = A.b[i];
      A.x[i] = 0.0;
      G.RP[0][i] = make_double2(bi, 0.0);
      part = fma(bi, bi, part);
    }
  }
  double rr = grid_allreduce(part, sm, A.slots, epoch);

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
  int a = 0;  // RP[a] holds (r_k, p_{k-1})

  for (long long k = 1; k <= max_it; ++k) {
    const double2* rpa = G.RP[a];
    double2* rpb = G.RP[a ^ 1];
    // pass A: p_k folded into the gather, q = A p_k, x += alpha_{k-1} p_{k-1}
    double pq = 0.0;
    auto lineA = [&](int, int i, const LineOut& o) {
      if (k > 1) A.x[i] = mul_add_rn(o.xo, alpha, rpa[i].y);
      if (!ATOM) A.q[i] = o.q;
      if (FMT == K_SCSR_ATOMIC) red_add_f64(A.q + i, o.q);
      pq += line_pq<FMT>(o);
    };
    if (k == 1) {
      SrcPairFirst sf{rpa};
      run_tiles<FMT, true, TWO, false>(P, sm, M, sf, A.q, lineA);
    } else {
      SrcPairFold sf{rpa, beta};
      run_tiles<FMT, true, TWO, false>(P, sm, M, sf, A.q, lineA, A.x);
    }
    pq = grid_allreduce(pq, sm, A.slots, epoch);
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
    // pass B: (r_{k+1}, p_k) -> RP[b]
    part = 0.0;
    const double na = -alpha;
    const double bb = (k == 1) ? 0.0 : beta;
    auto upd = [&](long long i, const double2 t, double qi) {
      const double pk = (k == 1) ? t.x : __dadd_rn(t.x, __dmul_rn(bb, t.y));
      const double rn = mul_add_rn(t.x, na, qi);
      rpb[i] = make_double2(rn, pk);
      part = fma(rn, rn, part);
    };
    long long i = gtid;
    for (; i + gstride < n; i += 2 * gstride) {  // two rows in flight per thread
      const double2 t0 = rpa[i], t1 = rpa[i + gstride];
      const double q0 = A.q[i], q1 = A.q[i + gstride];
      if (ATOM) {
        A.q[i] = 0.0;
        A.q[i + gstride] = 0.0;
      }
      upd(i, t0, q0);
      upd(i + gstride, t1, q1);
    }
    if (i < n) {
      const double2 t0 = rpa[i];
      const double q0 = A.q[i];
      if (ATOM) A.q[i] = 0.0;
      upd(i, t0, q0);
    }
    const double rr_new = grid_allreduce(part, sm, A.slots, epoch);
    a ^= 1;
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
  }

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
  // x += alpha_K p_K  (p_K is the .y of the pair written last)
  if (iterations > 0) {
    const double2* rp = G.RP[a];
    for (long long i = gtid; i < n; i += gstride) A.x[i] = mul_add_rn(A.x[i], alpha, rp[i].y);
  }
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
