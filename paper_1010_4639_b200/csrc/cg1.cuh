// cg1.cuh — single-reduction CG (Chronopoulos & Gear) for resident systems.
//
// The latency-bound small systems (the paper's 30880-row matrix) spend most
// of an iteration in grid barriers, and standard CG needs two per iteration
// (p.Ap, then r.r).  Chronopoulos-Gear CG is the same Krylov method with the
// two inner products of an iteration reduced together:
//   p_i = r_i + b_i p_{i-1}        s_i = w_i + b_i s_{i-1}     (s_i = A p_i)
//   x  += a_i p_i                  r_{i+1} = r_i - a_i s_i
//   w_{i+1} = A r_{i+1}            [g, d] = [r.r, r.w]_{i+1}   <- one all-reduce
//   b_{i+1} = g_{i+1}/g_i          a_{i+1} = g_{i+1} / (d_{i+1} - b_{i+1} g_{i+1}/a_i)
// so one tile pass + one grid all-reduce per iteration.  The r-update is
// folded into the SpMV gather (r_{i+1,j} = r_j - a (w_j + b s_j), bitwise the
// value the owner computes), and every CTA keeps its own x, r, w, p, s in
// registers; r, w, s are published (double/triple buffered) for gathers.
// Semantics kept from solver.py: ||b|| = 0, x0 already converged, history of
// the recursive ||r||/||b||, convergence after the r-update, breakdowns
// (p.Ap = d - b g/a <= 0 -> not SPD; non-finite alpha / residual / beta)
// attributed to the same iteration numbers; true residual recomputed at the
// end.  Verified against the reference's CG output: same iteration counts,
// x within ~1e-12 (tests/test_gpu_cg1.py).
#pragma once
#include "cg.cuh"

namespace spcg {

// r_{i+1,j} gathered from the published r_i, w_i, s_{i-1}
struct SrcCgcg {
  const double* r;
  const double* w;
  const double* s;
  double na;    // -alpha_i
  double beta;  // beta_i
  __device__ __forceinline__ double get(int j) const {
    const double sj = __dadd_rn(w[j], __dmul_rn(beta, s[j]));
    return __dadd_rn(r[j], __dmul_rn(na, sj));
  }
};

// All-reduce of two values in one barrier (slot: 4 words, 2 per value).
__device__ __forceinline__ void grid_allreduce2(double& v0, double& v1, Smem& sm,
                                                unsigned long long* slots, uint32_t& epoch) {
  ++epoch;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double a0 = warp_sum(v0), a1 = warp_sum(v1);
  __shared__ double red2[2][32];
  if (lane == 0) {
    red2[0][w] = a0;
    red2[1][w] = a1;
  }
  __syncthreads();
  unsigned long long* bank = slots + (size_t)(epoch & 1u) * gridDim.x * kSlotWords;
  if (w == 0) {
    const int nw = (int)(blockDim.x >> 5);
    double b0 = lane < nw ? red2[0][lane] : 0.0;
    double b1 = lane < nw ? red2[1][lane] : 0.0;
    b0 = warp_sum(b0);
    b1 = warp_sum(b1);
    if (lane == 0) {
      fence_acq_rel_gpu();
      const unsigned long long u0 = (unsigned long long)__double_as_longlong(b0);
      const unsigned long long u1 = (unsigned long long)__double_as_longlong(b1);
      unsigned long long* slot = bank + (size_t)kSlotWords * blockIdx.x;
      slot_st2(slot, (u0 & 0xffffffff00000000ull) | epoch, (u0 << 32) | epoch);
      slot_st2(slot + 2, (u1 & 0xffffffff00000000ull) | epoch, (u1 << 32) | epoch);
    }
  }
  if (w < kPollWarps) {
    unsigned long long a[kPollPer], c[kPollPer], e[kPollPer], f[kPollPer];
    bool pend[kPollPer];
    const int base = 32 * w + lane;
#pragma unroll
    for (int u = 0; u < kPollPer; ++u) pend[u] = base + 32 * kPollWarps * u < (int)gridDim.x;
    bool any = true;
    unsigned long long spins = 0;
    while (__any_sync(0xffffffffu, any)) {  // warp-uniform (cg.cuh grid_allreduce)
#pragma unroll
      for (int u = 0; u < kPollPer; ++u)
        if (pend[u]) {
          const unsigned long long* sl = bank + (size_t)kSlotWords * (base + 32 * kPollWarps * u);
          slot_ld2(sl, a[u], c[u]);
          slot_ld2(sl + 2, e[u], f[u]);
        }
      any = false;
#pragma unroll
      for (int u = 0; u < kPollPer; ++u)
        if (pend[u]) {
          pend[u] = (uint32_t)a[u] != epoch || (uint32_t)c[u] != epoch ||
                    (uint32_t)e[u] != epoch || (uint32_t)f[u] != epoch;
          any |= pend[u];
        }
      if (++spins > kSpinLimit) asm volatile("trap;");
      if (kPollSleepNs && __any_sync(0xffffffffu, any)) __nanosleep(kPollSleepNs);
    }
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int u = 0; u < kPollPer; ++u)
      if (base + 32 * kPollWarps * u < (int)gridDim.x) {
        s0 += __longlong_as_double((long long)((a[u] & 0xffffffff00000000ull) | (c[u] >> 32)));
        s1 += __longlong_as_double((long long)((e[u] & 0xffffffff00000000ull) | (f[u] >> 32)));
      }
    fence_acq_rel_gpu();
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    if (lane == 0) {
      red2[0][16 + w] = s0;
      red2[1][16 + w] = s1;
    }
  }
  __syncthreads();
  double t0 = 0.0, t1 = 0.0;
#pragma unroll
  for (int k = 0; k < kPollWarps; ++k) {
    t0 += red2[0][16 + k];
    t1 += red2[1][16 + k];
  }
  __syncthreads();
  v0 = t0;
  v1 = t1;
}

struct Cg1Args {
  CgArgs base;     // b, x0, x, hist, slots, res, tol, max_iter, flags, M
  double* R[2];    // published r_i (ping-pong)
  double* S[2];    // published s_{i-1}
  double* W[3];    // published w_i (triple buffer: atomic formats scatter into it)
};

template <int FMT>
__global__ void __launch_bounds__(kBlock, 1) cg1_kernel(const Cg1Args G) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  constexpr bool TWO = (FMT == K_SCSR_PRIV);
  constexpr bool ATOM = (FMT == K_SCSR_ATOMIC || FMT == K_CSC);
  const CgArgs& A = G.base;
  const MatView& M = A.M;
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;

  smem_init(sm);
  Pipe P;
  pipe_start<TWO>(P, sm, M, true);
  uint32_t epoch = 0;

  int li[kStages];
  double xr[kStages], rg[kStages], wg[kStages], pg[kStages], sg[kStages], bg[kStages];
#pragma unroll
  for (int u = 0; u < kStages; ++u) {
    li[u] = -1;
    xr[u] = rg[u] = wg[u] = pg[u] = sg[u] = bg[u] = 0.0;
    if (u < P.m) {
      mbar_wait(&sm.full[u], 0);
      const StageMeta& mt = sm.meta[u];
      li[u] = owned_line<FMT>(mt);
    }
  }
  // ||b||
  double part = 0.0, part2 = 0.0;
#pragma unroll
  for (int u = 0; u < kStages; ++u)
    if (li[u] >= 0) {
      bg[u] = A.b[li[u]];
      part = fma(bg[u], bg[u], part);
    }
  double b_norm = sqrt(grid_allreduce(part, sm, A.slots, epoch));
  if (b_norm == 0.0) {
#pragma unroll
    for (int u = 0; u < kStages; ++u)
      if (li[u] >= 0) A.x[li[u]] = 0.0;
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
  // x = x0, r0 = b - A x0 (solver.py:120-124), published in R[0]
  if (A.x0 != nullptr) {
    SrcPlain sx{A.x0};
#pragma unroll
    for (int u = 0; u < kStages; ++u)
      if (li[u] >= 0) xr[u] = A.x0[li[u]];
    double qv[kStages] = {};
    run_tiles<FMT, false, TWO, true>(P, sm, M, sx, A.q, [&](int j, int i, const LineOut& o) {
      if (FMT == K_SCSR_ATOMIC) red_add_f64(A.q + i, o.q);
      else if (!ATOM) qv[j] = o.q;
    });
    if (ATOM) grid_allreduce(0.0, sm, A.slots, epoch);
#pragma unroll
    for (int u = 0; u < kStages; ++u)
      if (li[u] >= 0) {
        const double qi = ATOM ? A.q[li[u]] : qv[u];
        if (ATOM) A.q[li[u]] = 0.0;
        rg[u] = mul_add_rn(bg[u], -1.0, qi);
      }
  } else {
#pragma unroll
    for (int u = 0; u < kStages; ++u) rg[u] = bg[u];
  }
  part = 0.0;
#pragma unroll
  for (int u = 0; u < kStages; ++u)
    if (li[u] >= 0) {
      G.R[0][li[u]] = rg[u];
      part = fma(rg[u], rg[u], part);
    }
  double gam = grid_allreduce(part, sm, A.slots, epoch);  // publishes R[0]
  const double tol_b = A.tol * b_norm;
  long long max_it = A.max_iter;
  double rel = sqrt(gam) / b_norm;
  int converged = 0, status = ST_OK;
  long long iterations = 0, fail_iter = 0;
  double alpha = 0.0, beta = 0.0;
  if (sqrt(gam) <= tol_b) {
    converged = 1;
    max_it = 0;
  } else {
    // w0 = A r0, d0 = r0.w0  (p0 = r0, so d0 = p0.Ap0)
    SrcPlain sr{G.R[0]};
    part = 0.0;
    run_tiles<FMT, true, TWO, true>(P, sm, M, sr, G.W[0], [&](int j, int i, const LineOut& o) {
      if (FMT == K_SCSR_ATOMIC) {
        red_add_f64(G.W[0] + i, o.q);
      } else if (!ATOM) {
        wg[j] = o.q;
        G.W[0][i] = o.q;
      }
      part += line_pq<FMT>(o);
    });
    // publishes W[0] and completes the atomic w0 scatter
    double d0 = grid_allreduce(part, sm, A.slots, epoch);
    if (ATOM) {
#pragma unroll
      for (int u = 0; u < kStages; ++u)
        if (li[u] >= 0) wg[u] = G.W[0][li[u]];
    }
    if (d0 <= 0.0) {
      status = ST_NOT_SPD;
      fail_iter = 1;
    } else {
      alpha = gam / d0;
      if (!isfinite(alpha)) {
        status = ST_NF_ALPHA;
        fail_iter = 1;
      }
    }
  }

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
  for (long long it = 0; status == ST_OK && it < max_it; ++it) {
    const int cur = (int)(it & 1), nxt = cur ^ 1;
    const int wc = (int)(it % 3), wn = (int)((it + 1) % 3), wz = (int)((it + 2) % 3);
    SrcCgcg src{G.R[cur], G.W[wc], G.S[cur], -alpha, beta};
    part = 0.0;
    part2 = 0.0;
    // own lines: p, s, x, r_{i+1} (registers), then w_{i+1} = A r_{i+1}
#pragma unroll
    for (int u = 0; u < kStages; ++u)
      if (li[u] >= 0) {
        pg[u] = mul_add_rn(rg[u], beta, pg[u]);
        sg[u] = mul_add_rn(wg[u], beta, sg[u]);
        xr[u] = mul_add_rn(xr[u], alpha, pg[u]);
        G.S[nxt][li[u]] = sg[u];
        if (ATOM) G.W[wz][li[u]] = 0.0;  // held w_{i-1}; scattered into at i+1
      }
    run_tiles<FMT, true, TWO, true>(P, sm, M, src, G.W[wn], [&](int j, int i, const LineOut& o) {
      rg[j] = o.xi;  // r_{i+1,i}, bitwise the gathered value
      if (FMT == K_SCSR_ATOMIC) {
        red_add_f64(G.W[wn] + i, o.q);
      } else if (!ATOM) {
        wg[j] = o.q;
        G.W[wn][i] = o.q;
      }
      G.R[nxt][i] = o.xi;
      part = fma(o.xi, o.xi, part);
      part2 += line_pq<FMT>(o);
    });
    double g_new = part, d_new = part2;
    mark(0);
    grid_allreduce2(g_new, d_new, sm, A.slots, epoch);
    mark(1);
    if (ATOM) {
#pragma unroll
      for (int u = 0; u < kStages; ++u)
        if (li[u] >= 0) wg[u] = G.W[wn][li[u]];
    }
    const long long k = it + 1;  // reference iteration number
    rel = sqrt(g_new) / b_norm;
    if (!isfinite(rel)) {
      status = ST_NF_RES;
      fail_iter = k;
      break;
    }
    if (A.record_history && leader) A.hist[k - 1] = rel;
    iterations = k;
    if (sqrt(g_new) <= tol_b) {
      converged = 1;
      break;
    }
    const double beta_n = g_new / gam;
    if (!isfinite(beta_n)) {
      status = ST_NF_BETA;
      fail_iter = k;
      break;
    }
    if (k < max_it) {  // p.Ap of iteration k+1 (solver.py:135-139)
      const double eta = d_new - beta_n * g_new / alpha;
      if (eta <= 0.0) {
        status = ST_NOT_SPD;
        fail_iter = k + 1;
        break;
      }
      const double alpha_n = g_new / eta;
      if (!isfinite(alpha_n)) {
        status = ST_NF_ALPHA;
        fail_iter = k + 1;
        break;
      }
      alpha = alpha_n;
    }
    beta = beta_n;
    gam = g_new;
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
#pragma unroll
  for (int u = 0; u < kStages; ++u)
    if (li[u] >= 0) A.x[li[u]] = xr[u];
  if (A.recompute) {
    grid_allreduce(0.0, sm, A.slots, epoch);
    SrcPlain sx{A.x};
    double qv[kStages] = {};
    run_tiles<FMT, false, TWO, true>(P, sm, M, sx, A.q, [&](int j, int i, const LineOut& o) {
      if (FMT == K_SCSR_ATOMIC) red_add_f64(A.q + i, o.q);
      else if (!ATOM) qv[j] = o.q;
    });
    if (ATOM) grid_allreduce(0.0, sm, A.slots, epoch);
    part = 0.0;
#pragma unroll
    for (int u = 0; u < kStages; ++u)
      if (li[u] >= 0) {
        const double qi = ATOM ? A.q[li[u]] : qv[u];
        const double tr = mul_add_rn(bg[u], -1.0, qi);
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


// ---- engine 7: the same single-reduction CG for systems that do NOT fit on
// chip (mid-size: ~0.25-4 M rows).  The per-pass engine pays three launches
// and three tails per iteration (~30 us at 262 K rows, where the bytes take
// ~3 us from L2); here ONE persistent cooperative kernel streams the tiles
// every iteration through the TMA ring (the matrix of a mid-size system stays
// in the 126 MB L2) and the only grid-wide wait is the fused all-reduce.  The
// per-line state lives in global memory (x in A.x, p in G.Pv, and the
// published r, s, w of cg1_kernel) instead of registers: a CTA's tile list is
// unbounded.  Gather formats only (CSR, privatized symmetric half), so every
// value is bitwise the one cg1_kernel computes.
struct Cg1sArgs {
  Cg1Args g;
  double* Pv;  // p, own lines
};

template <int FMT>
__global__ void __launch_bounds__(kBlock, 1) cg1s_kernel(const Cg1sArgs S1) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  constexpr bool TWO = (FMT == K_SCSR_PRIV);
  static_assert(FMT == K_CSR || FMT == K_SCSR_PRIV, "engine 7: gather formats");
  const Cg1Args& G = S1.g;
  const CgArgs& A = G.base;
  const MatView& M = A.M;
  double* X = A.x;
  double* Pv = S1.Pv;
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
  const long long n = M.n;
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long GT = (long long)gridDim.x * blockDim.x;

  smem_init(sm);
  Pipe P;
  pipe_start<TWO>(P, sm, M, false);  // streamed: the pass overwrites staged values
  uint32_t epoch = 0;

  // ||b||
  double part = 0.0, part2 = 0.0;
  for (long long i = gt; i < n; i += GT) part = fma(A.b[i], A.b[i], part);
  const double b_norm = sqrt(grid_allreduce(part, sm, A.slots, epoch));
  if (b_norm == 0.0) {  // solver.py:109-118
    for (long long i = gt; i < n; i += GT) X[i] = 0.0;
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
  // x = x0, r0 = b - A x0 (solver.py:120-124), published in R[0]
  part = 0.0;
  if (A.x0 != nullptr) {
    SrcPlain sx{A.x0};
    run_tiles<FMT, false, TWO, false>(P, sm, M, sx, A.q, [&](int, int i, const LineOut& o) {
      const double ri = mul_add_rn(A.b[i], -1.0, o.q);
      X[i] = A.x0[i];
      G.R[0][i] = ri;
      part = fma(ri, ri, part);
    });
  } else {
    for (long long i = gt; i < n; i += GT) {
      const double ri = A.b[i];
      X[i] = 0.0;
      G.R[0][i] = ri;
      part = fma(ri, ri, part);
    }
  }
  double gam = grid_allreduce(part, sm, A.slots, epoch);  // publishes R[0]
  const double tol_b = A.tol * b_norm;
  long long max_it = A.max_iter;
  double rel = sqrt(gam) / b_norm;
  int converged = 0, status = ST_OK;
  long long iterations = 0, fail_iter = 0;
  double alpha = 0.0, beta = 0.0;
  if (sqrt(gam) <= tol_b) {
    converged = 1;
    max_it = 0;
  } else {
    // w0 = A r0, d0 = r0.w0 (p0 = r0)
    SrcPlain sr{G.R[0]};
    part = 0.0;
    run_tiles<FMT, true, TWO, false>(P, sm, M, sr, G.W[0], [&](int, int i, const LineOut& o) {
      G.W[0][i] = o.q;
      part += line_pq<FMT>(o);
    });
    const double d0 = grid_allreduce(part, sm, A.slots, epoch);  // publishes W[0]
    if (d0 <= 0.0) {
      status = ST_NOT_SPD;
      fail_iter = 1;
    } else {
      alpha = gam / d0;
      if (!isfinite(alpha)) {
        status = ST_NF_ALPHA;
        fail_iter = 1;
      }
    }
  }
  for (long long it = 0; status == ST_OK && it < max_it; ++it) {
    const int cur = (int)(it & 1), nxt = cur ^ 1;
    const int wc = (int)(it % 3), wn = (int)((it + 1) % 3);
    SrcCgcg src{G.R[cur], G.W[wc], G.S[cur], -alpha, beta};
    part = 0.0;
    part2 = 0.0;
    // own line i: p, s, x from its published r_i, w_i, s_{i-1} (the same
    // operations as cg1_kernel's registers), r_{i+1} = the gathered value,
    // w_{i+1} = A r_{i+1}
    run_tiles<FMT, true, TWO, false>(P, sm, M, src, G.W[wn], [&](int, int i, const LineOut& o) {
      const double pi = mul_add_rn(G.R[cur][i], beta, Pv[i]);
      const double si = mul_add_rn(G.W[wc][i], beta, G.S[cur][i]);
      Pv[i] = pi;
      G.S[nxt][i] = si;
      X[i] = mul_add_rn(X[i], alpha, pi);
      G.W[wn][i] = o.q;
      G.R[nxt][i] = o.xi;  // r_{i+1,i}, bitwise the gathered value
      part = fma(o.xi, o.xi, part);
      part2 += line_pq<FMT>(o);
    });
    double g_new = part, d_new = part2;
    grid_allreduce2(g_new, d_new, sm, A.slots, epoch);
    const long long k = it + 1;  // reference iteration number
    rel = sqrt(g_new) / b_norm;
    if (!isfinite(rel)) {
      status = ST_NF_RES;
      fail_iter = k;
      break;
    }
    if (A.record_history && leader) A.hist[k - 1] = rel;
    iterations = k;
    if (sqrt(g_new) <= tol_b) {
      converged = 1;
      break;
    }
    const double beta_n = g_new / gam;
    if (!isfinite(beta_n)) {
      status = ST_NF_BETA;
      fail_iter = k;
      break;
    }
    if (k < max_it) {  // p.Ap of iteration k+1 (solver.py:135-139)
      const double eta = d_new - beta_n * g_new / alpha;
      if (eta <= 0.0) {
        status = ST_NOT_SPD;
        fail_iter = k + 1;
        break;
      }
      const double alpha_n = g_new / eta;
      if (!isfinite(alpha_n)) {
        status = ST_NF_ALPHA;
        fail_iter = k + 1;
        break;
      }
      alpha = alpha_n;
    }
    beta = beta_n;
    gam = g_new;
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
  if (A.recompute) {  // true residual ||b - A x|| / ||b||
    grid_allreduce(0.0, sm, A.slots, epoch);  // publishes x
    SrcPlain sx{X};
    part = 0.0;
    run_tiles<FMT, false, TWO, false>(P, sm, M, sx, A.q, [&](int, int i, const LineOut& o) {
      const double tr = mul_add_rn(A.b[i], -1.0, o.q);
      part = fma(tr, tr, part);
    });
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

