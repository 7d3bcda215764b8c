// cg.cuh — the whole CG solve (solver.py:65-172) as ONE persistent
// cooperative kernel.
//
// Per iteration k the grid makes two passes and two grid-wide all-reduce
// barriers (the minimum for unmodified CG: p.Ap and r.r are sequential):
//   pass A  (tiles)  p_k = r + beta p_{k-1} folded into the gather,
//                    q = A p_k, x += alpha_{k-1} p_{k-1} (deferred x update),
//                    partial p.q                                 -> allreduce
//   scalar           pq<=0 / non-finite alpha checks, alpha = rr/pq
//   pass B           r -= alpha q, partial r.r (atomic formats: q := 0) -> allreduce
//   scalar           rel, history, convergence, beta = rr_new/rr
// Scalars are reduced in a fixed order and are bitwise identical in every
// CTA, so control flow stays grid-uniform without any host round trip.
//
// RES (resident) variant: every CTA owns <= kStages tiles; the tiles stay in
// shared memory and the CTA's own x, r, p, q, b entries stay in registers for
// the entire solve; only r and p are published (stored) for other CTAs'
// gathers.  Used when the matrix fits in the grid's shared memory.
#pragma once
#include "lines.cuh"

namespace spcg {

struct CgDevResult {
  long long iterations;
  long long fail_iter;
  int converged;
  int status;
  double final_rel;
  double b_norm;
};

struct CgArgs {
  MatView M;
  const double* b;
  const double* x0;  // nullable
  double* x;
  double* r;
  double* p0;
  double* p1;
  double* q;  // zero on entry for atomic formats
  double* hist;
  unsigned long long* trace;  // nullable: per-CTA phase nanoseconds [G][4]
  unsigned long long* slots;  // 2 * gridDim.x * 2 words, zero on entry
  CgDevResult* res;
  double tol;
  long long max_iter;
  int record_history;
  int recompute;
};

enum : int {
  ST_OK = 0,
  ST_NOT_SPD = 3,
  ST_NF_ALPHA = 4,
  ST_NF_RES = 5,
  ST_NF_BETA = 6,
  ST_BAD_LAUNCH = 100  // cluster engine launched with another cluster shape
};

// Grid-wide all-reduce + barrier.  Each CTA publishes its fixed-order block
// sum in its own 256-byte slot (one L2 line per CTA, so polls spread over
// many L2 slices instead of hammering a few lines) as two 64-bit words
// {hi32(sum)|epoch, lo32(sum)|epoch}; each word is single-copy atomic, so a
// reader that sees the epoch in both words has the whole value: one polling
// round trip, no atomics, no counter, no second hop.  Slots alternate between
// two banks by epoch parity, which makes reuse safe (a CTA can only run one
// barrier ahead of the slowest reader).
// Release: thread 0's fence.acq_rel.gpu after the CTA barrier publishes all
// of the CTA's prior global writes.  Acquire: warp 0 polls every slot (lane
// l reads slots l, l+32, ...), then fences once for the CTA.
// The total is summed in the same fixed order in every CTA (bitwise equal).
constexpr int kSlotWords = 32;  // 256 bytes per CTA slot
#ifndef SPCG_POLL_WARPS
#define SPCG_POLL_WARPS 8
#endif
#ifndef SPCG_POLL_NS
#define SPCG_POLL_NS 200
#endif
constexpr int kPollWarps = (kBlock / 32) < SPCG_POLL_WARPS ? (kBlock / 32) : SPCG_POLL_WARPS;
constexpr int kPollPer = (384 + 32 * kPollWarps - 1) / (32 * kPollWarps);  // grids <= 384 CTAs
constexpr unsigned kPollSleepNs = SPCG_POLL_NS;  // back-off between polling rounds

__device__ __forceinline__ double grid_allreduce(double v, Smem& sm, unsigned long long* slots,
                                                 uint32_t& epoch) {
  ++epoch;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) sm.red[w] = v;
  __syncthreads();
  unsigned long long* bank = slots + (size_t)(epoch & 1u) * gridDim.x * kSlotWords;
  if (w == 0) {
    double bs = lane < (int)(blockDim.x >> 5) ? sm.red[lane] : 0.0;
    bs = warp_sum(bs);
    if (lane == 0) {
      fence_acq_rel_gpu();
      const unsigned long long bits = (unsigned long long)__double_as_longlong(bs);
      slot_st2(bank + (size_t)kSlotWords * blockIdx.x,
                        (bits & 0xffffffff00000000ull) | epoch, (bits << 32) | epoch);
    }
  }
  if (w < kPollWarps) {
    // slot t = 32*w + lane + 128*u; all of a lane's loads are in flight at once
    unsigned long long a[kPollPer], c[kPollPer];
    bool pend[kPollPer];
    const int base = 32 * w + lane;
#pragma unroll
    for (int u = 0; u < kPollPer; ++u) pend[u] = base + 32 * kPollWarps * u < (int)gridDim.x;
    bool any = true;
    unsigned long long spins = 0;
    while (any) {
#pragma unroll
      for (int u = 0; u < kPollPer; ++u)
        if (pend[u])
          slot_ld2(bank + (size_t)kSlotWords * (base + 32 * kPollWarps * u), a[u], c[u]);
      any = false;
#pragma unroll
      for (int u = 0; u < kPollPer; ++u)
        if (pend[u]) {
          pend[u] = (uint32_t)a[u] != epoch || (uint32_t)c[u] != epoch;
          any |= pend[u];
        }
      if (++spins > kSpinLimit) asm volatile("trap;");
      if (kPollSleepNs && any) __nanosleep(kPollSleepNs);
    }
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < kPollPer; ++u)
      if (base + 32 * kPollWarps * u < (int)gridDim.x)
        s += __longlong_as_double((long long)((a[u] & 0xffffffff00000000ull) | (c[u] >> 32)));
    fence_acq_rel_gpu();
    s = warp_sum(s);
    if (lane == 0) sm.red[16 + w] = s;  // red[0..15] is not reread after the barrier
  }
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int k = 0; k < kPollWarps; ++k) t += sm.red[16 + k];  // fixed order, every thread
  __syncthreads();  // red reuse by the next call
  return t;
}

// Resident tiles keep their values: the CSR-stream products go to a separate
// shared-memory buffer placed after Smem (kResProdBytes extra dynamic smem).
constexpr size_t kResProdBytes = sizeof(double) * kStages * kNzCap;
__device__ __forceinline__ double* res_prod(Smem& sm, int j) {
  return reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(&sm) + sizeof(Smem)) +
         (size_t)j * kNzCap;
}

// Iterate this CTA's tiles; fn(j, line, LineOut) for every owned line.
// Resident CTAs unroll over the (<= kStages) stages so that j is a
// compile-time index into the per-thread register arrays.
template <int FMT, bool GATHER_CSC, bool TWO, bool RES, class Src, class Fn>
__device__ __forceinline__ void run_tiles(Pipe& P, Smem& sm, const MatView& M, const Src& src,
                                          double* y, Fn fn, const double* xpre = nullptr) {
  if (RES) {
#pragma unroll
    for (int j = 0; j < kStages; ++j) {
      if (j < P.m) {
        mbar_wait(&sm.full[j], 0);
        bool active = false;
        int line = -1;
        // resident (latency-bound) tiles: thread-per-row beats the two-phase
        // stream body (one fewer CTA barrier on the critical path)
        const LineOut o = tile_line<FMT, GATHER_CSC, Src, false>(sm, j, M, src, y, active, line,
                                                                 res_prod(sm, j));
        if (active) fn(j, line, o);
      }
    }
    return;
  }
  for (int j = 0; j < P.m; ++j) {
    const int s = pipe_acquire(P, sm, j);
    bool active = false;
    int line = -1;
    const LineOut o =
        tile_line<FMT, GATHER_CSC>(sm, s, M, src, y, active, line, sm.val[s], xpre);
    if (active) fn(j, line, o);
    pipe_release<TWO>(P, sm, M, s);
  }
}

template <int FMT, bool RES>
__global__ void __launch_bounds__(kBlock, RES ? 1 : kStreamMinBlocks) cg_kernel(const CgArgs A) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  constexpr bool TWO = (FMT == K_SCSR_PRIV);
  constexpr bool ATOM = (FMT == K_SCSR_ATOMIC || FMT == K_CSC);
  const MatView& M = A.M;
  const int n = M.n;
  const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long gstride = (long long)gridDim.x * blockDim.x;
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;

  smem_init(sm);
  Pipe P;
  pipe_start<TWO>(P, sm, M, /*allow_resident=*/RES);
  uint32_t epoch = 0;

  // RES: per-thread owned lines and their register-resident vector entries.
  int li[kStages];
  double xr[kStages], rg[kStages], pg[kStages], qg[kStages], bg[kStages];
#pragma unroll
  for (int u = 0; u < kStages; ++u) {
    li[u] = -1;
    xr[u] = rg[u] = pg[u] = qg[u] = bg[u] = 0.0;
  }
  if (RES) {
#pragma unroll
    for (int u = 0; u < kStages; ++u) {
      if (u < P.m) {
        mbar_wait(&sm.full[u], 0);
        const StageMeta& mt = sm.meta[u];
        li[u] = owned_line<FMT>(mt);
      }
    }
  }

  // ---- ||b|| (solver.py:107) --------------------------------------------------
  double part = 0.0;
  if (RES) {
#pragma unroll
    for (int u = 0; u < kStages; ++u)
      if (li[u] >= 0) {
        bg[u] = A.b[li[u]];
        part = fma(bg[u], bg[u], part);
      }
  } else {
    for (long long i = gtid; i < n; i += gstride) part = fma(A.b[i], A.b[i], part);
  }
  const double b_norm = sqrt(grid_allreduce(part, sm, A.slots, epoch));

  if (b_norm == 0.0) {  // solver.py:109-118: x = 0 even when x0 != 0
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

  // ---- x = x0, r = b - A x0 (solver.py:120-124) -------------------------------
  if (A.x0 != nullptr) {
    SrcPlain sx{A.x0};
    if (RES) {
#pragma unroll
      for (int u = 0; u < kStages; ++u)
        if (li[u] >= 0) xr[u] = A.x0[li[u]];
      run_tiles<FMT, false, TWO, RES>(P, sm, M, sx, A.q, [&](int j, int i, const LineOut& o) {
        if (FMT == K_SCSR_ATOMIC) red_add_f64(A.q + i, o.q);
        else if (!ATOM) qg[j] = o.q;
      });
      if (ATOM) grid_allreduce(0.0, sm, A.slots, epoch);
#pragma unroll
      for (int u = 0; u < kStages; ++u)
        if (li[u] >= 0) {
          const int i = li[u];
          double qi = qg[u];
          if (ATOM) {
            qi = A.q[i];
            A.q[i] = 0.0;
          }
          rg[u] = mul_add_rn(bg[u], -1.0, qi);
          A.r[i] = rg[u];
        }
    } else {
      for (long long i = gtid; i < n; i += gstride) A.x[i] = A.x0[i];
      run_tiles<FMT, false, TWO, RES>(P, sm, M, sx, A.q, [&](int, int i, const LineOut& o) {
        finish_plain<FMT>(o, i, A.q);
      });
      grid_allreduce(0.0, sm, A.slots, epoch);
      for (long long i = gtid; i < n; i += gstride) {
        const double qi = A.q[i];
        if (ATOM) A.q[i] = 0.0;
        A.r[i] = mul_add_rn(A.b[i], -1.0, qi);
      }
    }
  } else {
    if (RES) {
#pragma unroll
      for (int u = 0; u < kStages; ++u)
        if (li[u] >= 0) {
          rg[u] = bg[u];
          A.r[li[u]] = bg[u];
        }
    } else {
      for (long long i = gtid; i < n; i += gstride) {
        A.x[i] = 0.0;
        A.r[i] = A.b[i];
      }
    }
  }
  part = 0.0;
  if (RES) {
#pragma unroll
    for (int u = 0; u < kStages; ++u)
      if (li[u] >= 0) part = fma(rg[u], rg[u], part);
  } else {
    for (long long i = gtid; i < n; i += gstride) part = fma(A.r[i], A.r[i], part);
  }
  double rr = grid_allreduce(part, sm, A.slots, epoch);

  // ---- CG loop (solver.py:126-157) ---------------------------------------------
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
  double* p_old = A.p1;
  double* p_new = A.p0;
  double* p_cur = nullptr;

#if SPCG_TRACE
  unsigned long long tr[4] = {0, 0, 0, 0};
  P.trace = A.trace != nullptr;
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
    // pass A
    double pq = 0.0;
    auto lineA = [&](int j, int i, const LineOut& o) {
      if (RES) {
        if (k > 1) xr[j] = mul_add_rn(xr[j], alpha, pg[j]);
        pg[j] = o.xi;
        if (!ATOM) qg[j] = o.q;
      } else {
        if (k > 1) A.x[i] = mul_add_rn(SPCG_NO_XPRE ? A.x[i] : o.xo, alpha, p_old[i]);
        if (!ATOM) A.q[i] = o.q;
      }
      p_new[i] = o.xi;
      if (FMT == K_SCSR_ATOMIC) red_add_f64(A.q + i, o.q);
      pq += line_pq<FMT>(o);
    };
    if (k == 1) {
      SrcFirst sf{A.r};
      run_tiles<FMT, true, TWO, RES>(P, sm, M, sf, A.q, lineA);
    } else {
      SrcFold sf{A.r, p_old, beta};
      run_tiles<FMT, true, TWO, RES>(P, sm, M, sf, A.q, lineA, RES ? nullptr : A.x);
    }
    p_cur = p_new;
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
    // pass B
    part = 0.0;
    if (RES) {
#pragma unroll
      for (int u = 0; u < kStages; ++u)
        if (li[u] >= 0) {
          const int i = li[u];
          double qi = qg[u];
          if (ATOM) {
            qi = A.q[i];
            A.q[i] = 0.0;
          }
          rg[u] = mul_add_rn(rg[u], -alpha, qi);
          A.r[i] = rg[u];
          part = fma(rg[u], rg[u], part);
        }
    } else {
      // r -= alpha q over 16-byte pairs, two pairs in flight per thread
      // (q, r are 256-byte-aligned workspace arrays).
      const double2* q2 = reinterpret_cast<const double2*>(A.q);
      double2* r2 = reinterpret_cast<double2*>(A.r);
      double2* z2 = reinterpret_cast<double2*>(A.q);
      const long long np = (long long)n >> 1;
      const double na = -alpha;
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
    mark(3);
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
    double* t = p_old;
    p_old = p_new;
    p_new = t;
  }

#if SPCG_TRACE
  if (A.trace && threadIdx.x == 0) {
#pragma unroll
    for (int ph = 0; ph < 4; ++ph) A.trace[blockIdx.x * 5 + ph] = tr[ph];
    A.trace[blockIdx.x * 5 + 4] = P.wait_ns;
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

  // ---- deferred x += alpha_K p_K, then the true residual (solver.py:159-162) --
  if (RES) {
#pragma unroll
    for (int u = 0; u < kStages; ++u)
      if (li[u] >= 0) {
        if (iterations > 0) xr[u] = mul_add_rn(xr[u], alpha, pg[u]);
        A.x[li[u]] = xr[u];
      }
  } else if (iterations > 0) {
    for (long long i = gtid; i < n; i += gstride) A.x[i] = mul_add_rn(A.x[i], alpha, p_cur[i]);
  }
  if (A.recompute) {
    grid_allreduce(0.0, sm, A.slots, epoch);
    SrcPlain sx{A.x};
    part = 0.0;
    if (RES) {
      run_tiles<FMT, false, TWO, RES>(P, sm, M, sx, A.q, [&](int j, int i, const LineOut& o) {
        if (FMT == K_SCSR_ATOMIC) red_add_f64(A.q + i, o.q);
        else if (!ATOM) qg[j] = o.q;
      });
      if (ATOM) grid_allreduce(0.0, sm, A.slots, epoch);
#pragma unroll
      for (int u = 0; u < kStages; ++u)
        if (li[u] >= 0) {
          const double qi = ATOM ? A.q[li[u]] : qg[u];
          const double tr = mul_add_rn(bg[u], -1.0, qi);
          part = fma(tr, tr, part);
        }
    } else {
      run_tiles<FMT, false, TWO, RES>(P, sm, M, sx, A.q, [&](int, int i, const LineOut& o) {
        finish_plain<FMT>(o, i, A.q);
      });
      grid_allreduce(0.0, sm, A.slots, epoch);
      for (long long i = gtid; i < n; i += gstride) {
        const double tr = mul_add_rn(A.b[i], -1.0, A.q[i]);
        part = fma(tr, tr, part);
      }
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
