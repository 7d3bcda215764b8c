// clus.cuh — cluster-resident single-reduction CG (engine 5) for systems
// that fit one thread-block cluster (the paper's 30880-row FEM matrix).
//
// Why: on F-class systems a grid-wide all-reduce through global memory costs
// ~5.5 µs inside the solve (the writer fence waits for the CTA's published
// vector stores), against ~2.8 µs of SpMV.  One cluster of up to 16 CTAs
// (one per SM) replaces it with a hardware cluster barrier and DSMEM stores:
// ~0.8 µs per all-reduce (scripts/cluster_bench.cu).  Nothing is published
// through global memory inside the loop.
//
// Layout (built on the host, cluster_plan in spcg_b200.cu):
// * CTA c owns a contiguous row block [row_lo, row_hi) (<= 2048 rows) and
//   keeps the window [wlo, wlo+wn) of r that its rows gather, in shared
//   memory: own rows plus a lower and an upper halo (banded matrices: the
//   FEM mesh's bandwidth is 177 rows).
// * Its rows are stored as SELL-32 slices of 32 consecutive rows (natural
//   order: the window gathers of banded rows hit consecutive banks; sorting
//   by length saved padding but cost more in bank conflicts, host_cluster.cuh):
//   entry u of the slice's 32 rows is contiguous, so a
//   warp reads values and 16-bit window-relative columns conflict-free.  Each
//   row keeps its storage order, so a row sum is the reference's sequential
//   sum (bitwise equal to csr_gather / the privatized two-segment sum).
//   Slices that fit stay in shared memory for the whole solve; the rest are
//   re-read from L2 every iteration (coalesced, same layout).
// * Warp w handles slices w, w+16, w+32, w+48; each thread keeps its (up to
//   four) rows' x, r, p, s, w in registers.
//
// Iteration (Chronopoulos–Gear, the recurrences of cg1.cuh):
//   own rows:  p = r + b p,  s = w + b s,  x += a p,  r -= a s
//   halo rows: s = w + b s,  r -= a s     (redundant, bitwise the owner's
//              values: same inputs, same operations; w arrives by DSMEM)
//   w = A r, [r.r, r.w] partials -> every CTA's slot (DSMEM), boundary w ->
//   the neighbours' halo buffers (DSMEM)  ->  ONE barrier.cluster
// Double-buffered halo w and slots make one barrier per iteration race-free.
#pragma once
#include <cooperative_groups.h>

#include "cg.cuh"

namespace spcg {

#ifndef SPCG_CLUS_THREADS
#define SPCG_CLUS_THREADS 512
#endif
constexpr int kClusThreads = SPCG_CLUS_THREADS;
constexpr int kClusWarps = kClusThreads / 32;
constexpr int kClusSlicesPerWarp = 2048 / kClusThreads;
constexpr int kClusMaxRows = kClusWarps * kClusSlicesPerWarp * 32;  // 2048 per CTA
constexpr int kClusMax = 16;      // CTAs in one cluster (non-portable above 8)
constexpr int kClusGridMax = 256;  // CTAs of a multi-cluster grid (K clusters of 8)
#ifndef SPCG_PHASE_TIMERS
#define SPCG_PHASE_TIMERS 1  // leader-thread phase times for SolveReport.timings
#endif
#ifndef SPCG_CLUS_POST_FENCE
#define SPCG_CLUS_POST_FENCE 0  // (A/B) fence after the leader's post
#endif
constexpr int kClusSlotWords = 32;  // 256-byte global slot per cluster (own L2 line pair)

struct ClusCta {
  int row_lo, row_hi;  // own rows
  int clo, chi;        // rows of this CTA's cluster (halo rows outside come via global)
  int wlo, wn;         // r window [wlo, wlo + wn)
  int nslices, slice0; // slices [slice0, slice0 + nslices) of the global table
  int nsend, send0;    // DSMEM sends of boundary w
  int hlo;             // lower-halo rows (row_lo - wlo); halo index h -> row
  int nrecv;           // halo rows received from this cluster's CTAs per iteration
};
struct ClusSlice {
  int width;  // entries per row slot (max row length in the slice)
  int goff;   // first entry in the global SELL arrays
  int soff;   // first entry in shared memory, -1: streamed from L2
  int pad;
};
struct ClusSend {
  int dst;      // destination CTA (grid index; same cluster -> DSMEM, else global)
  int lo, hi;   // global rows [lo, hi) of this CTA
  int dst_off;  // halo index of row lo in dst
};

struct ClusArgs {
  const ClusCta* ctas;
  const ClusSlice* slices;
  const ClusSend* sends;
  const int2* rowmeta;  // per slice slot: {row (-1 pad), lenA << 16 | len}
  const double* gval;
  const unsigned short* gcol;
  const double* b;
  const double* x0;  // nullable
  double* x;
  double* scratch;   // n doubles (window initialisation)
  double* scratch2;  // n doubles (engine 6: the window of w0 = A r0)
  double* hist;
  CgDevResult* res;
  double tol;
  long long max_iter;
  int record_history;
  int recompute;
  int off_rwin, off_shalo, off_whalo, off_val, off_col;  // smem byte offsets
  int hcap;  // halo capacity (entries per halo buffer)
  unsigned long long* trace;  // nullable (SPCG_TRACE builds): [G][4] ns
  double* ghalo;              // K > 1: [2][G][hcap] halo w between clusters
  unsigned long long* gslots; // K > 1: [2][K][4] epoch-tagged cluster partials (zeroed)
  int cluster_size;           // the plan's cluster size (checked against the launch)
  double* coef;               // nullable (engine 6): (alpha, beta) of every update
};

constexpr int kClusSendCache = 8;  // send descriptors staged in shared memory

struct ClusShared {  // static part
  double slot[2][kClusMax][2];
  double red[2][kClusWarps];
  double tot[2][2];  // K > 1: grid totals broadcast by the cluster leader
  ClusSend send[kClusSendCache];
};

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// One row of a slice: sequential sum(s) in storage order.  TWO: the row is
// (L+D segment, L^T segment) summed separately and added (privatized mode).
#ifndef SPCG_CLUS_UNROLL
#define SPCG_CLUS_UNROLL 4
#endif
template <bool TWO, int U = SPCG_CLUS_UNROLL>
__device__ __forceinline__ double clus_row(const double* val, const unsigned short* col, int base,
                                           int width, int len, int lenA, const double* win) {
  double acc = 0.0, g = 0.0;
  for (int u = 0; u < width; u += U) {
    double a[U];
    int c[U];
#pragma unroll
    for (int t = 0; t < U; ++t) {
      a[t] = 0.0;
      c[t] = 0;
      if (u + t < len) {
        a[t] = val[base + (u + t) * 32];
        c[t] = col[base + (u + t) * 32];
      }
    }
#pragma unroll
    for (int t = 0; t < U; ++t)
      if (u + t < len) {
        if (TWO && u + t == lenA) {
          g = acc;
          acc = 0.0;
        }
        acc = __dadd_rn(acc, __dmul_rn(a[t], win[c[t]]));
      }
  }
  if (!TWO) return acc;
  if (lenA >= len) {
    g = acc;
    acc = 0.0;
  }
  return __dadd_rn(g, acc);
}

template <bool TWO>
__global__ void __launch_bounds__(kClusThreads, 1) clus_cg_kernel(const ClusArgs A) {
  namespace cgp = cooperative_groups;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ ClusShared cs;
  cgp::cluster_group cl = cgp::this_cluster();
  const int me = (int)cl.block_rank();   // rank in the cluster
  const int C = (int)cl.num_blocks();
  const int G = (int)gridDim.x;          // K clusters of C CTAs
  const int K = G / C;
  const int kc = (int)blockIdx.x / C;    // this CTA's cluster
  const int gme = (int)blockIdx.x;
  if (C != A.cluster_size) {  // launched without the plan's cluster shape: refuse
    if (gme == 0 && threadIdx.x == 0) {
      A.res->iterations = 0;
      A.res->fail_iter = 0;
      A.res->converged = 0;
      A.res->status = ST_BAD_LAUNCH;
      A.res->final_rel = 0.0;
      A.res->b_norm = 0.0;
    }
    return;
  }
  const ClusCta P = A.ctas[gme];
  double* rwin = reinterpret_cast<double*>(smem_raw + A.off_rwin);
  double* shalo = reinterpret_cast<double*>(smem_raw + A.off_shalo);
  double* whalo = reinterpret_cast<double*>(smem_raw + A.off_whalo);  // [2][hcap]
  double* sval = reinterpret_cast<double*>(smem_raw + A.off_val);
  unsigned short* scol = reinterpret_cast<unsigned short*>(smem_raw + A.off_col);
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  const bool leader = gme == 0 && tid == 0;
  const int nhalo = P.wn - (P.row_hi - P.row_lo);
  const int own0 = P.row_lo - P.wlo;  // window index of the first own row

  // resident slices -> shared memory (once)
  for (int s = 0; s < P.nslices; ++s) {
    const ClusSlice sd = A.slices[P.slice0 + s];
    if (sd.soff < 0) continue;
    const int cnt = sd.width * 32;
    for (int e = tid; e < cnt; e += kClusThreads) {
      sval[sd.soff + e] = A.gval[sd.goff + e];
      scol[sd.soff + e] = A.gcol[sd.goff + e];
    }
  }
  if (tid < min(P.nsend, kClusSendCache)) cs.send[tid] = A.sends[P.send0 + tid];
  // this thread's row slots
  int rrow[kClusSlicesPerWarp], rlen[kClusSlicesPerWarp], rlenA[kClusSlicesPerWarp];
  int swidth[kClusSlicesPerWarp], sbase[kClusSlicesPerWarp];
  bool sres[kClusSlicesPerWarp];
  double xr[kClusSlicesPerWarp], rg[kClusSlicesPerWarp], pg[kClusSlicesPerWarp],
      sg[kClusSlicesPerWarp], wg[kClusSlicesPerWarp];
#pragma unroll
  for (int k = 0; k < kClusSlicesPerWarp; ++k) {
    const int s = wp + kClusWarps * k;
    rrow[k] = -1;
    rlen[k] = rlenA[k] = swidth[k] = sbase[k] = 0;
    sres[k] = false;
    xr[k] = rg[k] = pg[k] = sg[k] = wg[k] = 0.0;
    if (s < P.nslices) {
      const ClusSlice sd = A.slices[P.slice0 + s];
      const int2 rm = A.rowmeta[(size_t)(P.slice0 + s) * 32 + lane];
      rrow[k] = rm.x;
      rlen[k] = rm.y & 0xffff;
      rlenA[k] = (int)((unsigned)rm.y >> 16);
      swidth[k] = sd.width;
      sres[k] = sd.soff >= 0;
      sbase[k] = (sres[k] ? sd.soff : sd.goff) + lane;
    }
  }
  __syncthreads();

  // w_k = A win for this thread's rows; only rows with rrow >= 0 matter
  auto spmv = [&](double* out) {
#pragma unroll
    for (int k = 0; k < kClusSlicesPerWarp; ++k) {
      out[k] = 0.0;
      if (swidth[k] > 0) {  // warp-uniform
        const double q = sres[k] ? clus_row<TWO>(sval, scol, sbase[k], swidth[k], rlen[k], rlenA[k], rwin)
                                 : clus_row<TWO>(A.gval, A.gcol, sbase[k], swidth[k], rlen[k], rlenA[k], rwin);
        out[k] = rrow[k] >= 0 ? q : 0.0;
      }
    }
  };
  // cluster all-reduce of two values (fixed order: warps, then CTA ranks)
  uint32_t epoch = 0;
#if SPCG_TRACE
  unsigned long long tlv[4] = {0, 0, 0, 0};  // exchange, b1exit->b2exit, b1 wait, send_w
  unsigned long long tpost = 0;               // leader: sum of slot-post times since start
  const unsigned long long tstart = globaltimer_ns();
#endif
  auto allreduce2 = [&](double& v0, double& v1) {
    const int bank = (int)(epoch++ & 1u);
    double a0 = warp_sum(v0), a1 = warp_sum(v1);
    if (lane == 0) {
      cs.red[0][wp] = a0;
      cs.red[1][wp] = a1;
    }
    __syncthreads();
    if (wp == 0) {
      double b0 = lane < kClusWarps ? cs.red[0][lane] : 0.0;
      double b1 = lane < kClusWarps ? cs.red[1][lane] : 0.0;
      b0 = warp_sum(b0);
      b1 = warp_sum(b1);
      if (lane < C) {
        double* dst = cl.map_shared_rank(&cs.slot[bank][me][0], lane);
        dst[0] = b0;
        dst[1] = b1;
      }
    }
#if SPCG_TRACE
    const unsigned long long tb0 = (A.trace && tid == 0) ? globaltimer_ns() : 0;
#endif
    cluster_sync_all();
#if SPCG_TRACE
    if (A.trace && tid == 0) tlv[2] += globaltimer_ns() - tb0;
#endif
    double t0 = 0.0, t1 = 0.0;
    for (int c = 0; c < C; ++c) {
      t0 += cs.slot[bank][c][0];
      t1 += cs.slot[bank][c][1];
    }
    if (K > 1) {
      // second level through global memory: the cluster leader posts the
      // cluster's partials in its own 256-byte slot as epoch-tagged 64-bit
      // words (volatile scalar accesses; one fence before the post — the
      // cluster barrier above made the cluster's global halo stores part of
      // it — and one after the poll); the leader polls the K slots and
      // broadcasts over DSMEM behind a second cluster barrier (letting every
      // CTA poll was 2.3x slower).  Sums run in cluster order in every CTA.
      const uint32_t tag = epoch;  // identical sequence in every CTA, never 0
      unsigned long long* gb = A.gslots + (size_t)bank * K * kClusSlotWords;
#if SPCG_TRACE
      unsigned long long ta = (A.trace && tid == 0) ? globaltimer_ns() : 0;
#endif
      if (me == 0 && tid == 0) {
        fence_acq_rel_gpu();
        const unsigned long long u0 = (unsigned long long)__double_as_longlong(t0);
        const unsigned long long u1 = (unsigned long long)__double_as_longlong(t1);
#if SPCG_TRACE
        if (A.trace) tpost += globaltimer_ns() - tstart;
#endif
        volatile unsigned long long* dst = gb + kClusSlotWords * kc;
        dst[0] = (u0 & 0xffffffff00000000ull) | tag;
        dst[1] = (u0 << 32) | tag;
        dst[2] = (u1 & 0xffffffff00000000ull) | tag;
        dst[3] = (u1 << 32) | tag;
#if SPCG_CLUS_POST_FENCE
        // performed before this warp starts polling (see clus_pipe.cuh:
        // an unfenced post could stay invisible to the pollers for ~6.5 us)
        fence_acq_rel_gpu();
#endif
      }
      if (me == 0 && wp == 0) {
        double c0 = 0.0, c1 = 0.0;
        {
          // warp-uniform poll (see clus_pipe.cuh: a divergent spin loop let
          // an early leader finish ~7 us after its last slot was visible)
          const volatile unsigned long long* src = gb + kClusSlotWords * (lane < K ? lane : 0);
          unsigned long long a = 0, b = 0, c = 0, d = 0, spins = 0;
          bool ok = lane >= K;
          while (!__all_sync(0xffffffffu, ok)) {
            if (!ok) {
              // spin on the last-written word only (one load per round keeps
              // the pollers' pressure on the slot lines low), then validate all
              d = src[3];
              if ((uint32_t)d == tag) {
                a = src[0];
                b = src[1];
                c = src[2];
                ok = (uint32_t)a == tag && (uint32_t)b == tag && (uint32_t)c == tag;
              }
            }
            if (++spins > kSpinLimit) asm volatile("trap;");
          }
          if (lane < K) {
            c0 = __longlong_as_double((long long)((a & 0xffffffff00000000ull) | (b >> 32)));
            c1 = __longlong_as_double((long long)((c & 0xffffffff00000000ull) | (d >> 32)));
          }
        }
        fence_acq_rel_gpu();
#if SPCG_TRACE
        if (A.trace && tid == 0) {
          const unsigned long long tb = globaltimer_ns();
          tlv[0] += tb - ta;
          ta = tb;
        }
#endif
        double s0 = 0.0, s1 = 0.0;
        for (int k = 0; k < K; ++k) {  // fixed order over clusters
          s0 += __shfl_sync(0xffffffffu, c0, k);
          s1 += __shfl_sync(0xffffffffu, c1, k);
        }
        if (lane < C) {
          double* d2 = cl.map_shared_rank(&cs.tot[bank][0], lane);
          d2[0] = s0;
          d2[1] = s1;
        }
      }
      cluster_sync_all();
#if SPCG_TRACE
      if (A.trace && tid == 0) tlv[1] += globaltimer_ns() - ta;
#endif
      t0 = cs.tot[bank][0];
      t1 = cs.tot[bank][1];
    }
    v0 = t0;
    v1 = t1;
  };
  // boundary w of this CTA -> the halo buffers of the CTAs that gather it
  auto send_w = [&](int buf) {
    for (int e = 0; e < P.nsend; ++e) {
      const ClusSend sd = e < kClusSendCache ? cs.send[e] : A.sends[P.send0 + e];
      const bool remote_cluster = sd.dst / C != kc;
      double* dst = remote_cluster ? A.ghalo + ((size_t)buf * G + sd.dst) * A.hcap
                                   : cl.map_shared_rank(whalo + (size_t)buf * A.hcap, sd.dst % C);
#pragma unroll
      for (int k = 0; k < kClusSlicesPerWarp; ++k)
        if (rrow[k] >= sd.lo && rrow[k] < sd.hi) dst[sd.dst_off + rrow[k] - sd.lo] = wg[k];
    }
  };
  // window index of halo index h
  auto halo_win = [&](int h) { return h < P.hlo ? h : own0 + (P.row_hi - P.row_lo) + (h - P.hlo); };
  // w of halo index h from buffer buf: DSMEM-delivered (same cluster) or
  // global (other cluster, L2 only)
  auto halo_w = [&](int buf, int h) {
    const int hrow = h < P.hlo ? P.wlo + h : P.row_hi + (h - P.hlo);
    return (hrow >= P.clo && hrow < P.chi) ? whalo[(size_t)buf * A.hcap + h]
                                           : __ldcg(A.ghalo + ((size_t)buf * G + gme) * A.hcap + h);
  };
  double wpre = 0.0;  // halo w of h = tid for the next update, loaded right after the barrier

  // ||b||
  double part = 0.0, dummy = 0.0;
#pragma unroll
  for (int k = 0; k < kClusSlicesPerWarp; ++k)
    if (rrow[k] >= 0) {
      const double bv = A.b[rrow[k]];
      part = fma(bv, bv, part);
    }
  allreduce2(part, dummy);
  const double b_norm = sqrt(part);
  if (b_norm == 0.0) {  // solver.py:109-118
#pragma unroll
    for (int k = 0; k < kClusSlicesPerWarp; ++k)
      if (rrow[k] >= 0) A.x[rrow[k]] = 0.0;
    if (leader) {
      A.res->iterations = 0;
      A.res->fail_iter = 0;
      A.res->converged = 1;
      A.res->status = ST_OK;
      A.res->final_rel = 0.0;
      A.res->b_norm = 0.0;
    }
    return;
  }
  // x = x0, r0 = b - A x0 (solver.py:120-124)
  if (A.x0 != nullptr) {
    for (int j = tid; j < P.wn; j += kClusThreads) rwin[j] = A.x0[P.wlo + j];
    __syncthreads();
    double qv[kClusSlicesPerWarp];
    spmv(qv);
#pragma unroll
    for (int k = 0; k < kClusSlicesPerWarp; ++k)
      if (rrow[k] >= 0) {
        xr[k] = A.x0[rrow[k]];
        rg[k] = mul_add_rn(A.b[rrow[k]], -1.0, qv[k]);
      }
    __syncthreads();  // window reads done before it is overwritten
  } else {
#pragma unroll
    for (int k = 0; k < kClusSlicesPerWarp; ++k)
      if (rrow[k] >= 0) rg[k] = A.b[rrow[k]];
  }
  // r0 window: own rows through global scratch (once), gamma0
  part = 0.0;
  dummy = 0.0;
#pragma unroll
  for (int k = 0; k < kClusSlicesPerWarp; ++k)
    if (rrow[k] >= 0) {
      A.scratch[rrow[k]] = rg[k];
      part = fma(rg[k], rg[k], part);
    }
  allreduce2(part, dummy);  // release/acquire at cluster scope covers scratch
  double gam = part;
  for (int j = tid; j < P.wn; j += kClusThreads) rwin[j] = __ldcg(A.scratch + P.wlo + j);
  for (int h = tid; h < A.hcap; h += kClusThreads) shalo[h] = 0.0;
  __syncthreads();

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
    // w0 = A r0, d0 = r0.w0; boundary w0 -> neighbours' whalo[0]
    spmv(wg);
    part = 0.0;
#pragma unroll
    for (int k = 0; k < kClusSlicesPerWarp; ++k)
      if (rrow[k] >= 0) part += rg[k] * wg[k];
    send_w(0);
    allreduce2(part, dummy);
    if (tid < nhalo) wpre = halo_w(0, tid);
    const double d0 = part;
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

  // phase times: the leader thread always (SolveReport.timings), every CTA's
  // thread 0 when tracing
  unsigned long long tr[4] = {0, 0, 0, 0};
  const bool tl = tid == 0 && ((SPCG_PHASE_TIMERS && gme == 0) || (SPCG_TRACE && A.trace));
  unsigned long long tlast = tl ? globaltimer_ns() : 0;
  auto mark = [&](int ph) {
    if (tl) {
      const unsigned long long t = globaltimer_ns();
      tr[ph] += t - tlast;
      tlast = t;
    }
  };
  for (long long it = 0; status == ST_OK && it < max_it; ++it) {
    const int rb = (int)(it & 1), wb = rb ^ 1;
    const double na = -alpha;
    // own rows (registers) and halo rows (shared) advance to r_{i+1}
#pragma unroll
    for (int k = 0; k < kClusSlicesPerWarp; ++k)
      if (rrow[k] >= 0) {
        pg[k] = mul_add_rn(rg[k], beta, pg[k]);
        sg[k] = mul_add_rn(wg[k], beta, sg[k]);
        xr[k] = mul_add_rn(xr[k], alpha, pg[k]);
        rg[k] = mul_add_rn(rg[k], na, sg[k]);
        rwin[own0 + rrow[k] - P.row_lo] = rg[k];
      }
    for (int h = tid; h < nhalo; h += kClusThreads) {
      const double wv = h == tid ? wpre : halo_w(rb, h);
      const double sh = mul_add_rn(wv, beta, shalo[h]);
      shalo[h] = sh;
      const int j = halo_win(h);
      rwin[j] = mul_add_rn(rwin[j], na, sh);
    }
    __syncthreads();
    mark(0);
    spmv(wg);
    mark(1);
    double g_new = 0.0, d_new = 0.0;
#pragma unroll
    for (int k = 0; k < kClusSlicesPerWarp; ++k)
      if (rrow[k] >= 0) {
        g_new = fma(rg[k], rg[k], g_new);
        d_new += rg[k] * wg[k];
      }
#if SPCG_TRACE
    const unsigned long long ts0 = (A.trace && tid == 0) ? globaltimer_ns() : 0;
#endif
    send_w(wb);
#if SPCG_TRACE
    if (A.trace && tid == 0) tlv[3] += globaltimer_ns() - ts0;
#endif
    allreduce2(g_new, d_new);
    if (tid < nhalo) wpre = halo_w(wb, tid);  // in flight during the scalar updates
    mark(2);
    const long long kk = it + 1;  // reference iteration number
    rel = sqrt(g_new) / b_norm;
    if (!isfinite(rel)) {
      status = ST_NF_RES;
      fail_iter = kk;
      break;
    }
    if (A.record_history && leader) A.hist[kk - 1] = rel;
    iterations = kk;
    if (sqrt(g_new) <= tol_b) {
      converged = 1;
      break;
    }
    const double beta_n = g_new / gam;
    if (!isfinite(beta_n)) {
      status = ST_NF_BETA;
      fail_iter = kk;
      break;
    }
    if (kk < max_it) {  // p.Ap of iteration kk+1 (solver.py:135-139)
      const double eta = d_new - beta_n * g_new / alpha;
      if (eta <= 0.0) {
        status = ST_NOT_SPD;
        fail_iter = kk + 1;
        break;
      }
      const double alpha_n = g_new / eta;
      if (!isfinite(alpha_n)) {
        status = ST_NF_ALPHA;
        fail_iter = kk + 1;
        break;
      }
      alpha = alpha_n;
    }
    beta = beta_n;
    gam = g_new;
  }

#if SPCG_TRACE
  if (A.trace && tid == 0) {
    for (int ph = 0; ph < 3; ++ph) A.trace[gme * 8 + ph] = tr[ph];
    for (int ph = 0; ph < 4; ++ph) A.trace[gme * 8 + 3 + ph] = tlv[ph];
    A.trace[gme * 8 + 7] = tpost;
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
    return;
  }
#pragma unroll
  for (int k = 0; k < kClusSlicesPerWarp; ++k)
    if (rrow[k] >= 0) A.x[rrow[k]] = xr[k];
  if (A.recompute) {  // true residual ||b - A x|| / ||b||
    part = 0.0;
    dummy = 0.0;
    allreduce2(part, dummy);  // x visible cluster-wide
    for (int j = tid; j < P.wn; j += kClusThreads) rwin[j] = __ldcg(A.x + P.wlo + j);
    __syncthreads();
    double qv[kClusSlicesPerWarp];
    spmv(qv);
    part = 0.0;
#pragma unroll
    for (int k = 0; k < kClusSlicesPerWarp; ++k)
      if (rrow[k] >= 0) {
        const double tr = mul_add_rn(A.b[rrow[k]], -1.0, qv[k]);
        part = fma(tr, tr, part);
      }
    allreduce2(part, dummy);
    rel = sqrt(part) / b_norm;
  }
  if (leader) {
    A.res->iterations = iterations;
    A.res->fail_iter = 0;
    A.res->converged = converged;
    A.res->status = ST_OK;
    A.res->final_rel = rel;
    A.res->b_norm = b_norm;
    A.res->phase_ns[0] = tr[1];  // SpMV
    A.res->phase_ns[1] = tr[2];  // all-reduce
    A.res->phase_ns[2] = tr[0];  // update
  }
}

}  // namespace spcg
