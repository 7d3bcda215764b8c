// clus_pipe.cuh — pipelined cluster-resident CG (engine 6): the plan, data
// layout and row slots of engine 5 (clus.cuh), with the Ghysels–Vanroose
// recurrences so that the iteration's SpMV overlaps its all-reduce.
//
// Why: on F the engine-5 iteration is update (~0.85 us) + SpMV (~1.2 us) +
// all-reduce (~3.5 us: two cluster barriers and the leaders' exchange through
// global memory), strictly in sequence, because the SpMV input r needs the
// scalars of the previous reduction.  Pipelined CG reduces (r.r, w.r) and
// computes n = A w at the same time (w = A r by recurrence, so the SpMV needs
// no scalar of the current iteration):
//   gamma = r.r, delta = w.r   (all-reduce in flight)  ||  n = A w
//   beta = gamma / gamma_old,  alpha = gamma / (delta - beta gamma / alpha_old)
//   z = n + beta z,  s = w + beta s,  p = r + beta p,
//   x += alpha p,  r -= alpha s,  w -= alpha z
// (reference CG order, solver.py:132-157: the same alpha/beta formulas as the
// single-reduction engines, fp64; scripts/pipecg_numerics.py: F converges in
// the reference's 329 iterations, x within 4.9e-11 of the reference).
//
// Synchronisation per iteration i (one CTA per SM, 15 row warps + 1 comm
// warp; no cluster barrier inside the loop):
//   row warps: n = A w from the shared window of w; boundary n -> the cluster
//              neighbours' shared memory by st.async (completing on their
//              mbarrier mbB) and to other clusters as epoch-tagged words in
//              global memory; wait on the own mbB (totals + neighbours' n);
//              scalars; update; (r.r, w.r) of i+1 -> rank 0 by st.async (mbA);
//              halo rows; named barrier of the row warps
//   comm warp (cluster rank 0): wait on mbA (every row warp's partials),
//              sum in fixed order; K > 1: post to the own epoch-tagged global
//              slot, poll the K slots, sum; st.async the totals to every
//              cluster CTA (mbB)
// so the leaders' global exchange runs while the row warps do the SpMV.
// Halo rows of w advance redundantly in every CTA that gathers them
// (z = n + beta z, w -= alpha z: the owner's operations on the owner's
// inputs, so bitwise the owner's values), which needs only the neighbours'
// boundary n of the same iteration.
#pragma once
#include "clus.cuh"

namespace spcg {

// 15 row warps + the communication warp: a 17th warp would cap the kernel at
// 96 registers (5 warps on one SM sub-partition) and spill the row slots
constexpr int kPipeThreads = kClusThreads;
constexpr int kPipeWarps = kPipeThreads / 32;
constexpr int kPipeRowWarps = kPipeWarps - 1;
constexpr int kPipeRowThreads = kPipeRowWarps * 32;
constexpr int kPipeMaxSlices = kPipeRowWarps * kClusSlicesPerWarp;  // per CTA (host-checked)
constexpr int kPipeMaxSlices2 = kPipeRowWarps * 2;

struct PipeShared {
  double slot[2][kClusMax][2];  // setup / tail all-reduce (cluster barriers)
  double red[2][kPipeWarps];
  double tot[2][2];
  ClusSend send[kClusSendCache];
  // the loop's messages (by iteration parity): rank 0 gathers every row warp's
  // partials of the cluster in wslot (mbA); every CTA receives the totals in
  // ltot and its cluster neighbours' boundary n in nhalo (mbB)
  double wslot[2][kClusMax][kPipeRowWarps][2];
  double ltot[3][2];
  uint64_t mbA[2], mbB[3];
  unsigned long long fine[16];  // SPCG_PIPE_FINE sub-phase totals
};
// static shared memory of the larger of the two cluster kernels (the plan's
// dynamic budget is shared by engines 5 and 6)
constexpr size_t kClusStatic = sizeof(PipeShared) > sizeof(ClusShared) ? sizeof(PipeShared) : sizeof(ClusShared);

// SpMV unroll of the 2-slot kernel (4: 2.91 vs 2.86 us per iteration on F);
// the 4-slot kernel uses SPCG_CLUS_UNROLL (clus.cuh)
#ifndef SPCG_PIPE_SENDMASK
#define SPCG_PIPE_SENDMASK 1  // per-warp mask of the send descriptors
#endif
#ifndef SPCG_PIPE_UNROLL_ONE2
#define SPCG_PIPE_UNROLL_ONE2 8
#endif
// instrumented builds (dev): SM-cycle sub-phase timers; the leaders' exchange
// timeline of iterations 100-107 (both written through SPCG_CLUS_DEBUG)
#ifndef SPCG_PIPE_FINE
#define SPCG_PIPE_FINE 0
#endif
#ifndef SPCG_XCHG_TRACE
#define SPCG_XCHG_TRACE 0
#endif
// Measured and removed A/B variants: deferral of the remote halo
// rows to the next iteration (replaced by loads issued right after the wait),
// the privatized two-sum SpMV of symmetric-half rows (one chain instead),
// warp-uniform tagged halo loads, back-off in the polls, a fence or a release
// store on the leaders' post, aligned cluster barriers, every CTA polling the
// leaders' slots, system-scope 8-byte tagged words.
// An epoch-tagged double: {hi32 | tag, lo32 << 32 | tag}, written as one
// 16-byte relaxed store at gpu scope (each 8-byte word is single-copy atomic
// and carries the tag, so a reader never takes a torn value for a new one)
__device__ __forceinline__ void tagged_store(unsigned long long* dst, double v, uint32_t tag) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(dst),
               "l"((u & 0xffffffff00000000ull) | tag), "l"((u << 32) | tag) : "memory");
}
// both words in one 16-byte load; tagged_finish validates them when the
// value is consumed and re-polls until both carry the tag
__device__ __forceinline__ void tagged_issue(const unsigned long long* src, unsigned long long& a,
                                             unsigned long long& b) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(src) : "memory");
}
__device__ __forceinline__ double tagged_finish(const unsigned long long* src, unsigned long long a,
                                                unsigned long long b, uint32_t tag) {
  unsigned long long spins = 0;
  while ((uint32_t)a != tag || (uint32_t)b != tag) {
    tagged_issue(src, a, b);
    if (++spins > kSpinLimit) asm volatile("trap;");
  }
  return __longlong_as_double((long long)((a & 0xffffffff00000000ull) | (b >> 32)));
}
__device__ __forceinline__ double tagged_load(const unsigned long long* src, uint32_t tag) {
  unsigned long long a, b;
  tagged_issue(src, a, b);
  return tagged_finish(src, a, b, tag);
}

// NS: row slots per thread (2 when the plan's CTAs have <= 30 slices: fewer
// live registers, no spills; 4 otherwise)
// (A/B knobs) register rows: entries per row and CTA threads; 320 threads
// (9 row warps) never applied to F, whose fullest CTA has 10 slices
#ifndef SPCG_REG_W
#define SPCG_REG_W 24
#endif
#ifndef SPCG_REG_THREADS
#define SPCG_REG_THREADS 384
#endif
constexpr int kRegW = SPCG_REG_W;  // register rows: entries per row (the F-mesh's longest row)
constexpr int kRegThreads = SPCG_REG_THREADS;  // register rows: 11 row warps + the comm warp
constexpr int kRegW2 = 8;  // register rows with two slots per thread: short rows (stencils)

// TH: threads of the CTA (512, or 384 for the register-row variant: the
// 168-register budget); REG: each thread keeps its row's values and columns
// in registers (one row slot, rows of <= kRegW entries) so the SpMV reads
// only the window gathers from shared memory
template <int NS, int TH = kPipeThreads, int RW = 0>
__global__ void __launch_bounds__(TH, 1) clus_pcg_kernel(const ClusArgs A) {
  constexpr int PW_ = TH / 32, PRW_ = PW_ - 1, PRT_ = PRW_ * 32;
  constexpr bool REG = RW > 0;  // RW: register-row width (entries), 0: rows from shared memory
  namespace cgp = cooperative_groups;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ PipeShared cs;
  cgp::cluster_group cl = cgp::this_cluster();
  const int me = (int)cl.block_rank();
  const int C = (int)cl.num_blocks();
  const int G = (int)gridDim.x;
  const int K = G / C;
  const int kc = (int)blockIdx.x / C;
  const int gme = (int)blockIdx.x;
  if (C != A.cluster_size) {
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
  double* wwin = reinterpret_cast<double*>(smem_raw + A.off_rwin);   // window of w (SpMV input)
  double* zhalo = reinterpret_cast<double*>(smem_raw + A.off_shalo); // z of the halo rows
  double* nhalo = reinterpret_cast<double*>(smem_raw + A.off_whalo); // [3][hcap] halo n (DSMEM)
  double* sval = reinterpret_cast<double*>(smem_raw + A.off_val);
  unsigned short* scol = reinterpret_cast<unsigned short*>(smem_raw + A.off_col);
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  const bool comm = wp == PRW_;
  const bool leader = gme == 0 && tid == 0;
  const int nh = P.wn - (P.row_hi - P.row_lo);
  const int own0 = P.row_lo - P.wlo;
  unsigned long long* gh = reinterpret_cast<unsigned long long*>(A.ghalo);  // [3][G][hcap][2]

  // (REG: the SpMV reads its operands from registers, loaded below; the
  // shared-memory copy would only add a chain of dependent cold loads to the
  // prologue)
  if (!REG) {
    for (int s = 0; s < P.nslices; ++s) {
      const ClusSlice sd = A.slices[P.slice0 + s];
      if (sd.soff < 0) continue;
      const int cnt = sd.width * 32;
      for (int e = tid; e < cnt; e += TH) {
        sval[sd.soff + e] = A.gval[sd.goff + e];
        scol[sd.soff + e] = A.gcol[sd.goff + e];
      }
    }
  }
  if (tid < min(P.nsend, kClusSendCache)) cs.send[tid] = A.sends[P.send0 + tid];
  int rrow[NS], rlen[NS], rlenA[NS];
  int swidth[NS], sbase[NS];
  bool sres[NS];
  double xr[NS], rg[NS], pg[NS],
      sg[NS], wg[NS], zg[NS];
#pragma unroll
  for (int k = 0; k < NS; ++k) {
    const int s = wp + PRW_ * k;
    rrow[k] = -1;
    rlen[k] = rlenA[k] = swidth[k] = sbase[k] = 0;
    sres[k] = false;
    xr[k] = rg[k] = pg[k] = sg[k] = wg[k] = zg[k] = 0.0;
    if (!comm && s < P.nslices) {
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
  // REG: each slot's row values and window-relative columns, read once
  constexpr int RWA = REG ? RW : 2;
  double vreg[NS][RWA];
  uint32_t creg[NS][RWA / 2];
  if (REG) {
    // from the global SELL arrays: the shared-memory copy above is still in
    // flight in other threads (no barrier yet)
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const int s = wp + PRW_ * k;
      const int gb = (!comm && s < P.nslices) ? A.slices[P.slice0 + s].goff + lane : 0;
#pragma unroll
      for (int u = 0; u < RWA; ++u) {
        const bool in = u < rlen[k];
        vreg[k][u] = in ? A.gval[gb + u * 32] : 0.0;
        const uint32_t c = in ? (uint32_t)A.gcol[gb + u * 32] : 0u;
        if (u & 1) creg[k][u >> 1] |= c << 16;
        else creg[k][u >> 1] = c;
      }
    }
  }
  if (tid == 0) {
    for (int i = 0; i < 3; ++i) {
      if (i < 2) mbar_init(&cs.mbA[i], 1);
      mbar_init(&cs.mbB[i], 1);
    }
    fence_mbar_init();  // visible to the cluster at the first cluster barrier
  }
  __syncthreads();
  // bytes this CTA receives per iteration on mbB: the totals and one double
  // per halo row its cluster neighbours send (host-counted from the sends)
  const int bbytes = 16 + 8 * P.nrecv;

  auto spmv = [&](double* out) {
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      out[k] = 0.0;
      if (swidth[k] > 0) {
        // two-segment rows: unroll 2 (unroll 4 spilled at the 128-register cap)
        // a symmetric-half row (stored L+D entries, then its L^T entries:
        // column order) is summed in ONE chain like a full row -- engine 6's
        // recurrences differ from the reference's anyway, so the privatized
        // two-sum order bought nothing (S: 3.77 -> 2.86 us per iteration,
        // bitwise the full-row solve)
        constexpr int U = NS == 2 ? SPCG_PIPE_UNROLL_ONE2 : SPCG_CLUS_UNROLL;
        double q;
        if (REG) {  // the same storage-order sum, operands from registers
          q = 0.0;
#pragma unroll
          for (int u = 0; u < RWA; ++u)
            if (u < rlen[k]) {
              const uint32_t c = (u & 1) ? (creg[k][u >> 1] >> 16) : (creg[k][u >> 1] & 0xffffu);
              q = __dadd_rn(q, __dmul_rn(vreg[k][u], wwin[c]));
            }
        } else {
          q = sres[k] ? clus_row<false, U>(sval, scol, sbase[k], swidth[k], rlen[k], rlenA[k], wwin)
                      : clus_row<false, U>(A.gval, A.gcol, sbase[k], swidth[k], rlen[k], rlenA[k], wwin);
        }
        out[k] = rrow[k] >= 0 ? q : 0.0;
      }
    }
  };
  uint32_t epoch = 0;
  // block + cluster partial sums of (v0, v1) -> every cluster CTA's slot[bank]
  auto post_partials = [&](double v0, double v1, int bank) {
    const double a0 = warp_sum(v0), a1 = warp_sum(v1);
    if (lane == 0) {
      cs.red[0][wp] = a0;
      cs.red[1][wp] = a1;
    }
    __syncthreads();
    if (wp == 0) {
      double b0 = lane < PW_ ? cs.red[0][lane] : 0.0;
      double b1 = lane < PW_ ? cs.red[1][lane] : 0.0;
      b0 = warp_sum(b0);
      b1 = warp_sum(b1);
      if (lane < C) {
        double* dst = cl.map_shared_rank(&cs.slot[bank][me][0], lane);
        dst[0] = b0;
        dst[1] = b1;
      }
    }
  };
  // second level (K > 1, one warp of cluster rank 0, after the slots are
  // complete): cluster sum -> own epoch-tagged global slot, poll the K slots,
  // sum in cluster order, broadcast to the cluster's tot[bank] by DSMEM
  // fenced: the exchange also publishes the CTAs' earlier global stores
  // (setup / tail: scratch and x windows); inside the loop it carries only
  // its own epoch-tagged words, so it needs no fence
  long long cur_it = -1;  // loop iteration of the exchange (exchange trace)
  // v0, v1: this cluster's sums in, the grid's sums (cluster order) out
  auto exchange_core = [&](int bank, uint32_t tag, bool fenced, double& v0, double& v1, bool post = true) {
    // exchange trace (A.trace): iterations 100..107 of every cluster leader:
    // [post time, done time, time lane k saw cluster k's slot]
    unsigned long long* xr = (SPCG_XCHG_TRACE && A.trace && cur_it >= 100 && cur_it < 108)
        ? A.trace + 8 * (size_t)gridDim.x + ((size_t)kc * 8 + (size_t)(cur_it - 100)) * 34
        : nullptr;
    const double t0 = v0, t1 = v1;
    unsigned long long* gb = A.gslots + (size_t)bank * K * kClusSlotWords;
    if (post && lane == 0) {
      if (fenced) fence_acq_rel_gpu();
      unsigned long long* dst = gb + kClusSlotWords * kc;
      const unsigned long long u0 = (unsigned long long)__double_as_longlong(t0);
      const unsigned long long u1 = (unsigned long long)__double_as_longlong(t1);
      asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(dst),
                   "l"((u0 & 0xffffffff00000000ull) | tag), "l"((u0 << 32) | tag) : "memory");
      asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(dst + 2),
                   "l"((u1 & 0xffffffff00000000ull) | tag), "l"((u1 << 32) | tag) : "memory");
      if (xr) xr[0] = globaltimer_ns();
    }
    double c0 = 0.0, c1 = 0.0;
    {
      // warp-uniform poll: every lane stays in the loop until all K slots
      // are in (__all_sync), so no lane spins alone while finished lanes
      // wait at a reconvergence point -- a divergent spin loop let a leader
      // that arrived early finish ~7 us after its last slot was visible
      // (profiles/r02/bimodal.md)
      const unsigned long long* src = gb + kClusSlotWords * (lane < K ? lane : 0);
      unsigned long long a = 0, b = 0, c = 0, d = 0, spins = 0;
      bool ok = lane >= K;
      while (!__all_sync(0xffffffffu, ok)) {
        if (!ok) {
          // the slot's four words in one round trip (two 16-byte loads in
          // flight together); every word carries the tag
          asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];"
                       : "=l"(a), "=l"(b) : "l"(src) : "memory");
          asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];"
                       : "=l"(c), "=l"(d) : "l"(src + 2) : "memory");
          ok = (uint32_t)a == tag && (uint32_t)b == tag && (uint32_t)c == tag && (uint32_t)d == tag;
          if (ok && xr) xr[2 + lane] = globaltimer_ns();
        }
        if (++spins > kSpinLimit) asm volatile("trap;");
      }
      if (lane < K) {
        c0 = __longlong_as_double((long long)((a & 0xffffffff00000000ull) | (b >> 32)));
        c1 = __longlong_as_double((long long)((c & 0xffffffff00000000ull) | (d >> 32)));
      }
    }
    if (fenced) fence_acq_rel_gpu();
    // the K cluster sums in a fixed xor tree: IEEE addition commutes, so every
    // lane -- and every leader -- ends with the same bits
    const double s0 = warp_sum(c0), s1 = warp_sum(c1);
    if (xr && lane == 0) xr[1] = globaltimer_ns();
    v0 = s0;
    v1 = s1;
  };
  // blocking form (setup and tail): the cluster's slots in, the grid totals
  // out to every cluster CTA's tot[bank] (DSMEM)
  auto exchange = [&](int bank, uint32_t tag, bool fenced) {
    double s0 = 0.0, s1 = 0.0;
    for (int c = 0; c < C; ++c) {
      s0 += cs.slot[bank][c][0];
      s1 += cs.slot[bank][c][1];
    }
    exchange_core(bank, tag, fenced, s0, s1);
    if (lane < C) {
      double* d2 = cl.map_shared_rank(&cs.tot[bank][0], lane);
      d2[0] = s0;
      d2[1] = s1;
    }
  };
  auto totals = [&](int bank, double& v0, double& v1) {
    if (K > 1) {
      v0 = cs.tot[bank][0];
      v1 = cs.tot[bank][1];
    } else {
      v0 = v1 = 0.0;
      for (int c = 0; c < C; ++c) {
        v0 += cs.slot[bank][c][0];
        v1 += cs.slot[bank][c][1];
      }
    }
  };
  // blocking all-reduce (setup and tail)
  auto allreduce2 = [&](double& v0, double& v1) {
    const int bank = (int)(epoch++ & 1u);
    const uint32_t tag = epoch;
    post_partials(v0, v1, bank);
    cluster_sync_all();
    if (K > 1) {
      if (me == 0 && wp == 0) exchange(bank, tag, true);
      cluster_sync_all();
    }
    totals(bank, v0, v1);
  };
  auto halo_win = [&](int h) { return h < P.hlo ? h : own0 + (P.row_hi - P.row_lo) + (h - P.hlo); };
  // n of halo index h from buffer buf: DSMEM (same cluster) or tagged global
  auto halo_local = [&](int h) {
    const int hrow = h < P.hlo ? P.wlo + h : P.row_hi + (h - P.hlo);
    return hrow >= P.clo && hrow < P.chi;
  };
  auto halo_n = [&](bool act, int buf, int h, uint32_t tag) {
    if (!act) return 0.0;
    if (halo_local(h)) return nhalo[(size_t)buf * A.hcap + h];
    return tagged_load(gh + (((size_t)buf * G + gme) * A.hcap + h) * 2, tag);
  };
  // (SPCG_PIPE_SENDMASK) bit e: a row of this warp is in send descriptor e
  // (all bits when there are more than 32 descriptors).  In a register:
  // 2.328 vs 2.341 us per F iteration without the mask; read from shared
  // memory in the loop instead (fewer spills) it ran 2.369.  One-slot
  // variants only: the two-slot register variant would spill (0 -> 28 B)
  constexpr bool kSendMask = SPCG_PIPE_SENDMASK && NS == 1;
  uint32_t smask = 0xffffffffu;
  if (kSendMask && P.nsend <= 32) {
    smask = 0;
    for (int e = 0; e < P.nsend; ++e) {
      const ClusSend sd = e < kClusSendCache ? cs.send[e] : A.sends[P.send0 + e];
      bool in = false;
#pragma unroll
      for (int k = 0; k < NS; ++k) in = in || (rrow[k] >= sd.lo && rrow[k] < sd.hi);
      if (__ballot_sync(0xffffffffu, in)) smask |= 1u << e;
    }
  }
  // boundary n to the neighbours of this iteration: st.async into the cluster
  // neighbours' nhalo[buf] (completing on their mbB[buf]), epoch-tagged global
  // words for other clusters' CTAs
  auto send_one = [&](const double* nv, int buf, uint32_t tag, int e) {
    const ClusSend sd = e < kClusSendCache ? cs.send[e] : A.sends[P.send0 + e];
    if (sd.dst / C != kc) {
      unsigned long long* dst = gh + ((size_t)buf * G + sd.dst) * A.hcap * 2;
#pragma unroll
      for (int k = 0; k < NS; ++k)
        if (rrow[k] >= sd.lo && rrow[k] < sd.hi)
          tagged_store(dst + 2 * (size_t)(sd.dst_off + rrow[k] - sd.lo), nv[k], tag);
    } else {
      const uint32_t r = (uint32_t)(sd.dst % C);
      const uint32_t base = mapa_u32(nhalo + (size_t)buf * A.hcap, r);
      const uint32_t bar = mapa_u32(&cs.mbB[buf], r);
#pragma unroll
      for (int k = 0; k < NS; ++k)
        if (rrow[k] >= sd.lo && rrow[k] < sd.hi)
          st_async_f64(base + 8u * (uint32_t)(sd.dst_off + rrow[k] - sd.lo), nv[k], bar);
    }
  };
  auto send_n = [&](const double* nv, int buf, uint32_t tag) {
    if constexpr (kSendMask) {
      // only the descriptors some row of this warp belongs to (warp-uniform)
      for (uint32_t msk = smask; msk; msk &= msk - 1) send_one(nv, buf, tag, __ffs(msk) - 1);
    } else {
      for (int e = 0; e < P.nsend; ++e) send_one(nv, buf, tag, e);
    }
  };

  // ||b||.  Without x0, r0 = b: ||b||^2 is gamma0 bit for bit (the same
  // fmas, the same fixed-order all-reduce), and w0 is computed before it
  // (three blocking all-reduces fewer in the prologue than x0 given)
  double part = 0.0, dummy = 0.0;
  const bool zero_x0 = A.x0 == nullptr;
#pragma unroll
  for (int k = 0; k < NS; ++k)
    if (rrow[k] >= 0) {
      const double bv = A.b[rrow[k]];
      part = fma(bv, bv, part);
      if (zero_x0) rg[k] = bv;
    }
  // x0 = 0: r0's window is b's, read straight from b, so w0 = A r0 needs no
  // barrier first; its window goes out through scratch2 before this
  // all-reduce, which is then also the barrier before w0's window reads
  if (zero_x0) {
    for (int j = tid; j < P.wn; j += TH) wwin[j] = A.b[P.wlo + j];
    for (int h = tid; h < A.hcap; h += TH) zhalo[h] = 0.0;
    __syncthreads();
    spmv(wg);  // w0 = A r0
#pragma unroll
    for (int k = 0; k < NS; ++k)
      if (rrow[k] >= 0) A.scratch2[rrow[k]] = wg[k];
  }
  allreduce2(part, dummy);
  const double b_norm = sqrt(part);
  const double bb = part;
  if (b_norm == 0.0) {  // solver.py:109-118
#pragma unroll
    for (int k = 0; k < NS; ++k)
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
    for (int j = tid; j < P.wn; j += TH) wwin[j] = A.x0[P.wlo + j];
    __syncthreads();
    double qv[NS];
    spmv(qv);
#pragma unroll
    for (int k = 0; k < NS; ++k)
      if (rrow[k] >= 0) {
        xr[k] = A.x0[rrow[k]];
        rg[k] = mul_add_rn(A.b[rrow[k]], -1.0, qv[k]);
      }
    __syncthreads();
  }
  // window of r0 (through global scratch, once), gamma0
  double gam = bb;
  if (!zero_x0) {
    part = 0.0;
    dummy = 0.0;
#pragma unroll
    for (int k = 0; k < NS; ++k)
      if (rrow[k] >= 0) {
        A.scratch[rrow[k]] = rg[k];
        part = fma(rg[k], rg[k], part);
      }
    allreduce2(part, dummy);
    gam = part;
  }
  const double tol_b = A.tol * b_norm;
  // the largest g with sqrt(g) <= tol_b (sqrt is monotone: that set is [0, gthr])
  double gthr = tol_b * tol_b;
  for (int i = 0; i < 64 && gthr > 0.0 && sqrt(gthr) > tol_b; ++i) gthr = nextafter(gthr, 0.0);
  for (int i = 0; i < 64 && sqrt(nextafter(gthr, HUGE_VAL)) <= tol_b; ++i) gthr = nextafter(gthr, HUGE_VAL);
  long long max_it = A.max_iter;
  double rel = sqrt(gam) / b_norm;
  double g_rel = gam;  // r.r of the last relative residual (rel, computed after the loop)
  auto hist_w = [&](long long i, double g) {
    if (A.record_history && leader) A.hist[i - 1] = sqrt(g) / b_norm;
  };
  int converged = 0, status = ST_OK;
  long long iterations = 0, fail_iter = 0;
  if (sqrt(gam) <= tol_b) {
    converged = 1;
    max_it = 0;
  } else {
    if (!zero_x0) {
      for (int j = tid; j < P.wn; j += TH) wwin[j] = __ldcg(A.scratch + P.wlo + j);
      for (int h = tid; h < A.hcap; h += TH) zhalo[h] = 0.0;
      __syncthreads();
      spmv(wg);  // w0 = A r0
      // the window of w0 through a second scratch vector: no barrier for the
      // other CTAs' reads of r0's window first
#pragma unroll
      for (int k = 0; k < NS; ++k)
        if (rrow[k] >= 0) A.scratch2[rrow[k]] = wg[k];
      part = dummy = 0.0;
      allreduce2(part, dummy);  // (a barrier: every CTA sees the whole w0)
    }
    for (int j = tid; j < P.wn; j += TH) wwin[j] = __ldcg(A.scratch2 + P.wlo + j);
    __syncthreads();
  }

  // per-phase trace (A.trace set: SPCG_TRACE / SPCG_CLUS_DEBUG): thread 0 of
  // every CTA accumulates [iteration start + SpMV, -, sends + wait for the
  // totals, scalars + update + halo rows + barrier] ns, then records its SM
  // id and start / end times; the leader thread always (SolveReport.timings),
  // every CTA when tracing
  const bool tr = tid == 0 && (A.trace != nullptr || (SPCG_PHASE_TIMERS && gme == 0));
  // (SPCG_XCHG_TRACE) thread 0's timeline of iterations 100-107: [start,
  // SpMV done, sends done, totals in, partials posted, halo rows + barrier]
  unsigned long long* const tl_base =
      (SPCG_XCHG_TRACE && A.trace && tid == 0)
          ? A.trace + 8 * (size_t)G + (size_t)max(K * 8 * 34, 16 * G) + (size_t)gme * 8 * 6
          : nullptr;
  long long tl_it = -1;
#define SPCG_TL(j)                                                              \
  if (SPCG_XCHG_TRACE && tl_base && tl_it >= 100 && tl_it < 108)                \
    tl_base[(tl_it - 100) * 6 + (j)] = globaltimer_ns();
  unsigned long long tph[4] = {0, 0, 0, 0};
  // SPCG_PIPE_FINE (SM cycles), thread 0: [iteration start, -, SpMV, send n,
  // wait mbB, scalars, own-row update + partials, halo rows + sync]; the leader
  // CTA's comm warp: [12] iteration start -> partials in, [13] sum + exchange
  unsigned long long* tfine = cs.fine;  // (shared: no registers in the loop)
  unsigned long long tfl = 0;
  if (SPCG_PIPE_FINE) {
    if (tid < 16) cs.fine[tid] = 0;
    __syncthreads();
  }
#define SPCG_FT(j)                                          \
  if (SPCG_PIPE_FINE && tr) {                               \
    const unsigned long long tn_ = clock64();               \
    tfine[j] += tn_ - tfl;                                  \
    tfl = tn_;                                              \
  }
  const unsigned long long tkern0 = tr ? globaltimer_ns() : 0;
  double alpha = 0.0, beta = 0.0;
  // in-loop messages (no cluster barrier): every row warp's partials go by
  // st.async to cluster rank 0 (wslot[it & 1], completing on its mbA); rank
  // 0's comm warp sums them in (CTA, warp) order, runs the leaders' exchange
  // (K > 1) and st.asyncs the totals to every CTA's ltot (completing on mbB),
  // where the boundary n of the cluster neighbours (st.async into nhalo) land
  // too.  A CTA waits only for its own mbB: no CTA waits for the slowest of
  // the cluster.  The partials of iteration i+1 leave right after the own
  // rows' update of i, before the halo rows, so the reduction starts ~0.4 us
  // earlier.  Reuse distances (causality, not timing): partials by parity (a
  // CTA posts those of i+2 after the totals of i+1, i.e. after rank 0 read
  // i's); totals and halo n (nhalo, mbB, ghalo) by iteration mod 3 (the sends
  // of i+3 need the totals of i+2, i.e. every CTA's partials of i+2, posted
  // after that CTA's reads of i's halo rows).
  const uint32_t bA0 = mapa_u32(&cs.mbA[0], 0), bA1 = mapa_u32(&cs.mbA[1], 0);
  const uint32_t wsl0 = mapa_u32(&cs.wslot[0][me][wp][0], 0);
  const uint32_t wsl1 = mapa_u32(&cs.wslot[1][me][wp][0], 0);
  auto post_msg = [&](int pb) {  // row warps: this warp's (r.r, w.r) -> rank 0
    double g = 0.0, d = 0.0;
#pragma unroll
    for (int k = 0; k < NS; ++k)
      if (rrow[k] >= 0) {
        g = fma(rg[k], rg[k], g);
        d += rg[k] * wg[k];
      }
    g = warp_sum(g);
    d = warp_sum(d);
    if (lane == 0) st_async_v2f64(pb ? wsl1 : wsl0, g, d, pb ? bA1 : bA0);
  };
  if (!comm && max_it > 0) post_msg(0);
  int h3 = 0;  // iteration mod 3
  for (long long it = 0; max_it > 0; ++it, h3 = h3 == 2 ? 0 : h3 + 1) {
    const int bank = (int)(epoch++ & 1u), pb = (int)(it & 1);
    const uint32_t tag = epoch;
    const uint32_t parA = (uint32_t)(it >> 1) & 1u;  // mbA[pb]'s phase parity
    const uint32_t parB = (uint32_t)(it / 3) & 1u;   // mbB[h3]'s
    const unsigned long long t0 = tr ? globaltimer_ns() : 0;
    if (SPCG_PIPE_FINE) tfl = clock64();
    cur_it = it;
    tl_it = it;
    SPCG_TL(0)
    if (tid == 0) mbar_arrive_expect_tx(&cs.mbB[h3], (uint32_t)bbytes);
    // reciprocals of the last step's scalars, off the critical path: the
    // scalar step after the wait is then one division deep
    const double inv_gam = 1.0 / gam, inv_alpha = 1.0 / alpha;
    asm volatile("" ::"d"(inv_gam), "d"(inv_alpha));  // computed here, before the waits
    if (comm) {
      if (me == 0) {
        if (lane == 0) mbar_arrive_expect_tx(&cs.mbA[pb], (uint32_t)(C * PRW_ * 16));
        const bool trc = SPCG_PIPE_FINE && A.trace && lane == 0;
        unsigned long long tc0 = trc ? clock64() : 0;
        mbar_wait_cluster(&cs.mbA[pb], parA);
        if (trc) {
          const unsigned long long tn = clock64();
          tfine[12] += tn - tc0;
          tc0 = tn;
        }
        // lane w: warp w's partials over the cluster's CTAs; then the warps in
        // a fixed tree (the same bits on every lane after the broadcast)
        double c0 = 0.0, c1 = 0.0;
        if (lane < PRW_)
          for (int c = 0; c < C; ++c) {
            c0 += cs.wslot[pb][c][lane][0];
            c1 += cs.wslot[pb][c][lane][1];
          }
        c0 = warp_sum(c0);  // (xor tree: the same bits on every lane)
        c1 = warp_sum(c1);
        if (K > 1) exchange_core(bank, tag, false, c0, c1);
        if (trc) {
          const unsigned long long tn = clock64();
          tfine[13] += tn - tc0;
        }
        if (lane < C) st_async_v2f64(mapa_u32(&cs.ltot[h3][0], lane), c0, c1, mapa_u32(&cs.mbB[h3], lane));
      }
    } else {
      SPCG_FT(0)
      SPCG_FT(1)
    }
    double ng[NS];
    spmv(ng);  // n = A w (the comm warp has no rows), overlapped with the all-reduce
    SPCG_FT(2)
    SPCG_TL(1)
    const unsigned long long t1 = tr ? globaltimer_ns() : 0;
    const unsigned long long t2 = t1;
    if (!comm) send_n(ng, h3, tag);
    SPCG_FT(3)
    SPCG_TL(2)
    mbar_wait_cluster(&cs.mbB[h3], parB);  // totals + the cluster neighbours' boundary n
    SPCG_TL(3)
    // the first halo row of this thread, if another cluster owns it: its
    // tagged words are loaded now and consumed after the scalars, the update
    // and the partials' post (the L2 round trip off the path: 2.94 vs 3.12 us
    // per iteration on F against deferring the remote rows to the next
    // iteration's start)
    unsigned long long ea = 0, eb = 0;
    const bool e_act = !comm && tid < nh && !halo_local(tid);
    const unsigned long long* esrc = gh + (((size_t)h3 * G + gme) * A.hcap + (e_act ? tid : 0)) * 2;
    if (e_act) tagged_issue(esrc, ea, eb);
    SPCG_FT(4)
    const unsigned long long t3 = tr ? globaltimer_ns() : 0;
    if (tr) {
      tph[0] += t1 - t0;
      tph[1] += t2 - t1;
      tph[2] += t3 - t2;
    }
    const double g_new = cs.ltot[h3][0], d_new = cs.ltot[h3][1];
    if (it >= 1) {
      // one division deep: beta and eta from last step's reciprocals; the
      // convergence test sqrt(g) <= tol ||b|| as g <= gthr (the same set of
      // doubles); rel = sqrt(g) / ||b|| (history, report) off the path
      const double beta_n = g_new * inv_gam;
      const double eta = d_new - beta_n * g_new * inv_alpha;  // p.Ap of iteration it+1
      const double alpha_n = g_new / eta;
      g_rel = g_new;
      if (!isfinite(g_new)) {  // rel non-finite (||b|| > 0 finite)
        status = ST_NF_RES;
        fail_iter = it;
        break;
      }
      iterations = it;
      if (g_new <= gthr) {
        converged = 1;
        hist_w(it, g_new);
        break;
      }
      if (!isfinite(beta_n)) {
        status = ST_NF_BETA;
        fail_iter = it;
        hist_w(it, g_new);
        break;
      }
      if (it >= max_it) {
        hist_w(it, g_new);
        break;
      }
      if (eta <= 0.0) {
        status = ST_NOT_SPD;
        fail_iter = it + 1;
        hist_w(it, g_new);
        break;
      }
      if (!isfinite(alpha_n)) {
        status = ST_NF_ALPHA;
        fail_iter = it + 1;
        hist_w(it, g_new);
        break;
      }
      alpha = alpha_n;
      beta = beta_n;
    } else {
      if (d_new <= 0.0) {
        status = ST_NOT_SPD;
        fail_iter = 1;
        break;
      }
      alpha = g_new / d_new;
      if (!isfinite(alpha)) {
        status = ST_NF_ALPHA;
        fail_iter = 1;
        break;
      }
      beta = 0.0;
    }
    gam = g_new;
    // the CG coefficients of this step (Lanczos tridiagonal -> the host's
    // condition estimate of the auto-mode guard)
    if (leader && A.coef) {
      A.coef[2 * it] = alpha;
      A.coef[2 * it + 1] = beta;
    }
    const double na = -alpha;
    SPCG_FT(5)
    if (!comm) {
      // every row warp's SpMV has read the window of w before any warp writes
      // it (a warp with two slices is still reading when a one-slice warp
      // gets here; the cluster barrier of the barrier protocol did this)
      asm volatile("bar.sync 1, %0;" ::"r"(PRT_) : "memory");
#pragma unroll
      for (int k = 0; k < NS; ++k)
        if (rrow[k] >= 0) {
          zg[k] = mul_add_rn(ng[k], beta, zg[k]);
          sg[k] = mul_add_rn(wg[k], beta, sg[k]);
          pg[k] = mul_add_rn(rg[k], beta, pg[k]);
          xr[k] = mul_add_rn(xr[k], alpha, pg[k]);
          rg[k] = mul_add_rn(rg[k], na, sg[k]);
          wg[k] = mul_add_rn(wg[k], na, zg[k]);
          wwin[own0 + rrow[k] - P.row_lo] = wg[k];
        }
      post_msg(pb ^ 1);  // the partials of iteration it+1
      SPCG_TL(4)
      if (it >= 1) hist_w(it, g_new);
      SPCG_FT(6)
      for (int hb = tid - lane; hb < nh; hb += PRT_) {  // warp-uniform trip count
        const int h = hb + lane;
        const bool act = h < nh;
        const double nv = (e_act && h == tid) ? tagged_finish(esrc, ea, eb, tag)
                                                                 : halo_n(act, h3, h, tag);
        if (act) {
          const double zh = mul_add_rn(nv, beta, zhalo[h]);
          zhalo[h] = zh;
          const int j = halo_win(h);
          wwin[j] = mul_add_rn(wwin[j], na, zh);
        }
      }

      // the window of w is complete before the next SpMV (row warps only: the
      // comm warp never touches it)
      asm volatile("bar.sync 1, %0;" ::"r"(PRT_) : "memory");
    }
    SPCG_FT(7)
    SPCG_TL(5)
    if (tr) tph[3] += globaltimer_ns() - t3;
  }
  // every CTA leaves the loop at the same iteration (identical totals); the
  // barrier retires the loop's messages before the tail reuses shared memory
  cluster_sync_all();
  rel = sqrt(g_rel) / b_norm;
#undef SPCG_FT
#undef SPCG_TL
  if (tr && A.trace) {
    unsigned int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    for (int ph = 0; ph < 4; ++ph) A.trace[gme * 8 + ph] = tph[ph];
    A.trace[gme * 8 + 4] = smid;
    A.trace[gme * 8 + 5] = tkern0;
    A.trace[gme * 8 + 6] = globaltimer_ns();
    A.trace[gme * 8 + 7] = (unsigned long long)iterations;
    if (SPCG_PIPE_FINE)
      for (int j = 0; j < 12; ++j) A.trace[8 * (size_t)G + gme * 16 + j] = tfine[j];  // (tid 0's)
  }
  if (SPCG_PIPE_FINE && A.trace && comm && lane == 0 && me == 0)
    for (int j = 12; j < 14; ++j) A.trace[8 * (size_t)G + gme * 16 + j] = tfine[j];

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
  for (int k = 0; k < NS; ++k)
    if (rrow[k] >= 0) A.x[rrow[k]] = xr[k];
  const double rec_rel = rel;
  if (A.recompute) {  // true residual ||b - A x|| / ||b||
    part = 0.0;
    dummy = 0.0;
    allreduce2(part, dummy);
    for (int j = tid; j < P.wn; j += TH) wwin[j] = __ldcg(A.x + P.wlo + j);
    __syncthreads();
    double qv[NS];
    spmv(qv);
    part = 0.0;
#pragma unroll
    for (int k = 0; k < NS; ++k)
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
    A.res->rec_rel = rec_rel;
    A.res->phase_ns[0] = tph[0];            // SpMV
    A.res->phase_ns[1] = tph[1] + tph[2];   // sends + wait for the totals (exchange)
    A.res->phase_ns[2] = tph[3];            // scalars, update, partials, halo rows
  }
}

}  // namespace spcg
