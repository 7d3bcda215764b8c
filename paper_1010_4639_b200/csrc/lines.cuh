// lines.cuh — per-line SpMV bodies over a staged tile (one thread per line).
//
// The gathered vector is abstracted as a "source" (SrcPlain: x_j; the
// resident single-reduction engine's folded r-update: SrcCgcg in cg1.cuh).
// Row sums are formed sequentially in storage order with IEEE mul-then-add, so
// a CSR row equals _ckernels.csr_gather (_ckernels.pyx:42-47) bit for bit.
#pragma once
#include "tiles.cuh"

namespace spcg {

struct SrcPlain {
  const double* x;
  __device__ __forceinline__ double get(int j) const { return x[j]; }
};

#ifndef SPCG_UNROLL
#define SPCG_UNROLL 8
#endif
constexpr int kUnroll = SPCG_UNROLL;

// acc = sum_k v[k]*src(ix[k]) over [ks,ke), sequential order; loads batched
// kUnroll-deep so each thread keeps many gathers in flight.
template <class Src>
__device__ __forceinline__ double seq_row(const double* v, const int* ix, int ks, int ke,
                                          const Src& src) {
  double acc = 0.0;
  for (int k = ks; k < ke; k += kUnroll) {
    double pr[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      pr[u] = (k + u < ke) ? __dmul_rn(v[k + u], src.get(ix[k + u])) : 0.0;
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (k + u < ke) acc = __dadd_rn(acc, pr[u]);
  }
  return acc;
}

// Phase 1 of a CSR / SCSR_PRIV tile ("CSR-stream"): every thread forms
// products prod[k] = val[k] * src(idx[k]) for staged entries k = tid,
// tid+kBlock, ...  (kUnroll of them in flight), so all 512 threads gather
// regardless of row lengths; phase 2 sums each line's products sequentially
// in storage order (same bits as a sequential row sum).  prod may alias
// sm.val[s] (streamed tiles) or be a separate buffer (resident tiles).
template <class Src>
__device__ __forceinline__ void stream_products(const Smem& sm, int s, const Src& src,
                                                double* prod) {
  const int cnt = sm.meta[s].cnt;
  const double* v = sm.val[s];
  const int* ix = sm.idx[s];
  for (int k0 = threadIdx.x; k0 < cnt; k0 += kBlock * kUnroll) {
    double pr[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int k = k0 + u * kBlock;
      pr[u] = (k < cnt) ? __dmul_rn(v[k], src.get(ix[k])) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int k = k0 + u * kBlock;
      if (k < cnt) prod[k] = pr[u];
    }
  }
  __syncthreads();
}

__device__ __forceinline__ double seq_sum(const double* prod, int ks, int ke) {
  double acc = 0.0;
  for (int k = ks; k < ke; ++k) acc = __dadd_rn(acc, prod[k]);
  return acc;
}

// Symmetric L+D row i (diagonal last): g = sum_{j<=i} a_ij x_j, and the
// transpose contributions a_ij * x_i scattered into y_j (j<i) with fp64 red.
// Phase order matters: every gather of the round is issued before the first
// red (a red is an asm statement with a memory clobber, so no load can be
// hoisted above it, and each red waits for x_i -- the line's own, usually
// uncached, value).  Interleaving "gather u, red u" serialised the round's
// gathers behind that x_i load.
// FIX (K_SCSR_FIX): the transposed contributions go to the 64-bit
// fixed-point accumulator ytx, scaled by the power of two c (exact sums).
template <bool FIX = false, class Src>
__device__ __forceinline__ double sym_row_atomic(const double* v, const int* ix, int ks, int ke,
                                                 int i, double xi, const Src& src, double* y,
                                                 unsigned long long* ytx = nullptr,
                                                 double c = 0.0) {
  double acc = 0.0;
  for (int k = ks; k < ke; k += kUnroll) {
    int jj[kUnroll];
    double gx[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) jj[u] = (k + u < ke) ? ix[k + u] : i;
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) gx[u] = (k + u < ke) ? src.get(jj[u]) : 0.0;
    // one shared-memory read of each value serves its red and its product
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (k + u < ke) {
        const double a = v[k + u];
        if (jj[u] != i) {
          if (FIX) red_add_s64(ytx + jj[u], f64_to_s64_rn(__dmul_rn(a, xi) * c));
          else red_add_f64(y + jj[u], __dmul_rn(a, xi));
        }
        acc = __dadd_rn(acc, __dmul_rn(a, gx[u]));
      }
    }
  }
  return acc;
}

// CSC column j: y[row_k] += a_kj * xj (red), and (if GATHER) the transposed
// gather g = sum_k a_kj x_{row_k} that makes p.Ap = sum_j p_j g_j.  Gathers
// of a round go out before its reds (see sym_row_atomic).
template <bool GATHER, class Src>
__device__ __forceinline__ double csc_col(const double* v, const int* ix, int ks, int ke,
                                          double xj, const Src& src, double* y) {
  double acc = 0.0;
  for (int k = ks; k < ke; k += kUnroll) {
    int rr[kUnroll];
    double gx[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) rr[u] = (k + u < ke) ? ix[k + u] : 0;
    if (GATHER) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) gx[u] = (k + u < ke) ? src.get(rr[u]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (k + u < ke) {
        const double a = v[k + u];
        red_add_f64(y + rr[u], __dmul_rn(a, xj));
        if (GATHER) acc = __dadd_rn(acc, __dmul_rn(a, gx[u]));
      }
    }
  }
  return acc;
}

// ---- long lines: one line with > kTileNnz entries, read from global by the
// whole CTA.  Scatter formats (order unspecified anyway) use strided partial
// sums + a fixed-order block reduction (tile_line).
// Long line of a gather format, bitwise the reference's sequential row sum:
// chunk by chunk all threads form the products (coalesced loads, every
// gather in flight) into `prod` (>= kTileNnz doubles: the stage's unused
// value buffer), then thread 0 adds them in storage order.  The dependent
// add chain costs ~17 us per 4096 entries -- fine for the rare rows longer
// than a tile.  Result valid in thread 0.
template <class Src>
__device__ __forceinline__ double long_gather_seq(const double* val, const int* idx, int k0, int k1,
                                                  const Src& src, double* prod) {
  double acc = 0.0;
  for (int base = k0; base < k1; base += kTileNnz) {
    const int cnt = min(kTileNnz, k1 - base);
    for (int e = (int)threadIdx.x; e < cnt; e += blockDim.x)
      prod[e] = __dmul_rn(ld_stream_f64(val + base + e), src.get(ld_stream_s32(idx + base + e)));
    __syncthreads();
    if (threadIdx.x == 0)
      for (int e = 0; e < cnt; ++e) acc = __dadd_rn(acc, prod[e]);
    __syncthreads();  // prod is rewritten by the next chunk
  }
  return acc;
}

// Result of one line of a tile pass: the line's output value and the line's
// p.Ap contribution pieces (only meaningful where the caller needs them).
struct LineOut {
  double q;    // (A x)_i for CSR / SCSR_PRIV; g_i for SCSR_ATOMIC / CSC
  double xi;   // src(i): the gathered-vector value of the line itself
  double dg;   // SCSR_ATOMIC: diagonal a_ii
  double xo;   // xpre[i] prefetched with the line's loads (CG x update)
};

// Tiles averaging more than this many entries per line use the two-phase
// CSR-stream body; shorter rows (e.g. the 7-point stencil) keep one thread
// per row, which already has all of its gathers in flight.
#ifndef SPCG_STREAM_MIN
#define SPCG_STREAM_MIN 8
#endif
constexpr int kStreamMinPerLine = SPCG_STREAM_MIN;

// A line of a short tile gets 2^lg adjacent lanes when the tile has at most
// kBlock/2 (kBlock/4) lines (long-row matrices: see tile_line_cap).
// Gather formats (CSR, SCSR privatized) split only in the streaming passes:
// in the latency-bound resident kernels the shuffle chain costs more than
// the idle lanes (S: 8.6 vs 9.5 us per iteration).
template <int FMT, bool STREAMING>
__device__ __forceinline__ int split_lg(const StageMeta& mt) {
  if (!STREAMING && (FMT == K_CSR || FMT == K_SCSR_PRIV)) return 0;
  const int rows = mt.row1 - mt.row0;
  return (rows * 4 <= kBlock) ? 2 : (rows * 2 <= kBlock ? 1 : 0);
}

// Sequential (storage-order) sum of one line segment [ks, ke) of a staged
// tile, computed by the line's 2^lg adjacent lanes: lane g gathers entries
// u = g, g + T, g + 2T, ... (up to 8 per round, so each lane keeps 8 gathers
// in flight) and every lane of the group then adds all products in entry
// order, taking them by shuffles.  Bitwise the reference's row sum, with no
// product round trip through shared memory.  Warp-uniform: all 32 lanes
// call it (lanes without a line pass ks == ke).
template <class Src>
__device__ __forceinline__ double lane_seq_sum(const double* v, const int* ix, int ks, int ke,
                                               int lg, const Src& src) {
  const int T = 1 << lg;
  const int lane = (int)threadIdx.x & 31;
  const int g = lane & (T - 1), owner = lane & ~(T - 1);
  const int L = ke - ks;
  const int Lmax = __reduce_max_sync(0xffffffffu, L);
  double acc = 0.0;
  for (int base = 0; base < Lmax; base += 8 * T) {
    double p[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int u = base + t * T + g;
      p[t] = (u < L) ? __dmul_rn(v[ks + u], src.get(ix[ks + u])) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < 8; ++t)
#pragma unroll
      for (int gg = 0; gg < 4; ++gg)
        if (gg < T) {
          const double q = __shfl_sync(0xffffffffu, p[t], owner + gg);
          if (base + t * T + gg < L) acc = __dadd_rn(acc, q);
        }
  }
  return acc;
}

// The line this thread reports for staged tile mt (-1: none); matches
// tile_line's `active` / `line` outputs.
template <int FMT>
__device__ __forceinline__ int owned_line(const StageMeta& mt) {
  if (mt.is_long) return threadIdx.x == 0 ? mt.row0 : -1;
  const int lg = split_lg<FMT, false>(mt);  // resident kernels
  if ((int)threadIdx.x & ((1 << lg) - 1)) return -1;
  const int i = mt.row0 + ((int)threadIdx.x >> lg);
  return i < mt.row1 ? i : -1;
}

// Reassociated (but deterministic) variant for the CG passes: lane g sums
// its entries u = g, g+T, ... in order, then the partials combine by a fixed
// shuffle tree ((s0+s1)+(s2+s3)); valid in the group's first lane.  No
// per-product shuffles: the long-row bodies run at streaming speed.
template <class Src>
__device__ __forceinline__ double lane_tree_sum(const double* v, const int* ix, int ks, int ke,
                                                int lg, const Src& src) {
  const int T = 1 << lg;
  const int g = (int)threadIdx.x & (T - 1);
  const int L = ke - ks;
  double acc = 0.0;
  for (int base = 0; base < L; base += 8 * T) {
    double p[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int u = base + t * T + g;
      p[t] = (u < L) ? __dmul_rn(v[ks + u], src.get(ix[ks + u])) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < 8; ++t)
      if (base + t * T + g < L) acc = __dadd_rn(acc, p[t]);
  }
  if (lg >= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, 1));
  if (lg == 2) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, 2));
  return acc;
}

// Both segments of a privatized SCSR line in the same rounds (the gathers
// of L+D and L^T in flight together), each reduced by its own fixed tree.
template <class Src>
__device__ __forceinline__ double lane_tree_sum2(const double* v, const int* ix, int ka, int kae,
                                                 int kb, int kbe, int lg, const Src& src) {
  const int T = 1 << lg;
  const int g = (int)threadIdx.x & (T - 1);
  const int LA = kae - ka, LB = kbe - kb;
  const int L = max(LA, LB);
  double acc = 0.0, acc2 = 0.0;
  for (int base = 0; base < L; base += 4 * T) {
    double p[4], q[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int u = base + t * T + g;
      p[t] = (u < LA) ? __dmul_rn(v[ka + u], src.get(ix[ka + u])) : 0.0;
      q[t] = (u < LB) ? __dmul_rn(v[kb + u], src.get(ix[kb + u])) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int u = base + t * T + g;
      if (u < LA) acc = __dadd_rn(acc, p[t]);
      if (u < LB) acc2 = __dadd_rn(acc2, q[t]);
    }
  }
  if (lg >= 1) {
    acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, 1));
    acc2 = __dadd_rn(acc2, __shfl_down_sync(0xffffffffu, acc2, 1));
  }
  if (lg == 2) {
    acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, 2));
    acc2 = __dadd_rn(acc2, __shfl_down_sync(0xffffffffu, acc2, 2));
  }
  return __dadd_rn(acc, acc2);
}

// Two segments (SCSR privatized: L+D then L^T) in the same rounds, so the
// gathers of both are in flight together; sums kept separate (g, t).
template <class Src>
__device__ __forceinline__ void lane_seq_sum2(const double* v, const int* ix, int ka, int kae,
                                              int kb, int kbe, int lg, const Src& src,
                                              double& ga, double& gb) {
  const int T = 1 << lg;
  const int lane = (int)threadIdx.x & 31;
  const int g = lane & (T - 1), owner = lane & ~(T - 1);
  const int LA = kae - ka, LB = kbe - kb;
  const int Lmax = __reduce_max_sync(0xffffffffu, max(LA, LB));
  double acc = 0.0, acc2 = 0.0;
  for (int base = 0; base < Lmax; base += 4 * T) {
    double p[4], q[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int u = base + t * T + g;
      p[t] = (u < LA) ? __dmul_rn(v[ka + u], src.get(ix[ka + u])) : 0.0;
      q[t] = (u < LB) ? __dmul_rn(v[kb + u], src.get(ix[kb + u])) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int gg = 0; gg < 4; ++gg)
        if (gg < T) {
          const int u = base + t * T + gg;
          const double a = __shfl_sync(0xffffffffu, p[t], owner + gg);
          const double b = __shfl_sync(0xffffffffu, q[t], owner + gg);
          if (u < LA) acc = __dadd_rn(acc, a);
          if (u < LB) acc2 = __dadd_rn(acc2, b);
        }
  }
  ga = acc;
  gb = acc2;
}

// Computes line i (the tid-th line of staged tile s).  For FMT in
// {SCSR_ATOMIC, CSC} the scatter goes to y (must be zeroed beforehand) and
// the line's own gather is returned in q; for CSR / SCSR_PRIV the caller
// stores q.  `active` = this thread owns a line.  Long tiles: every thread
// must call (CTA-wide reductions); the line's result is valid in thread 0.
template <int FMT, bool GATHER_CSC, class Src, bool ALLOW_STREAM = true>
__device__ __forceinline__ LineOut tile_line(Smem& sm, int s, const MatView& M, const Src& src,
                                             double* y, bool& active, int& line, double* prod,
                                             const double* xpre = nullptr) {
  const StageMeta& mt = sm.meta[s];
  LineOut o{0.0, 0.0, 0.0, 0.0};
  if (!mt.is_long) {
    const int i = mt.row0 + (int)threadIdx.x;
    active = i < mt.row1;
    line = i;
#ifndef SPCG_NO_XPRE
#define SPCG_NO_XPRE 0
#endif
    if (SPCG_NO_XPRE) xpre = nullptr;
    if (FMT == K_SCSR_ATOMIC || FMT == K_SCSR_FIX || FMT == K_CSC) {
      // split lines: tiles of <= 256 (128) lines give each line 2 (4)
      // adjacent lanes (512-line tiles: one lane per line); lane g takes the g-th contiguous segment of the
      // line's entries (gather partial + its scatters), and the partials
      // combine in fixed order (s0+s1)+(s2+s3), so the gather half stays
      // deterministic.  Warp-uniform: every lane reaches the shuffles.
      const int lg = split_lg<FMT, ALLOW_STREAM>(mt);
      {
        const int tpl = 1 << lg;
        const int g = (int)threadIdx.x & (tpl - 1);
        const int li = mt.row0 + ((int)threadIdx.x >> lg);
        const bool has = li < mt.row1;
        double acc = 0.0;
        if (has) {
          const int l = li - mt.r0a;
          const int a0 = sm.rpA[s][l] - mt.kA0a;
          const int a1 = sm.rpA[s][l + 1] - mt.kA0a;
          const int c = (a1 - a0 + tpl - 1) >> lg;
          const int ks = min(a1, a0 + g * c);
          const int ke = min(a1, ks + c);
          o.xi = src.get(li);
          if (xpre) o.xo = xpre[li];
          if (FMT == K_SCSR_ATOMIC) {
            acc = sym_row_atomic(sm.val[s], sm.idx[s], ks, ke, li, o.xi, src, y);
            o.dg = (a1 > a0) ? sm.val[s][a1 - 1] : 0.0;
          } else if (FMT == K_SCSR_FIX) {
            acc = sym_row_atomic<true>(sm.val[s], sm.idx[s], ks, ke, li, o.xi, src, y, M.ytx,
                                       fix_scale(M.txmax, M.tx_eM));
            o.dg = (a1 > a0) ? sm.val[s][a1 - 1] : 0.0;
          } else {
            acc = csc_col<GATHER_CSC>(sm.val[s], sm.idx[s], ks, ke, o.xi, src, y);
          }
        }
        double t = acc;
        if (lg >= 1) t = __dadd_rn(t, __shfl_down_sync(0xffffffffu, t, 1));
        if (lg == 2) t = __dadd_rn(t, __shfl_down_sync(0xffffffffu, t, 2));
        o.q = t;
        active = has && g == 0;
        line = li;
        return o;
      }
    }
    if (FMT == K_CSR || FMT == K_SCSR_PRIV) {
      // long-row tiles capped at <= 256 (128) lines: split lines, every
      // lane of the group gets the line's sequential sum(s)
      const int lg = split_lg<FMT, ALLOW_STREAM>(mt);
      if (lg > 0) {
        const int g = (int)threadIdx.x & ((1 << lg) - 1);
        const int li = mt.row0 + ((int)threadIdx.x >> lg);
        const bool has = li < mt.row1;
        int ks = 0, ke = 0, kb = 0, kbe = 0;
        if (has) {
          const int l = li - mt.r0a;
          ks = sm.rpA[s][l] - mt.kA0a;
          ke = sm.rpA[s][l + 1] - mt.kA0a;
          if (FMT == K_SCSR_PRIV) {
            kb = sm.rpB[s][l] - mt.kB0a + mt.offB;
            kbe = sm.rpB[s][l + 1] - mt.kB0a + mt.offB;
          }
          if (g == 0) {
            o.xi = src.get(li);
            if (xpre) o.xo = xpre[li];
          }
        }
        if (M.tree) {  // warp-uniform
          o.q = FMT == K_SCSR_PRIV
                    ? lane_tree_sum2(sm.val[s], sm.idx[s], ks, ke, kb, kbe, lg, src)
                    : lane_tree_sum(sm.val[s], sm.idx[s], ks, ke, lg, src);
        } else if (FMT == K_SCSR_PRIV) {
          double ga, gb;
          lane_seq_sum2(sm.val[s], sm.idx[s], ks, ke, kb, kbe, lg, src, ga, gb);
          o.q = __dadd_rn(ga, gb);
        } else {
          o.q = lane_seq_sum(sm.val[s], sm.idx[s], ks, ke, lg, src);
        }
        active = has && g == 0;
        line = li;
        return o;
      }
    }
    const bool stream = ALLOW_STREAM && (FMT == K_CSR || FMT == K_SCSR_PRIV) &&
                        mt.cnt > kStreamMinPerLine * (mt.row1 - mt.row0);
    const double* v = sm.val[s];
    const int* ix = sm.idx[s];
    const int lr = i - mt.r0a;
    if (stream) {
      if (active) {  // own-line loads go out before the gather phase
        o.xi = src.get(i);
        if (xpre) o.xo = xpre[i];
      }
      stream_products(sm, s, src, prod);
      if (!active) return o;
      const int ks = sm.rpA[s][lr] - mt.kA0a;
      const int ke = sm.rpA[s][lr + 1] - mt.kA0a;
      if (FMT == K_CSR) {
        o.q = seq_sum(prod, ks, ke);
      } else {
        const int kb = sm.rpB[s][lr] - mt.kB0a + mt.offB;
        const int kbe = sm.rpB[s][lr + 1] - mt.kB0a + mt.offB;
        o.q = __dadd_rn(seq_sum(prod, ks, ke), seq_sum(prod, kb, kbe));
      }
      return o;
    }
    if (!active) return o;
    if (xpre) o.xo = xpre[i];
    const int ks = sm.rpA[s][lr] - mt.kA0a;
    const int ke = sm.rpA[s][lr + 1] - mt.kA0a;
    if (FMT == K_CSR) {
      o.q = seq_row(v, ix, ks, ke, src);
      o.xi = src.get(i);
    } else if (FMT == K_SCSR_PRIV) {
      const int kb = sm.rpB[s][lr] - mt.kB0a + mt.offB;
      const int kbe = sm.rpB[s][lr + 1] - mt.kB0a + mt.offB;
      const double g = seq_row(v, ix, ks, ke, src);
      const double t = seq_row(v, ix, kb, kbe, src);
      o.q = __dadd_rn(g, t);
      o.xi = src.get(i);
    } else if (FMT == K_SCSR_ATOMIC) {
      o.xi = src.get(i);
      o.q = sym_row_atomic(v, ix, ks, ke, i, o.xi, src, y);
      o.dg = (ke > ks) ? v[ke - 1] : 0.0;
    } else if (FMT == K_SCSR_FIX) {
      o.xi = src.get(i);
      o.q = sym_row_atomic<true>(v, ix, ks, ke, i, o.xi, src, y, M.ytx, fix_scale(M.txmax, M.tx_eM));
      o.dg = (ke > ks) ? v[ke - 1] : 0.0;
    } else {  // K_CSC
      o.xi = src.get(i);
      o.q = csc_col<GATHER_CSC>(v, ix, ks, ke, o.xi, src, y);
    }
    return o;
  }
  // long tile: one line, entries from global memory
  const int i = mt.row0;
  line = i;
  active = threadIdx.x == 0;
  if (xpre) o.xo = xpre[i];
  const int k0 = M.ptrA[i], k1 = M.ptrA[i + 1];
  if (FMT == K_CSR) {
    o.q = long_gather_seq(M.valA, M.idxA, k0, k1, src, prod);
    o.xi = src.get(i);
  } else if (FMT == K_SCSR_PRIV) {
    const double g = long_gather_seq(M.valA, M.idxA, k0, k1, src, prod);
    const double t = long_gather_seq(M.valB, M.idxB, M.ptrB[i], M.ptrB[i + 1], src, prod);
    o.q = __dadd_rn(g, t);
    o.xi = src.get(i);
  } else if (FMT == K_SCSR_ATOMIC || FMT == K_SCSR_FIX) {
    const double xi = src.get(i);
    const double c = FMT == K_SCSR_FIX ? fix_scale(M.txmax, M.tx_eM) : 0.0;
    double part = 0.0;
    for (int k = k0 + (int)threadIdx.x; k < k1; k += blockDim.x) {
      const int j = ld_stream_s32(M.idxA + k);
      const double a = ld_stream_f64(M.valA + k);
      part = __dadd_rn(part, __dmul_rn(a, src.get(j)));
      if (j != i) {
        if (FMT == K_SCSR_FIX) red_add_s64(M.ytx + j, f64_to_s64_rn(__dmul_rn(a, xi) * c));
        else red_add_f64(y + j, __dmul_rn(a, xi));
      }
    }
    o.q = block_sum(part, sm);
    o.xi = xi;
    o.dg = (k1 > k0) ? M.valA[k1 - 1] : 0.0;
  } else {
    const double xj = src.get(i);
    double part = 0.0;
    for (int k = k0 + (int)threadIdx.x; k < k1; k += blockDim.x) {
      const int row = ld_stream_s32(M.idxA + k);
      const double a = ld_stream_f64(M.valA + k);
      red_add_f64(y + row, __dmul_rn(a, xj));
      if (GATHER_CSC) part = __dadd_rn(part, __dmul_rn(a, src.get(row)));
    }
    o.q = GATHER_CSC ? block_sum(part, sm) : 0.0;
    o.xi = xj;
  }
  return o;
}

// Wide CSR tile (more than kBlock lines, thread-per-row rows): thread t
// computes lines row0 + t and row0 + t + kBlock with both lines' gathers in
// flight together; each line is summed sequentially in storage order
// (bitwise csr_gather).  Warp-uniform control flow.
template <class Src>
__device__ __forceinline__ void csr_line_pair(const Smem& sm, int s, const Src& src,
                                              LineOut (&o)[2], bool (&act)[2], int (&li)[2],
                                              const double* xpre) {
  const StageMeta& mt = sm.meta[s];
  const double* v = sm.val[s];
  const int* ix = sm.idx[s];
  int ks[2], len[2];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    li[t] = mt.row0 + (int)threadIdx.x + t * kBlock;
    act[t] = li[t] < mt.row1;
    o[t] = LineOut{0.0, 0.0, 0.0, 0.0};
    ks[t] = 0;
    len[t] = 0;
    if (act[t]) {
      const int lr = li[t] - mt.r0a;
      ks[t] = sm.rpA[s][lr] - mt.kA0a;
      len[t] = sm.rpA[s][lr + 1] - mt.kA0a - ks[t];
      o[t].xi = src.get(li[t]);
      if (xpre) o[t].xo = xpre[li[t]];
    }
  }
  constexpr int U = 8;
  double acc0 = 0.0, acc1 = 0.0;
  const int L = max(len[0], len[1]);
  for (int base = 0; base < L; base += U) {
    double p0[U], p1[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      p0[u] = (base + u < len[0]) ? __dmul_rn(v[ks[0] + base + u], src.get(ix[ks[0] + base + u])) : 0.0;
      p1[u] = (base + u < len[1]) ? __dmul_rn(v[ks[1] + base + u], src.get(ix[ks[1] + base + u])) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (base + u < len[0]) acc0 = __dadd_rn(acc0, p0[u]);
      if (base + u < len[1]) acc1 = __dadd_rn(acc1, p1[u]);
    }
  }
  o[0].q = acc0;
  o[1].q = acc1;
}

// True when staged tile s is a wide CSR tile (handled by csr_line_pair).
template <int FMT>
__device__ __forceinline__ bool wide_tile(const Smem& sm, int s) {
  return FMT == K_CSR && !sm.meta[s].is_long && sm.meta[s].row1 - sm.meta[s].row0 > kBlock;
}

// Finish a line of a plain SpMV y = A x (no CG bookkeeping).
template <int FMT>
__device__ __forceinline__ void finish_plain(const LineOut& o, int i, double* y) {
  if (FMT == K_CSR || FMT == K_SCSR_PRIV || FMT == K_SCSR_FIX) y[i] = o.q;  // FIX: the gather part
  else if (FMT == K_SCSR_ATOMIC) red_add_f64(y + i, o.q);
  // CSC: the column scatter already wrote everything
}

// p.Ap contribution of a line (p_i = o.xi):
//   CSR / SCSR_PRIV: p_i q_i;  SCSR_ATOMIC: p_i (2 g_i - a_ii p_i)
//   (p'Ap = 2 p'(L+D)p - p'Dp);  CSC: p_j g_j  (p'A p = p'A^T p).
template <int FMT>
__device__ __forceinline__ double line_pq(const LineOut& o) {
  if (FMT == K_SCSR_ATOMIC || FMT == K_SCSR_FIX) return o.xi * (2.0 * o.q - o.dg * o.xi);
  return o.xi * o.q;
}

}  // namespace spcg
