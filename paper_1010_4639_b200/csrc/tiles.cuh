// tiles.cuh — row-tile staging of CSR/SCSR/CSC arrays into shared memory.
//
// HBM layout (built by matrix.cu at upload):
//   ptr  int32[n+1 (+8 pad)]   idx int32[nnz (+8 pad)]   val f64[nnz (+8 pad)]
//   every array 256-byte aligned; pads are zero so 16-byte-rounded bulk copies
//   never read past an allocation.
//   tdesc int4[ntiles] = {row0, row1, k0, k1}: lines [row0,row1) hold stored
//   entries [k0,k1); a tile has <= kTileLines lines and <= kTileNnz entries,
//   except a "long" tile = one line with more entries than kTileNnz.
//   For the privatized symmetric mode a second segment (CSR of L^T) rides in
//   the same tile: tdescB int2[ntiles] = {k0B, k1B}.
//
// One tile = one stage of the shared-memory ring: its row-pointer slice, index
// slice and value slice arrive by 1-D bulk async copies (cp.async.bulk,
// completion on an mbarrier), issued by thread 0 one or more tiles ahead of the
// consumer, so HBM streaming overlaps the x-gathers and the grid barriers.
#pragma once
#include "ptx.cuh"

namespace spcg {

// SPCG_TRACE=1 builds per-phase timing into the CG kernels (dev builds only:
// even runtime-disabled, the hooks cost registers in the hot loops).
#ifndef SPCG_TRACE
#define SPCG_TRACE 0
#endif
#ifndef SPCG_BLOCK
#define SPCG_BLOCK 512
#endif
#ifndef SPCG_TILE_NNZ
#define SPCG_TILE_NNZ 4096
#endif
constexpr int kBlock = SPCG_BLOCK;     // threads per CTA == lines per tile
constexpr int kTileLines = kBlock;
constexpr int kTileNnz = SPCG_TILE_NNZ;  // stored entries per tile (both segments)
#ifndef SPCG_STAGES
#define SPCG_STAGES 2
#endif
constexpr int kStages = SPCG_STAGES;  // TMA ring depth (tiles in flight + 1)
#ifndef SPCG_STREAM_MINB
#define SPCG_STREAM_MINB (1024 / SPCG_BLOCK)
#endif
constexpr int kStreamMinBlocks = SPCG_STREAM_MINB;  // CTAs/SM targeted by streaming kernels
constexpr int kRpCap = kTileLines + 8;
// Streaming passes over short-row CSR matrices use "wide" tiles of up to
// kWideLines lines (two per thread), so a stage carries up to kTileNnz
// entries instead of 512 x (row length): more bytes in flight per SM
// (P2's 5-entry rows filled only 2,560 of a stage's 4,096 entries).
#ifndef SPCG_WIDE
#define SPCG_WIDE 2
#endif
constexpr int kWideLines = SPCG_WIDE * kBlock;
constexpr int kRpCapA = kWideLines + 8;
constexpr int kNzCap = kTileNnz + 16;

// Kernel-level storage variants.
// K_SCSR_FIX: the single pass over L+D of K_SCSR_ATOMIC, with the transposed
// contributions accumulated EXACTLY in 64-bit fixed point (integer reds are
// order-independent): the deterministic symmetric SpMV of the per-pass CG
// engine without a stored L^T (dist.cuh).
enum KFmt : int { K_CSR = 0, K_SCSR_ATOMIC = 1, K_SCSR_PRIV = 2, K_CSC = 3, K_SCSR_FIX = 4 };

struct MatView {
  int n;
  int ntiles;
  const int4* tdesc;     // {row0,row1,k0,k1}
  const int2* tdescB;    // {k0B,k1B} (K_SCSR_PRIV only)
  const int* ptrA;
  const int* idxA;
  const double* valA;
  const int* ptrB;       // CSR of L^T (K_SCSR_PRIV only)
  const int* idxB;
  const double* valB;
  const int2* twin;      // per tile: new gathered columns [lo,hi] vs the previous tile
  int rev;               // visit tiles last-to-first (per-pass engine: alternate passes
                         // start where the previous one ended, on its L2-resident lines)
  int tree;              // split long lines: per-lane partial sums + a fixed shuffle tree
                         // (reassociated, deterministic) instead of the in-order sum
  int wide;              // tiles may exceed kBlock lines (launch the WIDE instantiation)
  int cta0, ncta;        // CTAs [cta0, cta0 + ncta) work this view (ncta 0: the grid)
  // K_SCSR_FIX: fixed-point accumulator of the transposed contributions, the
  // bits of max|x| of the gathered vector, and ceil(log2(max_j sum_i |a_ij|))
  unsigned long long* ytx;
  const unsigned long long* txmax;
  int tx_eM;
};

struct StageMeta {
  int row0, row1;   // lines [row0,row1)
  int r0a;          // row-pointer slice starts at ptr[r0a]
  int kA0a, kB0a;   // first staged entry of each segment (4-aligned)
  int offB;         // segment B's offset inside the stage buffers
  int is_long;      // 1: entries not staged, read from global
  int cnt;          // staged entries (both segments)
};

struct __align__(16) Smem {
  double val[kStages][kNzCap];
  int idx[kStages][kNzCap];
  int rpA[kStages][kRpCapA];
  int rpB[kStages][kRpCap];
  uint64_t full[kStages];
  StageMeta meta[kStages];
  double red[32];
  double bcast;
};

__device__ __forceinline__ int view_cta(const MatView& M) { return (int)blockIdx.x - M.cta0; }
__device__ __forceinline__ int view_ctas(const MatView& M) {
  return M.ncta ? M.ncta : (int)gridDim.x;
}
__device__ __forceinline__ int my_tile(const MatView& M, int j) {
  const int t = view_cta(M) + j * view_ctas(M);
  return M.rev ? M.ntiles - 1 - t : t;
}
__device__ __forceinline__ int my_tile_count(const MatView& M) {
  const int b = view_cta(M), g = view_ctas(M);
  return (M.ntiles > b) ? (M.ntiles - 1 - b) / g + 1 : 0;
}

// Tile descriptor(s), fetched ahead of the issue so thread 0 never waits on
// a global load between a tile's barrier and the next bulk copy.
struct TileDesc {
  int4 a;   // {row0,row1,k0,k1}
  int2 b;   // {k0B,k1B}
  int2 w;   // leading-edge column window to prefetch (lo > hi: none)
};
template <bool TWO>
__device__ __forceinline__ TileDesc load_desc(const MatView& M, int t) {
  TileDesc d;
  d.a = M.tdesc[t];
  d.b = TWO ? M.tdescB[t] : make_int2(0, 0);
  d.w = M.twin ? M.twin[t] : make_int2(1, 0);
  return d;
}

// Vectors a pass may ask to be pulled into L2 (leading-edge window of each
// tile, issued with the tile's staging copies kStages tiles ahead).  Measured
// neutral-to-negative on the stencil workloads (profiles/r01/), so the
// passes leave it unset; kept for matrices with poor gather locality.
struct Prefetch {
  const double* v0 = nullptr;  // gathered vectors: leading-edge window
  const double* v1 = nullptr;
  const double* own = nullptr; // read at the tile's own rows
};

__device__ __forceinline__ void prefetch_window(const double* v, int2 w) {
  if (v == nullptr || w.x > w.y) return;
  const int lo = w.x & ~1;             // 16-byte aligned
  const int hi = (w.y + 2) & ~1;       // exclusive, even
  bulk_prefetch_l2(v + lo, (uint32_t)(hi - lo) * 8u);
}

// Thread 0 only: stage the tile described by `dd` into ring slot `s`.
template <bool TWO>
__device__ __forceinline__ void issue_tile_desc(Smem& sm, const MatView& M, const TileDesc& dd,
                                                int s, const Prefetch* pf = nullptr) {
  if (pf) {
    prefetch_window(pf->v0, dd.w);
    prefetch_window(pf->v1, dd.w);
    prefetch_window(pf->own, make_int2(dd.a.x, dd.a.y - 1));
  }
  const int4 d = dd.a;
  const int row0 = d.x, row1 = d.y, kA0 = d.z, kA1 = d.w;
  const int kB0 = TWO ? dd.b.x : 0, kB1 = TWO ? dd.b.y : 0;
  StageMeta& mt = sm.meta[s];
  mt.row0 = row0;
  mt.row1 = row1;
  const int r0a = row0 & ~3;
  const int rcnt = ((row1 + 1 + 3) & ~3) - r0a;
  mt.r0a = r0a;
  const int nA = kA1 - kA0, nB = kB1 - kB0;
  const bool is_long = (nA + nB) > kTileNnz;
  mt.is_long = is_long;
  uint32_t bytes = (uint32_t)rcnt * 4u * (TWO ? 2u : 1u);
  int kA0a = kA0 & ~3, cA = 0, kB0a = kB0 & ~3, cB = 0;
  if (!is_long) {
    cA = (nA > 0) ? ((kA1 + 3) & ~3) - kA0a : 0;
    cB = (TWO && nB > 0) ? ((kB1 + 3) & ~3) - kB0a : 0;
    bytes += (uint32_t)(cA + cB) * 12u;
  }
  mt.kA0a = kA0a;
  mt.kB0a = kB0a;
  mt.offB = cA;
  mt.cnt = cA + cB;
  fence_proxy_async_smem();
  mbar_arrive_expect_tx(&sm.full[s], bytes);
  bulk_g2s(sm.rpA[s], M.ptrA + r0a, (uint32_t)rcnt * 4u, &sm.full[s]);
  if (TWO) bulk_g2s(sm.rpB[s], M.ptrB + r0a, (uint32_t)rcnt * 4u, &sm.full[s]);
  if (cA > 0) {
    bulk_g2s_stream(sm.idx[s], M.idxA + kA0a, (uint32_t)cA * 4u, &sm.full[s]);
    bulk_g2s_stream(sm.val[s], M.valA + kA0a, (uint32_t)cA * 8u, &sm.full[s]);
  }
  if (TWO && cB > 0) {
    bulk_g2s_stream(sm.idx[s] + cA, M.idxB + kB0a, (uint32_t)cB * 4u, &sm.full[s]);
    bulk_g2s_stream(sm.val[s] + cA, M.valB + kB0a, (uint32_t)cB * 8u, &sm.full[s]);
  }
}

template <bool TWO>
__device__ __forceinline__ void issue_tile(Smem& sm, const MatView& M, int t, int s) {
  issue_tile_desc<TWO>(sm, M, load_desc<TWO>(M, t), s);
}

// Ring of kStages stages over this CTA's tile list (t = blockIdx.x + j*gridDim.x).
// If the CTA owns <= kStages tiles they are loaded once and stay resident in
// shared memory for the whole kernel (the 30880-row matrix fits this way);
// otherwise the list is streamed cyclically, prefetching kStages tiles ahead,
// across pass and iteration boundaries.
struct Pipe {
  int m;
  bool resident;
  long long c;    // tiles consumed (streaming mode)
  TileDesc next;  // thread 0: descriptor of the next tile to issue
  Prefetch pf;    // gathered vectors of the pass that will consume issued tiles
#if SPCG_TRACE
  unsigned long long wait_ns;  // thread 0: time blocked on tile data (tracing)
  bool trace;
#endif
};

// allow_resident=false forces cyclic streaming even for <= kStages tiles
// (needed when a pass overwrites staged values in place and the tiles are
// visited again, e.g. every CG iteration).
template <bool TWO>
__device__ __forceinline__ void pipe_start(Pipe& P, Smem& sm, const MatView& M,
                                           bool allow_resident = true) {
  P.m = my_tile_count(M);
  P.resident = allow_resident && P.m <= kStages;
  P.c = 0;
#if SPCG_TRACE
  P.wait_ns = 0;
  P.trace = false;
#endif
  if (threadIdx.x == 0 && P.m > 0) {
    const int pre = P.resident ? P.m : kStages;
    for (int j = 0; j < pre; ++j) issue_tile<TWO>(sm, M, my_tile(M, j % P.m), j);
    if (!P.resident) P.next = load_desc<TWO>(M, my_tile(M, kStages % P.m));
  }
}

// Stage holding the j-th tile of the current pass (waits for its bytes).
__device__ __forceinline__ int pipe_acquire(Pipe& P, Smem& sm, int j) {
  if (P.resident) {
    mbar_wait(&sm.full[j], 0);
    return j;
  }
  const int s = (int)(P.c % kStages);
#if SPCG_TRACE
  if (P.trace && threadIdx.x == 0) {
    const unsigned long long t0 = globaltimer_ns();
    mbar_wait(&sm.full[s], (uint32_t)((P.c / kStages) & 1));
    P.wait_ns += globaltimer_ns() - t0;
    return s;
  }
#endif
  mbar_wait(&sm.full[s], (uint32_t)((P.c / kStages) & 1));
  return s;
}

// Done with the stage returned by pipe_acquire: recycle it for a later tile.
template <bool TWO>
__device__ __forceinline__ void pipe_release(Pipe& P, Smem& sm, const MatView& M, int s) {
  if (P.resident) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    issue_tile_desc<TWO>(sm, M, P.next, s, &P.pf);
    P.next = load_desc<TWO>(M, my_tile(M, (int)((P.c + kStages + 1) % P.m)));
  }
  P.c++;
}

// Wait for copies still in flight before the CTA exits.
__device__ __forceinline__ void pipe_drain(Pipe& P, Smem& sm) {
  if (P.m == 0) return;
  if (P.resident) {
    for (int j = 0; j < P.m; ++j) mbar_wait(&sm.full[j], 0);
    return;
  }
  for (int u = 0; u < kStages; ++u) {
    const long long q = P.c + u;
    mbar_wait(&sm.full[q % kStages], (uint32_t)((q / kStages) & 1));
  }
}

__device__ __forceinline__ void smem_init(Smem& sm) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&sm.full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
}

// ---- deterministic reductions ------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Fixed-order block sum, result broadcast to every thread.  S: any shared
// struct with `double red[32]; double bcast;`.
template <class S>
__device__ __forceinline__ double block_sum(double v, S& sm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();  // protects sm.red / sm.bcast reuse
  if (lane == 0) sm.red[w] = v;
  __syncthreads();
  if (w == 0) {
    double t = (lane < (int)(blockDim.x >> 5)) ? sm.red[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) sm.bcast = t;
  }
  __syncthreads();
  return sm.bcast;
}

}  // namespace spcg
