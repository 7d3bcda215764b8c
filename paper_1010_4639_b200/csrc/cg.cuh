// cg.cuh — shared pieces of the persistent (grid-resident) CG engine:
// the device result record, the solve arguments, and the grid-wide
// all-reduce barrier and resident tile iteration used by cg1.cuh
// (engine 3, single-reduction CG).  The two-reduction persistent kernels of
// round 1 (engines 1 and 4) were removed: no default path used them and the
// per-pass engine (dist.cuh) is faster on every streaming system.
//
// Scalars are reduced in a fixed order and are bitwise identical in every
// CTA, so control flow stays grid-uniform without any host round trip.

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
  double rec_rel;  // engine 6: the recursive rel of the last iteration
  // resident cluster engines: the leader thread's loop time by phase (ns):
  // [0] SpMV (with the partials' post), [1] reductions / waits, [2] updates
  unsigned long long phase_ns[3];
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
    // warp-uniform loop (every lane until the warp's last slot is in): a
    // divergent spin let finished lanes wait ~7 us at the reconvergence
    // point (profiles/r02/bimodal.md)
    while (__any_sync(0xffffffffu, any)) {
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
      if (kPollSleepNs && __any_sync(0xffffffffu, any)) __nanosleep(kPollSleepNs);
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

}  // namespace spcg
