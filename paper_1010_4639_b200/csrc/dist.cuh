// dist.cuh — per-pass CG kernels: the row-sharded multi-GPU solve and the
// single-GPU streaming engine (the same engine with no peers).
//
// Each rank owns lines [row0,row1) of A (a "local" handle whose column
// indices are localized: owned columns -> [0,nloc), halo columns ->
// [nloc, nloc+nhalo)).  The search direction is stored extended,
// p_ext = [own p | neighbours' p], so pass A is a plain SpMV over p_ext.
// One iteration (unfolded CG: every pass streams at full speed, and each
// kernel keeps the whole register budget for its own loop):
//   A  q = A p_ext, partial p.q              -> all-reduce -> alpha
//   B  r -= alpha q, partial r.r             -> all-reduce -> beta, flags
//   C  x += alpha p, p = r + beta p          -> p's halo to the neighbours
// Scalars live in a device StepState; dot products are reduced in fixed
// order on each rank (last-CTA-done) and then across ranks, so every rank
// computes bitwise identical alpha/beta/flags and stops at the same iteration.
//
// Transports of the cross-rank steps (DistArgs::fused):
//  * fused = 0 (host-launched): the last CTA leaves the rank's partial in
//    StepState::red; the host enqueues ncclAllReduce (or the host-callback
//    transport's exchange) and a one-thread dist_scalar kernel, and the halo
//    goes by ncclSend/Recv after a pack kernel.
//  * fused = 1 (device-initiated, no host collective): the last CTA of a
//    reducing pass posts the rank partial into EVERY rank's mailbox slot (an
//    epoch-tagged word pair per source: peers' mailboxes are mapped through
//    CUDA IPC, or are plain device memory for ranks sharing a GPU), polls
//    its own mailbox until every rank's tag arrived, sums the R partials in
//    rank order (bitwise identical on every rank) and runs the scalar step
//    itself.  Pass C stores the boundary p values straight into the
//    neighbours' p_ext halo slots (remote stores over NVLink), each CTA
//    fences at system scope, and the last one posts a halo tag to every
//    receiving neighbour; the next pass A waits for the tags only before its
//    first tile that gathers halo columns, so interior tiles overlap the
//    neighbours' tail.  3 launches per iteration, no host work between them.
//
// Several ranks can run in ONE launch ("virtual ranks": rank v owns CTAs
// [v*G, (v+1)*G) and reads its own DistArgs) — how the device protocol is
// exercised on a single GPU (tests/test_gpu_p2p.py) without ever running
// kernels that wait on each other as separate launches.
#pragma once
#include "lines.cuh"

namespace spcg {

// Block size of the elementwise passes (B, C, x): independent of the tile
// kernels' kBlock so their grid-stride parallelism does not shrink with it.
constexpr int kElemBlock = 512;
constexpr int kMaxRanks = 16;   // peers of the device-initiated transport
constexpr int kRunCache = 8;    // send runs fused into pass C (else a push kernel)

struct StepState {
  double rr, alpha, beta, b_norm, rel, tol;
  double red;  // local partial sum (host transports all-reduce it in place)
  double pad0;
  long long k, max_it, fail_iter;
  long long kc;  // iterations whose pass C ran
  int status, converged, done, x0_given;
  unsigned int counter;  // last-CTA-done ticket
  int record;
  // K_SCSR_FIX: bits of max|p| per iteration parity (pass C fills the next
  // slot, pass A / B read the current one, pass B clears the next); slot 2:
  // the x0 / true-residual SpMVs
  unsigned long long pmax[3];
  unsigned int rseq;  // device transport: reductions done (mailbox tag/bank)
  unsigned int hseq;  // device transport: halo pushes done (halo tag)
};

// Contiguous run of send rows: own rows [lo,hi) go to peer `peer`'s extended
// vector at [dst, dst + hi - lo).
struct SendRun {
  int lo, hi, peer, pad;
  long long dst;
};

// Where a rank's device-transport traffic goes: its own mailbox / halo tags
// and the peers' buffers (device memory; only the exchange steps read it).
struct PeerTab {
  unsigned long long* mbox;                // own mailbox [2 banks][nranks][2]
  unsigned long long* hflag;               // own halo tags [nranks][2]
  int recv_from[kMaxRanks];                // ranks this one receives halo values from
  int send_to[kMaxRanks];                  // ranks this one sends halo values to
  unsigned long long* peer_mbox[kMaxRanks];
  unsigned long long* peer_hflag[kMaxRanks];
  double* peer_p[kMaxRanks];               // peers' p_ext
  double* peer_tmp[kMaxRanks];             // peers' tmp (x0 / x halos)
  double* peer_q[kMaxRanks];               // peers' q (reverse halo)
};

// Everything one rank's kernels need (by value as a kernel parameter for a
// single rank; an array in device memory for a launch over virtual ranks).
struct DistArgs {
  MatView M;          // localized rows (streaming tile view)
  StepState* S;
  double* p;          // p_ext: own p | halo
  double* r;
  double* q;          // extended: ghost slots of the single-pass SCSR scatter
  double* x;
  const double* b;
  const double* x0;   // nullable
  double* tmp;        // extended scratch (x0 / x with their halos)
  double* hist;
  double* part;       // per-CTA partials
  long long nloc;
  int rank, nranks;
  int zq;             // atomic formats: pass B re-zeroes q
  int xv;             // x is 16-byte aligned
  unsigned long long* txnext;  // K_SCSR_FIX: the max|p| slot pass C fills (pass B clears it)
  // device transport
  const PeerTab* peer;
  const unsigned char* thalo;  // per tile of M: gathers halo columns
  int nrecv, nsendpeers;
  int gpu_scope;               // every peer is on this device: gpu-scope exchange
  int nruns;                   // send runs (<= kRunCache: fused into pass C)
  const SendRun* runs;
  long long send_total;        // generic push: every send entry
  const int* send_idx;
  const int* send_peer;
  const long long* send_dst;
  long long nghost;            // reverse halo (SCSR atomic)
  const int* ghost_peer;
  const int* ghost_dst;
};

// This CTA's rank and its block index / count inside the rank.
struct RankCta {
  int v, lb, G;
};
__device__ __forceinline__ RankCta rank_cta(int G) {
  RankCta c;
  c.G = G;
  c.v = (int)blockIdx.x / G;
  c.lb = (int)blockIdx.x - c.v * G;
  return c;
}
// The rank's tile view with its CTA range (tiles.cuh: my_tile / my_tile_count).
__device__ __forceinline__ MatView rank_view(const DistArgs& A, const RankCta& c) {
  MatView M = A.M;
  M.cta0 = c.v * c.G;
  M.ncta = c.G;
  return M;
}

// Kernel transport modes (compile time): 0 = host transport, one rank, its
// DistArgs by value (the parameter bank, as lean as a plain kernel); 1 =
// device transport, one rank by value; 2 = device transport, several virtual
// ranks of one launch reading their DistArgs from the device array DAs.
#define SPCG_RANK_ARGS(MODE)                                              \
  const RankCta c = rank_cta(MODE == 2 ? G : (int)gridDim.x);             \
  const DistArgs& A = (MODE == 2) ? DAs[c.v] : A1;

// ---- scalar steps ------------------------------------------------------------
// op 0: after ||b||^2          op 1: after r0.r0 (start)
// op 2: after p.q (alpha)      op 3: after r.r (convergence, beta)
// op 4: after the true residual
__device__ __noinline__ void scalar_step(int op, StepState* S, double* hist) {
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
  if (op == 4) {
    S->rel = sqrt(S->red) / S->b_norm;
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

// Host-transport scalar step (one thread), operating on the all-reduced S->red.
__global__ void dist_scalar(int op, StepState* S, double* hist) { scalar_step(op, S, hist); }

// ---- system-scope memory operations (peer memory over NVLink) ---------------
// Scope of the exchange: system (peers are other GPUs: NVLink peer memory)
// or gpu (virtual ranks of one launch on one device, DistArgs::gpu_scope).
__device__ __forceinline__ void fence_acq_rel_sys(bool gpu = false) {
  if (gpu) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  else asm volatile("fence.acq_rel.sys;" ::: "memory");
}
__device__ __forceinline__ void st_relaxed_sys_u64(unsigned long long* p, unsigned long long v,
                                                   bool gpu = false) {
  if (gpu) asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const unsigned long long* p,
                                                                 bool gpu = false) {
  unsigned long long v;
  if (gpu) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v,
                                                   bool gpu = false) {
  if (gpu) asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p,
                                                                 bool gpu = false) {
  unsigned long long v;
  if (gpu) asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
constexpr unsigned long long kP2PSpinLimit = 1ull << 34;  // ~minutes: a lost peer traps

// Device all-reduce of the rank partial s (thread 0 of the rank's last CTA):
// post {hi32|tag, lo32|tag} into every rank's mailbox slot of this rank,
// poll the own mailbox until all R tags are in, sum in rank order.  Two
// banks by reduction parity make slot reuse safe (a rank can be at most one
// reduction ahead of a slower reader).
//
// Called by a whole warp (lane k posts to rank k and polls rank k's slot, in
// parallel; a warp-uniform loop, see the resident engines' exchange); the
// rank-ordered total is returned in every lane, and lane 0 owns S.
__device__ __noinline__ double mailbox_allreduce(const DistArgs& A, double s) {
  const int lane = threadIdx.x & 31;
  StepState* S = A.S;
  const unsigned int seq = S->rseq + 1;
  __syncwarp();
  if (lane == 0) S->rseq = seq;
  const int R = A.nranks, bank = (int)(seq & 1u);
  const unsigned long long u = (unsigned long long)__double_as_longlong(s);
  const unsigned long long w0 = (u & 0xffffffff00000000ull) | seq, w1 = (u << 32) | seq;
  if (lane < R) {
    unsigned long long* dst = A.peer->peer_mbox[lane] + ((size_t)bank * R + A.rank) * 2;
    st_relaxed_sys_u64(dst, w0, A.gpu_scope);
    st_relaxed_sys_u64(dst + 1, w1, A.gpu_scope);
  }
  const unsigned long long* src = A.peer->mbox + ((size_t)bank * R + (lane < R ? lane : 0)) * 2;
  unsigned long long a = 0, b = 0, spins = 0;
  bool ok = lane >= R;
  while (!__all_sync(0xffffffffu, ok)) {
    if (!ok) {
      a = ld_relaxed_sys_u64(src, A.gpu_scope);
      b = ld_relaxed_sys_u64(src + 1, A.gpu_scope);
      ok = (uint32_t)a == seq && (uint32_t)b == seq;
    }
    if (++spins > kP2PSpinLimit) asm volatile("trap;");
  }
  const double mine = __longlong_as_double((long long)((a & 0xffffffff00000000ull) | (b >> 32)));
  double tot = 0.0;
  for (int k = 0; k < R; ++k) tot += __shfl_sync(0xffffffffu, mine, k);  // rank order
  return tot;
}

// Fixed-order reduction of one rank's grid without a grid barrier: every CTA
// writes its block sum to part[], the last CTA to arrive sums part[] in index
// order; then (op >= 0) the cross-rank step: host transport -> S->red only;
// device transport -> mailbox all-reduce + the scalar step in place.
// post = false: leave the local sum in S->red (a later kernel posts it).
struct RedSmem {
  double red[32];
  double bcast;
};

template <bool FUSED, class SM>
__device__ __forceinline__ void rank_sum(double v, SM& sm, const DistArgs& A, const RankCta& c,
                                         int op, bool post = true) {
  const double bs = block_sum(v, sm);
  __shared__ bool last;
  StepState* S = A.S;
  if (threadIdx.x == 0) {
    A.part[c.lb] = bs;
    __threadfence();
    const unsigned int t = atomicAdd(&S->counter, 1u);
    last = (t == (unsigned)c.G - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double s = 0.0;
  for (int i = threadIdx.x; i < c.G; i += blockDim.x) s += __ldcg(A.part + i);
  s = block_sum(s, sm);
  if (FUSED && post && op >= 0) {
    if (threadIdx.x < 32) {
      const double tot = mailbox_allreduce(A, s);
      if (threadIdx.x == 0) {
        S->counter = 0;
        S->red = tot;
        scalar_step(op, S, A.hist);
      }
    }
  } else if (threadIdx.x == 0) {
    S->counter = 0;
    S->red = s;
  }
}

// Device transport: wait (thread 0, then the CTA) for the halo of push number
// `tag` from every rank this one receives from.
__device__ __noinline__ void wait_halo(const DistArgs& A, unsigned int tag) {
  if (threadIdx.x < 32) {  // warp 0, lane i polls source i (warp-uniform loop)
    const int lane = threadIdx.x;
    const unsigned long long* f =
        lane < A.nrecv ? A.peer->hflag + 2 * (size_t)A.peer->recv_from[lane] : nullptr;
    bool ok = f == nullptr;
    unsigned long long spins = 0;
    while (!__all_sync(0xffffffffu, ok)) {
      if (!ok) ok = (uint32_t)ld_acquire_sys_u64(f, A.gpu_scope) >= tag;
      if (++spins > kP2PSpinLimit) asm volatile("trap;");
    }
  }
  __syncthreads();
}

// After a CTA's remote halo stores: system-scope fence, ticket; the last CTA
// of the rank posts the halo tag to every receiving peer.
template <class SM>
__device__ __forceinline__ void halo_done(const DistArgs& A, const RankCta& c, SM& sm,
                                          unsigned int tag) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_acq_rel_sys(A.gpu_scope);
    const unsigned int t = atomicAdd(&A.S->counter, 1u);
    last = (t == (unsigned)c.G - 1);
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  A.S->counter = 0;
  A.S->hseq = tag;
  fence_acq_rel_sys(A.gpu_scope);
  for (int i = 0; i < A.nsendpeers; ++i)
    st_release_sys_u64(A.peer->peer_hflag[A.peer->send_to[i]] + 2 * (size_t)A.rank, tag,
                       A.gpu_scope);
}

// Virtual-rank launches: the CTA's rank arguments copied into shared memory
// (word by word by the first warps) with the rank's CTA range and the pass's
// traversal flags patched in.
__device__ __forceinline__ void stage_args(DistArgs& sA, const DistArgs& g, const RankCta& c,
                                           int rev, int tree) {
  static_assert(sizeof(DistArgs) % 8 == 0, "DistArgs copied in 8-byte words");
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(&g);
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(&sA);
  for (int w = threadIdx.x; w < (int)(sizeof(DistArgs) / 8); w += blockDim.x) dst[w] = src[w];
  __syncthreads();
  if (threadIdx.x == 0) {
    sA.M.cta0 = c.v * c.G;
    sA.M.ncta = c.G;
    sA.M.rev = rev;
    sA.M.tree = tree;
  }
  __syncthreads();
}

// ---- pass A: q = A p_ext, red = p.q partial (skipped once done) -------------
// WIDE: the view carries wide tiles (short-row CSR); a separate
// instantiation so the other kernels do not pay the two-line body's registers.
// Body of pass A over rank A's view M (M carries rev / tree / the CTA range).
template <int FMT, bool WIDE, bool FUSED>
__device__ __forceinline__ void spmv_pq_body(const DistArgs& A, const MatView& M, const RankCta& c,
                                             int post) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  StepState* S = A.S;
  if (S->done) {
    // what the alpha step records when it has nothing to do: pass C of an
    // exhausted max_iter ran once and must not run again
    if (c.lb == 0 && threadIdx.x == 0) S->kc = S->k;
    return;
  }
  constexpr bool TWO = (FMT == K_SCSR_PRIV);
  smem_init(sm);
  Pipe P;
  pipe_start<TWO>(P, sm, M);
  const bool waits = FUSED && A.nrecv > 0;
  const unsigned int htag = waits ? S->hseq : 0u;
  bool have_halo = !waits;
  SrcPlain src{A.p};
  double pq = 0.0;
  for (int j = 0; j < P.m; ++j) {
    const int s = pipe_acquire(P, sm, j);
    if (!have_halo && A.thalo[my_tile(M, j)]) {  // CTA-uniform
      wait_halo(A, htag);
      have_halo = true;
    }
    if (WIDE && wide_tile<FMT>(sm, s)) {
      LineOut o2[2];
      bool act[2];
      int li[2];
      csr_line_pair(sm, s, src, o2, act, li, nullptr);
#pragma unroll
      for (int t = 0; t < 2; ++t)
        if (act[t]) {
          A.q[li[t]] = o2[t].q;
          pq += o2[t].xi * o2[t].q;
        }
    } else {
      bool active = false;
      int i = -1;
      // atomic formats: transposed scatter into q (zeroed by pass B), p.Ap
      // from the line's own gather (line_pq)
      const LineOut o = tile_line<FMT, true>(sm, s, M, src, A.q, active, i, sm.val[s]);
      if (active) {
        finish_plain<FMT>(o, i, A.q);
        pq += line_pq<FMT>(o);
      }
    }
    pipe_release<TWO>(P, sm, M, s);
  }
  pipe_drain(P, sm);
  rank_sum<FUSED>(pq, sm, A, c, 2, post != 0);
}

// pass A: q = A p_ext, red = p.q partial (skipped once done).  WIDE: the
// view carries wide tiles (short-row CSR); a separate instantiation so the
// other kernels do not pay the two-line body's registers.  MODE 0 / 1: one
// rank, its DistArgs passed by value (the view stays in the parameter bank;
// the host sets M.rev / M.tree per launch); MODE 2: several virtual ranks of
// one launch, each reading its DistArgs from DAs.
// post = 0: leave the p.q partial for dist_ghost_push (device transport,
// single-pass SCSR with peers: uniform over the ranks of a launch)
template <int FMT, bool WIDE, int MODE>
__global__ void __launch_bounds__(kBlock, kStreamMinBlocks)
    dist_spmv_pq(const __grid_constant__ DistArgs A1, const DistArgs* __restrict__ DAs, int G,
                 int rev, int tree, int post) {
  if (MODE == 2) {
    // the rank's arguments staged in shared memory (a register copy of the
    // view spilled in the tile loop)
    __shared__ DistArgs sA;
    const RankCta c = rank_cta(G);
    stage_args(sA, DAs[c.v], c, rev, tree);
    spmv_pq_body<FMT, WIDE, true>(sA, sA.M, c, post);
  } else {
    spmv_pq_body<FMT, WIDE, MODE == 1>(A1, A1.M, rank_cta((int)gridDim.x), post);
  }
}

// Device transport, SCSR atomic with peers: the transposed contributions that
// landed in this rank's ghost slots go straight into their owners' q (remote
// fp64 reds over NVLink; this format's summation order is unspecified
// anyway), the ghosts are re-zeroed, and the last CTA posts pass A's p.q.
// op = -1: a barrier after the ghost reds (x0 / true-residual SpMVs, whose
// q the owners read next) instead of the p.q step.
template <int MODE>
__global__ void __launch_bounds__(kElemBlock)
    dist_ghost_push(const __grid_constant__ DistArgs A1, const DistArgs* __restrict__ DAs, int G,
                    int op) {
  SPCG_RANK_ARGS(MODE)
  StepState* S = A.S;
  if (op >= 0 && S->done) return;
  double* ghost = A.q + A.nloc;
  const long long GT = (long long)c.G * blockDim.x;
  for (long long h = (long long)c.lb * blockDim.x + threadIdx.x; h < A.nghost; h += GT) {
    const double v = ghost[h];
    ghost[h] = 0.0;
    if (v != 0.0) red_add_f64(A.peer->peer_q[A.ghost_peer[h]] + A.ghost_dst[h], v);
  }
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_acq_rel_sys(A.gpu_scope);  // the reds are visible before the p.q post
    const unsigned int t = atomicAdd(&S->counter, 1u);
    last = (t == (unsigned)c.G - 1);
  }
  __syncthreads();
  if (!last || threadIdx.x >= 32) return;
  const double tot = mailbox_allreduce(A, op >= 0 ? S->red : 0.0);
  if (threadIdx.x != 0) return;
  S->counter = 0;
  if (op >= 0) {
    S->red = tot;
    scalar_step(op, S, A.hist);
  }
}

// Reverse halo of the single-pass symmetric SpMV (host transports): partial
// sums of the transposed scatters that landed in this rank's ghost slots
// (halo columns owned by lower ranks) arrive in buf, aligned with the send
// list; add them into q at those rows.  Atomic adds: a row can be in several
// peers' halos, and this format's summation order is unspecified anyway.
__global__ void __launch_bounds__(256) dist_unpack_add(long long total, const int* idx,
                                                       const double* buf, double* q) {
  const long long G = (long long)gridDim.x * blockDim.x;
  for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < total; s += G)
    red_add_f64(q + idx[s], buf[s]);
}

// q = A tmp (plain gather; initial / true residual).  Device transport: waits
// for the halo of the push just done (number S->hseq) first.
template <int FMT, bool WIDE, bool FUSED>
__device__ __forceinline__ void spmv_body(const DistArgs& A, const MatView& M) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  constexpr bool TWO = (FMT == K_SCSR_PRIV);
  smem_init(sm);
  if (FUSED && A.nrecv > 0) wait_halo(A, A.S->hseq);
  Pipe P;
  pipe_start<TWO>(P, sm, M);
  SrcPlain src{A.tmp};
  for (int j = 0; j < P.m; ++j) {
    const int s = pipe_acquire(P, sm, j);
    if (WIDE && wide_tile<FMT>(sm, s)) {
      LineOut o2[2];
      bool act[2];
      int li[2];
      csr_line_pair(sm, s, src, o2, act, li, nullptr);
#pragma unroll
      for (int t = 0; t < 2; ++t)
        if (act[t]) A.q[li[t]] = o2[t].q;
    } else {
      bool active = false;
      int i = -1;
      const LineOut o = tile_line<FMT, false>(sm, s, M, src, A.q, active, i, sm.val[s]);
      if (active) finish_plain<FMT>(o, i, A.q);
    }
    pipe_release<TWO>(P, sm, M, s);
  }
  pipe_drain(P, sm);
}

template <int FMT, bool WIDE, int MODE>
__global__ void __launch_bounds__(kBlock, kStreamMinBlocks)
    dist_spmv(const __grid_constant__ DistArgs A1, const DistArgs* __restrict__ DAs, int G,
              int /*unused: launch-macro symmetry*/) {
  if (MODE == 2) {
    __shared__ DistArgs sA;
    const RankCta c = rank_cta(G);
    stage_args(sA, DAs[c.v], c, 0, 0);
    spmv_body<FMT, WIDE, true>(sA, sA.M);
  } else {
    spmv_body<FMT, WIDE, MODE == 1>(A1, A1.M);
  }
}

// Elementwise kernels over the nloc own lines (grid-stride, fixed order).
// mode 0: red = b.b                       -> op 0
// mode 1: r = b - q (or b), red = r.r, p = r  -> op 1  (useq: q holds A x0)
// mode 2: r -= alpha q, red = r.r         -> op 3
// mode 3: red = |b - q|^2 (true residual) -> op 4
// Mode 2 moves 16-byte pairs, two in flight per thread (r, q 16-B aligned).
template <int MODE>
__global__ void __launch_bounds__(kElemBlock)
    dist_elem(const __grid_constant__ DistArgs A1, const DistArgs* __restrict__ DAs, int G,
              int mode, int useq, int rev) {
  __shared__ RedSmem sm;
  SPCG_RANK_ARGS(MODE)
  StepState* S = A.S;
  if (mode == 2 && S->done) return;
  const long long nloc = A.nloc;
  double* q = A.q;
  double* r = A.r;
  const double* b = A.b;
  const int zq = A.zq;
  const double alpha = S->alpha;
  const long long g = (long long)c.lb * blockDim.x + threadIdx.x;
  const long long GT = (long long)c.G * blockDim.x;
  // K_SCSR_FIX: q = gather part + fixed-point transposed part (then cleared)
  unsigned long long* Y = A.M.ytx;
  const double iy = (Y && mode != 0) ? 1.0 / fix_scale(A.M.txmax, A.M.tx_eM) : 0.0;  // exact
  if (Y && mode == 2 && c.lb == 0 && threadIdx.x == 0 && A.txnext) *A.txnext = 0ull;
  double acc = 0.0;
  if (mode == 2) {
    const double na = -alpha;
    const long long np = nloc >> 1;
    const double2* q2 = reinterpret_cast<const double2*>(q);
    double2* r2 = reinterpret_cast<double2*>(r);
    // every load of a round is issued before its stores (the Y / q stores
    // may alias later loads as far as the compiler knows: interleaving them
    // serialised the round -- 0.43 ms instead of 0.2 for Q27's pass B)
    auto fixq = [&](double2 qv, ulonglong2 t) {
      qv.x = __dadd_rn(qv.x, s64_to_f64((long long)t.x) * iy);
      qv.y = __dadd_rn(qv.y, s64_to_f64((long long)t.y) * iy);
      return qv;
    };
    ulonglong2* y2 = reinterpret_cast<ulonglong2*>(Y);
    const ulonglong2 z2 = make_ulonglong2(0ull, 0ull);
    long long i = g;
    for (; i + GT < np; i += 2 * GT) {
      const long long ia = rev ? np - 1 - i : i, ib = rev ? np - 1 - (i + GT) : i + GT;
      double2 qa = q2[ia], qb = q2[ib];
      const double2 ra = r2[ia], rb = r2[ib];
      if (Y) {
        const ulonglong2 ya = y2[ia], yb = y2[ib];
        qa = fixq(qa, ya);
        qb = fixq(qb, yb);
      }
      const double2 oa = make_double2(mul_add_rn(ra.x, na, qa.x), mul_add_rn(ra.y, na, qa.y));
      const double2 ob = make_double2(mul_add_rn(rb.x, na, qb.x), mul_add_rn(rb.y, na, qb.y));
      r2[ia] = oa;
      r2[ib] = ob;
      if (Y) {
        y2[ia] = z2;
        y2[ib] = z2;
      }
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
      double2 qa = q2[ia];
      const double2 ra = r2[ia];
      if (Y) qa = fixq(qa, y2[ia]);
      const double2 oa = make_double2(mul_add_rn(ra.x, na, qa.x), mul_add_rn(ra.y, na, qa.y));
      r2[ia] = oa;
      if (Y) y2[ia] = z2;
      if (zq) reinterpret_cast<double2*>(q)[ia] = make_double2(0.0, 0.0);
      acc = fma(oa.x, oa.x, acc);
      acc = fma(oa.y, oa.y, acc);
    }
    if ((nloc & 1) && g == 0) {
      double qv = q[nloc - 1];
      if (Y) {
        qv = __dadd_rn(qv, s64_to_f64((long long)Y[nloc - 1]) * iy);
        Y[nloc - 1] = 0ull;
      }
      const double v = mul_add_rn(r[nloc - 1], na, qv);
      if (zq) q[nloc - 1] = 0.0;
      r[nloc - 1] = v;
      acc = fma(v, v, acc);
    }
  } else {
    for (long long i = g; i < nloc; i += GT) {
      double v;
      double qv = 0.0;
      if (mode != 0 && (mode == 3 || useq)) {
        qv = q[i];
        if (Y) {
          qv = __dadd_rn(qv, s64_to_f64((long long)Y[i]) * iy);
          Y[i] = 0ull;
        }
      }
      if (mode == 0) {
        v = b[i];
      } else if (mode == 1) {
        v = useq ? mul_add_rn(b[i], -1.0, qv) : b[i];
        if (useq && zq) q[i] = 0.0;
        r[i] = v;
        A.p[i] = v;
      } else {
        v = mul_add_rn(b[i], -1.0, qv);
      }
      acc = fma(v, v, acc);
    }
  }
  const int op = mode == 0 ? 0 : mode == 1 ? 1 : mode == 2 ? 3 : 4;
  rank_sum<MODE != 0>(acc, sm, A, c, op);
}

// Send runs of this rank cached in shared memory (pass C's fused halo push).
struct RunCache {
  SendRun run[kRunCache];
  int n;
};

// Device transport: store own row i's new p into every neighbour that
// receives it (runs sorted by peer, rows ascending within a run).
__device__ __forceinline__ void push_row(const DistArgs& A, const RunCache& rc, long long i,
                                         double v) {
  for (int k = 0; k < rc.n; ++k) {
    const SendRun& R = rc.run[k];
    if (i >= R.lo && i < R.hi) A.peer->peer_p[R.peer][R.dst + (i - R.lo)] = v;
  }
}

// pass C: x += alpha p, p = r + beta p, for an iteration that neither
// converged nor failed (a converged solve applies its last x update at the
// end; an exhausted max_iter runs its pass C).  Device transport: the new p
// of send rows goes straight into the neighbours' halo slots (runs <=
// kRunCache; else dist_push afterwards), then the halo tag.
template <int MODE>
__global__ void __launch_bounds__(kElemBlock)
    dist_update(const __grid_constant__ DistArgs A1, const DistArgs* __restrict__ DAs, int G,
                int rev) {
  __shared__ RunCache rc;
  __shared__ RedSmem sm;
  SPCG_RANK_ARGS(MODE)
  StepState* S = A.S;
  if (S->status != 0 || S->converged || S->kc >= S->k) return;
  // device transport, send runs that fit the cache (also none): the push and
  // the halo tag happen here; otherwise dist_push does both after this pass
  const bool push = MODE != 0 && A.nruns <= kRunCache;
  if (threadIdx.x == 0) rc.n = push ? A.nruns : 0;
  if (threadIdx.x < kRunCache && push && (int)threadIdx.x < A.nruns) rc.run[threadIdx.x] = A.runs[threadIdx.x];
  if (push) __syncthreads();
  const double alpha = S->alpha, beta = S->beta;
  const long long nloc = A.nloc;
  const double* r = A.r;
  double* p = A.p;
  double* x = A.x;
  const long long g = (long long)c.lb * blockDim.x + threadIdx.x;
  const long long GT = (long long)c.G * blockDim.x;
  const long long np = nloc >> 1;
  const double2* r2 = reinterpret_cast<const double2*>(r);
  double2* p2 = reinterpret_cast<double2*>(p);
  double pm = 0.0;
  for (long long j = g; j < np; j += GT) {
    const long long i = rev ? np - 1 - j : j;
    const double2 pv = p2[i], rv = r2[i];
    if (A.xv) {
      double2* x2 = reinterpret_cast<double2*>(x);
      const double2 xo = x2[i];
      x2[i] = make_double2(mul_add_rn(xo.x, alpha, pv.x), mul_add_rn(xo.y, alpha, pv.y));
    } else {
      x[2 * i] = mul_add_rn(x[2 * i], alpha, pv.x);
      x[2 * i + 1] = mul_add_rn(x[2 * i + 1], alpha, pv.y);
    }
    const double2 pn = make_double2(mul_add_rn(rv.x, beta, pv.x), mul_add_rn(rv.y, beta, pv.y));
    p2[i] = pn;
    pm = fmax(pm, fmax(fabs(pn.x), fabs(pn.y)));
    if (push) {
      push_row(A, rc, 2 * i, pn.x);
      push_row(A, rc, 2 * i + 1, pn.y);
    }
  }
  if ((nloc & 1) && g == 0) {
    const long long i = nloc - 1;
    const double pv = p[i];
    x[i] = mul_add_rn(x[i], alpha, pv);
    p[i] = mul_add_rn(r[i], beta, pv);
    if (push) push_row(A, rc, i, p[i]);
    pm = fmax(pm, fabs(p[i]));
  }
  if (A.txnext) {  // K_SCSR_FIX: max|p| of the new direction (bits are monotone for >= 0)
    pm = warp_max(pm);
    if ((threadIdx.x & 31) == 0 && pm > 0.0)
      atomicMax(A.txnext, (unsigned long long)__double_as_longlong(pm));
  }
  if (push) halo_done(A, c, sm, S->hseq + 1);
}

// Device transport, generic halo push of an own vector (src: 0 = p, 1 = x0,
// 2 = x) into the neighbours' extended vectors (dst: 0 = p, 1 = tmp) over the
// whole send list, then the halo tag.  `iter`: the p push of an iteration
// (skipped exactly when its pass C was).
template <int MODE>
__global__ void __launch_bounds__(kElemBlock)
    dist_push(const __grid_constant__ DistArgs A1, const DistArgs* __restrict__ DAs, int G,
              int srcsel, int dstsel, int iter) {
  __shared__ RedSmem sm;
  SPCG_RANK_ARGS(MODE)
  StepState* S = A.S;
  if (iter && (S->status != 0 || S->converged || S->kc >= S->k || A.nruns <= kRunCache)) return;
  const double* src = srcsel == 0 ? A.p : srcsel == 1 ? A.x0 : A.x;
  const long long GT = (long long)c.G * blockDim.x;
  for (long long s = (long long)c.lb * blockDim.x + threadIdx.x; s < A.send_total; s += GT) {
    double* dst = dstsel == 0 ? A.peer->peer_p[A.send_peer[s]] : A.peer->peer_tmp[A.send_peer[s]];
    dst[A.send_dst[s]] = src[A.send_idx[s]];
  }
  halo_done(A, c, sm, S->hseq + 1);
}

// Halo values to send (host transports): v[idx] for every send row.
__global__ void dist_pack(long long cnt, const int* idx, const double* v, double* out) {
  const long long G = (long long)gridDim.x * blockDim.x;
  for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < cnt; s += G)
    out[s] = v[idx[s]];
}

// x = x0 (or 0) and tmp = x0 (own part of the x0 gather vector); final
// x += alpha_K p_K of a converged solve (its pass C was skipped)
template <int MODE>
__global__ void dist_x(const __grid_constant__ DistArgs A1, const DistArgs* __restrict__ DAs,
                       int G, int mode) {
  SPCG_RANK_ARGS(MODE)
  const StepState* S = A.S;
  const long long GT = (long long)c.G * blockDim.x;
  const double alpha = S->alpha;
  const bool upd = S->k > 0 && S->status == 0 && S->converged;
  const bool zero_b = S->b_norm == 0.0;  // solver.py:109-118: x = 0 even for x0 != 0
  for (long long i = (long long)c.lb * blockDim.x + threadIdx.x; i < A.nloc; i += GT) {
    if (mode == 0) {
      const double v = (A.x0 && !zero_b) ? A.x0[i] : 0.0;
      A.x[i] = v;
      if (A.x0) A.tmp[i] = A.x0[i];
    } else if (mode == 1) {
      if (upd) A.x[i] = mul_add_rn(A.x[i], alpha, A.p[i]);
    } else {  // mode 2: tmp = x (own part of the true-residual gather)
      A.tmp[i] = A.x[i];
    }
  }
}

// out = bits of max |v| (atomicMax on the bit patterns of non-negative
// doubles: exact and order-independent); *out must be cleared first
__global__ void vec_absmax_kernel(long long n, const double* v, unsigned long long* out) {
  double m = 0.0;
  const long long G = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += G)
    m = fmax(m, fabs(v[i]));
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0 && m > 0.0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// 2^eM bound of max_j sum_i |a_ij| over the strictly lower part, from the
// rows of L^T summed in storage order: out = bits of the max row sum
__global__ void lt_rowsum_max_kernel(int n, const int* ptr, const double* val,
                                     unsigned long long* out) {
  double m = 0.0;
  const int G = gridDim.x * blockDim.x;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += G) {
    double s = 0.0;
    for (int k = ptr[j]; k < ptr[j + 1]; ++k) s = __dadd_rn(s, fabs(val[k]));
    m = fmax(m, s);
  }
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0 && m > 0.0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// Per tile of a localized view: 1 when any of its entries gathers a halo
// column (>= nloc): the tiles pass A must hold until the halo has arrived.
__global__ void tile_halo_kernel(const int4* desc, const int2* descB, int ntiles, const int* idxA,
                                 const int* idxB, long long nloc, unsigned char* out) {
  __shared__ int any;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    if (threadIdx.x == 0) any = 0;
    __syncthreads();
    const int4 d = desc[t];
    int hit = 0;
    for (int k = d.z + threadIdx.x; k < d.w; k += blockDim.x) hit |= (idxA[k] >= nloc);
    if (descB) {
      const int2 e = descB[t];
      for (int k = e.x + threadIdx.x; k < e.y; k += blockDim.x) hit |= (idxB[k] >= nloc);
    }
    if (hit) any = 1;
    __syncthreads();
    if (threadIdx.x == 0) out[t] = (unsigned char)any;
    __syncthreads();
  }
}

}  // namespace spcg
