/*
 * spcg_b200.h — C-ABI of the B200-native fp64 CG solve path.
 *
 * This is the drop-in boundary for the solve path of the reference package
 * `spcg` (arxiv/paper_1010_4639).  The reference binds its hot path from
 * Python into a Cython/OpenMP extension, one call per kernel:
 *
 *   reference call site                               replaced by
 *   ------------------------------------------------  -----------------------------
 *   _ckernels.csr_gather     (_ckernels.pyx:31-47)     spcg_spmv(CSR)
 *   _ckernels.scatter_atomic (_ckernels.pyx:50-62)     spcg_spmv(SCSR, ATOMIC),
 *                                                      spcg_spmv(CSC)
 *   _ckernels.scatter_privatized (_ckernels.pyx:65-91) spcg_spmv(SCSR, PRIVATIZED)
 *   _ckernels.dot_partials + config.pairwise_merge
 *                (_ckernels.pyx:94-108, config.py:43-56) spcg_dot
 *   _ckernels.axpy_kernel    (_ckernels.pyx:111-117)   spcg_axpy
 *   solver.cg_solve loop body (solver.py:107-162)      spcg_cg_solve / spcg_cg_solve_host
 *   core.CsrMatrix / SymHalfMatrix (core.py:57-156)    spcg_matrix_create_host
 *   genprob.poisson2d/3d (genprob.py:50-93)            spcg_matrix_generate
 *
 * Conventions: plain pointers and sizes only.  Pointers named d_* are device
 * pointers (any allocator: cudaMalloc, a torch tensor's data_ptr, ...); h_*
 * are host pointers.  `stream` is a cudaStream_t passed as void* (0 = legacy
 * default stream).  Every call returns an spcg_status; spcg_last_error()
 * gives the message of the most recent failure on the calling thread.
 * No call falls back to the CPU: without a usable sm_100 device every call
 * returns SPCG_ERR_CUDA (spcg_cg_cond_estimate, a host-side analysis of a
 * finished solve's CG coefficients, needs no device and computes no solve).
 */
#ifndef SPCG_B200_H
#define SPCG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPCG_ABI_VERSION 2

typedef enum {
  SPCG_OK = 0,
  SPCG_ERR_ARG = 1,          /* invalid argument (ValueError in Python)            */
  SPCG_ERR_CUDA = 2,         /* CUDA runtime failure / no device                   */
  SPCG_ERR_NOT_SPD = 3,      /* p'Ap <= 0  -> NotPositiveDefiniteError (solver.py:135) */
  SPCG_ERR_NONFINITE_ALPHA = 4, /* solver.py:138-139 */
  SPCG_ERR_NONFINITE_RESIDUAL = 5, /* solver.py:144-145 */
  SPCG_ERR_NONFINITE_BETA = 6,  /* solver.py:154-155 */
  SPCG_ERR_UNSUPPORTED = 7
} spcg_status;

/* Storage formats (core.py:57 CsrMatrix, core.py:103 SymHalfMatrix; CSC is new). */
typedef enum {
  SPCG_FMT_CSR = 0,   /* full CSR: row_start[n+1], col_idx[nnz], values[nnz]          */
  SPCG_FMT_SCSR = 1,  /* symmetric half: CSR of L+D, col<=row, diagonal last per row  */
  SPCG_FMT_CSC = 2    /* full CSC: col_start[n+1], row_idx[nnz], values[nnz]          */
} spcg_format;

/* Accumulation contract of the symmetric scatter (config.py:13-35). */
typedef enum {
  SPCG_ACC_ATOMIC = 0,      /* single pass over L+D, transpose scattered with fp64 red.add */
  SPCG_ACC_PRIVATIZED = 1   /* deterministic.  spcg_spmv: owner-computes gather over the
                               stored L^T, bitwise the reference privatized mode at
                               workers=1.  CG: resident engines gather the stored L^T
                               rows on chip; the per-pass engine makes ONE pass over L+D
                               and sums the transposed part exactly in 64-bit fixed
                               point (row_sums = 1: the stored L^T instead) */
} spcg_accumulation;

typedef struct spcg_matrix_s* spcg_matrix_t;

/* ---- matrix handles ---------------------------------------------------- */

/* Upload host CSR/SCSR/CSC arrays (int64 offsets and indices as in
 * core.INDEX_DTYPE, fp64 values).  The device copy uses int32 indices,
 * 16-byte-aligned arrays padded to a multiple of 4 entries, and a row-tile
 * table (rows binned into tiles of <= 512 rows / <= 4096 entries).
 * For SCSR the privatized-mode transpose L^T is built on the device lazily. */
int spcg_matrix_create_host(int fmt, int64_t n, int64_t nnz,
                            const int64_t* h_ptr, const int64_t* h_idx,
                            const double* h_val, spcg_matrix_t* out);

/* Same, from the u64 offsets / u32 indices of a .spcg container
 * (matio.py:162-168) without widening to int64 first. */
int spcg_matrix_create_host_u32(int fmt, int64_t n, int64_t nnz,
                                const uint64_t* h_ptr, const uint32_t* h_idx,
                                const double* h_val, spcg_matrix_t* out);

/* Generate a reference-identical matrix directly in HBM.
 * kind: 0 = poisson2d(d0,d1)      (genprob.py:50-70, diag 4, -1 per neighbour)
 *       1 = poisson3d(d0,d1,d2)   (genprob.py:73-93, diag 6)
 *       2 = stencil27(d0,d1,d2)   (27-point, diag 26, off-diagonal -1; new)
 * fmt CSR emits the full matrix, SCSR its L+D (same as core.extract_lower). */
int spcg_matrix_generate(int kind, int fmt, int64_t d0, int64_t d1, int64_t d2,
                         spcg_matrix_t* out);

/* Assemble in HBM the symmetric SPD matrix of genprob.random_spd / the
 * FEM-shaped generator (genprob.py:96-129) from the generator's own random
 * draws: m strictly-lower pairs (h_I[k] > h_J[k]) with values h_v[k] in draw
 * order, mirrored; diagonal i = the |v| of row i's entries summed in the
 * order [I-occurrences, J-occurrences] (np.bincount's order) + diag_shift.
 * Sorting, mirroring, the diagonal and the CSR / SCSR (+ L^T) / CSC layout
 * run on the device; the result is bitwise the host generator's matrix. */
int spcg_matrix_assemble_pairs(int fmt, int64_t n, int64_t m, const int64_t* h_I,
                               const int64_t* h_J, const double* h_v, double diag_shift,
                               spcg_matrix_t* out);

/* From DEVICE arrays in the .spcg layout (u64 offsets, u32 indices, fp64
 * values; matio.py:162-168): converted and validated on the device (the
 * checks of spcg_matrix_create_host); SCSR's L^T built by a device radix
 * sort.  The caller keeps ownership of its arrays (copied). */
int spcg_matrix_create_device_u32(int fmt, int64_t n, int64_t nnz, const uint64_t* d_ptr,
                                  const uint32_t* d_idx, const double* d_val, spcg_matrix_t* out);

int spcg_matrix_destroy(spcg_matrix_t m);

/* n, stored entries, format, number of row tiles, device bytes held. */
int spcg_matrix_info(spcg_matrix_t m, int64_t* n, int64_t* nnz, int* fmt,
                     int64_t* ntiles, int64_t* device_bytes);

/* Copy the device arrays back (int64 offsets/indices) — test helper. */
int spcg_matrix_download(spcg_matrix_t m, int64_t* h_ptr, int64_t* h_idx, double* h_val);

/* ---- kernel API (kernels/__init__.py:67-103) --------------------------- */

/* y = A x.  CSR: sequential per-row sums, bitwise equal to csr_gather.
 * SCSR: (L+D)x + L^T x per `accumulation`.  CSC: column scatter (atomic). */
int spcg_spmv(spcg_matrix_t m, const double* d_x, double* d_y, int accumulation,
              void* stream);

/* *d_out = sum u[i] v[i], fixed-order two-level reduction (deterministic). */
int spcg_dot(int64_t n, const double* d_u, const double* d_v, double* d_out,
             void* stream);

/* d_out = v + alpha*u elementwise (mul then add, no FMA: bitwise equal to
 * axpy_kernel); alpha == 0 copies v (_compiled.py:50-51). */
int spcg_axpy(int64_t n, double alpha, const double* d_u, const double* d_v,
              double* d_out, void* stream);

/* ---- CG solve (solver.py:65-172) -------------------------------------- */

typedef struct {
  double tol;                    /* CgOptions.tol (> 0)                        */
  int64_t max_iter;              /* <= 0 -> max(1, n)  (solver.py:96)          */
  int32_t record_history;        /* write rel residual per iteration to hist   */
  int32_t recompute_final_residual; /* default 1 (solver.py:159-162)           */
  int32_t accumulation;          /* spcg_accumulation, SCSR only               */
  int32_t engine;                /* 0 = auto: banded systems whose rows fit
                                    the co-resident clusters -> 6 (guarded,
                                    falls back to 5); other systems resident
                                    on chip -> 3; full CSR with <= 16 tiles
                                    per co-resident CTA (~1 M rows) -> 7;
                                    everything else -> 2.
                                    2 = per-pass kernels (the sharded engine),
                                    3 = persistent single-reduction CG
                                        (Chronopoulos-Gear, resident only),
                                    5 = cluster-resident single-reduction CG
                                        (banded systems),
                                    6 = engine 5's plan with pipelined CG
                                        (Ghysels-Vanroose: the SpMV overlaps
                                        the all-reduce),
                                    7 = engine 3's recurrences in one
                                        persistent kernel that streams the
                                        tiles every iteration (gather formats:
                                        CSR, privatized symmetric half).
                                    Other values: SPCG_ERR_ARG.             */
  int32_t timing;                /* per-pass engine: CUDA-event time of every
                                    SpMV pass -> result.spmv_ms / launches   */
  int32_t row_sums;              /* 0 = auto: in the streaming CG passes, lines
                                    split over 2-4 lanes sum per-lane partials
                                    + a fixed shuffle tree (deterministic,
                                    fp64-reassociated like the reference's
                                    parallel modes); 1 = every row sum in
                                    storage order (bitwise the reference's
                                    sequential sums).  SpMV entry points are
                                    always in storage order.                  */
} spcg_cg_options;

typedef struct {
  int64_t iterations;
  int32_t converged;
  int32_t status;                /* spcg_status of the solve                   */
  int64_t fail_iteration;        /* iteration k named in breakdown messages    */
  double final_relative_residual;
  double b_norm;
  double device_ms;              /* CUDA-event time of the solve on `stream`   */
  int64_t kernel_launches;       /* kernels launched by this solve             */
  double spmv_ms;                /* with opts.timing: summed SpMV-pass time    */
  int64_t spmv_launches;         /* with opts.timing: SpMV passes timed        */
  /* ABI 2 */
  int32_t engine_used;           /* engine that produced x (after auto routing
                                    and the pipelined engine's guard)         */
  int32_t fallbacks;             /* 1: auto's pipelined solve was re-run on
                                    engine 5 (cond estimate or true residual
                                    above the guard's limits)                */
  double cond_estimate;          /* engine 6: Ritz estimate of cond(A) from the
                                    CG coefficients (0 when not computed)     */
  double phase_ms[3];            /* device time split as in SolveReport.timings:
                                    [0] SpMV (with its fused dot partial),
                                    [1] reductions / scalar steps ("dot"),
                                    [2] vector updates ("axpy"); zeros when the
                                    engine did not measure them              */
} spcg_cg_result;

/* Device-resident solve.  d_x0 may be NULL (zeros).  d_x receives x.
 * d_hist (may be NULL unless record_history) must hold max_iter doubles.
 * Breakdowns are reported in result->status and returned. */
int spcg_cg_solve(spcg_matrix_t m, const double* d_b, const double* d_x0,
                  double* d_x, double* d_hist, const spcg_cg_options* opts,
                  spcg_cg_result* result, void* stream);

/* Same from host buffers: H2D of b (and x0), solve, D2H of x (and history). */
int spcg_cg_solve_host(spcg_matrix_t m, const double* h_b, const double* h_x0,
                       double* h_x, double* h_hist, const spcg_cg_options* opts,
                       spcg_cg_result* result, void* stream);

/* ---- row-sharded multi-GPU solve (new: the reference has no distribution,
 *      SPEC.md:489) ---------------------------------------- */

/* NCCL bootstrap: rank 0 makes an id, the host framework broadcasts the 128
 * bytes, every rank creates its communicator (one rank per GPU; the current
 * CUDA device is used).  nranks == 1 with id == NULL makes no NCCL
 * communicator (the collectives are no-ops); with an id it makes a real
 * one-rank NCCL communicator, so the NCCL data plane runs on one GPU too. */
#define SPCG_COMM_ID_BYTES 128
typedef struct spcg_comm_s* spcg_comm_t;
int spcg_comm_unique_id(unsigned char* out_id);
int spcg_comm_create(int nranks, int rank, const unsigned char* id, spcg_comm_t* out);
int spcg_comm_destroy(spcg_comm_t comm);

/* Host-callback communicator (no NCCL): the engine stages its collectives
 * through host memory and calls back into the host framework -- the same
 * sharded kernels over another transport (tests run two ranks as two
 * processes on ONE GPU over torch.distributed/gloo this way).  allreduce:
 * in-place sum of n doubles over all ranks.  sendrecv: for peer k send
 * send[send_off[k] .. send_off[k+1]) and receive recv[recv_off[k] ..
 * recv_off[k+1]).  Callbacks return 0 on success; they run on the calling
 * thread, after the stream has been synchronised. */
typedef int (*spcg_host_allreduce_fn)(double* buf, int64_t n, void* user);
typedef int (*spcg_host_sendrecv_fn)(int npeers, const int32_t* peers, const double* send,
                                     const int64_t* send_off, double* recv,
                                     const int64_t* recv_off, void* user);
int spcg_comm_create_host(int nranks, int rank, spcg_host_allreduce_fn allreduce,
                          spcg_host_sendrecv_fn sendrecv, void* user, spcg_comm_t* out);

/* Rows [row0,row1) of an n_global-row matrix, GLOBAL column ids (int64 host
 * arrays; ptr may be a slice of a global offsets array).  SCSR: A = the L+D
 * rows, B = the same rows of L^T (strict upper), needed for sharded solves. */
int spcg_matrix_create_rows(int fmt, int64_t n_global, int64_t row0, int64_t row1,
                            int64_t nnzA, const int64_t* ptrA, const int64_t* idxA,
                            const double* valA, int64_t nnzB, const int64_t* ptrB,
                            const int64_t* idxB, const double* valB, spcg_matrix_t* out);
/* Same rows of an in-HBM generated stencil (kinds of spcg_matrix_generate). */
int spcg_matrix_generate_rows(int kind, int fmt, int64_t d0, int64_t d1, int64_t d2,
                              int64_t row0, int64_t row1, spcg_matrix_t* out);
/* Remap columns: owned -> [0,nloc), others -> nloc + rank in the sorted halo
 * list.  After this the handle gathers from extended vectors of nloc+nhalo. */
int spcg_matrix_localize(spcg_matrix_t m, int64_t* nhalo);
int spcg_matrix_halo(spcg_matrix_t m, int64_t* halo_global_cols);

/* One rank's share of a row-sharded CG solve (solver.py:65-172 semantics on
 * the global system).  Halo plan: peers[npeers] (ranks, ascending);
 * recv_off[npeers+1] partitions the halo list by owner; send_off[npeers+1]
 * partitions send_idx (local rows each peer needs).  Per iteration: pack +
 * ncclSend/ncclRecv of the halo, pass A, ncclAllReduce(p.q), pass B,
 * ncclAllReduce(r.r); scalars stay on the device.  d_b/d_x0/d_x are local
 * (nloc); d_hist (max_iter) is written identically on every rank. */
int spcg_dist_cg_solve(spcg_matrix_t local, spcg_comm_t comm, int npeers,
                       const int32_t* peers, const int64_t* recv_off,
                       const int64_t* send_off, const int32_t* send_idx,
                       const double* d_b, const double* d_x0, double* d_x, double* d_hist,
                       const spcg_cg_options* opts, spcg_cg_result* result, void* stream);

/* ---- device-initiated transport (no host collective per iteration) -------
 * A per-rank plan of the same halo layout as spcg_dist_cg_solve.  Peers write
 * straight into this rank's memory: the two scalar all-reduces of every
 * iteration go through epoch-tagged mailboxes (each rank's last CTA of a
 * reducing pass posts its partial to every rank, polls its own mailbox and
 * sums the partials in rank order), the halo of p is stored by the pass that
 * computes it into the neighbours' p_ext (remote stores over NVLink), and the
 * single-pass SCSR scatter sends its transposed contributions to their
 * owners as remote fp64 reds.  Bootstrap: every rank exports a blob (CUDA IPC
 * handles of the buffers peers write, its row layout), the host framework
 * all-gathers the nranks blobs in rank order, every rank connects.  Ranks of
 * ONE process on ONE device are connected by plain pointers and can be
 * solved together in one launch per pass (spcg_dist_group_solve: "virtual
 * ranks", how the protocol is tested on a single GPU). */
#define SPCG_P2P_BLOB_BYTES 1024
typedef struct spcg_dist_plan_s* spcg_dist_plan_t;
int spcg_dist_plan_create(spcg_matrix_t local, int rank, int nranks, int npeers,
                          const int32_t* peers, const int64_t* recv_off, const int64_t* send_off,
                          const int32_t* send_idx, spcg_dist_plan_t* out);
int spcg_dist_plan_destroy(spcg_dist_plan_t plan);
int spcg_dist_plan_export(spcg_dist_plan_t plan, unsigned char* blob /* SPCG_P2P_BLOB_BYTES */);
int spcg_dist_plan_connect(spcg_dist_plan_t plan,
                           const unsigned char* blobs /* nranks x SPCG_P2P_BLOB_BYTES */);
/* One rank's share (one process per GPU), same semantics as spcg_dist_cg_solve. */
int spcg_dist_plan_solve(spcg_dist_plan_t plan, const double* d_b, const double* d_x0, double* d_x,
                         double* d_hist, const spcg_cg_options* opts, spcg_cg_result* result,
                         void* stream);
/* All nranks plans of this process (same device): every pass is ONE launch
 * over all ranks' data.  d_b / d_x0 (NULL or per rank) / d_x: per-rank
 * device vectors; d_hist: rank 0's history; results[nranks]. */
int spcg_dist_group_solve(int nranks, spcg_dist_plan_t* plans, const double* const* d_b,
                          const double* const* d_x0, double* const* d_x, double* d_hist,
                          const spcg_cg_options* opts, spcg_cg_result* results, void* stream);

/* ---- library ------------------------------------------------------------ */

const char* spcg_last_error(void);
int spcg_abi_version(void);
/* SMs of the current device and the cooperative grid the solver uses. */
int spcg_device_info(int* sm_count, int* coop_grid, int* cc_major, int* cc_minor);
/* Ritz estimate of cond(A) from k CG step coefficients, h_ab[2j] = alpha_j,
 * h_ab[2j+1] = beta_j (the beta that formed p_j; beta_0 ignored):
 * theta_max / theta_min of the Lanczos tridiagonal, ~1e-3 relative.  The
 * engine-6 auto guard's estimate (spcg_cg_result.cond_estimate); host only,
 * needs no device.  *cond = 0 when k < 2 or a coefficient is not positive. */
int spcg_cg_cond_estimate(const double* h_ab, int64_t k, double* cond);

#ifdef __cplusplus
}
#endif
#endif /* SPCG_B200_H */
