// spcg_b200.cu — host runtime behind include/spcg_b200.h: matrix handles
// (upload, int32 narrowing, row tiling, L^T construction, in-HBM generators),
// solver workspaces, kernel launches and the extern "C" entry points.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <dlfcn.h>
#include <unistd.h>
#include <cstddef>
#include <nccl.h>

#include "../../include/spcg_b200.h"
#include "cg.cuh"
#include "cg1.cuh"
#include "clus.cuh"
#include "clus_pipe.cuh"
#include "dist.cuh"
#include "ops.cuh"
#include "assemble.cuh"

using namespace spcg;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

// A handle's arrays live on the device that was current at its creation;
// using it from another device would hand foreign pointers to the kernels.
int on_device(int device) {
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess) return fail(SPCG_ERR_CUDA, "cudaGetDevice failed");
  if (cur != device)
    return fail(SPCG_ERR_ARG, "matrix handle lives on device " + std::to_string(device) +
                                  " but the current device is " + std::to_string(cur));
  return SPCG_OK;
}

#define CUDA_TRY(expr)                                                                  \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      return fail(SPCG_ERR_CUDA, std::string(#expr " failed: ") + cudaGetErrorString(_e)); \
  } while (0)

struct DevInfo {
  int device = -1;
  int sms = 0;
  int major = 0, minor = 0;
  int coop_res = 0;     // co-resident CTAs of the resident CG kernel
  int spmv_grid = 0;
  // stream-ordered scratch (dot partials): a library-owned pool that keeps
  // its memory (the default pool's release threshold of 0 would hand the
  // pages back at every synchronize and re-map them, ~ms, at the next call)
  cudaMemPool_t pool = nullptr;
};

std::mutex g_dev_mutex;
DevInfo g_dev[64];

template <class K>
int occupancy(K kernel, int* blocks, size_t smem = sizeof(Smem)) {
  CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, kernel, kBlock, smem));
  return SPCG_OK;
}
constexpr size_t kSmemRes = sizeof(Smem) + kResProdBytes;

int dev_info(DevInfo** out) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return fail(SPCG_ERR_CUDA, "device ordinal out of range");
  std::lock_guard<std::mutex> lk(g_dev_mutex);
  DevInfo& d = g_dev[dev];
  if (d.device != dev) {
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, dev));
    if (prop.major < 10)
      return fail(SPCG_ERR_CUDA, "spcg_b200 needs an sm_100 (Blackwell) device, found sm_" +
                                     std::to_string(prop.major) + std::to_string(prop.minor));
    if (!prop.cooperativeLaunch) return fail(SPCG_ERR_CUDA, "device lacks cooperative launch");
    d.sms = prop.multiProcessorCount;
    d.major = prop.major;
    d.minor = prop.minor;
    int br = 0, bp = 0, t = 0;
    int rc;
    // engine 3's resident kernel: every instantiation shares one shape
    if ((rc = occupancy(cg1_kernel<K_CSR>, &br, kSmemRes))) return rc;
    if ((rc = occupancy(cg1_kernel<K_SCSR_ATOMIC>, &t, kSmemRes))) return rc;
    br = std::min(br, t);
    if ((rc = occupancy(cg1_kernel<K_SCSR_PRIV>, &t, kSmemRes))) return rc;
    br = std::min(br, t);
    if ((rc = occupancy(cg1_kernel<K_CSC>, &t, kSmemRes))) return rc;
    br = std::min(br, t);
    if ((rc = occupancy(spmv_kernel<K_CSR>, &bp))) return rc;
    if ((rc = occupancy(spmv_kernel<K_SCSR_ATOMIC>, &t))) return rc;
    if ((rc = occupancy(spmv_kernel<K_SCSR_PRIV>, &t))) return rc;
    if ((rc = occupancy(spmv_kernel<K_CSC>, &t))) return rc;
    // (these calls also raise each kernel's dynamic shared-memory limit)
    if ((rc = occupancy(spmv_kernel<K_CSR, true>, &t))) return rc;
#define SPCG_OCC_DIST(F, W)                                                    \
  if ((rc = occupancy(dist_spmv_pq<F, W, 0>, &t))) return rc;                  \
  if ((rc = occupancy(dist_spmv_pq<F, W, 1>, &t))) return rc;                  \
  if ((rc = occupancy(dist_spmv_pq<F, W, 2>, &t))) return rc;                  \
  if ((rc = occupancy(dist_spmv<F, W, 0>, &t))) return rc;                     \
  if ((rc = occupancy(dist_spmv<F, W, 1>, &t))) return rc;                     \
  if ((rc = occupancy(dist_spmv<F, W, 2>, &t))) return rc;
    SPCG_OCC_DIST(K_CSR, false)
    SPCG_OCC_DIST(K_CSR, true)
    SPCG_OCC_DIST(K_SCSR_PRIV, false)
    SPCG_OCC_DIST(K_SCSR_ATOMIC, false)
    SPCG_OCC_DIST(K_CSC, false)
    SPCG_OCC_DIST(K_SCSR_FIX, false)
#undef SPCG_OCC_DIST
    if (br < 1 || bp < 1) return fail(SPCG_ERR_CUDA, "CG kernel does not fit on an SM");
    d.coop_res = std::min(br * d.sms, 32 * kPollWarps * kPollPer);
    d.spmv_grid = bp * d.sms;
    cudaMemPoolProps pp = {};
    pp.allocType = cudaMemAllocationTypePinned;
    pp.handleTypes = cudaMemHandleTypeNone;
    pp.location.type = cudaMemLocationTypeDevice;
    pp.location.id = dev;
    CUDA_TRY(cudaMemPoolCreate(&d.pool, &pp));
    unsigned long long keep = ~0ULL;
    CUDA_TRY(cudaMemPoolSetAttribute(d.pool, cudaMemPoolAttrReleaseThreshold, &keep));
    d.device = dev;
  }
  *out = &d;
  return SPCG_OK;
}

struct Seg {
  int* ptr = nullptr;
  int* idx = nullptr;
  double* val = nullptr;
  long long nnz = 0;
};

struct Tiles {
  int4* desc = nullptr;
  int2* descB = nullptr;
  int2* win = nullptr;  // leading-edge prefetch windows
  int ntiles = 0;
};

struct Workspace {
  int n = -1;
  int slots_g = 0;
  double* r = nullptr;
  double* p0 = nullptr;
  double* p1 = nullptr;
  double* q = nullptr;
  double* part = nullptr;
  unsigned long long* slots = nullptr;
  CgDevResult* res = nullptr;
  CgDevResult* h_res = nullptr;  // pinned
  double* cg1 = nullptr;         // single-reduction engine: R[2], S[2], W[3]
  // host-API staging
  double* b = nullptr;
  double* x = nullptr;
  double* x0 = nullptr;
  double* hist = nullptr;
  long long hist_cap = 0;
  double* coef = nullptr;  // engine-6 guard: (alpha, beta) per update
  long long coef_cap = 0;
  double* h_coef = nullptr;  // pinned: the first kCoefHost pairs come back with the result
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t ev_res = nullptr;  // after the result copy (guarded solves)
  // host-API solve: x's destination, so a guarded engine-6 solve can start
  // x's copy before its host-side guard runs (x_early_done: it did)
  double* h_x_early = nullptr;
  bool x_early_done = false;
};

// Workspace of the row-sharded (per-pass) engine.
struct DistWorkspace {
  long long next = -1;  // nloc + nhalo
  double* r_ext = nullptr;
  double* p_ext[2] = {nullptr, nullptr};
  double* tmp_ext = nullptr;
  double* q = nullptr;
  double* part = nullptr;
  StepState* S = nullptr;
  StepState* h_S = nullptr;  // pinned
  StepState* h_Sc[2] = {nullptr, nullptr};  // pinned, per in-flight chunk
  cudaEvent_t cev[2] = {nullptr, nullptr};  // chunk copies done
  double* send_buf = nullptr;
  long long send_cap = 0;
  int* send_idx = nullptr;
  long long send_idx_cap = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // [chunk buffer][A0 A1 B0 B1 C0 C1][iteration]: per-pass timing (opts.timing:
  // 1 = pass A only, 2 = all three passes for the spmv/dot/axpy split)
  cudaEvent_t tev[2][6][16] = {};
  DistArgs* args = nullptr;  // device copy of the rank's DistArgs (host transports)
  unsigned long long* ytx = nullptr;  // K_SCSR_FIX: fixed-point transposed part (n words)
  long long ytx_n = 0;
};

}  // namespace

// Cluster-resident engine plan (clus.cuh), built once per handle on demand.
struct ClusPlan {
  bool built = false;  // plan attempted
  bool ok = false;     // feasible
  std::string why;     // reason when not feasible
  bool two = false;    // two segments per row (SCSR: L+D, L^T)
  int C = 0;           // CTAs (grid)
  int cs = 0;          // cluster size; K = C / cs clusters
  double* ghalo = nullptr;              // K > 1: [2][C][hcap]
  unsigned long long* gslots = nullptr; // K > 1: [2][K][4]
  ClusCta* ctas = nullptr;
  ClusSlice* slices = nullptr;
  ClusSend* sends = nullptr;
  int2* rowmeta = nullptr;
  double* gval = nullptr;
  unsigned short* gcol = nullptr;
  int off_rwin = 0, off_shalo = 0, off_whalo = 0, off_val = 0, off_col = 0, hcap = 1;
  size_t smem = 0;
  long long resident = 0, streamed = 0;  // entries (stats)
  int max_slices = 0;                     // SELL-32 slices of the fullest CTA
  int max_width = 0;                      // longest row (entries) of the plan
  void* arena = nullptr;                  // the one allocation the pointers above live in
};

struct spcg_matrix_s {
  int fmt = 0;
  int n = 0;          // lines held (all rows, or the rows block of a shard)
  long long nnz = 0;
  int device = 0;
  Seg A, B;
  bool hasB = false;
  Tiles t1, t2;
  Tiles t1w;  // wide tiles (<= kWideLines lines) for the streaming passes; short-row CSR only
  long long bytes = 0;
  Workspace ws;
  // row block of a sharded matrix (rows [row0,row1) of an n_global system)
  bool is_rows = false;
  bool localized = false;
  long long row0 = 0, row1 = 0, n_global = 0;
  std::vector<long long> halo;  // sorted global ids of the halo columns
  DistWorkspace dw;
  ClusPlan cp;
  int tx_eM = -100000;  // K_SCSR_FIX: ceil(log2(max_j sum_i |a_ij|)) (unset: -100000)
  std::mutex mu;  // one solve at a time per handle (workspace reuse)
};

struct spcg_comm_s {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  // host-callback transport (spcg_comm_create_host): data staged through
  // host memory, collectives done by the caller's framework
  spcg_host_allreduce_fn host_ar = nullptr;
  spcg_host_sendrecv_fn host_sr = nullptr;
  void* host_user = nullptr;
};

namespace {

#include "host_matrix.cuh"
#include "host_cluster.cuh"
#include "host_solve.cuh"
#include "host_assemble.cuh"
#include "host_dist.cuh"

}  // namespace

// ============================================================================
extern "C" {

const char* spcg_last_error(void) { return g_last_error.c_str(); }
int spcg_abi_version(void) { return SPCG_ABI_VERSION; }

int spcg_device_info(int* sm_count, int* coop_grid, int* cc_major, int* cc_minor) {
  DevInfo* d;
  int rc;
  if ((rc = dev_info(&d))) return rc;
  if (sm_count) *sm_count = d->sms;
  if (coop_grid) *coop_grid = d->coop_res;
  if (cc_major) *cc_major = d->major;
  if (cc_minor) *cc_minor = d->minor;
  return SPCG_OK;
}

int spcg_matrix_create_host(int fmt, int64_t n, int64_t nnz, const int64_t* h_ptr,
                            const int64_t* h_idx, const double* h_val, spcg_matrix_t* out) {
  if (!out) return fail(SPCG_ERR_ARG, "null out");
  return create_from_host(fmt, n, nnz, h_ptr, h_idx, h_val, out);
}

int spcg_matrix_create_host_u32(int fmt, int64_t n, int64_t nnz, const uint64_t* h_ptr,
                                const uint32_t* h_idx, const double* h_val, spcg_matrix_t* out) {
  if (!out) return fail(SPCG_ERR_ARG, "null out");
  return create_from_host(fmt, n, nnz, h_ptr, h_idx, h_val, out);
}

int spcg_matrix_generate(int kind, int fmt, int64_t d0, int64_t d1, int64_t d2,
                         spcg_matrix_t* out) {
  if (!out) return fail(SPCG_ERR_ARG, "null out");
  if (kind < 0 || kind > 2) return fail(SPCG_ERR_ARG, "unknown generator kind");
  if (fmt != SPCG_FMT_CSR && fmt != SPCG_FMT_SCSR && fmt != SPCG_FMT_CSC)
    return fail(SPCG_ERR_ARG, "unknown format");
  if (kind == 0) d2 = 1;
  if (d0 < 1 || d1 < 1 || d2 < 1) return fail(SPCG_ERR_ARG, "extents must be >= 1");
  const long long n = d0 * d1 * d2;
  if (n >= (1LL << 31) - 16) return fail(SPCG_ERR_UNSUPPORTED, "grid exceeds int32 rows");
  DevInfo* d;
  int rc;
  if ((rc = dev_info(&d))) return rc;
  spcg_matrix_s* m = new spcg_matrix_s();
  m->fmt = fmt;
  m->n = (int)n;
  CUDA_TRY(cudaGetDevice(&m->device));
  std::vector<int> ptr, tptr;
  // CSC of a symmetric stencil is its CSR
  const int part = fmt == SPCG_FMT_SCSR ? 1 : 0;
  if ((rc = gen_seg(kind, part, 0, n, (int)d0, (int)d1, (int)d2, m->A, ptr, &m->bytes)) ||
      (rc = finish_matrix(m, ptr, nullptr, nullptr, true))) {
    free_matrix(m);
    delete m;
    return rc;
  }
  m->nnz = m->A.nnz;
  if (fmt == SPCG_FMT_SCSR) {
    if ((rc = gen_seg(kind, 2, 0, n, (int)d0, (int)d1, (int)d2, m->B, tptr, &m->bytes)) ||
        (rc = finish_transpose(m, ptr, tptr, nullptr, nullptr, true))) {
      free_matrix(m);
      delete m;
      return rc;
    }
  }
  if ((rc = refresh_windows(m))) {
    free_matrix(m);
    delete m;
    return rc;
  }
  *out = m;
  return SPCG_OK;
}

int spcg_matrix_assemble_pairs(int fmt, int64_t n, int64_t m, const int64_t* h_I,
                               const int64_t* h_J, const double* h_v, double diag_shift,
                               spcg_matrix_t* out) {
  if (!out) return fail(SPCG_ERR_ARG, "null out");
  return assemble_pairs(fmt, n, m, h_I, h_J, h_v, diag_shift, out);
}

int spcg_matrix_create_device_u32(int fmt, int64_t n, int64_t nnz, const uint64_t* d_ptr,
                                  const uint32_t* d_idx, const double* d_val, spcg_matrix_t* out) {
  if (!out) return fail(SPCG_ERR_ARG, "null out");
  return create_from_device(fmt, n, nnz, d_ptr, d_idx, d_val, out);
}

int spcg_matrix_destroy(spcg_matrix_t m) {
  if (!m) return SPCG_OK;
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != m->device) cudaSetDevice(m->device);
  cudaDeviceSynchronize();
  free_matrix(m);
  if (cur != m->device) cudaSetDevice(cur);
  delete m;
  return SPCG_OK;
}

int spcg_matrix_info(spcg_matrix_t m, int64_t* n, int64_t* nnz, int* fmt, int64_t* ntiles,
                     int64_t* device_bytes) {
  if (!m) return fail(SPCG_ERR_ARG, "null matrix");
  if (n) *n = m->n;
  if (nnz) *nnz = m->nnz;
  if (fmt) *fmt = m->fmt;
  if (ntiles) *ntiles = m->t1.ntiles;
  if (device_bytes) *device_bytes = m->bytes;
  return SPCG_OK;
}

int spcg_matrix_download(spcg_matrix_t m, int64_t* h_ptr, int64_t* h_idx, double* h_val) {
  if (!m) return fail(SPCG_ERR_ARG, "null matrix");
  std::vector<int> p((size_t)m->n + 1), ix((size_t)m->nnz);
  CUDA_TRY(cudaMemcpy(p.data(), m->A.ptr, sizeof(int) * p.size(), cudaMemcpyDeviceToHost));
  if (m->nnz) {
    CUDA_TRY(cudaMemcpy(ix.data(), m->A.idx, sizeof(int) * ix.size(), cudaMemcpyDeviceToHost));
    if (h_val)
      CUDA_TRY(cudaMemcpy(h_val, m->A.val, sizeof(double) * (size_t)m->nnz, cudaMemcpyDeviceToHost));
  }
  if (h_ptr)
    for (size_t i = 0; i < p.size(); ++i) h_ptr[i] = p[i];
  if (h_idx)
    for (size_t i = 0; i < ix.size(); ++i) h_idx[i] = ix[i];
  return SPCG_OK;
}

int spcg_spmv(spcg_matrix_t m, const double* d_x, double* d_y, int accumulation, void* stream) {
  if (!m || (m->n > 0 && (!d_x || !d_y))) return fail(SPCG_ERR_ARG, "null argument");
  if (int rc = on_device(m->device)) return rc;
  return do_spmv(m, d_x, d_y, accumulation, (cudaStream_t)stream);
}

int spcg_dot(int64_t n, const double* d_u, const double* d_v, double* d_out, void* stream) {
  DevInfo* d;
  int rc;
  if ((rc = dev_info(&d))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0 || !d_out) return fail(SPCG_ERR_ARG, "bad dot arguments");
  if (n == 0) {
    CUDA_TRY(cudaMemsetAsync(d_out, 0, sizeof(double), st));
    return SPCG_OK;
  }
  // per-call partials, stream-ordered (dots in flight on several streams,
  // or on several devices, never share a buffer)
  const int nb = (int)std::min<long long>(2LL * d->sms, (n + kBlock - 1) / kBlock);
  double* part = nullptr;
  CUDA_TRY(cudaMallocFromPoolAsync((void**)&part, sizeof(double) * (size_t)nb, d->pool, st));
  dot_partial_kernel<<<nb, kBlock, 0, st>>>(n, d_u, d_v, part);
  CUDA_TRY(cudaGetLastError());
  dot_final_kernel<<<1, kBlock, 0, st>>>(nb, part, d_out);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaFreeAsync(part, st));
  return SPCG_OK;
}

int spcg_axpy(int64_t n, double alpha, const double* d_u, const double* d_v, double* d_out,
              void* stream) {
  DevInfo* d;
  int rc;
  if ((rc = dev_info(&d))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0) return fail(SPCG_ERR_ARG, "bad axpy arguments");
  if (n == 0) return SPCG_OK;
  if (alpha == 0.0) {
    if (d_out != d_v)
      CUDA_TRY(cudaMemcpyAsync(d_out, d_v, sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, st));
    return SPCG_OK;
  }
  const int nb = (int)std::min<long long>(8LL * d->sms, (n + kBlock - 1) / kBlock);
  axpy_kernel<<<nb, kBlock, 0, st>>>(n, alpha, d_u, d_v, d_out);
  CUDA_TRY(cudaGetLastError());
  return SPCG_OK;
}

int spcg_cg_solve(spcg_matrix_t m, const double* d_b, const double* d_x0, double* d_x,
                  double* d_hist, const spcg_cg_options* opts, spcg_cg_result* result,
                  void* stream) {
  if (!m || !opts || !result) return fail(SPCG_ERR_ARG, "null argument");
  if (m->n > 0 && (!d_b || !d_x)) return fail(SPCG_ERR_ARG, "null vector");
  if (int rc = on_device(m->device)) return rc;
  std::lock_guard<std::mutex> lk(m->mu);
  return do_cg(m, d_b, d_x0, d_x, d_hist, opts, result, (cudaStream_t)stream);
}

int spcg_cg_solve_host(spcg_matrix_t m, const double* h_b, const double* h_x0, double* h_x,
                       double* h_hist, const spcg_cg_options* opts, spcg_cg_result* result,
                       void* stream) {
  if (!m || !opts || !result) return fail(SPCG_ERR_ARG, "null argument");
  if (m->n > 0 && (!h_b || !h_x)) return fail(SPCG_ERR_ARG, "null vector");
  if (int rc = on_device(m->device)) return rc;
  std::lock_guard<std::mutex> lk(m->mu);
  cudaStream_t st = (cudaStream_t)stream;
  Workspace& w = m->ws;
  int rc;
  const size_t vb = sizeof(double) * (size_t)std::max(1, m->n);
  if (!w.b) {
    if ((rc = dmalloc((void**)&w.b, vb, nullptr))) return rc;
    if ((rc = dmalloc((void**)&w.x, vb, nullptr))) return rc;
    if ((rc = dmalloc((void**)&w.x0, vb, nullptr))) return rc;
  }
  const long long max_iter = opts->max_iter > 0 ? opts->max_iter : std::max(1, m->n);
  if (opts->record_history && w.hist_cap < max_iter) {
    if (w.hist) cudaFree(w.hist);
    w.hist = nullptr;
    if ((rc = dmalloc((void**)&w.hist, sizeof(double) * (size_t)max_iter, nullptr))) return rc;
    w.hist_cap = max_iter;
  }
  const size_t nb = sizeof(double) * (size_t)m->n;
  static const bool etime = getenv("SPCG_E2E_TIMING") != nullptr;  // (dev)
  const auto th0 = std::chrono::steady_clock::now();
  if (m->n) CUDA_TRY(cudaMemcpyAsync(w.b, h_b, nb, cudaMemcpyHostToDevice, st));
  if (h_x0 && m->n) CUDA_TRY(cudaMemcpyAsync(w.x0, h_x0, nb, cudaMemcpyHostToDevice, st));
  const auto th1 = std::chrono::steady_clock::now();
  w.h_x_early = m->n ? h_x : nullptr;
  w.x_early_done = false;
  rc = do_cg(m, w.b, h_x0 ? w.x0 : nullptr, w.x, opts->record_history ? w.hist : nullptr, opts,
             result, st);
  w.h_x_early = nullptr;
  if (rc != SPCG_OK && rc != SPCG_ERR_NOT_SPD && rc != SPCG_ERR_NONFINITE_ALPHA &&
      rc != SPCG_ERR_NONFINITE_RESIDUAL && rc != SPCG_ERR_NONFINITE_BETA) {
    cudaStreamSynchronize(st);  // no copy into h_x (an early one) outlives the call
    w.x_early_done = false;
    return rc;
  }
  const std::string err = g_last_error;
  if (m->n && !w.x_early_done) CUDA_TRY(cudaMemcpyAsync(h_x, w.x, nb, cudaMemcpyDeviceToHost, st));
  w.x_early_done = false;
  if (opts->record_history && h_hist && result->iterations > 0)
    CUDA_TRY(cudaMemcpyAsync(h_hist, w.hist, sizeof(double) * (size_t)result->iterations,
                             cudaMemcpyDeviceToHost, st));
  const auto th2 = std::chrono::steady_clock::now();
  CUDA_TRY(cudaStreamSynchronize(st));
  if (etime) {
    auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
    fprintf(stderr, "[spcg e2e] host call: h2d enqueue %.1f, to x-copy %.1f x-copy+sync %.1f us\n",
            us(th0, th1), us(th0, th2),
            us(th2, std::chrono::steady_clock::now()));
  }
  g_last_error = err;
  return rc;
}

// ---- row-sharded multi-GPU solve ------------------------------------------
int spcg_comm_unique_id(unsigned char* out) {
  if (!out) return fail(SPCG_ERR_ARG, "null out");
  NcclApi& N = nccl();
  if (!N.ok) return fail(SPCG_ERR_CUDA, N.err);
  ncclUniqueId id;
  NCCL_TRY(N.GetUniqueId(&id));
  memcpy(out, id.internal, SPCG_COMM_ID_BYTES);
  return SPCG_OK;
}

int spcg_comm_create(int nranks, int rank, const unsigned char* id_bytes, spcg_comm_t* out) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks) return fail(SPCG_ERR_ARG, "bad comm args");
  spcg_comm_s* c = new spcg_comm_s();
  c->nranks = nranks;
  c->rank = rank;
  // nranks == 1 with a NULL id: no NCCL (collectives are no-ops); with an id
  // a real one-rank NCCL communicator, so the NCCL calls and their stream
  // ordering execute even on one GPU
  if (nranks > 1 || id_bytes) {
    NcclApi& N = nccl();
    if (!N.ok) {
      delete c;
      return fail(SPCG_ERR_CUDA, N.err);
    }
    if (!id_bytes) {
      delete c;
      return fail(SPCG_ERR_ARG, "null unique id");
    }
    ncclUniqueId id;
    memcpy(id.internal, id_bytes, SPCG_COMM_ID_BYTES);
    ncclResult_t r = N.CommInitRank(&c->comm, nranks, id, rank);
    if (r != ncclSuccess) {
      delete c;
      return fail(SPCG_ERR_CUDA, std::string("ncclCommInitRank: ") + N.GetErrorString(r));
    }
  }
  *out = c;
  return SPCG_OK;
}

int spcg_comm_create_host(int nranks, int rank, spcg_host_allreduce_fn allreduce,
                          spcg_host_sendrecv_fn sendrecv, void* user, spcg_comm_t* out) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks || !allreduce || !sendrecv)
    return fail(SPCG_ERR_ARG, "bad host comm args");
  spcg_comm_s* c = new spcg_comm_s();
  c->nranks = nranks;
  c->rank = rank;
  c->host_ar = allreduce;
  c->host_sr = sendrecv;
  c->host_user = user;
  *out = c;
  return SPCG_OK;
}

int spcg_comm_destroy(spcg_comm_t c) {
  if (!c) return SPCG_OK;
  if (c->comm) nccl().CommDestroy(c->comm);
  delete c;
  return SPCG_OK;
}

int spcg_matrix_create_rows(int fmt, int64_t n_global, int64_t row0, int64_t row1, int64_t nnzA,
                            const int64_t* ptrA, const int64_t* idxA, const double* valA,
                            int64_t nnzB, const int64_t* ptrB, const int64_t* idxB,
                            const double* valB, spcg_matrix_t* out) {
  if (!out) return fail(SPCG_ERR_ARG, "null out");
  int rc;
  if ((rc = check_csr_host(fmt, n_global, nnzA))) return rc;
  if (fmt == SPCG_FMT_CSC) return fail(SPCG_ERR_UNSUPPORTED, "row blocks are CSR / SCSR");
  if (row0 < 0 || row1 < row0 || row1 > n_global) return fail(SPCG_ERR_ARG, "bad row range");
  const int nrows = (int)(row1 - row0);
  std::vector<int> pA, iA, pB, iB;
  if ((rc = seg_from_host(nrows, ptrA, idxA, nnzA, n_global, pA, iA))) return rc;
  const bool hasB = fmt == SPCG_FMT_SCSR && ptrB != nullptr;
  if (hasB && (rc = seg_from_host(nrows, ptrB, idxB, nnzB, n_global, pB, iB))) return rc;
  DevInfo* d;
  if ((rc = dev_info(&d))) return rc;
  spcg_matrix_s* m = new spcg_matrix_s();
  m->fmt = fmt;
  m->n = nrows;
  m->nnz = nnzA;
  m->is_rows = true;
  m->row0 = row0;
  m->row1 = row1;
  m->n_global = n_global;
  CUDA_TRY(cudaGetDevice(&m->device));
  if ((rc = finish_matrix(m, pA, iA.data(), valA, false)) ||
      (hasB && (rc = finish_transpose(m, pA, pB, iB.data(), valB, false)))) {
    free_matrix(m);
    delete m;
    return rc;
  }
  if ((rc = refresh_windows(m))) {
    free_matrix(m);
    delete m;
    return rc;
  }
  *out = m;
  return SPCG_OK;
}

int spcg_matrix_generate_rows(int kind, int fmt, int64_t d0, int64_t d1, int64_t d2, int64_t row0,
                              int64_t row1, spcg_matrix_t* out) {
  if (!out) return fail(SPCG_ERR_ARG, "null out");
  if (kind < 0 || kind > 2) return fail(SPCG_ERR_ARG, "unknown generator kind");
  if (fmt != SPCG_FMT_CSR && fmt != SPCG_FMT_SCSR) return fail(SPCG_ERR_ARG, "row blocks are CSR / SCSR");
  if (kind == 0) d2 = 1;
  if (d0 < 1 || d1 < 1 || d2 < 1) return fail(SPCG_ERR_ARG, "extents must be >= 1");
  const long long N = d0 * d1 * d2;
  if (N >= (1LL << 31) - 16) return fail(SPCG_ERR_UNSUPPORTED, "grid exceeds int32 rows");
  if (row0 < 0 || row1 < row0 || row1 > N) return fail(SPCG_ERR_ARG, "bad row range");
  DevInfo* d;
  int rc;
  if ((rc = dev_info(&d))) return rc;
  spcg_matrix_s* m = new spcg_matrix_s();
  m->fmt = fmt;
  m->n = (int)(row1 - row0);
  m->is_rows = true;
  m->row0 = row0;
  m->row1 = row1;
  m->n_global = N;
  CUDA_TRY(cudaGetDevice(&m->device));
  std::vector<int> ptr, tptr;
  const int part = fmt == SPCG_FMT_SCSR ? 1 : 0;
  if ((rc = gen_seg(kind, part, row0, m->n, (int)d0, (int)d1, (int)d2, m->A, ptr, &m->bytes)) ||
      (rc = finish_matrix(m, ptr, nullptr, nullptr, true))) {
    free_matrix(m);
    delete m;
    return rc;
  }
  m->nnz = m->A.nnz;
  if (fmt == SPCG_FMT_SCSR) {
    if ((rc = gen_seg(kind, 2, row0, m->n, (int)d0, (int)d1, (int)d2, m->B, tptr, &m->bytes)) ||
        (rc = finish_transpose(m, ptr, tptr, nullptr, nullptr, true))) {
      free_matrix(m);
      delete m;
      return rc;
    }
  }
  if ((rc = refresh_windows(m))) {
    free_matrix(m);
    delete m;
    return rc;
  }
  *out = m;
  return SPCG_OK;
}

int spcg_matrix_localize(spcg_matrix_t m, int64_t* nhalo) {
  if (!m) return fail(SPCG_ERR_ARG, "null matrix");
  if (int rc = on_device(m->device)) return rc;
  std::lock_guard<std::mutex> lk(m->mu);
  int rc = localize(m);
  if (rc) return rc;
  if (nhalo) *nhalo = (int64_t)m->halo.size();
  return SPCG_OK;
}

int spcg_matrix_halo(spcg_matrix_t m, int64_t* halo_cols) {
  if (!m) return fail(SPCG_ERR_ARG, "null matrix");
  if (!m->localized) return fail(SPCG_ERR_ARG, "matrix is not localized");
  for (size_t k = 0; k < m->halo.size(); ++k) halo_cols[k] = m->halo[k];
  return SPCG_OK;
}

int spcg_dist_cg_solve(spcg_matrix_t local, spcg_comm_t comm, int npeers, const int32_t* peers,
                       const int64_t* recv_off, const int64_t* send_off, const int32_t* send_idx,
                       const double* d_b, const double* d_x0, double* d_x, double* d_hist,
                       const spcg_cg_options* opts, spcg_cg_result* result, void* stream) {
  if (!local || !opts || !result) return fail(SPCG_ERR_ARG, "null argument");
  if (npeers < 0 || (npeers > 0 && (!peers || !recv_off || !send_off)))
    return fail(SPCG_ERR_ARG, "bad halo plan");
  if (int rc = on_device(local->device)) return rc;
  std::lock_guard<std::mutex> lk(local->mu);
  return do_dist_cg(local, comm, npeers, peers, recv_off, send_off, send_idx, d_b, d_x0, d_x,
                    d_hist, opts, result, (cudaStream_t)stream);
}

int spcg_dist_plan_create(spcg_matrix_t local, int rank, int nranks, int npeers,
                          const int32_t* peers, const int64_t* recv_off, const int64_t* send_off,
                          const int32_t* send_idx, spcg_dist_plan_t* out) {
  if (!local || !out) return fail(SPCG_ERR_ARG, "null argument");
  if (int rc = on_device(local->device)) return rc;
  std::lock_guard<std::mutex> lk(local->mu);
  return plan_create(local, rank, nranks, npeers, peers, recv_off, send_off, send_idx, out);
}

int spcg_dist_plan_destroy(spcg_dist_plan_t plan) {
  if (!plan) return SPCG_OK;
  cudaDeviceSynchronize();
  free_plan(plan);
  delete plan;
  return SPCG_OK;
}

int spcg_dist_plan_export(spcg_dist_plan_t plan, unsigned char* blob) {
  if (!plan || !blob) return fail(SPCG_ERR_ARG, "null argument");
  if (int rc = on_device(plan->m->device)) return rc;
  return plan_export(plan, blob);
}

int spcg_dist_plan_connect(spcg_dist_plan_t plan, const unsigned char* blobs) {
  if (!plan || !blobs) return fail(SPCG_ERR_ARG, "null argument");
  if (int rc = on_device(plan->m->device)) return rc;
  std::lock_guard<std::mutex> lk(plan->m->mu);
  return plan_connect(plan, blobs);
}

int spcg_dist_plan_solve(spcg_dist_plan_t plan, const double* d_b, const double* d_x0, double* d_x,
                         double* d_hist, const spcg_cg_options* opts, spcg_cg_result* result,
                         void* stream) {
  if (!plan || !opts || !result) return fail(SPCG_ERR_ARG, "null argument");
  if (plan->m->n > 0 && (!d_b || !d_x)) return fail(SPCG_ERR_ARG, "null vector");
  std::lock_guard<std::mutex> lk(plan->m->mu);
  spcg_dist_plan_s* P[1] = {plan};
  const double* b[1] = {d_b};
  const double* x0[1] = {d_x0};
  double* x[1] = {d_x};
  return plan_solve_checked(1, P, b, d_x0 ? x0 : nullptr, x, d_hist, opts, result,
                            (cudaStream_t)stream);
}

int spcg_dist_group_solve(int nranks, spcg_dist_plan_t* plans, const double* const* d_b,
                          const double* const* d_x0, double* const* d_x, double* d_hist,
                          const spcg_cg_options* opts, spcg_cg_result* results, void* stream) {
  if (nranks < 1 || !plans || !d_b || !d_x || !opts || !results)
    return fail(SPCG_ERR_ARG, "null argument");
  for (int r = 0; r < nranks; ++r) {
    if (!plans[r] || plans[r]->rank != r || plans[r]->nranks != nranks)
      return fail(SPCG_ERR_ARG, "plans[r] must be rank r of this group");
    if (plans[r]->m->n > 0 && (!d_b[r] || !d_x[r])) return fail(SPCG_ERR_ARG, "null vector");
  }
  if (d_x0) {
    int given = 0;
    for (int r = 0; r < nranks; ++r) given += d_x0[r] != nullptr || plans[r]->m->n == 0;
    if (given != nranks) return fail(SPCG_ERR_ARG, "x0 must be given for every rank or none");
  }
  return plan_solve_checked(nranks, plans, d_b, d_x0, d_x, d_hist, opts, results,
                            (cudaStream_t)stream);
}

int spcg_cg_cond_estimate(const double* h_ab, int64_t k, double* cond) {
  if (!cond || (k > 0 && !h_ab) || k < 0) return fail(SPCG_ERR_ARG, "null argument or k < 0");
  *cond = k < 2 ? 0.0 : lanczos_cond(std::vector<double>(h_ab, h_ab + 2 * k), (long long)k);
  return SPCG_OK;
}

}  // extern "C"
