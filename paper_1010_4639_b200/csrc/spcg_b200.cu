// spcg_b200.cu — host runtime behind include/spcg_b200.h: matrix handles
// (upload, int32 narrowing, row tiling, L^T construction, in-HBM generators),
// solver workspaces, kernel launches and the extern "C" entry points.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>

#include "../../include/spcg_b200.h"
#include "cg.cuh"
#include "cg1.cuh"
#include "cgs.cuh"
#include "cg3.cuh"
#include "clus.cuh"
#include "dist.cuh"
#include "ops.cuh"

using namespace spcg;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
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
  int coop_stream = 0;  // co-resident CTAs of the streaming CG kernel
  int spmv_grid = 0;
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
    int br = 0, bs = 0, bp = 0, t = 0;
    int rc;
    if ((rc = occupancy(cg_kernel<K_CSR, true>, &br, kSmemRes))) return rc;
    if ((rc = occupancy(cg_kernel<K_CSR, false>, &bs))) return rc;
    // every instantiation shares the same block/smem shape; check the rest
    if ((rc = occupancy(cg_kernel<K_SCSR_ATOMIC, true>, &t, kSmemRes))) return rc;
    br = std::min(br, t);
    if ((rc = occupancy(cg_kernel<K_SCSR_PRIV, true>, &t, kSmemRes))) return rc;
    br = std::min(br, t);
    if ((rc = occupancy(cg_kernel<K_CSC, true>, &t, kSmemRes))) return rc;
    br = std::min(br, t);
    if ((rc = occupancy(cg1_kernel<K_CSR>, &t, kSmemRes))) return rc;
    br = std::min(br, t);
    if ((rc = occupancy(cg1_kernel<K_SCSR_ATOMIC>, &t, kSmemRes))) return rc;
    br = std::min(br, t);
    if ((rc = occupancy(cg1_kernel<K_SCSR_PRIV>, &t, kSmemRes))) return rc;
    br = std::min(br, t);
    if ((rc = occupancy(cg1_kernel<K_CSC>, &t, kSmemRes))) return rc;
    br = std::min(br, t);
    if ((rc = occupancy(cg_kernel<K_SCSR_ATOMIC, false>, &t))) return rc;
    bs = std::min(bs, t);
    if ((rc = occupancy(cg_kernel<K_SCSR_PRIV, false>, &t))) return rc;
    bs = std::min(bs, t);
    if ((rc = occupancy(cg_kernel<K_CSC, false>, &t))) return rc;
    bs = std::min(bs, t);
    if ((rc = occupancy(spmv_kernel<K_CSR>, &bp))) return rc;
    if ((rc = occupancy(spmv_kernel<K_SCSR_ATOMIC>, &t))) return rc;
    if ((rc = occupancy(spmv_kernel<K_SCSR_PRIV>, &t))) return rc;
    if ((rc = occupancy(spmv_kernel<K_CSC>, &t))) return rc;
    if ((rc = occupancy(cg3_kernel<K_CSR>, &t))) return rc;
    bs = std::min(bs, t);
    if ((rc = occupancy(cg3_kernel<K_SCSR_ATOMIC>, &t))) return rc;
    bs = std::min(bs, t);
    if ((rc = occupancy(cg3_kernel<K_SCSR_PRIV>, &t))) return rc;
    bs = std::min(bs, t);
    if ((rc = occupancy(cg3_kernel<K_CSC>, &t))) return rc;
    bs = std::min(bs, t);
    if ((rc = occupancy(cgs_kernel<K_CSR>, &t))) return rc;
    bs = std::min(bs, t);
    if ((rc = occupancy(cgs_kernel<K_SCSR_PRIV>, &t))) return rc;
    bs = std::min(bs, t);
    if ((rc = occupancy(dist_spmv_pq<K_CSR>, &t))) return rc;
    if ((rc = occupancy(dist_spmv_pq<K_SCSR_PRIV>, &t))) return rc;
    if ((rc = occupancy(dist_spmv_pq<K_SCSR_ATOMIC>, &t))) return rc;
    if ((rc = occupancy(dist_spmv_pq<K_CSC>, &t))) return rc;
    if ((rc = occupancy(dist_spmv<K_SCSR_ATOMIC>, &t))) return rc;
    if ((rc = occupancy(dist_spmv<K_CSC>, &t))) return rc;
    if ((rc = occupancy(dist_spmv<K_CSR>, &t))) return rc;
    if ((rc = occupancy(dist_spmv<K_SCSR_PRIV>, &t))) return rc;
    if (br < 1 || bs < 1 || bp < 1) return fail(SPCG_ERR_CUDA, "CG kernel does not fit on an SM");
    d.coop_res = std::min(br * d.sms, 32 * kPollWarps * kPollPer);
    d.coop_stream = std::min(bs * d.sms, 32 * kPollWarps * kPollPer);
    d.spmv_grid = bp * d.sms;
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
  double2* rp = nullptr;         // streaming engine: RP[2] interleaved (r, p) pairs
  // host-API staging
  double* b = nullptr;
  double* x = nullptr;
  double* x0 = nullptr;
  double* hist = nullptr;
  long long hist_cap = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
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
  double* send_buf = nullptr;
  long long send_cap = 0;
  int* send_idx = nullptr;
  long long send_idx_cap = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t tev[2][16] = {};  // per-iteration SpMV-pass timing (opts.timing)
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
};

struct spcg_matrix_s {
  int fmt = 0;
  int n = 0;          // lines held (all rows, or the rows block of a shard)
  long long nnz = 0;
  int device = 0;
  Seg A, B;
  bool hasB = false;
  Tiles t1, t2;
  long long bytes = 0;
  Workspace ws;
  // row block of a sharded matrix (rows [row0,row1) of an n_global system)
  bool is_rows = false;
  bool localized = false;
  long long row0 = 0, row1 = 0, n_global = 0;
  std::vector<long long> halo;  // sorted global ids of the halo columns
  DistWorkspace dw;
  ClusPlan cp;
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

int dmalloc(void** p, size_t bytes, long long* acct) {
  if (bytes < 256) bytes = 256;
  CUDA_TRY(cudaMalloc(p, bytes));
  if (acct) *acct += (long long)bytes;
  return SPCG_OK;
}

// Upload one CSR-like segment from host int32 arrays (+8 zero pad each).
int upload_seg(Seg& s, int n, const std::vector<int>& ptr, const int* idx, const double* val,
               long long nnz, long long* acct) {
  int rc;
  if ((rc = dmalloc((void**)&s.ptr, sizeof(int) * (size_t)(n + 1 + 8), acct))) return rc;
  if ((rc = dmalloc((void**)&s.idx, sizeof(int) * (size_t)(nnz + 8), acct))) return rc;
  if ((rc = dmalloc((void**)&s.val, sizeof(double) * (size_t)(nnz + 8), acct))) return rc;
  CUDA_TRY(cudaMemset(s.ptr, 0, sizeof(int) * (size_t)(n + 1 + 8)));
  CUDA_TRY(cudaMemset(s.idx + nnz, 0, sizeof(int) * 8));
  CUDA_TRY(cudaMemset(s.val + nnz, 0, sizeof(double) * 8));
  CUDA_TRY(cudaMemcpy(s.ptr, ptr.data(), sizeof(int) * (size_t)(n + 1), cudaMemcpyHostToDevice));
  // pad the tail of ptr with nnz so out-of-range slice reads stay monotone
  std::vector<int> tail(8, (int)nnz);
  CUDA_TRY(cudaMemcpy(s.ptr + n + 1, tail.data(), sizeof(int) * 8, cudaMemcpyHostToDevice));
  if (nnz > 0) {
    if (idx) CUDA_TRY(cudaMemcpy(s.idx, idx, sizeof(int) * (size_t)nnz, cudaMemcpyHostToDevice));
    if (val)
      CUDA_TRY(cudaMemcpy(s.val, val, sizeof(double) * (size_t)nnz, cudaMemcpyHostToDevice));
  }
  s.nnz = nnz;
  return SPCG_OK;
}

// Row tiles: first a balanced split into >= target pieces by the weight
// W(i) = ptrA[i] + ptrB[i] + i (entries + lines), then any piece over the
// caps (kTileLines lines, kTileNnz entries) is split greedily; a single line
// over kTileNnz becomes a "long" one-line tile.
void build_tiles(int n, const std::vector<int>& pA, const std::vector<int>* pB, int target,
                 std::vector<int4>& desc, std::vector<int2>* descB, int line_cap = kTileLines) {
  desc.clear();
  if (descB) descB->clear();
  if (n == 0) return;
  auto W = [&](int i) -> long long {
    return (long long)pA[i] + (pB ? (long long)(*pB)[i] : 0LL) + (long long)i;
  };
  auto nz = [&](int s, int e) -> long long {
    return (long long)(pA[e] - pA[s]) + (pB ? (long long)((*pB)[e] - (*pB)[s]) : 0LL);
  };
  const long long tot = W(n);
  const long long nzt = nz(0, n);
  long long T = std::max<long long>(target, (nzt + kTileNnz - 1) / kTileNnz);
  T = std::max<long long>(T, ((long long)n + line_cap - 1) / line_cap);
  T = std::max<long long>(1, std::min<long long>(T, n));
  auto push = [&](int s, int e) {
    desc.push_back(make_int4(s, e, pA[s], pA[e]));
    if (descB) descB->push_back(make_int2((*pB)[s], (*pB)[e]));
  };
  int s = 0;
  for (long long t = 1; t <= T && s < n; ++t) {
    int e;
    if (t == T) {
      e = n;
    } else {
      const long long goal = (tot * t + T - 1) / T;
      int lo = s, hi = n;  // first i >= s with W(i) >= goal
      while (lo < hi) {
        const int mid = lo + (hi - lo) / 2;
        if (W(mid) >= goal) hi = mid;
        else lo = mid + 1;
      }
      e = lo;
    }
    if (e <= s) continue;
    // enforce caps
    int a = s;
    while (a < e) {
      int lim = std::min(e, a + line_cap);
      int lo = a + 1, hi = lim;  // largest b in [a+1, lim] with nz(a,b) <= cap
      if (nz(a, a + 1) > kTileNnz) {
        push(a, a + 1);
        a = a + 1;
        continue;
      }
      while (lo < hi) {
        const int mid = lo + (hi - lo + 1) / 2;
        if (nz(a, mid) <= kTileNnz) lo = mid;
        else hi = mid - 1;
      }
      push(a, lo);
      a = lo;
    }
    s = e;
  }
}

int upload_tiles(Tiles& t, const std::vector<int4>& desc, const std::vector<int2>* descB,
                 long long* acct) {
  int rc;
  t.ntiles = (int)desc.size();
  if ((rc = dmalloc((void**)&t.desc, sizeof(int4) * std::max<size_t>(1, desc.size()), acct)))
    return rc;
  if (!desc.empty())
    CUDA_TRY(cudaMemcpy(t.desc, desc.data(), sizeof(int4) * desc.size(), cudaMemcpyHostToDevice));
  if (descB) {
    if ((rc = dmalloc((void**)&t.descB, sizeof(int2) * std::max<size_t>(1, descB->size()), acct)))
      return rc;
    if (!descB->empty())
      CUDA_TRY(cudaMemcpy(t.descB, descB->data(), sizeof(int2) * descB->size(),
                          cudaMemcpyHostToDevice));
  }
  return SPCG_OK;
}

// CSR of L^T from L+D host arrays: stable counting sort of the strictly
// lower entries by column (rows ascending within a column).
void transpose_strict_lower(int n, const std::vector<int>& ptr, const int* idx, const double* val,
                            std::vector<int>& tptr, std::vector<int>& tidx,
                            std::vector<double>& tval) {
  tptr.assign((size_t)n + 1, 0);
  for (int i = 0; i < n; ++i)
    for (int k = ptr[i]; k < ptr[i + 1]; ++k)
      if (idx[k] < i) tptr[idx[k] + 1]++;
  for (int j = 0; j < n; ++j) tptr[j + 1] += tptr[j];
  tidx.resize((size_t)tptr[n]);
  tval.resize((size_t)tptr[n]);
  std::vector<int> fill(tptr.begin(), tptr.end() - 1);
  for (int i = 0; i < n; ++i)
    for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
      const int j = idx[k];
      if (j < i) {
        tidx[fill[j]] = i;
        tval[fill[j]] = val[k];
        fill[j]++;
      }
    }
}

// (Re)compute the per-tile leading-edge windows from the device indices.
int compute_windows(Tiles& t, const Seg& A, const Seg* B, long long* acct) {
  if (t.ntiles == 0) return SPCG_OK;
  int rc;
  if (!t.win && (rc = dmalloc((void**)&t.win, sizeof(int2) * (size_t)t.ntiles, acct))) return rc;
  int *cmax = nullptr, *cmin = nullptr;
  if ((rc = dmalloc((void**)&cmax, sizeof(int) * (size_t)t.ntiles, nullptr))) return rc;
  if ((rc = dmalloc((void**)&cmin, sizeof(int) * (size_t)t.ntiles, nullptr))) return rc;
  tile_colext_kernel<<<std::min(t.ntiles, 148 * 16), 256>>>(t.desc, B ? t.descB : nullptr, t.ntiles,
                                                           A.idx, B ? B->idx : nullptr, cmax, cmin);
  tile_window_kernel<<<(t.ntiles + 255) / 256, 256>>>(t.ntiles, cmax, cmin, 4 * kTileLines, t.win);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaDeviceSynchronize());
  cudaFree(cmax);
  cudaFree(cmin);
  return SPCG_OK;
}

int target_tiles() {
  DevInfo* d = nullptr;
  if (dev_info(&d)) return 148;
  return d->sms;
}

// Long-row matrices split a line over 2 or 4 lanes when a full 512-line
// tile would not fit kTileNnz (tile_line): cap their tiles at 256 / 128
// lines so every thread of the CTA has a segment.  Rows averaging more than
// 32 entries keep 512-line tiles (CSR-stream body for the gather formats).
int tile_line_cap(long long entries, int n) {
  if (n == 0) return kTileLines;
  const double avg = (double)entries / (double)n;
  if (avg * kTileLines <= kTileNnz) return kTileLines;
  if (avg * (kTileLines / 2) <= kTileNnz) return kTileLines / 2;
  if (avg * (kTileLines / 4) <= kTileNnz) return kTileLines / 4;
  return kTileLines;
}

// Finish a handle from host int32 arrays (ptrA, idxA, valA).
int finish_matrix(spcg_matrix_s* m, const std::vector<int>& ptr, const int* idx, const double* val,
                  bool device_arrays_ready) {
  int rc;
  if (!device_arrays_ready) {
    if ((rc = upload_seg(m->A, m->n, ptr, idx, val, m->nnz, &m->bytes))) return rc;
  }
  const int target = target_tiles();
  std::vector<int4> desc;
  build_tiles(m->n, ptr, nullptr, target, desc, nullptr, tile_line_cap(m->n ? ptr[m->n] : 0, m->n));
  if ((rc = upload_tiles(m->t1, desc, nullptr, &m->bytes))) return rc;
  return SPCG_OK;
}

int finish_transpose(spcg_matrix_s* m, const std::vector<int>& ptr, const std::vector<int>& tptr,
                     const int* tidx, const double* tval, bool device_arrays_ready) {
  int rc;
  if (!device_arrays_ready) {
    if ((rc = upload_seg(m->B, m->n, tptr, tidx, tval, (long long)tptr[m->n], &m->bytes)))
      return rc;
  }
  std::vector<int4> desc;
  std::vector<int2> descB;
  build_tiles(m->n, ptr, &tptr, target_tiles(), desc, &descB,
              tile_line_cap(m->n ? (long long)ptr[m->n] + tptr[m->n] : 0, m->n));
  if ((rc = upload_tiles(m->t2, desc, &descB, &m->bytes))) return rc;
  m->hasB = true;
  return SPCG_OK;
}

// Windows for both tile tables (after the indices are final / localized).
int refresh_windows(spcg_matrix_s* m) {
  int rc;
  if ((rc = compute_windows(m->t1, m->A, nullptr, &m->bytes))) return rc;
  if (m->hasB && (rc = compute_windows(m->t2, m->A, &m->B, &m->bytes))) return rc;
  return SPCG_OK;
}

void free_matrix(spcg_matrix_s* m) {
  auto F = [](void* p) {
    if (p) cudaFree(p);
  };
  F(m->A.ptr); F(m->A.idx); F(m->A.val);
  F(m->B.ptr); F(m->B.idx); F(m->B.val);
  F(m->t1.desc); F(m->t1.descB); F(m->t2.desc); F(m->t2.descB); F(m->t1.win); F(m->t2.win);
  Workspace& w = m->ws;
  F(w.r); F(w.p0); F(w.p1); F(w.q); F(w.part); F(w.slots); F(w.res);
  F(w.b); F(w.x); F(w.x0); F(w.hist); F(w.cg1); F(w.rp);
  if (w.h_res) cudaFreeHost(w.h_res);
  if (w.ev0) cudaEventDestroy(w.ev0);
  if (w.ev1) cudaEventDestroy(w.ev1);
  DistWorkspace& d = m->dw;
  F(d.r_ext); F(d.p_ext[0]); F(d.p_ext[1]); F(d.tmp_ext); F(d.q); F(d.part); F(d.S);
  F(d.send_buf); F(d.send_idx);
  F(m->cp.ctas); F(m->cp.slices); F(m->cp.sends); F(m->cp.rowmeta); F(m->cp.gval); F(m->cp.gcol);
  F(m->cp.ghalo); F(m->cp.gslots);
  if (d.h_S) cudaFreeHost(d.h_S);
  if (d.ev0) cudaEventDestroy(d.ev0);
  if (d.ev1) cudaEventDestroy(d.ev1);
  for (int a = 0; a < 2; ++a)
    for (int c = 0; c < 16; ++c)
      if (d.tev[a][c]) cudaEventDestroy(d.tev[a][c]);
}

MatView view(const spcg_matrix_s* m, bool priv) {
  MatView v{};
  v.n = m->n;
  const Tiles& t = priv ? m->t2 : m->t1;
  v.ntiles = t.ntiles;
  v.tdesc = t.desc;
  v.tdescB = t.descB;
  v.ptrA = m->A.ptr;
  v.idxA = m->A.idx;
  v.valA = m->A.val;
  v.ptrB = m->B.ptr;
  v.idxB = m->B.idx;
  v.valB = m->B.val;
  v.twin = t.win;
  return v;
}

int kfmt_of(const spcg_matrix_s* m, int accumulation) {
  if (m->fmt == SPCG_FMT_CSR) return K_CSR;
  if (m->fmt == SPCG_FMT_CSC) return K_CSC;
  return accumulation == SPCG_ACC_PRIVATIZED ? K_SCSR_PRIV : K_SCSR_ATOMIC;
}

int ensure_ws(spcg_matrix_s* m, int grid) {
  Workspace& w = m->ws;
  int rc;
  if (w.n != m->n) {
    const size_t vb = sizeof(double) * (size_t)std::max(1, m->n);
    if ((rc = dmalloc((void**)&w.r, vb, nullptr))) return rc;
    if ((rc = dmalloc((void**)&w.p0, vb, nullptr))) return rc;
    if ((rc = dmalloc((void**)&w.p1, vb, nullptr))) return rc;
    if ((rc = dmalloc((void**)&w.q, vb, nullptr))) return rc;
    if ((rc = dmalloc((void**)&w.part, sizeof(double) * 4096, nullptr))) return rc;
    if ((rc = dmalloc((void**)&w.res, sizeof(CgDevResult), nullptr))) return rc;
    CUDA_TRY(cudaMallocHost((void**)&w.h_res, sizeof(CgDevResult)));
    CUDA_TRY(cudaEventCreate(&w.ev0));
    CUDA_TRY(cudaEventCreate(&w.ev1));
    w.n = m->n;
  }
  if (w.slots_g < grid) {
    if (w.slots) cudaFree(w.slots);
    if ((rc = dmalloc((void**)&w.slots, sizeof(unsigned long long) * 2 * kSlotWords * (size_t)grid, nullptr)))
      return rc;
    w.slots_g = grid;
  }
  return SPCG_OK;
}

template <int FMT>
int launch_cg(const CgArgs& a, bool res, int grid, cudaStream_t st, double2* rp, int n,
              bool three = false) {
  if (!res && three) {
    void* args[] = {(void*)&a};
    CUDA_TRY(cudaLaunchCooperativeKernel((const void*)cg3_kernel<FMT>, dim3(grid), dim3(kBlock),
                                         args, sizeof(Smem), st));
    return SPCG_OK;
  }
  if (res || rp == nullptr) {
    void* args[] = {(void*)&a};
    const void* fn = res ? (const void*)cg_kernel<FMT, true> : (const void*)cg_kernel<FMT, false>;
    CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kBlock), args,
                                         res ? kSmemRes : sizeof(Smem), st));
    return SPCG_OK;
  }
  CgsArgs g{};
  g.base = a;
  g.RP[0] = rp;
  g.RP[1] = rp + std::max(1, n);
  void* args[] = {(void*)&g};
  CUDA_TRY(cudaLaunchCooperativeKernel((const void*)cgs_kernel<FMT>, dim3(grid), dim3(kBlock), args,
                                       sizeof(Smem), st));
  return SPCG_OK;
}

template <int FMT>
int launch_cg1(const Cg1Args& a, int grid, cudaStream_t st) {
  void* args[] = {(void*)&a};
  const void* fn = (const void*)cg1_kernel<FMT>;
  CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kBlock), args, kSmemRes, st));
  return SPCG_OK;
}

template <int FMT>
int launch_spmv(const MatView& v, const double* x, double* y, int grid, cudaStream_t st) {
  spmv_kernel<FMT><<<grid, kBlock, sizeof(Smem), st>>>(v, x, y);
  CUDA_TRY(cudaGetLastError());
  return SPCG_OK;
}

int do_spmv(spcg_matrix_s* m, const double* x, double* y, int accumulation, cudaStream_t st) {
  DevInfo* d;
  int rc;
  if ((rc = dev_info(&d))) return rc;
  const int kf = kfmt_of(m, accumulation);
  if (kf == K_SCSR_PRIV && !m->hasB) return fail(SPCG_ERR_UNSUPPORTED, "no L^T for privatized mode");
  const MatView v = view(m, kf == K_SCSR_PRIV);
  if (m->n == 0) return SPCG_OK;
  if (kf == K_SCSR_ATOMIC || kf == K_CSC)
    CUDA_TRY(cudaMemsetAsync(y, 0, sizeof(double) * (size_t)m->n, st));
  const int grid = std::max(1, std::min(v.ntiles, d->spmv_grid));
  switch (kf) {
    case K_CSR: return launch_spmv<K_CSR>(v, x, y, grid, st);
    case K_SCSR_ATOMIC: return launch_spmv<K_SCSR_ATOMIC>(v, x, y, grid, st);
    case K_SCSR_PRIV: return launch_spmv<K_SCSR_PRIV>(v, x, y, grid, st);
    default: return launch_spmv<K_CSC>(v, x, y, grid, st);
  }
}

int do_dist_cg(spcg_matrix_s* m, spcg_comm_s* comm, int npeers, const int32_t* peers,
               const int64_t* recv_off, const int64_t* send_off, const int32_t* send_idx,
               const double* b, const double* x0, double* x, double* hist,
               const spcg_cg_options* o, spcg_cg_result* out, cudaStream_t st);

// ---- cluster-resident engine (engine 5, clus.cuh) ---------------------------

int clus_fail(ClusPlan& P, const char* why) {
  P.ok = false;
  P.why = why;
  return SPCG_OK;
}

int download_seg(const Seg& sg, int n, std::vector<int>& ptr, std::vector<int>& idx,
                 std::vector<double>& val) {
  ptr.resize((size_t)n + 1);
  CUDA_TRY(cudaMemcpy(ptr.data(), sg.ptr, sizeof(int) * ((size_t)n + 1), cudaMemcpyDeviceToHost));
  const size_t nz = (size_t)ptr[n];
  idx.resize(nz);
  val.resize(nz);
  if (nz) {
    CUDA_TRY(cudaMemcpy(idx.data(), sg.idx, sizeof(int) * nz, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(val.data(), sg.val, sizeof(double) * nz, cudaMemcpyDeviceToHost));
  }
  return SPCG_OK;
}

// Host CSR transpose (entries of each output row in ascending source-row
// order: the reference's privatized / sequential-scatter order).
void host_transpose(int n, const std::vector<int>& ptr, const std::vector<int>& idx,
                    const std::vector<double>& val, bool strict_lower, std::vector<int>& tp,
                    std::vector<int>& ti, std::vector<double>& tv) {
  tp.assign((size_t)n + 1, 0);
  for (int i = 0; i < n; ++i)
    for (int k = ptr[i]; k < ptr[i + 1]; ++k)
      if (!strict_lower || idx[k] < i) ++tp[(size_t)idx[k] + 1];
  for (int i = 0; i < n; ++i) tp[(size_t)i + 1] += tp[i];
  ti.resize((size_t)tp[n]);
  tv.resize((size_t)tp[n]);
  std::vector<int> pos(tp.begin(), tp.end() - 1);
  for (int i = 0; i < n; ++i)
    for (int k = ptr[i]; k < ptr[i + 1]; ++k)
      if (!strict_lower || idx[k] < i) {
        const int j = idx[k];
        ti[(size_t)pos[j]] = i;
        tv[(size_t)pos[j]++] = val[k];
      }
}

// Builds the cluster plan: row blocks, windows, SELL-32 slices (rows sorted
// by length), resident/streamed split, halo sends.  Infeasible systems keep
// P.ok = false (the caller falls back to the grid engines).
int build_clus_plan(spcg_matrix_s* m) {
  ClusPlan& P = m->cp;
  if (P.built) return SPCG_OK;
  P.built = true;
  const int n = m->n;
  if (m->is_rows) return clus_fail(P, "row block");
  if (n <= 0) return clus_fail(P, "empty");
  if ((long long)n > (long long)kClusGridMax * kClusMaxRows) return clus_fail(P, "too many rows");
  // rows as (segment A, segment B) entry lists
  std::vector<int> pA, iA, pB, iB;
  std::vector<double> vA, vB;
  int rc;
  if ((rc = download_seg(m->A, n, pA, iA, vA))) return rc;
  P.two = m->fmt == SPCG_FMT_SCSR;
  if (m->fmt == SPCG_FMT_CSC) {  // rows of A = transpose of the column store
    std::vector<int> tp, ti;
    std::vector<double> tv;
    host_transpose(n, pA, iA, vA, false, tp, ti, tv);
    pA.swap(tp);
    iA.swap(ti);
    vA.swap(tv);
  } else if (P.two) {
    if (m->hasB) {
      if ((rc = download_seg(m->B, n, pB, iB, vB))) return rc;
    } else {
      host_transpose(n, pA, iA, vA, true, pB, iB, vB);
    }
  }
  auto lenA = [&](int i) { return pA[(size_t)i + 1] - pA[i]; };
  auto lenB = [&](int i) { return P.two ? pB[(size_t)i + 1] - pB[i] : 0; };
  long long tot = 0;
  for (int i = 0; i < n; ++i) {
    const int l = lenA(i) + lenB(i);
    if (l > 4096 || lenA(i) > 32767) return clus_fail(P, "row too long");
    tot += l + 1;
  }
  // grid shape: one cluster of <= 16 CTAs, or K clusters of 8 (as many as
  // are co-resident) with ~4K entries per CTA so the whole matrix stays in
  // shared memory
  const int cmin = (n + kClusMaxRows - 1) / kClusMaxRows;
  const long long want = std::max<long long>(cmin, (tot + 3999) / 4000);
  const void* kfn = P.two ? (const void*)clus_cg_kernel<true> : (const void*)clus_cg_kernel<false>;
  int optin0 = 0, dev0 = 0;
  CUDA_TRY(cudaGetDevice(&dev0));
  CUDA_TRY(cudaDeviceGetAttribute(&optin0, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev0));
  const int smem_probe = optin0 - (int)sizeof(ClusShared) - 1024;
  auto max_clusters = [&](int csz) -> int {
    CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_probe));
    if (csz > 8) CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(csz);
    cfg.blockDim = dim3(kClusThreads);
    cfg.dynamicSmemBytes = (size_t)smem_probe;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csz;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, kfn, &cfg) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    return ncl;
  };
  int C, csz;
  static const int force_k = getenv("SPCG_CLUS_K") ? atoi(getenv("SPCG_CLUS_K")) : 0;  // dev A/B
  if ((want <= kClusMax && force_k <= 1) || force_k == 1) {
    C = csz = (int)std::min<long long>(kClusMax, std::max<long long>(1, want));
    if (max_clusters(csz) < 1) return clus_fail(P, "cluster not launchable");
  } else {
    csz = 8;
    const int kmax = std::min(max_clusters(csz), kClusGridMax / 8);
    int K = (int)std::min<long long>(kmax, (want + csz - 1) / csz);
    if (force_k > 1) K = std::min(kmax, force_k);
    if (K < 1) return clus_fail(P, "cluster not launchable");
    if ((long long)K * csz * kClusMaxRows < n) {  // fall back to one big cluster
      csz = kClusMax;
      K = 1;
      if (max_clusters(csz) < 1 || (long long)csz * kClusMaxRows < n)
        return clus_fail(P, "too many rows for the co-resident clusters");
    }
    C = K * csz;
  }
  // contiguous row blocks balanced by entries + rows, <= kClusMaxRows each
  std::vector<int> lo(C), hi(C);
  {
    int r = 0;
    long long acc = 0;
    for (int c = 0; c < C; ++c) {
      lo[c] = r;
      const long long goal = tot * (c + 1) / C;
      while (r < n && (r - lo[c]) < kClusMaxRows && (acc < goal || c == C - 1)) {
        acc += lenA(r) + lenB(r) + 1;
        ++r;
      }
      hi[c] = r;
    }
    if (r < n) return clus_fail(P, "row blocks exceed the cluster");
  }
  // windows
  std::vector<int> wlo(C), whi(C);
  for (int c = 0; c < C; ++c) {
    int a = lo[c], z = hi[c];
    for (int i = lo[c]; i < hi[c]; ++i) {
      for (int k = pA[i]; k < pA[(size_t)i + 1]; ++k) {
        a = std::min(a, iA[k]);
        z = std::max(z, iA[k] + 1);
      }
      if (P.two)
        for (int k = pB[i]; k < pB[(size_t)i + 1]; ++k) {
          a = std::min(a, iB[k]);
          z = std::max(z, iB[k] + 1);
        }
    }
    wlo[c] = a;
    whi[c] = z;
    if (z - a > 8192) return clus_fail(P, "gather window too wide (not banded)");
  }
  int wmax = 1, hcap = 1;
  for (int c = 0; c < C; ++c) {
    wmax = std::max(wmax, whi[c] - wlo[c]);
    hcap = std::max(hcap, (whi[c] - wlo[c]) - (hi[c] - lo[c]));
  }
  // slices: rows of a block sorted by length (descending, stable)
  std::vector<ClusCta> ctas(C);
  std::vector<ClusSlice> slices;
  std::vector<int2> rowmeta;
  std::vector<std::vector<int>> order(C);
  for (int c = 0; c < C; ++c) {
    std::vector<int>& o = order[c];
    for (int i = lo[c]; i < hi[c]; ++i) o.push_back(i);
    std::stable_sort(o.begin(), o.end(),
                     [&](int a, int b2) { return lenA(a) + lenB(a) > lenA(b2) + lenB(b2); });
    ClusCta& t = ctas[c];
    t.row_lo = lo[c];
    t.row_hi = hi[c];
    t.clo = lo[(c / csz) * csz];
    t.chi = hi[(c / csz) * csz + csz - 1];
    t.wlo = wlo[c];
    t.wn = whi[c] - wlo[c];
    t.hlo = lo[c] - wlo[c];
    t.slice0 = (int)slices.size();
    t.nslices = ((int)o.size() + 31) / 32;
    for (int s = 0; s < t.nslices; ++s) {
      ClusSlice sd{};
      int wdt = 0;
      for (int l = 0; l < 32; ++l) {
        const int q = 32 * s + l;
        if (q < (int)o.size()) wdt = std::max(wdt, lenA(o[q]) + lenB(o[q]));
      }
      sd.width = wdt;
      sd.soff = -1;
      slices.push_back(sd);
      for (int l = 0; l < 32; ++l) {
        const int q = 32 * s + l;
        if (q < (int)o.size()) {
          const int i = o[q];
          rowmeta.push_back(make_int2(i, (lenA(i) << 16) | (lenA(i) + lenB(i))));
        } else {
          rowmeta.push_back(make_int2(-1, 0));
        }
      }
    }
  }
  // shared-memory layout and the resident budget
  DevInfo* d;
  if ((rc = dev_info(&d))) return rc;
  int optin = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, d->device));
  auto al = [](size_t v) { return (v + 127) & ~(size_t)127; };
  size_t off = 0;
  P.off_rwin = (int)off;
  off = al(off + sizeof(double) * (size_t)wmax);
  P.off_shalo = (int)off;
  off = al(off + sizeof(double) * (size_t)hcap);
  P.off_whalo = (int)off;
  off = al(off + sizeof(double) * 2 * (size_t)hcap);
  P.off_val = (int)off;
  const long long budget = (long long)optin - (long long)sizeof(ClusShared) - (long long)off - 1024;
  if (budget < 0) return clus_fail(P, "window does not fit shared memory");
  const long long E = budget / 10;  // 8 B value + 2 B column per resident entry
  long long goff = 0;
  for (int c = 0; c < C; ++c) {
    long long used = 0;
    const ClusCta& t = ctas[c];
    for (int k = 0; k < kClusSlicesPerWarp; ++k)
      for (int w = 0; w < kClusWarps; ++w) {
        const int s = w + kClusWarps * k;
        if (s >= t.nslices) continue;
        ClusSlice& sd = slices[(size_t)t.slice0 + s];
        const long long cnt = 32LL * sd.width;
        if (used + cnt <= E) {
          sd.soff = (int)used;
          used += cnt;
          P.resident += cnt;
        } else {
          P.streamed += cnt;
        }
      }
    for (int s = 0; s < t.nslices; ++s) {
      slices[(size_t)t.slice0 + s].goff = (int)goff;
      goff += 32LL * slices[(size_t)t.slice0 + s].width;
    }
  }
  if (goff >= (1LL << 31)) return clus_fail(P, "too many entries");
  P.off_col = (int)(P.off_val + 8 * E);
  P.smem = (size_t)P.off_col + 2 * (size_t)E;
  // SELL values / window-relative columns
  std::vector<double> gval((size_t)goff + 8, 0.0);
  std::vector<unsigned short> gcol((size_t)goff + 8, 0);
  for (int c = 0; c < C; ++c) {
    const ClusCta& t = ctas[c];
    for (int s = 0; s < t.nslices; ++s) {
      const ClusSlice& sd = slices[(size_t)t.slice0 + s];
      for (int l = 0; l < 32; ++l) {
        const int2 rm = rowmeta[((size_t)t.slice0 + s) * 32 + l];
        if (rm.x < 0) continue;
        const int i = rm.x;
        int u = 0;
        for (int k = pA[i]; k < pA[(size_t)i + 1]; ++k, ++u) {
          gval[(size_t)sd.goff + (size_t)u * 32 + l] = vA[k];
          gcol[(size_t)sd.goff + (size_t)u * 32 + l] = (unsigned short)(iA[k] - t.wlo);
        }
        if (P.two)
          for (int k = pB[i]; k < pB[(size_t)i + 1]; ++k, ++u) {
            gval[(size_t)sd.goff + (size_t)u * 32 + l] = vB[k];
            gcol[(size_t)sd.goff + (size_t)u * 32 + l] = (unsigned short)(iB[k] - t.wlo);
          }
      }
    }
  }
  // halo sends: owner d -> every CTA c whose window holds d's rows
  std::vector<ClusSend> sends;
  for (int dd = 0; dd < C; ++dd) {
    ctas[dd].send0 = (int)sends.size();
    for (int c = 0; c < C; ++c) {
      if (c == dd) continue;
      const int a1 = std::max(wlo[c], lo[dd]), z1 = std::min(lo[c], hi[dd]);  // lower halo
      if (a1 < z1) sends.push_back(ClusSend{c, a1, z1, a1 - wlo[c]});
      const int a2 = std::max(hi[c], lo[dd]), z2 = std::min(whi[c], hi[dd]);  // upper halo
      if (a2 < z2) sends.push_back(ClusSend{c, a2, z2, ctas[c].hlo + (a2 - hi[c])});
    }
    ctas[dd].nsend = (int)sends.size() - ctas[dd].send0;
  }
  if (sends.empty()) sends.push_back(ClusSend{0, 0, 0, 0});
  // the grid of C CTAs in clusters of csz must be co-resident with this smem
  CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.smem));
  if (csz > 8) CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(csz);
    cfg.blockDim = dim3(kClusThreads);
    cfg.dynamicSmemBytes = P.smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csz;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, kfn, &cfg) != cudaSuccess || ncl < C / csz) {
      cudaGetLastError();
      return clus_fail(P, "clusters not co-resident");
    }
  }
  long long acct = 0;
  if ((rc = dmalloc((void**)&P.ctas, sizeof(ClusCta) * ctas.size(), &acct)) ||
      (rc = dmalloc((void**)&P.slices, sizeof(ClusSlice) * slices.size(), &acct)) ||
      (rc = dmalloc((void**)&P.sends, sizeof(ClusSend) * sends.size(), &acct)) ||
      (rc = dmalloc((void**)&P.rowmeta, sizeof(int2) * rowmeta.size(), &acct)) ||
      (rc = dmalloc((void**)&P.gval, sizeof(double) * gval.size(), &acct)) ||
      (rc = dmalloc((void**)&P.gcol, sizeof(unsigned short) * gcol.size(), &acct)))
    return rc;
  CUDA_TRY(cudaMemcpy(P.ctas, ctas.data(), sizeof(ClusCta) * ctas.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(P.slices, slices.data(), sizeof(ClusSlice) * slices.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(P.sends, sends.data(), sizeof(ClusSend) * sends.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(P.rowmeta, rowmeta.data(), sizeof(int2) * rowmeta.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(P.gval, gval.data(), sizeof(double) * gval.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(P.gcol, gcol.data(), sizeof(unsigned short) * gcol.size(), cudaMemcpyHostToDevice));
  if (C > csz) {
    if ((rc = dmalloc((void**)&P.ghalo, sizeof(double) * 2 * (size_t)C * hcap, &acct)) ||
        (rc = dmalloc((void**)&P.gslots,
                      sizeof(unsigned long long) * 2 * kClusSlotWords * (size_t)(C / csz),
                      &acct)))
      return rc;
    CUDA_TRY(cudaMemset(P.ghalo, 0, sizeof(double) * 2 * (size_t)C * hcap));
  }
  m->bytes += acct;
  P.hcap = hcap;
  P.C = C;
  P.cs = csz;
  P.ok = true;
  return SPCG_OK;
}

int launch_clus(const ClusPlan& P, const ClusArgs& a, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P.C);
  cfg.blockDim = dim3(kClusThreads);
  cfg.dynamicSmemBytes = P.smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = P.cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeCooperative;  // K > 1 clusters poll each other
  at[1].val.cooperative = 1;
  cfg.attrs = at;
  // SPCG_CLUS_NONCOOP=1 (profiling only): ncu drops the cluster shape of a
  // cooperative cluster launch; the K clusters still fit on the device at
  // once, and the kernel refuses a launch whose cluster size is not the plan's
  static const bool noncoop = getenv("SPCG_CLUS_NONCOOP") != nullptr;
  cfg.numAttrs = (P.C > P.cs && !noncoop) ? 2 : 1;
  if (P.two) CUDA_TRY(cudaLaunchKernelEx(&cfg, clus_cg_kernel<true>, a));
  else CUDA_TRY(cudaLaunchKernelEx(&cfg, clus_cg_kernel<false>, a));
  return SPCG_OK;
}

int do_clus_cg(spcg_matrix_s* m, const double* b, const double* x0, double* x, double* hist,
               const spcg_cg_options* o, spcg_cg_result* out, cudaStream_t st) {
  int rc;
  const ClusPlan& P = m->cp;
  if ((rc = ensure_ws(m, 1))) return rc;
  Workspace& w = m->ws;
  const long long max_iter = o->max_iter > 0 ? o->max_iter : std::max(1, m->n);
  if (o->record_history && hist == nullptr)
    return fail(SPCG_ERR_ARG, "record_history needs a history buffer");
  ClusArgs a{};
  a.ctas = P.ctas;
  a.slices = P.slices;
  a.sends = P.sends;
  a.rowmeta = P.rowmeta;
  a.gval = P.gval;
  a.gcol = P.gcol;
  a.b = b;
  a.x0 = x0;
  a.x = x;
  a.scratch = w.q;
  a.hist = hist;
  a.res = w.res;
  a.tol = o->tol;
  a.max_iter = max_iter;
  a.record_history = o->record_history;
  a.recompute = o->recompute_final_residual;
  a.off_rwin = P.off_rwin;
  a.off_shalo = P.off_shalo;
  a.off_whalo = P.off_whalo;
  a.off_val = P.off_val;
  a.off_col = P.off_col;
  a.hcap = P.hcap;
  a.ghalo = P.ghalo;
  a.gslots = P.gslots;
  a.cluster_size = P.cs;
  if (P.gslots)
    CUDA_TRY(cudaMemsetAsync(P.gslots, 0,
                             sizeof(unsigned long long) * 2 * kClusSlotWords * (size_t)(P.C / P.cs),
                             st));
  static const bool tracing = getenv("SPCG_TRACE") != nullptr;
  if (tracing) {
    CUDA_TRY(cudaMalloc((void**)&a.trace, sizeof(unsigned long long) * 8 * (size_t)P.C));
    CUDA_TRY(cudaMemsetAsync(a.trace, 0, sizeof(unsigned long long) * 8 * (size_t)P.C, st));
  }
  CUDA_TRY(cudaEventRecord(w.ev0, st));
  if ((rc = launch_clus(P, a, st))) return rc;
  CUDA_TRY(cudaEventRecord(w.ev1, st));
  CUDA_TRY(cudaMemcpyAsync(w.h_res, w.res, sizeof(CgDevResult), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  float ms = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&ms, w.ev0, w.ev1));
  const CgDevResult& r = *w.h_res;
  if (r.status == ST_BAD_LAUNCH)
    return fail(SPCG_ERR_CUDA, "cluster engine: kernel ran with a different cluster shape than "
                               "planned (cluster launch attribute not honoured)");
  if (a.trace) {
    std::vector<unsigned long long> tv(8 * (size_t)P.C);
    CUDA_TRY(cudaMemcpy(tv.data(), a.trace, sizeof(unsigned long long) * tv.size(),
                        cudaMemcpyDeviceToHost));
    cudaFree(a.trace);
    double mean[7] = {0}, mx[7] = {0}, lead[7] = {0};
    int nl = 0;
    for (int c = 0; c < P.C; ++c)
      for (int ph = 0; ph < 7; ++ph) {
        mean[ph] += (double)tv[8 * c + ph] / P.C;
        mx[ph] = std::max(mx[ph], (double)tv[8 * c + ph]);
        if (c % std::max(1, P.cs) == 0) lead[ph] += (double)tv[8 * c + ph];
      }
    nl = std::max(1, P.C / std::max(1, P.cs));
    const double it = (double)std::max<long long>(1, r.iterations) * 1e3;
    fprintf(stderr,
            "[spcg trace] ctas=%d cs=%d resident=%lld streamed=%lld us/iter mean(max): update %.3f(%.3f) "
            "spmv %.3f(%.3f) allreduce %.3f(%.3f) | send_w %.3f b1wait %.3f b1exit->b2exit %.3f "
            "| leaders: exchange %.3f b1wait %.3f poll->b2exit %.3f\n",
            P.C, P.cs, P.resident, P.streamed, mean[0] / it, mx[0] / it, mean[1] / it, mx[1] / it,
            mean[2] / it, mx[2] / it, mean[6] / it, mean[5] / it, mean[4] / it, lead[3] / nl / it,
            lead[5] / nl / it, lead[4] / nl / it);
    if (P.C > P.cs) {  // mean slot-post time of each cluster relative to the earliest
      double mn = 1e300;
      std::vector<double> pt;
      for (int c = 0; c < P.C; c += P.cs) {
        pt.push_back((double)tv[8 * c + 7] / it);
        mn = std::min(mn, pt.back());
      }
      fprintf(stderr, "[spcg trace] cluster post offsets (us):");
      for (double v : pt) fprintf(stderr, " %.2f", v - mn);
      fprintf(stderr, "\n");
    }
  }
  out->iterations = r.iterations;
  out->converged = r.converged;
  out->status = r.status;
  out->fail_iteration = r.fail_iter;
  out->final_relative_residual = r.final_rel;
  out->b_norm = r.b_norm;
  out->device_ms = ms;
  out->kernel_launches = 1;
  out->spmv_ms = 0.0;
  out->spmv_launches = 0;
  if (r.status != SPCG_OK) {
    const char* what = r.status == SPCG_ERR_NOT_SPD ? "matrix not positive definite"
                       : r.status == SPCG_ERR_NONFINITE_ALPHA ? "non-finite alpha"
                       : r.status == SPCG_ERR_NONFINITE_RESIDUAL ? "non-finite residual"
                                                                  : "non-finite beta";
    return fail(r.status, std::string(what) + " at iteration " + std::to_string(r.fail_iter));
  }
  return SPCG_OK;
}

int do_cg(spcg_matrix_s* m, const double* b, const double* x0, double* x, double* hist,
          const spcg_cg_options* o, spcg_cg_result* out, cudaStream_t st) {
  DevInfo* d;
  int rc;
  if ((rc = dev_info(&d))) return rc;
  if (!(o->tol > 0.0)) return fail(SPCG_ERR_ARG, "tol must be > 0");
  if (m->is_rows) return fail(SPCG_ERR_ARG, "a row block is solved with spcg_dist_cg_solve");
  if (m->n == 0) {  // ||b|| = 0: x = [] converged in 0 iterations, any engine (solver.py:109-118)
    *out = spcg_cg_result{};
    out->converged = 1;
    return SPCG_OK;
  }
  const int kf = kfmt_of(m, o->accumulation);
  if (kf == K_SCSR_PRIV && !m->hasB) return fail(SPCG_ERR_UNSUPPORTED, "no L^T for privatized mode");
  const MatView v = view(m, kf == K_SCSR_PRIV);
  const bool fits = v.ntiles <= d->coop_res * kStages;
  // engine 2, and auto for systems that stream from HBM: per-pass kernels
  // (the sharded engine with no peers) — each pass keeps the whole register
  // budget, which the persistent kernel cannot (P3: 0.99 vs 0.82 of roofline)
  if (o->engine == 2 || (o->engine == 0 && !fits))
    return do_dist_cg(m, nullptr, 0, nullptr, nullptr, nullptr, nullptr, b, x0, x, hist, o, out, st);
  // engine 5, and auto for banded systems whose rows fit the co-resident
  // clusters' shared memory: cluster-resident single-reduction CG (DSMEM +
  // hardware cluster barriers; K clusters of 8 exchange through global
  // memory).  F: 5.35 us/iteration vs 8.45 on engine 3; S: 6.23 vs 8.58.
  if (o->engine == 5 || (o->engine == 0 && m->n <= kClusGridMax * kClusMaxRows)) {
    if ((rc = build_clus_plan(m))) return rc;
    // auto only when (nearly) everything stays in shared memory: streamed
    // slices are re-read from L2 every iteration at L2 latency
    const bool resident = m->cp.streamed * 9 <= m->cp.resident;
    if (m->cp.ok && (o->engine == 5 || resident)) return do_clus_cg(m, b, x0, x, hist, o, out, st);
    if (o->engine == 5)
      return fail(SPCG_ERR_UNSUPPORTED, "cluster engine not applicable: " + m->cp.why);
  }
  const bool res = fits;
  // resident: the balanced tiles map one-to-one onto CTAs where possible
  const int grid = res ? std::max(1, std::min(d->coop_res, std::max(1, v.ntiles)))
                       : d->coop_stream;
  if ((rc = ensure_ws(m, grid))) return rc;
  Workspace& w = m->ws;
  const long long max_iter = o->max_iter > 0 ? o->max_iter : std::max(1, m->n);
  if (o->record_history && hist == nullptr)
    return fail(SPCG_ERR_ARG, "record_history needs a history buffer");
  CUDA_TRY(cudaMemsetAsync(w.slots, 0, sizeof(unsigned long long) * 2 * kSlotWords * (size_t)grid, st));
  if (kf == K_SCSR_ATOMIC || kf == K_CSC)
    CUDA_TRY(cudaMemsetAsync(w.q, 0, sizeof(double) * (size_t)std::max(1, m->n), st));
  CgArgs a{};
  a.M = v;
  a.b = b;
  a.x0 = x0;
  a.x = x;
  a.r = w.r;
  a.p0 = w.p0;
  a.p1 = w.p1;
  a.q = w.q;
  a.hist = hist;
  a.slots = w.slots;
  unsigned long long* trace = nullptr;
  static const bool tracing = getenv("SPCG_TRACE") != nullptr;
  if (tracing) {
    CUDA_TRY(cudaMalloc((void**)&trace, sizeof(unsigned long long) * 5 * (size_t)grid));
    CUDA_TRY(cudaMemsetAsync(trace, 0, sizeof(unsigned long long) * 5 * (size_t)grid, st));
  }
  a.trace = trace;
  a.res = w.res;
  a.tol = o->tol;
  a.max_iter = max_iter;
  a.record_history = o->record_history;
  a.recompute = o->recompute_final_residual;
  // engine 3 (or auto on resident systems): single-reduction CG, one grid
  // barrier per iteration; engine 1 forces the two-reduction form
  const bool single = res && (o->engine == 3 || o->engine == 0);
  Cg1Args g{};
  if (single) {
    const size_t vb = sizeof(double) * (size_t)std::max(1, m->n);
    if (!w.cg1 && (rc = dmalloc((void**)&w.cg1, 7 * vb, nullptr))) return rc;
    CUDA_TRY(cudaMemsetAsync(w.cg1, 0, 7 * vb, st));
    g.base = a;
    for (int k = 0; k < 2; ++k) g.R[k] = w.cg1 + (size_t)k * std::max(1, m->n);
    for (int k = 0; k < 2; ++k) g.S[k] = w.cg1 + (size_t)(2 + k) * std::max(1, m->n);
    for (int k = 0; k < 3; ++k) g.W[k] = w.cg1 + (size_t)(4 + k) * std::max(1, m->n);
  }
  CUDA_TRY(cudaEventRecord(w.ev0, st));
  if (single) {
    switch (kf) {
      case K_CSR: rc = launch_cg1<K_CSR>(g, grid, st); break;
      case K_SCSR_ATOMIC: rc = launch_cg1<K_SCSR_ATOMIC>(g, grid, st); break;
      case K_SCSR_PRIV: rc = launch_cg1<K_SCSR_PRIV>(g, grid, st); break;
      default: rc = launch_cg1<K_CSC>(g, grid, st); break;
    }
  } else {
    // streaming systems: interleaved (r, p) pairs pay off for the gather-only
    // formats with long rows (27-point class: 20% on full CSR); short rows
    // (5/7-point) and the atomic scatters keep separate r and p arrays
    const double per_line = (double)(m->nnz + (kf == K_SCSR_PRIV ? m->B.nnz : 0)) /
                            std::max(1, m->n);
    const bool three = !res && o->engine == 4;  // persistent three-pass (unfolded) CG
    const bool pairs = !res && !three && (kf == K_CSR || kf == K_SCSR_PRIV) && per_line > 8.0;
    if (pairs && !w.rp &&
        (rc = dmalloc((void**)&w.rp, sizeof(double2) * 2 * (size_t)std::max(1, m->n), nullptr)))
      return rc;
    double2* rp = pairs ? w.rp : nullptr;
    switch (kf) {
      case K_CSR: rc = launch_cg<K_CSR>(a, res, grid, st, rp, m->n, three); break;
      case K_SCSR_ATOMIC: rc = launch_cg<K_SCSR_ATOMIC>(a, res, grid, st, rp, m->n, three); break;
      case K_SCSR_PRIV: rc = launch_cg<K_SCSR_PRIV>(a, res, grid, st, rp, m->n, three); break;
      default: rc = launch_cg<K_CSC>(a, res, grid, st, rp, m->n, three); break;
    }
  }
  if (rc) return rc;
  CUDA_TRY(cudaEventRecord(w.ev1, st));
  CUDA_TRY(cudaMemcpyAsync(w.h_res, w.res, sizeof(CgDevResult), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  float ms = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&ms, w.ev0, w.ev1));
  const CgDevResult& r = *w.h_res;
  if (trace) {
    std::vector<unsigned long long> tv(5 * (size_t)grid);
    CUDA_TRY(cudaMemcpy(tv.data(), trace, sizeof(unsigned long long) * tv.size(),
                        cudaMemcpyDeviceToHost));
    cudaFree(trace);
    double mean[5] = {0, 0, 0, 0, 0}, mx[5] = {0, 0, 0, 0, 0};
    for (int b = 0; b < grid; ++b)
      for (int ph = 0; ph < 5; ++ph) {
        mean[ph] += (double)tv[5 * b + ph] / grid;
        mx[ph] = std::max(mx[ph], (double)tv[5 * b + ph]);
      }
    const double it = (double)std::max<long long>(1, r.iterations);
    fprintf(stderr,
            "[spcg trace] grid=%d res=%d iters=%lld us/iter mean(max): passA %.3f(%.3f) "
            "reduce1 %.3f(%.3f) passB %.3f(%.3f) reduce2 %.3f(%.3f) tilewait %.3f(%.3f)\n",
            grid, (int)res, r.iterations, mean[0] / it / 1e3, mx[0] / it / 1e3, mean[1] / it / 1e3,
            mx[1] / it / 1e3, mean[2] / it / 1e3, mx[2] / it / 1e3, mean[3] / it / 1e3,
            mx[3] / it / 1e3, mean[4] / it / 1e3, mx[4] / it / 1e3);
  }
  out->iterations = r.iterations;
  out->converged = r.converged;
  out->status = r.status;
  out->fail_iteration = r.fail_iter;
  out->final_relative_residual = r.final_rel;
  out->b_norm = r.b_norm;
  out->device_ms = ms;
  out->kernel_launches = 1;
  out->spmv_ms = 0.0;
  out->spmv_launches = 0;
  if (r.status != SPCG_OK) {
    const char* what = r.status == SPCG_ERR_NOT_SPD ? "matrix not positive definite"
                       : r.status == SPCG_ERR_NONFINITE_ALPHA ? "non-finite alpha"
                       : r.status == SPCG_ERR_NONFINITE_RESIDUAL ? "non-finite residual"
                                                                  : "non-finite beta";
    return fail(r.status, std::string(what) + " at iteration " + std::to_string(r.fail_iter));
  }
  return SPCG_OK;
}

int check_csr_host(int fmt, int64_t n, int64_t nnz) {
  if (fmt < 0 || fmt > 2) return fail(SPCG_ERR_ARG, "unknown format");
  if (n < 0 || nnz < 0) return fail(SPCG_ERR_ARG, "negative size");
  if (n >= (1LL << 31) - 16 || nnz >= (1LL << 31) - 16)
    return fail(SPCG_ERR_UNSUPPORTED, "n and nnz must fit 32-bit indices");
  return SPCG_OK;
}

template <class PT, class IT>
int create_from_host(int fmt, int64_t n, int64_t nnz, const PT* hp, const IT* hi, const double* hv,
                     spcg_matrix_t* out) {
  int rc;
  if ((rc = check_csr_host(fmt, n, nnz))) return rc;
  if (n > 0 && (hp == nullptr)) return fail(SPCG_ERR_ARG, "null offsets");
  if (nnz > 0 && (hi == nullptr || hv == nullptr)) return fail(SPCG_ERR_ARG, "null arrays");
  std::vector<int> ptr((size_t)n + 1);
  if (n == 0) {
    ptr[0] = 0;
  } else {
    if ((long long)hp[0] != 0 || (long long)hp[n] != nnz)
      return fail(SPCG_ERR_ARG, "offsets must start at 0 and end at nnz");
    for (int64_t i = 0; i <= n; ++i) {
      if (i > 0 && hp[i] < hp[i - 1]) return fail(SPCG_ERR_ARG, "offsets must be non-decreasing");
      ptr[(size_t)i] = (int)hp[i];
    }
  }
  std::vector<int> idx((size_t)nnz);
  for (int64_t k = 0; k < nnz; ++k) {
    const long long c = (long long)hi[k];
    if (c < 0 || c >= n) return fail(SPCG_ERR_ARG, "index out of range at entry " + std::to_string(k));
    idx[(size_t)k] = (int)c;
  }
  if (fmt == SPCG_FMT_SCSR) {
    for (int64_t i = 0; i < n; ++i) {
      const int a = ptr[i], b = ptr[i + 1];
      if (b <= a || idx[b - 1] != (int)i)
        return fail(SPCG_ERR_ARG, "row " + std::to_string(i) + " has no stored diagonal entry");
      for (int k = a; k < b; ++k)
        if (idx[k] > (int)i) return fail(SPCG_ERR_ARG, "symmetric-half storage requires col <= row");
    }
  }
  DevInfo* d;
  if ((rc = dev_info(&d))) return rc;
  spcg_matrix_s* m = new spcg_matrix_s();
  m->fmt = fmt;
  m->n = (int)n;
  m->nnz = nnz;
  CUDA_TRY(cudaGetDevice(&m->device));
  if ((rc = finish_matrix(m, ptr, idx.data(), hv, false))) {
    free_matrix(m);
    delete m;
    return rc;
  }
  if (fmt == SPCG_FMT_SCSR) {
    std::vector<int> tptr, tidx;
    std::vector<double> tval;
    transpose_strict_lower((int)n, ptr, idx.data(), hv, tptr, tidx, tval);
    if ((rc = finish_transpose(m, ptr, tptr, tidx.data(), tval.data(), false))) {
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

// Device generator: counts -> host prefix sum -> ptr upload -> device fill.
int gen_seg(int kind, int part, long long row0, long long n, int nx, int ny, int nz, Seg& s,
            std::vector<int>& ptr, long long* acct) {
  int rc;
  int* counts = nullptr;
  if ((rc = dmalloc((void**)&counts, sizeof(int) * (size_t)std::max<long long>(1, n), nullptr)))
    return rc;
  const int grid = 148 * 8;
  stencil_count_kernel<<<grid, 256>>>(kind, part, row0, n, nx, ny, nz, counts);
  CUDA_TRY(cudaGetLastError());
  std::vector<int> c((size_t)n);
  CUDA_TRY(cudaMemcpy(c.data(), counts, sizeof(int) * (size_t)n, cudaMemcpyDeviceToHost));
  cudaFree(counts);
  ptr.assign((size_t)n + 1, 0);
  long long acc = 0;
  for (long long i = 0; i < n; ++i) {
    acc += c[(size_t)i];
    if (acc >= (1LL << 31) - 16) return fail(SPCG_ERR_UNSUPPORTED, "generated nnz exceeds int32");
    ptr[(size_t)i + 1] = (int)acc;
  }
  if ((rc = upload_seg(s, (int)n, ptr, nullptr, nullptr, acc, acct))) return rc;
  stencil_fill_kernel<<<grid, 256>>>(kind, part, row0, n, nx, ny, nz, s.ptr, s.idx, s.val);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaDeviceSynchronize());
  return SPCG_OK;
}


// ---- NCCL, loaded at run time ---------------------------------------------
// dlopen keeps the library loadable without NCCL and lets it share the NCCL
// a host framework (torch) already loaded (RTLD_NOLOAD first).
struct NcclApi {
  bool ok = false;
  std::string err;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
};

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return a;
    }
#define SPCG_NCCL_SYM(f)                                     \
  a.f = reinterpret_cast<decltype(a.f)>(dlsym(h, "nccl" #f)); \
  if (!a.f) {                                                \
    a.err = "libnccl.so.2 lacks nccl" #f;                    \
    return a;                                                \
  }
    SPCG_NCCL_SYM(GetUniqueId)
    SPCG_NCCL_SYM(CommInitRank)
    SPCG_NCCL_SYM(CommDestroy)
    SPCG_NCCL_SYM(AllReduce)
    SPCG_NCCL_SYM(Send)
    SPCG_NCCL_SYM(Recv)
    SPCG_NCCL_SYM(GroupStart)
    SPCG_NCCL_SYM(GroupEnd)
    SPCG_NCCL_SYM(GetErrorString)
#undef SPCG_NCCL_SYM
    a.ok = true;
    return a;
  }();
  return api;
}

#define NCCL_TRY(expr)                                                                   \
  do {                                                                                   \
    ncclResult_t _r = (expr);                                                            \
    if (_r != ncclSuccess)                                                               \
      return fail(SPCG_ERR_CUDA, std::string(#expr " failed: ") + nccl().GetErrorString(_r)); \
  } while (0)

// ---- row blocks ------------------------------------------------------------
// Rows [row0,row1) of an n_global system with GLOBAL column ids; becomes
// solvable after localize().
template <class IT>
int seg_from_host(int nrows, const IT* hp, const IT* hi, long long nnz, long long ncols,
                  std::vector<int>& ptr, std::vector<int>& idx) {
  ptr.assign((size_t)nrows + 1, 0);
  if (nrows > 0) {
    const long long base = (long long)hp[0];
    if ((long long)hp[nrows] - base != nnz) return fail(SPCG_ERR_ARG, "offsets do not span nnz");
    for (int i = 0; i <= nrows; ++i) {
      if (i > 0 && hp[i] < hp[i - 1]) return fail(SPCG_ERR_ARG, "offsets must be non-decreasing");
      ptr[(size_t)i] = (int)((long long)hp[i] - base);
    }
  }
  idx.resize((size_t)nnz);
  for (long long k = 0; k < nnz; ++k) {
    const long long c = (long long)hi[k];
    if (c < 0 || c >= ncols) return fail(SPCG_ERR_ARG, "column index out of range");
    idx[(size_t)k] = (int)c;
  }
  return SPCG_OK;
}

// Map global column ids to [0,nloc) (owned) / nloc + rank in the sorted halo
// list, for segment A (and B).  Host pass over the indices: O(nnz + n/64).
int localize(spcg_matrix_s* m) {
  if (!m->is_rows) return fail(SPCG_ERR_ARG, "localize needs a row-block matrix");
  if (m->localized) return SPCG_OK;
  const long long N = m->n_global, r0 = m->row0, r1 = m->row1;
  const size_t words = (size_t)((N + 63) / 64);
  std::vector<unsigned long long> bits(words, 0ull);
  Seg* segs[2] = {&m->A, m->hasB ? &m->B : nullptr};
  std::vector<std::vector<int>> host(2);
  for (int t = 0; t < 2; ++t) {
    if (!segs[t]) continue;
    host[t].resize((size_t)segs[t]->nnz);
    if (segs[t]->nnz)
      CUDA_TRY(cudaMemcpy(host[t].data(), segs[t]->idx, sizeof(int) * (size_t)segs[t]->nnz,
                          cudaMemcpyDeviceToHost));
    for (int c : host[t])
      if (c < r0 || c >= r1) bits[(size_t)c >> 6] |= 1ull << (c & 63);
  }
  std::vector<long long> prefix(words + 1, 0);
  for (size_t w = 0; w < words; ++w) prefix[w + 1] = prefix[w] + __builtin_popcountll(bits[w]);
  m->halo.clear();
  m->halo.reserve((size_t)prefix[words]);
  for (size_t w = 0; w < words; ++w)
    for (unsigned long long b = bits[w]; b; b &= b - 1)
      m->halo.push_back((long long)(w * 64 + __builtin_ctzll(b)));
  const long long nloc = r1 - r0;
  if (nloc + (long long)m->halo.size() >= (1LL << 31) - 16)
    return fail(SPCG_ERR_UNSUPPORTED, "local extended vector exceeds int32");
  for (int t = 0; t < 2; ++t) {
    if (!segs[t]) continue;
    for (int& c : host[t]) {
      if (c >= r0 && c < r1) {
        c = (int)(c - r0);
      } else {
        const size_t w = (size_t)c >> 6;
        const unsigned long long below = bits[w] & ((1ull << (c & 63)) - 1ull);
        c = (int)(nloc + prefix[w] + __builtin_popcountll(below));
      }
    }
    if (segs[t]->nnz)
      CUDA_TRY(cudaMemcpy(segs[t]->idx, host[t].data(), sizeof(int) * (size_t)segs[t]->nnz,
                          cudaMemcpyHostToDevice));
  }
  m->localized = true;
  return refresh_windows(m);
}

int ensure_dist_ws(spcg_matrix_s* m, long long send_total) {
  DistWorkspace& d = m->dw;
  int rc;
  const long long next = (long long)m->n + (long long)m->halo.size();
  if (d.next != next) {
    for (double* q : {d.r_ext, d.p_ext[0], d.p_ext[1], d.tmp_ext, d.q, d.part})
      if (q) cudaFree(q);
    if (d.S) cudaFree(d.S);
    if (d.h_S) cudaFreeHost(d.h_S);
    if (d.ev0) cudaEventDestroy(d.ev0);
    if (d.ev1) cudaEventDestroy(d.ev1);
    const size_t eb = sizeof(double) * (size_t)std::max<long long>(1, next);
    if ((rc = dmalloc((void**)&d.r_ext, eb, nullptr))) return rc;
    if ((rc = dmalloc((void**)&d.p_ext[0], eb, nullptr))) return rc;
    if ((rc = dmalloc((void**)&d.p_ext[1], eb, nullptr))) return rc;
    if ((rc = dmalloc((void**)&d.tmp_ext, eb, nullptr))) return rc;
    // q is extended too: the single-pass SCSR scatter puts the transposed
    // contributions of halo columns in q[nloc ..] (reverse halo)
    if ((rc = dmalloc((void**)&d.q, eb, nullptr))) return rc;
    if ((rc = dmalloc((void**)&d.part, sizeof(double) * 4096, nullptr))) return rc;
    if ((rc = dmalloc((void**)&d.S, sizeof(StepState), nullptr))) return rc;
    CUDA_TRY(cudaMallocHost((void**)&d.h_S, sizeof(StepState)));
    CUDA_TRY(cudaEventCreate(&d.ev0));
    CUDA_TRY(cudaEventCreate(&d.ev1));
    d.next = next;
  }
  if (d.send_cap < std::max(1LL, send_total)) {
    if (d.send_buf) cudaFree(d.send_buf);
    if (d.send_idx) cudaFree(d.send_idx);
    d.send_buf = nullptr;
    d.send_idx = nullptr;
    d.send_cap = std::max(1LL, send_total);
    if ((rc = dmalloc((void**)&d.send_buf, sizeof(double) * (size_t)d.send_cap, nullptr))) return rc;
    if ((rc = dmalloc((void**)&d.send_idx, sizeof(int) * (size_t)d.send_cap, nullptr))) return rc;
  }
  return SPCG_OK;
}

struct HaloPlan {
  ncclComm_t comm = nullptr;
  const spcg_comm_s* hc = nullptr;  // host-callback transport when set
  int npeers = 0;
  const int32_t* peers = nullptr;
  const int64_t* recv_off = nullptr;
  const int64_t* send_off = nullptr;
  long long nloc = 0;
};

// Pack v at the send rows, then exchange into dst_ext's halo.
// Host-callback transport: stage the send buffer, exchange through the
// caller's sendrecv, upload the received halo.  Synchronous (bring-up/tests).
int host_sendrecv(const HaloPlan& H, const double* d_send, double* d_recv, const int64_t* soff,
                  const int64_t* roff, cudaStream_t st) {
  const long long sn = soff[H.npeers], rn = roff[H.npeers];
  std::vector<double> hs((size_t)std::max(1LL, sn)), hr((size_t)std::max(1LL, rn));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (sn) CUDA_TRY(cudaMemcpy(hs.data(), d_send, sizeof(double) * (size_t)sn, cudaMemcpyDeviceToHost));
  if (H.hc->host_sr(H.npeers, H.peers, hs.data(), soff, hr.data(), roff, H.hc->host_user) != 0)
    return fail(SPCG_ERR_CUDA, "host sendrecv callback failed");
  if (rn) CUDA_TRY(cudaMemcpy(d_recv, hr.data(), sizeof(double) * (size_t)rn, cudaMemcpyHostToDevice));
  return SPCG_OK;
}

int halo_exchange(const HaloPlan& H, DistWorkspace& d, const double* v, double* dst_ext,
                  cudaStream_t st, long long* launches) {
  if (H.npeers == 0) return SPCG_OK;
  const long long total = H.send_off[H.npeers];
  if (total > 0) {
    const int g = (int)std::min<long long>(1184, (total + 255) / 256);
    dist_pack<<<g, 256, 0, st>>>(total, d.send_idx, v, d.send_buf);
    CUDA_TRY(cudaGetLastError());
    ++*launches;
  }
  if (H.hc) return host_sendrecv(H, d.send_buf, dst_ext + H.nloc, H.send_off, H.recv_off, st);
  NcclApi& N = nccl();
  NCCL_TRY(N.GroupStart());
  for (int k = 0; k < H.npeers; ++k) {
    const long long sc = H.send_off[k + 1] - H.send_off[k];
    const long long rc = H.recv_off[k + 1] - H.recv_off[k];
    if (sc > 0)
      NCCL_TRY(N.Send(d.send_buf + H.send_off[k], (size_t)sc, ncclDouble, H.peers[k], H.comm, st));
    if (rc > 0)
      NCCL_TRY(N.Recv(dst_ext + H.nloc + H.recv_off[k], (size_t)rc, ncclDouble, H.peers[k], H.comm,
                      st));
  }
  NCCL_TRY(N.GroupEnd());
  return SPCG_OK;
}

// Reverse halo: ghost partial sums q[nloc + recv_off[k] ..] go back to
// their owner k, which adds them at its send rows; ghosts are then zeroed
// for the next scatter.
int reverse_halo(const HaloPlan& H, DistWorkspace& d, double* q, long long nhalo,
                 cudaStream_t st, long long* launches) {
  if (H.npeers == 0) return SPCG_OK;
  if (H.hc) {  // roles swapped: ghosts (halo order) out, owner rows (send order) in
    int rc;
    if ((rc = host_sendrecv(H, q + H.nloc, d.send_buf, H.recv_off, H.send_off, st))) return rc;
  } else {
    NcclApi& N = nccl();
    NCCL_TRY(N.GroupStart());
    for (int k = 0; k < H.npeers; ++k) {
      const long long sc = H.send_off[k + 1] - H.send_off[k];
      const long long rc = H.recv_off[k + 1] - H.recv_off[k];
      if (rc > 0)
        NCCL_TRY(N.Send(q + H.nloc + H.recv_off[k], (size_t)rc, ncclDouble, H.peers[k], H.comm, st));
      if (sc > 0)
        NCCL_TRY(N.Recv(d.send_buf + H.send_off[k], (size_t)sc, ncclDouble, H.peers[k], H.comm, st));
    }
    NCCL_TRY(N.GroupEnd());
  }
  const long long total = H.send_off[H.npeers];
  if (total > 0) {
    const int g = (int)std::min<long long>(1184, (total + 255) / 256);
    dist_unpack_add<<<g, 256, 0, st>>>(total, d.send_idx, d.send_buf, q);
    CUDA_TRY(cudaGetLastError());
    ++*launches;
  }
  if (nhalo > 0) CUDA_TRY(cudaMemsetAsync(q + H.nloc, 0, sizeof(double) * (size_t)nhalo, st));
  return SPCG_OK;
}

int allreduce_red(const HaloPlan& H, StepState* S, cudaStream_t st) {
  if (H.hc) {
    double v = 0.0;
    CUDA_TRY(cudaStreamSynchronize(st));
    CUDA_TRY(cudaMemcpy(&v, &S->red, sizeof(double), cudaMemcpyDeviceToHost));
    if (H.hc->host_ar(&v, 1, H.hc->host_user) != 0)
      return fail(SPCG_ERR_CUDA, "host allreduce callback failed");
    CUDA_TRY(cudaMemcpy(&S->red, &v, sizeof(double), cudaMemcpyHostToDevice));
    return SPCG_OK;
  }
  if (!H.comm) return SPCG_OK;
  NCCL_TRY(nccl().AllReduce(&S->red, &S->red, 1, ncclDouble, ncclSum, H.comm, st));
  return SPCG_OK;
}

template <int FMT>
int dist_solve_t(spcg_matrix_s* m, const HaloPlan& H, const double* b, const double* x0, double* x,
                 double* hist, const spcg_cg_options* o, spcg_cg_result* out, cudaStream_t st) {
  DevInfo* di;
  int rc;
  if ((rc = dev_info(&di))) return rc;
  DistWorkspace& d = m->dw;
  const MatView v = view(m, FMT == K_SCSR_PRIV);
  const long long nloc = m->n, next = d.next;
  const int G = std::max(1, std::min(std::max(1, v.ntiles), di->spmv_grid));
  const int GE = 2 * di->sms;
  const size_t sm = sizeof(Smem);
  const int xv = (((uintptr_t)x) & 15) == 0;
  constexpr int kAtom = (FMT == K_SCSR_ATOMIC || FMT == K_CSC) ? 1 : 0;
  double* p = d.p_ext[0];  // p_ext = [own p | halo]
  double* r = d.r_ext;
  long long launches = 0;
  StepState init{};
  init.tol = o->tol;
  init.max_it = o->max_iter > 0 ? o->max_iter
                                : std::max<long long>(1, std::max<long long>(m->n_global, m->n));
  init.record = o->record_history && hist;
  init.x0_given = x0 != nullptr;
  CUDA_TRY(cudaMemcpyAsync(d.S, &init, sizeof(StepState), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemsetAsync(p, 0, sizeof(double) * (size_t)next, st));
  if (kAtom) CUDA_TRY(cudaMemsetAsync(d.q, 0, sizeof(double) * (size_t)std::max(1LL, next), st));
  const long long nhalo = next - nloc;
  constexpr bool kRev = (FMT == K_SCSR_ATOMIC);  // transposed scatters reach halo rows
  CUDA_TRY(cudaEventRecord(d.ev0, st));
  // ||b|| (solver.py:107)
  dist_elem<<<GE, kBlock, 0, st>>>(0, nloc, d.S, b, nullptr, nullptr, nullptr, d.part, 0);
  if ((rc = allreduce_red(H, d.S, st))) return rc;
  dist_scalar<<<1, 1, 0, st>>>(0, d.S, hist);
  // x = x0, r = b - A x0, p = r (solver.py:120-124)
  dist_x<<<GE, kBlock, 0, st>>>(0, nloc, d.S, x0, x);
  launches += 3;
  if (x0) {
    CUDA_TRY(cudaMemcpyAsync(d.tmp_ext, x0, sizeof(double) * (size_t)nloc,
                             cudaMemcpyDeviceToDevice, st));
    if ((rc = halo_exchange(H, d, x0, d.tmp_ext, st, &launches))) return rc;
    dist_spmv<FMT><<<G, kBlock, sm, st>>>(v, d.tmp_ext, d.q);
    if (kRev && (rc = reverse_halo(H, d, d.q, nhalo, st, &launches))) return rc;
    dist_elem<<<GE, kBlock, 0, st>>>(1, nloc, d.S, b, d.q, r, p, d.part, kAtom);
    launches += 2;
  } else {
    dist_elem<<<GE, kBlock, 0, st>>>(1, nloc, d.S, b, nullptr, r, p, d.part, 0);
    ++launches;
  }
  if ((rc = allreduce_red(H, d.S, st))) return rc;
  dist_scalar<<<1, 1, 0, st>>>(1, d.S, hist);
  ++launches;
  if ((rc = halo_exchange(H, d, p, p, st, &launches))) return rc;
  CUDA_TRY(cudaGetLastError());
  // CG loop; the host enqueues chunks of iterations and polls the device-side
  // done flag between chunks (iterations after `done` are no-ops on every
  // rank, so the NCCL calls stay matched)
  const int chunk = 16;
  const bool timing = o->timing != 0;
  if (timing && !d.tev[0][0])
    for (int a = 0; a < 2; ++a)
      for (int c = 0; c < chunk; ++c) CUDA_TRY(cudaEventCreate(&d.tev[a][c]));
  double spmv_ms = 0.0;
  long long spmv_n = 0, k_before = 0, iter_enq = 0;
#ifndef SPCG_ALTERNATE
#define SPCG_ALTERNATE 1
#endif
  constexpr bool kAlternate = SPCG_ALTERNATE != 0;
  for (;;) {
    for (int c = 0; c < chunk; ++c) {
      if (timing) CUDA_TRY(cudaEventRecord(d.tev[0][c], st));
      // alternate traversal directions pass to pass (A, B, C, A, ...): each
      // pass starts on the lines the previous one wrote last (still in L2)
      const int dirA = kAlternate ? (int)((iter_enq & 1) == 0) : 0;
      MatView va = v;
      va.rev = dirA;
      va.tree = o->row_sums == 0;  // auto: reassociated long-row sums in pass A
      dist_spmv_pq<FMT><<<G, kBlock, sm, st>>>(va, d.S, p, d.q, d.part);
      if (timing) CUDA_TRY(cudaEventRecord(d.tev[1][c], st));
      if ((rc = allreduce_red(H, d.S, st))) return rc;
      if (kRev && (rc = reverse_halo(H, d, d.q, nhalo, st, &launches))) return rc;
      dist_scalar<<<1, 1, 0, st>>>(2, d.S, hist);
      dist_elem<<<GE, kBlock, 0, st>>>(2, nloc, d.S, nullptr, d.q, r, nullptr, d.part, kAtom,
                                       kAlternate ? 1 - dirA : 0);
      if ((rc = allreduce_red(H, d.S, st))) return rc;
      dist_scalar<<<1, 1, 0, st>>>(3, d.S, hist);
      dist_update<<<GE, kBlock, 0, st>>>(nloc, d.S, r, p, x, xv, dirA);
      ++iter_enq;
      launches += 5;
      if ((rc = halo_exchange(H, d, p, p, st, &launches))) return rc;
    }
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(d.h_S, d.S, sizeof(StepState), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (timing) {  // only the passes that did work (later ones returned at once)
      const long long ran = std::min<long long>(chunk, d.h_S->k - k_before +
                                                           (d.h_S->status != 0 ? 1 : 0));
      for (long long c = 0; c < ran; ++c) {
        float t = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&t, d.tev[0][c], d.tev[1][c]));
        spmv_ms += t;
        ++spmv_n;
      }
      k_before = d.h_S->k;
    }
    if (d.h_S->done) break;
  }
  // a converged solve skipped its pass C: x += alpha_K p_K; then the true residual
  dist_x<<<GE, kBlock, 0, st>>>(1, nloc, d.S, p, x);
  ++launches;
  if (o->recompute_final_residual && d.h_S->status == 0 && d.h_S->b_norm != 0.0) {
    CUDA_TRY(cudaMemcpyAsync(d.tmp_ext, x, sizeof(double) * (size_t)nloc,
                             cudaMemcpyDeviceToDevice, st));
    if ((rc = halo_exchange(H, d, x, d.tmp_ext, st, &launches))) return rc;
    dist_spmv<FMT><<<G, kBlock, sm, st>>>(v, d.tmp_ext, d.q);
    if (kRev && (rc = reverse_halo(H, d, d.q, nhalo, st, &launches))) return rc;
    dist_elem<<<GE, kBlock, 0, st>>>(3, nloc, d.S, b, d.q, nullptr, nullptr, d.part, 0);
    if ((rc = allreduce_red(H, d.S, st))) return rc;
    dist_true_rel<<<1, 1, 0, st>>>(d.S);
    launches += 3;
  }
  CUDA_TRY(cudaEventRecord(d.ev1, st));
  CUDA_TRY(cudaMemcpyAsync(d.h_S, d.S, sizeof(StepState), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  CUDA_TRY(cudaGetLastError());
  float ms = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&ms, d.ev0, d.ev1));
  const StepState& S = *d.h_S;
  out->iterations = S.k;
  out->converged = S.converged;
  out->status = S.status;
  out->fail_iteration = S.fail_iter;
  out->final_relative_residual = S.rel;
  out->b_norm = S.b_norm;
  out->device_ms = ms;
  out->kernel_launches = launches;
  out->spmv_ms = spmv_ms;
  out->spmv_launches = spmv_n;
  if (S.status != 0) {
    const char* what = S.status == SPCG_ERR_NOT_SPD ? "matrix not positive definite"
                       : S.status == SPCG_ERR_NONFINITE_ALPHA ? "non-finite alpha"
                       : S.status == SPCG_ERR_NONFINITE_RESIDUAL ? "non-finite residual"
                                                                  : "non-finite beta";
    return fail(S.status, std::string(what) + " at iteration " + std::to_string(S.fail_iter));
  }
  return SPCG_OK;
}

int do_dist_cg(spcg_matrix_s* m, spcg_comm_s* comm, int npeers, const int32_t* peers,
               const int64_t* recv_off, const int64_t* send_off, const int32_t* send_idx,
               const double* b, const double* x0, double* x, double* hist,
               const spcg_cg_options* o, spcg_cg_result* out, cudaStream_t st) {
  if (!(o->tol > 0.0)) return fail(SPCG_ERR_ARG, "tol must be > 0");
  // single GPU: every format; sharded: CSR, owner-computes SCSR, and the
  // single-pass SCSR whose transposed scatters into halo rows travel back to
  // their owners (reverse halo)
  const int kf = kfmt_of(m, o->accumulation);
  if (npeers > 0 && kf == K_CSC) return fail(SPCG_ERR_UNSUPPORTED, "sharded CSC is not supported");
  if (kf == K_SCSR_PRIV && !m->hasB) return fail(SPCG_ERR_UNSUPPORTED, "SCSR needs its L^T rows");
  if (m->is_rows && !m->localized) return fail(SPCG_ERR_ARG, "call spcg_matrix_localize first");
  const bool host_comm = comm && comm->host_ar;
  if (npeers > 0 && (!comm || (!comm->comm && !host_comm)))
    return fail(SPCG_ERR_ARG, "peers need a communicator");
  if (npeers > 0 && !host_comm && !nccl().ok) return fail(SPCG_ERR_CUDA, nccl().err);
  if (o->record_history && !hist) return fail(SPCG_ERR_ARG, "record_history needs a history buffer");
  HaloPlan H;
  H.comm = comm ? comm->comm : nullptr;
  H.hc = (comm && comm->host_ar) ? comm : nullptr;
  H.npeers = npeers;
  H.peers = peers;
  H.recv_off = recv_off;
  H.send_off = send_off;
  H.nloc = m->n;
  const long long nhalo = (long long)m->halo.size();
  if (npeers > 0 && recv_off[npeers] != nhalo)
    return fail(SPCG_ERR_ARG, "receive plan does not cover the halo");
  const long long send_total = npeers > 0 ? send_off[npeers] : 0;
  int rc;
  if ((rc = ensure_dist_ws(m, send_total))) return rc;
  if (send_total > 0) {
    for (long long s = 0; s < send_total; ++s)
      if (send_idx[s] < 0 || send_idx[s] >= m->n) return fail(SPCG_ERR_ARG, "send index out of range");
    CUDA_TRY(cudaMemcpyAsync(m->dw.send_idx, send_idx, sizeof(int) * (size_t)send_total,
                             cudaMemcpyHostToDevice, st));
  }
  if (m->n == 0 && npeers == 0) {
    out->iterations = 0;
    out->converged = 1;
    out->status = 0;
    out->final_relative_residual = 0.0;
    return SPCG_OK;
  }
  switch (kf) {
    case K_CSR: return dist_solve_t<K_CSR>(m, H, b, x0, x, hist, o, out, st);
    case K_SCSR_PRIV: return dist_solve_t<K_SCSR_PRIV>(m, H, b, x0, x, hist, o, out, st);
    case K_SCSR_ATOMIC: return dist_solve_t<K_SCSR_ATOMIC>(m, H, b, x0, x, hist, o, out, st);
    default: return dist_solve_t<K_CSC>(m, H, b, x0, x, hist, o, out, st);
  }
}
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
  static thread_local double* part = nullptr;
  static thread_local int part_dev = -1;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (part == nullptr || part_dev != dev) {
    CUDA_TRY(cudaMalloc((void**)&part, sizeof(double) * 4096));
    part_dev = dev;
  }
  const int nb = (int)std::min<long long>(2LL * d->sms, (n + kBlock - 1) / kBlock);
  dot_partial_kernel<<<nb, kBlock, 0, st>>>(n, d_u, d_v, part);
  CUDA_TRY(cudaGetLastError());
  dot_final_kernel<<<1, kBlock, 0, st>>>(nb, part, d_out);
  CUDA_TRY(cudaGetLastError());
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
  std::lock_guard<std::mutex> lk(m->mu);
  return do_cg(m, d_b, d_x0, d_x, d_hist, opts, result, (cudaStream_t)stream);
}

int spcg_cg_solve_host(spcg_matrix_t m, const double* h_b, const double* h_x0, double* h_x,
                       double* h_hist, const spcg_cg_options* opts, spcg_cg_result* result,
                       void* stream) {
  if (!m || !opts || !result) return fail(SPCG_ERR_ARG, "null argument");
  if (m->n > 0 && (!h_b || !h_x)) return fail(SPCG_ERR_ARG, "null vector");
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
  if (m->n) CUDA_TRY(cudaMemcpyAsync(w.b, h_b, nb, cudaMemcpyHostToDevice, st));
  if (h_x0 && m->n) CUDA_TRY(cudaMemcpyAsync(w.x0, h_x0, nb, cudaMemcpyHostToDevice, st));
  rc = do_cg(m, w.b, h_x0 ? w.x0 : nullptr, w.x, opts->record_history ? w.hist : nullptr, opts,
             result, st);
  if (rc != SPCG_OK && rc != SPCG_ERR_NOT_SPD && rc != SPCG_ERR_NONFINITE_ALPHA &&
      rc != SPCG_ERR_NONFINITE_RESIDUAL && rc != SPCG_ERR_NONFINITE_BETA)
    return rc;
  const std::string err = g_last_error;
  if (m->n) CUDA_TRY(cudaMemcpyAsync(h_x, w.x, nb, cudaMemcpyDeviceToHost, st));
  if (opts->record_history && h_hist && result->iterations > 0)
    CUDA_TRY(cudaMemcpyAsync(h_hist, w.hist, sizeof(double) * (size_t)result->iterations,
                             cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
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
  if (nranks > 1) {
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
  std::lock_guard<std::mutex> lk(local->mu);
  return do_dist_cg(local, comm, npeers, peers, recv_off, send_off, send_idx, d_b, d_x0, d_x,
                    d_hist, opts, result, (cudaStream_t)stream);
}

}  // extern "C"
