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

#include "../../include/spcg_b200.h"
#include "cg.cuh"
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
  // host-API staging
  double* b = nullptr;
  double* x = nullptr;
  double* x0 = nullptr;
  double* hist = nullptr;
  long long hist_cap = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

}  // namespace

struct spcg_matrix_s {
  int fmt = 0;
  int n = 0;
  long long nnz = 0;
  int device = 0;
  Seg A, B;
  bool hasB = false;
  Tiles t1, t2;
  long long bytes = 0;
  Workspace ws;
  std::mutex mu;  // one solve at a time per handle (workspace reuse)
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
                 std::vector<int4>& desc, std::vector<int2>* descB) {
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
  T = std::max<long long>(T, ((long long)n + kTileLines - 1) / kTileLines);
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
      int lim = std::min(e, a + kTileLines);
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

int target_tiles() {
  DevInfo* d = nullptr;
  if (dev_info(&d)) return 148;
  return d->sms;
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
  build_tiles(m->n, ptr, nullptr, target, desc, nullptr);
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
  build_tiles(m->n, ptr, &tptr, target_tiles(), desc, &descB);
  if ((rc = upload_tiles(m->t2, desc, &descB, &m->bytes))) return rc;
  m->hasB = true;
  return SPCG_OK;
}

void free_matrix(spcg_matrix_s* m) {
  auto F = [](void* p) {
    if (p) cudaFree(p);
  };
  F(m->A.ptr); F(m->A.idx); F(m->A.val);
  F(m->B.ptr); F(m->B.idx); F(m->B.val);
  F(m->t1.desc); F(m->t1.descB); F(m->t2.desc); F(m->t2.descB);
  Workspace& w = m->ws;
  F(w.r); F(w.p0); F(w.p1); F(w.q); F(w.part); F(w.slots); F(w.res);
  F(w.b); F(w.x); F(w.x0); F(w.hist);
  if (w.h_res) cudaFreeHost(w.h_res);
  if (w.ev0) cudaEventDestroy(w.ev0);
  if (w.ev1) cudaEventDestroy(w.ev1);
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
int launch_cg(const CgArgs& a, bool res, int grid, cudaStream_t st) {
  void* args[] = {(void*)&a};
  const void* fn = res ? (const void*)cg_kernel<FMT, true> : (const void*)cg_kernel<FMT, false>;
  CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kBlock), args,
                                       res ? kSmemRes : sizeof(Smem), st));
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

int do_cg(spcg_matrix_s* m, const double* b, const double* x0, double* x, double* hist,
          const spcg_cg_options* o, spcg_cg_result* out, cudaStream_t st) {
  DevInfo* d;
  int rc;
  if ((rc = dev_info(&d))) return rc;
  if (!(o->tol > 0.0)) return fail(SPCG_ERR_ARG, "tol must be > 0");
  const int kf = kfmt_of(m, o->accumulation);
  if (kf == K_SCSR_PRIV && !m->hasB) return fail(SPCG_ERR_UNSUPPORTED, "no L^T for privatized mode");
  const MatView v = view(m, kf == K_SCSR_PRIV);
  const bool res = o->engine != 2 && v.ntiles <= d->coop_res * kStages;
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
    CUDA_TRY(cudaMalloc((void**)&trace, sizeof(unsigned long long) * 4 * (size_t)grid));
    CUDA_TRY(cudaMemsetAsync(trace, 0, sizeof(unsigned long long) * 4 * (size_t)grid, st));
  }
  a.trace = trace;
  a.res = w.res;
  a.tol = o->tol;
  a.max_iter = max_iter;
  a.record_history = o->record_history;
  a.recompute = o->recompute_final_residual;
  CUDA_TRY(cudaEventRecord(w.ev0, st));
  switch (kf) {
    case K_CSR: rc = launch_cg<K_CSR>(a, res, grid, st); break;
    case K_SCSR_ATOMIC: rc = launch_cg<K_SCSR_ATOMIC>(a, res, grid, st); break;
    case K_SCSR_PRIV: rc = launch_cg<K_SCSR_PRIV>(a, res, grid, st); break;
    default: rc = launch_cg<K_CSC>(a, res, grid, st); break;
  }
  if (rc) return rc;
  CUDA_TRY(cudaEventRecord(w.ev1, st));
  CUDA_TRY(cudaMemcpyAsync(w.h_res, w.res, sizeof(CgDevResult), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  float ms = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&ms, w.ev0, w.ev1));
  const CgDevResult& r = *w.h_res;
  if (trace) {
    std::vector<unsigned long long> tv(4 * (size_t)grid);
    CUDA_TRY(cudaMemcpy(tv.data(), trace, sizeof(unsigned long long) * tv.size(),
                        cudaMemcpyDeviceToHost));
    cudaFree(trace);
    double mean[4] = {0, 0, 0, 0}, mx[4] = {0, 0, 0, 0};
    for (int b = 0; b < grid; ++b)
      for (int ph = 0; ph < 4; ++ph) {
        mean[ph] += (double)tv[4 * b + ph] / grid;
        mx[ph] = std::max(mx[ph], (double)tv[4 * b + ph]);
      }
    const double it = (double)std::max<long long>(1, r.iterations);
    fprintf(stderr,
            "[spcg trace] grid=%d res=%d iters=%lld us/iter mean(max): passA %.3f(%.3f) "
            "reduce1 %.3f(%.3f) passB %.3f(%.3f) reduce2 %.3f(%.3f)\n",
            grid, (int)res, r.iterations, mean[0] / it / 1e3, mx[0] / it / 1e3, mean[1] / it / 1e3,
            mx[1] / it / 1e3, mean[2] / it / 1e3, mx[2] / it / 1e3, mean[3] / it / 1e3,
            mx[3] / it / 1e3);
  }
  out->iterations = r.iterations;
  out->converged = r.converged;
  out->status = r.status;
  out->fail_iteration = r.fail_iter;
  out->final_relative_residual = r.final_rel;
  out->b_norm = r.b_norm;
  out->device_ms = ms;
  out->kernel_launches = 1;
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
  *out = m;
  return SPCG_OK;
}

// Device generator: counts -> host prefix sum -> ptr upload -> device fill.
int gen_seg(int kind, int part, long long n, int nx, int ny, int nz, Seg& s, std::vector<int>& ptr,
            long long* acct) {
  int rc;
  int* counts = nullptr;
  if ((rc = dmalloc((void**)&counts, sizeof(int) * (size_t)std::max<long long>(1, n), nullptr)))
    return rc;
  const int grid = 148 * 8;
  stencil_count_kernel<<<grid, 256>>>(kind, part, n, nx, ny, nz, counts);
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
  stencil_fill_kernel<<<grid, 256>>>(kind, part, n, nx, ny, nz, s.ptr, s.idx, s.val);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaDeviceSynchronize());
  return SPCG_OK;
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
  if ((rc = gen_seg(kind, part, n, (int)d0, (int)d1, (int)d2, m->A, ptr, &m->bytes)) ||
      (rc = finish_matrix(m, ptr, nullptr, nullptr, true))) {
    free_matrix(m);
    delete m;
    return rc;
  }
  m->nnz = m->A.nnz;
  if (fmt == SPCG_FMT_SCSR) {
    if ((rc = gen_seg(kind, 2, n, (int)d0, (int)d1, (int)d2, m->B, tptr, &m->bytes)) ||
        (rc = finish_transpose(m, ptr, tptr, nullptr, nullptr, true))) {
      free_matrix(m);
      delete m;
      return rc;
    }
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

}  // extern "C"
