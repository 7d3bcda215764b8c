// host_assemble.cuh — host side of assemble.cuh: generator assembly in HBM and
// the device-side conversion / validation of uploaded CSR arrays.
// Included exactly once, by spcg_b200.cu inside its anonymous namespace.
#pragma once

// Scoped device allocations of the assembly (freed on every exit path).
struct DevTmp {
  std::vector<void*> p;
  template <class T>
  int get(T** out, size_t count) {
    void* q = nullptr;
    CUDA_TRY(cudaMalloc(&q, std::max<size_t>(1, count) * sizeof(T)));
    p.push_back(q);
    *out = static_cast<T*>(q);
    return SPCG_OK;
  }
  ~DevTmp() {
    for (void* q : p) cudaFree(q);
  }
};

template <class K, class V>
int radix_sort_pairs(DevTmp& T, const K* kin, K* kout, const V* vin, V* vout, long long count,
                     int end_bit) {
  if (count <= 0) return SPCG_OK;
  size_t bytes = 0;
  CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, (int)count, 0,
                                           end_bit));
  void* tmp = nullptr;
  int rc;
  if ((rc = T.get((unsigned char**)&tmp, bytes))) return rc;
  CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, bytes, kin, kout, vin, vout, (int)count, 0,
                                           end_bit));
  return SPCG_OK;
}

int bits_for(long long v) {
  int b = 1;
  while ((1LL << b) <= v) ++b;
  return b;
}

int asm_error(int err) {
  if (err & ASM_ERR_RANGE) return fail(SPCG_ERR_ARG, "pair outside 0 <= J < I < n");
  if (err & ASM_ERR_DUPLICATE) return fail(SPCG_ERR_ARG, "duplicate (row, col) entry");
  if (err & ASM_ERR_OFFSETS)
    return fail(SPCG_ERR_ARG, "offsets must start at 0, end at nnz and be non-decreasing");
  if (err & ASM_ERR_INDEX) return fail(SPCG_ERR_ARG, "index out of range");
  if (err & ASM_ERR_DIAG) return fail(SPCG_ERR_ARG, "a row has no stored diagonal entry");
  if (err & ASM_ERR_UPPER) return fail(SPCG_ERR_ARG, "symmetric-half storage requires col <= row");
  return SPCG_OK;
}

std::vector<int> host_prefix(const std::vector<int>& cnt) {
  std::vector<int> ptr(cnt.size() + 1, 0);
  for (size_t i = 0; i < cnt.size(); ++i) ptr[i + 1] = ptr[i] + cnt[i];
  return ptr;
}

// Generators: m mirrored pairs (I > J) with values v in draw order, diagonal
// = np.bincount order sums of |v| + shift (genprob.py:96-129).
int assemble_pairs(int fmt, int64_t n, int64_t m, const int64_t* hI, const int64_t* hJ,
                   const double* hv, double shift, spcg_matrix_t* out) {
  int rc;
  if ((rc = check_csr_host(fmt, n, 2 * m + n))) return rc;
  if (m < 0) return fail(SPCG_ERR_ARG, "negative pair count");
  if (m > 0 && (!hI || !hJ || !hv)) return fail(SPCG_ERR_ARG, "null arrays");
  DevInfo* di;
  if ((rc = dev_info(&di))) return rc;
  DevTmp T;
  long long *I, *J;
  double *v, *diag;
  int *rows, *ids, *rows_s, *ids_s, *seg, *err;
  if ((rc = T.get(&I, m)) || (rc = T.get(&J, m)) || (rc = T.get(&v, m)) || (rc = T.get(&diag, n)) ||
      (rc = T.get(&rows, 2 * m)) || (rc = T.get(&ids, 2 * m)) || (rc = T.get(&rows_s, 2 * m)) ||
      (rc = T.get(&ids_s, 2 * m)) || (rc = T.get(&seg, n + 1)) || (rc = T.get(&err, 1)))
    return rc;
  if (m > 0) {
    CUDA_TRY(cudaMemcpy(I, hI, sizeof(long long) * m, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(J, hJ, sizeof(long long) * m, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(v, hv, sizeof(double) * m, cudaMemcpyHostToDevice));
  }
  CUDA_TRY(cudaMemset(err, 0, sizeof(int)));
  const int grid = 8 * di->sms;
  // diagonal: stable sort of the 2m entries by row, in-order sums per row
  std::vector<int> cnt((size_t)n, 0);
  if (m > 0) {
    asm_rows_kernel<<<grid, 256>>>(m, (int)n, I, J, rows, ids, err);
    CUDA_TRY(cudaGetLastError());
    if ((rc = radix_sort_pairs(T, rows, rows_s, ids, ids_s, 2 * m, bits_for(n)))) return rc;
    CUDA_TRY(cudaMemset(seg, 0, sizeof(int) * (size_t)(n + 1)));
    asm_hist_kernel<<<grid, 256>>>(2 * m, rows_s, seg);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpy(cnt.data(), seg, sizeof(int) * (size_t)n, cudaMemcpyDeviceToHost));
  }
  {
    const std::vector<int> off = host_prefix(cnt);
    CUDA_TRY(cudaMemcpy(seg, off.data(), sizeof(int) * off.size(), cudaMemcpyHostToDevice));
  }
  asm_diag_kernel<<<grid, 256>>>((int)n, seg, ids_s, m, v, shift, diag);
  CUDA_TRY(cudaGetLastError());
  // all entries sorted by (row, col): CSR / CSC (the symmetric arrays) or
  // SCSR = the col <= row part, with the col > row part as L^T
  const bool scsr = fmt == SPCG_FMT_SCSR;
  const long long total = 2 * m + n;
  unsigned long long *keys, *keys_s;
  int *vid, *vid_s, *cA, *cB;
  if ((rc = T.get(&keys, total)) || (rc = T.get(&keys_s, total)) || (rc = T.get(&vid, total)) ||
      (rc = T.get(&vid_s, total)) || (rc = T.get(&cA, n)) || (rc = T.get(&cB, n)))
    return rc;
  asm_keys_kernel<<<grid, 256>>>(m, (int)n, I, J, 0, keys, vid);
  CUDA_TRY(cudaGetLastError());
  if ((rc = radix_sort_pairs(T, keys, keys_s, vid, vid_s, total, 32 + bits_for(n)))) return rc;
  CUDA_TRY(cudaMemset(cA, 0, sizeof(int) * (size_t)std::max<int64_t>(1, n)));
  CUDA_TRY(cudaMemset(cB, 0, sizeof(int) * (size_t)std::max<int64_t>(1, n)));
  asm_count_kernel<<<grid, 256>>>(total, keys_s, scsr ? 1 : 0, cA, cB, err);
  CUDA_TRY(cudaGetLastError());
  int herr = 0;
  CUDA_TRY(cudaMemcpy(&herr, err, sizeof(int), cudaMemcpyDeviceToHost));
  if (herr) return asm_error(herr);
  std::vector<int> hA((size_t)n), hB((size_t)n);
  CUDA_TRY(cudaMemcpy(hA.data(), cA, sizeof(int) * (size_t)n, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(hB.data(), cB, sizeof(int) * (size_t)n, cudaMemcpyDeviceToHost));
  const std::vector<int> ptrA = host_prefix(hA), ptrB = host_prefix(hB);
  spcg_matrix_s* M = new spcg_matrix_s();
  M->fmt = fmt;
  M->n = (int)n;
  M->nnz = ptrA.back();
  CUDA_TRY(cudaGetDevice(&M->device));
  auto bail = [&](int code) {
    free_matrix(M);
    delete M;
    return code;
  };
  if ((rc = upload_seg(M->A, (int)n, ptrA, nullptr, nullptr, ptrA.back(), &M->bytes))) return bail(rc);
  if (scsr && (rc = upload_seg(M->B, (int)n, ptrB, nullptr, nullptr, ptrB.back(), &M->bytes)))
    return bail(rc);
  asm_scatter_kernel<<<grid, 256>>>(total, keys_s, vid_s, m, v, diag, M->A.ptr,
                                    scsr ? M->B.ptr : nullptr, M->A.idx, M->A.val,
                                    scsr ? M->B.idx : nullptr, scsr ? M->B.val : nullptr);
  if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
    return bail(fail(SPCG_ERR_CUDA, "assembly scatter failed"));
  if ((rc = finish_matrix(M, ptrA, nullptr, nullptr, true))) return bail(rc);
  if (scsr && (rc = finish_transpose(M, ptrA, ptrB, nullptr, nullptr, true))) return bail(rc);
  if ((rc = refresh_windows(M))) return bail(rc);
  *out = M;
  return SPCG_OK;
}

// Device arrays (offsets PT, indices IT, fp64 values) -> a matrix handle:
// conversion to int32 and the checks of create_from_host, on the device; for
// SCSR the privatized mode's L^T is built by a radix sort of the strict
// entries by (column, row).  The caller's arrays are not kept.
template <class PT, class IT>
int create_from_device(int fmt, int64_t n, int64_t nnz, const PT* dp, const IT* di_,
                       const double* dv, spcg_matrix_t* out) {
  int rc;
  if ((rc = check_csr_host(fmt, n, nnz))) return rc;
  if (nnz > 0 && (!di_ || !dv)) return fail(SPCG_ERR_ARG, "null arrays");
  if (!dp) return fail(SPCG_ERR_ARG, "null offsets");
  DevInfo* dinfo;
  if ((rc = dev_info(&dinfo))) return rc;
  const int grid = 8 * dinfo->sms;
  DevTmp T;
  int* err;
  int* p32;
  if ((rc = T.get(&err, 1)) || (rc = T.get(&p32, n + 1))) return rc;
  CUDA_TRY(cudaMemset(err, 0, sizeof(int)));
  conv_ptr_kernel<PT><<<grid, 256>>>(n, nnz, dp, p32, err);
  CUDA_TRY(cudaGetLastError());
  int herr = 0;
  CUDA_TRY(cudaMemcpy(&herr, err, sizeof(int), cudaMemcpyDeviceToHost));
  if (herr) return asm_error(herr);
  std::vector<int> ptr((size_t)n + 1);
  CUDA_TRY(cudaMemcpy(ptr.data(), p32, sizeof(int) * ptr.size(), cudaMemcpyDeviceToHost));
  spcg_matrix_s* M = new spcg_matrix_s();
  M->fmt = fmt;
  M->n = (int)n;
  M->nnz = nnz;
  CUDA_TRY(cudaGetDevice(&M->device));
  auto bail = [&](int code) {
    free_matrix(M);
    delete M;
    return code;
  };
  if ((rc = upload_seg(M->A, (int)n, ptr, nullptr, nullptr, nnz, &M->bytes))) return bail(rc);
  if (nnz > 0) {
    CUDA_TRY(cudaMemcpy(M->A.val, dv, sizeof(double) * (size_t)nnz, cudaMemcpyDeviceToDevice));
  }
  const bool scsr = fmt == SPCG_FMT_SCSR;
  unsigned long long* tk = nullptr;
  int *tv = nullptr, *tcount = nullptr;
  if (scsr && ((rc = T.get(&tk, nnz)) || (rc = T.get(&tv, nnz)) || (rc = T.get(&tcount, 1))))
    return bail(rc);
  if (scsr) CUDA_TRY(cudaMemset(tcount, 0, sizeof(int)));
  if (n > 0) {
    conv_idx_kernel<IT><<<grid, 256>>>((int)n, scsr ? 1 : 0, M->A.ptr, di_, M->A.idx, err, tk, tv,
                                       tcount);
    CUDA_TRY(cudaGetLastError());
  }
  CUDA_TRY(cudaMemcpy(&herr, err, sizeof(int), cudaMemcpyDeviceToHost));
  if (herr) return bail(asm_error(herr));
  if ((rc = finish_matrix(M, ptr, nullptr, nullptr, true))) return bail(rc);
  if (scsr) {
    int cnt = 0;
    CUDA_TRY(cudaMemcpy(&cnt, tcount, sizeof(int), cudaMemcpyDeviceToHost));
    unsigned long long* tks;
    int *tvs, *hist;
    if ((rc = T.get(&tks, cnt)) || (rc = T.get(&tvs, cnt)) || (rc = T.get(&hist, n))) return bail(rc);
    if ((rc = radix_sort_pairs(T, tk, tks, tv, tvs, cnt, 32 + bits_for(n)))) return bail(rc);
    CUDA_TRY(cudaMemset(hist, 0, sizeof(int) * (size_t)std::max<int64_t>(1, n)));
    if (cnt > 0) lt_hist_kernel<<<grid, 256>>>(cnt, tks, hist);
    std::vector<int> hc((size_t)n);
    CUDA_TRY(cudaMemcpy(hc.data(), hist, sizeof(int) * (size_t)n, cudaMemcpyDeviceToHost));
    const std::vector<int> tptr = host_prefix(hc);
    if ((rc = upload_seg(M->B, (int)n, tptr, nullptr, nullptr, cnt, &M->bytes))) return bail(rc);
    if (cnt > 0) lt_scatter_kernel<<<grid, 256>>>(cnt, tks, tvs, M->A.val, M->B.idx, M->B.val);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaDeviceSynchronize());
    if ((rc = finish_transpose(M, ptr, tptr, nullptr, nullptr, true))) return bail(rc);
  }
  if ((rc = refresh_windows(M))) return bail(rc);
  *out = M;
  return SPCG_OK;
}

template <class PT, class IT>
int create_from_host(int fmt, int64_t n, int64_t nnz, const PT* hp, const IT* hi, const double* hv,
                     spcg_matrix_t* out) {
  int rc;
  if ((rc = check_csr_host(fmt, n, nnz))) return rc;
  if (n > 0 && hp == nullptr) return fail(SPCG_ERR_ARG, "null offsets");
  if (nnz > 0 && (hi == nullptr || hv == nullptr)) return fail(SPCG_ERR_ARG, "null arrays");
  DevInfo* d;
  if ((rc = dev_info(&d))) return rc;
  DevTmp T;
  PT* dp;
  IT* dix;
  double* dv;
  if ((rc = T.get(&dp, n + 1)) || (rc = T.get(&dix, nnz)) || (rc = T.get(&dv, nnz))) return rc;
  if (n > 0) {
    CUDA_TRY(cudaMemcpy(dp, hp, sizeof(PT) * (size_t)(n + 1), cudaMemcpyHostToDevice));
  } else {
    CUDA_TRY(cudaMemset(dp, 0, sizeof(PT)));
  }
  if (nnz > 0) {
    CUDA_TRY(cudaMemcpy(dix, hi, sizeof(IT) * (size_t)nnz, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(dv, hv, sizeof(double) * (size_t)nnz, cudaMemcpyHostToDevice));
  }
  return create_from_device(fmt, n, nnz, dp, dix, dv, out);
}
