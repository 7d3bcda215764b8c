// host_matrix.cuh — host side of spcg_b200.cu: matrix handles: uploads, row tiles, windows, workspaces, single-GPU launchers.
// Included exactly once, by spcg_b200.cu inside its anonymous namespace
// (one translation unit: the kernels' templates are instantiated there).
#pragma once

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
  const int cap = tile_line_cap(m->n ? ptr[m->n] : 0, m->n);
  build_tiles(m->n, ptr, nullptr, target, desc, nullptr, cap);
  if ((rc = upload_tiles(m->t1, desc, nullptr, &m->bytes))) return rc;
  // wide tiles only where their second line slot fills well (>= 3/4 of a
  // kTileLines tile at the average row length: P2's 5-entry rows, not P3's
  // 7, where the mostly idle second slot cost 17 % on the 7-point stencil)
  const long long ent = m->n ? (long long)ptr[m->n] : 0;
  if (kWideLines > kTileLines && m->fmt == SPCG_FMT_CSR && cap == kTileLines && m->n > 0 &&
      ent * (long long)(kTileLines + kTileLines / 2) <= (long long)kTileNnz * m->n) {
    build_tiles(m->n, ptr, nullptr, target, desc, nullptr, kWideLines);
    if ((rc = upload_tiles(m->t1w, desc, nullptr, &m->bytes))) return rc;
  }
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
  F(m->t1.desc); F(m->t1.descB); F(m->t1w.desc); F(m->t2.desc); F(m->t2.descB); F(m->t1.win); F(m->t2.win);
  Workspace& w = m->ws;
  F(w.r); F(w.p0); F(w.p1); F(w.q); F(w.part); F(w.slots); F(w.res);
  F(w.b); F(w.x); F(w.x0); F(w.hist); F(w.cg1); F(w.coef);
  if (w.h_res) cudaFreeHost(w.h_res);
  if (w.h_coef) cudaFreeHost(w.h_coef);
  if (w.ev0) cudaEventDestroy(w.ev0);
  if (w.ev1) cudaEventDestroy(w.ev1);
  if (w.ev_res) cudaEventDestroy(w.ev_res);
  DistWorkspace& d = m->dw;
  F(d.r_ext); F(d.p_ext[0]); F(d.p_ext[1]); F(d.tmp_ext); F(d.q); F(d.part); F(d.S);
  F(d.send_buf); F(d.send_idx); F(d.args); F(d.ytx);
  F(m->cp.arena);  // every device array of the cluster plan
  if (d.h_S) cudaFreeHost(d.h_S);
  if (d.ev0) cudaEventDestroy(d.ev0);
  if (d.ev1) cudaEventDestroy(d.ev1);
  for (int bb = 0; bb < 2; ++bb) {
    if (d.h_Sc[bb]) cudaFreeHost(d.h_Sc[bb]);
    if (d.cev[bb]) cudaEventDestroy(d.cev[bb]);
    for (int a = 0; a < 6; ++a)
      for (int c = 0; c < 16; ++c)
        if (d.tev[bb][a][c]) cudaEventDestroy(d.tev[bb][a][c]);
  }
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

// Tile table of the streaming passes (per-pass engine, standalone SpMV):
// the wide table when the matrix has one.
MatView view_stream(const spcg_matrix_s* m, bool priv) {
  MatView v = view(m, priv);
  if (!priv && m->t1w.ntiles > 0) {
    v.ntiles = m->t1w.ntiles;
    v.tdesc = m->t1w.desc;
    v.tdescB = nullptr;
    v.twin = nullptr;
    v.wide = 1;
  }
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
    CUDA_TRY(cudaEventCreateWithFlags(&w.ev_res, cudaEventDisableTiming));
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
int launch_cg1(const Cg1Args& a, int grid, cudaStream_t st) {
  void* args[] = {(void*)&a};
  const void* fn = (const void*)cg1_kernel<FMT>;
  CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kBlock), args, kSmemRes, st));
  return SPCG_OK;
}

// engine 7: co-resident CTAs of cg1s_kernel<FMT> on this device (cooperative)
template <int FMT>
int cg1s_grid(const DevInfo* d, int* grid) {
  static int cached[64] = {0};
  int& c = cached[d->device & 63];
  if (c == 0) {
    int per_sm = 0;
    const void* fn = (const void*)cg1s_kernel<FMT>;
    CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem)));
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kBlock, sizeof(Smem)));
    // the grid all-reduce polls at most 384 slots (cg.cuh kPollPer)
    c = std::max(1, std::min(per_sm * d->sms, 384));
  }
  *grid = c;
  return SPCG_OK;
}
template <int FMT>
int launch_cg1s(const Cg1sArgs& a, int grid, cudaStream_t st) {
  void* args[] = {(void*)&a};
  CUDA_TRY(cudaLaunchCooperativeKernel((const void*)cg1s_kernel<FMT>, dim3(grid), dim3(kBlock), args,
                                       sizeof(Smem), st));
  return SPCG_OK;
}

template <int FMT>
int launch_spmv(const MatView& v, const double* x, double* y, int grid, cudaStream_t st) {
  if (FMT == K_CSR && v.wide) spmv_kernel<K_CSR, true><<<grid, kBlock, sizeof(Smem), st>>>(v, x, y);
  else spmv_kernel<FMT><<<grid, kBlock, sizeof(Smem), st>>>(v, x, y);
  CUDA_TRY(cudaGetLastError());
  return SPCG_OK;
}

int do_spmv(spcg_matrix_s* m, const double* x, double* y, int accumulation, cudaStream_t st) {
  DevInfo* d;
  int rc;
  if ((rc = dev_info(&d))) return rc;
  const int kf = kfmt_of(m, accumulation);
  if (kf == K_SCSR_PRIV && !m->hasB) return fail(SPCG_ERR_UNSUPPORTED, "no L^T for privatized mode");
  const MatView v = view_stream(m, kf == K_SCSR_PRIV);
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
