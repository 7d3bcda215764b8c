// host_dist.cuh — host side of spcg_b200.cu: row-sharded solve: NCCL loading, localization, halo / reverse halo, per-pass engine.
// Included exactly once, by spcg_b200.cu inside its anonymous namespace
// (one translation unit: the kernels' templates are instantiated there).
#pragma once

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
    for (int c = 0; c < 2; ++c) {
      if (d.h_Sc[c]) cudaFreeHost(d.h_Sc[c]);
      if (d.cev[c]) cudaEventDestroy(d.cev[c]);
      d.h_Sc[c] = nullptr;
      d.cev[c] = nullptr;
    }
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
    for (int c = 0; c < 2; ++c) {
      CUDA_TRY(cudaMallocHost((void**)&d.h_Sc[c], sizeof(StepState)));
      CUDA_TRY(cudaEventCreateWithFlags(&d.cev[c], cudaEventDisableTiming));
    }
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
  const MatView v = view_stream(m, FMT == K_SCSR_PRIV);
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
  dist_elem<<<GE, kElemBlock, 0, st>>>(0, nloc, d.S, b, nullptr, nullptr, nullptr, d.part, 0);
  if ((rc = allreduce_red(H, d.S, st))) return rc;
  dist_scalar<<<1, 1, 0, st>>>(0, d.S, hist);
  // x = x0, r = b - A x0, p = r (solver.py:120-124)
  dist_x<<<GE, kElemBlock, 0, st>>>(0, nloc, d.S, x0, x);
  launches += 3;
  if (x0) {
    CUDA_TRY(cudaMemcpyAsync(d.tmp_ext, x0, sizeof(double) * (size_t)nloc,
                             cudaMemcpyDeviceToDevice, st));
    if ((rc = halo_exchange(H, d, x0, d.tmp_ext, st, &launches))) return rc;
    if (FMT == K_CSR && v.wide) dist_spmv<K_CSR, true><<<G, kBlock, sm, st>>>(v, d.tmp_ext, d.q);
    else dist_spmv<FMT><<<G, kBlock, sm, st>>>(v, d.tmp_ext, d.q);
    if (kRev && (rc = reverse_halo(H, d, d.q, nhalo, st, &launches))) return rc;
    dist_elem<<<GE, kElemBlock, 0, st>>>(1, nloc, d.S, b, d.q, r, p, d.part, kAtom);
    launches += 2;
  } else {
    dist_elem<<<GE, kElemBlock, 0, st>>>(1, nloc, d.S, b, nullptr, r, p, d.part, 0);
    ++launches;
  }
  if ((rc = allreduce_red(H, d.S, st))) return rc;
  dist_scalar<<<1, 1, 0, st>>>(1, d.S, hist);
  ++launches;
  if ((rc = halo_exchange(H, d, p, p, st, &launches))) return rc;
  CUDA_TRY(cudaGetLastError());
  // CG loop; the host enqueues chunks of iterations and polls the device-side
  // done flag of chunk c while chunk c + 1 is already queued (double
  // buffered), so the GPU never idles while the host enqueues.  Iterations
  // after `done` are no-ops on every rank, so the NCCL calls stay matched;
  // the one chunk enqueued past convergence costs only empty launches.
  const int chunk = 16;
  const bool timing = o->timing != 0;
  const bool split = o->timing >= 2;  // events around passes B and C too
  if (timing && !d.tev[0][0][0])
    for (int bb = 0; bb < 2; ++bb)
      for (int a = 0; a < 6; ++a)
        for (int c = 0; c < chunk; ++c) CUDA_TRY(cudaEventCreate(&d.tev[bb][a][c]));
  double spmv_ms = 0.0, axpy_ms = 0.0;
  long long spmv_n = 0, k_before = 0, iter_enq = 0;
#ifndef SPCG_ALTERNATE
#define SPCG_ALTERNATE 1
#endif
  constexpr bool kAlternate = SPCG_ALTERNATE != 0;
  auto enqueue_chunk = [&](int bb) -> int {
    for (int c = 0; c < chunk; ++c) {
      if (timing) CUDA_TRY(cudaEventRecord(d.tev[bb][0][c], st));
      // alternate traversal directions pass to pass (A, B, C, A, ...): each
      // pass starts on the lines the previous one wrote last (still in L2)
      const int dirA = kAlternate ? (int)((iter_enq & 1) == 0) : 0;
      MatView va = v;
      va.rev = dirA;
      va.tree = o->row_sums == 0;  // auto: reassociated long-row sums in pass A
      if (FMT == K_CSR && v.wide)
        dist_spmv_pq<K_CSR, true><<<G, kBlock, sm, st>>>(va, d.S, p, d.q, d.part);
      else
        dist_spmv_pq<FMT><<<G, kBlock, sm, st>>>(va, d.S, p, d.q, d.part);
      if (timing) CUDA_TRY(cudaEventRecord(d.tev[bb][1][c], st));
      int rc2;
      if ((rc2 = allreduce_red(H, d.S, st))) return rc2;
      if (kRev && (rc2 = reverse_halo(H, d, d.q, nhalo, st, &launches))) return rc2;
      dist_scalar<<<1, 1, 0, st>>>(2, d.S, hist);
      if (split) CUDA_TRY(cudaEventRecord(d.tev[bb][2][c], st));
      dist_elem<<<GE, kElemBlock, 0, st>>>(2, nloc, d.S, nullptr, d.q, r, nullptr, d.part, kAtom,
                                       kAlternate ? 1 - dirA : 0);
      if (split) CUDA_TRY(cudaEventRecord(d.tev[bb][3][c], st));
      if ((rc2 = allreduce_red(H, d.S, st))) return rc2;
      dist_scalar<<<1, 1, 0, st>>>(3, d.S, hist);
      if (split) CUDA_TRY(cudaEventRecord(d.tev[bb][4][c], st));
      dist_update<<<GE, kElemBlock, 0, st>>>(nloc, d.S, r, p, x, xv, dirA);
      if (split) CUDA_TRY(cudaEventRecord(d.tev[bb][5][c], st));
      ++iter_enq;
      launches += 5;
      if ((rc2 = halo_exchange(H, d, p, p, st, &launches))) return rc2;
    }
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(d.h_Sc[bb], d.S, sizeof(StepState), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaEventRecord(d.cev[bb], st));
    return SPCG_OK;
  };
  // the host-callback transport synchronises inside every exchange: no
  // point (and no room) for a second chunk in flight
  const bool two = H.hc == nullptr;
  if ((rc = enqueue_chunk(0))) return rc;
  for (long long ci = 0;; ++ci) {
    const int bb = (int)(ci & 1);
    if (two && (rc = enqueue_chunk(bb ^ 1))) return rc;
    CUDA_TRY(cudaEventSynchronize(d.cev[bb]));
    const StepState& hs = *d.h_Sc[bb];
    if (timing) {  // only the passes that did work (later ones returned at once)
      const long long ran = std::min<long long>(chunk, hs.k - k_before + (hs.status != 0 ? 1 : 0));
      for (long long c = 0; c < ran; ++c) {
        float t = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&t, d.tev[bb][0][c], d.tev[bb][1][c]));
        spmv_ms += t;
        ++spmv_n;
        if (split) {
          float tb = 0.f, tc = 0.f;
          CUDA_TRY(cudaEventElapsedTime(&tb, d.tev[bb][2][c], d.tev[bb][3][c]));
          CUDA_TRY(cudaEventElapsedTime(&tc, d.tev[bb][4][c], d.tev[bb][5][c]));
          axpy_ms += (double)tb + (double)tc;
        }
      }
      k_before = hs.k;
    }
    if (hs.done) {
      *d.h_S = hs;
      break;
    }
    if (!two && (rc = enqueue_chunk(bb ^ 1))) return rc;
  }
  // a converged solve skipped its pass C: x += alpha_K p_K; then the true residual
  dist_x<<<GE, kElemBlock, 0, st>>>(1, nloc, d.S, p, x);
  ++launches;
  if (o->recompute_final_residual && d.h_S->status == 0 && d.h_S->b_norm != 0.0) {
    CUDA_TRY(cudaMemcpyAsync(d.tmp_ext, x, sizeof(double) * (size_t)nloc,
                             cudaMemcpyDeviceToDevice, st));
    if ((rc = halo_exchange(H, d, x, d.tmp_ext, st, &launches))) return rc;
    if (FMT == K_CSR && v.wide) dist_spmv<K_CSR, true><<<G, kBlock, sm, st>>>(v, d.tmp_ext, d.q);
    else dist_spmv<FMT><<<G, kBlock, sm, st>>>(v, d.tmp_ext, d.q);
    if (kRev && (rc = reverse_halo(H, d, d.q, nhalo, st, &launches))) return rc;
    dist_elem<<<GE, kElemBlock, 0, st>>>(3, nloc, d.S, b, d.q, nullptr, nullptr, d.part, 0);
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
  out->engine_used = 2;
  out->fallbacks = 0;
  out->cond_estimate = 0.0;
  // split: SpMV passes (with the fused p.q partial); the vector-update passes
  // B and C (with the fused r.r partial); the rest (reductions' completion,
  // scalar steps, collectives, halo, prologue/epilogue) under "dot"
  out->phase_ms[0] = split ? spmv_ms : 0.0;
  out->phase_ms[2] = split ? axpy_ms : 0.0;
  out->phase_ms[1] = split ? std::max(0.0, (double)ms - spmv_ms - axpy_ms) : 0.0;
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
  // an empty shard with no peers may return at once only when it is alone:
  // with other ranks it must still join every collective of the solve
  const bool alone = !comm || comm->nranks <= 1;
  if (m->n == 0 && npeers == 0 && alone) {
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
