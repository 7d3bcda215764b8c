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
    CUDA_TRY(cudaMemset(d.S, 0, sizeof(StepState)));
    if (!d.args && (rc = dmalloc((void**)&d.args, sizeof(DistArgs), nullptr))) return rc;
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

// ---- device-initiated transport: per-rank plan (spcg_dist_plan_t) ----------
// What peers write into lives in plain cudaMalloc allocations of this rank,
// exported by CUDA IPC (one process per GPU) or shared as raw pointers (ranks
// of one process on one GPU: the virtual-rank group launch).
struct P2PBlob {
  uint32_t magic, version;
  int32_t rank, nranks, device, pid;
  int64_t nloc, row0;
  int64_t recv_off_by_src[kMaxRanks];  // offset of src's values in my halo (-1: none)
  cudaIpcMemHandle_t h_mbox, h_hflag, h_p, h_tmp, h_q;
  uint64_t mbox, hflag, p, tmp, q;     // raw pointers (same-process connect)
};
static_assert(sizeof(P2PBlob) <= SPCG_P2P_BLOB_BYTES, "blob too large");
constexpr uint32_t kBlobMagic = 0x50324350u;  // "PC2P"

}  // namespace

struct spcg_dist_plan_s {
  spcg_matrix_s* m = nullptr;
  int rank = 0, nranks = 1;
  std::vector<int32_t> peers;
  std::vector<int64_t> recv_off, send_off;
  std::vector<int32_t> send_idx;
  unsigned long long* mbox = nullptr;   // [2][R][2]
  unsigned long long* hflag = nullptr;  // [R][2]
  unsigned char* thalo = nullptr;
  SendRun* runs = nullptr;
  int nruns = 0;
  int nrecv = 0, nsendpeers = 0;
  bool same_device = true;           // every peer mapped by pointer on this device
  int* send_peer = nullptr;
  long long* send_dst = nullptr;
  int* ghost_peer = nullptr;
  int* ghost_dst = nullptr;
  long long nghost = 0;
  bool connected = false;
  PeerTab peer{};                    // peer pointer tables (filled by connect)
  PeerTab* d_peer = nullptr;         // their device copy
  std::vector<void*> opened;         // IPC mappings to close
  DistArgs* d_args = nullptr;        // device copy for solo solves
};

namespace {

void free_plan(spcg_dist_plan_s* P) {
  for (void* q : P->opened) cudaIpcCloseMemHandle(q);
  P->opened.clear();
  for (void* q : {(void*)P->mbox, (void*)P->hflag, (void*)P->thalo, (void*)P->runs,
                  (void*)P->send_peer, (void*)P->send_dst, (void*)P->ghost_peer,
                  (void*)P->ghost_dst, (void*)P->d_args, (void*)P->d_peer})
    if (q) cudaFree(q);
}

// The streaming tile view of a (localized) handle and its per-tile halo flags.
MatView dist_view(const spcg_matrix_s* m, int kf) { return view_stream(m, kf == K_SCSR_PRIV); }

int build_thalo(spcg_matrix_s* m, int kf, unsigned char** out) {
  const MatView v = dist_view(m, kf);
  int rc;
  if ((rc = dmalloc((void**)out, std::max<size_t>(1, (size_t)v.ntiles), nullptr))) return rc;
  if (v.ntiles > 0) {
    tile_halo_kernel<<<std::min(v.ntiles, 148 * 8), 256>>>(
        v.tdesc, kf == K_SCSR_PRIV ? v.tdescB : nullptr, v.ntiles, v.idxA,
        kf == K_SCSR_PRIV ? v.idxB : nullptr, (long long)m->n, *out);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaDeviceSynchronize());
  }
  return SPCG_OK;
}

// ---- the per-pass loop, shared by every transport ----------------------------
// nv DistArgs (device array dA, host copies hA): nv = 1 for one rank per
// process (host transports, or the device transport across GPUs), nv = R for
// the virtual-rank group on one GPU.  H: the host transport (fused == 0 only).
template <int FMT>
int run_dist(const std::vector<DistArgs>& hA, DistArgs* dA, const HaloPlan* H, const MatView& v,
             const spcg_cg_options* o, std::vector<StepState*> h_state,
             const std::vector<spcg_matrix_s*>& mats, spcg_cg_result* out, cudaStream_t st) {
  DevInfo* di;
  int rc;
  if ((rc = dev_info(&di))) return rc;
  const int nv = (int)hA.size();
  const bool fused = hA[0].peer != nullptr;
  const bool wide = FMT == K_CSR && v.wide;
  // virtual ranks share the GPU: each gets 1/nv of the CTAs a lone rank
  // would use, so a launch over all of them is one wave, as for one rank
  int G = 1;
  for (const DistArgs& a : hA)
    G = std::max(G, std::min(std::max(1, a.M.ntiles), std::max(1, di->spmv_grid / nv)));
  const int GE = std::max(1, 2 * di->sms / nv);
  const size_t sm = sizeof(Smem);
  constexpr int kAtom = (FMT == K_SCSR_ATOMIC || FMT == K_CSC) ? 1 : 0;
  constexpr bool kRev = (FMT == K_SCSR_ATOMIC);  // transposed scatters reach halo rows
  const bool ghosts = fused && kRev && hA[0].nranks > 1;
  bool any_push = false;  // some rank's send runs do not fit pass C
  for (const DistArgs& a : hA) any_push |= fused && a.nruns > kRunCache;
  DistWorkspace& d0 = mats[0]->dw;
  long long launches = 0;
  // solve state (the device transport's sequence counters rseq / hseq at the
  // end of StepState persist across solves: every rank keeps them in step)
  for (int r = 0; r < nv; ++r) {
    StepState init{};
    init.tol = o->tol;
    init.max_it = o->max_iter > 0
                      ? o->max_iter
                      : std::max<long long>(1, std::max<long long>(mats[r]->n_global, mats[r]->n));
    init.record = o->record_history && hA[r].hist;
    init.x0_given = hA[r].x0 != nullptr;
    CUDA_TRY(cudaMemcpyAsync(hA[r].S, &init, offsetof(StepState, rseq), cudaMemcpyHostToDevice, st));
    const long long next = mats[r]->dw.next;
    CUDA_TRY(cudaMemsetAsync(hA[r].p, 0, sizeof(double) * (size_t)next, st));
    if (kAtom) CUDA_TRY(cudaMemsetAsync(hA[r].q, 0, sizeof(double) * (size_t)std::max(1LL, next), st));
  }
  const int GG = nv * G, GGE = nv * GE;
  // K_SCSR_FIX (one rank): the max|p| slots of StepState and the accumulator
  constexpr bool kFix = (FMT == K_SCSR_FIX);
  auto pmax_slot = [&](int k) {
    return reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(hA[0].S) +
                                                 offsetof(StepState, pmax) + 8 * (size_t)k);
  };
  if (kFix) {
    if (nv != 1 || hA[0].M.ytx == nullptr) return fail(SPCG_ERR_ARG, "fixed-point SCSR: one rank");
    CUDA_TRY(cudaMemsetAsync(hA[0].M.ytx, 0, sizeof(unsigned long long) *
                                                 (size_t)std::max<long long>(2, hA[0].nloc + 1), st));
  }
  auto absmax = [&](const double* v, int slot) -> int {  // max|v| into a pmax slot
    CUDA_TRY(cudaMemsetAsync(pmax_slot(slot), 0, sizeof(unsigned long long), st));
    vec_absmax_kernel<<<GE, kElemBlock, 0, st>>>(hA[0].nloc, v, pmax_slot(slot));
    CUDA_TRY(cudaGetLastError());
    return SPCG_OK;
  };
  // kernel transport mode: 0 host transport, 1 device transport (one rank
  // per process), 2 device transport over nv virtual ranks in one launch
  // (SPCG_FORCE_GROUP=1: one rank through the virtual-rank kernels, to
  // measure what the group form itself costs; scripts/p2p_overhead.py)
  static const bool force_group = getenv("SPCG_FORCE_GROUP") != nullptr;
  const int mode = !fused ? 0 : ((nv > 1 || force_group) ? 2 : 1);
  DistArgs a1 = hA[0];  // MODE 0 / 1: the rank's arguments by value
  a1.M.cta0 = 0;
  a1.M.ncta = 0;
  a1.txnext = nullptr;
  if (kFix) a1.M.txmax = pmax_slot(2);  // always a valid slot
#define SPCG_ELEM(KERNEL, ...)                                                        \
  do {                                                                                \
    if (mode == 0) KERNEL<0><<<GE, kElemBlock, 0, st>>>(a1, dA, GE, __VA_ARGS__);      \
    else if (mode == 1) KERNEL<1><<<GE, kElemBlock, 0, st>>>(a1, dA, GE, __VA_ARGS__); \
    else KERNEL<2><<<GGE, kElemBlock, 0, st>>>(a1, dA, GE, __VA_ARGS__);              \
    ++launches;                                                                       \
  } while (0)
#define SPCG_TILE(KERNEL, ...)                                                                    \
  do {                                                                                            \
    if (wide) {                                                                                   \
      if (mode == 0) KERNEL<K_CSR, true, 0><<<G, kBlock, sm, st>>>(a1, dA, G, __VA_ARGS__);        \
      else if (mode == 1) KERNEL<K_CSR, true, 1><<<G, kBlock, sm, st>>>(a1, dA, G, __VA_ARGS__);   \
      else KERNEL<K_CSR, true, 2><<<GG, kBlock, sm, st>>>(a1, dA, G, __VA_ARGS__);                \
    } else {                                                                                      \
      if (mode == 0) KERNEL<FMT, false, 0><<<G, kBlock, sm, st>>>(a1, dA, G, __VA_ARGS__);         \
      else if (mode == 1) KERNEL<FMT, false, 1><<<G, kBlock, sm, st>>>(a1, dA, G, __VA_ARGS__);    \
      else KERNEL<FMT, false, 2><<<GG, kBlock, sm, st>>>(a1, dA, G, __VA_ARGS__);                 \
    }                                                                                             \
    ++launches;                                                                                   \
  } while (0)
  StepState* S0 = hA[0].S;
  double* hist0 = hA[0].hist;
  auto host_reduce = [&](int op) -> int {  // host transports: all-reduce + scalar kernel
    if (fused) return SPCG_OK;
    int rc2;
    if ((rc2 = allreduce_red(*H, S0, st))) return rc2;
    dist_scalar<<<1, 1, 0, st>>>(op, S0, hist0);
    ++launches;
    return SPCG_OK;
  };
  // halo of an own vector into the neighbours' extended `dst`
  auto halo = [&](int srcsel, int dstsel, const double* hsrc, double* hdst) -> int {
    if (fused) {
      if (hA[0].nranks > 1) SPCG_ELEM(dist_push, srcsel, dstsel, 0);
      return SPCG_OK;
    }
    return halo_exchange(*H, d0, hsrc, hdst, st, &launches);
  };
  auto spmv_once = [&]() -> int {  // q = A tmp (x0 / true residual)
    // device transport: the kernel waits for the halo of the push just done
    a1.M.rev = 0;
    a1.M.tree = 0;
    if (kFix) {  // slot 2: max|tmp|, read by this SpMV and the elementwise pass after it
      int rc2;
      if ((rc2 = absmax(hA[0].tmp, 2))) return rc2;
      a1.M.txmax = pmax_slot(2);
      a1.txnext = nullptr;
  if (kFix) a1.M.txmax = pmax_slot(2);  // always a valid slot
    }
    SPCG_TILE(dist_spmv, 0);
    if (kRev) {
      if (ghosts) {
        SPCG_ELEM(dist_ghost_push, -1);
      } else if (!fused) {
        int rc2;
        if ((rc2 = reverse_halo(*H, d0, hA[0].q, d0.next - hA[0].nloc, st, &launches))) return rc2;
      }
    }
    return SPCG_OK;
  };
  CUDA_TRY(cudaEventRecord(d0.ev0, st));
  // ||b|| (solver.py:107)
  SPCG_ELEM(dist_elem, 0, 0, 0);
  if ((rc = host_reduce(0))) return rc;
  // x = x0, r = b - A x0, p = r (solver.py:120-124)
  SPCG_ELEM(dist_x, 0);
  const bool have_x0 = hA[0].x0 != nullptr;
  if (have_x0) {
    if ((rc = halo(1, 1, hA[0].x0, hA[0].tmp))) return rc;
    if ((rc = spmv_once())) return rc;
  }
  SPCG_ELEM(dist_elem, 1, have_x0 ? 1 : 0, 0);
  if ((rc = host_reduce(1))) return rc;
  if (kFix && (rc = absmax(hA[0].p, 0))) return rc;  // p_1 = r_0 -> slot 0
  if ((rc = halo(0, 0, hA[0].p, hA[0].p))) return rc;
  CUDA_TRY(cudaGetLastError());
  // CG loop; the host enqueues chunks of iterations and polls the device-side
  // done flag of chunk c while chunk c + 1 is already queued (double
  // buffered), so the GPU never idles while the host enqueues.  Iterations
  // after `done` are no-ops on every rank, so the collectives stay matched;
  // the one chunk enqueued past convergence costs only empty launches.
  const int chunk = 16;
  const bool timing = o->timing != 0;
  const bool split = o->timing >= 2;  // events around passes B and C too
  if (timing && !d0.tev[0][0][0])
    for (int bb = 0; bb < 2; ++bb)
      for (int a = 0; a < 6; ++a)
        for (int c = 0; c < chunk; ++c) CUDA_TRY(cudaEventCreate(&d0.tev[bb][a][c]));
  double spmv_ms = 0.0, axpy_ms = 0.0;
  long long spmv_n = 0, k_before = 0, iter_enq = 0;
#ifndef SPCG_ALTERNATE
#define SPCG_ALTERNATE 1
#endif
  constexpr bool kAlternate = SPCG_ALTERNATE != 0;
  const int tree = o->row_sums == 0;  // auto: reassociated long-row sums in pass A
  const int post = ghosts ? 0 : 1;
  static const int dir_mode = getenv("SPCG_PASS_DIR") ? atoi(getenv("SPCG_PASS_DIR")) : -1;
  auto enqueue_chunk = [&](int bb) -> int {
    for (int c = 0; c < chunk; ++c) {
      if (timing) CUDA_TRY(cudaEventRecord(d0.tev[bb][0][c], st));
      // alternate traversal directions pass to pass (A, B, C, A, ...): each
      // pass starts on the lines the previous one wrote last (still in L2)
      // pass A runs last-to-first always on the regular tiles (P3 1,676 ->
      // 1,653 us per iteration: its reverse traversal streams 5 % faster,
      // more than the L2 reuse alternation bought; Q27 neutral) and
      // alternates on the wide tiles (P2 417.7 vs 420.1); scripts/phase_split.py
      int dirA = kAlternate ? (wide ? (int)((iter_enq & 1) == 0) : 1) : 0;
      // (A/B) SPCG_PASS_DIR: 0 / 1 a fixed pass-A direction, 2 alternate
      if (dir_mode == 0 || dir_mode == 1) dirA = dir_mode;
      if (dir_mode == 2) dirA = (int)((iter_enq & 1) == 0);
      a1.M.rev = dirA;
      a1.M.tree = tree;
      if (kFix) {  // iteration parity: A / B read slot k&1, C fills (B clears) slot (k+1)&1
        a1.M.txmax = pmax_slot((int)(iter_enq & 1));
        a1.txnext = pmax_slot((int)((iter_enq + 1) & 1));
      }
      SPCG_TILE(dist_spmv_pq, dirA, tree, post);
      if (timing) CUDA_TRY(cudaEventRecord(d0.tev[bb][1][c], st));
      int rc2;
      if (!fused) {
        if ((rc2 = allreduce_red(*H, S0, st))) return rc2;
        if (kRev && (rc2 = reverse_halo(*H, d0, hA[0].q, d0.next - hA[0].nloc, st, &launches)))
          return rc2;
        dist_scalar<<<1, 1, 0, st>>>(2, S0, hist0);
        ++launches;
      } else if (ghosts) {
        SPCG_ELEM(dist_ghost_push, 2);
      }
      if (split) CUDA_TRY(cudaEventRecord(d0.tev[bb][2][c], st));
      SPCG_ELEM(dist_elem, 2, 0, kAlternate ? 1 - dirA : 0);
      if (split) CUDA_TRY(cudaEventRecord(d0.tev[bb][3][c], st));
      if ((rc2 = host_reduce(3))) return rc2;
      if (split) CUDA_TRY(cudaEventRecord(d0.tev[bb][4][c], st));
      SPCG_ELEM(dist_update, dirA);
      if (split) CUDA_TRY(cudaEventRecord(d0.tev[bb][5][c], st));
      ++iter_enq;
      if (fused) {
        if (any_push) SPCG_ELEM(dist_push, 0, 0, 1);
      } else if ((rc2 = halo_exchange(*H, d0, hA[0].p, hA[0].p, st, &launches))) {
        return rc2;
      }
    }
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(d0.h_Sc[bb], S0, sizeof(StepState), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaEventRecord(d0.cev[bb], st));
    return SPCG_OK;
  };
  // the host-callback transport synchronises inside every exchange: no
  // point (and no room) for a second chunk in flight
  const bool two = fused || H->hc == nullptr;
  if ((rc = enqueue_chunk(0))) return rc;
  StepState fin{};
  for (long long ci = 0;; ++ci) {
    const int bb = (int)(ci & 1);
    if (two && (rc = enqueue_chunk(bb ^ 1))) return rc;
    CUDA_TRY(cudaEventSynchronize(d0.cev[bb]));
    const StepState& hs = *d0.h_Sc[bb];
    if (timing) {  // only the passes that did work (later ones returned at once)
      const long long ran = std::min<long long>(chunk, hs.k - k_before + (hs.status != 0 ? 1 : 0));
      for (long long c = 0; c < ran; ++c) {
        float t = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&t, d0.tev[bb][0][c], d0.tev[bb][1][c]));
        spmv_ms += t;
        ++spmv_n;
        if (split) {
          float tb = 0.f, tc = 0.f;
          CUDA_TRY(cudaEventElapsedTime(&tb, d0.tev[bb][2][c], d0.tev[bb][3][c]));
          CUDA_TRY(cudaEventElapsedTime(&tc, d0.tev[bb][4][c], d0.tev[bb][5][c]));
          axpy_ms += (double)tb + (double)tc;
        }
      }
      k_before = hs.k;
    }
    if (hs.done) {
      fin = hs;
      break;
    }
    if (!two && (rc = enqueue_chunk(bb ^ 1))) return rc;
  }
  // a converged solve skipped its pass C: x += alpha_K p_K; then the true residual
  SPCG_ELEM(dist_x, 1);
  if (o->recompute_final_residual && fin.status == 0 && fin.b_norm != 0.0) {
    SPCG_ELEM(dist_x, 2);
    if ((rc = halo(2, 1, hA[0].x, hA[0].tmp))) return rc;
    if ((rc = spmv_once())) return rc;
    SPCG_ELEM(dist_elem, 3, 0, 0);
    if ((rc = host_reduce(4))) return rc;
  }
#undef SPCG_ELEM
#undef SPCG_TILE
  CUDA_TRY(cudaEventRecord(d0.ev1, st));
  for (int r = 0; r < nv; ++r)
    CUDA_TRY(cudaMemcpyAsync(h_state[r], hA[r].S, sizeof(StepState), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  CUDA_TRY(cudaGetLastError());
  float ms = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&ms, d0.ev0, d0.ev1));
  for (int r = 0; r < nv; ++r) {
    const StepState& S = *h_state[r];
    spcg_cg_result& R = out[r];
    R = spcg_cg_result{};
    R.iterations = S.k;
    R.converged = S.converged;
    R.status = S.status;
    R.fail_iteration = S.fail_iter;
    R.final_relative_residual = S.rel;
    R.b_norm = S.b_norm;
    R.device_ms = ms;
    R.kernel_launches = launches;
    R.spmv_ms = spmv_ms;
    R.spmv_launches = spmv_n;
    R.engine_used = 2;
    // split: SpMV passes (with the fused p.q partial); the vector-update
    // passes B and C (with the fused r.r partial); the rest (reductions'
    // completion, scalar steps, collectives, halo, prologue) under "dot"
    R.phase_ms[0] = split ? spmv_ms : 0.0;
    R.phase_ms[2] = split ? axpy_ms : 0.0;
    R.phase_ms[1] = split ? std::max(0.0, (double)ms - spmv_ms - axpy_ms) : 0.0;
  }
  const StepState& S = *h_state[0];
  if (S.status != 0) {
    const char* what = S.status == SPCG_ERR_NOT_SPD ? "matrix not positive definite"
                       : S.status == SPCG_ERR_NONFINITE_ALPHA ? "non-finite alpha"
                       : S.status == SPCG_ERR_NONFINITE_RESIDUAL ? "non-finite residual"
                                                                  : "non-finite beta";
    return fail(S.status, std::string(what) + " at iteration " + std::to_string(S.fail_iter));
  }
  return SPCG_OK;
}

// Host-side DistArgs of one rank (no device-transport fields).
DistArgs base_args(spcg_matrix_s* m, int kf, const double* b, const double* x0, double* x,
                   double* hist, const spcg_cg_options* o) {
  DistWorkspace& d = m->dw;
  DistArgs A{};
  A.M = dist_view(m, kf);
  A.S = d.S;
  A.p = d.p_ext[0];
  A.r = d.r_ext;
  A.q = d.q;
  A.x = x;
  A.b = b;
  A.x0 = x0;
  A.tmp = d.tmp_ext;
  A.hist = o->record_history ? hist : nullptr;
  A.part = d.part;
  A.nloc = m->n;
  A.rank = 0;
  A.nranks = 1;
  A.zq = (kf == K_SCSR_ATOMIC || kf == K_CSC) ? 1 : 0;
  A.xv = (((uintptr_t)x) & 15) == 0;
  if (kf == K_SCSR_FIX) {
    A.M.ytx = d.ytx;
    A.M.tx_eM = m->tx_eM;
  }
  return A;
}

// K_SCSR_FIX setup: the accumulator and 2^eM >= max_j sum_{i>j} |a_ij| (from
// the rows of L^T, summed in order: deterministic), once per handle.
int ensure_fix(spcg_matrix_s* m) {
  DistWorkspace& d = m->dw;
  int rc;
  if (d.ytx_n < (long long)m->n + 2) {
    if (d.ytx) cudaFree(d.ytx);
    d.ytx = nullptr;
    if ((rc = dmalloc((void**)&d.ytx, sizeof(unsigned long long) * ((size_t)m->n + 2), nullptr)))
      return rc;
    d.ytx_n = (long long)m->n + 2;
  }
  if (m->tx_eM == -100000) {
    if (!m->hasB) return fail(SPCG_ERR_UNSUPPORTED, "fixed-point SCSR needs the L^T rows");
    unsigned long long* mx = nullptr;
    if ((rc = dmalloc((void**)&mx, sizeof(unsigned long long), nullptr))) return rc;
    CUDA_TRY(cudaMemset(mx, 0, sizeof(unsigned long long)));
    if (m->n > 0) lt_rowsum_max_kernel<<<592, 256>>>(m->n, m->B.ptr, m->B.val, mx);
    unsigned long long bits = 0;
    CUDA_TRY(cudaMemcpy(&bits, mx, sizeof(bits), cudaMemcpyDeviceToHost));
    cudaFree(mx);
    int e = 0;
    const double Mmax = __builtin_bit_cast(double, bits);
    if (Mmax > 0.0) std::frexp(Mmax, &e);
    m->tx_eM = e;
  }
  return SPCG_OK;
}

template <int FMT>
int dispatch_fmt_host(spcg_matrix_s* m, const HaloPlan& H, const double* b, const double* x0,
                      double* x, double* hist, const spcg_cg_options* o, spcg_cg_result* out,
                      cudaStream_t st) {
  DistWorkspace& d = m->dw;
  std::vector<DistArgs> hA{base_args(m, FMT, b, x0, x, hist, o)};
  CUDA_TRY(cudaMemcpyAsync(d.args, hA.data(), sizeof(DistArgs), cudaMemcpyHostToDevice, st));
  return run_dist<FMT>(hA, d.args, &H, hA[0].M, o, {d.h_S}, {m}, out, st);
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
    *out = spcg_cg_result{};
    out->converged = 1;
    out->engine_used = 2;
    return SPCG_OK;
  }
  // deterministic symmetric mode on one GPU: one pass over L+D with the
  // transposed part accumulated exactly in fixed point (K_SCSR_FIX), unless
  // the caller asked for the reference's sequential sums (row_sums = 1: the
  // stored L^T, bitwise the reference privatized mode at workers = 1)
  if (kf == K_SCSR_PRIV && npeers == 0 && alone && !m->is_rows && o->row_sums == 0) {
    if ((rc = ensure_fix(m))) return rc;
    return dispatch_fmt_host<K_SCSR_FIX>(m, H, b, x0, x, hist, o, out, st);
  }
  switch (kf) {
    case K_CSR: return dispatch_fmt_host<K_CSR>(m, H, b, x0, x, hist, o, out, st);
    case K_SCSR_PRIV: return dispatch_fmt_host<K_SCSR_PRIV>(m, H, b, x0, x, hist, o, out, st);
    case K_SCSR_ATOMIC: return dispatch_fmt_host<K_SCSR_ATOMIC>(m, H, b, x0, x, hist, o, out, st);
    default: return dispatch_fmt_host<K_CSC>(m, H, b, x0, x, hist, o, out, st);
  }
}

// ---- device transport: plan creation, export / connect, solves --------------
int plan_create(spcg_matrix_s* m, int rank, int nranks, int npeers, const int32_t* peers,
                const int64_t* recv_off, const int64_t* send_off, const int32_t* send_idx,
                spcg_dist_plan_s** out) {
  if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks)
    return fail(SPCG_ERR_ARG, "device transport: 1 <= nranks <= " + std::to_string(kMaxRanks));
  if (m->is_rows && !m->localized) return fail(SPCG_ERR_ARG, "call spcg_matrix_localize first");
  if (npeers < 0 || (npeers > 0 && (!peers || !recv_off || !send_off)))
    return fail(SPCG_ERR_ARG, "bad halo plan");
  const long long nhalo = (long long)m->halo.size();
  if ((npeers > 0 ? recv_off[npeers] : 0) != nhalo)
    return fail(SPCG_ERR_ARG, "receive plan does not cover the halo");
  const long long send_total = npeers > 0 ? send_off[npeers] : 0;
  for (int k = 0; k < npeers; ++k)
    if (peers[k] < 0 || peers[k] >= nranks || peers[k] == rank || (k && peers[k] <= peers[k - 1]))
      return fail(SPCG_ERR_ARG, "peers must be ascending ranks other than this one");
  for (long long s = 0; s < send_total; ++s)
    if (!send_idx || send_idx[s] < 0 || send_idx[s] >= m->n)
      return fail(SPCG_ERR_ARG, "send index out of range");
  int rc;
  if ((rc = ensure_dist_ws(m, send_total))) return rc;
  auto* P = new spcg_dist_plan_s();
  P->m = m;
  P->rank = rank;
  P->nranks = nranks;
  P->peers.assign(peers, peers + npeers);
  P->recv_off.assign(recv_off ? recv_off : nullptr, recv_off ? recv_off + npeers + 1 : nullptr);
  P->send_off.assign(send_off ? send_off : nullptr, send_off ? send_off + npeers + 1 : nullptr);
  if (npeers == 0) {
    P->recv_off.assign(1, 0);
    P->send_off.assign(1, 0);
  }
  P->send_idx.assign(send_idx ? send_idx : nullptr, send_idx ? send_idx + send_total : nullptr);
  const size_t mb = sizeof(unsigned long long) * 2 * 2 * (size_t)nranks;
  const size_t hb = sizeof(unsigned long long) * 2 * (size_t)nranks;
  if ((rc = dmalloc((void**)&P->mbox, mb, nullptr)) || (rc = dmalloc((void**)&P->hflag, hb, nullptr)) ||
      (rc = dmalloc((void**)&P->d_args, sizeof(DistArgs), nullptr))) {
    free_plan(P);
    delete P;
    return rc;
  }
  CUDA_TRY(cudaMemset(P->mbox, 0, mb));
  CUDA_TRY(cudaMemset(P->hflag, 0, hb));
  // the sequence counters start at 0 on every rank
  CUDA_TRY(cudaMemset(m->dw.S, 0, sizeof(StepState)));
  *out = P;
  return SPCG_OK;
}

int plan_export(spcg_dist_plan_s* P, unsigned char* blob_out) {
  spcg_matrix_s* m = P->m;
  P2PBlob B;
  memset(&B, 0, sizeof(B));
  B.magic = kBlobMagic;
  B.version = SPCG_ABI_VERSION;
  B.rank = P->rank;
  B.nranks = P->nranks;
  B.device = m->device;
  B.pid = (int32_t)getpid();
  B.nloc = m->n;
  B.row0 = m->is_rows ? m->row0 : 0;
  for (int s = 0; s < kMaxRanks; ++s) B.recv_off_by_src[s] = -1;
  for (size_t k = 0; k < P->peers.size(); ++k) B.recv_off_by_src[P->peers[k]] = P->recv_off[k];
  DistWorkspace& d = m->dw;
  CUDA_TRY(cudaIpcGetMemHandle(&B.h_mbox, P->mbox));
  CUDA_TRY(cudaIpcGetMemHandle(&B.h_hflag, P->hflag));
  CUDA_TRY(cudaIpcGetMemHandle(&B.h_p, d.p_ext[0]));
  CUDA_TRY(cudaIpcGetMemHandle(&B.h_tmp, d.tmp_ext));
  CUDA_TRY(cudaIpcGetMemHandle(&B.h_q, d.q));
  B.mbox = (uint64_t)(uintptr_t)P->mbox;
  B.hflag = (uint64_t)(uintptr_t)P->hflag;
  B.p = (uint64_t)(uintptr_t)d.p_ext[0];
  B.tmp = (uint64_t)(uintptr_t)d.tmp_ext;
  B.q = (uint64_t)(uintptr_t)d.q;
  memset(blob_out, 0, SPCG_P2P_BLOB_BYTES);
  memcpy(blob_out, &B, sizeof(B));
  return SPCG_OK;
}

// Map every peer's buffers (IPC, or raw pointers within this process) and
// build this rank's sender tables: send runs / entries with destinations in
// the receivers' extended vectors, and the reverse-halo ghost destinations.
int plan_connect(spcg_dist_plan_s* P, const unsigned char* blobs) {
  if (P->connected) return SPCG_OK;
  const int R = P->nranks, me = P->rank;
  std::vector<P2PBlob> B((size_t)R);
  for (int k = 0; k < R; ++k) {
    memcpy(&B[(size_t)k], blobs + (size_t)k * SPCG_P2P_BLOB_BYTES, sizeof(P2PBlob));
    if (B[k].magic != kBlobMagic || B[k].rank != k || B[k].nranks != R)
      return fail(SPCG_ERR_ARG, "peer blob " + std::to_string(k) + " is not a plan export of rank " +
                                    std::to_string(k) + " of " + std::to_string(R));
  }
  const int mypid = (int)getpid();
  PeerTab& T = P->peer;
  T.mbox = P->mbox;
  T.hflag = P->hflag;
  auto open = [&](int k, const cudaIpcMemHandle_t& h, uint64_t raw, void** dst) -> int {
    if (k == me || B[k].pid == mypid) {
      if (B[k].device != P->m->device)
        return fail(SPCG_ERR_UNSUPPORTED, "ranks of one process must share the device");
      *dst = (void*)(uintptr_t)raw;
      return SPCG_OK;
    }
    CUDA_TRY(cudaIpcOpenMemHandle(dst, h, cudaIpcMemLazyEnablePeerAccess));
    P->opened.push_back(*dst);
    P->same_device = false;  // another process: another GPU (system scope)
    return SPCG_OK;
  };
  int rc;
  std::vector<bool> sendto((size_t)R, false), recvfrom((size_t)R, false);
  for (size_t k = 0; k < P->peers.size(); ++k) {
    const int pk = P->peers[k];
    if (P->send_off[k + 1] > P->send_off[k]) sendto[(size_t)pk] = true;
    if (P->recv_off[k + 1] > P->recv_off[k]) recvfrom[(size_t)pk] = true;
  }
  for (int k = 0; k < R; ++k) {
    if ((rc = open(k, B[k].h_mbox, B[k].mbox, (void**)&T.peer_mbox[k]))) return rc;
    if (k == me) continue;
    if (sendto[k]) {
      if ((rc = open(k, B[k].h_hflag, B[k].hflag, (void**)&T.peer_hflag[k]))) return rc;
      if ((rc = open(k, B[k].h_p, B[k].p, (void**)&T.peer_p[k]))) return rc;
      if ((rc = open(k, B[k].h_tmp, B[k].tmp, (void**)&T.peer_tmp[k]))) return rc;
    }
    if (recvfrom[k] && (rc = open(k, B[k].h_q, B[k].q, (void**)&T.peer_q[k]))) return rc;
  }
  P->nrecv = 0;
  P->nsendpeers = 0;
  for (int k = 0; k < R; ++k) {
    if (recvfrom[k]) T.recv_from[P->nrecv++] = k;
    if (sendto[k]) T.send_to[P->nsendpeers++] = k;
  }
  if ((rc = dmalloc((void**)&P->d_peer, sizeof(PeerTab), nullptr))) return rc;
  CUDA_TRY(cudaMemcpy(P->d_peer, &T, sizeof(PeerTab), cudaMemcpyHostToDevice));
  // sender tables
  const long long total = P->send_off.back();
  std::vector<int> speer((size_t)std::max(1LL, total));
  std::vector<long long> sdst((size_t)std::max(1LL, total));
  std::vector<SendRun> runs;
  for (size_t k = 0; k < P->peers.size(); ++k) {
    const int pk = P->peers[k];
    const long long roff = B[pk].recv_off_by_src[me];
    if (P->send_off[k + 1] > P->send_off[k] && roff < 0)
      return fail(SPCG_ERR_ARG, "rank " + std::to_string(pk) + " expects no values from rank " +
                                    std::to_string(me));
    for (long long s = P->send_off[k]; s < P->send_off[k + 1]; ++s) {
      speer[(size_t)s] = pk;
      sdst[(size_t)s] = B[pk].nloc + roff + (s - P->send_off[k]);
      const int row = P->send_idx[(size_t)s];
      if (!runs.empty() && runs.back().peer == pk && runs.back().hi == row &&
          runs.back().dst + (runs.back().hi - runs.back().lo) == sdst[(size_t)s]) {
        runs.back().hi++;
      } else {
        runs.push_back(SendRun{row, row + 1, pk, 0, sdst[(size_t)s]});
      }
    }
  }
  P->nruns = (int)runs.size();
  if ((rc = dmalloc((void**)&P->runs, sizeof(SendRun) * std::max<size_t>(1, runs.size()), nullptr)) ||
      (rc = dmalloc((void**)&P->send_peer, sizeof(int) * speer.size(), nullptr)) ||
      (rc = dmalloc((void**)&P->send_dst, sizeof(long long) * sdst.size(), nullptr)))
    return rc;
  if (!runs.empty())
    CUDA_TRY(cudaMemcpy(P->runs, runs.data(), sizeof(SendRun) * runs.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(P->send_peer, speer.data(), sizeof(int) * speer.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(P->send_dst, sdst.data(), sizeof(long long) * sdst.size(), cudaMemcpyHostToDevice));
  if (total > 0)
    CUDA_TRY(cudaMemcpy(P->m->dw.send_idx, P->send_idx.data(), sizeof(int) * (size_t)total,
                        cudaMemcpyHostToDevice));
  // reverse halo: ghost h (a halo column owned by peer k) -> k's local row
  const std::vector<long long>& halo = P->m->halo;
  P->nghost = (long long)halo.size();
  std::vector<int> gpeer((size_t)std::max(1LL, P->nghost)), gdst((size_t)std::max(1LL, P->nghost));
  for (size_t k = 0; k < P->peers.size(); ++k)
    for (long long h = P->recv_off[k]; h < P->recv_off[k + 1]; ++h) {
      gpeer[(size_t)h] = P->peers[k];
      gdst[(size_t)h] = (int)(halo[(size_t)h] - B[P->peers[k]].row0);
    }
  if ((rc = dmalloc((void**)&P->ghost_peer, sizeof(int) * gpeer.size(), nullptr)) ||
      (rc = dmalloc((void**)&P->ghost_dst, sizeof(int) * gdst.size(), nullptr)))
    return rc;
  CUDA_TRY(cudaMemcpy(P->ghost_peer, gpeer.data(), sizeof(int) * gpeer.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(P->ghost_dst, gdst.data(), sizeof(int) * gdst.size(), cudaMemcpyHostToDevice));
  P->connected = true;
  return SPCG_OK;
}

// DistArgs of a connected plan for one solve.
int plan_args(spcg_dist_plan_s* P, int kf, const double* b, const double* x0, double* x,
              double* hist, const spcg_cg_options* o, DistArgs& A) {
  spcg_matrix_s* m = P->m;
  A = base_args(m, kf, b, x0, x, hist, o);
  if (!P->thalo) {
    int rc;
    if ((rc = build_thalo(m, kf, &P->thalo))) return rc;
  }
  A.thalo = P->thalo;
  A.rank = P->rank;
  A.nranks = P->nranks;
  A.peer = P->d_peer;
  A.nrecv = P->nrecv;
  A.nsendpeers = P->nsendpeers;
  A.gpu_scope = P->same_device ? 1 : 0;
  A.nruns = P->nruns;
  A.runs = P->runs;
  A.send_total = P->send_off.back();
  A.send_idx = m->dw.send_idx;
  A.send_peer = P->send_peer;
  A.send_dst = P->send_dst;
  A.nghost = P->nghost;
  A.ghost_peer = P->ghost_peer;
  A.ghost_dst = P->ghost_dst;
  return SPCG_OK;
}

template <int FMT>
int group_solve_t(int nranks, spcg_dist_plan_s* const* plans, const double* const* b,
                  const double* const* x0, double* const* x, double* hist,
                  const spcg_cg_options* o, spcg_cg_result* out, cudaStream_t st,
                  DistArgs* d_args) {
  std::vector<DistArgs> hA((size_t)nranks);
  std::vector<StepState*> hs((size_t)nranks);
  std::vector<spcg_matrix_s*> ms((size_t)nranks);
  int rc;
  for (int r = 0; r < nranks; ++r) {
    spcg_dist_plan_s* P = plans[r];
    if ((rc = plan_args(P, FMT, b[r], x0 ? x0[r] : nullptr, x[r], r == 0 ? hist : nullptr, o,
                        hA[(size_t)r])))
      return rc;
    hs[(size_t)r] = P->m->dw.h_S;
    ms[(size_t)r] = P->m;
  }
  for (int r = 1; r < nranks; ++r)
    if (hA[(size_t)r].M.wide != hA[0].M.wide)
      return fail(SPCG_ERR_UNSUPPORTED, "ranks of one launch need the same tile layout");
  CUDA_TRY(cudaMemcpyAsync(d_args, hA.data(), sizeof(DistArgs) * (size_t)nranks,
                           cudaMemcpyHostToDevice, st));
  return run_dist<FMT>(hA, d_args, nullptr, hA[0].M, o, hs, ms, out, st);
}

int plan_solve_checked(int nranks, spcg_dist_plan_s* const* plans, const double* const* b,
                       const double* const* x0, double* const* x, double* hist,
                       const spcg_cg_options* o, spcg_cg_result* out, cudaStream_t st) {
  if (!(o->tol > 0.0)) return fail(SPCG_ERR_ARG, "tol must be > 0");
  if (o->record_history && !hist) return fail(SPCG_ERR_ARG, "record_history needs a history buffer");
  const int kf = kfmt_of(plans[0]->m, o->accumulation);
  for (int r = 0; r < nranks; ++r) {
    spcg_dist_plan_s* P = plans[r];
    if (!P->connected) return fail(SPCG_ERR_ARG, "plan not connected (spcg_dist_plan_connect)");
    if (kfmt_of(P->m, o->accumulation) != kf) return fail(SPCG_ERR_ARG, "ranks differ in format");
    if (int rc = on_device(P->m->device)) return rc;
  }
  if (kf == K_CSC && plans[0]->nranks > 1) return fail(SPCG_ERR_UNSUPPORTED, "sharded CSC is not supported");
  if (kf == K_SCSR_PRIV && !plans[0]->m->hasB) return fail(SPCG_ERR_UNSUPPORTED, "SCSR needs its L^T rows");
  // the launch's DistArgs array: the plan's own slot for one rank, a
  // temporary one for a group
  DistArgs* d_args = plans[0]->d_args;
  if (nranks > 1) {
    int rc;
    if ((rc = dmalloc((void**)&d_args, sizeof(DistArgs) * (size_t)nranks, nullptr))) return rc;
  }
  int rc;
  switch (kf) {
    case K_CSR: rc = group_solve_t<K_CSR>(nranks, plans, b, x0, x, hist, o, out, st, d_args); break;
    case K_SCSR_PRIV:
      rc = group_solve_t<K_SCSR_PRIV>(nranks, plans, b, x0, x, hist, o, out, st, d_args);
      break;
    case K_SCSR_ATOMIC:
      rc = group_solve_t<K_SCSR_ATOMIC>(nranks, plans, b, x0, x, hist, o, out, st, d_args);
      break;
    default: rc = group_solve_t<K_CSC>(nranks, plans, b, x0, x, hist, o, out, st, d_args); break;
  }
  if (nranks > 1) {
    cudaStreamSynchronize(st);
    cudaFree(d_args);
  }
  return rc;
}
