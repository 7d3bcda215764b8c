// host_cluster.cuh — host side of spcg_b200.cu: cluster-resident engine (engine 5): plan builder, launch, solve.
// Included exactly once, by spcg_b200.cu inside its anonymous namespace
// (one translation unit: the kernels' templates are instantiated there).
#pragma once

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
  // (dev) SPCG_PLAN_TIMING: host time of the plan's steps on stderr
  static const bool ptime = getenv("SPCG_PLAN_TIMING") != nullptr;
  auto tnow = [] { return std::chrono::steady_clock::now(); };
  auto t_last = tnow();
  auto mark = [&](const char* what) {
    if (!ptime) return;
    const auto t = tnow();
    fprintf(stderr, "[spcg plan] %-14s %.3f ms\n", what,
            std::chrono::duration<double, std::milli>(t - t_last).count());
    t_last = t;
  };
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
  mark("download");
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
  const int smem_probe = optin0 - (int)kClusStatic - 1024;
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
  mark("row lengths");
  int C, csz;
  static const int force_k = getenv("SPCG_CLUS_K") ? atoi(getenv("SPCG_CLUS_K")) : 0;  // dev A/B
  if ((want <= kClusMax && force_k <= 1) || force_k == 1) {
    C = csz = (int)std::min<long long>(kClusMax, std::max<long long>(1, want));
    if (max_clusters(csz) < 1) return clus_fail(P, "cluster not launchable");
  } else {
    static const int force_csz = getenv("SPCG_CLUS_CSZ") ? atoi(getenv("SPCG_CLUS_CSZ")) : 0;  // dev A/B
    csz = (force_csz == 16 || force_csz == 4) ? force_csz : 8;
    // <= 32 clusters: the leaders' exchange polls one cluster slot per lane
    const int kmax = std::min(std::min(max_clusters(csz), kClusGridMax / csz), 32);
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
  mark("cluster shape");
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
  // slices: 32 rows of a block each
  std::vector<ClusCta> ctas(C);
  std::vector<ClusSlice> slices;
  std::vector<int2> rowmeta;
  std::vector<std::vector<int>> order(C);
  for (int c = 0; c < C; ++c) {
    std::vector<int>& o = order[c];
    for (int i = lo[c]; i < hi[c]; ++i) o.push_back(i);
    // row order inside a CTA's slices: natural (consecutive rows per slice:
    // the window gathers of banded rows hit consecutive banks) -- F 2.76 vs
    // 2.85 us per iteration on engine 6 and 5.96 vs 6.06 on engine 5 against
    // rows sorted by length (less padding, ~37 % excess shared-memory
    // wavefronts from bank conflicts); Poisson neutral.  (dev A/B)
    // SPCG_CLUS_SORT=1: by length, 2: by length within groups of
    // 32*SPCG_CLUS_SORTG rows
    static const int sort_mode = getenv("SPCG_CLUS_SORT") ? atoi(getenv("SPCG_CLUS_SORT")) : 0;
    static const int sort_g = getenv("SPCG_CLUS_SORTG") ? atoi(getenv("SPCG_CLUS_SORTG")) : 4;
    auto by_len = [&](int a, int b2) { return lenA(a) + lenB(a) > lenA(b2) + lenB(b2); };
    if (sort_mode == 1) std::stable_sort(o.begin(), o.end(), by_len);
    if (sort_mode == 2)
      for (size_t g0 = 0; g0 < o.size(); g0 += 32 * (size_t)std::max(1, sort_g))
        std::stable_sort(o.begin() + g0, o.begin() + std::min(o.size(), g0 + 32 * (size_t)std::max(1, sort_g)),
                         by_len);
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
    P.max_slices = std::max(P.max_slices, t.nslices);
    for (int s = 0; s < t.nslices; ++s) {
      ClusSlice sd{};
      int wdt = 0;
      for (int l = 0; l < 32; ++l) {
        const int q = 32 * s + l;
        if (q < (int)o.size()) wdt = std::max(wdt, lenA(o[q]) + lenB(o[q]));
      }
      sd.width = wdt;
      P.max_width = std::max(P.max_width, wdt);
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
  mark("blocks+slices");
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
  off = al(off + sizeof(double) * 3 * (size_t)hcap);  // engine 6: 3 buffers of halo n
  P.off_val = (int)off;
  const long long budget = (long long)optin - (long long)kClusStatic - (long long)off - 1024;
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
  mark("SELL pack");
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
  // per receiver: the in-cluster halo rows its neighbours send each iteration
  // (engine 6 expects exactly these bytes on its mbarrier)
  for (int c = 0; c < C; ++c) ctas[c].nrecv = 0;
  for (int dd = 0; dd < C; ++dd)
    for (int e = ctas[dd].send0; e < ctas[dd].send0 + ctas[dd].nsend; ++e)
      if (dd / csz == sends[e].dst / csz) ctas[sends[e].dst].nrecv += sends[e].hi - sends[e].lo;
  if (getenv("SPCG_CLUS_DEBUG"))
    for (int c = 0; c < C; ++c) {  // against the halo rows the receiver counts as in-cluster
      int nl = 0;
      const int clo = lo[(c / csz) * csz], chi = hi[(c / csz) * csz + csz - 1];
      for (int r = wlo[c]; r < whi[c]; ++r)
        if ((r < lo[c] || r >= hi[c]) && r >= clo && r < chi) ++nl;
      if (nl != ctas[c].nrecv)
        fprintf(stderr, "[spcg plan] cta %d: %d in-cluster halo rows, %d sent\n", c, nl, ctas[c].nrecv);
    }
  if (sends.empty()) sends.push_back(ClusSend{0, 0, 0, 0});
  // the grid of C CTAs in clusters of csz must be co-resident with this smem
  CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.smem));
  if (csz > 8) CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  // the pipelined kernel (engine 6) runs the same plan with one more warp
  const void* kpipes[4] = {(const void*)clus_pcg_kernel<2>, (const void*)clus_pcg_kernel<4>,
                           (const void*)clus_pcg_kernel<1, kRegThreads, kRegW>,
                           (const void*)clus_pcg_kernel<2, kRegThreads, kRegW2>};
  for (const void* kp : kpipes) {
    CUDA_TRY(cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.smem));
    if (csz > 8) CUDA_TRY(cudaFuncSetAttribute(kp, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  }
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
  mark("sends+attrs");
  // one device arena for the plan (one allocation, one copy of a host image
  // of the read-only part, one memset of the halo words): the first solve of
  // a matrix pays ~2 ms here instead of ~6 (SPCG_PLAN_TIMING)
  auto al256 = [](size_t v) { return (v + 255) & ~(size_t)255; };
  size_t o_ctas = 0;
  size_t o_slices = al256(o_ctas + sizeof(ClusCta) * ctas.size());
  size_t o_sends = al256(o_slices + sizeof(ClusSlice) * slices.size());
  size_t o_rowmeta = al256(o_sends + sizeof(ClusSend) * sends.size());
  size_t o_gval = al256(o_rowmeta + sizeof(int2) * rowmeta.size());
  size_t o_gcol = al256(o_gval + sizeof(double) * gval.size());
  const size_t ro_bytes = al256(o_gcol + sizeof(unsigned short) * gcol.size());
  const bool multi = C > csz;
  // [2][C][hcap] doubles (engine 5) or [3][C][hcap] epoch-tagged word pairs (engine 6)
  const size_t ghalo_bytes = multi ? sizeof(double) * 6 * (size_t)C * hcap : 0;
  const size_t gslot_bytes = multi ? sizeof(unsigned long long) * 2 * kClusSlotWords * (size_t)(C / csz) : 0;
  const size_t o_ghalo = ro_bytes, o_gslots = al256(o_ghalo + ghalo_bytes);
  const size_t total = al256(o_gslots + gslot_bytes);
  long long acct = 0;
  unsigned char* base = nullptr;
  if ((rc = dmalloc((void**)&base, total, &acct))) return rc;
  P.arena = base;
  std::vector<unsigned char> img(ro_bytes, 0);
  memcpy(img.data() + o_ctas, ctas.data(), sizeof(ClusCta) * ctas.size());
  memcpy(img.data() + o_slices, slices.data(), sizeof(ClusSlice) * slices.size());
  memcpy(img.data() + o_sends, sends.data(), sizeof(ClusSend) * sends.size());
  memcpy(img.data() + o_rowmeta, rowmeta.data(), sizeof(int2) * rowmeta.size());
  memcpy(img.data() + o_gval, gval.data(), sizeof(double) * gval.size());
  memcpy(img.data() + o_gcol, gcol.data(), sizeof(unsigned short) * gcol.size());
  CUDA_TRY(cudaMemcpy(base, img.data(), ro_bytes, cudaMemcpyHostToDevice));
  P.ctas = reinterpret_cast<ClusCta*>(base + o_ctas);
  P.slices = reinterpret_cast<ClusSlice*>(base + o_slices);
  P.sends = reinterpret_cast<ClusSend*>(base + o_sends);
  P.rowmeta = reinterpret_cast<int2*>(base + o_rowmeta);
  P.gval = reinterpret_cast<double*>(base + o_gval);
  P.gcol = reinterpret_cast<unsigned short*>(base + o_gcol);
  if (multi) {
    P.ghalo = reinterpret_cast<double*>(base + o_ghalo);
    P.gslots = reinterpret_cast<unsigned long long*>(base + o_gslots);
    CUDA_TRY(cudaMemset(P.ghalo, 0, ghalo_bytes));
  }
  mark("upload");
  m->bytes += acct;
  P.hcap = hcap;
  P.C = C;
  P.cs = csz;
  P.ok = true;
  return SPCG_OK;
}

int launch_clus(const ClusPlan& P, const ClusArgs& a, cudaStream_t st, bool pipe) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P.C);
  // engine 6 with register rows: every slice in one 384-thread CTA's 11 row
  // warps (one slot each) and rows of <= kRegW entries (SPCG_PIPE_REG=0: off)
  static const bool reg_ok = !getenv("SPCG_PIPE_REG") || atoi(getenv("SPCG_PIPE_REG")) != 0;
  const int rw_ = kRegThreads / 32 - 1;  // row warps of the register variants
  const bool reg = pipe && reg_ok && P.max_slices <= rw_ && P.max_width <= kRegW;
  // two register rows per thread for short rows (stencils): <= 2 * 11 slices
  const bool reg2 = pipe && reg_ok && !reg && P.max_slices <= 2 * rw_ && P.max_width <= kRegW2;
  cfg.blockDim = dim3((reg || reg2) ? kRegThreads : pipe ? kPipeThreads : kClusThreads);
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
  if (reg) {
    CUDA_TRY(cudaLaunchKernelEx(&cfg, clus_pcg_kernel<1, kRegThreads, kRegW>, a));
  } else if (reg2) {
    CUDA_TRY(cudaLaunchKernelEx(&cfg, clus_pcg_kernel<2, kRegThreads, kRegW2>, a));
  } else if (pipe) {
    const bool ns2 = P.max_slices <= kPipeMaxSlices2;
    // (two-segment plans too: engine 6 sums their rows in one chain)
    if (ns2) CUDA_TRY(cudaLaunchKernelEx(&cfg, clus_pcg_kernel<2>, a));
    else CUDA_TRY(cudaLaunchKernelEx(&cfg, clus_pcg_kernel<4>, a));
  } else if (P.two) {
    CUDA_TRY(cudaLaunchKernelEx(&cfg, clus_cg_kernel<true>, a));
  } else {
    CUDA_TRY(cudaLaunchKernelEx(&cfg, clus_cg_kernel<false>, a));
  }
  return SPCG_OK;
}

// Extreme eigenvalues of CG's Lanczos tridiagonal T_k from the step
// coefficients (alpha_j, beta_j), beta_0 = 0:
//   T_jj = 1/alpha_j + beta_j/alpha_{j-1},  T_{j-1,j} = sqrt(beta_j)/alpha_{j-1}
// by Sturm-count multisection (below); returns theta_max / theta_min (the Ritz
// estimate of cond(A): the extreme Ritz values converge first) or 0.
double lanczos_cond(const std::vector<double>& ab, long long k) {
  if (k < 2) return 0.0;
  std::vector<double> d((size_t)k), e2((size_t)k, 0.0);
  double lo = 1e300, hi = -1e300;
  for (long long j = 0; j < k; ++j) {
    const double a = ab[2 * j], bb = j ? ab[2 * j + 1] : 0.0, ap = j ? ab[2 * (j - 1)] : 1.0;
    if (!(a > 0.0) || !(bb >= 0.0)) return 0.0;
    d[j] = 1.0 / a + (j ? bb / ap : 0.0);
    e2[j] = j ? bb / (ap * ap) : 0.0;
  }
  for (long long j = 0; j < k; ++j) {  // Gershgorin interval of T
    const double r = (j ? std::sqrt(e2[j]) : 0.0) + (j + 1 < k ? std::sqrt(e2[j + 1]) : 0.0);
    lo = std::min(lo, d[j] - r);
    hi = std::max(hi, d[j] + r);
  }
  // brackets: T is SPD (its extreme eigenvalues enclose the diagonal), so
  // theta_min in [max(0, lo), min d] and theta_max in [max d, hi]
  double dmin = d[0], dmax = d[0];
  for (long long j = 1; j < k; ++j) {
    dmin = std::min(dmin, d[j]);
    dmax = std::max(dmax, d[j]);
  }
  // multisection with division-free Sturm counts: the leading principal
  // minors p_j = (d_j - x) p_{j-1} - e_j^2 p_{j-2} change sign exactly
  // (number of eigenvalues below x) times.  T is scaled by 1/hi first (the
  // ratio is scale-free), so a step grows |p| at most ~2x and a rescale
  // every 4 steps keeps it in range.  NP points per bracket per round, all
  // 2 NP recurrences in one pass over T, branch-free (independent
  // multiply-adds that vectorise), so a round narrows each bracket (NP + 1)x
  // for about the cost of one count.  2e-3 relative is ample for a guard
  // threshold of 1e5 (this host time sits on every auto solve's path)
  constexpr int NP = 8, NX = 2 * NP;
  const double sc = 1.0 / hi;
  for (long long j = 0; j < k; ++j) {
    d[j] *= sc;
    e2[j] *= sc * sc;
  }
  double a0 = std::max(0.0, lo) * sc, z0 = dmin * sc, a1 = dmax * sc, z1 = 1.0;
  auto done = [](double a, double z) { return z - a <= 2e-3 * std::max(std::fabs(a), std::fabs(z)); };
  for (int round = 0; round < 64 && !(done(a0, z0) && done(a1, z1)); ++round) {
    // (gcc vector extensions: two lanes per op on any host ISA)
    typedef double v2d __attribute__((vector_size(16)));
    typedef long long v2l __attribute__((vector_size(16)));
    constexpr int NV = NX / 2;
    alignas(64) double x[NX], c[NX];
    // a bracket already narrow enough gives its points to the other one
    const int n0 = done(a1, z1) ? NX : done(a0, z0) ? 0 : NP, n1 = NX - n0;
    for (int i = 0; i < n0; ++i) x[i] = a0 + (z0 - a0) * (i + 1) / (n0 + 1);
    for (int i = 0; i < n1; ++i) x[n0 + i] = a1 + (z1 - a1) * (i + 1) / (n1 + 1);
    v2d vx[NV], pm[NV], pc[NV], vc[NV];
    const v2d one = {1.0, 1.0}, zero = {0.0, 0.0}, tiny = {1e-300, 1e-300};
    for (int v = 0; v < NV; ++v) {
      vx[v] = v2d{x[2 * v], x[2 * v + 1]};
      pm[v] = one;  // p_{-1}
      pc[v] = d[0] - vx[v];
      vc[v] = (v2d)((v2l)one & (pc[v] < zero));
    }
    auto step = [&](long long j) {
      const double dj = d[j], ej = e2[j];
      for (int v = 0; v < NV; ++v) {
        v2d pn = (dj - vx[v]) * pc[v] - ej * pm[v];
        pn += tiny;  // an exact zero takes a sign (probability ~0); a no-op otherwise
        vc[v] += (v2d)((v2l)one & (pn * pc[v] < zero));
        pm[v] = pc[v];
        pc[v] = pn;
      }
    };
    long long j = 1;
    for (; j + 4 <= k; j += 4) {
      step(j);
      step(j + 1);
      step(j + 2);
      step(j + 3);
      for (int v = 0; v < NV; ++v) {
        const v2d apc = (v2d)((v2l)pc[v] & 0x7fffffffffffffffLL), apm = (v2d)((v2l)pm[v] & 0x7fffffffffffffffLL);
        const v2d m = one / (apc + apm);
        pc[v] *= m;
        pm[v] *= m;
      }
    }
    for (; j < k; ++j) step(j);
    for (int v = 0; v < NV; ++v) {
      c[2 * v] = vc[v][0];
      c[2 * v + 1] = vc[v][1];
    }
    // theta_min: the first point with an eigenvalue below it
    double na = a0, nz = z0;
    for (int i = 0; i < n0; ++i)
      if (c[i] > 0.5) {
        nz = x[i];
        break;
      } else {
        na = x[i];
      }
    a0 = na;
    z0 = nz;
    // theta_max: the first point with every eigenvalue below it
    na = a1;
    nz = z1;
    for (int i = n0; i < NX; ++i)
      if (c[i] > (double)k - 0.5) {
        nz = x[i];
        break;
      } else {
        na = x[i];
      }
    a1 = na;
    z1 = nz;
  }
  const double tmin = 0.5 * (a0 + z0), tmax = 0.5 * (a1 + z1);
  return tmin > 0.0 ? tmax / tmin : 0.0;
}

// Auto-mode guard of the pipelined engine: Ghysels-Vanroose CG follows the
// reference's iterates to fp64 reassociation only while the system is
// reasonably conditioned; measured on the F-mesh family and 2-D Poisson
// (tests/test_gpu_conditioning.py, profiles/r02/cond_sweep.jsonl):
// ||x6 - x_ref|| / ||x_ref|| <= 3e-9 up to cond ~ 8e4, 6.5e-8 at 1.9e5,
// 1e-6 at 1.9e6; and at tol 1e-12 the true residual ends 16x above tol.
// Above either limit the auto mode re-solves on engine 5 (standard-order
// single-reduction CG, within 1e-9 of the reference in the same sweep).
constexpr double kPipeCondMax = 1.0e5;
constexpr long long kCoefHost = 4096;  // guard coefficients copied with the result
constexpr double kPipeTrueResMax = 2.0;  // true rel residual / tol

int do_clus_cg(spcg_matrix_s* m, const double* b, const double* x0, double* x, double* hist,
               const spcg_cg_options* o, spcg_cg_result* out, cudaStream_t st, bool pipe = false,
               bool guard = false) {
  int rc;
  const auto tentry = std::chrono::steady_clock::now();
  const ClusPlan& P = m->cp;
  if ((rc = ensure_ws(m, 1))) return rc;
  Workspace& w = m->ws;
  const long long max_iter = o->max_iter > 0 ? o->max_iter : std::max(1, m->n);
  if (o->record_history && hist == nullptr)
    return fail(SPCG_ERR_ARG, "record_history needs a history buffer");
  guard = guard && pipe;
  if (guard && w.coef_cap < max_iter) {
    if (w.coef) cudaFree(w.coef);
    w.coef = nullptr;
    if ((rc = dmalloc((void**)&w.coef, sizeof(double) * 2 * (size_t)max_iter, nullptr))) return rc;
    w.coef_cap = max_iter;
  }
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
  a.scratch2 = w.p0;
  a.hist = hist;
  a.res = w.res;
  a.tol = o->tol;
  a.max_iter = max_iter;
  a.record_history = o->record_history;
  // the guard judges the TRUE residual, computed even when not requested
  a.recompute = o->recompute_final_residual || guard;
  a.coef = guard ? w.coef : nullptr;
  a.off_rwin = P.off_rwin;
  a.off_shalo = P.off_shalo;
  a.off_whalo = P.off_whalo;
  a.off_val = P.off_val;
  a.off_col = P.off_col;
  a.hcap = P.hcap;
  a.ghalo = P.ghalo;
  a.gslots = P.gslots;
  a.cluster_size = P.cs;
  if (P.gslots) {
    // tags restart at 1 every solve: engine 6 clears its halo words too, in
    // the same memset (the arena holds ghalo right before gslots)
    const unsigned char* end =
        reinterpret_cast<const unsigned char*>(P.gslots + 2 * kClusSlotWords * (size_t)(P.C / P.cs));
    unsigned char* from = reinterpret_cast<unsigned char*>(pipe && P.ghalo ? (void*)P.ghalo : (void*)P.gslots);
    CUDA_TRY(cudaMemsetAsync(from, 0, (size_t)(end - from), st));
  }
  static const bool tracing = getenv("SPCG_TRACE") != nullptr;
  static const char* dbg_path = getenv("SPCG_CLUS_DEBUG");  // per-solve CTA trace lines
  // [C][8] per-CTA phases + [K][8 iterations][34] exchange trace (engine 6)
  // (SPCG_PIPE_FINE builds: [C][16] sub-phase totals in place of the exchange trace)
  // (SPCG_XCHG_TRACE builds: + [C][8 iterations][6] per-CTA timeline)
  const size_t tl0 = 8 * (size_t)P.C +
                     std::max((size_t)(P.C / std::max(1, P.cs)) * 8 * 34, 16 * (size_t)P.C);
  const size_t trace_words = tl0 + (size_t)P.C * 8 * 6;
  if (tracing || dbg_path) {
    CUDA_TRY(cudaMalloc((void**)&a.trace, sizeof(unsigned long long) * trace_words));
    CUDA_TRY(cudaMemsetAsync(a.trace, 0, sizeof(unsigned long long) * trace_words, st));
  }
  static const bool etime = getenv("SPCG_E2E_TIMING") != nullptr;  // (dev)
  const auto te0 = std::chrono::steady_clock::now();
  CUDA_TRY(cudaEventRecord(w.ev0, st));
  if ((rc = launch_clus(P, a, st, pipe))) return rc;
  CUDA_TRY(cudaEventRecord(w.ev1, st));
  const auto te1 = std::chrono::steady_clock::now();
  // the guard's coefficients ride along with the result (one wait, not two)
  const long long coef_pre = guard ? std::min<long long>(max_iter, kCoefHost) : 0;
  if (coef_pre > 0) {
    if (!w.h_coef) CUDA_TRY(cudaMallocHost((void**)&w.h_coef, sizeof(double) * 2 * kCoefHost));
    CUDA_TRY(cudaMemcpyAsync(w.h_coef, w.coef, sizeof(double) * 2 * (size_t)coef_pre,
                             cudaMemcpyDeviceToHost, st));
  }
  CUDA_TRY(cudaMemcpyAsync(w.h_res, w.res, sizeof(CgDevResult), cudaMemcpyDeviceToHost, st));
  const auto te2 = std::chrono::steady_clock::now();
  // a guarded host-API solve: x's copy to the caller runs while the host
  // computes the guard (re-copied after a fallback re-solve)
  const bool early = guard && w.h_x_early && x == w.x && !(tracing || dbg_path);
  if (early) {
    CUDA_TRY(cudaEventRecord(w.ev_res, st));
    CUDA_TRY(cudaMemcpyAsync(w.h_x_early, w.x, sizeof(double) * (size_t)m->n,
                             cudaMemcpyDeviceToHost, st));
    w.x_early_done = true;
    CUDA_TRY(cudaEventSynchronize(w.ev_res));
  } else {
    CUDA_TRY(cudaStreamSynchronize(st));
  }
  const auto te3 = std::chrono::steady_clock::now();
  float ms = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&ms, w.ev0, w.ev1));
  if (etime) {
    auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
    fprintf(stderr, "[spcg e2e] entry->launch %.1f launch %.1f copies %.1f sync-wait %.1f (kernel %.1f) us\n",
            us(tentry, te0), us(te0, te1), us(te1, te2), us(te2, te3), 1e3 * ms);
  }
  const CgDevResult& r = *w.h_res;
  if (r.status == ST_BAD_LAUNCH)
    return fail(SPCG_ERR_CUDA, "cluster engine: kernel ran with a different cluster shape than "
                               "planned (cluster launch attribute not honoured)");
  if (a.trace && pipe) {
    std::vector<unsigned long long> tv(trace_words);
    CUDA_TRY(cudaMemcpy(tv.data(), a.trace, sizeof(unsigned long long) * tv.size(),
                        cudaMemcpyDeviceToHost));
    cudaFree(a.trace);
    a.trace = nullptr;
    const double it = (double)std::max<long long>(1, r.iterations) * 1e3;
    double mean[4] = {0, 0, 0, 0}, mx[4] = {0, 0, 0, 0};
    unsigned long long t0 = ~0ull, t1 = 0;
    for (int c = 0; c < P.C; ++c) {
      for (int ph = 0; ph < 4; ++ph) {
        mean[ph] += (double)tv[8 * c + ph] / P.C;
        mx[ph] = std::max(mx[ph], (double)tv[8 * c + ph]);
      }
      t0 = std::min(t0, tv[8 * c + 5]);
      t1 = std::max(t1, tv[8 * c + 6]);
    }
    if (tracing)
      fprintf(stderr,
              "[spcg trace] engine 6 ctas=%d cs=%d two=%d us/iter mean(max): partials+spmv %.3f(%.3f) "
              "waitA %.3f(%.3f) send+barrierB %.3f(%.3f) update %.3f(%.3f); kernel %.1f us\n",
              P.C, P.cs, (int)P.two, mean[0] / it, mx[0] / it, mean[1] / it, mx[1] / it,
              mean[2] / it, mx[2] / it, mean[3] / it, mx[3] / it, (double)(t1 - t0) / 1e3);
    if (dbg_path) {
      if (FILE* f = fopen(dbg_path, "a")) {
        fprintf(f, "{\"engine\": 6, \"two\": %d, \"cs\": %d, \"ms\": %.6f, \"iters\": %lld, \"ctas\": [",
                (int)P.two, P.cs, ms, (long long)r.iterations);
        for (int c = 0; c < P.C; ++c)
          fprintf(f, "%s[%llu, %llu, %llu, %llu, %llu, %llu, %llu]", c ? ", " : "", tv[8 * c + 4],
                  tv[8 * c + 5] - t0, tv[8 * c + 6] - t0, tv[8 * c + 0], tv[8 * c + 1],
                  tv[8 * c + 2], tv[8 * c + 3]);
        fprintf(f, "], \"xch\": [");
        const int K = P.C / std::max(1, P.cs);
        for (size_t w = 8 * (size_t)P.C; w < 8 * (size_t)P.C + (size_t)K * 8 * 34; ++w)
          fprintf(f, "%s%lld", w > 8 * (size_t)P.C ? ", " : "",
                  tv[w] ? (long long)(tv[w] - t0) : -1LL);
        fprintf(f, "], \"fine\": [");
        for (size_t w = 0; w < 16 * (size_t)P.C; ++w)
          fprintf(f, "%s%llu", w ? ", " : "", tv[8 * (size_t)P.C + w]);
        fprintf(f, "], \"tl\": [");
        for (size_t w = tl0; w < trace_words; ++w)
          fprintf(f, "%s%lld", w > tl0 ? ", " : "", tv[w] ? (long long)(tv[w] - t0) : -1LL);
        fprintf(f, "], \"K\": %d}\n", K);
        fclose(f);
      }
    }
  }
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
  double cond = 0.0;
  if (guard && r.status == SPCG_OK && r.iterations >= 2) {
    std::vector<double> ab(2 * (size_t)r.iterations);
    if (r.iterations <= coef_pre)
      std::copy(w.h_coef, w.h_coef + ab.size(), ab.begin());
    else
      CUDA_TRY(cudaMemcpy(ab.data(), w.coef, sizeof(double) * ab.size(), cudaMemcpyDeviceToHost));
    static const bool gtime = getenv("SPCG_GUARD_TIMING") != nullptr;  // (dev)
    const auto tg0 = std::chrono::steady_clock::now();
    cond = lanczos_cond(ab, r.iterations);
    if (gtime)
      fprintf(stderr, "[spcg guard] lanczos %.1f us (k = %lld)\n",
              std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tg0).count(),
              (long long)r.iterations);
    if (cond > kPipeCondMax || r.final_rel > kPipeTrueResMax * o->tol) {
      // re-solve on engine 5; the reported time covers both solves
      w.x_early_done = false;  // (the copy already queued carries engine 6's x)
      rc = do_clus_cg(m, b, x0, x, hist, o, out, st, false, false);
      out->device_ms += ms;
      out->kernel_launches += 1;
      out->fallbacks = 1;
      out->cond_estimate = cond;
      return rc;
    }
  }
  out->iterations = r.iterations;
  out->converged = r.converged;
  out->status = r.status;
  out->fail_iteration = r.fail_iter;
  out->final_relative_residual =
      (pipe && !o->recompute_final_residual && r.status == SPCG_OK) ? r.rec_rel : r.final_rel;
  out->b_norm = r.b_norm;
  out->device_ms = ms;
  out->kernel_launches = 1;
  out->spmv_ms = 0.0;
  out->spmv_launches = 0;
  out->engine_used = pipe ? 6 : 5;
  out->fallbacks = 0;
  out->cond_estimate = cond;
  out->phase_ms[0] = out->phase_ms[1] = out->phase_ms[2] = 0.0;
  if (r.status == SPCG_OK && r.iterations > 0) {  // the leader's loop phases
    out->phase_ms[0] = (double)r.phase_ns[0] / 1e6;
    out->phase_ms[2] = (double)r.phase_ns[2] / 1e6;
    out->phase_ms[1] = std::max(0.0, (double)ms - out->phase_ms[0] - out->phase_ms[2]);
  }
  if (r.status != SPCG_OK) {
    const char* what = r.status == SPCG_ERR_NOT_SPD ? "matrix not positive definite"
                       : r.status == SPCG_ERR_NONFINITE_ALPHA ? "non-finite alpha"
                       : r.status == SPCG_ERR_NONFINITE_RESIDUAL ? "non-finite residual"
                                                                  : "non-finite beta";
    return fail(r.status, std::string(what) + " at iteration " + std::to_string(r.fail_iter));
  }
  return SPCG_OK;
}
