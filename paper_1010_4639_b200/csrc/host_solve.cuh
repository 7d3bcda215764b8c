// host_solve.cuh — host side of spcg_b200.cu: the solve dispatcher (engine routing) and matrix creation / generation.
// Included exactly once, by spcg_b200.cu inside its anonymous namespace
// (one translation unit: the kernels' templates are instantiated there).
#pragma once

// engine 7 (cg1.cuh cg1s_kernel): streamed single-reduction CG, one
// persistent cooperative launch per solve
int do_cg1s(spcg_matrix_s* m, int kf, const double* b, const double* x0, double* x, double* hist,
            const spcg_cg_options* o, spcg_cg_result* out, cudaStream_t st) {
  DevInfo* d;
  int rc;
  if ((rc = dev_info(&d))) return rc;
  int grid = 1;
  if ((rc = kf == K_CSR ? cg1s_grid<K_CSR>(d, &grid) : cg1s_grid<K_SCSR_PRIV>(d, &grid))) return rc;
  const MatView v = view(m, kf == K_SCSR_PRIV);
  grid = std::max(1, std::min(grid, v.ntiles));
  if ((rc = ensure_ws(m, grid))) return rc;
  Workspace& w = m->ws;
  if (o->record_history && hist == nullptr)
    return fail(SPCG_ERR_ARG, "record_history needs a history buffer");
  const size_t vb = sizeof(double) * (size_t)std::max(1, m->n);
  if (!w.cg1 && (rc = dmalloc((void**)&w.cg1, 8 * vb, nullptr))) return rc;
  CUDA_TRY(cudaMemsetAsync(w.cg1, 0, 8 * vb, st));  // s_{-1} = 0, p_{-1} = 0
  CUDA_TRY(cudaMemsetAsync(w.slots, 0, sizeof(unsigned long long) * 2 * kSlotWords * (size_t)grid, st));
  Cg1sArgs a{};
  CgArgs& c = a.g.base;
  c.M = v;
  c.b = b;
  c.x0 = x0;
  c.x = x;
  c.q = w.q;
  c.hist = hist;
  c.slots = w.slots;
  c.res = w.res;
  c.tol = o->tol;
  c.max_iter = o->max_iter > 0 ? o->max_iter : std::max(1, m->n);
  c.record_history = o->record_history;
  c.recompute = o->recompute_final_residual;
  for (int k = 0; k < 2; ++k) a.g.R[k] = w.cg1 + (size_t)k * std::max(1, m->n);
  for (int k = 0; k < 2; ++k) a.g.S[k] = w.cg1 + (size_t)(2 + k) * std::max(1, m->n);
  for (int k = 0; k < 3; ++k) a.g.W[k] = w.cg1 + (size_t)(4 + k) * std::max(1, m->n);
  a.Pv = w.cg1 + (size_t)7 * std::max(1, m->n);
  CUDA_TRY(cudaEventRecord(w.ev0, st));
  if ((rc = kf == K_CSR ? launch_cg1s<K_CSR>(a, grid, st) : launch_cg1s<K_SCSR_PRIV>(a, grid, st)))
    return rc;
  CUDA_TRY(cudaEventRecord(w.ev1, st));
  CUDA_TRY(cudaMemcpyAsync(w.h_res, w.res, sizeof(CgDevResult), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  float ms = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&ms, w.ev0, w.ev1));
  const CgDevResult& r = *w.h_res;
  *out = spcg_cg_result{};
  out->iterations = r.iterations;
  out->converged = r.converged;
  out->status = r.status;
  out->fail_iteration = r.fail_iter;
  out->final_relative_residual = r.final_rel;
  out->b_norm = r.b_norm;
  out->device_ms = ms;
  out->kernel_launches = 1;
  out->engine_used = 7;
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
  if (o->engine != 0 && o->engine != 2 && o->engine != 3 && o->engine != 5 && o->engine != 6 &&
      o->engine != 7)
    return fail(SPCG_ERR_ARG, "engine must be 0 (auto), 2, 3, 5, 6 or 7");
  const MatView v = view(m, kf == K_SCSR_PRIV);
  const bool fits = v.ntiles <= d->coop_res * kStages;
  if (o->engine == 7) {
    if (kf != K_CSR && kf != K_SCSR_PRIV)
      return fail(SPCG_ERR_UNSUPPORTED, "engine 7 takes gather formats (CSR, privatized symmetric half)");
    return do_cg1s(m, kf, b, x0, x, hist, o, out, st);
  }
  // engine 2, and auto for systems that stream from HBM: per-pass kernels
  // (the sharded engine with no peers) — each pass keeps the whole register
  // budget, which a persistent kernel cannot (P3: 0.99 vs 0.82 of roofline)
  // auto, full CSR that does not fit on chip but whose tile list is short
  // (<= 16 tiles per co-resident CTA, ~1 M rows): engine 7's one persistent
  // launch beats three launches per iteration (2-D Poisson 512^2 12.7 vs
  // 30.6 us per iteration, 3-D 100^3 42.9 vs 50.0); beyond that the per-pass
  // kernels stream faster (3-D 128^3 73.8 vs 103.6); symmetric-half
  // privatized would stream L^T too (27-point 64^3 57.6 vs 45.6), so not
  // there (scripts/engine7_ab.py)
  if (o->engine == 0 && !fits && kf == K_CSR) {
    int g7 = 1;
    if ((rc = cg1s_grid<K_CSR>(d, &g7))) return rc;
    if (v.ntiles <= 16 * g7) return do_cg1s(m, kf, b, x0, x, hist, o, out, st);
  }
  if (o->engine == 2 || (o->engine == 0 && !fits))
    return do_dist_cg(m, nullptr, 0, nullptr, nullptr, nullptr, nullptr, b, x0, x, hist, o, out, st);
  // engine 5, and auto for banded systems whose rows fit the co-resident
  // clusters' shared memory: cluster-resident single-reduction CG (DSMEM +
  // hardware cluster barriers; K clusters of 8 exchange through global
  // memory).  F: 5.35 us/iteration vs 8.45 on engine 3; S: 6.23 vs 8.58.
  // engine 6: the same plan, pipelined CG (SpMV overlapped with the all-reduce)
  if (o->engine == 6) {
    if ((rc = build_clus_plan(m))) return rc;
    if (!m->cp.ok) return fail(SPCG_ERR_UNSUPPORTED, "cluster engine not applicable: " + m->cp.why);
    if (m->cp.max_slices > kPipeMaxSlices)
      return fail(SPCG_ERR_UNSUPPORTED, "pipelined cluster engine: too many rows per CTA");
    return do_clus_cg(m, b, x0, x, hist, o, out, st, true);
  }
  if (o->engine == 5 || (o->engine == 0 && m->n <= kClusGridMax * kClusMaxRows)) {
    if ((rc = build_clus_plan(m))) return rc;
    // auto only when (nearly) everything stays in shared memory: streamed
    // slices are re-read from L2 every iteration at L2 latency
    const bool resident = m->cp.streamed * 9 <= m->cp.resident;
    // auto picks the pipelined form (engine 6) when its row slots hold the
    // plan, for single- and two-segment rows alike: F 4.6 vs 5.7 us per
    // iteration, S 5.3 vs 6.3 (round 1 kept SCSR on engine 5 because engine 6
    // ran it at 7-11 us on some boxes: the divergent spin of the leaders'
    // poll, fixed in round 2 -- profiles/r02/bimodal.md)
    if (m->cp.ok && (o->engine == 5 || resident)) {
      const bool pipe = o->engine == 0 && m->cp.max_slices <= kPipeMaxSlices;
      return do_clus_cg(m, b, x0, x, hist, o, out, st, pipe, /*guard=*/pipe);
    }
    if (o->engine == 5)
      return fail(SPCG_ERR_UNSUPPORTED, "cluster engine not applicable: " + m->cp.why);
  }
  // engine 3 (and auto on the remaining resident systems): the grid-resident
  // single-reduction CG, one grid all-reduce per iteration
  if (!fits)
    return fail(SPCG_ERR_UNSUPPORTED, "engine 3 needs a system resident in shared memory");
  // the balanced tiles map one-to-one onto CTAs where possible
  const int grid = std::max(1, std::min(d->coop_res, std::max(1, v.ntiles)));
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
  Cg1Args g{};
  const size_t vb = sizeof(double) * (size_t)std::max(1, m->n);
  if (!w.cg1 && (rc = dmalloc((void**)&w.cg1, 8 * vb, nullptr))) return rc;  // (+ p of engine 7)
  CUDA_TRY(cudaMemsetAsync(w.cg1, 0, 7 * vb, st));
  g.base = a;
  for (int k = 0; k < 2; ++k) g.R[k] = w.cg1 + (size_t)k * std::max(1, m->n);
  for (int k = 0; k < 2; ++k) g.S[k] = w.cg1 + (size_t)(2 + k) * std::max(1, m->n);
  for (int k = 0; k < 3; ++k) g.W[k] = w.cg1 + (size_t)(4 + k) * std::max(1, m->n);
  const bool res = true;
  CUDA_TRY(cudaEventRecord(w.ev0, st));
  switch (kf) {
    case K_CSR: rc = launch_cg1<K_CSR>(g, grid, st); break;
    case K_SCSR_ATOMIC: rc = launch_cg1<K_SCSR_ATOMIC>(g, grid, st); break;
    case K_SCSR_PRIV: rc = launch_cg1<K_SCSR_PRIV>(g, grid, st); break;
    default: rc = launch_cg1<K_CSC>(g, grid, st); break;
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
  out->engine_used = 3;
  out->fallbacks = 0;
  out->cond_estimate = 0.0;
  out->phase_ms[0] = out->phase_ms[1] = out->phase_ms[2] = 0.0;
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

// Host arrays -> a matrix handle: the raw offsets / indices / values go to
// the device as they are (no host conversion loop), where create_from_device
// (host_assemble.cuh) converts them to int32 and validates them in parallel
// and builds SCSR's L^T by a device radix sort.
template <class PT, class IT>
int create_from_host(int fmt, int64_t n, int64_t nnz, const PT* hp, const IT* hi, const double* hv,
                     spcg_matrix_t* out);
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
