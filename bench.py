"""Benchmark: fp64 CG iterations/s (and SpMV HBM GB/s, % of roofline) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload p3|p2|q27|q27p|f|s|csc] [--max-iter M]

Workload (BASELINE.json configs[3]; the largest single-GPU config and the one
the metric's 1/2/4/8-GPU scaling is quoted on): 3-D 7-point Poisson 400^3
(n = 64,000,000, nnz = 447,040,000), full CSR, fp64, x0 = 0, b = A x_gen with
x_gen = default_rng(1).standard_normal(n), tol 1e-10.  One step = one complete
cg_solve (944 iterations + the true-residual recompute).  Inputs (5.6 GB of
matrix) are far larger than L2 (126 MB), so no L2 flush is needed.

`value` = total CG iterations / device time of K solves (CUDA events on the
solve stream, barrier + synchronize on both sides, max over ranks);
`e2e` = the same through the C-ABI host entry point spcg_cg_solve_host with
b in pinned host memory and x copied back every step.
`roofline` = algorithmic bytes of one solve-kernel launch / its CUDA-event
duration vs MEASURED_PEAKS.json hbm_gbs.  `cpu_baseline` = the reference's own
compiled kernels (oracle/_ref, built from the reference sources) driven by
the reference CG loop on this host, on a 20-iteration window of the same
system.  `--impl reference` times that CPU path alone (the driver's reference
arm).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # name: (generator kind, dims, storage, accumulation, description)
    "p3": ("poisson3d", (400, 400, 400), "csr", 1, "3D 7-point Poisson 400^3, CSR fp64 CG"),
    "p2": ("poisson2d", (4096, 4096), "csr", 1, "2D 5-point Poisson 4096^2, CSR fp64 CG"),
    "q27": ("stencil27", (256, 256, 256), "scsr", 0,
            "3D 27-point stencil 256^3, symmetric CSR (L+D, atomic scatter) fp64 CG"),
    "q27p": ("stencil27", (256, 256, 256), "scsr", 1,
             "3D 27-point stencil 256^3, symmetric CSR (L+D and L^T rows, privatized: "
             "deterministic, the reference's default accumulation) fp64 CG"),
    "f": ("fem", None, "csr", 1, "FEM-shaped 30880x30880 / 449,798 nnz, full CSR fp64 CG"),
    "s": ("fem", None, "scsr", 1, "FEM-shaped 30880, symmetric CSR (L+D) fp64 CG"),
    "csc": ("fem", None, "csc", 1, "FEM-shaped 30880, CSC fp64 CG"),
}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def iter_bytes(n, nnz):
    """algorithmic bytes of one CG iteration."""
    return 12 * nnz + 4 * (n + 1) + 88 * n


def spmv_bytes(n, nnz):
    return 12 * nnz + 4 * (n + 1) + 16 * n


def solve_bytes(n, nnz, iterations, recompute=True):
    """Algorithmic bytes of one solve-kernel launch: ||b|| (8n), x=0 & r=b
    (24n), r.r (8n); per iteration iter_bytes; x += alpha p (24n); true
    residual = SpMV + b - q (spmv_bytes + 16n)."""
    b = 40 * n + iterations * iter_bytes(n, nnz) + 24 * n
    if recompute:
        b += spmv_bytes(n, nnz) + 16 * n
    return b


# ---- clocks ---------------------------------------------------------------
class ClockSampler:
    """SM clock / power / throttle reasons sampled DURING the timed region:
    NVML polled every 2 ms from a thread (short regions such as a 10 ms F
    run still get samples); nvidia-smi -lms 200 as the fallback."""
    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
               ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4))

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None
        self.path = None
        self.thread = None
        self.stop = None

    def __enter__(self):
        try:
            import threading

            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(max(0, self.idx))
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.stop = threading.Event()

            def poll():
                while not self.stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.rows.append((float(sm), float(mx), pw, int(rs)))
                    except Exception:  # noqa: BLE001
                        pass
                    self.stop.wait(0.002)

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return self
        except Exception:  # noqa: BLE001 - no NVML: nvidia-smi
            self.thread = None
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            sel = ["-i", str(self.idx)] if self.idx >= 0 else []
            self.proc = subprocess.Popen(
                ["nvidia-smi", *sel, "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.thread is not None:
            self.stop.set()
            self.thread.join(timeout=2)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            try:
                for line in open(self.path):
                    p = [x.strip() for x in line.split(",")]
                    if len(p) >= 7 and p[0].replace(".", "").isdigit():
                        bits = sum(m for (_, m), v in zip(self.REASONS, p[3:7]) if v == "Active")
                        self.rows.append((float(p[0]), float(p[1]),
                                          float(p[2]) if p[2].replace(".", "").isdigit() else 0.0,
                                          bits))
            except OSError:
                pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [r[0] for r in self.rows]
        mx = max(r[1] for r in self.rows)
        reasons = sorted({name for r in self.rows for name, bit in self.REASONS if r[3] & bit})
        loaded = [v for v in sm if v > 0.5 * mx] or sm
        return {"sm_mhz": float(np.median(loaded)), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows), "power_w_max": max(r[2] for r in self.rows),
                "source": "nvml" if self.thread is not None else "nvidia-smi"}


# ---- system construction ----------------------------------------------------------
def build_device_system(workload: str):
    """(DeviceMatrix, b (cuda tensor), n, stored nnz, x_gen numpy)."""
    import torch

    from paper_1010_4639_b200 import _native as N
    from paper_1010_4639_b200.core import extract_lower
    from paper_1010_4639_b200.device import DeviceMatrix
    from paper_1010_4639_b200.genprob import fem_mesh, rhs_for

    kind, dims, fmt, acc, _ = WORKLOADS[workload]
    if kind == "fem":
        F = fem_mesh()
        b, xg = rhs_for(F, seed=1)
        m = {"csr": F, "scsr": extract_lower(F) if fmt == "scsr" else None,
             "csc": F.to_csc() if fmt == "csc" else None}[fmt]
        dm = m.device()
        return dm, torch.from_numpy(b).cuda(), m.n, m.nnz, xg, acc
    dm = DeviceMatrix.generate(kind, dims, fmt)
    n = dm.n
    xg = np.random.default_rng(1).standard_normal(n)
    xt = torch.from_numpy(xg).cuda()
    full = dm if fmt == "csr" else DeviceMatrix.generate(kind, dims, "csr")
    bt = torch.empty_like(xt)
    N.check(N.load().spcg_spmv(full.handle, xt.data_ptr(), bt.data_ptr(), 1,
                               torch.cuda.current_stream().cuda_stream), "rhs spmv")
    torch.cuda.synchronize()
    if full is not dm:
        full.close()
    del xt
    return dm, bt, n, dm.nnz, xg, acc


_HOST_CACHE: dict = {}


def host_system(workload: str):
    """Host int64 arrays of the same system for the CPU path: (kind, rs, ci, v, b).
    The last system is cached (q27 and q27p share theirs)."""
    key = WORKLOADS[workload][:3]
    if key in _HOST_CACHE:
        return _HOST_CACHE[key]
    _HOST_CACHE.clear()
    _HOST_CACHE[key] = _host_system(workload)
    return _HOST_CACHE[key]


def _host_system(workload: str):
    from oracle import oracle as O
    from paper_1010_4639_b200.core import extract_lower
    from paper_1010_4639_b200.genprob import fem_mesh, rhs_for

    kind, dims, fmt, acc, _ = WORKLOADS[workload]
    if kind == "fem":
        F = fem_mesh()
        b, _ = rhs_for(F, seed=1)
        if fmt == "scsr":
            s = extract_lower(F)
            return "sym", s.row_start, s.col_idx, s.values, b
        return "csr", F.row_start, F.col_idx, F.values, b
    rs, ci, v = O.stencil(kind, dims, "full")
    xg = np.random.default_rng(1).standard_normal(len(rs) - 1)
    b = O.spmv_full(rs, ci, v, xg, workers=O.host_cores())
    if fmt == "scsr":
        rs, ci, v = O.stencil(kind, dims, "lower")
        return "sym", rs, ci, v, b
    return "csr", rs, ci, v, b


def cpu_sample(workload: str, steps: int, warmup: int, window: int):
    """Time the reference's compiled kernels (reference CG loop) on host cores."""
    from oracle import oracle as O

    kind, rs, ci, v, b = host_system(workload)
    n = len(rs) - 1
    cores = O.host_cores()
    acc = "atomic" if WORKLOADS[workload][3] == 0 else "privatized"
    use_ref = O.load_ref() is not None
    solve = O.cg_solve_ref if use_ref else O.cg_solve
    full_solve = kind != "sym" and n < 100_000  # small systems: whole solve
    mi = None if full_solve else window
    times, its = [], []
    for k in range(warmup + steps):
        t0 = time.perf_counter()
        r = solve(kind, rs, ci, v, b, max_iter=mi, recompute=full_solve, workers=cores,
                  accumulation=acc)
        dt = time.perf_counter() - t0
        if k >= warmup:
            times.append(dt)
            its.append(r.iterations)
    value = sum(its) / sum(times)
    sample = (f"{'full solve' if full_solve else f'{window}-iteration window (max_iter={window}, x0=0)'}"
              f" of the same {n}-row system, {steps} timed + {warmup} warm-up, "
              f"{'reference _ckernels (oracle/_ref) + reference CG loop' if use_ref else 'oracle C port'}")
    return {"value": value, "unit": "iterations/s", "cores": cores,
            "kind": "reference" if use_ref else "port", "sample": sample,
            "iterations_per_step": its[0], "s_per_step": float(np.median(times))}


def time_upload(workload: str):
    """The drop-in path's first-use cost: cg_solve(CsrMatrix(...)) uploads the
    host matrix once (spcg_matrix_create_host: raw int64 / fp64 arrays copied
    to the device, converted to int32 and validated there, row tiles built).
    Timed on the host arrays of the CPU baseline (same system)."""
    import ctypes

    import torch

    from paper_1010_4639_b200 import _native as N

    kind, rs, ci, v, _ = host_system(workload)
    fmt = N.FMT_SCSR if kind == "sym" else N.FMT_CSR
    n, nnz = len(rs) - 1, len(ci)
    lib = N.load()
    times = []
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h = ctypes.c_void_p()
        N.check(lib.spcg_matrix_create_host(fmt, n, nnz, rs.ctypes.data, ci.ctypes.data,
                                            v.ctypes.data, ctypes.byref(h)), "upload")
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        lib.spcg_matrix_destroy(h)
    host_bytes = 8 * (n + 1) + 16 * nnz
    return {"s": round(min(times), 3), "host_GB": round(host_bytes / 1e9, 2),
            "GBs": round(host_bytes / min(times) / 1e9, 1),
            "what": "spcg_matrix_create_host on the int64/fp64 host arrays (pageable), "
                    "device-side conversion + validation + tiles; best of 2"}


# ---- our arm ---------------------------------------------------------------------
def _opts(N, acc, max_iter=0, timing=1):
    return N.CgOptionsC(tol=1e-10, max_iter=max_iter, record_history=0,
                        recompute_final_residual=1, accumulation=acc, engine=0, timing=timing)


def measure_ours(workload: str, steps: int, warmup: int, peak: float, max_iter: int = 0,
                 clocks: bool = False, spmv: bool = False):
    """One workload through spcg_cg_solve (device-resident, `value`) and
    spcg_cg_solve_host (pinned host b in, x out every step: `e2e`).  Returns
    the fields of a bench line (no metric/header keys)."""
    import torch

    from paper_1010_4639_b200 import _native as N

    lib = N.load()
    t0 = time.time()
    dm, bt, n, nnz, xg, acc = build_device_system(workload)
    setup_s = time.time() - t0
    st = torch.cuda.current_stream()
    x = torch.empty_like(bt)
    opts = _opts(N, acc, max_iter)

    def solve_dev():
        r = N.CgResultC()
        N.check(lib.spcg_cg_solve(dm.handle, bt.data_ptr(), None, x.data_ptr(), None, opts, r,
                                  st.cuda_stream), "spcg_cg_solve")
        return r

    for _ in range(warmup):
        solve_dev()
    torch.cuda.synchronize()
    # working sets below 256 MB would stay in the 126 MB L2 between steps:
    # flush L2 (512 MB write) before every step, outside its timed window
    small = solve_bytes(n, nnz, 1) < 256e6
    flush = torch.empty(64 << 20, dtype=torch.float64, device="cuda") if small else None
    results = []
    clk = ClockSampler(torch.cuda.current_device()) if clocks else None
    if clk:
        clk.__enter__()
    torch.cuda.synchronize()
    if small:
        # per step: flush, then the solve; its time is the library's CUDA
        # event pair on the solve stream around the launch (device_ms),
        # which host-side stalls between steps cannot inflate
        for i in range(steps):
            flush.fill_(float(i))
            results.append(solve_dev())
            torch.cuda.synchronize()
        ms = float(sum(r.device_ms for r in results))
    else:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(steps):
            results.append(solve_dev())
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    if clk:
        clk.__exit__(None, None, None)
    iters = sum(r.iterations for r in results)
    solve_ms = float(np.mean([r.device_ms for r in results]))
    it_per = results[-1].iterations
    alg_solve = solve_bytes(n, nnz, it_per)
    achieved_solve = alg_solve / (solve_ms / 1e3) / 1e9
    # dominant kernel: the SpMV pass (q = A p, p.q) of the per-pass engine,
    # timed by CUDA events on the solve stream around every launch
    sp_launch = sum(r.spmv_launches for r in results)
    sp_kms = sum(r.spmv_ms for r in results)
    if sp_launch > 0:
        kern = "dist_spmv_pq (SpMV pass of the per-pass engine: q = A p, partial p.q)"
        kern_ms = sp_kms / sp_launch
        alg = spmv_bytes(n, nnz)
        model = "SpMV pass 12*nnz + 4*(n+1) + 16*n (SURVEY 8d)"
    else:  # resident systems: the whole solve is one persistent kernel
        kern = ("clus_pcg_kernel / clus_cg_kernel (cluster-resident CG solve, one launch) or "
                "cg1_kernel (grid-resident, unbanded systems)")
        kern_ms = solve_ms
        alg = alg_solve
        model = "per iteration 12*nnz + 4*(n+1) + 88*n (SURVEY 8d) + prologue/epilogue"
    achieved = alg / (kern_ms / 1e3) / 1e9

    # e2e through the C-ABI host entry point: pinned b in, x out, every step
    b_host = torch.empty(n, dtype=torch.float64, pin_memory=True)
    b_host.copy_(bt.cpu())
    x_host = torch.empty(n, dtype=torch.float64, pin_memory=True)
    bh, xh = b_host.numpy(), x_host.numpy()
    opts_e = _opts(N, acc, max_iter, timing=0)

    def solve_host():
        r = N.CgResultC()
        N.check(lib.spcg_cg_solve_host(dm.handle, bh.ctypes.data, None, xh.ctypes.data, None,
                                       opts_e, r, st.cuda_stream), "spcg_cg_solve_host")
        return r

    solve_host()
    torch.cuda.synchronize()
    e2e_ms, e2e_its = 0.0, 0
    for i in range(steps):
        if small:
            flush.fill_(float(i))
        torch.cuda.synchronize()
        e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2.record(st)
        e2e_its += solve_host().iterations
        e3.record(st)
        torch.cuda.synchronize()
        e2e_ms += e2.elapsed_time(e3)
    x_check = xh.copy()

    out = {
        "value": round(iters / (ms / 1e3), 3), "unit": "iterations/s",
        "ms_per_step": ms / steps, "steps": steps, "warmup": warmup,
        "n": n, "nnz_stored": nnz, "iterations_per_solve": it_per,
        "l2": ("L2 flushed (512 MB write) before every timed step (step time = CUDA events "
               "around the solve launch); working set %.1f MB" % (solve_bytes(n, nnz, 1) / 1e6))
        if small else ("inputs (matrix %.1f GB) >> 126 MB L2, no flush needed" % (12 * nnz / 1e9)),
        "engine": "per-pass" if sp_launch > 0 else "resident",
        "e2e": {"value": round(e2e_its / (e2e_ms / 1e3), 3), "unit": "iterations/s",
                "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n + 40,
                "path": "spcg_cg_solve_host (C-ABI, pinned host b -> x), matrix handle resident"},
        "gpu_launches": int(sum(r.kernel_launches for r in results)),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": None,
                     "kernel": kern, "algorithmic_bytes_per_launch": alg, "kernel_ms": kern_ms,
                     "launches_timed": int(sp_launch) if sp_launch else steps,
                     "bytes_model": model},
        "roofline_iteration": {"achieved": round(achieved_solve, 1),
                               "frac": round(achieved_solve / peak, 4), "unit": "GB/s",
                               "solve_ms": solve_ms, "us_per_iteration": 1e3 * solve_ms / it_per,
                               "algorithmic_bytes_per_solve": alg_solve,
                               "bytes_model": "per iteration 12*nnz + 4*(n+1) + 88*n "
                                              "(SURVEY 8d) + prologue/epilogue"},
        "final_relative_residual": results[-1].final_relative_residual,
        "converged": bool(results[-1].converged),
        "max_abs_err_vs_xgen": float(np.max(np.abs(x_check - xg)) / max(1.0, np.max(np.abs(xg)))),
        "setup_s": round(setup_s, 2),
    }
    if clk:
        out["clocks"] = clk.summary()
    if spmv:  # standalone SpMV kernel (the metric's "SpMV HBM GB/s")
        y = torch.empty_like(bt)
        for _ in range(3):
            lib.spcg_spmv(dm.handle, bt.data_ptr(), y.data_ptr(), acc, st.cuda_stream)
        reps = 20 if n > 1_000_000 else 200
        e4, e5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e4.record(st)
        for _ in range(reps):
            lib.spcg_spmv(dm.handle, bt.data_ptr(), y.data_ptr(), acc, st.cuda_stream)
        e5.record(st)
        torch.cuda.synchronize()
        sp_ms = e4.elapsed_time(e5) / reps
        sp_gbs = spmv_bytes(n, nnz) / (sp_ms / 1e3) / 1e9
        out["spmv"] = {"ms": sp_ms, "GBs": round(sp_gbs, 1), "frac": round(sp_gbs / peak, 4),
                       "bytes": spmv_bytes(n, nnz)}
    dm.close()
    del bt, x, b_host, x_host, flush
    torch.cuda.empty_cache()
    return out


METRIC = "fp64 CG iterations/sec (and SpMV HBM GB/s, % of roofline)"


def run_ours(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1 or args.engine == "sharded":
        return run_distributed(args)
    torch.cuda.set_device(0)
    torch.cuda.init()
    peak, peak_src = peaks()
    m = measure_ours(args.workload, args.steps, args.warmup, peak, args.max_iter, clocks=True,
                     spmv=True)
    tfile = ROOT / "profiles" / "r02" / "p3_spmv_traffic.json"
    if args.workload == "p3" and m["engine"] == "per-pass" and tfile.exists():
        # DRAM bytes of one dist_spmv_pq launch on this system (ncu --metrics
        # dram__bytes_read.sum,dram__bytes_write.sum; profiles/r01)
        m["roofline"]["traffic"] = int(json.loads(tfile.read_text())["dram_bytes_per_launch"])
        m["roofline"]["traffic_source"] = ("profiles/r02/p3_spmv_traffic.json (ncu dram__bytes "
                                           "of one launch)")
    m["roofline"]["peak_source"] = peak_src
    _, _, _, _, desc = WORKLOADS[args.workload]
    line = {
        "metric": METRIC,
        "value": m["value"],
        "unit": "iterations/s",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": m["ms_per_step"],
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (reference generators rebuilt in HBM; b = A x_gen, x_gen ~ N(0,1) seed 1)",
        "config": {"workload": desc, "n": m["n"], "nnz_stored": m["nnz_stored"], "tol": 1e-10,
                   "x0": "zeros", "iterations_per_solve": m["iterations_per_solve"],
                   "step": "one full cg_solve", "l2": m["l2"],
                   "parallelism": ("1 GPU; per-pass engine (tiled SpMV pass + 2 streaming passes, "
                                   "device-resident scalars, no host round trip per iteration)")
                                  if m["engine"] == "per-pass" else
                                  ("1 GPU; cluster-resident engine (one kernel per solve: "
                                   "matrix in shared memory, K clusters of 8 CTAs)")},
    }
    for k in ("e2e", "gpu_launches", "roofline", "roofline_iteration", "spmv", "clocks",
              "final_relative_residual", "converged", "max_abs_err_vs_xgen", "setup_s"):
        line[k] = m[k]
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_sample(args.workload, steps=3, warmup=1,
                                          window=WINDOW.get(args.workload, 20))
        line["upload"] = time_upload(args.workload)
    if not args.no_secondary and args.workload == "p3":
        line["secondary"] = secondary(peak, cpu=not args.no_cpu_baseline)
    print(json.dumps(line), flush=True)


def run_distributed(args):
    """N ranks (torchrun, one per GPU).  Stencil workloads are row-sharded
    (contiguous z-slabs; halo exchange + 2 all-reduces per iteration over
    NCCL): strong scaling of one global solve.  The 30880-row FEM configs do
    not shard (SURVEY §8e "replicas only"): each rank solves its own copy."""
    import torch
    import torch.distributed as dist

    from paper_1010_4639_b200 import _native as N
    from paper_1010_4639_b200 import distributed as D

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        gather, bcast = D.torch_collectives()
    else:
        gather, bcast = (lambda o: [o]), (lambda o: o)
    peak, peak_src = peaks()
    kind, dims, fmt, acc, desc = WORKLOADS[args.workload]
    st = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier(device_ids=[local])

    def max_over_ranks(v):
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    if kind == "fem":  # replicas
        dm, bt, n, nnz, xg, acc = build_device_system(args.workload)
        lib = N.load()
        x = torch.empty_like(bt)
        o = N.CgOptionsC(tol=1e-10, max_iter=args.max_iter, record_history=0,
                         recompute_final_residual=1, accumulation=acc, engine=0, timing=0)

        def step():
            r = N.CgResultC()
            N.check(lib.spcg_cg_solve(dm.handle, bt.data_ptr(), None, x.data_ptr(), None, o, r,
                                      st.cuda_stream), "solve")
            return r
        for _ in range(args.warmup):
            step()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        its = sum(step().iterations for _ in range(args.steps))
        e1.record(st)
        barrier()
        ms = max_over_ranks(e0.elapsed_time(e1))
        if rank == 0:
            print(json.dumps({
                "metric": "fp64 CG iterations/sec (and SpMV HBM GB/s, % of roofline)",
                "value": round(world * its / (ms / 1e3), 3), "unit": "iterations/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": desc, "parallelism": f"{world} independent replicas"},
                "gpu_launches": args.steps}), flush=True)
        if world > 1:
            dist.destroy_process_group()
        return

    comm = D.Comm(rank, world, bcast)
    t0 = time.time()
    sm = D.ShardedMatrix.from_stencil(kind, dims, fmt, rank, world, gather)
    n = sm.n_global
    xg = np.random.default_rng(1).standard_normal(n)
    x_ext = torch.from_numpy(np.concatenate([xg[sm.row0:sm.row1], xg[sm.halo]])).cuda()
    b_loc = sm.spmv_ext(x_ext)
    del x_ext
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    nnz_loc = sm.dm.nnz
    nnz_tot = int(sum(gather(nnz_loc))) if world > 1 else nnz_loc

    accum = "atomic" if acc == 0 else "privatized"  # SCSR shards: reverse halo vs stored L^T
    # transport of the per-iteration exchange: "nccl" (host-enqueued NCCL
    # all-reduces + send/recv) or "p2p" (device-initiated: mailbox all-reduce
    # and halo stores in CUDA-IPC-mapped peer memory, no host collective)
    plan = None
    if args.transport == "p2p":
        plan = D.P2PPlan(sm, rank, world)
        plan.connect(gather(plan.export()) if world > 1 else [plan.export()])

    def step():
        if plan is not None:
            x, res, _ = plan.solve(b_loc, max_iter=args.max_iter or None, timing=True,
                                   accumulation=accum)
        else:
            x, res, _ = D.dist_cg_solve(sm, comm, b_loc, max_iter=args.max_iter or None,
                                        timing=True, accumulation=accum)
        return x, res

    for _ in range(args.warmup):
        step()
    results = []
    with ClockSampler(local if world == 1 else -1) as clk:
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(args.steps):
            x, r = step()
            results.append((r.iterations, r.device_ms, r.kernel_launches, r.final_relative_residual,
                            r.spmv_ms, r.spmv_launches))
        e1.record(st)
        barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    clocks = clk.summary() if rank == 0 else None
    its = sum(r[0] for r in results)
    it_per = results[-1][0]
    solve_ms = max_over_ranks(float(np.mean([r[1] for r in results])))
    alg_solve = solve_bytes(n, nnz_tot, it_per)
    # dominant kernel: the SpMV pass, CUDA-event timed per launch, max over ranks
    kern_ms = max_over_ranks(sum(r[4] for r in results) / max(1, sum(r[5] for r in results)))
    alg = spmv_bytes(n, nnz_tot)
    achieved = alg / (kern_ms / 1e3) / 1e9
    err = float(np.max(np.abs(x.cpu().numpy() - xg[sm.row0:sm.row1])))
    err = max_over_ranks(err)
    # e2e: pinned host b in, x out, every step, through the sharded entry point
    bh = torch.empty(sm.nloc, dtype=torch.float64, pin_memory=True)
    bh.copy_(b_loc.cpu())
    xh = torch.empty(sm.nloc, dtype=torch.float64, pin_memory=True)
    barrier()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(st)
    e2e_its = 0
    for _ in range(args.steps):
        bd = bh.to("cuda", non_blocking=True)
        if plan is not None:
            xd, r, _ = plan.solve(bd, max_iter=args.max_iter or None, accumulation=accum)
        else:
            xd, r, _ = D.dist_cg_solve(sm, comm, bd, max_iter=args.max_iter or None,
                                       accumulation=accum)
        xh.copy_(xd, non_blocking=True)
        e2e_its += r.iterations
    e3.record(st)
    barrier()
    e2e_ms = max_over_ranks(e2.elapsed_time(e3))
    if rank == 0:
        print(json.dumps({
            "metric": "fp64 CG iterations/sec (and SpMV HBM GB/s, % of roofline)",
            "value": round(its / (ms / 1e3), 3), "unit": "iterations/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generator rebuilt in HBM per shard; b = A x_gen)",
            "config": {"workload": desc, "n": n, "nnz_stored": nnz_tot, "tol": 1e-10,
                       "iterations_per_solve": it_per, "step": "one full cg_solve",
                       "parallelism": (f"row-sharded over {world} GPU(s): z-slabs, NCCL halo "
                                       "send/recv + 2 all-reduces per iteration")
                                      if plan is None else
                                      (f"row-sharded over {world} GPU(s): z-slabs, device-initiated "
                                       "exchange (mailbox all-reduce + halo stores in peer memory)"),
                       "engine": "per-pass kernels + NCCL (spcg_dist_cg_solve)" if plan is None
                                 else "per-pass kernels, device transport (spcg_dist_plan_solve)",
                       "transport": args.transport},
            "e2e": {"value": round(e2e_its / (e2e_ms / 1e3), 3), "unit": "iterations/s",
                    "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                    "path": "spcg_dist_cg_solve per rank, pinned host b -> x"},
            "gpu_launches": int(sum(r[2] for r in results)),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1),
                         "peak": round(peak * world, 1), "unit": "GB/s",
                         "frac": round(achieved / (peak * world), 4), "traffic": None,
                         "peak_source": peak_src + f" x {world} GPUs",
                         "kernel": "dist_spmv_pq (SpMV pass, all ranks)",
                         "algorithmic_bytes_per_launch": alg, "kernel_ms": kern_ms},
            "roofline_iteration": {"achieved": round(alg_solve / (solve_ms / 1e3) / 1e9, 1),
                                   "frac": round(alg_solve / (solve_ms / 1e3) / 1e9 /
                                                 (peak * world), 4), "solve_ms": solve_ms},
            "clocks": clocks, "final_relative_residual": results[-1][3],
            "max_abs_err_vs_xgen": err, "setup_s": round(setup_s, 2)}), flush=True)
    if plan is not None:
        plan.close()
    comm.close()
    if world > 1:
        dist.destroy_process_group()


# reference CPU window (iterations) per workload: a bounded sample of ~5-15 s
WINDOW = {"p3": 20, "p2": 20, "q27": 10, "q27p": 10}


def secondary(peak, cpu=True):
    """Every other BASELINE config, each with its own roofline,
    e2e and reference-CPU baseline: P2 4096^2, Q27 256^3 in both
    accumulations, and the 30880-row FEM-shaped F (full CSR), S (symmetric
    CSR) and CSC (BASELINE configs[0..2,4])."""
    out = {}
    for w in ("p2", "q27", "q27p", "f", "s", "csc"):
        big = w in ("p2", "q27", "q27p")
        m = measure_ours(w, steps=3 if big else 10, warmup=1 if big else 3, peak=peak)
        d = {"workload": WORKLOADS[w][4]}
        for k in ("value", "unit", "ms_per_step", "steps", "warmup", "n", "nnz_stored",
                  "iterations_per_solve", "l2", "engine", "e2e", "roofline", "roofline_iteration",
                  "final_relative_residual", "converged"):
            d[k] = m[k]
        if cpu:
            d["cpu_baseline"] = cpu_sample(w, steps=3 if big else 5, warmup=1,
                                           window=WINDOW.get(w, 20))
        out[w] = d
    return out


def run_table1(args):
    """Table I of the paper on the 30880 FEM-shaped matrix: device op rows
    (CUDA events) next to the reference's compiled kernels on host cores."""
    import statistics

    from oracle import oracle as O
    from paper_1010_4639_b200.genprob import fem_mesh, rhs_for
    from paper_1010_4639_b200.table1 import run_table1 as gpu_rows

    F = fem_mesh()
    b, _ = rhs_for(F, seed=1)
    rep = gpu_rows(F, b, reps=15)
    # reference CPU rows (workers = host cores), median of 15 after a warm-up
    cores = O.host_cores()
    K = O.RefKernels(workers=cores, accumulation="atomic")
    Kp = O.RefKernels(workers=cores, accumulation="privatized")
    rng = np.random.default_rng(0)
    u, v = rng.standard_normal(F.n), rng.standard_normal(F.n)
    from paper_1010_4639_b200.core import extract_lower

    S = extract_lower(F)
    rows_s = np.repeat(np.arange(S.n, dtype=np.int64), np.diff(S.row_start))
    mk = S.col_idx < rows_s
    strict = (np.ascontiguousarray(rows_s[mk]), np.ascontiguousarray(S.col_idx[mk]),
              np.ascontiguousarray(S.values[mk]))
    rsF, ciF, vF = (np.ascontiguousarray(a) for a in (F.row_start, F.col_idx, F.values))
    rsS, ciS, vS = (np.ascontiguousarray(a) for a in (S.row_start, S.col_idx, S.values))
    cpu_ops = {
        "dotProd": lambda: K.dot(u, v),
        "AXPY": lambda: K.axpy(1.5, u, v),
        "SpMV": lambda: K.spmv_full(rsF, ciF, vF, u),
        "SpMV(sym)/atomic": lambda: K.spmv_sym(rsS, ciS, vS, strict, u),
        "SpMV(sym)/privatized": lambda: Kp.spmv_sym(rsS, ciS, vS, strict, u),
    }

    def med(fn, reps=15):
        fn()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            ts.append((time.perf_counter() - t0) * 1e3)
        return statistics.median(ts)

    for row in rep["ops"]:
        if row["op"] in cpu_ops:
            row["cpu_ms"] = med(cpu_ops[row["op"]])
            row["speedup_vs_cpu"] = row["cpu_ms"] / row["median_ms"]
    for row in rep["cg"]:
        if row["storage"] in ("full", "sym"):
            kind = "csr" if row["storage"] == "full" else "sym"
            arrs = (rsF, ciF, vF) if kind == "csr" else (rsS, ciS, vS)
            O.cg_solve_ref(kind, *arrs, b, workers=cores, accumulation="atomic")
            t0 = time.perf_counter()
            r = O.cg_solve_ref(kind, *arrs, b, workers=cores, accumulation="atomic")
            row["cpu_ms"] = (time.perf_counter() - t0) * 1e3
            row["cpu_iterations"] = r.iterations
            row["speedup_vs_cpu"] = row["cpu_ms"] / row["time_ms"]
    rep["meta"]["cpu_cores"] = cores
    rep["meta"]["cpu_kind"] = "reference _ckernels (oracle/_ref)"
    print(json.dumps(rep), flush=True)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    _, _, _, _, desc = WORKLOADS[args.workload]
    s = cpu_sample(args.workload, steps=args.steps, warmup=args.warmup,
                   window=WINDOW.get(args.workload, 20))
    line = {
        "impl": "reference",
        "metric": "fp64 CG iterations/sec (and SpMV HBM GB/s, % of roofline)",
        "value": round(s["value"], 4),
        "unit": "iterations/s",
        "n_gpus": int(os.environ.get("WORLD_SIZE", str(args.gpus))),
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": s["s_per_step"] * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (same system as the ours arm)",
        "config": {"workload": desc},
        "cpu_baseline": {k: s[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": round(s["value"], 4), "unit": "iterations/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` (N > 1) run directly, without torchrun: launch the
    N ranks ourselves (one process per GPU, torch.distributed.run on
    127.0.0.1) with the same arguments; rank 0 prints the line."""
    import socket

    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    env = dict(os.environ)
    # communicator bring-up is logged (NCCL_DEBUG=INFO lines go to stderr)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.run(cmd, env=env).returncode


def run_dry(args):
    """CPU dry run of the multi-rank plumbing (gloo; no GPU, no solve): the
    rank env, the P3 z-slab partition and halo plan built collectively, the
    max-over-ranks reduction and the rank-0 line.  `value` is null: this is
    a plumbing check, never a measurement."""
    import torch
    import torch.distributed as dist

    from paper_1010_4639_b200 import distributed as D

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    gather = (lambda o: [o]) if world == 1 else D.torch_collectives()[0]
    kind, dims, fmt, _, desc = WORKLOADS[args.workload]
    if kind == "fem":
        dims = (16, 10, 193)
    nx, ny, nz = (list(dims) + [1, 1])[:3]
    plane = nx * ny if nz > 1 else nx
    n = nx * ny * nz
    bounds = D.row_partition(n, world, align=plane)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    # halo of a 7-point slab: one plane on each interior side
    halo = np.concatenate([np.arange(max(0, r0 - plane), r0), np.arange(r1, min(n, r1 + plane))])
    plan = D.halo_plan(halo, bounds, rank, gather)
    t = torch.tensor([float(plan.send_off[-1])], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": None, "unit": "iterations/s", "n_gpus": world,
            "steps": 0, "warmup": 0, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "none (dry run)", "dry_run": True,
            "config": {"workload": desc, "n": n, "ranks_rows": [int(b) for b in bounds],
                       "max_halo_send": int(t.item()), "backend": "gloo (CPU)"}}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=tuple(WORKLOADS), default="p3")
    ap.add_argument("--max-iter", type=int, default=0, help="cap iterations (profiling only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--table1", action="store_true",
                    help="paper Table-I per-op rows (F matrix) on GPU vs the reference CPU path")
    ap.add_argument("--engine", choices=("auto", "sharded"), default="auto",
                    help="sharded: run the row-sharded engine even on one GPU")
    ap.add_argument("--transport", choices=("nccl", "p2p"), default="nccl",
                    help="sharded runs: host-enqueued NCCL or the device-initiated transport")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU check of the N-rank plumbing (gloo), no GPU and no measurement")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours" and args.max_iter == 0:
        print("note: contract requires warmup >= 3", file=sys.stderr)
    launched = "WORLD_SIZE" in os.environ
    if args.gpus > 1 and not launched and (args.impl == "ours" or args.dry_run):
        sys.exit(spawn_ranks(args))
    if args.dry_run:
        run_dry(args)
    elif args.table1:
        run_table1(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
