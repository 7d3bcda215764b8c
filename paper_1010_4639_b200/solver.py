"""Conjugate gradient on the B200: the reference's `cg_solve` API
(solver.py:65-172) over the device engines of the C library (one
persistent cluster-resident kernel for systems that fit on chip, per-pass
streaming kernels for the rest).

Semantics kept from the reference, in order (solver.py:86-162):
  * b and x0 are cast to the matrix dtype; shape errors raise ValueError
    ("dimension mismatch ...");  x0=None means zeros;
  * max_iter defaults to max(1, n);
  * ||b|| = 0 returns x = 0 (even for x0 != 0), 0 iterations, converged;
  * an x0 already within tolerance returns 0 iterations, converged;
  * per iteration: q = A p, p.q <= 0 -> NotPositiveDefiniteError, non-finite
    alpha / residual / beta -> NumericalBreakdownError naming iteration k,
    the history holds the recursive ||r||/||b||, convergence is
    ||r|| <= tol * ||b|| tested after the r-update;
  * hitting max_iter returns converged=False (no exception);
  * final_relative_residual is the true ||b - A x||/||b|| unless
    recompute_final_residual is False.
All of it runs on the device: no host round trip per iteration; the host
reads back a small result record, x and (optionally) the history.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .core import CscMatrix, CsrMatrix, SymHalfMatrix
from .kernels import KernelConfig, _acc_code


class CgBreakdownError(RuntimeError):
    """Base for failures that abort the CG iteration (solver.py:22-23)."""


class NotPositiveDefiniteError(CgBreakdownError):
    """p'Ap <= 0 with a nonzero residual (solver.py:26-27)."""


class NumericalBreakdownError(CgBreakdownError):
    """A non-finite alpha, beta or residual appeared (solver.py:30-31)."""


@dataclass(frozen=True)
class CgOptions:
    tol: float = 1e-10
    max_iter: int | None = None
    record_history: bool = False
    recompute_final_residual: bool = True

    def __post_init__(self):
        if not self.tol > 0:
            raise ValueError("tol must be > 0")
        if self.max_iter is not None and self.max_iter < 1:
            raise ValueError("max_iter must be >= 1")


@dataclass
class SolveReport:
    x: np.ndarray
    iterations: int
    converged: bool
    final_relative_residual: float
    residual_history: list[float] | None = None
    timings: dict[str, float] = field(default_factory=dict)
    # (new, not in the reference's record) which device engine produced x:
    # {"engine": 2|3|5|6|7, "fallback": bool, "cond_estimate": float}
    engine_info: dict = field(default_factory=dict, compare=False, repr=False)


def check_convergence(residual_norm: float, b_norm: float, opts: CgOptions) -> bool:
    """residual_norm <= tol*b_norm; b = 0 demands an exact zero (solver.py:58-62)."""
    if b_norm == 0.0:
        return residual_norm == 0.0
    return residual_norm <= opts.tol * b_norm


_BREAKDOWN = {
    N.ERR_NOT_SPD: lambda k: NotPositiveDefiniteError("matrix not positive definite"),
    N.ERR_NONFINITE_ALPHA: lambda k: NumericalBreakdownError(f"non-finite alpha at iteration {k}"),
    N.ERR_NONFINITE_RESIDUAL: lambda k: NumericalBreakdownError(
        f"non-finite residual at iteration {k}"),
    N.ERR_NONFINITE_BETA: lambda k: NumericalBreakdownError(f"non-finite beta at iteration {k}"),
}


def _is_torch_cuda(v) -> bool:
    mod = type(v).__module__
    return mod.startswith("torch") and getattr(v, "is_cuda", False)


def cg_solve(a, b, x0=None, opts: CgOptions | None = None, cfg: KernelConfig | None = None,
             engine: int = 0) -> SolveReport:
    """Solve A x = b for SPD A stored as CsrMatrix, SymHalfMatrix or CscMatrix.

    `b`/`x0` may be numpy arrays (x returned as numpy) or CUDA torch tensors
    (device-resident solve; x returned as a CUDA tensor).  `cfg.accumulation`
    selects the symmetric-half mode: "privatized" (default, deterministic:
    resident engines use the stored L^T rows on chip, the streaming engine a
    single pass over L+D with the transposed part summed exactly in 64-bit
    fixed point) or "atomic" (single pass over L+D with fp64 atomics).
    `engine` 0 = auto; `report.engine_info` names the engine that ran.
    """
    opts = opts or CgOptions()
    cfg = cfg or KernelConfig()
    if not isinstance(a, (CsrMatrix, SymHalfMatrix, CscMatrix)):
        raise TypeError(f"unsupported matrix type {type(a).__name__}")
    n = a.n
    t0 = time.perf_counter()
    device_io = _is_torch_cuda(b)
    if not device_io:
        b = np.ascontiguousarray(b, dtype=a.dtype)
        if b.shape != (n,):
            raise ValueError(f"dimension mismatch: b has shape {b.shape}, expected ({n},)")
        if x0 is not None:
            x0 = np.ascontiguousarray(x0, dtype=a.dtype)
            if x0.shape != (n,):
                raise ValueError(
                    f"dimension mismatch: x0 has shape {x0.shape}, expected ({n},)")
    else:
        if tuple(b.shape) != (n,):
            raise ValueError(f"dimension mismatch: b has shape {tuple(b.shape)}, expected ({n},)")
        if x0 is not None and tuple(x0.shape) != (n,):
            raise ValueError(
                f"dimension mismatch: x0 has shape {tuple(x0.shape)}, expected ({n},)")
    max_iter = opts.max_iter if opts.max_iter is not None else max(1, n)

    dev = a.device()
    lib = N.load()
    o = N.CgOptionsC(tol=float(opts.tol), max_iter=int(max_iter),
                     record_history=int(bool(opts.record_history)),
                     recompute_final_residual=int(bool(opts.recompute_final_residual)),
                     accumulation=_acc_code(cfg), engine=int(engine),
                     row_sums=1 if cfg.row_sums == "sequential" else 0, timing=2)
    res = N.CgResultC()
    if device_io:
        import torch

        bt = b.to(torch.float64).contiguous()
        x0t = x0.to(device=bt.device, dtype=torch.float64).contiguous() if x0 is not None else None
        xt = torch.empty(n, dtype=torch.float64, device=bt.device)
        ht = torch.empty(max(1, max_iter) if opts.record_history else 1, dtype=torch.float64,
                         device=bt.device)
        rc = lib.spcg_cg_solve(dev.handle, bt.data_ptr(), x0t.data_ptr() if x0t is not None else None,
                               xt.data_ptr(), ht.data_ptr() if opts.record_history else None,
                               o, res, torch.cuda.current_stream(bt.device).cuda_stream)
        hist_arr = ht[: res.iterations].cpu().numpy() if opts.record_history else None
        x_out = xt
    else:
        bb = np.ascontiguousarray(b, dtype=np.float64)
        xx0 = np.ascontiguousarray(x0, dtype=np.float64) if x0 is not None else None
        x = np.empty(n, dtype=np.float64)
        hist = np.empty(max(1, max_iter), dtype=np.float64) if opts.record_history else None
        rc = lib.spcg_cg_solve_host(
            dev.handle, bb.ctypes.data if n else None,
            xx0.ctypes.data if xx0 is not None and n else None,
            x.ctypes.data if n else None,
            hist.ctypes.data if hist is not None else None, o, res, N.current_stream())
        hist_arr = hist[: res.iterations] if hist is not None else None
        x_out = x if a.dtype == np.float64 else x.astype(a.dtype)
    if rc in _BREAKDOWN:
        raise _BREAKDOWN[rc](int(res.fail_iteration))
    N.check(rc, "spcg_cg_solve")
    total = time.perf_counter() - t0
    # Device time per phase (solver.py:98-105 keys).  The kernels fuse the
    # dot partials into the SpMV and update passes, so: "spmv" = the SpMV
    # passes, "axpy" = the vector-update passes, "dot" = the rest of the
    # device time (reductions' completion, scalar steps, collectives).
    ph = [float(v) / 1e3 for v in res.phase_ms]
    if sum(ph) > 0.0:
        timings = {"spmv": ph[0], "dot": ph[1], "axpy": ph[2], "total": total}
    else:  # an engine that did not split its one kernel: all under "spmv"
        timings = {"spmv": res.device_ms / 1e3, "dot": 0.0, "axpy": 0.0, "total": total}
    return SolveReport(
        x=x_out,
        iterations=int(res.iterations),
        converged=bool(res.converged),
        final_relative_residual=float(res.final_relative_residual),
        residual_history=[float(v) for v in hist_arr] if hist_arr is not None else None,
        timings=timings,
        engine_info={"engine": int(res.engine_used), "fallback": bool(res.fallbacks),
                     "cond_estimate": float(res.cond_estimate)},
    )
