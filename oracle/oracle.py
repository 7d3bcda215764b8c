"""TEST INFRASTRUCTURE ONLY — the parity oracle for the B200 solve path.

Two CPU implementations of the reference's solve path (arxiv/paper_1010_4639,
package `spcg`), used by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs, never by the product:

  * `liboracle.so` (oracle.c): a C restatement of the kernels and of the
    cg_solve loop (solver.py:65-172), OpenMP-parallel like the reference's
    compiled backend ("port").
  * `_ref/_ckernels*.so`: the reference's OWN compiled kernels, built from
    /root/reference/pkg/src/spcg/kernels/_ckernels.pyx by oracle/Makefile,
    driven by `cg_solve_ref` below, a line-by-line restatement of
    solver.py:65-172 + the _compiled.py adapter ("reference").

Parity is pinned: tests/test_oracle.py checks both against golden vectors
produced by the reference package itself (tests/golden/, made by
scripts/make_golden.py).
"""

from __future__ import annotations

import ctypes
import glob
import importlib.util
import math
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"

_i64 = ctypes.c_int64
_vp = ctypes.c_void_p


class OrcMatrix(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("acc", ctypes.c_int), ("n", _i64),
                ("row_start", _vp), ("col_idx", _vp), ("values", _vp), ("m_strict", _i64),
                ("s_rows", _vp), ("s_cols", _vp), ("s_vals", _vp)]


class OrcResult(ctypes.Structure):
    _fields_ = [("iterations", _i64), ("converged", ctypes.c_int), ("status", ctypes.c_int),
                ("fail_iteration", _i64), ("final_rel", ctypes.c_double),
                ("b_norm", ctypes.c_double)]


_lib = None


def build():
    """Compile liboracle.so (and the reference kernels when /root/reference exists)."""
    targets = ["liboracle.so"]
    if Path("/root/reference/pkg/src/spcg/kernels/_ckernels.pyx").exists():
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", str(HERE), *targets], check=True)


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = ctypes.CDLL(str(LIB))
        L.orc_csr_gather.argtypes = [_i64, _vp, _vp, _vp, _vp, _vp, ctypes.c_int]
        L.orc_dot.argtypes = [_i64, _vp, _vp, ctypes.c_int, _i64]
        L.orc_dot.restype = ctypes.c_double
        L.orc_axpy.argtypes = [_i64, ctypes.c_double, _vp, _vp, _vp, ctypes.c_int]
        L.orc_scatter_seq.argtypes = [_i64, _vp, _vp, _vp, _vp, _vp]
        L.orc_scatter_privatized.argtypes = [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp,
                                             ctypes.c_int, _i64]
        L.orc_cg_solve.argtypes = [ctypes.POINTER(OrcMatrix), _vp, _vp, _vp, ctypes.c_double, _i64,
                                   ctypes.c_int, _vp, ctypes.c_int, _i64,
                                   ctypes.POINTER(OrcResult)]
        L.orc_cg_solve.restype = ctypes.c_int
        L.orc_stencil.argtypes = [ctypes.c_int, ctypes.c_int, _i64, _i64, _i64, _vp, _vp, _vp]
        L.orc_stencil.restype = _i64
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data if a is not None and a.size else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i(a):
    return np.ascontiguousarray(a, dtype=np.int64)


# ---- kernels (C restatement) ---------------------------------------------------
def spmv_full(row_start, col_idx, values, x, workers: int = 1) -> np.ndarray:
    """_ckernels.csr_gather (_ckernels.pyx:31-47)."""
    n = len(row_start) - 1
    rs, ci, v, x = _i(row_start), _i(col_idx), _f64(values), _f64(x)
    y = np.zeros(n)
    lib().orc_csr_gather(n, _p(rs), _p(ci), _p(v), _p(x), _p(y), workers)
    return y


def spmv_sym(row_start, col_idx, values, x, accumulation="privatized", workers=1, chunk=None):
    """_compiled.spmv_sym (_compiled.py:22-35): gather over L+D, then scatter
    of the strictly-lower entries (sequential for "atomic", reference
    privatized chunking otherwise)."""
    n = len(row_start) - 1
    rs, ci, v, x = _i(row_start), _i(col_idx), _f64(values), _f64(x)
    y = spmv_full(rs, ci, v, x, workers)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rs))
    keep = ci < rows
    r, c, vv = _i(rows[keep]), _i(ci[keep]), _f64(v[keep])
    m = r.shape[0]
    if accumulation == "atomic":
        lib().orc_scatter_seq(m, _p(r), _p(c), _p(vv), _p(x), _p(y))
    else:
        ch = chunk if chunk else max(1, math.ceil(m / (8 * workers)))
        priv = np.zeros(workers * max(n, 1))
        lib().orc_scatter_privatized(m, n, _p(r), _p(c), _p(vv), _p(x), _p(y), _p(priv), workers,
                                     ch)
    return y


def spmv_csc(col_start, row_idx, values, x) -> np.ndarray:
    """CSC column scatter y[row_idx[k]] += val[k] * x[col(k)] — the reference's
    scatter_atomic (_ckernels.pyx:50-62) applied to CSC arrays."""
    n = len(col_start) - 1
    cs = _i(col_start)
    cols = _i(np.repeat(np.arange(n, dtype=np.int64), np.diff(cs)))
    y = np.zeros(n)
    ri, v, x = _i(row_idx), _f64(values), _f64(x)
    lib().orc_scatter_seq(v.shape[0], _p(cols), _p(ri), _p(v), _p(x), _p(y))
    return y


def dot(u, v, workers: int = 1, chunk: int | None = None) -> float:
    """dot_partials + pairwise_merge (_ckernels.pyx:94-108, config.py:43-56)."""
    u, v = _f64(u), _f64(v)
    return float(lib().orc_dot(u.shape[0], _p(u), _p(v), workers, chunk or 0))


def axpy(alpha, u, v, workers: int = 1) -> np.ndarray:
    """v + alpha*u (_ckernels.pyx:111-117, alpha == 0 copies v)."""
    u, v = _f64(u), _f64(v)
    out = np.empty_like(v)
    lib().orc_axpy(u.shape[0], float(alpha), _p(u), _p(v), _p(out), workers)
    return out


class Result(dict):
    __getattr__ = dict.__getitem__


def cg_solve(kind: str, row_start, col_idx, values, b, x0=None, tol=1e-10, max_iter=None,
             recompute=True, record_history=False, workers=1, chunk=None,
             accumulation="privatized") -> Result:
    """solver.py:65-172 restated in C.  kind: 'csr' (full) or 'sym' (L+D)."""
    n = len(row_start) - 1
    keep = []
    rs, ci, v = _i(row_start), _i(col_idx), _f64(values)
    keep += [rs, ci, v]
    M = OrcMatrix(kind=0 if kind == "csr" else 1, acc=0 if accumulation == "atomic" else 1, n=n,
                  row_start=_p(rs), col_idx=_p(ci), values=_p(v))
    if kind == "sym":
        rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rs))
        mk = ci < rows
        sr, sc, sv = _i(rows[mk]), _i(ci[mk]), _f64(v[mk])
        keep += [sr, sc, sv]
        M.m_strict, M.s_rows, M.s_cols, M.s_vals = sr.shape[0], _p(sr), _p(sc), _p(sv)
    b = _f64(b)
    x0a = _f64(x0) if x0 is not None else None
    x = np.zeros(n)
    mi = max_iter if max_iter else max(1, n)
    hist = np.zeros(mi) if record_history else None
    res = OrcResult()
    lib().orc_cg_solve(ctypes.byref(M), _p(b), _p(x0a), _p(x), float(tol), int(mi), int(recompute),
                       _p(hist), int(workers), int(chunk or 0), ctypes.byref(res))
    return Result(x=x, iterations=int(res.iterations), converged=bool(res.converged),
                  status=int(res.status), fail_iteration=int(res.fail_iteration),
                  final_relative_residual=float(res.final_rel), b_norm=float(res.b_norm),
                  residual_history=list(hist[: res.iterations]) if hist is not None else None)


def stencil(kind: str, dims, part: str = "full"):
    """(row_start, col_idx, values) int64/f64 of poisson2d/poisson3d/stencil27."""
    k = {"poisson2d": 0, "poisson3d": 1, "stencil27": 2}[kind]
    d = list(dims) + [1] * (3 - len(dims))
    pt = 0 if part == "full" else 1
    n = d[0] * d[1] * d[2]
    nnz = lib().orc_stencil(k, pt, d[0], d[1], d[2], None, None, None)
    rs = np.empty(n + 1, dtype=np.int64)
    ci = np.empty(nnz, dtype=np.int64)
    v = np.empty(nnz, dtype=np.float64)
    lib().orc_stencil(k, pt, d[0], d[1], d[2], _p(rs), _p(ci), _p(v))
    return rs, ci, v


# ---- the reference's own compiled kernels ------------------------------------------
def load_ref():
    """Import oracle/_ref/_ckernels*.so (the reference's Cython/OpenMP kernels)."""
    cands = glob.glob(str(HERE / "_ref" / "_ckernels*.so"))
    if not cands:
        return None
    spec = importlib.util.spec_from_file_location("_ckernels", cands[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _pairwise(arr):
    arr = np.asarray(arr)
    if arr.size == 0:
        return 0.0
    while arr.size > 1:
        h = arr.size // 2
        head = arr[0:2 * h:2] + arr[1:2 * h:2]
        arr = np.concatenate([head, arr[2 * h:]]) if arr.size % 2 else head
    return float(arr[0])


class RefKernels:
    """_compiled.py:13-57 restated around the reference's own _ckernels."""

    def __init__(self, workers: int = 1, chunk: int | None = None, accumulation="privatized"):
        self.ck = load_ref()
        if self.ck is None:
            raise RuntimeError("oracle/_ref is not built (needs /root/reference at build time)")
        self.w, self.chunk, self.acc = workers, chunk, accumulation

    def _chunk(self, items):
        return self.chunk or max(1, math.ceil(items / (8 * self.w)))

    def spmv_full(self, rs, ci, v, x):
        y = np.zeros(len(rs) - 1)
        self.ck.csr_gather(rs, ci, v, x, y, self.w, self._chunk(len(rs) - 1))
        return y

    def spmv_sym(self, rs, ci, v, strict, x):
        n = len(rs) - 1
        y = np.zeros(n)
        self.ck.csr_gather(rs, ci, v, x, y, self.w, self._chunk(n))
        rows, cols, vals = strict
        ch = self._chunk(rows.shape[0])
        if self.acc == "atomic":
            self.ck.scatter_atomic(rows, cols, vals, x, y, self.w, ch)
        else:
            priv = np.zeros((self.w, n))
            self.ck.scatter_privatized(rows, cols, vals, x, y, priv, self.w, ch)
        return y

    def dot(self, u, v):
        m = u.shape[0]
        if m == 0:
            return 0.0
        ch = self._chunk(m)
        part = np.empty(-(-m // ch))
        self.ck.dot_partials(u, v, part, self.w, ch)
        return _pairwise(part)

    def axpy(self, alpha, u, v):
        if alpha == 0.0:
            return v.copy()
        out = np.empty_like(v)
        self.ck.axpy_kernel(float(alpha), u, v, out, self.w, self._chunk(u.shape[0]))
        return out


_STRICT: dict = {}


def _strict_of(rs, ci, v):
    """SymHalfMatrix.strict_lower (core.py:145-156): a cached property of the
    reference's matrix object, so it is built once per matrix, not per solve."""
    key = (rs.ctypes.data, ci.ctypes.data, v.ctypes.data, rs.shape[0], ci.shape[0])
    if key not in _STRICT:
        n = len(rs) - 1
        rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rs))
        mk = ci < rows
        _STRICT.clear()
        _STRICT[key] = (np.ascontiguousarray(rows[mk]), np.ascontiguousarray(ci[mk]),
                        np.ascontiguousarray(v[mk]))
    return _STRICT[key]


def cg_solve_ref(kind, row_start, col_idx, values, b, x0=None, tol=1e-10, max_iter=None,
                 recompute=True, record_history=False, workers=1, chunk=None,
                 accumulation="privatized") -> Result:
    """solver.py:65-172 over the reference's compiled kernels (same op order)."""
    K = RefKernels(workers, chunk, accumulation)
    rs, ci, v = _i(row_start), _i(col_idx), _f64(values)
    n = len(rs) - 1
    if kind == "sym":
        strict = _strict_of(rs, ci, v)
        spmv = lambda x: K.spmv_sym(rs, ci, v, strict, x)  # noqa: E731
    else:
        spmv = lambda x: K.spmv_full(rs, ci, v, x)  # noqa: E731
    b = _f64(b)
    mi = max_iter if max_iter else max(1, n)
    hist = [] if record_history else None
    b_norm = math.sqrt(K.dot(b, b))
    if b_norm == 0.0:
        return Result(x=np.zeros(n), iterations=0, converged=True, status=0, fail_iteration=0,
                      final_relative_residual=0.0, b_norm=0.0, residual_history=hist)
    x = _f64(x0).copy() if x0 is not None else np.zeros(n)
    r = K.axpy(-1.0, spmv(x), b)
    p = r.copy()
    rr = K.dot(r, r)
    rel = math.sqrt(rr) / b_norm
    conv, its, status, fail = False, 0, 0, 0
    if math.sqrt(rr) <= tol * b_norm:
        conv, mi = True, 0
    for k in range(1, mi + 1):
        q = spmv(p)
        pq = K.dot(p, q)
        if pq <= 0.0:
            status, fail = 3, k
            break
        alpha = rr / pq
        if not math.isfinite(alpha):
            status, fail = 4, k
            break
        x = K.axpy(alpha, p, x)
        r = K.axpy(-alpha, q, r)
        rr_new = K.dot(r, r)
        rel = math.sqrt(rr_new) / b_norm
        if not math.isfinite(rel):
            status, fail = 5, k
            break
        if hist is not None:
            hist.append(rel)
        its = k
        if math.sqrt(rr_new) <= tol * b_norm:
            conv, rr = True, rr_new
            break
        beta = rr_new / rr
        if not math.isfinite(beta):
            status, fail = 6, k
            break
        p = K.axpy(beta, p, r)
        rr = rr_new
    if status == 0 and recompute:
        tr = K.axpy(-1.0, spmv(x), b)
        rel = math.sqrt(K.dot(tr, tr)) / b_norm
    return Result(x=x, iterations=its, converged=conv, status=status, fail_iteration=fail,
                  final_relative_residual=rel, b_norm=b_norm, residual_history=hist)


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
