"""The reference's kernel API (kernels/__init__.py:67-103) on the B200.

`spmv_full`, `spmv_sym`, `spmv_csc`, `dot`, `axpy`, `norm2` take numpy arrays
(results come back as numpy) or CUDA torch tensors (results stay on the
device).  torch is used only to hold device buffers.  There is exactly one
backend, "cuda"; `set_backend` accepts "auto"/"cuda" and the reference's
backend names "compiled"/"python" (aliases of the one backend, also through
SPCG_BACKEND) so code written against the reference's registry keeps working,
and anything else raises ValueError like the reference does for unknown names
(kernels/__init__.py:35-44).

Numerical contracts:
  spmv_full   sequential row sums, IEEE mul-then-add: bitwise equal to
              _ckernels.csr_gather for rows of <= 4096 entries
  spmv_sym    privatized: (L+D)x then + L^T x per row (owner-computes, no
              atomics) = reference privatized at workers=1, bit for bit;
              atomic: single pass, fp64 red.add scatter (order unspecified)
  cg_solve    accumulation="privatized" (the default) is deterministic in
              every engine: the streaming engine makes ONE pass over L+D
              and accumulates the transposed part exactly in 64-bit fixed
              point (order-independent integer reds; no L^T streamed);
              row_sums="sequential" selects the stored-L^T rows instead
              (bitwise the reference's privatized row sums at workers=1)
  dot         fixed-order two-level reduction (deterministic, reassociated)
  axpy        v + alpha*u with IEEE mul-then-add; alpha == 0 copies v
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np

from . import _native as N

ACCUMULATION_MODES = ("atomic", "privatized")


@dataclass(frozen=True)
class KernelConfig:
    """Execution contract (config.py:13-40).  On the GPU `workers`/`chunk`
    have no meaning (the grid is sized to the SM count) but are validated;
    `accumulation` selects the symmetric scatter mode.  `row_sums` (new):
    "auto" lets the streaming CG passes sum long rows as per-lane partials +
    a fixed tree (deterministic, fp64-reassociated); "sequential" keeps every
    row sum in storage order (bitwise the reference's sequential sums)."""

    workers: int = 1
    chunk: int | None = None
    accumulation: str = "privatized"
    row_sums: str = "auto"

    def __post_init__(self):
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.chunk is not None and self.chunk < 1:
            raise ValueError("chunk must be >= 1")
        if self.accumulation not in ACCUMULATION_MODES:
            raise ValueError(f"accumulation must be one of {ACCUMULATION_MODES}")
        if self.row_sums not in ("auto", "sequential"):
            raise ValueError("row_sums must be 'auto' or 'sequential'")

    def resolve_chunk(self, work_items: int) -> int:
        if self.chunk is not None:
            return self.chunk
        return max(1, math.ceil(work_items / (8 * self.workers)))


_DEFAULT_CFG = KernelConfig()


def _acc_code(cfg: KernelConfig | None) -> int:
    cfg = cfg or _DEFAULT_CFG
    return N.ACC_ATOMIC if cfg.accumulation == "atomic" else N.ACC_PRIVATIZED


class _CudaBackend:
    """Backend module interface of the reference (_compiled.py:10-57: name,
    spmv_full, spmv_sym, dot, axpy); filled in below."""

    name = "cuda"


# The reference's backend registry (kernels/__init__.py:21-50).  There is ONE
# implementation (the device kernels, no CPU fallback); the reference's names
# "compiled" and "python" are aliases of it, so code that selects a backend
# by name -- set_backend("compiled"), SPCG_BACKEND=python -- keeps working.
BACKENDS = {"cuda": _CudaBackend, "compiled": _CudaBackend, "python": _CudaBackend}


def available_backends() -> tuple[str, ...]:
    """Distinct implementations (the aliases above resolve to "cuda")."""
    return ("cuda",)


def set_backend(name: str):
    """Select a backend by name and return it (kernels/__init__.py:35-41);
    "auto" and the reference's names resolve to the one device backend,
    unknown names raise ValueError like the reference."""
    global _active
    if name == "auto":
        name = "cuda"
    if name not in BACKENDS:
        raise ValueError(f"unknown backend {name!r}; available: {tuple(BACKENDS)}")
    _active = BACKENDS[name]
    return _active


def get_backend() -> str:
    return _active.name


# SPCG_BACKEND is honoured at import (kernels/__init__.py:50)
_active = set_backend(os.environ.get("SPCG_BACKEND", "auto"))


# ---- device buffer plumbing --------------------------------------------------
def _torch():
    import torch

    if not torch.cuda.is_available():
        raise N.NativeUnavailableError("no CUDA device: the B200 kernels have no CPU fallback")
    return torch


def _is_dev(v) -> bool:
    return type(v).__module__.startswith("torch") and getattr(v, "is_cuda", False)


def _to_dev(v, n: int | None = None):
    """(device tensor f64, was_device) for a numpy array / CUDA tensor."""
    torch = _torch()
    if _is_dev(v):
        t = v.to(torch.float64).contiguous()
    else:
        a = np.ascontiguousarray(v)
        if a.dtype not in (np.float32, np.float64):
            a = a.astype(np.float64)
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to("cuda")
    if t.ndim != 1 or (n is not None and t.shape[0] != n):
        raise ValueError(
            f"dimension mismatch: expected vector of length {n}, got shape {tuple(t.shape)}")
    return t


def _host_dtype(*vs):
    for v in vs:
        if not _is_dev(v):
            a = np.asarray(v)
            if a.dtype in (np.float32, np.float64):
                return a.dtype
    return np.dtype(np.float64)


def _back(t, like_dev: bool, dtype=np.float64):
    if like_dev:
        return t
    out = t.cpu().numpy()
    return out if out.dtype == dtype else out.astype(dtype)


def _check_vec(x, n):
    shape = tuple(x.shape) if _is_dev(x) else np.shape(x)
    if len(shape) != 1 or shape[0] != n:
        raise ValueError(f"dimension mismatch: expected vector of length {n}, got shape {shape}")


def _spmv(m, x, cfg):
    _check_vec(x, m.n)
    dev = m.device()
    torch = _torch()
    xt = _to_dev(x, m.n)
    yt = torch.empty(m.n, dtype=torch.float64, device=xt.device)
    rc = N.load().spcg_spmv(dev.handle, xt.data_ptr(), yt.data_ptr(), _acc_code(cfg),
                            torch.cuda.current_stream().cuda_stream)
    N.check(rc, "spcg_spmv")
    return _back(yt, _is_dev(x), m.dtype)


def spmv_full(m, x, cfg: KernelConfig | None = None):
    """y = M x over full CSR (or CSC) storage; bitwise independent of cfg."""
    from .core import CscMatrix, CsrMatrix

    if not isinstance(m, (CsrMatrix, CscMatrix)):
        raise TypeError(f"spmv_full needs CsrMatrix/CscMatrix, got {type(m).__name__}")
    return _spmv(m, x, cfg)


def spmv_sym(s, x, cfg: KernelConfig | None = None):
    """y = (L+D) x + L^T x per cfg.accumulation (kernels/__init__.py:73-82)."""
    from .core import SymHalfMatrix

    if not isinstance(s, SymHalfMatrix):
        raise TypeError(f"spmv_sym needs SymHalfMatrix, got {type(s).__name__}")
    return _spmv(s, x, cfg)


def spmv_csc(c, x, cfg: KernelConfig | None = None):
    """y = C x by column scatter over CSC storage (fp64 atomics)."""
    from .core import CscMatrix

    if not isinstance(c, CscMatrix):
        raise TypeError(f"spmv_csc needs CscMatrix, got {type(c).__name__}")
    return _spmv(c, x, cfg)


def dot(u, v, cfg: KernelConfig | None = None) -> float:
    """Inner product with a fixed-order device reduction (deterministic)."""
    torch = _torch()
    ut = _to_dev(u)
    vt = _to_dev(v, ut.shape[0])
    out = torch.empty(1, dtype=torch.float64, device=ut.device)
    rc = N.load().spcg_dot(int(ut.shape[0]), ut.data_ptr(), vt.data_ptr(), out.data_ptr(),
                           torch.cuda.current_stream().cuda_stream)
    N.check(rc, "spcg_dot")
    return float(out.item())


def axpy(alpha: float, u, v, cfg: KernelConfig | None = None):
    """v + alpha*u elementwise; bitwise independent of cfg."""
    torch = _torch()
    ut = _to_dev(u)
    vt = _to_dev(v, ut.shape[0])
    out = torch.empty_like(vt)
    rc = N.load().spcg_axpy(int(ut.shape[0]), float(alpha), ut.data_ptr(), vt.data_ptr(),
                            out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    N.check(rc, "spcg_axpy")
    return _back(out, _is_dev(v), _host_dtype(u, v))


def norm2(u, cfg: KernelConfig | None = None) -> float:
    """Euclidean norm through the deterministic dot."""
    return math.sqrt(dot(u, u, cfg))


def pairwise_merge(partials) -> float:
    """Fixed-order pairwise tree sum (config.py:43-56); host helper kept for API
    compatibility — the device reductions do their own fixed-order trees."""
    arr = np.asarray(partials, dtype=np.float64)
    if arr.size == 0:
        return 0.0
    while arr.size > 1:
        half = arr.size // 2
        head = arr[0:2 * half:2] + arr[1:2 * half:2]
        arr = np.concatenate([head, arr[2 * half:]]) if arr.size % 2 else head
    return float(arr[0])


for _n in ("spmv_full", "spmv_sym", "dot", "axpy"):
    setattr(_CudaBackend, _n, staticmethod(globals()[_n]))
del _n

__all__ = [
    "KernelConfig", "ACCUMULATION_MODES", "pairwise_merge", "spmv_full", "spmv_sym", "spmv_csc",
    "dot", "axpy", "norm2", "set_backend", "get_backend", "available_backends", "BACKENDS",
]
