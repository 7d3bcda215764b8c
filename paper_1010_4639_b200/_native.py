"""ctypes binding of the C-ABI in include/spcg_b200.h.

The shared library is built in-tree (``paper_1010_4639_b200/_lib/libspcg_b200.so``,
see ``build.py``).  There is no CPU fallback: if the library is missing, or the
process has no sm_100 device, every compute entry point raises
``NativeUnavailableError``.  ctypes releases the GIL for the duration of each
call, matching the reference's ``nogil`` OpenMP kernels (_ckernels.pyx:42).
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

LIB_PATH = Path(os.environ.get("SPCG_LIB") or Path(__file__).resolve().parent / "_lib" / "libspcg_b200.so")
HEADER_PATH = Path(__file__).resolve().parent.parent / "include" / "spcg_b200.h"

# spcg_status (spcg_b200.h)
OK = 0
ERR_ARG = 1
ERR_CUDA = 2
ERR_NOT_SPD = 3
ERR_NONFINITE_ALPHA = 4
ERR_NONFINITE_RESIDUAL = 5
ERR_NONFINITE_BETA = 6
ERR_UNSUPPORTED = 7

FMT_CSR, FMT_SCSR, FMT_CSC = 0, 1, 2
ACC_ATOMIC, ACC_PRIVATIZED = 0, 1
GEN_POISSON2D, GEN_POISSON3D, GEN_STENCIL27 = 0, 1, 2


class NativeUnavailableError(RuntimeError):
    """The CUDA library is not built or no usable B200 device is present."""


class CgOptionsC(ctypes.Structure):
    _fields_ = [
        ("tol", ctypes.c_double),
        ("max_iter", ctypes.c_int64),
        ("record_history", ctypes.c_int32),
        ("recompute_final_residual", ctypes.c_int32),
        ("accumulation", ctypes.c_int32),
        ("engine", ctypes.c_int32),
        ("timing", ctypes.c_int32),
        ("row_sums", ctypes.c_int32),
    ]


class CgResultC(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int64),
        ("converged", ctypes.c_int32),
        ("status", ctypes.c_int32),
        ("fail_iteration", ctypes.c_int64),
        ("final_relative_residual", ctypes.c_double),
        ("b_norm", ctypes.c_double),
        ("device_ms", ctypes.c_double),
        ("kernel_launches", ctypes.c_int64),
        ("spmv_ms", ctypes.c_double),
        ("spmv_launches", ctypes.c_int64),
        ("engine_used", ctypes.c_int32),
        ("fallbacks", ctypes.c_int32),
        ("cond_estimate", ctypes.c_double),
        ("phase_ms", ctypes.c_double * 3),
    ]


_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int
_d = ctypes.c_double

# name -> (restype, argtypes); every symbol declared in include/spcg_b200.h
SIGNATURES = {
    "spcg_matrix_create_host": (_i32, [_i32, _i64, _i64, _vp, _vp, _vp, ctypes.POINTER(_vp)]),
    "spcg_matrix_create_host_u32": (_i32, [_i32, _i64, _i64, _vp, _vp, _vp, ctypes.POINTER(_vp)]),
    "spcg_matrix_generate": (_i32, [_i32, _i32, _i64, _i64, _i64, ctypes.POINTER(_vp)]),
    "spcg_matrix_assemble_pairs": (_i32, [_i32, _i64, _i64, _vp, _vp, _vp, _d, ctypes.POINTER(_vp)]),
    "spcg_matrix_create_device_u32": (_i32, [_i32, _i64, _i64, _vp, _vp, _vp, ctypes.POINTER(_vp)]),
    "spcg_matrix_destroy": (_i32, [_vp]),
    "spcg_matrix_info": (
        _i32,
        [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(_i32),
         ctypes.POINTER(_i64), ctypes.POINTER(_i64)],
    ),
    "spcg_matrix_download": (_i32, [_vp, _vp, _vp, _vp]),
    "spcg_spmv": (_i32, [_vp, _vp, _vp, _i32, _vp]),
    "spcg_dot": (_i32, [_i64, _vp, _vp, _vp, _vp]),
    "spcg_axpy": (_i32, [_i64, _d, _vp, _vp, _vp, _vp]),
    "spcg_cg_solve": (
        _i32,
        [_vp, _vp, _vp, _vp, _vp, ctypes.POINTER(CgOptionsC), ctypes.POINTER(CgResultC), _vp],
    ),
    "spcg_cg_solve_host": (
        _i32,
        [_vp, _vp, _vp, _vp, _vp, ctypes.POINTER(CgOptionsC), ctypes.POINTER(CgResultC), _vp],
    ),
    "spcg_comm_unique_id": (_i32, [_vp]),
    "spcg_comm_create": (_i32, [_i32, _i32, _vp, ctypes.POINTER(_vp)]),
    "spcg_comm_destroy": (_i32, [_vp]),
    "spcg_comm_create_host": (_i32, [_i32, _i32, _vp, _vp, _vp, ctypes.POINTER(_vp)]),
    "spcg_matrix_create_rows": (
        _i32,
        [_i32, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _i64, _vp, _vp, _vp, ctypes.POINTER(_vp)],
    ),
    "spcg_matrix_generate_rows": (_i32, [_i32, _i32, _i64, _i64, _i64, _i64, _i64,
                                         ctypes.POINTER(_vp)]),
    "spcg_matrix_localize": (_i32, [_vp, ctypes.POINTER(_i64)]),
    "spcg_matrix_halo": (_i32, [_vp, _vp]),
    "spcg_dist_cg_solve": (
        _i32,
        [_vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.POINTER(CgOptionsC),
         ctypes.POINTER(CgResultC), _vp],
    ),
    "spcg_dist_plan_create": (_i32, [_vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp, ctypes.POINTER(_vp)]),
    "spcg_dist_plan_destroy": (_i32, [_vp]),
    "spcg_dist_plan_export": (_i32, [_vp, _vp]),
    "spcg_dist_plan_connect": (_i32, [_vp, _vp]),
    "spcg_dist_plan_solve": (
        _i32, [_vp, _vp, _vp, _vp, _vp, ctypes.POINTER(CgOptionsC), ctypes.POINTER(CgResultC), _vp]),
    "spcg_dist_group_solve": (
        _i32, [_i32, _vp, _vp, _vp, _vp, _vp, ctypes.POINTER(CgOptionsC), _vp, _vp]),
    "spcg_last_error": (ctypes.c_char_p, []),
    "spcg_abi_version": (_i32, []),
    "spcg_cg_cond_estimate": (_i32, [_vp, _i64, ctypes.POINTER(_d)]),
    "spcg_device_info": (
        _i32,
        [ctypes.POINTER(_i32), ctypes.POINTER(_i32), ctypes.POINTER(_i32), ctypes.POINTER(_i32)],
    ),
}

_lock = threading.Lock()
_lib = None


def load(path: os.PathLike | str | None = None) -> ctypes.CDLL:
    """Load (once) and return the library with typed signatures."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise NativeUnavailableError(
                f"{p} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = ctypes.CDLL(str(p))
        lenient = os.environ.get("SPCG_LIB_LENIENT") == "1"  # dev: older library builds
        for name, (res, args) in SIGNATURES.items():
            if lenient and not hasattr(lib, name):
                continue
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def last_error() -> str:
    msg = load().spcg_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str) -> None:
    """Raise for a non-OK status that is not a CG breakdown."""
    if rc == OK:
        return
    msg = last_error()
    if rc == ERR_ARG:
        raise ValueError(f"{what}: {msg}")
    if rc == ERR_CUDA:
        raise NativeUnavailableError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: status {rc}: {msg}")


def device_info() -> dict:
    lib = load()
    sm, grid, ma, mi = _i32(), _i32(), _i32(), _i32()
    check(lib.spcg_device_info(ctypes.byref(sm), ctypes.byref(grid), ctypes.byref(ma),
                               ctypes.byref(mi)), "spcg_device_info")
    return {"sm_count": sm.value, "coop_grid": grid.value, "cc": (ma.value, mi.value)}


def cg_cond_estimate(alpha, beta) -> float:
    """Ritz estimate of cond(A) from CG's step coefficients (alpha_j, beta_j),
    beta_j the coefficient that formed p_j (beta_0 ignored); the engine-6
    guard's estimate, computed on the host (spcg_cg_cond_estimate)."""
    import numpy as np

    a = np.asarray(alpha, dtype=np.float64)
    b = np.asarray(beta, dtype=np.float64)
    if a.shape != b.shape or a.ndim != 1:
        raise ValueError("alpha and beta must be 1-D arrays of the same length")
    ab = np.ascontiguousarray(np.stack([a, b], axis=1).reshape(-1))
    out = ctypes.c_double()
    check(load().spcg_cg_cond_estimate(ab.ctypes.data if ab.size else None, a.size,
                                       ctypes.byref(out)), "spcg_cg_cond_estimate")
    return out.value


def current_stream() -> int:
    """torch's current CUDA stream handle (0 if torch CUDA is not initialised)."""
    try:
        import torch

        if torch.cuda.is_available() and torch.cuda.is_initialized():
            return int(torch.cuda.current_stream().cuda_stream)
    except Exception:  # pragma: no cover - torch is plumbing only
        pass
    return 0


# Host-callback communicator (spcg_comm_create_host)
HOST_ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.POINTER(ctypes.c_double), ctypes.c_int64,
                                     ctypes.c_void_p)
HOST_SENDRECV_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                                    ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64),
                                    ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64),
                                    ctypes.c_void_p)
