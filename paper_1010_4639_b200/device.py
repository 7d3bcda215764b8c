"""Device-resident matrix handles (the C-ABI's spcg_matrix_t).

A `DeviceMatrix` owns the HBM copy of one matrix: int32 offsets/indices,
fp64 values, 16-byte-aligned and padded arrays, the row-tile table, and for
symmetric half storage the L^T arrays used by the deterministic
(privatized-equivalent) mode.  Upload happens once per immutable host matrix
(`CsrMatrix.device()` caches it); in-HBM generators build the reference's
Poisson / 27-point matrices without touching host memory.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


def current_device() -> int:
    """Index of the current CUDA device (-1 without torch CUDA)."""
    try:
        import torch

        if torch.cuda.is_available():
            return int(torch.cuda.current_device())
    except Exception:  # pragma: no cover - torch is plumbing only
        pass
    return -1


class DeviceMatrix:
    FORMATS = {"csr": N.FMT_CSR, "scsr": N.FMT_SCSR, "csc": N.FMT_CSC}

    def __init__(self, handle: int, fmt: int, n: int, nnz: int, host_dtype=np.float64):
        self._h = ctypes.c_void_p(handle)
        self.fmt = fmt
        self.n = n
        self.nnz = nnz
        self.host_dtype = np.dtype(host_dtype)
        self._lib = N.load()

    # ---- construction -------------------------------------------------------
    @classmethod
    def from_host(cls, m) -> "DeviceMatrix":
        from .core import CscMatrix, CsrMatrix, SymHalfMatrix

        if isinstance(m, SymHalfMatrix):
            fmt, off, idx = N.FMT_SCSR, m.row_start, m.col_idx
        elif isinstance(m, CsrMatrix):
            fmt, off, idx = N.FMT_CSR, m.row_start, m.col_idx
        elif isinstance(m, CscMatrix):
            fmt, off, idx = N.FMT_CSC, m.col_start, m.row_idx
        else:
            raise TypeError(f"unsupported matrix type {type(m).__name__}")
        off = np.ascontiguousarray(off, dtype=np.int64)
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        val = np.ascontiguousarray(m.values, dtype=np.float64)
        lib = N.load()
        h = ctypes.c_void_p()
        rc = lib.spcg_matrix_create_host(fmt, m.n, int(val.shape[0]), _ptr(off), _ptr(idx),
                                         _ptr(val), ctypes.byref(h))
        N.check(rc, "spcg_matrix_create_host")
        return cls(h.value, fmt, m.n, int(val.shape[0]), m.dtype)

    @classmethod
    def from_spcg_arrays(cls, fmt: int, n: int, row_start_u64: np.ndarray, col_idx_u32: np.ndarray,
                         values: np.ndarray) -> "DeviceMatrix":
        """Upload the raw u64/u32 arrays of a .spcg container (matio.py:162-168)."""
        off = np.ascontiguousarray(row_start_u64, dtype=np.uint64)
        idx = np.ascontiguousarray(col_idx_u32, dtype=np.uint32)
        val = np.ascontiguousarray(values, dtype=np.float64)
        h = ctypes.c_void_p()
        rc = N.load().spcg_matrix_create_host_u32(fmt, n, int(val.shape[0]), _ptr(off), _ptr(idx),
                                                  _ptr(val), ctypes.byref(h))
        N.check(rc, "spcg_matrix_create_host_u32")
        return cls(h.value, fmt, n, int(val.shape[0]))

    @classmethod
    def from_pairs(cls, n: int, I: np.ndarray, J: np.ndarray, v: np.ndarray, diag_shift: float,
                   fmt: str = "csr") -> "DeviceMatrix":
        """Assemble a generator's mirrored pairs in HBM (spcg_matrix_assemble_pairs)."""
        I = np.ascontiguousarray(I, dtype=np.int64)
        J = np.ascontiguousarray(J, dtype=np.int64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        if not (I.shape == J.shape == v.shape):
            raise ValueError("I, J and v must have the same length")
        h = ctypes.c_void_p()
        N.check(N.load().spcg_matrix_assemble_pairs(cls.FORMATS[fmt], int(n), int(I.size), _ptr(I),
                                                    _ptr(J), _ptr(v), float(diag_shift),
                                                    ctypes.byref(h)), "spcg_matrix_assemble_pairs")
        dm = cls(h.value, cls.FORMATS[fmt], 0, 0)
        dm._refresh()
        return dm

    @classmethod
    def from_device_arrays_u32(cls, fmt: int, n: int, nnz: int, d_ptr: int, d_idx: int,
                               d_val: int) -> "DeviceMatrix":
        """From device arrays in the .spcg layout (u64 offsets, u32 indices, f64
        values; raw device pointers), converted and validated on the device."""
        h = ctypes.c_void_p()
        N.check(N.load().spcg_matrix_create_device_u32(fmt, int(n), int(nnz), d_ptr, d_idx, d_val,
                                                       ctypes.byref(h)),
                "spcg_matrix_create_device_u32")
        dm = cls(h.value, fmt, 0, 0)
        dm._refresh()
        return dm

    @classmethod
    def generate(cls, kind: str, dims: tuple[int, ...], fmt: str = "csr") -> "DeviceMatrix":
        """In-HBM generator: kind in {'poisson2d','poisson3d','stencil27'}."""
        kinds = {"poisson2d": N.GEN_POISSON2D, "poisson3d": N.GEN_POISSON3D,
                 "stencil27": N.GEN_STENCIL27}
        d = list(dims) + [1] * (3 - len(dims))
        h = ctypes.c_void_p()
        rc = N.load().spcg_matrix_generate(kinds[kind], cls.FORMATS[fmt], d[0], d[1], d[2],
                                           ctypes.byref(h))
        N.check(rc, "spcg_matrix_generate")
        dm = cls(h.value, cls.FORMATS[fmt], 0, 0)
        dm._refresh()
        return dm

    def _refresh(self):
        n, nnz, fmt, nt, nb = (ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int(),
                               ctypes.c_int64(), ctypes.c_int64())
        N.check(self._lib.spcg_matrix_info(self._h, ctypes.byref(n), ctypes.byref(nnz),
                                           ctypes.byref(fmt), ctypes.byref(nt), ctypes.byref(nb)),
                "spcg_matrix_info")
        self.n, self.nnz, self.fmt = n.value, nnz.value, fmt.value
        self.ntiles, self.device_bytes = nt.value, nb.value

    def info(self) -> dict:
        self._refresh()
        return {"n": self.n, "nnz": self.nnz, "fmt": self.fmt, "ntiles": self.ntiles,
                "device_bytes": self.device_bytes}

    def download(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """(offsets, indices, values) copied back to the host as int64/f64."""
        off = np.empty(self.n + 1, dtype=np.int64)
        idx = np.empty(self.nnz, dtype=np.int64)
        val = np.empty(self.nnz, dtype=np.float64)
        N.check(self._lib.spcg_matrix_download(self._h, _ptr(off), _ptr(idx), _ptr(val)),
                "spcg_matrix_download")
        return off, idx, val

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    def close(self):
        if self._h is not None and self._h.value:
            self._lib.spcg_matrix_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
