"""Sparse storage types on the host: full CSR, symmetric half (L+D) CSR and CSC.

Semantics follow the reference's `spcg.core` (core.py:57-309): immutable
objects with frozen int64 index arrays, duplicate-summing triplet assembly,
violation-list validation, tolerance-based symmetry checks and full<->half
conversion.  These are the *inputs* of the solve path; the device copy (int32
indices, row tiles) is created once per object by `DeviceMatrix` and cached.
`CscMatrix` is new: the reference has no CSC type.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

DEFAULT_SYMMETRY_TOL = 1e-12
INDEX_DTYPE = np.int64


class MatrixConstructionError(ValueError):
    """Input data cannot form a valid sparse matrix (core.py:21-22)."""


class AsymmetricMatrixError(ValueError):
    """A symmetric-only operation received an asymmetric matrix (core.py:25-26)."""


class MissingDiagonalError(ValueError):
    """Symmetric-half storage lacks a structural diagonal entry (core.py:29-30)."""


def _frozen(a, dtype=None) -> np.ndarray:
    arr = np.ascontiguousarray(a if dtype is None else np.asarray(a).astype(dtype, copy=False))
    if arr.flags.writeable and arr.base is not None:
        arr = arr.copy()
    arr.flags.writeable = False
    return arr


def as_vector(data, n: int | None = None, dtype=None) -> np.ndarray:
    """Boundary check for dense vectors (core.py:39-54): 1-D, real, finite."""
    v = np.ascontiguousarray(data, dtype=dtype)
    if v.ndim != 1:
        raise ValueError(f"expected a 1-D vector, got shape {v.shape}")
    if v.dtype not in (np.float32, np.float64):
        v = v.astype(np.float64)
    if n is not None and v.shape[0] != n:
        raise ValueError(f"expected length {n}, got {v.shape[0]}")
    if not np.isfinite(v).all():
        raise ValueError("vector contains non-finite entries")
    return v


def _rows_of(offsets: np.ndarray, n: int) -> np.ndarray:
    return np.repeat(np.arange(n, dtype=INDEX_DTYPE), np.diff(offsets))


class _Compressed:
    """Shared behaviour of the three compressed layouts."""

    n: int
    values: np.ndarray

    def _init_arrays(self, off_name: str, idx_name: str):
        object.__setattr__(self, off_name, _frozen(getattr(self, off_name), INDEX_DTYPE))
        object.__setattr__(self, idx_name, _frozen(getattr(self, idx_name), INDEX_DTYPE))
        object.__setattr__(self, "values", _frozen(self.values))
        object.__setattr__(self, "_cache", {})

    @property
    def dtype(self):
        return self.values.dtype

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])

    def device(self, accumulation: str | None = None):
        """Device copy on the CURRENT CUDA device (uploaded once per device;
        matrices are immutable)."""
        from .device import DeviceMatrix, current_device

        key = ("device", current_device())
        dev = self._cache.get(key)
        if dev is None:
            dev = DeviceMatrix.from_host(self)
            self._cache[key] = dev
        return dev


@dataclass(frozen=True, eq=False)
class CsrMatrix(_Compressed):
    """Square matrix in compressed sparse row form (core.py:57-100).

    row_start has n+1 entries, row_start[0] = 0, row_start[n] = nnz; column
    indices are 0-based and strictly increasing within a row.
    """

    n: int
    row_start: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    _cache: dict = field(default=None, init=False, repr=False, compare=False)

    def __post_init__(self):
        self._init_arrays("row_start", "col_idx")

    @property
    def entry_rows(self) -> np.ndarray:
        r = self._cache.get("entry_rows")
        if r is None:
            r = _frozen(_rows_of(self.row_start, self.n))
            self._cache["entry_rows"] = r
        return r

    def diagonal(self) -> np.ndarray:
        d = np.zeros(self.n, dtype=self.dtype)
        rows = self.entry_rows
        on = rows == self.col_idx
        d[rows[on]] = self.values[on]
        return d

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.n, self.n), dtype=self.dtype)
        out[self.entry_rows, self.col_idx] = self.values
        return out

    def to_csc(self) -> "CscMatrix":
        """Same matrix in CSC form (columns ascending, rows ascending within)."""
        return csc_from_triplets(self.entry_rows, self.col_idx, self.values, self.n)


@dataclass(frozen=True, eq=False)
class SymHalfMatrix(_Compressed):
    """CSR of L+D for a symmetric A = L + D + L^T (core.py:103-156).

    Every entry has col <= row and the diagonal is the last entry of its row.
    """

    n: int
    row_start: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    diag_present: bool = True
    _cache: dict = field(default=None, init=False, repr=False, compare=False)

    def __post_init__(self):
        self._init_arrays("row_start", "col_idx")
        rows = self.entry_rows
        if (self.col_idx > rows).any():
            raise MatrixConstructionError(
                "symmetric-half storage requires col <= row for every entry"
            )
        if self.n > 0 and self.col_idx.shape[0] < self.n:
            raise MissingDiagonalError("fewer stored entries than rows; some diagonal is missing")
        if self.n > 0:
            lens = np.diff(self.row_start)
            last = np.maximum(self.row_start[1:] - 1, 0)
            good = (lens > 0) & (self.col_idx[last] == np.arange(self.n))
            if not good.all():
                raise MissingDiagonalError(f"row {int(np.argmin(good))} has no stored diagonal entry")
        object.__setattr__(self, "diag_present", True)

    @property
    def entry_rows(self) -> np.ndarray:
        r = self._cache.get("entry_rows")
        if r is None:
            r = _frozen(_rows_of(self.row_start, self.n))
            self._cache["entry_rows"] = r
        return r

    @property
    def strict_lower(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """(rows, cols, values) of the strictly lower entries, storage order."""
        t = self._cache.get("strict_lower")
        if t is None:
            rows = self.entry_rows
            keep = self.col_idx < rows
            t = (_frozen(rows[keep]), _frozen(self.col_idx[keep]), _frozen(self.values[keep]))
            self._cache["strict_lower"] = t
        return t


@dataclass(frozen=True, eq=False)
class CscMatrix(_Compressed):
    """Square matrix in compressed sparse column form (new; no reference type).

    col_start has n+1 entries; row indices strictly increase within a column.
    For a symmetric matrix the CSC arrays equal the CSR arrays.
    """

    n: int
    col_start: np.ndarray
    row_idx: np.ndarray
    values: np.ndarray
    _cache: dict = field(default=None, init=False, repr=False, compare=False)

    def __post_init__(self):
        self._init_arrays("col_start", "row_idx")

    @property
    def entry_cols(self) -> np.ndarray:
        c = self._cache.get("entry_cols")
        if c is None:
            c = _frozen(_rows_of(self.col_start, self.n))
            self._cache["entry_cols"] = c
        return c

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.n, self.n), dtype=self.dtype)
        out[self.row_idx, self.entry_cols] = self.values
        return out

    def to_csr(self) -> CsrMatrix:
        return build_csr_from_triplets((self.row_idx, self.entry_cols, self.values), self.n,
                                       dtype=self.dtype)


@dataclass(frozen=True)
class ValidationReport:
    ok: bool
    violations: tuple

    def __post_init__(self):
        object.__setattr__(self, "violations", tuple(self.violations))
        if self.ok != (len(self.violations) == 0):
            raise AssertionError("ok must equal 'no violations'")


def _coerce_triplets(triplets, dtype):
    if isinstance(triplets, tuple) and len(triplets) == 3 and isinstance(triplets[0], np.ndarray):
        rows, cols, vals = triplets
    elif len(triplets) == 0:
        return (np.empty(0, INDEX_DTYPE), np.empty(0, INDEX_DTYPE), np.empty(0, dtype))
    else:
        rows, cols, vals = (np.asarray(col) for col in zip(*triplets))
    return (np.asarray(rows).astype(INDEX_DTYPE, copy=False),
            np.asarray(cols).astype(INDEX_DTYPE, copy=False),
            np.asarray(vals, dtype=dtype))


def _assemble(major, minor, vals, n, drop_zeros):
    """Sort by (major, minor), sum duplicates, return (offsets, minor, vals)."""
    if major.size:
        order = np.lexsort((minor, major))
        major, minor, vals = major[order], minor[order], vals[order]
        first = np.ones(major.size, dtype=bool)
        first[1:] = (major[1:] != major[:-1]) | (minor[1:] != minor[:-1])
        if not first.all():
            starts = np.flatnonzero(first)
            vals = np.add.reduceat(vals, starts)
            major, minor = major[starts], minor[starts]
    if drop_zeros and major.size:
        nz = vals != 0
        major, minor, vals = major[nz], minor[nz], vals[nz]
    offsets = np.zeros(n + 1, dtype=INDEX_DTYPE)
    np.cumsum(np.bincount(major, minlength=n), out=offsets[1:])
    return offsets, minor, vals


def _check_range(rows, cols, vals, n):
    bad = (rows < 0) | (rows >= n) | (cols < 0) | (cols >= n)
    if bad.any():
        k = int(np.argmax(bad))
        raise MatrixConstructionError(
            f"triplet ({int(rows[k])}, {int(cols[k])}, {vals[k]!r}) is outside [0, {n})"
        )


def build_csr_from_triplets(triplets, n: int, dtype=np.float64, drop_zeros: bool = False) -> CsrMatrix:
    """Assemble CSR from (row, col, value) triplets; duplicates are summed
    (core.py:169-212)."""
    rows, cols, vals = _coerce_triplets(triplets, dtype)
    _check_range(rows, cols, vals, n)
    off, idx, v = _assemble(rows, cols, vals, n, drop_zeros)
    return CsrMatrix(n=n, row_start=off, col_idx=idx, values=v)


def csc_from_triplets(rows, cols, vals, n: int, dtype=None, drop_zeros: bool = False) -> CscMatrix:
    """Assemble CSC from triplets (sorted by column, then row)."""
    rows, cols, vals = _coerce_triplets(
        (np.asarray(rows), np.asarray(cols), np.asarray(vals)),
        dtype if dtype is not None else np.asarray(vals).dtype if np.asarray(vals).size else np.float64,
    )
    _check_range(rows, cols, vals, n)
    off, idx, v = _assemble(cols, rows, vals, n, drop_zeros)
    return CscMatrix(n=n, col_start=off, row_idx=idx, values=v)


def validate_csr(m: CsrMatrix) -> ValidationReport:
    """Every CSR invariant as a list of (rule, row, position) (core.py:215-240)."""
    out: list[tuple[str, int, int]] = []
    n, nnz = m.n, m.values.shape[0]
    if m.row_start.shape[0] != n + 1:
        return ValidationReport(False, [("offsets-length", -1, -1)])
    if m.row_start[0] != 0:
        out.append(("offsets-start", 0, 0))
    steps = np.diff(m.row_start)
    out.extend(("offsets-monotone", int(i), -1) for i in np.flatnonzero(steps < 0))
    if m.row_start[n] != nnz:
        out.append(("offsets-end", n, -1))
    if m.col_idx.shape[0] != nnz:
        out.append(("arrays-length", -1, -1))
    out.extend(("col-range", -1, int(k)) for k in np.flatnonzero((m.col_idx < 0) | (m.col_idx >= n)))
    if not (steps < 0).any():
        for i in range(n):
            lo, hi = int(m.row_start[i]), int(m.row_start[i + 1])
            for p in np.flatnonzero(np.diff(m.col_idx[lo:hi]) <= 0):
                out.append(("col-order", i, lo + int(p) + 1))
    return ValidationReport(not out, out)


def first_asymmetric_pair(m: CsrMatrix, tol: float = DEFAULT_SYMMETRY_TOL):
    """First (i, j) with |A_ij - A_ji| > tol*max(1, min(|A_ij|,|A_ji|)), absent
    mirrors counting as zero (core.py:247-270); None if symmetric."""
    n = np.int64(m.n)
    rows, cols = m.entry_rows, m.col_idx
    keys = rows * n + cols
    tkeys = cols * n + rows
    allk = np.union1d(keys, tkeys)
    a = np.zeros(allk.shape[0])
    b = np.zeros(allk.shape[0])
    a[np.searchsorted(allk, keys)] = m.values
    b[np.searchsorted(allk, tkeys)] = m.values
    bound = tol * np.maximum(1.0, np.minimum(np.abs(a), np.abs(b)))
    bad = np.flatnonzero(np.abs(a - b) > bound)
    if bad.size == 0:
        return None
    key = int(allk[bad[0]])
    return key // m.n, key % m.n


def is_symmetric(m: CsrMatrix, tol: float = DEFAULT_SYMMETRY_TOL) -> bool:
    return first_asymmetric_pair(m, tol) is None


def extract_lower(m: CsrMatrix, tol: float = DEFAULT_SYMMETRY_TOL) -> SymHalfMatrix:
    """L+D of a symmetric matrix with a full structural diagonal (core.py:279-300)."""
    pair = first_asymmetric_pair(m, tol)
    if pair is not None:
        i, j = pair
        raise AsymmetricMatrixError(
            f"matrix is not symmetric: entries ({i}, {j}) and ({j}, {i}) disagree beyond tolerance"
        )
    rows = m.entry_rows
    has_diag = np.bincount(rows[rows == m.col_idx], minlength=m.n) > 0
    if not has_diag.all():
        raise MissingDiagonalError(f"row {int(np.argmin(has_diag))} has no stored diagonal entry")
    keep = m.col_idx <= rows
    off = np.zeros(m.n + 1, dtype=INDEX_DTYPE)
    np.cumsum(np.bincount(rows[keep], minlength=m.n), out=off[1:])
    return SymHalfMatrix(n=m.n, row_start=off, col_idx=m.col_idx[keep], values=m.values[keep])


def expand_symmetric(s: SymHalfMatrix) -> CsrMatrix:
    """A = L + D + L^T from half storage (core.py:303-309)."""
    lr, lc, lv = s.strict_lower
    return build_csr_from_triplets(
        (np.concatenate([s.entry_rows, lc]), np.concatenate([s.col_idx, lr]),
         np.concatenate([s.values, lv])),
        s.n,
        dtype=s.dtype,
    )
