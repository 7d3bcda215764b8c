"""Synthetic SPD systems of the benchmark configurations (host side).

`poisson2d`, `poisson3d`, `random_spd` reproduce the reference generators'
outputs bit for bit (genprob.py:50-129; same seeded PCG64 call sequence for
random_spd) so the oracle and the device solve identical systems.  Two
generators are new:
  * `fem_mesh`  — the "FEM-shaped" 30880x30880 / 449,798-nnz matrix (F-mesh):
    a 16x10x193 mesh, all 7-point edges plus 121,997 seeded edges of the
    27-point neighbourhood, off-diagonals -U(0.5,1), diagonal = |row sum| + shift;
  * `stencil27` — 27-point stencil (26 on the diagonal, -1 off it), full or L+D.
The device twins of poisson2d/poisson3d/stencil27 (`DeviceMatrix.generate`)
build the same arrays directly in HBM.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import INDEX_DTYPE, CsrMatrix, SymHalfMatrix, build_csr_from_triplets

_N_LIMIT = 2**31


@dataclass(frozen=True)
class ProblemSpec:
    kind: str  # poisson2d | poisson3d | random_spd | fem_mesh | stencil27
    dims: tuple[int, ...]
    density: float = 0.05
    seed: int = 0

    def __post_init__(self):
        if self.kind not in ("poisson2d", "poisson3d", "random_spd", "fem_mesh", "stencil27"):
            raise ValueError(f"unknown problem kind {self.kind!r}")
        if any(d < 1 for d in self.dims):
            raise ValueError("extents must be >= 1")
        if not (0 < self.density <= 1):
            raise ValueError("density must be in (0, 1]")


def generate(spec: ProblemSpec, dtype=np.float64) -> CsrMatrix:
    if spec.kind == "poisson2d":
        return poisson2d(*spec.dims, dtype=dtype)
    if spec.kind == "poisson3d":
        return poisson3d(*spec.dims, dtype=dtype)
    if spec.kind == "stencil27":
        return stencil27(*spec.dims, dtype=dtype)
    if spec.kind == "fem_mesh":
        return fem_mesh(*spec.dims, seed=spec.seed, dtype=dtype)
    return random_spd(spec.dims[0], spec.density, spec.seed, dtype=dtype)


def _guard(n: int):
    if n >= _N_LIMIT:
        raise OverflowError(f"grid of {n} points exceeds the supported size")


def _stencil_csr(dims, offsets, diag: float, part: str, dtype) -> CsrMatrix:
    """Natural-order stencil assembled directly in CSR (sorted columns).

    `offsets` are (dz, dy, dx) triples; a neighbour exists when it stays in
    the grid.  part: 'full' | 'lower' (L+D) | 'upper' (strict, = CSR of L^T).
    """
    nx, ny, nz = dims
    n = nx * ny * nz
    _guard(n)
    idx = np.arange(n, dtype=INDEX_DTYPE)
    ix = idx % nx
    iy = (idx // nx) % ny
    iz = idx // (nx * ny)
    offs = sorted(offsets, key=lambda o: o[0] * nx * ny + o[1] * nx + o[2])
    cols, masks, vals = [], [], []
    for dz, dy, dx in offs:
        lin = dz * nx * ny + dy * nx + dx
        if part == "lower" and lin > 0:
            continue
        if part == "upper" and lin <= 0:
            continue
        ok = ((ix + dx >= 0) & (ix + dx < nx) & (iy + dy >= 0) & (iy + dy < ny)
              & (iz + dz >= 0) & (iz + dz < nz))
        masks.append(ok)
        cols.append(idx + lin)
        vals.append(diag if lin == 0 else -1.0)
    m = np.stack(masks, axis=1)  # (n, k), columns ascending by offset
    counts = m.sum(axis=1)
    row_start = np.zeros(n + 1, dtype=INDEX_DTYPE)
    np.cumsum(counts, out=row_start[1:])
    c = np.stack(cols, axis=1)[m]
    v = np.broadcast_to(np.asarray(vals, dtype=dtype), m.shape)[m]
    cls = SymHalfMatrix if part == "lower" else CsrMatrix
    return cls(n=n, row_start=row_start, col_idx=c.astype(INDEX_DTYPE), values=np.ascontiguousarray(v))


_OFF5 = [(0, 0, 0), (0, 0, -1), (0, 0, 1), (0, -1, 0), (0, 1, 0)]
_OFF7 = _OFF5 + [(-1, 0, 0), (1, 0, 0)]
_OFF27 = [(dz, dy, dx) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]


def poisson2d(nx: int, ny: int, dtype=np.float64) -> CsrMatrix:
    """5-point Laplacian, 4 on the diagonal, -1 per grid neighbour (genprob.py:50-70)."""
    if nx < 1 or ny < 1:
        raise ValueError("extents must be >= 1")
    return _stencil_csr((nx, ny, 1), _OFF5, 4.0, "full", dtype)


def poisson3d(nx: int, ny: int, nz: int, dtype=np.float64) -> CsrMatrix:
    """7-point Laplacian, diagonal 6 (genprob.py:73-93)."""
    if min(nx, ny, nz) < 1:
        raise ValueError("extents must be >= 1")
    return _stencil_csr((nx, ny, nz), _OFF7, 6.0, "full", dtype)


def stencil27(nx: int, ny: int, nz: int, part: str = "full", dtype=np.float64):
    """27-point stencil: 26 on the diagonal, -1 for each of the <= 26
    neighbours (irreducibly diagonally dominant, hence SPD).  part='lower'
    returns the SymHalfMatrix L+D directly."""
    if min(nx, ny, nz) < 1:
        raise ValueError("extents must be >= 1")
    return _stencil_csr((nx, ny, nz), _OFF27, 26.0, part, dtype)


def random_spd_pairs(n: int, density: float, seed: int):
    """The random draws of random_spd (genprob.py:96-129): m distinct
    strictly-lower pairs (I > J) by rng.choice over the row-major pair
    enumeration and their values U(-1, 0), in draw order."""
    if n < 1:
        raise ValueError("n must be >= 1")
    rng = np.random.default_rng(seed)
    npairs = n * (n - 1) // 2
    m = min(npairs, int(round(density * n * n / 2)))
    if m == 0:
        e = np.empty(0, dtype=INDEX_DTYPE)
        return e, e.copy(), np.empty(0)
    ids = rng.choice(npairs, size=m, replace=False).astype(INDEX_DTYPE)
    # pair id -> (i, j): row i owns ids [i(i-1)/2, i(i+1)/2)
    i = ((1 + np.sqrt(1 + 8 * ids.astype(np.float64))) // 2).astype(INDEX_DTYPE)
    i -= (i * (i - 1) // 2 > ids)
    i += ((i + 1) * i // 2 <= ids)
    j = ids - i * (i - 1) // 2
    v = rng.uniform(-1.0, 0.0, size=m)
    return i, j, v


def _assemble_pairs(n, I, J, v, shift, dtype):
    rows, cols, vals = np.concatenate([I, J]), np.concatenate([J, I]), np.concatenate([v, v])
    diag = np.bincount(rows, weights=np.abs(vals), minlength=n) + shift
    ar = np.arange(n, dtype=INDEX_DTYPE)
    return build_csr_from_triplets(
        (np.concatenate([rows, ar]), np.concatenate([cols, ar]), np.concatenate([vals, diag])),
        n, dtype=dtype)


def random_spd(n: int, density: float, seed: int, dtype=np.float64) -> CsrMatrix:
    """Seeded strictly diagonally dominant symmetric matrix (genprob.py:96-129):
    m = round(density*n^2/2) distinct strictly-lower pairs drawn by
    rng.choice over the row-major pair enumeration, values U(-1,0), mirrored,
    diagonal = absolute row sum + 1."""
    I, J, v = random_spd_pairs(n, density, seed)
    return _assemble_pairs(n, I, J, v, 1.0, dtype)


def random_spd_device(n: int, density: float, seed: int, fmt: str = "csr"):
    """random_spd assembled in HBM (the draws on the host, numpy PCG64 like the
    reference; mirroring, diagonal and CSR / SCSR / CSC layout on the device):
    bitwise the host generator's matrix.  Returns a DeviceMatrix."""
    from .device import DeviceMatrix

    I, J, v = random_spd_pairs(n, density, seed)
    return DeviceMatrix.from_pairs(n, I, J, v, 1.0, fmt)


def _lower_edges(nx, ny, nz, offsets):
    """Lower (j < i) neighbour pairs (i, j) for each offset in the given
    order; within an offset, nodes ascending."""
    n = nx * ny * nz
    idx = np.arange(n, dtype=INDEX_DTYPE)
    ix, iy, iz = idx % nx, (idx // nx) % ny, idx // (nx * ny)
    I, J = [], []
    for dz, dy, dx in offsets:
        lin = dz * nx * ny + dy * nx + dx
        if lin >= 0:
            continue
        ok = ((ix + dx >= 0) & (ix + dx < nx) & (iy + dy >= 0) & (iy + dy < ny)
              & (iz + dz >= 0) & (iz + dz < nz))
        I.append(idx[ok])
        J.append(idx[ok] + lin)
    return np.concatenate(I), np.concatenate(J)


def fem_mesh_pairs(nx: int = 16, ny: int = 10, nz: int = 193, extra: int = 121_997,
                   seed: int = 1):
    """(n, I, J, v): the lower pairs of fem_mesh in draw order (I > J)."""
    off7 = [o for o in _OFF27 if sum(c != 0 for c in o) == 1]
    offx = [o for o in _OFF27 if sum(c != 0 for c in o) > 1]
    i7, j7 = _lower_edges(nx, ny, nz, off7)
    ie, je = _lower_edges(nx, ny, nz, offx)
    rng = np.random.default_rng(seed)
    pick = rng.choice(ie.shape[0], size=extra, replace=False)
    I = np.concatenate([i7, ie[pick]])
    J = np.concatenate([j7, je[pick]])
    v = -rng.uniform(0.5, 1.0, size=I.shape[0])
    return nx * ny * nz, I, J, v


def fem_mesh(nx: int = 16, ny: int = 10, nz: int = 193, extra: int = 121_997,
             shift: float = 0.004, seed: int = 1, dtype=np.float64) -> CsrMatrix:
    """FEM-shaped SPD matrix (SURVEY.md §8d "F-mesh"); defaults give the
    30880 x 30880, 449,798-nnz configuration of BASELINE.json configs[0].

    Pair order: the 7-point lower edges (offsets in (dz,dy,dx) nested order,
    nodes ascending), then the `extra` edges drawn with
    default_rng(seed).choice(len(E), extra, replace=False) from E = the other
    lower 27-point-neighbourhood edges (same enumeration), in draw order.
    Values -U(0.5, 1) from the same generator, mirrored; diagonal = sum of
    |off-diagonals| + shift.
    """
    n, I, J, v = fem_mesh_pairs(nx, ny, nz, extra, seed)
    return _assemble_pairs(n, I, J, v, shift, dtype)


def fem_mesh_device(nx: int = 16, ny: int = 10, nz: int = 193, extra: int = 121_997,
                    shift: float = 0.004, seed: int = 1, fmt: str = "csr"):
    """fem_mesh assembled in HBM (draws on the host, assembly on the device):
    bitwise the host generator's matrix.  Returns a DeviceMatrix."""
    from .device import DeviceMatrix

    n, I, J, v = fem_mesh_pairs(nx, ny, nz, extra, seed)
    return DeviceMatrix.from_pairs(n, I, J, v, shift, fmt)


def rhs_for(a, seed: int = 1) -> tuple[np.ndarray, np.ndarray]:
    """(b, x_gen) following cmd_gen (cli.py:91-93): x_gen =
    default_rng(seed).standard_normal(n) and b = A x_gen as a sequential
    row-order sum over the FULL matrix (what spmv_full computes)."""
    from .core import expand_symmetric

    full = expand_symmetric(a) if isinstance(a, SymHalfMatrix) else a
    x = np.random.default_rng(seed).standard_normal(full.n)
    b = np.bincount(full.entry_rows, weights=full.values * x[full.col_idx], minlength=full.n)
    return b, x
