"""Device kernel API vs the oracle / the reference's golden outputs."""

import numpy as np
import pytest

from conftest import dense_spmv_oracle, random_csr, rel_inf_err
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _csr(g, i, p="c"):
    from paper_1010_4639_b200.core import CsrMatrix, SymHalfMatrix

    cls = CsrMatrix if p == "c" else SymHalfMatrix
    rs = g[f"{p}{i}_rs"]
    return cls(n=len(rs) - 1, row_start=rs, col_idx=g[f"{p}{i}_ci"], values=g[f"{p}{i}_v"])


def test_spmv_full_bitwise_equals_reference(golden):
    from paper_1010_4639_b200 import spmv_full

    g = golden("kernels_small")
    for i in range(int(g["ncases"])):
        y = spmv_full(_csr(g, i), g[f"c{i}_x"])
        assert (y == g[f"c{i}_y"]).all(), i


def test_spmv_sym_privatized_bitwise_and_atomic_close(golden):
    from paper_1010_4639_b200 import KernelConfig, spmv_sym

    g = golden("kernels_small")
    for i in range(int(g["nsym"])):
        s = _csr(g, i, "s")
        x = g[f"s{i}_x"]
        yp = spmv_sym(s, x, KernelConfig(accumulation="privatized"))
        assert (yp == g[f"s{i}_ypriv1"]).all(), i
        ya = spmv_sym(s, x, KernelConfig(accumulation="atomic"))
        assert rel_inf_err(ya, g[f"s{i}_yatom"]) <= 1e-12, i


def test_spmv_csc_matches_column_scatter_oracle():
    from paper_1010_4639_b200 import spmv_csc

    rng = np.random.default_rng(5)
    for _ in range(30):
        n = int(rng.integers(1, 80))
        a = random_csr(rng, n, float(rng.uniform(0.01, 0.4)))
        c = a.to_csc()
        x = rng.standard_normal(n)
        y = spmv_csc(c, x)
        ref = O.spmv_csc(c.col_start, c.row_idx, c.values, x)
        assert rel_inf_err(y, ref) <= 1e-12
        assert rel_inf_err(y, dense_spmv_oracle(a.to_dense(), x)) <= 1e-13


def test_criterion1_random_vs_dense_oracle():
    from paper_1010_4639_b200 import spmv_full

    rng = np.random.default_rng(1001)
    worst = 0.0
    for _ in range(200):
        n = int(rng.integers(1, 65))
        m = random_csr(rng, n, float(rng.uniform(0.01, 0.3)))
        x = rng.standard_normal(n)
        worst = max(worst, rel_inf_err(spmv_full(m, x), dense_spmv_oracle(m.to_dense(), x)))
    assert worst <= 1e-13


def test_long_rows_and_tiles():
    """Rows longer than a tile (4096 entries) take the CTA-wide path."""
    from paper_1010_4639_b200 import KernelConfig, extract_lower, spmv_full, spmv_sym
    from paper_1010_4639_b200.core import build_csr_from_triplets

    rng = np.random.default_rng(9)
    n = 9000
    rows = np.concatenate([np.zeros(6000, np.int64), rng.integers(0, n, 20000)])
    cols = np.concatenate([rng.choice(n, 6000, replace=False), rng.integers(0, n, 20000)])
    a = build_csr_from_triplets((rows, cols, rng.standard_normal(rows.size)), n)
    x = rng.standard_normal(n)
    y = spmv_full(a, x)
    ref = O.spmv_full(a.row_start, a.col_idx, a.values, x)
    assert rel_inf_err(y, ref) <= 1e-12
    short = np.diff(a.row_start) <= 4096
    assert (y[short] == ref[short]).all()
    # symmetric with a dense first column (long last row in L+D)
    sym_rows = np.concatenate([np.arange(1, n), np.arange(n)])
    sym_cols = np.concatenate([np.zeros(n - 1, np.int64), np.arange(n)])
    vals = np.concatenate([-np.ones(n - 1) * 1e-3, np.full(n, 10.0)])
    full = build_csr_from_triplets((np.concatenate([sym_rows, sym_cols[: n - 1]]),
                                    np.concatenate([sym_cols, sym_rows[: n - 1]]),
                                    np.concatenate([vals, vals[: n - 1]])), n)
    s = extract_lower(full)
    for acc in ("atomic", "privatized"):
        ys = spmv_sym(s, x, KernelConfig(accumulation=acc))
        assert rel_inf_err(ys, O.spmv_full(full.row_start, full.col_idx, full.values, x)) <= 1e-12


def test_dot_axpy_norm():
    from paper_1010_4639_b200 import axpy, dot, norm2

    assert dot(np.zeros(10), np.ones(10)) == 0.0
    assert dot([1.0, 2.0, 3.0], [4.0, 5.0, 6.0]) == 32.0
    for n in (1, 7, 1000, 1 << 20):
        assert dot(np.ones(n), np.ones(n)) == float(n)
    rng = np.random.default_rng(8)
    u, v = rng.standard_normal(100_001), rng.standard_normal(100_001)
    d0 = dot(u, v)
    assert all(dot(u, v) == d0 for _ in range(5))  # deterministic
    assert abs(d0 - O.dot(u, v)) <= 1e-12 * max(1.0, abs(d0)) * 100
    assert (axpy(0.0, u, v) == v).all()
    assert (axpy(2.0, np.array([1.0, 1.0]), np.array([0.0, 3.0])) == [2.0, 5.0]).all()
    assert (axpy(-1.0, u, u.copy()) == 0.0).all()
    assert (axpy(1.7, u, v) == O.axpy(1.7, u, v)).all()  # bitwise
    assert norm2(np.array([3.0, 4.0])) == 5.0
    w = rng.standard_normal(100)
    exp = float(np.sqrt(sum(val * val for val in w)))
    assert abs(norm2(w) - exp) <= 1e-15 * exp


def test_dimension_mismatch():
    from paper_1010_4639_b200 import build_csr_from_triplets, spmv_full

    a = build_csr_from_triplets([(0, 0, 4.0), (0, 1, 1.0), (1, 0, 1.0), (1, 1, 3.0)], 2)
    with pytest.raises(ValueError, match="dimension mismatch"):
        spmv_full(a, np.ones(3))


def test_torch_device_io():
    import torch

    from paper_1010_4639_b200 import dot, spmv_full
    from paper_1010_4639_b200.genprob import poisson2d

    a = poisson2d(20, 30)
    x = torch.randn(a.n, dtype=torch.float64, device="cuda")
    y = spmv_full(a, x)
    assert y.is_cuda
    ref = O.spmv_full(a.row_start, a.col_idx, a.values, x.cpu().numpy())
    assert (y.cpu().numpy() == ref).all()
    assert dot(x, x) == pytest.approx(float((x * x).sum()), rel=1e-13)


@pytest.mark.parametrize("kind,dims", [("poisson2d", (37, 23)), ("poisson3d", (9, 7, 11)),
                                       ("stencil27", (6, 5, 7))])
def test_device_generators_match_host(kind, dims):
    from paper_1010_4639_b200.device import DeviceMatrix

    dm = DeviceMatrix.generate(kind, dims, "csr")
    rs, ci, v = O.stencil(kind, dims)
    off, idx, val = dm.download()
    assert (off == rs).all() and (idx == ci).all() and (val == v).all()
    if kind == "stencil27":
        dm = DeviceMatrix.generate(kind, dims, "scsr")
        rs, ci, v = O.stencil(kind, dims, part="lower")
        off, idx, val = dm.download()
        assert (off == rs).all() and (idx == ci).all() and (val == v).all()


@pytest.mark.parametrize("ragged", [False, True])
def test_spmv_wide_tiles_bitwise(ragged):
    """Short-row CSR matrices large enough for wide tiles (two lines per
    thread in the streaming passes) stay bitwise equal to csr_gather."""
    from paper_1010_4639_b200 import spmv_full
    from paper_1010_4639_b200.core import CsrMatrix

    rng = np.random.default_rng(77 + ragged)
    n = 400_000
    lens = (rng.choice([0, 1, 2, 3, 4, 5, 6, 9, 17, 24], size=n,
                       p=[.06, .1, .12, .2, .2, .17, .1, .03, .015, .005])
            if ragged else np.full(n, 5))
    rows = np.repeat(np.arange(n), lens)
    cols = np.clip(rows + rng.integers(-3000, 3000, size=len(rows)), 0, n - 1)
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    keep = np.ones(len(rows), bool)
    keep[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
    rows, cols = rows[keep], cols[keep]
    rs = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rs, rows + 1, 1)
    rs = np.cumsum(rs)
    vals = rng.standard_normal(len(cols))
    a = CsrMatrix(n=n, row_start=rs, col_idx=cols.astype(np.int64), values=vals)
    x = rng.standard_normal(n)
    y = spmv_full(a, x)
    ref = O.spmv_full(a.row_start, a.col_idx, a.values, x)
    assert (y == ref).all()


def test_cg_wide_tiles_poisson2d_matches_reference():
    """CG on a 2D Poisson system with wide tiles (640^2 rows) against the
    reference CG: same iteration count, x within 1e-8."""
    from paper_1010_4639_b200 import CgOptions, cg_solve
    from paper_1010_4639_b200.genprob import poisson2d, rhs_for

    a = poisson2d(640, 640)
    b, _ = rhs_for(a, seed=3)
    ref = O.cg_solve("csr", a.row_start, a.col_idx, a.values, b, max_iter=5000)
    r = cg_solve(a, b, opts=CgOptions(max_iter=5000))
    assert r.converged
    assert abs(r.iterations - ref.iterations) <= max(1, ref.iterations // 100)
    assert np.linalg.norm(r.x - ref.x) / np.linalg.norm(ref.x) <= 1e-8
