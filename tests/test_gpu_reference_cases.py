"""The reference's pinned kernel and solver cases (test_kernels.py
:35-179, test_solver.py:84-132 of the reference), re-pointed at the device
path and run for every storage and CG engine.  The reference runs these per
backend (python / compiled); here the "backends" are the storages
(CSR, SCSR privatized / atomic, CSC) and the engines of spcg_cg_options."""

import numpy as np
import pytest

from conftest import rel_inf_err

pytestmark = pytest.mark.gpu

STORAGES = ["csr", "sym_priv", "sym_atomic", "csc"]
ENGINES = [0, 2, 3, 5, 6]  # auto, per-pass, single-reduction, cluster, pipelined cluster


def as_storage(a, kind):
    from paper_1010_4639_b200 import KernelConfig, extract_lower

    if kind == "csr":
        return a, KernelConfig()
    if kind == "csc":
        return a.to_csc(), KernelConfig()
    acc = "privatized" if kind == "sym_priv" else "atomic"
    return extract_lower(a), KernelConfig(accumulation=acc)


def spmv_any(m, x, cfg):
    from paper_1010_4639_b200 import CscMatrix, SymHalfMatrix, spmv_csc, spmv_full, spmv_sym

    if isinstance(m, SymHalfMatrix):
        return spmv_sym(m, x, cfg)
    if isinstance(m, CscMatrix):
        return spmv_csc(m, x)
    return spmv_full(m, x, cfg)


# ---- SpMV (reference test_kernels.py:35-116) -------------------------------

@pytest.mark.parametrize("kind", STORAGES)
def test_identity_is_bitwise(kind):
    from paper_1010_4639_b200 import build_csr_from_triplets

    n = 50
    eye = build_csr_from_triplets([(i, i, 1.0) for i in range(n)], n)
    m, cfg = as_storage(eye, kind)
    x = np.random.default_rng(1).standard_normal(n)
    assert (spmv_any(m, x, cfg) == x).all()


@pytest.mark.parametrize("kind", STORAGES)
def test_two_by_two(kind):
    from paper_1010_4639_b200 import build_csr_from_triplets

    a = build_csr_from_triplets([(0, 0, 4.0), (0, 1, 1.0), (1, 0, 1.0), (1, 1, 3.0)], 2)
    m, cfg = as_storage(a, kind)
    assert (spmv_any(m, np.ones(2), cfg) == np.array([5.0, 4.0])).all()


@pytest.mark.parametrize("kind", STORAGES)
def test_poisson3x3_times_ones(kind):
    from paper_1010_4639_b200.genprob import poisson2d

    m, cfg = as_storage(poisson2d(3, 3), kind)
    y = spmv_any(m, np.ones(9), cfg)
    assert y[4] == 0.0  # interior row
    assert (np.delete(y, 4) > 0).all()


@pytest.mark.parametrize("kind", STORAGES)
def test_linearity(kind):
    from paper_1010_4639_b200.genprob import poisson3d

    m, cfg = as_storage(poisson3d(9, 8, 7), kind)
    rng = np.random.default_rng(3)
    u, v = rng.standard_normal(504), rng.standard_normal(504)
    a, b = 1.7, -0.3
    lhs = spmv_any(m, a * u + b * v, cfg)
    rhs = a * spmv_any(m, u, cfg) + b * spmv_any(m, v, cfg)
    assert rel_inf_err(lhs, rhs) <= 1e-12


@pytest.mark.parametrize("acc", ["privatized", "atomic"])
def test_sym_diagonal_only_is_bitwise(acc):
    from paper_1010_4639_b200 import KernelConfig, SymHalfMatrix, spmv_sym

    n = 40
    d = np.random.default_rng(4).uniform(1, 2, n)
    s = SymHalfMatrix(n=n, row_start=np.arange(n + 1), col_idx=np.arange(n), values=d)
    x = np.random.default_rng(5).standard_normal(n)
    assert (spmv_sym(s, x, KernelConfig(accumulation=acc)) == d * x).all()


@pytest.mark.parametrize("acc", ["privatized", "atomic"])
def test_sym_poisson_matches_full(acc):
    from paper_1010_4639_b200 import KernelConfig, extract_lower, spmv_full, spmv_sym
    from paper_1010_4639_b200.genprob import poisson2d

    a = poisson2d(17, 13)
    x = np.random.default_rng(6).standard_normal(a.n)
    y = spmv_sym(extract_lower(a), x, KernelConfig(accumulation=acc))
    assert rel_inf_err(y, spmv_full(a, x)) <= 1e-14


def test_axpy_self_cancels_and_dot_of_ones_exact():
    from paper_1010_4639_b200 import axpy, dot

    u = np.random.default_rng(7).standard_normal(100_003)
    assert (axpy(-1.0, u, u) == 0.0).all()
    assert dot(np.ones(1_000_000), np.ones(1_000_000)) == 1_000_000.0


# ---- CG (reference test_solver.py:84-132), every storage x engine ---------

def _solve(a, b, kind, engine, **kw):
    from paper_1010_4639_b200 import CgOptions, cg_solve

    m, cfg = as_storage(a, kind)
    return cg_solve(m, b, opts=CgOptions(**kw), cfg=cfg, engine=engine)


@pytest.mark.parametrize("engine", ENGINES)
def test_representation_equivalence(engine):
    from paper_1010_4639_b200.genprob import poisson2d

    a = poisson2d(8, 8)
    b = np.random.default_rng(5).standard_normal(64)
    full = _solve(a, b, "csr", engine)
    for kind in STORAGES[1:]:
        other = _solve(a, b, kind, engine)
        assert abs(full.iterations - other.iterations) <= 1, kind
        assert np.max(np.abs(full.x - other.x)) <= 1e-8, kind


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("kind", STORAGES)
def test_solution_certificate(kind, engine):
    from paper_1010_4639_b200.genprob import poisson2d

    a = poisson2d(10, 10)
    b = np.random.default_rng(8).standard_normal(100)
    r = _solve(a, b, kind, engine, tol=1e-10, recompute_final_residual=True)
    assert r.converged
    assert r.final_relative_residual <= 10 * 1e-10
    true = np.linalg.norm(b - a.to_dense() @ r.x) / np.linalg.norm(b)
    assert true <= 10 * 1e-10


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("kind", STORAGES)
def test_scaling_invariance(kind, engine):
    from paper_1010_4639_b200 import build_csr_from_triplets
    from paper_1010_4639_b200.genprob import poisson2d

    a = poisson2d(7, 7)
    b = np.random.default_rng(9).standard_normal(49)
    base = _solve(a, b, kind, engine)
    scaled = build_csr_from_triplets((a.entry_rows.copy(), a.col_idx.copy(), 3.0 * a.values), a.n)
    s = _solve(scaled, 3.0 * b, kind, engine)
    assert s.iterations == base.iterations
    assert np.max(np.abs(s.x - base.x)) <= 1e-9


@pytest.mark.parametrize("engine", [0, 2, 5])
def test_history_follows_dense_cg(engine):
    """Stronger form of the reference's Krylov-orthogonality check: the
    device's recorded recursive residual norms follow an independent dense
    CG of the same system step by step, and its successive residuals are
    nearly orthogonal."""
    from paper_1010_4639_b200.genprob import poisson2d

    a = poisson2d(6, 6)
    b = np.random.default_rng(6).standard_normal(36)
    rep = _solve(a, b, "csr", engine, record_history=True)
    dense = a.to_dense()
    x, r = np.zeros(36), b.copy()
    p = r.copy()
    rel = []
    for _ in range(rep.iterations):
        q = dense @ p
        alpha = (r @ r) / (p @ q)
        x = x + alpha * p
        r_new = r - alpha * q
        if np.linalg.norm(r_new) > 1e-13:
            cos = abs(r_new @ r) / (np.linalg.norm(r_new) * np.linalg.norm(r))
            assert cos <= 1e-6
        rel.append(np.linalg.norm(r_new) / np.linalg.norm(b))
        beta = (r_new @ r_new) / (r @ r)
        p = r_new + beta * p
        r = r_new
    h = np.asarray(rep.residual_history)
    assert len(h) == rep.iterations
    # early iterations agree to rounding; later ones within the drift of
    # two fp64 CG recurrences at this conditioning
    assert np.allclose(h[:10], rel[:10], rtol=1e-9, atol=0)
    assert np.allclose(h, rel, rtol=1e-4, atol=1e-14)
