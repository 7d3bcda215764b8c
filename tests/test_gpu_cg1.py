"""Single-reduction (Chronopoulos-Gear) resident engine vs the reference's
own CG output, and the two-reduction resident engine kept selectable."""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

STORAGES = ["csr", "sym_priv", "sym_atomic", "csc"]


def as_storage(a, kind):
    from paper_1010_4639_b200 import KernelConfig, extract_lower

    if kind == "csr":
        return a, KernelConfig()
    if kind == "csc":
        return a.to_csc(), KernelConfig()
    return extract_lower(a), KernelConfig(accumulation="privatized" if kind == "sym_priv"
                                          else "atomic")


@pytest.mark.parametrize("engine", [3])
@pytest.mark.parametrize("kind", STORAGES)
def test_fem_mesh_both_resident_engines(golden, kind, engine):
    from paper_1010_4639_b200 import CgOptions, cg_solve
    from paper_1010_4639_b200.genprob import fem_mesh

    g = golden("fem")
    m, cfg = as_storage(fem_mesh(), kind)
    r = cg_solve(m, g["F_b"], opts=CgOptions(record_history=True), cfg=cfg, engine=engine)
    assert abs(r.iterations - int(g["F_full_it"])) <= 3
    xr = g["F_full_x"]
    assert np.linalg.norm(r.x - xr) / np.linalg.norm(xr) <= 1e-8
    assert r.converged and r.final_relative_residual <= 1e-10
    assert np.allclose(r.residual_history[:50], g["F_full_hist"][:50], rtol=1e-8)


@pytest.mark.parametrize("kind", STORAGES)
def test_single_reduction_semantics(golden, kind):
    from paper_1010_4639_b200 import CgOptions, cg_solve
    from paper_1010_4639_b200.genprob import poisson3d

    g = golden("cg_small")
    a = poisson3d(12, 12, 12)
    m, cfg = as_storage(a, kind)
    r = cg_solve(m, g["p3_b"], x0=g["p3_x0"], opts=CgOptions(tol=1e-9, record_history=True),
                 cfg=cfg, engine=3)
    assert abs(r.iterations - int(g["p3_it"])) <= 1
    assert np.linalg.norm(r.x - g["p3_x"]) / np.linalg.norm(g["p3_x"]) <= 1e-8
    assert len(r.residual_history) == r.iterations
    t = cg_solve(m, g["p3_b"], x0=g["p3_x0"], opts=CgOptions(max_iter=7, record_history=True,
                                                             recompute_final_residual=False),
                 cfg=cfg, engine=3)
    assert t.iterations == 7 and not t.converged and len(t.residual_history) == 7
    assert abs(t.final_relative_residual - float(g["p3t_final"])) <= 1e-9 * float(g["p3t_final"])
    z = cg_solve(m, np.zeros(a.n), x0=g["p3_x0"], cfg=cfg, engine=3)
    assert z.iterations == 0 and (z.x == 0).all()


def test_single_reduction_breakdowns():
    from paper_1010_4639_b200 import NotPositiveDefiniteError, build_csr_from_triplets, cg_solve

    a = build_csr_from_triplets([(0, 0, 1.0), (1, 1, -1.0)], 2)
    with pytest.raises(NotPositiveDefiniteError, match="not positive definite"):
        cg_solve(a, np.array([1.0, 2.0]), engine=3)
    # indefinite but p0.Ap0 > 0: the breakdown appears at a later iteration,
    # which must be the iteration the reference reports
    d = build_csr_from_triplets([(0, 0, 4.0), (1, 1, 3.0), (2, 2, -0.5)], 3)
    b = np.array([1.0, 1.0, 0.1])
    with pytest.raises(NotPositiveDefiniteError):
        cg_solve(d, b, engine=3)
    ref = O.cg_solve("csr", d.row_start, d.col_idx, d.values, b)
    assert ref.status == 3


def test_engine3_is_deterministic():
    from paper_1010_4639_b200 import cg_solve
    from paper_1010_4639_b200.genprob import fem_mesh, rhs_for

    F = fem_mesh()
    b, _ = rhs_for(F, seed=1)
    r1 = cg_solve(F, b, engine=3)
    r2 = cg_solve(F, b, engine=3)
    assert r1.iterations == r2.iterations and (r1.x == r2.x).all()
