"""Cluster-resident engine (engine 5, csrc/clus.cuh) vs the reference's own
CG output: the paper-size FEM matrix in all four storages (16-CTA cluster,
SELL slices partly streamed from L2, DSMEM halo exchange), the solver.py
semantics (x0, max_iter, b = 0, history) and breakdown attribution."""

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


@pytest.mark.parametrize("kind", STORAGES)
def test_fem_mesh_cluster_engine(golden, kind):
    from paper_1010_4639_b200 import CgOptions, cg_solve
    from paper_1010_4639_b200.genprob import fem_mesh

    g = golden("fem")
    m, cfg = as_storage(fem_mesh(), kind)
    r = cg_solve(m, g["F_b"], opts=CgOptions(record_history=True), cfg=cfg, engine=5)
    assert abs(r.iterations - int(g["F_full_it"])) <= 3
    xr = g["F_full_x"]
    assert np.linalg.norm(r.x - xr) / np.linalg.norm(xr) <= 1e-8
    assert r.converged and r.final_relative_residual <= 1e-10
    assert np.allclose(r.residual_history[:50], g["F_full_hist"][:50], rtol=1e-8)


@pytest.mark.parametrize("kind", STORAGES)
def test_cluster_semantics(golden, kind):
    from paper_1010_4639_b200 import CgOptions, cg_solve
    from paper_1010_4639_b200.genprob import poisson3d

    g = golden("cg_small")
    a = poisson3d(12, 12, 12)
    m, cfg = as_storage(a, kind)
    r = cg_solve(m, g["p3_b"], x0=g["p3_x0"], opts=CgOptions(tol=1e-9, record_history=True),
                 cfg=cfg, engine=5)
    assert abs(r.iterations - int(g["p3_it"])) <= 1
    assert np.linalg.norm(r.x - g["p3_x"]) / np.linalg.norm(g["p3_x"]) <= 1e-8
    assert len(r.residual_history) == r.iterations
    t = cg_solve(m, g["p3_b"], x0=g["p3_x0"], opts=CgOptions(max_iter=7, record_history=True,
                                                             recompute_final_residual=False),
                 cfg=cfg, engine=5)
    assert t.iterations == 7 and not t.converged and len(t.residual_history) == 7
    assert abs(t.final_relative_residual - float(g["p3t_final"])) <= 1e-9 * float(g["p3t_final"])
    z = cg_solve(m, np.zeros(a.n), x0=g["p3_x0"], cfg=cfg, engine=5)
    assert z.iterations == 0 and (z.x == 0).all()


def test_cluster_unbanded_random_spd():
    """Random SPD (windows span the whole matrix): every CTA's halo is every
    other CTA's rows; the result must still match the reference CG."""
    from paper_1010_4639_b200 import CgOptions, cg_solve
    from paper_1010_4639_b200.genprob import random_spd

    a = random_spd(3000, 0.004, seed=5)
    rng = np.random.default_rng(3)
    b = rng.standard_normal(a.n)
    ref = O.cg_solve("csr", a.row_start, a.col_idx, a.values, b, tol=1e-10)
    r = cg_solve(a, b, opts=CgOptions(tol=1e-10), engine=5)
    assert abs(r.iterations - ref.iterations) <= max(1, ref.iterations // 100)
    assert np.linalg.norm(r.x - ref.x) / np.linalg.norm(ref.x) <= 1e-8


def test_cluster_breakdowns():
    from paper_1010_4639_b200 import NotPositiveDefiniteError, build_csr_from_triplets, cg_solve

    a = build_csr_from_triplets([(0, 0, 1.0), (1, 1, -1.0)], 2)
    with pytest.raises(NotPositiveDefiniteError, match="not positive definite"):
        cg_solve(a, np.array([1.0, 2.0]), engine=5)
    d = build_csr_from_triplets([(0, 0, 4.0), (1, 1, 3.0), (2, 2, -0.5)], 3)
    b = np.array([1.0, 1.0, 0.1])
    ref = O.cg_solve("csr", d.row_start, d.col_idx, d.values, b)
    assert ref.status == 3
    with pytest.raises(NotPositiveDefiniteError):
        cg_solve(d, b, engine=5)
    # the iteration the breakdown is attributed to (C-ABI) is the reference's
    from paper_1010_4639_b200 import _native as N
    import torch

    lib = N.load()
    bt = torch.from_numpy(b).cuda()
    xt = torch.empty_like(bt)
    o = N.CgOptionsC(tol=1e-10, max_iter=3, record_history=0, recompute_final_residual=1,
                     accumulation=1, engine=5)
    res = N.CgResultC()
    rc = lib.spcg_cg_solve(d.device().handle, bt.data_ptr(), None, xt.data_ptr(), None, o, res,
                           torch.cuda.current_stream().cuda_stream)
    assert rc == 3 and res.status == 3 and res.fail_iteration == ref.fail_iteration


def test_multi_cluster_grid_used_for_paper_matrix():
    """The 30880-row matrix runs on K clusters of 8 (two-level all-reduce,
    inter-cluster halo through global memory); a single 16-CTA cluster run of
    the same system (SPCG_CLUS_K unset would pick the multi-cluster grid) is
    checked by the storage tests above; here: determinism across runs."""
    from paper_1010_4639_b200 import CgOptions, cg_solve
    from paper_1010_4639_b200.genprob import fem_mesh, rhs_for

    F = fem_mesh()
    b, _ = rhs_for(F, seed=1)
    runs = [cg_solve(F, b, opts=CgOptions(record_history=True), engine=5) for _ in range(3)]
    for r in runs[1:]:
        assert r.iterations == runs[0].iterations and (r.x == runs[0].x).all()
        assert np.array_equal(r.residual_history, runs[0].residual_history)


def test_auto_engine_is_cluster_for_small_systems():
    from paper_1010_4639_b200 import cg_solve
    from paper_1010_4639_b200.genprob import fem_mesh, rhs_for

    F = fem_mesh()
    b, _ = rhs_for(F, seed=1)
    r0 = cg_solve(F, b)            # auto: the pipelined cluster engine
    r6 = cg_solve(F, b, engine=6)
    assert r0.iterations == r6.iterations and (r0.x == r6.x).all()  # deterministic
    r5 = cg_solve(F, b, engine=5)
    assert r5.iterations == r6.iterations
    assert np.linalg.norm(r6.x - r5.x) / np.linalg.norm(r5.x) <= 1e-9
    r3 = cg_solve(F, b, engine=3)  # grid-resident single reduction: same method
    assert r3.iterations == r5.iterations
    assert np.linalg.norm(r3.x - r5.x) / np.linalg.norm(r5.x) <= 1e-10


def test_multi_cluster_x0_truncation_and_zero_rhs():
    """The paper-size matrix on the K-cluster grid with the solver.py edge
    semantics: x0 (the initial residual goes through the global scratch
    window), max_iter truncation (history and final residual), b = 0."""
    from paper_1010_4639_b200 import CgOptions, cg_solve
    from paper_1010_4639_b200.genprob import fem_mesh, rhs_for

    F = fem_mesh()
    b, _ = rhs_for(F, seed=1)
    x0 = np.random.default_rng(11).standard_normal(F.n)
    ref = O.cg_solve("csr", F.row_start, F.col_idx, F.values, b, x0=x0, record_history=True)
    r = cg_solve(F, b, x0=x0, opts=CgOptions(record_history=True), engine=5)
    assert abs(r.iterations - ref.iterations) <= 3
    assert np.linalg.norm(r.x - ref.x) / np.linalg.norm(ref.x) <= 1e-8
    assert np.allclose(r.residual_history[:50], ref.residual_history[:50], rtol=1e-8)
    t = cg_solve(F, b, x0=x0, opts=CgOptions(max_iter=25, record_history=True,
                                             recompute_final_residual=False), engine=5)
    rt = O.cg_solve("csr", F.row_start, F.col_idx, F.values, b, x0=x0, max_iter=25,
                    record_history=True, recompute=False)
    assert t.iterations == 25 and not t.converged
    assert np.allclose(t.residual_history, rt.residual_history, rtol=1e-9)
    assert np.linalg.norm(t.x - rt.x) / np.linalg.norm(rt.x) <= 1e-9
    z = cg_solve(F, np.zeros(F.n), x0=x0, engine=5)
    assert z.iterations == 0 and (z.x == 0).all()
