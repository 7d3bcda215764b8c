"""Engine 7 (csrc/cg1.cuh cg1s_kernel): the single-reduction CG of engine 3
in one persistent kernel that streams the tiles every iteration.  The
solver.py edge semantics against the reference goldens (x0, b = 0,
truncation with the recursive residual, history), breakdown attribution
like the reference, a system larger than the chip's resident tiles against
the reference CG, repeatability, and the gather-format restriction."""

import numpy as np
import pytest

from oracle import oracle as O

from test_gpu_clus import as_storage

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind", ["csr", "sym_priv"])
def test_engine7_semantics(golden, kind):
    from paper_1010_4639_b200 import CgOptions, cg_solve
    from paper_1010_4639_b200.genprob import poisson3d

    g = golden("cg_small")
    a = poisson3d(12, 12, 12)
    m, cfg = as_storage(a, kind)
    r = cg_solve(m, g["p3_b"], x0=g["p3_x0"], opts=CgOptions(tol=1e-9, record_history=True),
                 cfg=cfg, engine=7)
    assert r.engine_info["engine"] == 7
    assert abs(r.iterations - int(g["p3_it"])) <= 1
    assert np.linalg.norm(r.x - g["p3_x"]) / np.linalg.norm(g["p3_x"]) <= 1e-8
    assert len(r.residual_history) == r.iterations
    t = cg_solve(m, g["p3_b"], x0=g["p3_x0"], opts=CgOptions(max_iter=7, record_history=True,
                                                             recompute_final_residual=False),
                 cfg=cfg, engine=7)
    assert t.iterations == 7 and not t.converged and len(t.residual_history) == 7
    assert abs(t.final_relative_residual - float(g["p3t_final"])) <= 1e-9 * float(g["p3t_final"])
    z = cg_solve(m, np.zeros(a.n), x0=g["p3_x0"], cfg=cfg, engine=7)
    assert z.iterations == 0 and z.converged and (z.x == 0).all()
    # x0 already converged: 0 iterations (solver.py:128-131)
    c = cg_solve(m, g["p3_b"], x0=r.x, opts=CgOptions(tol=1e-6), cfg=cfg, engine=7)
    assert c.iterations == 0 and c.converged


def test_engine7_breakdowns():
    from paper_1010_4639_b200 import NotPositiveDefiniteError, build_csr_from_triplets, cg_solve

    a = build_csr_from_triplets([(0, 0, 1.0), (1, 1, -1.0)], 2)
    with pytest.raises(NotPositiveDefiniteError, match="not positive definite"):
        cg_solve(a, np.array([1.0, 2.0]), engine=7)
    d = build_csr_from_triplets([(0, 0, 4.0), (1, 1, 3.0), (2, 2, -0.5)], 3)
    b = np.array([1.0, 1.0, 0.1])
    ref = O.cg_solve("csr", d.row_start, d.col_idx, d.values, b)
    assert ref.status == 3
    import torch

    from paper_1010_4639_b200 import _native as N

    bt = torch.from_numpy(b).cuda()
    xt = torch.empty_like(bt)
    o = N.CgOptionsC(tol=1e-10, max_iter=3, record_history=0, recompute_final_residual=1,
                     accumulation=1, engine=7)
    res = N.CgResultC()
    rc = N.load().spcg_cg_solve(d.device().handle, bt.data_ptr(), None, xt.data_ptr(), None, o,
                                res, torch.cuda.current_stream().cuda_stream)
    assert rc == 3 and res.status == 3 and res.fail_iteration == ref.fail_iteration


def test_engine7_streamed_system_repeatable():
    """A system whose tiles do not fit on chip (more tiles than the
    co-resident CTAs hold): reference iterations, x within 1e-8 of the
    reference CG, bitwise repeatable run to run."""
    from paper_1010_4639_b200 import CgOptions, cg_solve
    from paper_1010_4639_b200.genprob import poisson3d, rhs_for

    a = poisson3d(48, 48, 64)
    b, _ = rhs_for(a, seed=6)
    assert a.device().info()["ntiles"] > 2 * 148
    ref = O.cg_solve("csr", a.row_start, a.col_idx, a.values, b, record_history=True)
    r1 = cg_solve(a, b, opts=CgOptions(record_history=True), engine=7)
    r2 = cg_solve(a, b, opts=CgOptions(record_history=True), engine=7)
    assert abs(r1.iterations - ref.iterations) <= max(1, ref.iterations // 100)
    assert np.linalg.norm(r1.x - ref.x) / np.linalg.norm(ref.x) <= 1e-8
    assert np.allclose(r1.residual_history[:50], ref.residual_history[:50], rtol=1e-8)
    assert r1.iterations == r2.iterations and np.array_equal(r1.x, r2.x)


@pytest.mark.parametrize("kind", ["sym_atomic", "csc"])
def test_engine7_rejects_scatter_formats(kind):
    from paper_1010_4639_b200 import cg_solve
    from paper_1010_4639_b200.genprob import poisson2d

    a = poisson2d(16, 16)
    m, cfg = as_storage(a, kind)
    with pytest.raises(Exception, match="gather formats"):
        cg_solve(m, np.ones(a.n), cfg=cfg, engine=7)
