"""The oracle is pinned against golden vectors produced by the reference
package itself (scripts/make_golden.py) before anything is compared to it."""

import numpy as np
import pytest

from oracle import oracle as O


def test_spmv_full_bitwise_vs_reference(golden):
    g = golden("kernels_small")
    for i in range(int(g["ncases"])):
        y = O.spmv_full(g[f"c{i}_rs"], g[f"c{i}_ci"], g[f"c{i}_v"], g[f"c{i}_x"], workers=3)
        assert (y == g[f"c{i}_y"]).all(), i


def test_spmv_sym_privatized_bitwise_vs_reference(golden):
    g = golden("kernels_small")
    for i in range(int(g["nsym"])):
        y = O.spmv_sym(g[f"s{i}_rs"], g[f"s{i}_ci"], g[f"s{i}_v"], g[f"s{i}_x"],
                       accumulation="privatized", workers=1)
        assert (y == g[f"s{i}_ypriv1"]).all(), i
        ya = O.spmv_sym(g[f"s{i}_rs"], g[f"s{i}_ci"], g[f"s{i}_v"], g[f"s{i}_x"],
                        accumulation="atomic")
        ref = g[f"s{i}_yatom"]
        assert np.max(np.abs(ya - ref), initial=0) <= 1e-12 * max(1, np.max(np.abs(ref), initial=0))


def test_dot_axpy_vs_reference(golden):
    g = golden("kernels_small")
    for i in range(int(g["ncases"])):
        x = g[f"c{i}_x"]
        assert O.dot(x, x, workers=1) == float(g[f"c{i}_dot"])
        assert (O.axpy(1.7, x, x[::-1].copy()) == g[f"c{i}_axpy"]).all()


def test_pairwise_merge_and_edges():
    assert O.dot(np.zeros(0), np.zeros(0)) == 0.0
    assert O.dot(np.ones(1000), np.ones(1000), workers=8) == 1000.0
    u = np.random.default_rng(3).standard_normal(33)
    assert (O.axpy(-1.0, u, u.copy()) == 0).all()
    assert (O.axpy(0.0, u, u[::-1].copy()) == u[::-1]).all()


def test_cg_matches_reference_cg(golden):
    g = golden("cg_small")
    from paper_1010_4639_b200.genprob import poisson2d, poisson3d
    from paper_1010_4639_b200.core import extract_lower

    a = poisson2d(32, 32)
    r = O.cg_solve("csr", a.row_start, a.col_idx, a.values, g["p2_b"], max_iter=1029,
                   record_history=True)
    assert r.iterations == int(g["p2_full_it"])
    assert (r.x == g["p2_full_x"]).all()  # same op order, same kernels: bitwise
    assert r.residual_history == list(g["p2_full_hist"])
    s = extract_lower(a)
    r = O.cg_solve("sym", s.row_start, s.col_idx, s.values, g["p2_b"], max_iter=1029,
                   record_history=True, accumulation="privatized")
    assert r.iterations == int(g["p2_sym_it"])
    assert (r.x == g["p2_sym_x"]).all()
    a3 = poisson3d(12, 12, 12)
    r = O.cg_solve("csr", a3.row_start, a3.col_idx, a3.values, g["p3_b"], x0=g["p3_x0"], tol=1e-9)
    assert r.iterations == int(g["p3_it"]) and (r.x == g["p3_x"]).all()
    r = O.cg_solve("csr", a3.row_start, a3.col_idx, a3.values, g["p3_b"], x0=g["p3_x0"],
                   max_iter=7, recompute=False)
    assert r.iterations == 7 and not r.converged
    assert r.final_relative_residual == float(g["p3t_final"])


def test_cg_fem_mesh_matches_reference(golden):
    from paper_1010_4639_b200.genprob import fem_mesh

    g = golden("fem")
    F = fem_mesh()
    assert F.nnz == int(g["F_nnz"]) == 449_798
    r = O.cg_solve("csr", F.row_start, F.col_idx, F.values, g["F_b"], workers=1)
    assert r.iterations == int(g["F_full_it"]) == 329
    assert (r.x == g["F_full_x"]).all()


def test_reference_kernels_drive_same_cg(golden):
    ck = O.load_ref()
    if ck is None:
        pytest.skip("oracle/_ref not built")
    from paper_1010_4639_b200.genprob import poisson2d

    g = golden("cg_small")
    a = poisson2d(32, 32)
    r = O.cg_solve_ref("csr", a.row_start, a.col_idx, a.values, g["p2_b"], max_iter=1029)
    assert r.iterations == int(g["p2_full_it"]) and (r.x == g["p2_full_x"]).all()


def test_stencil_generator_matches_host_generators():
    from paper_1010_4639_b200.genprob import poisson2d, poisson3d, stencil27

    for kind, dims, ref in [("poisson2d", (6, 5), poisson2d(6, 5)),
                            ("poisson3d", (4, 5, 3), poisson3d(4, 5, 3)),
                            ("stencil27", (4, 3, 5), stencil27(4, 3, 5))]:
        rs, ci, v = O.stencil(kind, dims)
        assert (rs == ref.row_start).all() and (ci == ref.col_idx).all() and (v == ref.values).all()
    s = stencil27(3, 4, 5, part="lower")
    rs, ci, v = O.stencil("stencil27", (3, 4, 5), part="lower")
    assert (rs == s.row_start).all() and (ci == s.col_idx).all() and (v == s.values).all()
