"""BASELINE.json's full-size configurations on the B200, checked against the
reference's own golden runs (compiled reference backend,
tol 1e-10, x0 = 0, b = A x_gen with x_gen = default_rng(1).standard_normal(n)):
P2 4096^2 -> 7,387 iterations, P3 400^3 -> 944, Q27 256^3 (symmetric half) ->
457.  The reference's x is not stored at these sizes, so the size-independent
properties are checked instead: the iteration count (+-1 %), the true relative
residual, the error against x_gen (the survey's 3.1e-6 / 1.4e-7 level), and
that every storage of the same operator gives the same SpMV to 1e-12."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _system(kind, dims, fmt):
    import torch

    from paper_1010_4639_b200 import _native as N
    from paper_1010_4639_b200.device import DeviceMatrix

    dm = DeviceMatrix.generate(kind, dims, fmt)
    full = dm if fmt == "csr" else DeviceMatrix.generate(kind, dims, "csr")
    xg = torch.from_numpy(np.random.default_rng(1).standard_normal(dm.n)).cuda()
    b = torch.empty_like(xg)
    N.check(N.load().spcg_spmv(full.handle, xg.data_ptr(), b.data_ptr(), N.ACC_PRIVATIZED, 0), "b")
    return dm, full, xg, b


def _solve(dm, b, acc):
    import torch

    from paper_1010_4639_b200 import _native as N

    x = torch.empty_like(b)
    o = N.CgOptionsC(tol=1e-10, max_iter=0, record_history=0, recompute_final_residual=1,
                     accumulation=acc, engine=0)
    r = N.CgResultC()
    N.check(N.load().spcg_cg_solve(dm.handle, b.data_ptr(), None, x.data_ptr(), None, o, r, 0),
            "solve")
    return x, r


@pytest.mark.parametrize("kind,dims,ref_its,err_bound", [
    ("poisson2d", (4096, 4096), 7387, 1e-5),
    ("poisson3d", (400, 400, 400), 944, 1e-6),
])
def test_poisson_full_size(kind, dims, ref_its, err_bound):
    import torch

    dm, _, xg, b = _system(kind, dims, "csr")
    x, r = _solve(dm, b, 1)
    assert abs(r.iterations - ref_its) <= max(1, ref_its // 100)
    assert r.converged and r.final_relative_residual <= 1e-10
    err = float(torch.linalg.norm(x - xg) / torch.linalg.norm(xg))
    assert err <= err_bound, err


def test_q27_full_size_both_accumulations():
    import torch

    from paper_1010_4639_b200 import _native as N

    dm, full, xg, b = _system("stencil27", (256, 256, 256), "scsr")
    lib = N.load()
    # SpMV: privatized SCSR and atomic SCSR against the full CSR of the same operator
    y_full = torch.empty_like(xg)
    y_priv = torch.empty_like(xg)
    y_atom = torch.empty_like(xg)
    N.check(lib.spcg_spmv(full.handle, xg.data_ptr(), y_full.data_ptr(), 1, 0), "full")
    N.check(lib.spcg_spmv(dm.handle, xg.data_ptr(), y_priv.data_ptr(), 1, 0), "priv")
    N.check(lib.spcg_spmv(dm.handle, xg.data_ptr(), y_atom.data_ptr(), 0, 0), "atom")
    scale = float(torch.linalg.norm(y_full, ord=float("inf")))
    assert float((y_priv - y_full).abs().max()) <= 1e-12 * scale
    assert float((y_atom - y_full).abs().max()) <= 1e-12 * scale
    xs = []
    for acc in (1, 0):
        x, r = _solve(dm, b, acc)
        assert abs(r.iterations - 457) <= 4
        assert r.converged and r.final_relative_residual <= 1e-10
        assert float(torch.linalg.norm(x - xg) / torch.linalg.norm(xg)) <= 1e-6
        xs.append(x)
    assert float(torch.linalg.norm(xs[0] - xs[1]) / torch.linalg.norm(xs[0])) <= 1e-8
