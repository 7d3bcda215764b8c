"""The row-sharded (per-pass) engine on one GPU, and the C-side column
localization against the host numbering of distributed.py."""

import ctypes

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("storage", ["csr", "sym"])
def test_per_pass_engine_matches_golden(golden, storage):
    from paper_1010_4639_b200 import CgOptions, KernelConfig, cg_solve, extract_lower
    from paper_1010_4639_b200.genprob import fem_mesh

    g = golden("fem")
    F = fem_mesh()
    m = F if storage == "csr" else extract_lower(F)
    r = cg_solve(m, g["F_b"], opts=CgOptions(record_history=True),
                 cfg=KernelConfig(accumulation="privatized"), engine=2)
    assert abs(r.iterations - int(g["F_full_it"])) <= 3
    assert np.linalg.norm(r.x - g["F_full_x"]) / np.linalg.norm(g["F_full_x"]) <= 1e-8
    assert len(r.residual_history) == r.iterations


def test_per_pass_engine_edge_cases():
    from paper_1010_4639_b200 import (CgOptions, NotPositiveDefiniteError, build_csr_from_triplets,
                                      cg_solve)
    from paper_1010_4639_b200.genprob import poisson3d

    a = poisson3d(9, 8, 7)
    b = np.random.default_rng(2).standard_normal(a.n)
    x0 = np.random.default_rng(3).standard_normal(a.n)
    r = cg_solve(a, b, x0=x0, opts=CgOptions(tol=1e-9), engine=2)
    o = O.cg_solve("csr", a.row_start, a.col_idx, a.values, b, x0=x0, tol=1e-9)
    assert abs(r.iterations - o.iterations) <= 1
    assert np.linalg.norm(r.x - o.x) / np.linalg.norm(o.x) <= 1e-8
    t = cg_solve(a, b, opts=CgOptions(max_iter=5, recompute_final_residual=False), engine=2)
    ot = O.cg_solve("csr", a.row_start, a.col_idx, a.values, b, max_iter=5, recompute=False)
    assert t.iterations == 5 and not t.converged
    assert abs(t.final_relative_residual - ot.final_relative_residual) <= 1e-12
    z = cg_solve(a, np.zeros(a.n), x0=x0, engine=2)
    assert z.iterations == 0 and (z.x == 0).all()
    with pytest.raises(NotPositiveDefiniteError):
        cg_solve(build_csr_from_triplets([(0, 0, 1.0), (1, 1, -1.0)], 2), np.array([1.0, 2.0]),
                 engine=2)


def _rows_handle(a, r0, r1):
    from paper_1010_4639_b200 import _native as N

    rs = np.ascontiguousarray(a.row_start, dtype=np.int64)
    k0, k1 = int(rs[r0]), int(rs[r1])
    ci = np.ascontiguousarray(a.col_idx[k0:k1], dtype=np.int64)
    v = np.ascontiguousarray(a.values[k0:k1])
    p = np.ascontiguousarray(rs[r0:r1 + 1])
    h = ctypes.c_void_p()
    N.check(N.load().spcg_matrix_create_rows(N.FMT_CSR, a.n, r0, r1, v.size, p.ctypes.data,
                                             ci.ctypes.data, v.ctypes.data, 0, None, None, None,
                                             ctypes.byref(h)), "create_rows")
    return h


def test_c_localization_matches_host_numbering():
    from paper_1010_4639_b200 import _native as N
    from paper_1010_4639_b200.device import DeviceMatrix
    from paper_1010_4639_b200.distributed import localize_columns, row_partition
    from paper_1010_4639_b200.genprob import random_spd

    a = random_spd(500, 0.03, 7)
    bnd = row_partition(a.n, 3, a.row_start)
    lib = N.load()
    for rank in range(3):
        r0, r1 = int(bnd[rank]), int(bnd[rank + 1])
        h = _rows_handle(a, r0, r1)
        dm = DeviceMatrix(h.value, N.FMT_CSR, 0, 0)
        dm._refresh()
        nh = ctypes.c_int64()
        N.check(lib.spcg_matrix_localize(dm.handle, ctypes.byref(nh)), "localize")
        halo = np.empty(nh.value, dtype=np.int64)
        N.check(lib.spcg_matrix_halo(dm.handle, halo.ctypes.data), "halo")
        cols = a.col_idx[a.row_start[r0]:a.row_start[r1]]
        loc, hh = localize_columns(cols, r0, r1)
        assert (halo == hh).all()
        off, idx, val = dm.download()
        assert (idx == loc).all()
        # y_loc = A_loc x_ext equals the rows of the global product, bitwise
        x = np.random.default_rng(rank).standard_normal(a.n)
        import torch

        x_ext = torch.from_numpy(np.concatenate([x[r0:r1], x[halo]])).cuda()
        y = torch.empty(r1 - r0, dtype=torch.float64, device="cuda")
        N.check(lib.spcg_spmv(dm.handle, x_ext.data_ptr(), y.data_ptr(), 1, 0), "spmv")
        ref = O.spmv_full(a.row_start, a.col_idx, a.values, x)[r0:r1]
        assert (y.cpu().numpy() == ref).all()


def test_generated_rows_match_host_rows():
    from paper_1010_4639_b200 import _native as N
    from paper_1010_4639_b200.device import DeviceMatrix
    from paper_1010_4639_b200.distributed import localize_columns
    from paper_1010_4639_b200.genprob import poisson3d

    dims = (9, 7, 8)
    a = poisson3d(*dims)
    r0, r1 = 2 * 63, 5 * 63
    h = ctypes.c_void_p()
    N.check(N.load().spcg_matrix_generate_rows(N.GEN_POISSON3D, N.FMT_CSR, *dims, r0, r1,
                                               ctypes.byref(h)), "generate_rows")
    dm = DeviceMatrix(h.value, N.FMT_CSR, 0, 0)
    dm._refresh()
    off, idx, val = dm.download()
    k0, k1 = a.row_start[r0], a.row_start[r1]
    assert (off == a.row_start[r0:r1 + 1] - k0).all()
    assert (idx == a.col_idx[k0:k1]).all() and (val == a.values[k0:k1]).all()
    nh = ctypes.c_int64()
    N.check(N.load().spcg_matrix_localize(dm.handle, ctypes.byref(nh)), "localize")
    _, halo = localize_columns(a.col_idx[k0:k1], r0, r1)
    assert nh.value == halo.size == 2 * 63


def test_sharded_world1_solve():
    import torch

    from paper_1010_4639_b200.distributed import Comm, ShardedMatrix, dist_cg_solve
    from paper_1010_4639_b200.genprob import poisson3d, rhs_for

    a = poisson3d(16, 16, 16)
    b, _ = rhs_for(a, seed=1)
    sm = ShardedMatrix.from_stencil("poisson3d", (16, 16, 16), "csr", 0, 1, lambda o: [o])
    comm = Comm(0, 1)
    x, res, hist = dist_cg_solve(sm, comm, torch.from_numpy(b).cuda(), record_history=True)
    o = O.cg_solve("csr", a.row_start, a.col_idx, a.values, b)
    assert res.iterations == o.iterations
    assert np.linalg.norm(x.cpu().numpy() - o.x) / np.linalg.norm(o.x) <= 1e-8
    assert len(hist) == res.iterations


@pytest.mark.parametrize("accumulation", ["privatized", "atomic"])
def test_sharded_world1_symmetric_rows(accumulation):
    """Symmetric-half row blocks (generated 27-point stencil, L+D and L^T
    rows) through the sharded engine at world 1, both accumulation modes
    (atomic: reverse-halo path with no peers)."""
    import torch

    from paper_1010_4639_b200.distributed import Comm, ShardedMatrix, dist_cg_solve
    from paper_1010_4639_b200.genprob import rhs_for, stencil27

    a = stencil27(12, 10, 9)  # full matrix (the shards generate L+D / L^T rows)
    b, _ = rhs_for(a, seed=2)
    sm = ShardedMatrix.from_stencil("stencil27", (12, 10, 9), "scsr", 0, 1, lambda o: [o])
    comm = Comm(0, 1)
    x0 = np.random.default_rng(4).standard_normal(a.n)
    x, res, _ = dist_cg_solve(sm, comm, torch.from_numpy(b).cuda(), torch.from_numpy(x0).cuda(),
                              accumulation=accumulation)
    o = O.cg_solve("csr", a.row_start, a.col_idx, a.values, b, x0=x0)
    assert abs(res.iterations - o.iterations) <= 1
    assert np.linalg.norm(x.cpu().numpy() - o.x) / np.linalg.norm(o.x) <= 1e-8
    assert res.final_relative_residual <= 1e-10


_NCCL_SCRIPT = r"""
import sys, json
sys.path.insert(0, {root!r})
import numpy as np, torch
from paper_1010_4639_b200.distributed import Comm, ShardedMatrix, dist_cg_solve
sm = ShardedMatrix.from_stencil("poisson3d", (20, 18, 16), "csr", 0, 1, lambda o: [o])
from paper_1010_4639_b200.genprob import poisson3d, rhs_for
a = poisson3d(20, 18, 16)
b, _ = rhs_for(a, seed=1)
bt = torch.from_numpy(b).cuda()
out = {{}}
for name, nccl in (("none", False), ("nccl", True)):
    comm = Comm(0, 1, nccl=nccl)
    x, res, hist = dist_cg_solve(sm, comm, bt, record_history=True)
    out[name] = dict(x=x.cpu().numpy().tolist(), it=int(res.iterations), hist=hist.tolist(),
                     launches=int(res.kernel_launches))
    comm.close()
print("RESULT " + json.dumps(out))
"""


def test_nccl_one_rank_communicator():
    """A real one-rank NCCL communicator (spcg_comm_create with an id): the
    ncclAllReduce calls of the sharded engine execute on the solve stream
    (NCCL_DEBUG=INFO shows the communicator's bring-up), and the solve is
    bitwise the one without a communicator (a one-rank sum is the value)."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = str(Path(__file__).resolve().parent.parent)
    env = dict(os.environ, NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT,COLL")
    p = subprocess.run([sys.executable, "-c", _NCCL_SCRIPT.format(root=root)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    log = p.stdout + p.stderr
    assert "NCCL INFO" in log and "ncclCommInitRank" in log, log[-3000:]
    assert "AllReduce" in log, log[-3000:]  # COLL subsystem: the engine's all-reduces ran
    res = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("RESULT ")][0][7:])
    a, b = res["none"], res["nccl"]
    assert a["it"] == b["it"] and a["x"] == b["x"] and a["hist"] == b["hist"]
    o = O.cg_solve("csr", *_poisson_arrays(), _rhs())
    assert abs(a["it"] - o.iterations) <= 1


def _poisson_arrays():
    from paper_1010_4639_b200.genprob import poisson3d

    a = poisson3d(20, 18, 16)
    return a.row_start, a.col_idx, a.values


def _rhs():
    from paper_1010_4639_b200.genprob import poisson3d, rhs_for

    return rhs_for(poisson3d(20, 18, 16), seed=1)[0]
