"""§8f rows: the FEM-shaped / random_spd generators assembled in HBM
(genprob.py:96-129 of spcg; spcg_matrix_assemble_pairs) and the .spcg
container loaded straight to HBM with pinned, chunked, double-buffered
copies and device-side conversion (matio.py:171-208;
spcg_matrix_create_device_u32)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _same(dm, host):
    """The device handle's arrays equal the host matrix's, bit for bit."""
    p, i, v = dm.download()
    off = host.col_start if hasattr(host, "col_start") else host.row_start
    idx = host.row_idx if hasattr(host, "row_idx") else host.col_idx
    assert (p == off).all() and (i == idx).all()
    assert (v.view(np.uint64) == np.ascontiguousarray(host.values).view(np.uint64)).all()


@pytest.mark.parametrize("fmt", ["csr", "scsr", "csc"])
def test_fem_mesh_device_is_bitwise_host(fmt):
    from paper_1010_4639_b200 import extract_lower
    from paper_1010_4639_b200.genprob import fem_mesh, fem_mesh_device

    F = fem_mesh()
    host = {"csr": F, "scsr": extract_lower(F), "csc": F.to_csc()}[fmt]
    dm = fem_mesh_device(fmt=fmt)
    assert dm.n == 30880 and dm.nnz == host.nnz
    _same(dm, host)


@pytest.mark.parametrize("n,density,seed", [(30880, 418918 / 30880 ** 2, 1), (1, 0.5, 2),
                                            (7, 0.9, 3), (2000, 0.01, 4)])
def test_random_spd_device_is_bitwise_host(n, density, seed):
    from paper_1010_4639_b200 import extract_lower
    from paper_1010_4639_b200.genprob import random_spd, random_spd_device

    A = random_spd(n, density, seed)
    _same(random_spd_device(n, density, seed), A)
    _same(random_spd_device(n, density, seed, fmt="scsr"), extract_lower(A))


def test_device_generated_scsr_lt_matches_host_upload():
    """The device-built L^T (privatized mode) gives the host upload's SpMV
    bit for bit, and the CG solve on the generated handle is the host one's."""
    import torch

    from paper_1010_4639_b200 import _native as N
    from paper_1010_4639_b200 import extract_lower
    from paper_1010_4639_b200.genprob import fem_mesh, fem_mesh_device, rhs_for

    F = fem_mesh()
    S = extract_lower(F)
    dh, dd = S.device(), fem_mesh_device(fmt="scsr")
    x = torch.from_numpy(np.random.default_rng(1).standard_normal(F.n)).cuda()
    y1, y2 = torch.empty_like(x), torch.empty_like(x)
    lib = N.load()
    N.check(lib.spcg_spmv(dh.handle, x.data_ptr(), y1.data_ptr(), N.ACC_PRIVATIZED, 0), "a")
    N.check(lib.spcg_spmv(dd.handle, x.data_ptr(), y2.data_ptr(), N.ACC_PRIVATIZED, 0), "b")
    assert torch.equal(y1, y2)
    b, _ = rhs_for(F, seed=1)
    bt = torch.from_numpy(b).cuda()
    outs = []
    for dm in (dh, dd):
        xo = torch.empty_like(bt)
        o = N.CgOptionsC(tol=1e-10, max_iter=0, record_history=0, recompute_final_residual=1,
                         accumulation=1, engine=5)
        r = N.CgResultC()
        N.check(lib.spcg_cg_solve(dm.handle, bt.data_ptr(), None, xo.data_ptr(), None, o, r, 0), "s")
        outs.append((r.iterations, xo.cpu().numpy()))
    assert outs[0][0] == outs[1][0] and (outs[0][1] == outs[1][1]).all()


def test_assemble_rejects_bad_pairs():
    from paper_1010_4639_b200.device import DeviceMatrix

    with pytest.raises(ValueError):  # J >= I
        DeviceMatrix.from_pairs(4, np.array([1, 2]), np.array([1, 0]), np.array([-1.0, -1.0]), 1.0)
    with pytest.raises(ValueError):  # duplicate pair
        DeviceMatrix.from_pairs(4, np.array([2, 2]), np.array([0, 0]), np.array([-1.0, -1.0]), 1.0)


@pytest.mark.parametrize("storage", ["csr", "sym", "csc"])
def test_read_system_device_pinned_chunked(tmp_path, storage):
    from paper_1010_4639_b200 import extract_lower
    from paper_1010_4639_b200.genprob import poisson2d, rhs_for
    from paper_1010_4639_b200.matio import LinearSystem, read_system_device, write_system

    a = poisson2d(300, 300)  # 5.4 MB payload: several 1 MiB chunks through both buffers
    b, xg = rhs_for(a, seed=4)
    m = {"csr": a, "sym": extract_lower(a), "csc": a.to_csc()}[storage]
    p = tmp_path / f"s_{storage}.spcg"
    write_system(LinearSystem(matrix=m, b=b, x_ref=xg), p)
    dm, bd, xd = read_system_device(p, chunk_bytes=1 << 20)
    _same(dm, m)
    assert (bd == b).all() and (xd == xg).all()
    dm2, bt, xt = read_system_device(p, device_vectors=True)
    assert bt.is_cuda and (bt.cpu().numpy() == b).all()


def test_read_system_device_rejects_corrupt_files(tmp_path):
    from paper_1010_4639_b200.genprob import poisson2d
    from paper_1010_4639_b200.matio import (FileFormatError, LinearSystem, read_system_device,
                                            write_system)

    a = poisson2d(5, 5)
    p = tmp_path / "a.spcg"
    write_system(LinearSystem(matrix=a, b=np.ones(a.n)), p)
    raw = p.read_bytes()
    (tmp_path / "t.spcg").write_bytes(raw[:-8])
    with pytest.raises(FileFormatError):
        read_system_device(tmp_path / "t.spcg")
    (tmp_path / "m.spcg").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(FileFormatError):
        read_system_device(tmp_path / "m.spcg")
    # offsets that are not monotone: rejected by the device-side checks
    bad = bytearray(raw)
    bad[24 + 8 * 3: 24 + 8 * 4] = (10 ** 6).to_bytes(8, "little")
    (tmp_path / "o.spcg").write_bytes(bytes(bad))
    with pytest.raises(ValueError):
        read_system_device(tmp_path / "o.spcg")
