"""Host logic (no GPU): the C-ABI library loads and exports the header's
symbols, host storage types / loaders / generators behave like the
reference's, and the product refuses to run without a device (no CPU
fallback)."""

import os
import re

import numpy as np
import pytest

from conftest import HAS_GPU, ROOT


def test_library_exports_every_header_symbol():
    from paper_1010_4639_b200 import _native as N

    header = N.HEADER_PATH.read_text()
    declared = set(re.findall(r"^\s*(?:int|const char\*)\s+(spcg_\w+)\s*\(", header, re.M))
    assert declared == set(N.SIGNATURES), declared ^ set(N.SIGNATURES)
    lib = N.load()
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.spcg_abi_version() == 2


@pytest.mark.skipif(HAS_GPU, reason="checks the no-device failure mode")
def test_no_cpu_fallback_without_device():
    from paper_1010_4639_b200 import cg_solve
    from paper_1010_4639_b200._native import NativeUnavailableError
    from paper_1010_4639_b200.genprob import poisson2d

    with pytest.raises(NativeUnavailableError):
        cg_solve(poisson2d(3, 3), np.ones(9))


def test_generators_match_reference_bitwise(golden):
    from paper_1010_4639_b200.genprob import poisson2d, poisson3d, random_spd

    g = golden("generators")
    for name, a in [("p2", poisson2d(5, 7)), ("p3", poisson3d(4, 3, 5)),
                    ("rs", random_spd(40, 0.2, 3)), ("rs2", random_spd(7, 1.0, 9))]:
        assert (a.row_start == g[f"{name}_rs"]).all(), name
        assert (a.col_idx == g[f"{name}_ci"]).all(), name
        assert (a.values == g[f"{name}_v"]).all(), name


def test_fem_mesh_shape(golden):
    from paper_1010_4639_b200 import is_symmetric
    from paper_1010_4639_b200.genprob import fem_mesh

    g = golden("fem")
    F = fem_mesh()
    assert (F.n, F.nnz) == (30880, 449798)
    assert F.values.sum() == float(g["F_vsum"])
    assert int(F.col_idx.sum()) == int(g["F_colsum"])
    lens = np.diff(F.row_start)
    assert lens.min() >= 4 and lens.max() <= 27
    assert is_symmetric(F)


def two_by_two():
    from paper_1010_4639_b200 import build_csr_from_triplets

    return build_csr_from_triplets([(0, 0, 4.0), (0, 1, 1.0), (1, 0, 1.0), (1, 1, 3.0)], 2)


class TestCore:
    def test_triplets(self):
        from paper_1010_4639_b200 import build_csr_from_triplets
        from paper_1010_4639_b200.core import MatrixConstructionError

        m = two_by_two()
        assert list(m.row_start) == [0, 2, 4] and list(m.col_idx) == [0, 1, 0, 1]
        assert build_csr_from_triplets([], 3).nnz == 0
        assert build_csr_from_triplets([(0, 0, 1.0), (0, 0, 2.0)], 1).values[0] == 3.0
        with pytest.raises(MatrixConstructionError, match=r"\(0, 5,"):
            build_csr_from_triplets([(0, 5, 1.0)], 2)
        z = [(0, 1, 0.0), (0, 0, 1.0), (1, 1, 1.0)]
        assert build_csr_from_triplets(z, 2).nnz == 3
        assert build_csr_from_triplets(z, 2, drop_zeros=True).nnz == 2

    def test_validate(self):
        from paper_1010_4639_b200 import CsrMatrix, validate_csr

        assert validate_csr(two_by_two()).ok
        bad = CsrMatrix(n=2, row_start=np.array([0, 2, 1]), col_idx=np.array([0, 1]),
                        values=np.array([1.0, 2.0]))
        assert any(r == "offsets-monotone" for r, _, _ in validate_csr(bad).violations)
        unsorted = CsrMatrix(n=2, row_start=np.array([0, 2, 2]), col_idx=np.array([1, 0]),
                             values=np.array([1.0, 2.0]))
        assert any(r == "col-order" for r, _, _ in validate_csr(unsorted).violations)

    def test_symmetry_and_half_storage(self):
        from paper_1010_4639_b200 import (SymHalfMatrix, build_csr_from_triplets,
                                          expand_symmetric, extract_lower, is_symmetric)
        from paper_1010_4639_b200.core import (AsymmetricMatrixError, MatrixConstructionError,
                                               MissingDiagonalError)
        from paper_1010_4639_b200.genprob import poisson2d, random_spd

        assert is_symmetric(two_by_two())
        m = build_csr_from_triplets([(0, 0, 4.0), (0, 1, 1.0), (1, 0, 1.0 + 5e-13), (1, 1, 3.0)], 2)
        assert is_symmetric(m, tol=1e-12) and not is_symmetric(m, tol=1e-13)
        s = extract_lower(two_by_two())
        assert list(s.row_start) == [0, 1, 3] and list(s.values) == [4.0, 1.0, 3.0]
        a = poisson2d(3, 3)
        assert extract_lower(a).nnz == 21
        with pytest.raises(AsymmetricMatrixError, match=r"\(0, 1\)"):
            extract_lower(build_csr_from_triplets([(0, 0, 1.0), (0, 1, 2.0), (1, 1, 1.0)], 2))
        with pytest.raises(MissingDiagonalError, match="row 1"):
            extract_lower(build_csr_from_triplets([(0, 0, 1.0), (1, 2, 1.0), (2, 1, 1.0)], 3))
        with pytest.raises((MatrixConstructionError, MissingDiagonalError)):
            SymHalfMatrix(n=2, row_start=np.array([0, 2, 3]), col_idx=np.array([0, 1, 1]),
                          values=np.ones(3))
        rng = np.random.default_rng(11)
        for _ in range(20):
            r = random_spd(int(rng.integers(1, 40)), 0.2, int(rng.integers(1 << 30)))
            e = expand_symmetric(extract_lower(r))
            assert (e.row_start == r.row_start).all() and (e.values == r.values).all()

    def test_csc_round_trip(self):
        from paper_1010_4639_b200.genprob import random_spd

        from conftest import random_csr

        rng = np.random.default_rng(2)
        a = random_csr(rng, 30, 0.2)
        c = a.to_csc()
        assert (c.to_dense() == a.to_dense()).all()
        back = c.to_csr()
        assert (back.col_idx == a.col_idx).all() and (back.values == a.values).all()
        s = random_spd(25, 0.3, 4)
        cs = s.to_csc()
        assert (cs.col_start == s.row_start).all() and (cs.row_idx == s.col_idx).all()

    def test_immutability(self):
        m = two_by_two()
        with pytest.raises(ValueError):
            m.values[0] = 1.0


class TestMatio:
    def test_spcg_round_trip_all_storages(self, tmp_path):
        from paper_1010_4639_b200 import extract_lower
        from paper_1010_4639_b200.genprob import random_spd
        from paper_1010_4639_b200.matio import LinearSystem, read_system, write_system

        rng = np.random.default_rng(1008)
        for seed in range(30):
            n = int(rng.integers(1, 40))
            a = random_spd(n, 0.3, seed)
            m = [a, extract_lower(a), a.to_csc()][seed % 3]
            sys_ = LinearSystem(matrix=m, b=rng.standard_normal(n),
                                x_ref=rng.standard_normal(n) if seed % 2 else None)
            p = tmp_path / f"s{seed}.spcg"
            write_system(sys_, p)
            back = read_system(p)
            assert type(back.matrix) is type(m)
            assert (back.matrix.values == m.values).all()
            assert (back.b == sys_.b).all()
            assert (back.x_ref is None) == (sys_.x_ref is None)

    def test_matrix_market(self, tmp_path):
        from paper_1010_4639_b200 import CscMatrix, SymHalfMatrix, expand_symmetric, extract_lower
        from paper_1010_4639_b200.genprob import random_spd
        from paper_1010_4639_b200.matio import (FileFormatError, UnsupportedFormatError,
                                                read_matrix_market, write_matrix_market)

        a = random_spd(25, 0.25, 555)
        gp, sp = tmp_path / "g.mtx", tmp_path / "s.mtx"
        write_matrix_market(a, gp)
        write_matrix_market(extract_lower(a), sp)
        s = read_matrix_market(sp)
        assert isinstance(s, SymHalfMatrix)
        e = expand_symmetric(s)
        g = read_matrix_market(gp)
        assert (e.col_idx == g.col_idx).all() and np.max(np.abs(e.values - g.values)) <= 1e-15
        c = read_matrix_market(gp, as_csc=True)
        assert isinstance(c, CscMatrix) and (c.to_dense() == g.to_dense()).all()
        bad = tmp_path / "z.mtx"
        bad.write_text("%%MatrixMarket matrix coordinate real general\n0 0 0\n")
        with pytest.raises(FileFormatError, match="degenerate"):
            read_matrix_market(bad)
        cx = tmp_path / "c.mtx"
        cx.write_text("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1.0\n")
        with pytest.raises(UnsupportedFormatError):
            read_matrix_market(cx)


def test_kernel_config_and_backend():
    from paper_1010_4639_b200 import KernelConfig
    from paper_1010_4639_b200 import kernels

    with pytest.raises(ValueError):
        KernelConfig(workers=0)
    with pytest.raises(ValueError):
        KernelConfig(chunk=0)
    with pytest.raises(ValueError):
        KernelConfig(accumulation="racy")
    assert KernelConfig(workers=2).resolve_chunk(160) == 10
    assert kernels.available_backends() == ("cuda",)
    be = kernels.set_backend("auto")
    assert be.name == "cuda" and kernels.get_backend() == "cuda"
    # the reference's backend names select the one device backend
    for alias in ("compiled", "python", "cuda"):
        assert kernels.set_backend(alias) is be
        assert kernels.BACKENDS[alias] is be
    for fn in ("spmv_full", "spmv_sym", "dot", "axpy"):
        assert callable(getattr(be, fn))
    with pytest.raises(ValueError):
        kernels.set_backend("numba")
    assert kernels.pairwise_merge(np.array([1.0, 2.0, 3.0, 4.0, 5.0])) == 15.0


def test_cg_options_and_convergence():
    from paper_1010_4639_b200 import CgOptions, check_convergence

    with pytest.raises(ValueError):
        CgOptions(tol=0)
    with pytest.raises(ValueError):
        CgOptions(max_iter=0)
    assert check_convergence(0.0, 0.0, CgOptions())
    assert not check_convergence(1e-300, 0.0, CgOptions())
    assert check_convergence(5e-10, 10.0, CgOptions(tol=1e-10))


def test_spcg_backend_env_is_honoured():
    """SPCG_BACKEND (kernels/__init__.py:50) is read at import: a reference
    name selects the device backend, an unknown one fails the import."""
    import subprocess
    import sys

    code = "import paper_1010_4639_b200.kernels as k; print(k.get_backend())"
    for name, ok in (("compiled", True), ("python", True), ("bogus", False)):
        p = subprocess.run([sys.executable, "-c", code], cwd=str(ROOT),
                           env={**os.environ, "SPCG_BACKEND": name}, capture_output=True, text=True)
        assert (p.returncode == 0) == ok, p.stderr
        if ok:
            assert p.stdout.strip() == "cuda"
        else:
            assert "unknown backend" in p.stderr


def test_bench_report_schema_round_trips():
    """The Table-I report keeps the reference's schema (spcg bench.py:27-128)."""
    from paper_1010_4639_b200.table1 import BenchReport, CgTiming, OpTiming

    rep = BenchReport(meta={"n": 9, "nnz_full": 33, "nnz_sym": 21, "storage_kind": "full",
                            "backend": "cuda", "precision": "float64", "accumulation": "atomic",
                            "reps": 3, "load_time_ms": 0.5},
                      ops=[OpTiming("dotProd", 1, 0.0123, 1.0), OpTiming("SpMV", 1, 0.02, 1.0)],
                      cg=[CgTiming("full", 1, 1.5, 7, True, 3.2e-11, 1.0),
                          CgTiming("sym", 1, 1.7, 7, False, 2.0e-9, 1.0)])
    assert BenchReport.from_json(rep.to_json()) == rep
    assert BenchReport.from_csv(rep.to_csv()) == rep
    txt = rep.to_text()
    assert "CG/ # int (full)" in txt and "[NOT CONVERGED]" in txt and "workers=1" in txt


def test_csc_container_carries_its_own_version(tmp_path):
    """CSC .spcg files (new) are VERSION_CSC, so the reference reader (which
    accepts only VERSION and ignores unknown flags) rejects them rather than
    reading the CSC arrays as CSR; this reader round-trips both."""
    import struct

    from paper_1010_4639_b200.genprob import poisson2d
    from paper_1010_4639_b200.matio import (VERSION, VERSION_CSC, FileFormatError, LinearSystem,
                                            read_system, write_system)

    a = poisson2d(4, 3)
    for m, ver in ((a, VERSION), (a.to_csc(), VERSION_CSC)):
        p = tmp_path / f"v{ver}.spcg"
        write_system(LinearSystem(matrix=m, b=np.arange(a.n, dtype=float)), p)
        raw = p.read_bytes()
        assert struct.unpack_from("<I", raw, 4)[0] == ver
        back = read_system(p).matrix
        assert type(back) is type(m) and (back.values == m.values).all()
    # a CSC payload labelled VERSION 1 is refused
    raw = bytearray((tmp_path / f"v{VERSION_CSC}.spcg").read_bytes())
    raw[4:8] = struct.pack("<I", VERSION)
    (tmp_path / "bad.spcg").write_bytes(bytes(raw))
    with pytest.raises(FileFormatError):
        read_system(tmp_path / "bad.spcg")


def _cg_coefficients(ev, b, iters):
    """Textbook CG on diag(ev): (alpha_j, beta_j) with beta_j the coefficient
    that formed p_j (beta_0 = 0)."""
    r = b.copy()
    p = r.copy()
    rr = r @ r
    alpha, beta, prev = [], [], 0.0
    for _ in range(iters):
        ap = ev * p
        a = rr / (p @ ap)
        r -= a * ap
        rn = r @ r
        alpha.append(a)
        beta.append(prev)
        prev = rn / rr
        rr = rn
        p = r + prev * p
        if np.sqrt(rn) < 1e-12 * np.linalg.norm(b):
            break
    return np.array(alpha), np.array(beta)


@pytest.mark.parametrize("n,cond,scale,iters", [
    (500, 10.0, 1.0, 200), (2000, 1e3, 1e-9, 400), (30880, 1e4, 1e12, 329),
    (3000, 1e8, 1.0, 1500), (5000, 2e5, 1.0, 600), (100, 1.0001, 1.0, 50)])
def test_cg_cond_estimate_matches_tridiagonal_eigenvalues(n, cond, scale, iters):
    """The engine-6 guard's Ritz estimate (host multisection over Sturm
    counts, host_cluster.cuh lanczos_cond) equals theta_max / theta_min of
    CG's Lanczos tridiagonal computed by LAPACK, to its stated ~1e-3."""
    from paper_1010_4639_b200._native import cg_cond_estimate

    ev = np.geomspace(1.0, cond, n) * scale
    alpha, beta = _cg_coefficients(ev, np.random.default_rng(n).standard_normal(n), iters)
    d = 1.0 / alpha
    d[1:] += beta[1:] / alpha[:-1]
    e = np.sqrt(beta[1:]) / alpha[:-1]
    w = np.linalg.eigvalsh(np.diag(d) + np.diag(e, 1) + np.diag(e, -1))
    got = cg_cond_estimate(alpha, beta)
    assert abs(got / (w[-1] / w[0]) - 1.0) <= 2e-3, (got, w[-1] / w[0])


def test_cg_cond_estimate_degenerate_inputs():
    from paper_1010_4639_b200._native import cg_cond_estimate

    assert cg_cond_estimate([], []) == 0.0
    assert cg_cond_estimate([0.5], [0.0]) == 0.0
    assert cg_cond_estimate([0.5, -1.0], [0.0, 0.1]) == 0.0  # not positive
    with pytest.raises(ValueError):
        cg_cond_estimate([0.5, 0.4], [0.0])
