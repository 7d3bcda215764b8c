"""Generate tests/golden/*.npz from the REFERENCE package itself.

Run here (the container with /root/reference):  python scripts/make_golden.py
It imports `spcg` from /root/reference/pkg/src, with the reference's own
compiled kernels (oracle/_ref/_ckernels*.so, built by `make -C oracle ref`
from the reference's _ckernels.pyx) installed as spcg.kernels._ckernels so
the "compiled" backend is the one the reference ships.  The fixtures pin the
oracle (tests/test_oracle.py) and the device path (tests/test_gpu_*.py).
"""

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from oracle import oracle as O  # noqa: E402

ck = O.load_ref()
assert ck is not None, "run `make -C oracle ref` first"
sys.modules["spcg.kernels._ckernels"] = ck

import spcg  # noqa: E402
from spcg import genprob, kernels  # noqa: E402
from spcg.core import build_csr_from_triplets, extract_lower  # noqa: E402
from spcg.kernels import KernelConfig  # noqa: E402
from spcg.solver import CgOptions, cg_solve  # noqa: E402

assert "compiled" in kernels.available_backends()
kernels.set_backend("compiled")

from paper_1010_4639_b200 import genprob as mygen  # noqa: E402

OUT = ROOT / "tests" / "golden"
OUT.mkdir(parents=True, exist_ok=True)


def random_csr(rng, n, density):  # reference tests/conftest.py:29-35 recipe
    m = max(1, int(round(density * n * n)))
    rows = rng.integers(0, n, size=m).astype(np.int64)
    cols = rng.integers(0, n, size=m).astype(np.int64)
    vals = rng.standard_normal(m)
    return build_csr_from_triplets((rows, cols, vals), n)


def kernels_small():
    rng = np.random.default_rng(20261018)
    d = {}
    cases = []
    for k in range(40):
        n = int(rng.integers(1, 65))
        a = random_csr(rng, n, float(rng.uniform(0.01, 0.3)))
        cases.append(("rand", a))
    cases.append(("poisson2d_3x3", genprob.poisson2d(3, 3)))
    cases.append(("two_by_two", build_csr_from_triplets(
        [(0, 0, 4.0), (0, 1, 1.0), (1, 0, 1.0), (1, 1, 3.0)], 2)))
    cases.append(("long_rows", random_csr(rng, 300, 0.9)))  # rows > 4096? no: 270 each
    d["ncases"] = np.array(len(cases))
    for i, (name, a) in enumerate(cases):
        x = rng.standard_normal(a.n)
        d[f"c{i}_rs"], d[f"c{i}_ci"], d[f"c{i}_v"], d[f"c{i}_x"] = (
            a.row_start, a.col_idx, a.values, x)
        d[f"c{i}_y"] = kernels.spmv_full(a, x, KernelConfig(workers=4))
        d[f"c{i}_dot"] = np.array(kernels.dot(x, x, KernelConfig(workers=1)))
        d[f"c{i}_axpy"] = kernels.axpy(1.7, x, x[::-1].copy())
    # symmetric cases (criterion 2 style)
    sym = []
    for k in range(30):
        n = int(rng.integers(1, 65))
        sym.append(extract_lower(genprob.random_spd(n, 0.25, 40_000 + k)))
    sym.append(extract_lower(genprob.poisson2d(4, 5)))
    d["nsym"] = np.array(len(sym))
    for i, s in enumerate(sym):
        x = rng.standard_normal(s.n)
        d[f"s{i}_rs"], d[f"s{i}_ci"], d[f"s{i}_v"], d[f"s{i}_x"] = (
            s.row_start, s.col_idx, s.values, x)
        d[f"s{i}_ypriv1"] = kernels.spmv_sym(s, x, KernelConfig(workers=1, accumulation="privatized"))
        d[f"s{i}_yatom"] = kernels.spmv_sym(s, x, KernelConfig(workers=4, accumulation="atomic"))
    np.savez_compressed(OUT / "kernels_small.npz", **d)


def generators():
    d = {}
    for name, a in [("p2", genprob.poisson2d(5, 7)), ("p3", genprob.poisson3d(4, 3, 5)),
                    ("rs", genprob.random_spd(40, 0.2, 3)), ("rs2", genprob.random_spd(7, 1.0, 9))]:
        d[f"{name}_rs"], d[f"{name}_ci"], d[f"{name}_v"] = a.row_start, a.col_idx, a.values
    np.savez_compressed(OUT / "generators.npz", **d)


def cg_cases():
    d = {}
    # acceptance criterion 4 (tests/test_acceptance.py:78-94)
    a = genprob.poisson2d(32, 32)
    x_ref = np.random.default_rng(1004).standard_normal(1024)
    b = kernels.spmv_full(a, x_ref)
    opts = CgOptions(tol=1e-10, max_iter=1029, record_history=True)
    for tag, m, cfg in [("full", a, KernelConfig()),
                        ("sym", extract_lower(a), KernelConfig(accumulation="privatized"))]:
        r = cg_solve(m, b, opts=opts, cfg=cfg)
        d[f"p2_{tag}_x"] = r.x
        d[f"p2_{tag}_it"] = np.array(r.iterations)
        d[f"p2_{tag}_hist"] = np.array(r.residual_history)
        d[f"p2_{tag}_final"] = np.array(r.final_relative_residual)
    d["p2_b"] = b
    d["p2_xgen"] = x_ref
    # poisson3d 12^3 with x0 != 0 and max_iter truncation
    a3 = genprob.poisson3d(12, 12, 12)
    rng = np.random.default_rng(77)
    b3 = rng.standard_normal(a3.n)
    x03 = rng.standard_normal(a3.n)
    r = cg_solve(a3, b3, x0=x03, opts=CgOptions(tol=1e-9, record_history=True))
    d["p3_b"], d["p3_x0"], d["p3_x"], d["p3_it"] = b3, x03, r.x, np.array(r.iterations)
    d["p3_hist"] = np.array(r.residual_history)
    r = cg_solve(a3, b3, x0=x03, opts=CgOptions(max_iter=7, recompute_final_residual=False,
                                                record_history=True))
    d["p3t_x"], d["p3t_it"], d["p3t_final"] = r.x, np.array(r.iterations), np.array(
        r.final_relative_residual)
    d["p3t_conv"] = np.array(r.converged)
    np.savez_compressed(OUT / "cg_small.npz", **d)


def fem():
    """F-mesh (our FEM-shaped generator) and F-rand (reference random_spd) at
    the paper's 30880 / 449,798 size, solved by the reference CG."""
    d = {}
    F = mygen.fem_mesh()
    Fr = build_csr_from_triplets((F.entry_rows.copy(), F.col_idx.copy(), F.values.copy()), F.n)
    b, xg = mygen.rhs_for(F, seed=1)
    bref = kernels.spmv_full(Fr, xg)
    assert (b == bref).all()
    d["F_nnz"] = np.array(F.nnz)
    d["F_vsum"] = np.array(F.values.sum())
    d["F_colsum"] = np.array(int(F.col_idx.sum()))
    d["F_b"] = b
    for tag, m, cfg in [("full", Fr, KernelConfig(workers=1)),
                        ("sym", extract_lower(Fr), KernelConfig(workers=1, accumulation="privatized"))]:
        r = cg_solve(m, b, opts=CgOptions(record_history=True), cfg=cfg)
        d[f"F_{tag}_x"], d[f"F_{tag}_it"] = r.x, np.array(r.iterations)
        d[f"F_{tag}_hist"] = np.array(r.residual_history)
        d[f"F_{tag}_final"] = np.array(r.final_relative_residual)
        print("F", tag, r.iterations, r.final_relative_residual)
    R = genprob.random_spd(30880, 418918 / 30880**2, 1)
    assert R.nnz == 449798, R.nnz
    br = kernels.spmv_full(R, np.random.default_rng(1).standard_normal(R.n))
    r = cg_solve(R, br, opts=CgOptions(record_history=True), cfg=KernelConfig(workers=1))
    print("Frand", r.iterations, r.final_relative_residual)
    d["R_it"], d["R_x"], d["R_hist"] = np.array(r.iterations), r.x, np.array(r.residual_history)
    d["R_vsum"], d["R_colsum"] = np.array(R.values.sum()), np.array(int(R.col_idx.sum()))
    np.savez_compressed(OUT / "fem.npz", **d)


if __name__ == "__main__":
    kernels_small()
    generators()
    cg_cases()
    fem()
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)
