"""Full-size reference CG goldens for BASELINE's big configs (P3, P2, Q27).

Run HERE (the container with /root/reference; ~30 min, ~25 GB RSS peak):
    python scripts/make_golden_fullsize.py [p3 p2 q27]

For each config it runs the REFERENCE's own `spcg.solver.cg_solve`
(/root/reference/pkg/src/spcg/solver.py:65-172) with the reference's compiled
kernels (oracle/_ref, built from _ckernels.pyx by `make -C oracle ref`)
installed as the "compiled" backend, exactly as scripts/make_golden.py does
for the small fixtures.  Only the matrix arrays come from the C generator
(oracle.stencil, pinned bitwise against genprob.poisson2d/3d in
tests/test_oracle.py) because genprob.poisson3d(400^3) alone needs 38 GB.

Inputs follow cmd_gen (cli.py:91-93): x_gen = default_rng(1).standard_normal(n),
b = spmv_full(A_full, x_gen), x0 = 0, tol = 1e-10, max_iter = n.

Stored per config in tests/golden/fullsize_<cfg>.npz (small: the vector is
subsampled):
  iterations, converged, final_rel (true residual), residual_history (all
  iterations), x_norm = ||x_ref||_2, stride, x_sub = x_ref[::stride],
  x_sum (np.sum of x_ref), b_norm, kernel config.
The full x_ref also goes to fullsize_xref/ (git-ignored and gpurun-ignored;
un-ignored for the one full-vector comparison call, scripts/fullsize_parity.py).
"""

from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from oracle import oracle as O  # noqa: E402

ck = O.load_ref()
assert ck is not None, "run `make -C oracle ref` first"
sys.modules["spcg.kernels._ckernels"] = ck

from spcg import kernels  # noqa: E402
from spcg.core import CsrMatrix, SymHalfMatrix  # noqa: E402
from spcg.kernels import KernelConfig  # noqa: E402
from spcg.solver import CgOptions, cg_solve  # noqa: E402

assert "compiled" in kernels.available_backends()
kernels.set_backend("compiled")

OUT = ROOT / "tests" / "golden"
FULL = ROOT / "fullsize_xref"
STRIDE = 977

CONFIGS = {
    "p3": ("poisson3d", (400, 400, 400), "csr"),
    "p2": ("poisson2d", (4096, 4096), "csr"),
    "q27": ("stencil27", (256, 256, 256), "sym"),
}


def run(name: str) -> dict:
    kind, dims, storage = CONFIGS[name]
    workers = os.cpu_count() or 1
    cfg = KernelConfig(workers=workers, accumulation="privatized")
    t0 = time.perf_counter()
    rs, ci, v = O.stencil(kind, dims, "full")
    n = len(rs) - 1
    full = CsrMatrix(n, rs, ci, v)
    x_gen = np.random.default_rng(1).standard_normal(n)
    b = kernels.spmv_full(full, x_gen, cfg)
    if storage == "sym":
        del full, rs, ci, v
        rs, ci, v = O.stencil(kind, dims, "lower")
        a = SymHalfMatrix(n, rs, ci, v)
    else:
        a = full
    t1 = time.perf_counter()
    print(f"[{name}] n={n} stored={len(ci)} generated in {t1 - t0:.1f}s; solving "
          f"(workers={workers})", flush=True)
    rep = cg_solve(a, b, opts=CgOptions(tol=1e-10, record_history=True), cfg=cfg)
    t2 = time.perf_counter()
    x = rep.x
    res = dict(
        config=name, kind=kind, dims=list(dims), storage=storage, n=n, stored_nnz=int(len(ci)),
        iterations=int(rep.iterations), converged=bool(rep.converged),
        final_rel=float(rep.final_relative_residual),
        residual_history=np.asarray(rep.residual_history, dtype=np.float64),
        x_norm=float(np.linalg.norm(x)), x_sum=float(np.sum(x)), stride=STRIDE,
        x_sub=np.ascontiguousarray(x[::STRIDE]), b_norm=float(np.linalg.norm(b)),
        err_vs_gen=float(np.linalg.norm(x - x_gen) / np.linalg.norm(x_gen)),
        workers=workers, accumulation="privatized", solve_s=t2 - t1,
    )
    np.savez_compressed(OUT / f"fullsize_{name}.npz", **res)
    # the whole vector too, for the one GPU-box full-vector comparison
    # (scripts/fullsize_parity.py); git-ignored: 128-512 MB
    FULL.mkdir(parents=True, exist_ok=True)
    np.save(FULL / f"fullsize_{name}_x.npy", x)
    print(json.dumps({k: (v if not isinstance(v, np.ndarray) else f"<{v.shape}>")
                      for k, v in res.items()}), flush=True)
    return res


if __name__ == "__main__":
    names = sys.argv[1:] or ["q27", "p3", "p2"]
    for nm in names:
        run(nm)
