"""Whole-vector parity of the full-size BASELINE configs against the
reference's own CG output (scripts/make_golden_fullsize.py: /root/reference's
spcg.cg_solve over its compiled kernels).  The reference x ships as
x_ref - x_gen in float32 (fullsize_xref/*_d32.npy: the snapshot limit is
512 MiB; x_gen = default_rng(1).standard_normal(n) is regenerated here), which
reconstructs x_ref to 4e-16 .. 8e-14 relative -- far below the 1e-8 bar.
Run once on a GPU box with fullsize_xref/ shipped:
    python scripts/fullsize_parity.py > profiles/r02/fullsize_parity.json
Every entry of x is compared (not a subsample): relative 2-norm error, max
abs error, iterations, true residual, for every storage / accumulation."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1010_4639_b200 import _native as N  # noqa: E402
from paper_1010_4639_b200.device import DeviceMatrix  # noqa: E402

CASES = [("p3", "poisson3d", (400, 400, 400), "csr", [("privatized", 1, 0)]),
         ("p2", "poisson2d", (4096, 4096), "csr", [("privatized", 1, 0)]),
         ("q27", "stencil27", (256, 256, 256), "scsr",
          [("fixed-point (default privatized)", 1, 0), ("L^T sequential (bitwise ref rows)", 1, 1),
           ("atomic", 0, 0)])]
out = {"reference": "spcg.cg_solve (solver.py:65-172) over the reference _ckernels, workers=8, "
                    "privatized; tol 1e-10, x0 = 0, b = spmv_full(A, default_rng(1).standard_normal(n))",
       "cases": []}
lib = N.load()
for name, kind, dims, fmt, modes in CASES:
    g = np.load(ROOT / "tests" / "golden" / f"fullsize_{name}.npz")
    d32 = np.load(ROOT / "fullsize_xref" / f"fullsize_{name}_d32.npy")
    xref = np.random.default_rng(1).standard_normal(d32.size) + d32.astype(np.float64)
    del d32
    dm = DeviceMatrix.generate(kind, dims, fmt)
    full = dm if fmt == "csr" else DeviceMatrix.generate(kind, dims, "csr")
    xg = torch.from_numpy(np.random.default_rng(1).standard_normal(dm.n)).cuda()
    b = torch.empty_like(xg)
    N.check(lib.spcg_spmv(full.handle, xg.data_ptr(), b.data_ptr(), N.ACC_PRIVATIZED, 0), "b")
    if full is not dm:
        full.close()
    del xg
    for label, acc, row_sums in modes:
        x = torch.empty_like(b)
        o = N.CgOptionsC(tol=1e-10, max_iter=0, record_history=0, recompute_final_residual=1,
                         accumulation=acc, engine=0, row_sums=row_sums)
        r = N.CgResultC()
        N.check(lib.spcg_cg_solve(dm.handle, b.data_ptr(), None, x.data_ptr(), None, o, r, 0), name)
        xh = x.cpu().numpy()
        d = xh - xref
        rec = {"config": name, "mode": label, "n": int(dm.n), "iterations": int(r.iterations),
               "ref_iterations": int(g["iterations"]),
               "rel_err_2norm": float(np.linalg.norm(d) / np.linalg.norm(xref)),
               "max_abs_err": float(np.max(np.abs(d))), "max_abs_xref": float(np.max(np.abs(xref))),
               "true_rel_residual": float(r.final_relative_residual),
               "ref_true_rel_residual": float(g["final_rel"]), "engine": int(r.engine_used),
               "entries_compared": int(d.size)}
        rec["pass"] = bool(abs(rec["iterations"] - rec["ref_iterations"]) <= max(1, rec["ref_iterations"] // 100)
                           and rec["rel_err_2norm"] <= 1e-8)
        out["cases"].append(rec)
        print(json.dumps(rec), file=sys.stderr, flush=True)
    dm.close()
print(json.dumps(out, indent=1))
