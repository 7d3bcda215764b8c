"""Engine 7 (streamed single-reduction persistent kernel) vs engine 2 (per-pass)
on mid-size systems: us per iteration (flushed, median of 3), iterations, and
||x7 - x2|| / ||x2||.   python scripts/engine7_ab.py"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1010_4639_b200 import _native as N  # noqa: E402
from paper_1010_4639_b200.device import DeviceMatrix  # noqa: E402

lib = N.load()
flush = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
cases = [("poisson2d", (512, 512), "csr", 1), ("poisson3d", (64, 64, 64), "csr", 1),
         ("poisson3d", (100, 100, 100), "csr", 1), ("poisson2d", (1448, 1448), "csr", 1),
         ("poisson3d", (128, 128, 128), "csr", 1), ("poisson2d", (2048, 2048), "csr", 1),
         ("stencil27", (64, 64, 64), "scsr", 1), ("poisson3d", (200, 200, 200), "csr", 1),
         ("poisson2d", (4096, 4096), "csr", 1)]
if len(sys.argv) > 1:
    cases = cases[: int(sys.argv[1])]
for kind, dims, fmt, acc in cases:
    dm = DeviceMatrix.generate(kind, dims, fmt)
    b = torch.from_numpy(np.random.default_rng(1).standard_normal(dm.n)).cuda()
    res = {}
    xs = {}
    for eng in (2, 7, 0):
        ts, its = [], None
        for rep in range(3):
            flush.fill_(float(rep))
            x = torch.empty_like(b)
            o = N.CgOptionsC(tol=1e-10, max_iter=2000, record_history=0, recompute_final_residual=1,
                             accumulation=acc, engine=eng)
            r = N.CgResultC()
            rc = lib.spcg_cg_solve(dm.handle, b.data_ptr(), None, x.data_ptr(), None, o, r, 0)
            if rc:
                its = "rc %d" % rc
                break
            ts.append(1e3 * r.device_ms / max(1, r.iterations))
            its = (int(r.iterations), int(r.engine_used), float(r.final_relative_residual))
            xs[eng] = x
        res[eng] = (round(float(np.median(ts)), 2) if ts else None, its)
    d = (torch.linalg.norm(xs[7] - xs[2]) / torch.linalg.norm(xs[2])).item() if 7 in xs and 2 in xs else None
    print(kind, dims, fmt, dm.n, res, "x7-x2 %.2e" % d if d is not None else "", flush=True)
    del dm
    torch.cuda.empty_cache()
