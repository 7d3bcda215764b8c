"""(dev) engine 6 with / without register rows (SPCG_PIPE_REG=0 in the env
turns them off) on F and stencil systems: us per iteration (flushed, median)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1010_4639_b200 import _native as N  # noqa: E402
from paper_1010_4639_b200.genprob import fem_mesh, poisson2d, poisson3d, rhs_for  # noqa: E402

lib = N.load()
flush = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
out = {}
for name, a in (("F", fem_mesh()), ("p2d_160", poisson2d(160, 160)), ("p2d_256", poisson2d(256, 256)),
                ("p3d_32", poisson3d(32, 32, 32)), ("p3d_40", poisson3d(40, 40, 40))):
    b, _ = rhs_for(a, seed=1)
    bt = torch.from_numpy(b).cuda()
    dm = a.device()
    ts = []
    for rep in range(6):
        flush.fill_(float(rep))
        x = torch.empty_like(bt)
        o = N.CgOptionsC(tol=1e-10, max_iter=0, record_history=0, recompute_final_residual=1,
                         accumulation=1, engine=6)
        r = N.CgResultC()
        rc = lib.spcg_cg_solve(dm.handle, bt.data_ptr(), None, x.data_ptr(), None, o, r, 0)
        if rc:
            break
        ts.append(r.device_ms * 1e3 / r.iterations)
    out[name] = (round(float(np.median(ts[1:])), 3) if len(ts) > 2 else None, int(r.iterations))
print(out, flush=True)
