"""(dev) engine 5/6 device time per iteration under the current SPCG_CLUS_SORT
on F and a few banded systems (flushed, median of 5)."""
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
for name, a in (("F", fem_mesh()), ("p2d_256", poisson2d(256, 256)), ("p2d_400", poisson2d(400, 400)),
                ("p3d_48", poisson3d(48, 48, 48))):
    b, _ = rhs_for(a, seed=1)
    bt = torch.from_numpy(b).cuda()
    dm = a.device()
    for eng in (5, 6):
        ts = []
        for rep in range(6):
            flush.fill_(float(rep))
            x = torch.empty_like(bt)
            o = N.CgOptionsC(tol=1e-10, max_iter=0, record_history=0, recompute_final_residual=1,
                             accumulation=1, engine=eng)
            r = N.CgResultC()
            rc = lib.spcg_cg_solve(dm.handle, bt.data_ptr(), None, x.data_ptr(), None, o, r, 0)
            if rc:
                break
            ts.append(r.device_ms * 1e3 / r.iterations)
        out[f"{name}:{eng}"] = round(float(np.median(ts[1:])), 3) if len(ts) > 2 else None
print(out, flush=True)
