"""Per-engine device time per iteration on mid-size banded systems (is auto's
pick the fastest?):  python scripts/engine_pick.py"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1010_4639_b200 import _native as N  # noqa: E402
from paper_1010_4639_b200.genprob import poisson2d, poisson3d, rhs_for  # noqa: E402

lib = N.load()
flush = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
for name, a in (("p2d_256", poisson2d(256, 256)), ("p2d_512", poisson2d(512, 512)),
                ("p2d_724", poisson2d(724, 724)), ("p3d_48", poisson3d(48, 48, 48)),
                ("p3d_64", poisson3d(64, 64, 64))):
    b, _ = rhs_for(a, seed=1)
    bt = torch.from_numpy(b).cuda()
    dm = a.device()
    res = {}
    for eng in (0, 2, 3, 5, 6):
        ts = []
        info = None
        for rep in range(4):
            flush.fill_(float(rep))
            x = torch.empty_like(bt)
            o = N.CgOptionsC(tol=1e-10, max_iter=0, record_history=0, recompute_final_residual=1,
                             accumulation=1, engine=eng)
            r = N.CgResultC()
            rc = lib.spcg_cg_solve(dm.handle, bt.data_ptr(), None, x.data_ptr(), None, o, r, 0)
            if rc != 0:
                info = "rc %d" % rc
                break
            ts.append(r.device_ms * 1e3 / max(1, r.iterations))
            info = (r.iterations, r.engine_used)
        res[eng] = (round(float(np.median(ts[1:])), 2) if len(ts) > 1 else None, info)
    print(name, a.n, res, flush=True)
