"""Dev: per-pass engine solve time without per-pass timing events."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1010_4639_b200 import _native as N  # noqa
from paper_1010_4639_b200.device import DeviceMatrix  # noqa

for name, kind, dims, fmt, acc in (("P2", "poisson2d", (4096, 4096), "csr", 1),
                                   ("P3", "poisson3d", (400, 400, 400), "csr", 1),
                                   ("Q27", "stencil27", (256, 256, 256), "scsr", 0)):
    dm = DeviceMatrix.generate(kind, dims, fmt)
    b = torch.from_numpy(np.random.default_rng(1).standard_normal(dm.n)).cuda()
    x = torch.empty_like(b)
    o = N.CgOptionsC(tol=1e-10, max_iter=0, record_history=0, recompute_final_residual=1,
                     accumulation=acc, engine=0, timing=0)
    ts = []
    for _ in range(4):
        r = N.CgResultC()
        N.check(N.load().spcg_cg_solve(dm.handle, b.data_ptr(), None, x.data_ptr(), None, o, r, 0), "s")
        ts.append(r.device_ms * 1e3 / r.iterations)
    print(name, r.iterations, " ".join("%.1f" % t for t in ts), flush=True)
    dm.close()
