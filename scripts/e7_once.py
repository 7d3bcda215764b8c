"""(dev) one engine-7 solve of 2-D Poisson (side argv[1]) for ncu."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1010_4639_b200 import _native as N  # noqa: E402
from paper_1010_4639_b200.device import DeviceMatrix  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 512
dm = DeviceMatrix.generate("poisson2d", (side, side), "csr")
b = torch.from_numpy(np.random.default_rng(1).standard_normal(dm.n)).cuda()
x = torch.empty_like(b)
for _ in range(2):
    o = N.CgOptionsC(tol=1e-10, max_iter=200, record_history=0, recompute_final_residual=0,
                     accumulation=1, engine=7)
    r = N.CgResultC()
    N.check(N.load().spcg_cg_solve(dm.handle, b.data_ptr(), None, x.data_ptr(), None, o, r, 0), "s")
print(r.iterations, 1e3 * r.device_ms / r.iterations)
