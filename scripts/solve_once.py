"""Dev helper: one device-generated solve (for ncu launch lists).
python scripts/solve_once.py <P3|P2|Q27|Q27P> <max_iter> <engine>"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1010_4639_b200 import _native as N  # noqa: E402
from paper_1010_4639_b200.device import DeviceMatrix  # noqa: E402

CFG = {"P3": ("poisson3d", (400, 400, 400), "csr", 1), "P2": ("poisson2d", (4096, 4096), "csr", 1),
       "Q27": ("stencil27", (256, 256, 256), "scsr", 0), "Q27P": ("stencil27", (256, 256, 256), "scsr", 1)}
kind, dims, fmt, acc = CFG[sys.argv[1]]
mi, eng = int(sys.argv[2]), int(sys.argv[3])
dm = DeviceMatrix.generate(kind, dims, fmt)
b = torch.from_numpy(np.random.default_rng(1).standard_normal(dm.n)).cuda()
x = torch.empty_like(b)
o = N.CgOptionsC(tol=1e-10, max_iter=mi, record_history=0, recompute_final_residual=1,
                 accumulation=acc, engine=eng)
r = N.CgResultC()
N.check(N.load().spcg_cg_solve(dm.handle, b.data_ptr(), None, x.data_ptr(), None, o, r, 0), "solve")
print(r.iterations, r.device_ms, r.kernel_launches)
