"""Per-phase device time of the per-pass engine (opts.timing = 2): SpMV
passes / vector-update passes / the rest, per iteration, for a generated
system.   python scripts/phase_split.py Q27P"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1010_4639_b200 import _native as N  # noqa: E402
from paper_1010_4639_b200.device import DeviceMatrix  # noqa: E402

CFG = {"P3": ("poisson3d", (400, 400, 400), "csr", 1), "P2": ("poisson2d", (4096, 4096), "csr", 1),
       "Q27": ("stencil27", (256, 256, 256), "scsr", 0), "Q27P": ("stencil27", (256, 256, 256), "scsr", 1),
       "Q27S": ("stencil27", (256, 256, 256), "scsr", 1),
       "M512": ("poisson2d", (512, 512), "csr", 1), "M1024": ("poisson2d", (1024, 1024), "csr", 1)}
name = sys.argv[1]
kind, dims, fmt, acc = CFG[name]
dm = DeviceMatrix.generate(kind, dims, fmt)
b = torch.from_numpy(np.random.default_rng(1).standard_normal(dm.n)).cuda()
x = torch.empty_like(b)
for rep in range(3):
    o = N.CgOptionsC(tol=1e-10, max_iter=int(sys.argv[2]) if len(sys.argv) > 2 else 100,
                     record_history=0, recompute_final_residual=0, accumulation=acc, engine=2,
                     timing=2, row_sums=1 if name == "Q27S" else 0)
    r = N.CgResultC()
    N.check(N.load().spcg_cg_solve(dm.handle, b.data_ptr(), None, x.data_ptr(), None, o, r, 0), "s")
    it = r.iterations
    print(name, "its", it, "us/it total %.1f spmv %.1f update(B+C) %.1f rest %.1f" % (
        1e3 * r.device_ms / it, 1e3 * r.phase_ms[0] / it, 1e3 * r.phase_ms[2] / it,
        1e3 * r.phase_ms[1] / it), flush=True)
