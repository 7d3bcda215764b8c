"""Dev helper: repeated standalone SpMV on a generated matrix (for ncu)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1010_4639_b200 import _native as N  # noqa: E402
from paper_1010_4639_b200.device import DeviceMatrix  # noqa: E402

CFG = {"P3": ("poisson3d", (400, 400, 400), "csr", 1), "Q27F": ("stencil27", (256, 256, 256), "csr", 1),
       "Q27": ("stencil27", (256, 256, 256), "scsr", 0), "Q27P": ("stencil27", (256, 256, 256), "scsr", 1)}
kind, dims, fmt, acc = CFG[sys.argv[1]]
dm = DeviceMatrix.generate(kind, dims, fmt)
x = torch.from_numpy(np.random.default_rng(1).standard_normal(dm.n)).cuda()
y = torch.empty_like(x)
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    N.check(N.load().spcg_spmv(dm.handle, x.data_ptr(), y.data_ptr(), acc, 0), "spmv")
torch.cuda.synchronize()
print("ok")
