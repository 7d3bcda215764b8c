"""(dev) lone-rank per-pass engine: host-transport form (MODE 0, 5 launches per
iteration: 2 one-thread scalar kernels) vs the device-transport form (MODE 1,
3 launches: scalars in the passes' last CTA) on 3-D Poisson of several sides.
    python scripts/mode_ab.py 64 128 256"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1010_4639_b200 import _native as N  # noqa: E402
from paper_1010_4639_b200.device import DeviceMatrix  # noqa: E402
from paper_1010_4639_b200.distributed import ShardedMatrix, group_plans, group_solve  # noqa: E402

lib = N.load()
for arg in sys.argv[1:] or ["64", "128", "256"]:
    kind = "poisson2d" if arg.startswith("2d") else "poisson3d"
    side = int(arg[2:]) if arg.startswith("2d") else int(arg)
    dims = (side, side) if kind == "poisson2d" else (side, side, side)
    n = side ** len(dims)
    its = 200
    dm = DeviceMatrix.generate(kind, dims, "csr")
    b = torch.from_numpy(np.random.default_rng(1).standard_normal(n)).cuda()
    x = torch.empty_like(b)
    t0 = []
    for rep in range(3):
        o = N.CgOptionsC(tol=1e-30, max_iter=its, record_history=0, recompute_final_residual=0,
                         accumulation=1, engine=2)
        r = N.CgResultC()
        N.check(lib.spcg_cg_solve(dm.handle, b.data_ptr(), None, x.data_ptr(), None, o, r, 0), "s")
        t0.append(1e3 * r.device_ms / r.iterations)
    shards = ShardedMatrix.group_from_stencil(kind, dims, "csr", 1)
    plans = group_plans(shards)
    t1 = []
    for rep in range(3):
        _, rr, _ = group_solve(plans, [b], max_iter=its, recompute_final_residual=False, tol=1e-30)
        t1.append(1e3 * rr[0].device_ms / rr[0].iterations)
    print(side, n, "mode0 us/it %.2f" % np.median(t0), "mode1 us/it %.2f" % np.median(t1),
          "launches", r.kernel_launches, rr[0].kernel_launches, flush=True)
    del plans, shards, dm
    torch.cuda.empty_cache()
