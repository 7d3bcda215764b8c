"""Dev stress: many cluster-engine solves of F / S, every run must be bitwise
identical (x, iterations) -- a race in the inter-cluster exchange shows up as
a differing run or a breakdown."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1010_4639_b200 import _native as N  # noqa: E402
from paper_1010_4639_b200.core import extract_lower  # noqa: E402
from paper_1010_4639_b200.genprob import fem_mesh, rhs_for  # noqa: E402

F = fem_mesh()
b, _ = rhs_for(F, seed=1)
bt = torch.from_numpy(b).cuda()
lib = N.load()
runs = int(sys.argv[1]) if len(sys.argv) > 1 else 200
for name, m in (("F", F), ("S", extract_lower(F))):
    dm = m.device()
    ref = None
    bad = 0
    for i in range(runs):
        x = torch.empty_like(bt)
        o = N.CgOptionsC(tol=1e-10, max_iter=0, record_history=0, recompute_final_residual=1,
                         accumulation=1, engine=5)
        r = N.CgResultC()
        rc = lib.spcg_cg_solve(dm.handle, bt.data_ptr(), None, x.data_ptr(), None, o, r, 0)
        xs = x.cpu().numpy()
        if rc != 0 or (ref is not None and (r.iterations != ref[0] or not np.array_equal(xs, ref[1]))):
            bad += 1
            print(name, "run", i, "rc", rc, "its", r.iterations, flush=True)
        if ref is None and rc == 0:
            ref = (r.iterations, xs)
    print(name, "runs", runs, "bad", bad, "its", ref[0] if ref else None, flush=True)
