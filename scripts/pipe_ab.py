"""Dev A/B: engine 5 (cluster-resident Chronopoulos–Gear) vs engine 6
(pipelined) on the FEM matrix in each storage: iterations, x gap to the
engine-5 solution, device µs per iteration (best of N back-to-back solves)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1010_4639_b200 import KernelConfig, extract_lower  # noqa: E402
from paper_1010_4639_b200 import _native as N  # noqa: E402
from paper_1010_4639_b200.genprob import fem_mesh, rhs_for  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
F = fem_mesh()
b, _ = rhs_for(F, seed=1)
bt = torch.from_numpy(b).cuda()
lib = N.load()
for kind, m, acc in (("csr", F, 1), ("csc", F.to_csc(), 1), ("sym_priv", extract_lower(F), 1),
                     ("sym_atomic", extract_lower(F), 0)):
    dm = m.device()
    xs = {}
    for eng in (5, 6):
        x = torch.empty_like(bt)
        o = N.CgOptionsC(tol=1e-10, max_iter=0, record_history=0, recompute_final_residual=1,
                         accumulation=acc, engine=eng)
        best = 1e30
        for _ in range(reps):
            r = N.CgResultC()
            N.check(lib.spcg_cg_solve(dm.handle, bt.data_ptr(), None, x.data_ptr(), None, o, r,
                                      0), "solve")
            best = min(best, r.device_ms)
        xs[eng] = x.cpu().numpy()
        print(f"{kind:10s} engine {eng}: it {r.iterations} final_rel {r.final_relative_residual:.3e} "
              f"best {best * 1e3 / r.iterations:.3f} us/it ({r.iterations / best * 1e3:,.0f} it/s)",
              flush=True)
    gap = np.linalg.norm(xs[6] - xs[5]) / np.linalg.norm(xs[5])
    print(f"{kind:10s} |x6 - x5| / |x5| = {gap:.2e}", flush=True)
