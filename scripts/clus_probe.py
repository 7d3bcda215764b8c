"""Dev probe: cluster engine on the FEM matrix, fixed 300 iterations (A/B of
library variants under SPCG_TRACE; results of skip-variants are wrong)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1010_4639_b200 import _native as N  # noqa: E402
from paper_1010_4639_b200.genprob import fem_mesh, rhs_for  # noqa: E402
from paper_1010_4639_b200.core import extract_lower  # noqa: E402

F = fem_mesh()
b, _ = rhs_for(F, seed=1)
bt = torch.from_numpy(b).cuda()
lib = N.load()
for name, m, acc in (("F", F, 1), ("S", extract_lower(F), 1)):
    dm = m.device()
    x = torch.empty_like(bt)
    for eng in (5, 3):
        o = N.CgOptionsC(tol=1e-30, max_iter=300, record_history=0, recompute_final_residual=0,
                         accumulation=acc, engine=eng)
        best = 1e9
        for _ in range(3):
            r = N.CgResultC()
            lib.spcg_cg_solve(dm.handle, bt.data_ptr(), None, x.data_ptr(), None, o, r,
                              torch.cuda.current_stream().cuda_stream)
            best = min(best, r.device_ms)
        print(f"{name} engine {eng}: {r.iterations} its, {best * 1e3 / max(r.iterations, 1):.3f} us/it, "
              f"status {r.status}", flush=True)
