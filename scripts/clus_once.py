"""Dev helper: one cluster-engine solve on the FEM matrix (for ncu)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1010_4639_b200 import _native as N  # noqa: E402
from paper_1010_4639_b200.genprob import fem_mesh, rhs_for  # noqa: E402

F = fem_mesh()
b, _ = rhs_for(F, seed=1)
bt = torch.from_numpy(b).cuda()
kind = sys.argv[3] if len(sys.argv) > 3 else "csr"  # csr | sym (privatized L+D)
if kind == "sym":
    from paper_1010_4639_b200 import extract_lower  # noqa: E402
    dm = extract_lower(F).device()
else:
    dm = F.device()
x = torch.empty_like(bt)
o = N.CgOptionsC(tol=1e-10, max_iter=int(sys.argv[1]) if len(sys.argv) > 1 else 0,
                 record_history=0, recompute_final_residual=1, accumulation=1,
                 engine=int(sys.argv[2]) if len(sys.argv) > 2 else 5)
for _ in range(2):
    r = N.CgResultC()
    N.check(N.load().spcg_cg_solve(dm.handle, bt.data_ptr(), None, x.data_ptr(), None, o, r, 0), "solve")
print(r.iterations, r.device_ms)
