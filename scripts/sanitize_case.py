"""Small solves of every engine for compute-sanitizer (one tool per run):
    compute-sanitizer --tool racecheck python scripts/sanitize_case.py
Engines 6 / 5 / 3 on the 30880-row F-mesh (CSR and SCSR), the per-pass
engine on a small Poisson, and the device-transport group solve (2 virtual
ranks) -- the synchronisation-heavy paths of DESIGN §3-4."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1010_4639_b200 import CgOptions, KernelConfig, cg_solve, extract_lower  # noqa: E402
from paper_1010_4639_b200.distributed import ShardedMatrix, group_plans, group_solve  # noqa: E402
from paper_1010_4639_b200.genprob import fem_mesh, poisson3d, rhs_for  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
F = fem_mesh()
b, _ = rhs_for(F, seed=1)
S = extract_lower(F)
mi = int(sys.argv[2]) if len(sys.argv) > 2 else 40  # iterations per solve (sanitizers are slow)
opts = CgOptions(max_iter=mi)
for eng in (6, 5, 3):
    if which not in ("all", f"e{eng}"):
        continue
    for m, acc in ((F, "privatized"), (S, "privatized"), (S, "atomic")):
        r = cg_solve(m, b, opts=opts, cfg=KernelConfig(accumulation=acc), engine=eng)
        print("engine", eng, type(m).__name__, acc, r.iterations, flush=True)
if which in ("all", "e2"):
    a = poisson3d(24, 24, 24)
    bb, _ = rhs_for(a, seed=2)
    r = cg_solve(a, bb, opts=opts, engine=2)
    print("engine 2", r.iterations, flush=True)
if which in ("all", "p2p"):
    a = poisson3d(12, 12, 16)
    bb, _ = rhs_for(a, seed=2)
    sh = ShardedMatrix.group_from_stencil("poisson3d", (12, 12, 16), "csr", 2)
    plans = group_plans(sh)
    xs, res, _ = group_solve(plans, [torch.from_numpy(bb[s.row0:s.row1].copy()).cuda() for s in sh],
                             max_iter=mi)
    print("p2p group", res[0].iterations, flush=True)
torch.cuda.synchronize()
print("done")
