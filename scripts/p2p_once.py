"""One group solve (R virtual ranks, Poisson side^3) for ncu launch lists:
    python scripts/p2p_once.py R side iters"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1010_4639_b200.distributed import ShardedMatrix, group_plans, group_solve  # noqa: E402

R, side, its = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
shards = ShardedMatrix.group_from_stencil("poisson3d", (side,) * 3, "csr", R)
plans = group_plans(shards)
bl = [torch.ones(s.nloc, dtype=torch.float64, device="cuda") for s in shards]
xs, res, _ = group_solve(plans, bl, max_iter=its, recompute_final_residual=False)
torch.cuda.synchronize()
print(R, res[0].iterations, res[0].device_ms)
