"""Per-iteration cost of the device-initiated exchange in the one-GPU
virtual-rank model: the same system solved (a) as ONE rank (device transport,
no peers) and (b) as R virtual ranks in one launch per pass (mailbox
all-reduces + halo stores between the ranks' buffers).  Both stream the same
bytes, so (b) - (a) per iteration is what the exchange costs (an upper bound
for the NVLink case, where the R ranks also stream in parallel).
    python scripts/p2p_overhead.py [side] [R...]"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1010_4639_b200.distributed import ShardedMatrix, group_plans, group_solve  # noqa: E402
from paper_1010_4639_b200.genprob import poisson3d  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 256
Rs = [int(r) for r in sys.argv[2:]] or [1, 2, 4, 8]
dims = (side, side, side)
n = side ** 3
xg = np.random.default_rng(1).standard_normal(n)
res = []
for R in Rs:
    shards = ShardedMatrix.group_from_stencil("poisson3d", dims, "csr", R)
    plans = group_plans(shards)
    # b = A x_gen through the shards (each rank's rows)
    bl = []
    for s in shards:
        xe = torch.from_numpy(np.concatenate([xg[s.row0:s.row1], xg[s.halo]])).cuda()
        bl.append(s.spmv_ext(xe))
    its = 200
    for rep in range(3):
        torch.cuda.synchronize()
        xs, rr, _ = group_solve(plans, bl, max_iter=its, recompute_final_residual=False)
        torch.cuda.synchronize()
    ms = rr[0].device_ms
    _, rt, _ = group_solve(plans, bl, max_iter=its, recompute_final_residual=False, timing=2)
    it = rt[0].iterations
    out = {"R": R, "n": n, "iterations": int(rr[0].iterations), "ms": ms,
           "us_per_iteration": 1e3 * ms / rr[0].iterations,
           "phase_us_per_iteration": {"spmv_pass": 1e3 * rt[0].phase_ms[0] / it,
                                      "update_passes": 1e3 * rt[0].phase_ms[2] / it,
                                      "rest": 1e3 * rt[0].phase_ms[1] / it},
           "launches_per_iteration": None}
    _, r1, _ = group_solve(plans, bl, max_iter=100, recompute_final_residual=False)
    _, r2, _ = group_solve(plans, bl, max_iter=200, recompute_final_residual=False)
    out["launches_per_iteration"] = (r2[0].kernel_launches - r1[0].kernel_launches) / 100
    res.append(out)
    print(json.dumps(out), flush=True)
    del plans, shards, bl
    torch.cuda.empty_cache()
base = res[0]["us_per_iteration"]
for o in res:
    o["overhead_us_per_iteration_vs_R1"] = o["us_per_iteration"] - base
print(json.dumps({"side": side, "results": res}))
