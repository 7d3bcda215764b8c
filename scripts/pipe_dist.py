"""Dev: distribution of per-solve µs/iteration (L2 flushed before each solve)
for engines 5 and 6 on the FEM matrix storages (bimodality check)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1010_4639_b200 import extract_lower  # noqa: E402
from paper_1010_4639_b200 import _native as N  # noqa: E402
from paper_1010_4639_b200.genprob import fem_mesh, rhs_for  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
engines = [int(e) for e in sys.argv[2].split(",")] if len(sys.argv) > 2 else [5, 6]
F = fem_mesh()
b, _ = rhs_for(F, seed=1)
bt = torch.from_numpy(b).cuda()
lib = N.load()
flush = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
for kind, m, acc in (("csr", F, 1), ("sym_priv", extract_lower(F), 1),
                     ("sym_atomic", extract_lower(F), 0), ("csc", F.to_csc(), 1)):
    dm = m.device()
    x = torch.empty_like(bt)
    for eng in engines:
        o = N.CgOptionsC(tol=1e-10, max_iter=0, record_history=0, recompute_final_residual=1,
                         accumulation=acc, engine=eng)
        us = []
        for k in range(reps):
            flush.fill_(float(k))
            r = N.CgResultC()
            N.check(lib.spcg_cg_solve(dm.handle, bt.data_ptr(), None, x.data_ptr(), None, o, r,
                                      torch.cuda.current_stream().cuda_stream), "solve")
            us.append(r.device_ms * 1e3 / r.iterations)
        print(f"{kind:9s} e{eng}: median {np.median(us):.3f} us/it  " +
              " ".join(f"{u:.2f}" for u in us), flush=True)
