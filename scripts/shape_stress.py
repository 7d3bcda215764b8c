"""Engine-6 determinism across grid shapes (dev knobs SPCG_CLUS_K / _CSZ):
RUNS solves per case; prints failures and distinct (iterations, x hash).
    SPCG_CLUS_K=6 python scripts/shape_stress.py 30 csr,sympriv,csc [engine]"""
import hashlib
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1010_4639_b200 import _native as N  # noqa: E402
from paper_1010_4639_b200.core import extract_lower  # noqa: E402
from paper_1010_4639_b200.genprob import fem_mesh, rhs_for  # noqa: E402

runs = int(sys.argv[1])
cases = sys.argv[2].split(",")
eng = int(sys.argv[3]) if len(sys.argv) > 3 else 6
F = fem_mesh()
b, _ = rhs_for(F, seed=1)
bt = torch.from_numpy(b).cuda()
lib = N.load()
mats = {"csr": (F, 1), "sympriv": (extract_lower(F), 1), "csc": (F.to_csc(), 1)}
for case in cases:
    m, acc = mats[case]
    dm = m.device()
    fails, seen = 0, {}
    for i in range(runs):
        x = torch.zeros_like(bt)
        o = N.CgOptionsC(tol=1e-10, max_iter=0, record_history=0, recompute_final_residual=1,
                         accumulation=acc, engine=eng)
        r = N.CgResultC()
        rc = lib.spcg_cg_solve(dm.handle, bt.data_ptr(), None, x.data_ptr(), None, o, r, 0)
        if rc != 0:
            fails += 1
            key = ("rc", rc, r.fail_iteration if hasattr(r, "fail_iteration") else -1)
        else:
            key = (r.iterations, hashlib.md5(x.cpu().numpy().tobytes()).hexdigest()[:8])
        seen[key] = seen.get(key, 0) + 1
    print(case, "eng", eng, "runs", runs, "fails", fails, "distinct", seen, flush=True)
