"""Distribution of back-to-back L2-flushed cluster-engine solves (the
"occasional 2.2x slower solve" of DESIGN §3): N solves per (storage, engine),
device time per solve from the library's CUDA events, and with
SPCG_CLUS_DEBUG=<file> the per-CTA SM ids / phase times of every engine-6
solve for the analysis in scripts/bimodal_report.py.

    SPCG_CLUS_DEBUG=gpurun_out/clus_dbg.jsonl python scripts/bimodal.py 50
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1010_4639_b200 import _native as N  # noqa: E402
from paper_1010_4639_b200.core import extract_lower  # noqa: E402
from paper_1010_4639_b200.genprob import fem_mesh, rhs_for  # noqa: E402

runs = int(sys.argv[1]) if len(sys.argv) > 1 else 50
cases = sys.argv[2].split(",") if len(sys.argv) > 2 else ["csr:6", "csr:5", "sympriv:6", "sympriv:5",
                                                          "csc:6", "csr:0"]
F = fem_mesh()
b, _ = rhs_for(F, seed=1)
bt = torch.from_numpy(b).cuda()
lib = N.load()
flush = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
mats = {"csr": (F, 1), "sympriv": (extract_lower(F), 1), "symatom": (extract_lower(F), 0),
        "csc": (F.to_csc(), 1)}
for case in cases:
    st, eng = case.split(":")
    m, acc = mats[st]
    dm = m.device()
    x = torch.empty_like(bt)
    o = N.CgOptionsC(tol=1e-10, max_iter=0, record_history=0, recompute_final_residual=1,
                     accumulation=acc, engine=int(eng))
    ms, its = [], None
    for i in range(runs + 2):
        flush.fill_(float(i))
        r = N.CgResultC()
        N.check(lib.spcg_cg_solve(dm.handle, bt.data_ptr(), None, x.data_ptr(), None, o, r, 0), case)
        torch.cuda.synchronize()
        if i >= 2:
            ms.append(r.device_ms)
            its = r.iterations
    a = np.array(ms)
    med = float(np.median(a))
    print(json.dumps({"case": case, "runs": runs, "iterations": its,
                      "us_it_min": round(1e3 * a.min() / its, 3),
                      "us_it_median": round(1e3 * med / its, 3),
                      "us_it_mean": round(1e3 * a.mean() / its, 3),
                      "us_it_max": round(1e3 * a.max() / its, 3),
                      "slow_runs": int((a > 1.3 * med).sum()),
                      "ms": [round(v, 4) for v in ms]}), flush=True)
