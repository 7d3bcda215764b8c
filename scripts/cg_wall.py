import time, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1010_4639_b200.genprob import fem_mesh, rhs_for
from paper_1010_4639_b200.core import extract_lower
from paper_1010_4639_b200.solver import cg_solve, CgOptions
from paper_1010_4639_b200.kernels import KernelConfig
F = fem_mesh(); b, _ = rhs_for(F, seed=1)
for name, m in (("full", F), ("sym", extract_lower(F)), ("csc", F.to_csc())):
    t0 = time.perf_counter(); m.device(); torch.cuda.synchronize(); up = time.perf_counter() - t0
    for acc in ("atomic", "privatized"):
        ts = []
        for i in range(5):
            t0 = time.perf_counter_ns()
            r = cg_solve(m, b, opts=CgOptions(tol=1e-10), cfg=KernelConfig(accumulation=acc))
            ts.append((time.perf_counter_ns() - t0) / 1e6)
        print(name, acc, "upload %.1f ms" % (up * 1e3), "solves ms", ["%.2f" % t for t in ts], r.engine_info, r.timings, flush=True)
