"""Development probe: per-config device CG timing (not the bench contract).

python scripts/probe.py [configs...]   configs: F S SA CSC P2 P3 Q27 Q27P
"""

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_1010_4639_b200 import _native as N  # noqa: E402
from paper_1010_4639_b200.device import DeviceMatrix  # noqa: E402
from paper_1010_4639_b200.genprob import fem_mesh, rhs_for  # noqa: E402
from paper_1010_4639_b200.core import extract_lower  # noqa: E402

PEAK = 6547.8


def solve(dm, b_t, acc=1, tol=1e-10, max_iter=0, engine=0, reps=3):
    lib = N.load()
    x = torch.empty_like(b_t)
    o = N.CgOptionsC(tol=tol, max_iter=max_iter, record_history=0, recompute_final_residual=1,
                     accumulation=acc, engine=engine, timing=1)
    out = []
    for _ in range(reps):
        r = N.CgResultC()
        rc = lib.spcg_cg_solve(dm.handle, b_t.data_ptr(), None, x.data_ptr(), None, o, r,
                               torch.cuda.current_stream().cuda_stream)
        N.check(rc, "solve")
        out.append((r.device_ms, r.iterations, r.final_relative_residual, r.spmv_ms / max(r.spmv_launches, 1)))
    return out, x


def spmv_time(dm, acc, n, reps=20):
    lib = N.load()
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        lib.spcg_spmv(dm.handle, x.data_ptr(), y.data_ptr(), acc, st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        lib.spcg_spmv(dm.handle, x.data_ptr(), y.data_ptr(), acc, st)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def report(name, dm, n, nnz_stored, b_t, acc=1, max_iter=0, engine=0):
    t0 = time.time()
    res, x = solve(dm, b_t, acc=acc, max_iter=max_iter, engine=engine)
    ms, its, fr, pq_ms = res[-1]
    best = min(r[0] for r in res)
    it_bytes = 12 * nnz_stored + 4 * (n + 1) + 88 * n
    sp_bytes = 12 * nnz_stored + 4 * (n + 1) + 16 * n
    us_it = best * 1e3 / max(its, 1)
    spms = spmv_time(dm, acc, n)
    d = dict(cfg=name, n=n, nnz=nnz_stored, iterations=its, final_rel=fr, solve_ms=best,
             us_per_it=us_it, it_per_s=its / (best / 1e3),
             it_GBs=it_bytes / (us_it * 1e-6) / 1e9, it_frac=it_bytes / (us_it * 1e-6) / 1e9 / PEAK,
             spmv_ms=spms, pass_a_ms=pq_ms, pass_a_frac=sp_bytes / (pq_ms * 1e-3) / 1e9 / PEAK if pq_ms else None, spmv_GBs=sp_bytes / (spms * 1e-3) / 1e9,
             spmv_frac=sp_bytes / (spms * 1e-3) / 1e9 / PEAK, wall_s=time.time() - t0,
             all_ms=[r[0] for r in res])
    print(json.dumps(d), flush=True)


def main():
    cfgs = sys.argv[1:] or ["F", "S", "SA", "CSC", "P2", "P3", "Q27", "Q27P"]
    print(json.dumps(N.device_info()))
    if any(c in cfgs for c in ("F", "S", "SA", "CSC")):
        F = fem_mesh()
        b, _ = rhs_for(F, seed=1)
        bt = torch.from_numpy(b).cuda()
        if "F" in cfgs:
            report("F_csr", F.device(), F.n, F.nnz, bt)
        if "S" in cfgs or "SA" in cfgs:
            S = extract_lower(F)
            if "S" in cfgs:
                report("S_priv", S.device(), S.n, S.nnz, bt, acc=1)
            if "SA" in cfgs:
                report("S_atomic", S.device(), S.n, S.nnz, bt, acc=0)
        if "CSC" in cfgs:
            C = F.to_csc()
            report("F_csc", C.device(), C.n, C.nnz, bt)
    big = {"P2": ("poisson2d", (4096, 4096), "csr", 1),
           "P3": ("poisson3d", (400, 400, 400), "csr", 1),
           "Q27": ("stencil27", (256, 256, 256), "scsr", 0),
           "Q27P": ("stencil27", (256, 256, 256), "scsr", 1),
           "Q27F": ("stencil27", (256, 256, 256), "csr", 1)}
    for c in cfgs:
        if c not in big:
            continue
        kind, dims, fmt, acc = big[c]
        t0 = time.time()
        dm = DeviceMatrix.generate(kind, dims, fmt)
        gen_s = time.time() - t0
        n = dm.n
        xg = torch.from_numpy(np.random.default_rng(1).standard_normal(n)).cuda()
        full = DeviceMatrix.generate(kind, dims, "csr") if fmt != "csr" else dm
        bt = torch.empty_like(xg)
        N.check(N.load().spcg_spmv(full.handle, xg.data_ptr(), bt.data_ptr(), 1, 0), "rhs")
        torch.cuda.synchronize()
        if full is not dm:
            full.close()
        print(json.dumps({"gen_s": gen_s, "cfg": c}), flush=True)
        report(c, dm, n, dm.nnz, bt, acc=acc, engine=int(__import__("os").environ.get("ENGINE", "0")))
        dm.close()


if __name__ == "__main__":
    main()
