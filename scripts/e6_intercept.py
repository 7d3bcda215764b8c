import sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_1010_4639_b200 import _native as N
from paper_1010_4639_b200.genprob import fem_mesh, rhs_for
F = fem_mesh(); b, _ = rhs_for(F, seed=1)
dm = F.device(); lib = N.load()
bt = torch.from_numpy(b).cuda(); xt = torch.empty_like(bt)
st = torch.cuda.current_stream().cuda_stream
flush = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
for mi in (1, 2, 5, 10, 50, 100, 200, 329):
    ts = []
    for rep in range(12):
        o = N.CgOptionsC(tol=1e-30 if mi < 329 else 1e-10, max_iter=mi, record_history=0, recompute_final_residual=0,
                         accumulation=1, engine=6)
        r = N.CgResultC()
        flush.fill_(rep)
        torch.cuda.synchronize()
        lib.spcg_cg_solve(dm.handle, bt.data_ptr(), None, xt.data_ptr(), None, o, r, st)
        torch.cuda.synchronize()
        ts.append(r.device_ms * 1e3)
    print(mi, r.iterations, "median us %.1f" % np.median(ts[2:]))
# b = 0: launch + setup loads + the ||b|| all-reduce only
bz = torch.zeros_like(bt)
ts = []
for rep in range(12):
    o = N.CgOptionsC(tol=1e-10, max_iter=0, record_history=0, recompute_final_residual=0,
                     accumulation=1, engine=6)
    r = N.CgResultC()
    flush.fill_(rep)
    torch.cuda.synchronize()
    lib.spcg_cg_solve(dm.handle, bz.data_ptr(), None, xt.data_ptr(), None, o, r, st)
    torch.cuda.synchronize()
    ts.append(r.device_ms * 1e3)
print("b=0", r.iterations, "median us %.1f" % np.median(ts[2:]))
ts = []
for rep in range(12):
    o = N.CgOptionsC(tol=1e-10, max_iter=0, record_history=0, recompute_final_residual=0,
                     accumulation=1, engine=6)
    r = N.CgResultC()
    torch.cuda.synchronize()
    lib.spcg_cg_solve(dm.handle, bz.data_ptr(), None, xt.data_ptr(), None, o, r, st)
    torch.cuda.synchronize()
    ts.append(r.device_ms * 1e3)
print("b=0 no flush", r.iterations, "median us %.1f" % np.median(ts[2:]))
