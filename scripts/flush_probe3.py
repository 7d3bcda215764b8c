"""Dev: what about a preceding big memory kernel slows the next F solve?"""
import sys, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1010_4639_b200 import _native as N  # noqa
from paper_1010_4639_b200.genprob import fem_mesh, rhs_for  # noqa

F = fem_mesh(); b, _ = rhs_for(F, seed=1)
bt = torch.from_numpy(b).cuda(); dm = F.device(); x = torch.empty_like(bt)
lib = N.load(); st = torch.cuda.current_stream()
o = N.CgOptionsC(tol=1e-10, max_iter=0, record_history=0, recompute_final_residual=1, accumulation=1, engine=0)
big = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
small = torch.empty(16 << 20, dtype=torch.float64, device="cuda")
def solve():
    r = N.CgResultC()
    lib.spcg_cg_solve(dm.handle, bt.data_ptr(), None, x.data_ptr(), None, o, r, st.cuda_stream)
    torch.cuda.synchronize()
    return r.device_ms
def run(tag, pre, n=12):
    ks = []
    for i in range(n):
        pre(i)
        ks.append(solve())
    print("%-28s" % tag, " ".join("%.2f" % k for k in ks), flush=True)
for _ in range(3): solve()
run("write 512MB", lambda i: big.fill_(float(i)))
run("write 512MB + 2ms sleep", lambda i: (big.fill_(float(i)), torch.cuda.synchronize(), time.sleep(0.002)))
run("read 512MB", lambda i: big.sum())
run("write 128MB", lambda i: small.fill_(float(i)))
run("nothing", lambda i: None)
