"""Dev: fraction of slow F solves after a foreign kernel (bimodality check)."""
import sys
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
def solve():
    r = N.CgResultC()
    lib.spcg_cg_solve(dm.handle, bt.data_ptr(), None, x.data_ptr(), None, o, r, st.cuda_stream)
    torch.cuda.synchronize()
    return r.device_ms
for _ in range(3): solve()
for tag, pre in (("after fill", lambda i: big.fill_(float(i))), ("back-to-back", lambda i: None)):
    ks = []
    for i in range(60):
        pre(i); ks.append(solve())
    ks.sort()
    print(tag, "min %.2f median %.2f max %.2f slow(>2.5ms) %d/60" % (ks[0], ks[30], ks[-1], sum(k > 2.5 for k in ks)), flush=True)
