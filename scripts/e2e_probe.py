"""(dev) per-solve e2e overhead of spcg_cg_solve_host on F: engine 0 (auto,
with the engine-6 guard) vs engine 6 (no guard), CUDA events around the
host call vs the kernel's own device time."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1010_4639_b200 import _native as N  # noqa: E402
from paper_1010_4639_b200.genprob import fem_mesh, rhs_for  # noqa: E402

F = fem_mesh()
b, _ = rhs_for(F, seed=1)
dm = F.device()
lib = N.load()
st = torch.cuda.current_stream()
bh = torch.from_numpy(b).pin_memory()
xh = torch.empty_like(bh).pin_memory()
for eng in (0, 6, 0, 6):
    o = N.CgOptionsC(tol=1e-10, max_iter=0, record_history=0, recompute_final_residual=1,
                     accumulation=1, engine=eng)
    e2e, dev = [], []
    for i in range(30):
        r = N.CgResultC()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        N.check(lib.spcg_cg_solve_host(dm.handle, bh.numpy().ctypes.data, None, xh.numpy().ctypes.data,
                                       None, o, r, st.cuda_stream), "s")
        e1.record(st)
        torch.cuda.synchronize()
        e2e.append(e0.elapsed_time(e1) * 1e3)
        dev.append(r.device_ms * 1e3)
    print("engine", eng, "e2e us %.1f" % np.median(e2e[5:]), "device us %.1f" % np.median(dev[5:]),
          "overhead us %.1f" % (np.median(e2e[5:]) - np.median(dev[5:])), flush=True)
