import sys; sys.path.insert(0,'.')
import torch
from paper_1010_4639_b200 import _native as N
from paper_1010_4639_b200.genprob import poisson2d, poisson3d, rhs_for
lib=N.load()
for a in (poisson2d(512,512), poisson3d(64,64,64), poisson2d(400,400)):
    b,_=rhs_for(a,seed=1); bt=torch.from_numpy(b).cuda(); dm=a.device(); x=torch.empty_like(bt)
    for eng in (5,6):
        o=N.CgOptionsC(tol=1e-10,max_iter=0,record_history=0,recompute_final_residual=1,accumulation=1,engine=eng)
        r=N.CgResultC(); rc=lib.spcg_cg_solve(dm.handle,bt.data_ptr(),None,x.data_ptr(),None,o,r,0)
        try: N.check(rc,'s'); print(a.n, eng, 'ok', r.iterations, r.device_ms*1e3/r.iterations)
        except Exception as e: print(a.n, eng, e)
