"""The sharded engine with REAL halos on the GPU: world 2 and 4 as separate
processes on the one B200, the collectives over torch.distributed/gloo
through the host-callback communicator (spcg_comm_create_host) -- the same
kernels as the NCCL path (localized gathers, halo pack, reverse halo of the
single-pass symmetric SpMV), another transport.  No kernel waits on another
rank: every exchange is a host round trip.  Checked against the serial
reference CG."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_1010_4639_b200.distributed import (Comm, ShardedMatrix, dist_cg_solve,
                                                      torch_collectives, torch_host_transport)
        from paper_1010_4639_b200.genprob import poisson3d, random_spd, rhs_for, stencil27

        gather, _ = torch_collectives()
        acc = "privatized"
        if case == "p3":
            a = poisson3d(9, 8, 12)
            sm = ShardedMatrix.from_stencil("poisson3d", (9, 8, 12), "csr", rank, world, gather)
        elif case == "p3_empty":
            # 3 z-planes over 4 plane-aligned ranks: one rank owns no rows and
            # must still join every collective of the solve
            a = poisson3d(10, 10, 3)
            sm = ShardedMatrix.from_stencil("poisson3d", (10, 10, 3), "csr", rank, world, gather)
        elif case in ("q27_priv", "q27_atomic"):
            a = stencil27(10, 9, 16)
            sm = ShardedMatrix.from_stencil("stencil27", (10, 9, 16), "scsr", rank, world, gather)
            acc = "atomic" if case == "q27_atomic" else "privatized"
        else:
            a = random_spd(400, 0.03, 7)
            sm = ShardedMatrix.from_host(a, rank, world, gather)
        b, _ = rhs_for(a, seed=5)
        comm = Comm.host(rank, world, *torch_host_transport())
        b_loc = torch.from_numpy(b[sm.row0:sm.row1].copy()).cuda()
        x, res, hist = dist_cg_solve(sm, comm, b_loc, record_history=True, accumulation=acc)
        out = (rank, x.cpu().numpy(), int(res.iterations), float(res.final_relative_residual),
               int(sm.plan.npeers), int(sm.halo.size))
        allx = [None] * world
        dist.all_gather_object(allx, out)
        if rank == 0:
            q.put((a, b, allx))
        comm.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [(w, c) for w in (2, 4)
                                        for c in ("p3", "q27_priv", "q27_atomic", "rand")]
                         + [(4, "p3_empty")])
def test_sharded_world_n_on_one_gpu(case, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    a, b, allx = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    allx = sorted(allx, key=lambda t: t[0])
    x = np.concatenate([t[1] for t in allx])
    its = {t[2] for t in allx}
    assert len(its) == 1, its                      # every rank stops together
    assert all(t[4] >= 1 and t[5] >= 1 for t in allx if t[1].size)  # real halos on every rank
    if case == "p3_empty":
        assert any(t[1].size == 0 for t in allx)
    ref = O.cg_solve("csr", a.row_start, a.col_idx, a.values, b)
    assert abs(its.pop() - ref.iterations) <= max(1, ref.iterations // 100)
    assert np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x) <= 1e-8
    assert allx[0][3] <= 1e-10
