"""The device-initiated transport of the sharded engine (csrc/dist.cuh,
`fused`): per-iteration scalar all-reduces through epoch-tagged mailboxes in
peer memory and the halo of p stored by pass C straight into the
neighbours' p_ext, no host collective per iteration.

On one GPU the ranks run as VIRTUAL ranks: every pass is ONE launch over all
ranks' data (spcg_dist_group_solve), so the cross-rank waits (mailbox polls,
halo tags) only ever wait on CTAs of the same launch -- the emulation the
profiling guide prescribes instead of separate per-rank launches that wait on
each other.  Peers are connected by plain device pointers; across GPUs the
same kernels use CUDA-IPC-mapped peer memory (spcg_dist_plan_export /
connect).  Checked against the serial reference CG and, bit for bit, against
the host-callback transport (ranks as processes, all-reduce summed in rank
order) on the same partition."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _case(case, world):
    from paper_1010_4639_b200.distributed import ShardedMatrix
    from paper_1010_4639_b200.genprob import poisson2d, poisson3d, random_spd, stencil27

    acc = "privatized"
    if case == "p3":
        a = poisson3d(20, 18, 32)
        shards = ShardedMatrix.group_from_stencil("poisson3d", (20, 18, 32), "csr", world)
    elif case == "p2":
        a = poisson2d(96, 128)
        shards = ShardedMatrix.group_from_stencil("poisson2d", (96, 128), "csr", world)
    elif case == "p3_empty":
        a = poisson3d(10, 10, 3)
        shards = ShardedMatrix.group_from_stencil("poisson3d", (10, 10, 3), "csr", world)
    elif case in ("q27_priv", "q27_atomic"):
        a = stencil27(12, 10, 24)
        shards = ShardedMatrix.group_from_stencil("stencil27", (12, 10, 24), "scsr", world)
        acc = "atomic" if case == "q27_atomic" else "privatized"
    else:  # unstructured: many send runs -> the generic push kernel
        a = random_spd(600, 0.02, 11)
        shards = ShardedMatrix.group_from_host(a, world)
    return a, shards, acc


@pytest.mark.parametrize("world,case", [(w, c) for w in (2, 4)
                                        for c in ("p3", "p2", "q27_priv", "q27_atomic", "rand")]
                         + [(4, "p3_empty"), (8, "p3"), (3, "rand")])
def test_group_solve_matches_reference(case, world):
    import torch

    from paper_1010_4639_b200.distributed import group_plans, group_solve
    from paper_1010_4639_b200.genprob import rhs_for

    a, shards, acc = _case(case, world)
    b, _ = rhs_for(a, seed=5)
    plans = group_plans(shards)
    bl = [torch.from_numpy(b[s.row0:s.row1].copy()).cuda() for s in shards]
    xs, res, hist = group_solve(plans, bl, record_history=True, accumulation=acc)
    its = {int(r.iterations) for r in res}
    assert len(its) == 1, its  # every rank stops at the same iteration
    x = np.concatenate([v.cpu().numpy() for v in xs])
    ref = O.cg_solve("csr", a.row_start, a.col_idx, a.values, b, record_history=True)
    it = its.pop()
    assert abs(it - ref.iterations) <= max(1, ref.iterations // 100), (it, ref.iterations)
    assert np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x) <= 1e-8
    assert all(r.converged and r.final_relative_residual <= 1e-10 for r in res)
    assert len(hist) == it
    assert np.allclose(hist[:30], ref.residual_history[:30], rtol=1e-8)
    # the protocol is deterministic: a second solve is bitwise the first
    # (sequence counters continue across solves on every rank)
    xs2, res2, _ = group_solve(plans, bl, accumulation=acc)
    if acc == "privatized":
        assert all((u == v).all() for u, v in zip(xs, xs2))
    assert int(res2[0].iterations) == it


def test_group_solve_x0_truncation_and_zero_rhs():
    import torch

    from paper_1010_4639_b200.distributed import ShardedMatrix, group_plans, group_solve
    from paper_1010_4639_b200.genprob import poisson3d, rhs_for

    a = poisson3d(16, 12, 24)
    shards = ShardedMatrix.group_from_stencil("poisson3d", (16, 12, 24), "csr", 4)
    plans = group_plans(shards)
    b, _ = rhs_for(a, seed=2)
    x0 = np.random.default_rng(3).standard_normal(a.n)
    cut = lambda v: [torch.from_numpy(v[s.row0:s.row1].copy()).cuda() for s in shards]  # noqa: E731
    xs, res, _ = group_solve(plans, cut(b), cut(x0), tol=1e-9)
    ref = O.cg_solve("csr", a.row_start, a.col_idx, a.values, b, x0=x0, tol=1e-9)
    x = np.concatenate([v.cpu().numpy() for v in xs])
    assert abs(res[0].iterations - ref.iterations) <= 1
    assert np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x) <= 1e-8
    xs, res, _ = group_solve(plans, cut(b), max_iter=5, recompute_final_residual=False)
    rt = O.cg_solve("csr", a.row_start, a.col_idx, a.values, b, max_iter=5, recompute=False)
    assert res[0].iterations == 5 and not res[0].converged
    assert abs(res[0].final_relative_residual - rt.final_relative_residual) <= 1e-12
    xs, res, _ = group_solve(plans, cut(np.zeros(a.n)), cut(x0))
    assert res[0].iterations == 0 and all((v == 0).all() for v in xs)


def test_group_solve_launch_count():
    """3 launches per iteration on stencil shards (pass A, B, C: no scalar
    kernels, no host collectives, the halo push fused into pass C)."""
    import torch

    from paper_1010_4639_b200.distributed import ShardedMatrix, group_plans, group_solve
    from paper_1010_4639_b200.genprob import poisson3d, rhs_for

    a = poisson3d(16, 16, 32)
    shards = ShardedMatrix.group_from_stencil("poisson3d", (16, 16, 32), "csr", 4)
    plans = group_plans(shards)
    b, _ = rhs_for(a, seed=1)
    bl = [torch.from_numpy(b[s.row0:s.row1].copy()).cuda() for s in shards]
    _, r1, _ = group_solve(plans, bl, max_iter=32, recompute_final_residual=False)
    _, r2, _ = group_solve(plans, bl, max_iter=64, recompute_final_residual=False)
    assert r2[0].iterations - r1[0].iterations == 32
    assert (r2[0].kernel_launches - r1[0].kernel_launches) == 3 * 32


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _host_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_1010_4639_b200.distributed import (Comm, ShardedMatrix, dist_cg_solve,
                                                      torch_collectives, torch_host_transport)
        from paper_1010_4639_b200.genprob import poisson3d, rhs_for

        gather, _ = torch_collectives()
        a = poisson3d(20, 18, 32)
        sm = ShardedMatrix.from_stencil("poisson3d", (20, 18, 32), "csr", rank, world, gather)
        b, _ = rhs_for(a, seed=5)
        comm = Comm.host(rank, world, *torch_host_transport(rank_order=True))
        x, res, _ = dist_cg_solve(sm, comm, torch.from_numpy(b[sm.row0:sm.row1].copy()).cuda())
        allx = [None] * world
        dist.all_gather_object(allx, (rank, x.cpu().numpy(), int(res.iterations)))
        if rank == 0:
            q.put(allx)
        comm.close()
    finally:
        dist.destroy_process_group()


def test_device_transport_bitwise_equals_host_transport():
    """Same partition, same kernels, rank-ordered sums on both sides: the
    device-initiated transport reproduces the host-callback transport bit
    for bit."""
    import torch

    from paper_1010_4639_b200.distributed import group_plans, group_solve
    from paper_1010_4639_b200.genprob import rhs_for

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_host_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    allx = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    allx = sorted(allx, key=lambda t: t[0])
    a, shards, _ = _case("p3", world)
    b, _ = rhs_for(a, seed=5)
    plans = group_plans(shards)
    xs, res, _ = group_solve(plans, [torch.from_numpy(b[s.row0:s.row1].copy()).cuda()
                                     for s in shards])
    assert int(res[0].iterations) == allx[0][2]
    for (_, xh, _), xd in zip(allx, xs):
        assert (xh == xd.cpu().numpy()).all()


def test_plan_export_blob_and_bad_connect():
    from paper_1010_4639_b200.distributed import P2PPlan, ShardedMatrix

    shards = ShardedMatrix.group_from_stencil("poisson3d", (8, 8, 8), "csr", 2)
    plans = [P2PPlan(s, r, 2) for r, s in enumerate(shards)]
    blobs = [p.export() for p in plans]
    assert all(len(bb) == 1024 for bb in blobs) and blobs[0][:4] == b"PC2P"
    with pytest.raises(ValueError):
        plans[0].connect(blobs[::-1])  # rank order violated
