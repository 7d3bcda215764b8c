"""Row-sharded CG host logic on CPU with the gloo backend, world_size 2.

The partition / halo numbering / exchange plan of paper_1010_4639_b200.distributed
are exercised for real; the per-rank device kernels are emulated with numpy
following the engine's exact structure (csrc/dist.cuh: SpMV over the extended
p = [own | neighbours'], r-update, x/p-update, halo exchange of the new p,
local sums + all-reduce), and the result is compared with the serial
oracle.  The GPU side of the same engine is covered by
tests/test_gpu_dist.py (single rank) — multi-GPU runs need >1 GPU.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sym_rows(a, r0, r1):
    """Rows [r0,r1) of L+D and of L^T (global column ids) for SymHalfMatrix a."""
    from paper_1010_4639_b200.core import build_csr_from_triplets

    lr, lc, lv = a.strict_lower
    t = build_csr_from_triplets((lc, lr, lv), a.n)
    return t


def emulate_rank(rank, world, a, b, bounds, gather, allreduce, exchange, max_iter=None, tol=1e-10,
                 atomic=False, reverse=None):
    """One rank of the sharded CG in numpy (mirrors dist.cuh).  atomic: the
    single-pass symmetric SpMV over L+D only, its transposed scatters into
    halo rows sent back to their owners (reverse halo)."""
    from paper_1010_4639_b200.core import SymHalfMatrix
    from paper_1010_4639_b200.distributed import halo_plan, localize_columns

    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    nloc = r1 - r0
    rs = a.row_start
    segs = [(rs[r0:r1 + 1] - rs[r0], a.col_idx[rs[r0]:rs[r1]], a.values[rs[r0]:rs[r1]])]
    if isinstance(a, SymHalfMatrix) and not atomic:
        t = _sym_rows(a, r0, r1)
        segs.append((t.row_start[r0:r1 + 1] - t.row_start[r0],
                     t.col_idx[t.row_start[r0]:t.row_start[r1]],
                     t.values[t.row_start[r0]:t.row_start[r1]]))
    allc = np.concatenate([s[1] for s in segs])
    _, halo = localize_columns(allc, r0, r1)
    loc = [localize_columns(np.concatenate([s[1], allc]), r0, r1)[0][: s[1].size] for s in segs]
    plan = halo_plan(halo, bounds, rank, gather)
    next_ = nloc + halo.size

    def spmv2(v_ext):
        outs = []
        for (ptr, _, val), ci in zip(segs, loc):
            part = np.zeros(nloc)
            for i in range(nloc):
                acc = 0.0
                for k in range(ptr[i], ptr[i + 1]):
                    acc = acc + val[k] * v_ext[ci[k]]
                part[i] = acc
            outs.append(part)
        return outs[0] if len(outs) == 1 else outs[0] + outs[1]

    def spmv_atomic(v_ext):
        """(q, p.Ap partial): gather over L+D, scatter of the transpose into
        q_ext (ghost slots for halo columns), reverse halo, local p.Ap."""
        ptr, _, val = segs[0]
        ci = loc[0]
        q_ext = np.zeros(next_)
        pq = 0.0
        for i in range(nloc):
            g = 0.0
            dg = 0.0
            for k in range(ptr[i], ptr[i + 1]):
                g = g + val[k] * v_ext[ci[k]]
                if ci[k] != i:
                    q_ext[ci[k]] += val[k] * v_ext[i]
                else:
                    dg = val[k]
            q_ext[i] += g
            pq += v_ext[i] * (2.0 * g - dg * v_ext[i])
        back = reverse(plan, q_ext[nloc:])
        np.add.at(q_ext, plan.send_idx, back)
        return q_ext[:nloc], pq

    bl = b[r0:r1].copy()
    b_norm = np.sqrt(allreduce(float(np.dot(bl, bl))))
    x = np.zeros(nloc)
    r = bl.copy()
    p_ext = np.zeros(next_)          # [own p | neighbours' p]
    p_ext[:nloc] = r
    rr = allreduce(float(np.dot(r, r)))
    p_ext[nloc:] = exchange(plan, p_ext[plan.send_idx])
    mi = max_iter or a.n
    k, alpha = 0, 0.0
    converged = np.sqrt(rr) <= tol * b_norm
    while not converged and k < mi:
        if atomic:                                         # pass A
            q, pq_loc = spmv_atomic(p_ext)
            pq = allreduce(float(pq_loc))
        else:
            q = spmv2(p_ext)
            pq = allreduce(float(np.dot(p_ext[:nloc], q)))
        assert pq > 0
        alpha = rr / pq
        r = r - alpha * q                                  # pass B
        rr_new = allreduce(float(np.dot(r, r)))
        k += 1
        if np.sqrt(rr_new) <= tol * b_norm:
            converged = True
            break
        beta = rr_new / rr
        rr = rr_new
        x = x + alpha * p_ext[:nloc]                       # pass C
        p_ext[:nloc] = r + beta * p_ext[:nloc]
        p_ext[nloc:] = exchange(plan, p_ext[plan.send_idx])
    if converged and k > 0:
        x = x + alpha * p_ext[:nloc]
    return x, k, plan, halo


def _worker(rank, world, port, kind, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1010_4639_b200.core import extract_lower
        from paper_1010_4639_b200.distributed import row_partition, torch_collectives
        from paper_1010_4639_b200.genprob import poisson3d, random_spd, rhs_for

        gather, _ = torch_collectives()
        if kind == "p3":
            a = poisson3d(7, 6, 5)
        elif kind in ("sym", "sym_atomic"):
            a = extract_lower(poisson3d(6, 5, 6))
        else:
            a = random_spd(90, 0.08, 5)
        b, _ = rhs_for(a, seed=3)
        bounds = row_partition(a.n, world, a.row_start)

        def allreduce(v):
            t = torch.tensor([v], dtype=torch.float64)
            dist.all_reduce(t)
            return float(t.item())

        def exchange(plan, send):
            reqs = []
            out = np.zeros(int(plan.recv_off[-1]))
            bufs = []
            for k, peer in enumerate(plan.peers):
                s0, s1 = plan.send_off[k], plan.send_off[k + 1]
                r0, r1 = plan.recv_off[k], plan.recv_off[k + 1]
                if s1 > s0:
                    reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(send[s0:s1])), int(peer)))
                if r1 > r0:
                    t = torch.empty(int(r1 - r0), dtype=torch.float64)
                    bufs.append((r0, r1, t))
                    reqs.append(dist.irecv(t, int(peer)))
            for rq in reqs:
                rq.wait()
            for r0_, r1_, t in bufs:
                out[r0_:r1_] = t.numpy()
            return out

        def reverse(plan, ghosts):
            """Ghost partial sums -> their owners; returns the received values
            aligned with this rank's send list (dist_unpack_add's input)."""
            reqs, bufs = [], []
            out = np.zeros(int(plan.send_off[-1]))
            for k, peer in enumerate(plan.peers):
                s0, s1 = plan.send_off[k], plan.send_off[k + 1]
                r0_, r1_ = plan.recv_off[k], plan.recv_off[k + 1]
                if r1_ > r0_:
                    reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(ghosts[r0_:r1_])),
                                           int(peer)))
                if s1 > s0:
                    t = torch.empty(int(s1 - s0), dtype=torch.float64)
                    bufs.append((s0, s1, t))
                    reqs.append(dist.irecv(t, int(peer)))
            for rq in reqs:
                rq.wait()
            for s0, s1, t in bufs:
                out[s0:s1] = t.numpy()
            return out

        x, k, plan, halo = emulate_rank(rank, world, a, b, bounds, gather, allreduce, exchange,
                                        atomic=kind == "sym_atomic", reverse=reverse)
        xs = [None] * world
        dist.all_gather_object(xs, (rank, x, k, plan.npeers, halo.size))
        if rank == 0:
            q.put((kind, a, b, bounds, xs))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["p3", "sym", "sym_atomic", "rand"])
def test_sharded_cg_world2_matches_serial(kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    kind_, a, b, bounds, xs = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    xs = sorted(xs, key=lambda t: t[0])
    x = np.concatenate([t[1] for t in xs])
    its = {t[2] for t in xs}
    assert len(its) == 1, its  # every rank stops at the same iteration
    if kind in ("sym", "sym_atomic"):
        from paper_1010_4639_b200.core import expand_symmetric

        full = expand_symmetric(a)
    else:
        full = a
    ref = O.cg_solve("csr", full.row_start, full.col_idx, full.values, b)
    assert abs(its.pop() - ref.iterations) <= max(1, ref.iterations // 100)
    assert np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x) <= 1e-8
    assert all(t[3] >= 1 for t in xs)  # both ranks exchange a halo


def test_partition_and_localize():
    from paper_1010_4639_b200.distributed import localize_columns, row_partition
    from paper_1010_4639_b200.genprob import poisson3d

    a = poisson3d(10, 10, 16)
    for world in (1, 2, 4, 8):
        b = row_partition(a.n, world, align=100)
        assert b[0] == 0 and b[-1] == a.n and (np.diff(b) >= 0).all()
        assert all(v % 100 == 0 for v in b)
        assert max(np.diff(b)) - min(np.diff(b)) <= 100
    b = row_partition(a.n, 4, a.row_start)
    r0, r1 = b[1], b[2]
    cols = a.col_idx[a.row_start[r0]:a.row_start[r1]]
    loc, halo = localize_columns(cols, r0, r1)
    assert (halo == np.unique(cols[(cols < r0) | (cols >= r1)])).all()
    nloc = r1 - r0
    back = np.where(loc < nloc, loc + r0, halo[np.clip(loc - nloc, 0, None)])
    assert (back == cols).all()
