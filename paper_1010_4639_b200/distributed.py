"""Row-sharded CG across the GPUs of one node (new — the
reference has no distribution).

One process per GPU (torchrun).  Rows are split into contiguous blocks; each
rank holds its block as a *localized* matrix handle (owned columns ->
[0, nloc), halo columns -> nloc + position in the sorted halo list).  Per CG
iteration the C++ engine (spcg_dist_cg_solve; per-pass kernels, csrc/dist.cuh)
runs q = A p_ext, r -= alpha q, x += alpha p / p = r + beta p, sums the two
dot products with ncclAllReduce and exchanges the halo of the new p with
ncclSend/ncclRecv; all scalars stay on the device and are bitwise identical
on every rank, so all ranks stop at the same iteration.

Host-side logic here is plain numpy + torch.distributed object collectives
(works with the gloo backend on CPU, which tests/test_distributed.py uses):
  * `row_partition`  — contiguous, balanced by stored entries (+ optional
    alignment, e.g. whole z-planes of a stencil);
  * `localize_columns` — the halo numbering (also done in C for device
    handles; both must agree);
  * `halo_plan` — receive lists by owner and the matching send lists.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N


# ---- partition & plan (host logic) ---------------------------------------------
def row_partition(n: int, nranks: int, row_start: np.ndarray | None = None,
                  align: int = 1) -> np.ndarray:
    """Boundaries b[0..nranks] of contiguous row blocks.  Balanced by stored
    entries + rows when offsets are given, by rows otherwise; every interior
    boundary is a multiple of `align` (rounded to the nearest)."""
    if nranks < 1:
        raise ValueError("nranks must be >= 1")
    b = np.zeros(nranks + 1, dtype=np.int64)
    b[-1] = n
    if row_start is not None:
        w = np.asarray(row_start, dtype=np.int64) + np.arange(n + 1, dtype=np.int64)
        for k in range(1, nranks):
            b[k] = int(np.searchsorted(w, (w[-1] * k) // nranks))
    else:
        for k in range(1, nranks):
            b[k] = (n * k) // nranks
    if align > 1:
        b[1:-1] = np.clip(np.rint(b[1:-1] / align).astype(np.int64) * align, 0, n)
    return np.maximum.accumulate(b)


def localize_columns(cols: np.ndarray, row0: int, row1: int) -> tuple[np.ndarray, np.ndarray]:
    """(local column ids, sorted halo global ids) — the numbering the C
    library's spcg_matrix_localize produces."""
    cols = np.asarray(cols, dtype=np.int64)
    own = (cols >= row0) & (cols < row1)
    halo = np.unique(cols[~own])
    loc = np.empty_like(cols)
    nloc = row1 - row0
    loc[own] = cols[own] - row0
    loc[~own] = nloc + np.searchsorted(halo, cols[~own])
    return loc, halo


@dataclass
class HaloPlan:
    peers: np.ndarray      # int32, ascending ranks exchanged with
    recv_off: np.ndarray   # int64[npeers+1] into the halo list
    send_off: np.ndarray   # int64[npeers+1] into send_idx
    send_idx: np.ndarray   # int32 local rows to send, grouped by peer

    @property
    def npeers(self) -> int:
        return int(self.peers.shape[0])


def halo_plan(halo: np.ndarray, bounds: np.ndarray, rank: int, all_gather_object) -> HaloPlan:
    """Build the exchange plan.  `all_gather_object(obj) -> list` gathers one
    picklable object per rank (torch.distributed.all_gather_object)."""
    halo = np.asarray(halo, dtype=np.int64)
    owners = np.searchsorted(bounds, halo, side="right") - 1
    nranks = len(bounds) - 1
    if halo.size and (owners.min() < 0 or owners.max() >= nranks or (owners == rank).any()):
        raise ValueError("halo column outside the partition or owned by this rank")
    want = {int(q): halo[owners == q] for q in np.unique(owners)}
    everyone = all_gather_object(want)
    row0 = int(bounds[rank])
    send = {q: np.asarray(everyone[q][rank], dtype=np.int64) - row0
            for q in range(nranks) if q != rank and rank in everyone[q]}
    peers = sorted(set(want) | set(send))
    recv_off = [0]
    send_off = [0]
    send_idx = []
    for q in peers:
        recv_off.append(recv_off[-1] + (want[q].size if q in want else 0))
        s = send.get(q, np.empty(0, dtype=np.int64))
        send_off.append(send_off[-1] + s.size)
        send_idx.append(s)
    # receive order must follow the sorted halo list
    if halo.size and not np.array_equal(
            np.concatenate([want[q] for q in peers if q in want]), halo):
        raise AssertionError("halo is not grouped by ascending owner")
    si = np.concatenate(send_idx) if send_idx else np.empty(0, dtype=np.int64)
    if si.size and (si.min() < 0 or si.max() >= bounds[rank + 1] - row0):
        raise ValueError("a peer requested rows this rank does not own")
    return HaloPlan(np.asarray(peers, dtype=np.int32), np.asarray(recv_off, dtype=np.int64),
                    np.asarray(send_off, dtype=np.int64), si.astype(np.int32))


# ---- communicator ----------------------------------------------------------------
class Comm:
    """NCCL communicator of the C library, bootstrapped over torch.distributed."""

    def __init__(self, rank: int, world: int, broadcast_object=None, nccl: bool | None = None):
        """nccl: make an NCCL communicator (default: when world > 1); at
        world 1 `nccl=True` builds a real one-rank NCCL communicator so the
        ncclAllReduce path runs on a single GPU."""
        self.rank, self.world = rank, world
        lib = N.load()
        h = ctypes.c_void_p()
        if nccl is None:
            nccl = world > 1
        if broadcast_object is None:
            broadcast_object = lambda o: o  # noqa: E731 - world 1
        if nccl:
            idbuf = (ctypes.c_ubyte * 128)()
            if rank == 0:
                N.check(lib.spcg_comm_unique_id(idbuf), "spcg_comm_unique_id")
            data = broadcast_object(bytes(idbuf) if rank == 0 else None)
            idbuf = (ctypes.c_ubyte * 128).from_buffer_copy(data)
            N.check(lib.spcg_comm_create(world, rank, idbuf, ctypes.byref(h)), "spcg_comm_create")
        else:
            N.check(lib.spcg_comm_create(1, 0, None, ctypes.byref(h)), "spcg_comm_create")
        self._h = h

    @classmethod
    def host(cls, rank: int, world: int, allreduce, sendrecv) -> "Comm":
        """Communicator over the caller's own transport (spcg_comm_create_host):
        allreduce(np.ndarray) sums in place over all ranks; sendrecv(peers,
        send, send_off, recv_off) -> recv exchanges per-peer slices.  The
        engine stages data through host memory, so this is for bring-up and
        tests (e.g. several ranks on one GPU over gloo), not for speed."""
        import numpy as _np

        def _ar(buf, n, _user):
            try:
                a = _np.ctypeslib.as_array(buf, shape=(n,))
                a[:] = allreduce(a.copy())
                return 0
            except Exception:  # noqa: BLE001 - reported to the C side as failure
                import traceback

                traceback.print_exc()
                return 1

        def _sr(npeers, peers, send, soff, recv, roff, _user):
            try:
                pe = _np.ctypeslib.as_array(peers, shape=(npeers,)).copy()
                so = _np.ctypeslib.as_array(soff, shape=(npeers + 1,)).copy()
                ro = _np.ctypeslib.as_array(roff, shape=(npeers + 1,)).copy()
                sv = _np.ctypeslib.as_array(send, shape=(max(1, int(so[-1])),))[: int(so[-1])].copy()
                out = sendrecv(pe, sv, so, ro)
                if int(ro[-1]):
                    _np.ctypeslib.as_array(recv, shape=(int(ro[-1]),))[:] = out
                return 0
            except Exception:  # noqa: BLE001
                import traceback

                traceback.print_exc()
                return 1

        self = cls.__new__(cls)
        self.rank, self.world = rank, world
        self._cb = (N.HOST_ALLREDUCE_FN(_ar), N.HOST_SENDRECV_FN(_sr))  # keep alive
        h = ctypes.c_void_p()
        N.check(N.load().spcg_comm_create_host(world, rank, ctypes.cast(self._cb[0], ctypes.c_void_p),
                                               ctypes.cast(self._cb[1], ctypes.c_void_p), None,
                                               ctypes.byref(h)), "spcg_comm_create_host")
        self._h = h
        return self

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h is not None and self._h.value:
            N.load().spcg_comm_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def torch_host_transport(rank_order: bool = False):
    """(allreduce, sendrecv) callables for Comm.host over the default
    torch.distributed process group (any backend, e.g. gloo on CPU tensors).
    rank_order: sum the ranks' partials in rank order (all-gather + ordered
    sum), the order of the device-initiated transport's mailbox sum."""
    import torch
    import torch.distributed as dist

    def allreduce(a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        if rank_order:
            parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
            dist.all_gather(parts, t)
            acc = parts[0].numpy().copy()
            for q in parts[1:]:
                acc = acc + q.numpy()
            return acc
        dist.all_reduce(t)
        return t.numpy()

    def sendrecv(peers, send, soff, roff):
        reqs, bufs = [], []
        out = np.zeros(int(roff[-1]))
        for k, peer in enumerate(peers):
            s0, s1, r0, r1 = int(soff[k]), int(soff[k + 1]), int(roff[k]), int(roff[k + 1])
            if s1 > s0:
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(send[s0:s1])), int(peer)))
            if r1 > r0:
                t = torch.empty(r1 - r0, dtype=torch.float64)
                bufs.append((r0, r1, t))
                reqs.append(dist.irecv(t, int(peer)))
        for rq in reqs:
            rq.wait()
        for r0, r1, t in bufs:
            out[r0:r1] = t.numpy()
        return out

    return allreduce, sendrecv


def torch_collectives():
    """(all_gather_object, broadcast_object) over the default process group."""
    import torch.distributed as dist

    def gather(obj):
        out = [None] * dist.get_world_size()
        dist.all_gather_object(out, obj)
        return out

    def bcast(obj):
        box = [obj]
        dist.broadcast_object_list(box, src=0)
        return box[0]

    return gather, bcast


# ---- sharded matrices and the solve ------------------------------------------------
class ShardedMatrix:
    """This rank's localized row block + its halo plan."""

    def __init__(self, dm, row0: int, row1: int, n_global: int, halo: np.ndarray, plan: HaloPlan):
        self.dm, self.row0, self.row1, self.n_global = dm, row0, row1, n_global
        self.halo, self.plan = halo, plan

    @property
    def nloc(self) -> int:
        return self.row1 - self.row0

    @staticmethod
    def _finish(dm, bounds, rank, all_gather_object):
        lib = N.load()
        nh = ctypes.c_int64()
        N.check(lib.spcg_matrix_localize(dm.handle, ctypes.byref(nh)), "spcg_matrix_localize")
        halo = np.empty(nh.value, dtype=np.int64)
        N.check(lib.spcg_matrix_halo(dm.handle, halo.ctypes.data if halo.size else None),
                "spcg_matrix_halo")
        plan = halo_plan(halo, bounds, rank, all_gather_object)
        return ShardedMatrix(dm, int(bounds[rank]), int(bounds[rank + 1]), int(bounds[-1]), halo,
                             plan)

    @staticmethod
    def _stencil_rows(kind, dims, fmt, bounds, rank):
        from .device import DeviceMatrix

        kinds = {"poisson2d": N.GEN_POISSON2D, "poisson3d": N.GEN_POISSON3D,
                 "stencil27": N.GEN_STENCIL27}
        d = list(dims) + [1] * (3 - len(dims))
        h = ctypes.c_void_p()
        N.check(N.load().spcg_matrix_generate_rows(kinds[kind], DeviceMatrix.FORMATS[fmt], d[0], d[1],
                                                   d[2], int(bounds[rank]), int(bounds[rank + 1]),
                                                   ctypes.byref(h)), "spcg_matrix_generate_rows")
        dm = DeviceMatrix(h.value, DeviceMatrix.FORMATS[fmt], 0, 0)
        dm._refresh()
        return dm

    @staticmethod
    def stencil_bounds(kind: str, dims, world: int, align_planes: bool = True) -> np.ndarray:
        d = list(dims) + [1] * (3 - len(dims))
        n = d[0] * d[1] * d[2]
        plane = d[0] if kind == "poisson2d" else d[0] * d[1]
        return row_partition(n, world, align=plane if align_planes else 1)

    @classmethod
    def group_from_stencil(cls, kind: str, dims, fmt: str, world: int,
                           align_planes: bool = True) -> list["ShardedMatrix"]:
        """ALL `world` shards of a stencil in this process, on the current
        device (virtual ranks of spcg_dist_group_solve): the halo plans are
        built from every shard's halo without a process group."""
        bounds = cls.stencil_bounds(kind, dims, world, align_planes)
        return cls._group_finish([cls._stencil_rows(kind, dims, fmt, bounds, r)
                                  for r in range(world)], bounds)

    @staticmethod
    def _localize(dm):
        lib = N.load()
        nh = ctypes.c_int64()
        N.check(lib.spcg_matrix_localize(dm.handle, ctypes.byref(nh)), "spcg_matrix_localize")
        halo = np.empty(nh.value, dtype=np.int64)
        N.check(lib.spcg_matrix_halo(dm.handle, halo.ctypes.data if halo.size else None),
                "spcg_matrix_halo")
        return halo

    @classmethod
    def _group_finish(cls, dms, bounds) -> list["ShardedMatrix"]:
        halos = [cls._localize(dm) for dm in dms]
        wants = []
        for h in halos:
            owners = np.searchsorted(bounds, h, side="right") - 1
            wants.append({int(q): h[owners == q] for q in np.unique(owners)})
        out = []
        for r, (dm, h) in enumerate(zip(dms, halos)):
            plan = halo_plan(h, bounds, r, lambda _w: wants)
            out.append(ShardedMatrix(dm, int(bounds[r]), int(bounds[r + 1]), int(bounds[-1]), h,
                                     plan))
        return out

    @classmethod
    def group_from_host(cls, a, world: int) -> list["ShardedMatrix"]:
        """All shards of a host CsrMatrix / SymHalfMatrix in this process."""
        bounds = row_partition(a.n, world, a.row_start)
        dms = [cls._host_rows(a, bounds, r) for r in range(world)]
        return cls._group_finish(dms, bounds)

    @classmethod
    def from_stencil(cls, kind: str, dims, fmt: str, rank: int, world: int, all_gather_object,
                     align_planes: bool = True) -> "ShardedMatrix":
        """Rows of an in-HBM generated stencil; blocks aligned to whole
        z-planes (x-y planes for 2-D) so each halo is one plane per side."""
        from .device import DeviceMatrix

        kinds = {"poisson2d": N.GEN_POISSON2D, "poisson3d": N.GEN_POISSON3D,
                 "stencil27": N.GEN_STENCIL27}
        d = list(dims) + [1] * (3 - len(dims))
        n = d[0] * d[1] * d[2]
        plane = d[0] if kind == "poisson2d" else d[0] * d[1]
        bounds = row_partition(n, world, align=plane if align_planes else 1)
        h = ctypes.c_void_p()
        N.check(N.load().spcg_matrix_generate_rows(kinds[kind], DeviceMatrix.FORMATS[fmt], d[0], d[1],
                                                   d[2], int(bounds[rank]), int(bounds[rank + 1]),
                                                   ctypes.byref(h)), "spcg_matrix_generate_rows")
        dm = DeviceMatrix(h.value, DeviceMatrix.FORMATS[fmt], 0, 0)
        dm._refresh()
        return cls._finish(dm, bounds, rank, all_gather_object)

    @classmethod
    def from_host(cls, a, rank: int, world: int, all_gather_object) -> "ShardedMatrix":
        """Rows of a host CsrMatrix / SymHalfMatrix (SCSR also ships the rows
        of L^T, needed by the owner-computes transpose)."""
        from .core import CsrMatrix, SymHalfMatrix, build_csr_from_triplets
        from .device import DeviceMatrix

        bounds = row_partition(a.n, world, a.row_start)
        return cls._finish(cls._host_rows(a, bounds, rank), bounds, rank, all_gather_object)

    @staticmethod
    def _host_rows(a, bounds, rank):
        from .core import CsrMatrix, SymHalfMatrix, build_csr_from_triplets
        from .device import DeviceMatrix

        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        rs = np.ascontiguousarray(a.row_start, dtype=np.int64)
        k0, k1 = int(rs[r0]), int(rs[r1])
        ci = np.ascontiguousarray(a.col_idx[k0:k1], dtype=np.int64)
        v = np.ascontiguousarray(a.values[k0:k1], dtype=np.float64)
        ptrA = np.ascontiguousarray(rs[r0:r1 + 1])
        keep = [ptrA, ci, v]
        if isinstance(a, SymHalfMatrix):
            fmt = N.FMT_SCSR
            lr, lc, lv = a.strict_lower
            t = build_csr_from_triplets((lc, lr, lv), a.n)  # rows of L^T
            tb0, tb1 = int(t.row_start[r0]), int(t.row_start[r1])
            ptrB = np.ascontiguousarray(t.row_start[r0:r1 + 1], dtype=np.int64)
            ciB = np.ascontiguousarray(t.col_idx[tb0:tb1], dtype=np.int64)
            vB = np.ascontiguousarray(t.values[tb0:tb1], dtype=np.float64)
            keep += [ptrB, ciB, vB]
            b_args = (int(vB.size), ptrB.ctypes.data, ciB.ctypes.data if ciB.size else None,
                      vB.ctypes.data if vB.size else None)
        elif isinstance(a, CsrMatrix):
            fmt = N.FMT_CSR
            b_args = (0, None, None, None)
        else:
            raise TypeError(f"cannot shard {type(a).__name__}")
        h = ctypes.c_void_p()
        N.check(N.load().spcg_matrix_create_rows(
            fmt, a.n, r0, r1, int(v.size), ptrA.ctypes.data, ci.ctypes.data if ci.size else None,
            v.ctypes.data if v.size else None, *b_args, ctypes.byref(h)), "spcg_matrix_create_rows")
        dm = DeviceMatrix(h.value, fmt, 0, 0)
        dm._refresh()
        return dm

    def spmv_ext(self, x_ext):
        """y_loc = A_loc x_ext for an extended vector (own + halo values)."""
        import torch

        y = torch.empty(self.nloc, dtype=torch.float64, device=x_ext.device)
        N.check(N.load().spcg_spmv(self.dm.handle, x_ext.data_ptr(), y.data_ptr(), N.ACC_PRIVATIZED,
                                   torch.cuda.current_stream().cuda_stream), "spcg_spmv")
        return y


def dist_cg_solve(sm: ShardedMatrix, comm: Comm, b_loc, x0_loc=None, tol: float = 1e-10,
                  max_iter: int | None = None, record_history: bool = False,
                  recompute_final_residual: bool = True, timing: bool = False,
                  accumulation: str = "privatized"):
    """One rank's part of the sharded solve.  b_loc / x0_loc: CUDA tensors
    of this rank's rows.  accumulation (symmetric-half shards): "privatized"
    (owner-computes with the stored L^T rows, deterministic) or "atomic"
    (one pass over L+D; transposed contributions to other ranks' rows go back
    through a reverse halo).  Returns (x_loc, CgResultC, history or None)."""
    import torch

    p = sm.plan
    mi = max_iter if max_iter else max(1, sm.n_global)
    x = torch.empty(sm.nloc, dtype=torch.float64, device=b_loc.device)
    hist = torch.empty(mi if record_history else 1, dtype=torch.float64, device=b_loc.device)
    o = N.CgOptionsC(tol=float(tol), max_iter=int(mi), record_history=int(record_history),
                     recompute_final_residual=int(recompute_final_residual),
                     accumulation=N.ACC_ATOMIC if accumulation == "atomic" else N.ACC_PRIVATIZED,
                     engine=2, timing=int(timing))
    res = N.CgResultC()

    def ptr(a):
        return a.ctypes.data if a.size else None

    rc = N.load().spcg_dist_cg_solve(
        sm.dm.handle, comm.handle, p.npeers, ptr(p.peers), ptr(p.recv_off), ptr(p.send_off),
        ptr(p.send_idx), b_loc.data_ptr(), x0_loc.data_ptr() if x0_loc is not None else None,
        x.data_ptr(), hist.data_ptr() if record_history else None, o, res,
        torch.cuda.current_stream().cuda_stream)
    from .solver import _BREAKDOWN

    if rc in _BREAKDOWN:
        raise _BREAKDOWN[rc](int(res.fail_iteration))
    N.check(rc, "spcg_dist_cg_solve")
    h = hist[: res.iterations].cpu().numpy() if record_history else None
    return x, res, h


# ---- device-initiated transport (spcg_dist_plan_*) ---------------------------------
class P2PPlan:
    """One rank's device-initiated transport: the two scalar all-reduces of
    every iteration through epoch-tagged mailboxes in peer memory and the
    halo of p stored by pass C straight into the neighbours' p_ext (no host
    collective per iteration).  Bootstrap: export() -> all-gather the blobs
    in rank order -> connect(blobs).  Ranks sharing this process and device
    connect by plain pointers and can be solved together in one launch per
    pass (`group_solve`)."""

    BLOB = 1024  # SPCG_P2P_BLOB_BYTES

    def __init__(self, sm: "ShardedMatrix", rank: int, world: int):
        p = sm.plan
        self.sm, self.rank, self.world = sm, rank, world
        lib = N.load()
        h = ctypes.c_void_p()

        def ptr(a):
            return a.ctypes.data if a.size else None

        N.check(lib.spcg_dist_plan_create(sm.dm.handle, rank, world, p.npeers, ptr(p.peers),
                                          ptr(p.recv_off), ptr(p.send_off), ptr(p.send_idx),
                                          ctypes.byref(h)), "spcg_dist_plan_create")
        self._h = h

    @property
    def handle(self):
        return self._h

    def export(self) -> bytes:
        buf = (ctypes.c_ubyte * self.BLOB)()
        N.check(N.load().spcg_dist_plan_export(self._h, buf), "spcg_dist_plan_export")
        return bytes(buf)

    def connect(self, blobs: list[bytes]):
        if len(blobs) != self.world or any(len(b) != self.BLOB for b in blobs):
            raise ValueError("connect needs one export blob per rank, in rank order")
        buf = (ctypes.c_ubyte * (self.BLOB * self.world)).from_buffer_copy(b"".join(blobs))
        N.check(N.load().spcg_dist_plan_connect(self._h, buf), "spcg_dist_plan_connect")

    def solve(self, b_loc, x0_loc=None, tol: float = 1e-10, max_iter: int | None = None,
              record_history: bool = False, recompute_final_residual: bool = True,
              timing: bool = False, accumulation: str = "privatized"):
        """This rank's share of the solve (one process per GPU)."""
        import torch

        sm = self.sm
        mi = max_iter if max_iter else max(1, sm.n_global)
        x = torch.empty(sm.nloc, dtype=torch.float64, device=b_loc.device)
        hist = torch.empty(mi if record_history else 1, dtype=torch.float64, device=b_loc.device)
        o = _options(tol, mi, record_history, recompute_final_residual, timing, accumulation)
        res = N.CgResultC()
        rc = N.load().spcg_dist_plan_solve(
            self._h, b_loc.data_ptr(), x0_loc.data_ptr() if x0_loc is not None else None,
            x.data_ptr(), hist.data_ptr() if record_history else None, o, res,
            torch.cuda.current_stream().cuda_stream)
        _raise(rc, res, "spcg_dist_plan_solve")
        return x, res, (hist[: res.iterations].cpu().numpy() if record_history else None)

    def close(self):
        if self._h is not None and self._h.value:
            N.load().spcg_dist_plan_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _options(tol, mi, record_history, recompute_final_residual, timing, accumulation):
    return N.CgOptionsC(tol=float(tol), max_iter=int(mi), record_history=int(record_history),
                        recompute_final_residual=int(recompute_final_residual),
                        accumulation=N.ACC_ATOMIC if accumulation == "atomic" else N.ACC_PRIVATIZED,
                        engine=2, timing=int(timing))


def _raise(rc, res, what):
    from .solver import _BREAKDOWN

    if rc in _BREAKDOWN:
        raise _BREAKDOWN[rc](int(res.fail_iteration))
    N.check(rc, what)


def connect_all(plans: list[P2PPlan]):
    """Connect the plans of ranks that all live in this process."""
    blobs = [p.export() for p in plans]
    for p in plans:
        p.connect(blobs)


def group_plans(shards: list["ShardedMatrix"]) -> list[P2PPlan]:
    plans = [P2PPlan(sm, r, len(shards)) for r, sm in enumerate(shards)]
    connect_all(plans)
    return plans


def group_solve(plans: list[P2PPlan], b_locs, x0_locs=None, tol: float = 1e-10,
                max_iter: int | None = None, record_history: bool = False,
                recompute_final_residual: bool = True, timing: bool = False,
                accumulation: str = "privatized"):
    """Every rank of `plans` (this process, this device) in ONE launch per
    pass: the device-initiated protocol with all its waits inside single
    launches.  Returns ([x_loc per rank], [CgResultC per rank], rank 0's
    history or None)."""
    import torch

    R = len(plans)
    n_global = plans[0].sm.n_global
    mi = max_iter if max_iter else max(1, n_global)
    dev = b_locs[0].device
    xs = [torch.empty(p.sm.nloc, dtype=torch.float64, device=dev) for p in plans]
    hist = torch.empty(mi if record_history else 1, dtype=torch.float64, device=dev)
    o = _options(tol, mi, record_history, recompute_final_residual, timing, accumulation)
    res = (N.CgResultC * R)()
    P = (ctypes.c_void_p * R)(*[p.handle.value for p in plans])
    B = (ctypes.c_void_p * R)(*[b.data_ptr() for b in b_locs])
    X = (ctypes.c_void_p * R)(*[x.data_ptr() for x in xs])
    X0 = (ctypes.c_void_p * R)(*[x.data_ptr() for x in x0_locs]) if x0_locs is not None else None
    vp = ctypes.c_void_p
    rc = N.load().spcg_dist_group_solve(
        R, ctypes.cast(P, vp), ctypes.cast(B, vp), ctypes.cast(X0, vp) if X0 is not None else None,
        ctypes.cast(X, vp), hist.data_ptr() if record_history else None, o, ctypes.cast(res, vp),
        torch.cuda.current_stream().cuda_stream)
    _raise(rc, res[0], "spcg_dist_group_solve")
    return xs, list(res), (hist[: res[0].iterations].cpu().numpy() if record_history else None)
