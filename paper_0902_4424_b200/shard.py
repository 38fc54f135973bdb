"""Column sharding of the GPSS iteration.

Rank r of R owns columns [r*p/R, (r+1)*p/R) of K and that slice of x and g.  Per iteration
the ranks exchange two packets (allgather, NCCL inside the iteration graph):

  * the shard's tree values of K d (n per rank), joined by a pairwise tree over the ranks
    (fwd_finish_kernel with the rank values as its partials);
  * after the adjoint: the shard's new x and g slices plus its subtree values of s'z, s's,
    z'z and its clock (2 p/R + 8 per rank).  Every rank projects the gathered x - alpha g
    (the threshold, the escalation loop and the feasibility bumps need all of v), joining
    the secant dots over the ranks in the canonical tree order.

With p/R a power of two the shard trees are subtrees of the canonical column tree, so the
sharded run is bit-identical to the single-GPU run (tests/test_gpu_shard.py on one GPU with
in-process shards; tests/test_shard_gloo.py restates the exchange with gloo on CPU).

This module is the host side: shard planning, the NCCL unique-id exchange over an existing
torch.distributed group, and solver wrappers.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from ._lib import check, ptr

COL_ALIGN = 256  # COL_GROUP: columns per shard must be a multiple of this


@dataclass(frozen=True)
class Shard:
    rank: int
    nranks: int
    col0: int
    p_local: int

    @property
    def cols(self) -> slice:
        return slice(self.col0, self.col0 + self.p_local)


def shard_plan(p: int, nranks: int) -> list[Shard]:
    """Equal contiguous column blocks; raises ValueError when p does not split evenly into
    blocks of a multiple of 256 columns (the engine's column group)."""
    if nranks < 1:
        raise ValueError("shard_plan: nranks must be >= 1")
    if p % nranks:
        raise ValueError(f"shard_plan: p={p} is not divisible by {nranks} ranks")
    pl = p // nranks
    if nranks > 1 and pl % COL_ALIGN:
        raise ValueError(f"shard_plan: {pl} columns per rank is not a multiple of {COL_ALIGN}")
    return [Shard(r, nranks, r * pl, pl) for r in range(nranks)]


def bit_exact(p: int, nranks: int) -> bool:
    """True when the sharded reduction order equals the single-device canonical order."""
    pl = p // nranks
    return p % nranks == 0 and (pl & (pl - 1)) == 0


def rank_tree(parts: np.ndarray) -> np.ndarray:
    """Pairwise tree over the rank axis (axis 0) with power-of-two splits -- the order in
    which fwd_finish_kernel joins the gathered shard values of K d."""
    parts = np.asarray(parts, dtype=np.float64)
    m = parts.shape[0]
    if m == 0:
        return np.zeros(parts.shape[1:])
    if m == 1:
        return parts[0].copy()
    h = 1
    while h * 2 < m:
        h *= 2
    return rank_tree(parts[:h]) + rank_tree(parts[h:])


def exchange_id(pg, rank: int, make_id=None) -> bytes:
    """Rank 0 creates the NCCL unique id (l1g_comm_unique_id) and broadcasts its 128 bytes
    over the torch.distributed group `pg` (gloo: CPU tensor; nccl: CUDA tensor)."""
    import torch
    nbytes = 128
    if rank == 0:
        if make_id is None:
            buf = (C.c_uint8 * nbytes)()
            check(L.load().l1g_comm_unique_id(C.cast(buf, C.c_void_p)), "comm_unique_id")
            raw = bytes(buf)
        else:
            raw = bytes(make_id())
        if len(raw) != nbytes:
            raise ValueError("NCCL unique id must be 128 bytes")
        t = torch.tensor(list(raw), dtype=torch.uint8)
    else:
        t = torch.zeros(nbytes, dtype=torch.uint8)
    if pg.get_backend() == "nccl":
        t = t.cuda()
    pg.broadcast(t, src=0)
    return bytes(t.cpu().tolist())


class Comm:
    """NCCL communicator of the sharded solver (one rank per process and device)."""

    def __init__(self, ctx, rank: int, nranks: int, uid: bytes):
        self.h = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        check(L.load().l1g_comm_create(ctx.h, rank, nranks, C.cast(buf, C.c_void_p),
                                       C.byref(self.h)), "comm_create")
        self.rank, self.nranks = rank, nranks

    def close(self):
        if self.h:
            L.load().l1g_comm_destroy(self.h)
            self.h = C.c_void_p()


class HostComm:
    """Sharded-solver communicator over the caller's own host allgather (no NCCL): the
    engine stages every exchange through pinned host memory and calls `allgather` from a host
    node of its iteration graphs.  With a torch.distributed group (e.g. gloo) this runs the
    product's multi-rank path in processes that share one GPU (tests/test_gpu_shard_mp.py)."""

    def __init__(self, ctx, rank: int, nranks: int, pg=None, allgather=None):
        self.rank, self.nranks = rank, nranks
        self.errors = []
        if allgather is None:
            allgather = torch_allgather(pg, nranks)

        def _fn(send_p, recv_p, count, user):
            try:
                send = np.ctypeslib.as_array(send_p, shape=(count,))
                recv = np.ctypeslib.as_array(recv_p, shape=(nranks * count,))
                allgather(send, recv)
                return 0
            except BaseException as e:  # reported by the solver as a runtime failure
                self.errors.append(e)
                return 1

        self._fn = L.ALLGATHER_FN(_fn)  # kept alive as long as the communicator
        self.h = C.c_void_p()
        check(L.load().l1g_comm_create_host(ctx.h, rank, nranks, self._fn, None,
                                            C.byref(self.h)), "comm_create_host")

    def close(self):
        if self.h:
            L.load().l1g_comm_destroy(self.h)
            self.h = C.c_void_p()


def torch_allgather(pg, nranks: int):
    """recv[r * count:(r + 1) * count] = rank r's send, over a torch.distributed group."""
    import torch

    def ag(send, recv):
        src = torch.from_numpy(send.copy())
        out = [torch.empty_like(src) for _ in range(nranks)]
        pg.all_gather(out, src)
        recv[:] = torch.cat(out).numpy()
    return ag


def create_group_solver(ops, y, rho, cfg):
    """In-process shards on one device (ops[r] = columns of shard r), run in lockstep."""
    arr = (C.c_void_p * len(ops))(*[o.h for o in ops])
    h = C.c_void_p()
    yy = np.ascontiguousarray(y, dtype=np.float64)
    check(L.load().l1g_solver_create_group(arr, len(ops), ptr(yy), rho, C.byref(cfg._c()),
                                           C.byref(h)), "solver_create_group")
    return h


def create_sharded_solver(op, comm, y, rho, cfg):
    """This process's shard of a sharded solve (comm: Comm over NCCL, or HostComm)."""
    h = C.c_void_p()
    yy = np.ascontiguousarray(y, dtype=np.float64)
    check(L.load().l1g_solver_create_sharded(op.h, comm.h, ptr(yy), rho, C.byref(cfg._c()),
                                             C.byref(h)), "solver_create_sharded")
    return h


def solve(h, stop, x0=None, trace_cap: int = 0):
    """gp_init + the device-resident gpss_solve loop on a solver handle; returns
    (x, result struct, trace records)."""
    lib = L.load()
    x0a = None if x0 is None else np.ascontiguousarray(x0, dtype=np.float64)
    check(lib.l1g_solver_init(h, ptr(x0a)), "solver_init")
    res = L.ResultC()
    recs = (L.IterRecordC * max(trace_cap, 1))()
    check(lib.l1g_solver_run(h, C.byref(stop._c()), C.byref(res),
                             C.addressof(recs) if trace_cap else None, trace_cap), "solver_run")
    n_rec = min(trace_cap, res.iterations)
    return res, [recs[i] for i in range(n_rec)]


def solver_x(h, p: int) -> np.ndarray:
    x = np.empty(p)
    check(L.load().l1g_solver_get(h, ptr(x), None, None, None, None, None, None), "solver_get")
    return x
