"""Multi-GPU plumbing: one process per GPU, fitness cases sharded by rank.

`torch.distributed` only bootstraps: rank 0 creates an NCCL unique id inside
libgsgp_b200.so, it is broadcast over the existing process group, and every
rank joins the library's own NCCL communicator (`gsgp_comm_init`).  After
that `run_evolution` shards the train and test cases contiguously across
ranks (slices aligned to CASE_ALIGN cases) and the per-generation collectives
are two small NCCL allreduces of the canonical SSE — the rows' partial
exponent anchors (max) and their exact fixed-point digit sums (sum) — so the
SSE, and every decision, is bit-identical for any number of ranks (SURVEY
§8e); genomes, plans and survival are recomputed identically on each rank
from the counter RNG.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib, devices
from ._lib import check


CASE_ALIGN = 12288
"""Shard boundaries are multiples of this many cases (engine.cu kCaseAlign:
the lcm of every SSE tile), which keeps the SSE tile partials — and with the
canonical sum the whole run — identical for any number of shards."""


def shard_range(n: int, count: int, index: int, align: int = CASE_ALIGN) -> tuple[int, int]:
    """Contiguous slice [lo, hi) of shard `index` out of `count` (same
    formula as gsgp_shard_range in engine.cu for the default `align`)."""
    def cut(i):
        return n if i >= count else (n * i) // count // align * align
    return cut(index), cut(index + 1)


def init_from_torch(group=None) -> tuple[int, int]:
    """Create the library's NCCL communicator over the ranks of an
    initialised torch.distributed group; returns (world, rank)."""
    import torch.distributed as td
    world, rank = td.get_world_size(group), td.get_rank(group)
    lib = _lib.load()
    uid = (C.c_ubyte * 128)()
    if rank == 0:
        check(lib.gsgp_comm_unique_id(uid))
    payload = [bytes(uid)]
    td.broadcast_object_list(payload, src=0, group=group)
    buf = (C.c_ubyte * 128).from_buffer_copy(payload[0])
    devices.activate(None)
    check(lib.gsgp_comm_init(world, rank, buf))
    devices._process_comm = True
    return world, rank


HOST_ALLREDUCE = C.CFUNCTYPE(None, C.c_void_p, C.c_int64, C.c_int32)
_host_cb = None   # keep the ctypes callback alive while the library holds it


def init_host_exchange(group=None) -> tuple[int, int]:
    """Test transport: the engine's collectives go through host memory and
    torch.distributed (e.g. gloo) instead of NCCL, so several ranks can share
    one GPU (`gsgp_comm_init_host`).  Same partitioning and exchanged values
    as the NCCL path; runs use direct launches instead of a CUDA graph."""
    import torch
    import torch.distributed as td
    global _host_cb
    world, rank = td.get_world_size(group), td.get_rank(group)
    # engine.cu HostRed: 0 fp64 sum, 1 int32 sum, 2 uint64 sum, 3 int32 max
    kinds = {0: (np.float64, 8, td.ReduceOp.SUM), 1: (np.int32, 4, td.ReduceOp.SUM),
             2: (np.uint64, 8, td.ReduceOp.SUM), 3: (np.int32, 4, td.ReduceOp.MAX)}

    def allreduce(ptr, count, kind):
        npt, esz, op = kinds[int(kind)]
        buf = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_ubyte)), shape=(count * esz,))
        arr = buf.view(npt)
        # uint64 digit sums travel as int64: two's-complement addition is the
        # same bits (the sums stay far below 2^63)
        t = torch.from_numpy(arr.view(np.int64).copy() if npt is np.uint64 else arr.copy())
        td.all_reduce(t, op=op, group=group)
        arr[:] = t.numpy().view(npt) if npt is np.uint64 else t.numpy()

    _host_cb = HOST_ALLREDUCE(allreduce)
    devices.activate(None)
    check(_lib.load().gsgp_comm_init_host(world, rank, C.cast(_host_cb, C.c_void_p)))
    devices._process_comm = True
    return world, rank


def destroy() -> None:
    check(_lib.load().gsgp_comm_destroy())
    devices._process_comm = False


def gather_elite_semantics(result, n_train: int, group=None) -> np.ndarray:
    """Assemble the full elite train semantics from every rank's slice."""
    import torch
    import torch.distributed as td
    lo, hi = result.device["shard_train_range"]
    local = torch.from_numpy(np.ascontiguousarray(result.elite_train_semantics[lo:hi]))
    parts = [None] * td.get_world_size(group)
    td.all_gather_object(parts, (lo, hi, local.numpy()), group=group)
    full = np.zeros(n_train)
    for a, b, vals in parts:
        full[a:b] = vals
    return full
