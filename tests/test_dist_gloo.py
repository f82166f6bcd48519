"""Multi-process check of the case-sharding protocol on CPU.

Two gloo ranks each take their contiguous train/test slice
(`paper_2106_04034_b200.dist.shard_range`, the same formula as the C
library's `gsgp_shard_range`), run the engine arithmetic
(oracle/engine32.run32) on that slice only, and exchange exactly what the
device engine allreduces over NCCL: the per-row SSE vector every generation
plus the init-time overflow flags and non-finite count.  Every rank must then
take the same survival decisions as a single-process run over all cases and
as the reference itself (golden run).
"""

from __future__ import annotations

import ast
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as td
import torch.multiprocessing as mp

from conftest import golden


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import engine32, restate as R
        from paper_2106_04034_b200.dist import shard_range
        g = golden(name)
        cfg = R.Cfg(**ast.literal_eval(str(g["cfg"][0])))
        ntr, nte = g["Xtr"].shape[0], g["Xte"].shape[0]
        # align=1: these goldens are smaller than the engine's 12288-case
        # grid, and the protocol (not the grid) is what is checked here
        a, b = shard_range(ntr, world, rank, align=1)
        c, d = shard_range(nte, world, rank, align=1)

        def allreduce(_name, arr):
            t = torch.from_numpy(np.ascontiguousarray(arr))
            td.all_reduce(t, op=td.ReduceOp.SUM)
            return t.numpy()

        out = engine32.run32(cfg, g["Xtr"][a:b], g["ytr"][a:b], g["Xte"][c:d], g["yte"][c:d],
                             exchange=allreduce, n_total=(ntr, nte))
        out_q.put((rank, [e[:3] for e in out["elite"]], out["train"].tolist(),
                   out["test"].tolist(), out["overflow"]))
    finally:
        td.destroy_process_group()


@pytest.mark.parametrize("name,world", [("accept", 2), ("small", 2), ("c1", 3)])
def test_sharded_protocol_matches_single_process_and_reference(name, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = golden(name)
    ref_elite = [(("parent" if s == 0 else "offspring"), int(i), int(w))
                 for s, i, w in zip(g["src"], g["idx"], g["slot"])]
    for rank, elite, train, test, overflow in results:
        assert [tuple(e) for e in elite] == ref_elite, f"rank {rank}"
        np.testing.assert_allclose(train, g["train"], rtol=1e-5, atol=0)
        np.testing.assert_allclose(test, g["test"], rtol=1e-5, atol=0)
        assert overflow == int(g["overflow"][0])
    # all ranks hold bit-identical traces (same allreduced bits)
    assert all(r[2] == results[0][2] and r[3] == results[0][3] for r in results)


def _canon_worker(rank, world, port, out_q):
    """One rank of the canonical-SSE exchange (engine.cu canon_sse): local
    anchors -> allreduce MAX (int32) -> local digit limbs -> allreduce SUM
    (uint64 carried as int64, as dist.init_host_exchange does) -> finish."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import canon
        from paper_2106_04034_b200.dist import shard_range
        P = _canon_partials()
        lo, hi = shard_range(P.shape[1], world, rank, align=7)   # this rank's tiles
        mine = P[:, lo:hi]
        A = torch.tensor([canon.anchor(r) for r in mine], dtype=torch.int32)
        td.all_reduce(A, op=td.ReduceOp.MAX)
        L = np.array([canon.digits(r, int(a)) for r, a in zip(mine, A.tolist())], dtype=np.uint64)
        t = torch.from_numpy(L.view(np.int64).copy())
        td.all_reduce(t, op=td.ReduceOp.SUM)
        L = t.numpy().view(np.uint64)
        out_q.put((rank, [canon.finish([int(x) for x in l], int(a)) for l, a in zip(L, A.tolist())]))
    finally:
        td.destroy_process_group()


def _canon_partials():
    rng = np.random.default_rng(3)
    P = rng.lognormal(0.0, 5.0, (12, 61)) * 10.0 ** rng.integers(-20, 20, (12, 1))
    P[3] = 0.0
    P[4, 17] = np.inf
    P[5, :30] = 0.0
    P[6] = np.r_[2.0 ** 53, 1.0, 2.0 ** -60, np.zeros(58)]
    return P


@pytest.mark.parametrize("world", [2, 3])
def test_canonical_sse_exchange_is_rank_count_invariant(world):
    """The engine's two-collective SSE exchange gives every rank the
    single-process canonical sums bit for bit, whatever the split."""
    from oracle.canon import canonical_rows
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_canon_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = canonical_rows(_canon_partials())
    for rank, sums in got:
        np.testing.assert_array_equal(np.array(sums), want)
