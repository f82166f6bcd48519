"""The engine's multi-rank path (case sharding + per-generation exchange,
SURVEY §8e) with 2 and 3 real processes sharing this GPU: the collectives
go through `dist.init_host_exchange` (host memory + gloo) instead of NCCL —
same partition, same exchanged values, same decision logic in the library.
Every rank must return the single-process run's elite trace and traces
bit for bit (the canonical SSE does not depend on the split) and the
reference's golden elite trace; the gathered elite semantics must equal the
single-process elite semantics.  The goldens are smaller than one 12288-case
shard block, so here the leading ranks hold empty slices; real splits of
large datasets are in test_gpu_canonical.py."""

from __future__ import annotations

import ast
import os
import socket

import numpy as np
import pytest
import torch.distributed as td
import torch.multiprocessing as mp

from conftest import golden

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, vshards, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2106_04034_b200 as G
        from paper_2106_04034_b200 import dist
        dist.init_host_exchange()
        g = golden(name)
        cfg = G.RunConfig(**ast.literal_eval(str(g["cfg"][0])))
        res = G.run_evolution(cfg, G.Dataset(g["Xtr"], g["ytr"]), G.Dataset(g["Xte"], g["yte"]),
                              virtual_shards=vshards)
        full = dist.gather_elite_semantics(res, g["Xtr"].shape[0])
        elite = [(e.elite.source, e.elite.index, e.elite.slot) for e in res.lineage.entries]
        q.put((rank, elite, res.train_fitness.tolist(), res.test_fitness.tolist(),
               res.overflow_replacements, full.tolist()))
        dist.destroy()
    finally:
        td.destroy_process_group()


@pytest.mark.parametrize("name,world,vshards", [("accept", 2, 1), ("c1", 3, 1), ("c2s", 2, 2), ("wide", 2, 1),
                                                 ("n1", 2, 1)])
def test_ranks_sharing_a_gpu_reproduce_single_process_run(name, world, vshards):
    import paper_2106_04034_b200 as G
    g = golden(name)
    cfg = G.RunConfig(**ast.literal_eval(str(g["cfg"][0])))
    one = G.run_evolution(cfg, G.Dataset(g["Xtr"], g["ytr"]), G.Dataset(g["Xte"], g["yte"]))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, vshards, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref_elite = [(("parent" if s == 0 else "offspring"), int(i), int(w))
                 for s, i, w in zip(g["src"], g["idx"], g["slot"])]
    one_elite = [(e.elite.source, e.elite.index, e.elite.slot) for e in one.lineage.entries]
    assert one_elite == ref_elite
    for rank, elite, train, test, overflow, full in got:
        assert elite == one_elite, rank
        assert train == one.train_fitness.tolist() and test == one.test_fitness.tolist()
        assert overflow == one.overflow_replacements
        assert np.array_equal(np.array(full), one.elite_train_semantics)
    assert all(r[2] == got[0][2] and r[3] == got[0][3] for r in got)   # identical on every rank


def _replica_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["GSGP_SHARED_GPU"] = "1"
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import dataclasses

        import paper_2106_04034_b200 as G
        from paper_2106_04034_b200.runs import select_local_device
        select_local_device()
        g = golden("c1")
        cfg = dataclasses.replace(G.RunConfig(**ast.literal_eval(str(g["cfg"][0]))), runs=5,
                                  generations=12)
        ran = []
        out = G.run_many(cfg, G.Dataset(g["Xtr"], g["ytr"]), G.Dataset(g["Xte"], g["yte"]),
                         on_result=lambda i, r: ran.append(i))
        q.put((rank, ran, [None if o is None else o.train_fitness.tolist() for o in out]))
    finally:
        td.destroy_process_group()


def test_replica_runs_across_ranks_match_sequential_runs():
    """run_many with 2 real ranks on this GPU: run i on
    rank i % 2, full results gathered to rank 0 in run order, equal to the
    runs executed one by one in this process."""
    import dataclasses

    import paper_2106_04034_b200 as G
    g = golden("c1")
    cfg = dataclasses.replace(G.RunConfig(**ast.literal_eval(str(g["cfg"][0]))), runs=5, generations=12)
    tr, te = G.Dataset(g["Xtr"], g["ytr"]), G.Dataset(g["Xte"], g["yte"])
    seq = [G.run_evolution(cfg.with_seed(s), tr, te).train_fitness.tolist() for s in G.run_seeds(cfg)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_replica_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got[0][1] == [0, 2, 4] and got[1][1] == [1, 3]
    assert got[0][2] == seq


def _case(seed, tiny):
    from test_gpu_random_runs import _random_case
    kw, Xtr, ytr, Xte, yte = _random_case(seed)
    if tiny:                      # fewer cases than ranks: some slices are empty
        a, b = 1 + seed % 2, 1 + seed % 3
        Xtr, ytr, Xte, yte = Xtr[:a], ytr[:a], Xte[:b], yte[:b]
    return kw, Xtr, ytr, Xte, yte


def _random_worker(rank, world, port, seed, vshards, tiny, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2106_04034_b200 as G
        from paper_2106_04034_b200 import dist
        dist.init_host_exchange()
        kw, Xtr, ytr, Xte, yte = _case(seed, tiny)
        res = G.run_evolution(G.RunConfig(**kw), G.Dataset(Xtr, ytr), G.Dataset(Xte, yte),
                              virtual_shards=vshards)
        full = dist.gather_elite_semantics(res, Xtr.shape[0])
        q.put((rank, [(e.elite.source, e.elite.index, e.elite.slot) for e in res.lineage.entries],
               res.train_fitness.tolist(), full.tolist()))
        dist.destroy()
    finally:
        td.destroy_process_group()


@pytest.mark.parametrize("seed,world,vshards,tiny",
                         [(s, 2 + s % 3, 1 + s % 2, s >= 204) for s in range(200, 210)])
def test_random_configs_across_ranks(seed, world, vshards, tiny):
    """Random configurations (tiny case counts included, so some ranks hold
    no cases) over 2-4 ranks x 1-2 virtual shards == the single-process run."""
    import paper_2106_04034_b200 as G
    kw, Xtr, ytr, Xte, yte = _case(seed, tiny)
    one = G.run_evolution(G.RunConfig(**kw), G.Dataset(Xtr, ytr), G.Dataset(Xte, yte))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_random_worker, args=(r, world, port, seed, vshards, tiny, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    one_elite = [(e.elite.source, e.elite.index, e.elite.slot) for e in one.lineage.entries]
    for rank, elite, train, full in got:
        assert elite == one_elite, (rank, kw)
        assert train == one.train_fitness.tolist(), (rank, kw)
        assert np.array_equal(np.array(full), one.elite_train_semantics)
