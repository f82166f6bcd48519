"""Multi-run batching (paper_2106_04034_b200/runs.py).

CPU: the replica distribution over a 2- and 3-rank gloo group — run i on
rank i % world, results gathered to rank 0 in run order — with the oracle's
reference loop (oracle/restate.run) standing in for the device run, so the
host logic is checked without a GPU: every gathered run must equal the same
run executed alone, with the reference's per-run seeds
(gsgp/io_cli.py:288-289).
"""

from __future__ import annotations

import os
import socket
import types

import numpy as np
import pytest
import torch.distributed as td
import torch.multiprocessing as mp

from oracle import restate as R
from paper_2106_04034_b200.core import ConfigError, RunConfig
from paper_2106_04034_b200.runs import assign_runs, run_seeds

CFG = dict(population_size=12, random_trees=8, program_size=15, generations=4, runs=5, seed=9)


def _data():
    r = np.random.default_rng(3)
    Xtr, Xte = r.uniform(-1, 1, (40, 3)), r.uniform(-1, 1, (15, 3))
    return Xtr, Xtr[:, 0] * Xtr[:, 1] + Xtr[:, 2], Xte, Xte[:, 0] * Xte[:, 1] + Xte[:, 2]


def _oracle_run(cfg: RunConfig, train, test, **_):
    Xtr, ytr = train
    Xte, yte = test
    o = R.run(R.Cfg(**{k: getattr(cfg, k) for k in ("population_size", "random_trees", "program_size",
                                                     "generations", "seed")}), Xtr, ytr, Xte, yte)
    return types.SimpleNamespace(seed=cfg.seed, train_fitness=o["train"], test_fitness=o["test"],
                                 overflow_replacements=o["overflow"], timings=None,
                                 elite=[e[:3] for e in o["elite"]])


def test_assign_runs_round_robin_and_seeds():
    assert assign_runs(7, 3, 0) == [0, 3, 6] and assign_runs(7, 3, 2) == [2, 5]
    assert sorted(sum((assign_runs(10, 4, r) for r in range(4)), [])) == list(range(10))
    with pytest.raises(ConfigError):
        assign_runs(3, 2, 2)
    cfg = RunConfig(**CFG)
    assert run_seeds(cfg) == [R.run_seed(9, i) for i in range(5)]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, gather, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2106_04034_b200.runs import run_many
        Xtr, ytr, Xte, yte = _data()
        ran = []
        out = run_many(RunConfig(**CFG), (Xtr, ytr), (Xte, yte), gather=gather, run_fn=_oracle_run,
                       on_result=lambda i, res: ran.append(i))
        summary = [None if o is None else (list(map(float, o.train_fitness)), list(map(float, o.test_fitness)))
                   for o in out]
        q.put((rank, ran, summary))
    finally:
        td.destroy_process_group()


@pytest.mark.parametrize("world,gather", [(2, "results"), (3, "summary")])
def test_replicas_over_gloo_ranks_match_sequential_runs(world, gather):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, gather, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    Xtr, ytr, Xte, yte = _data()
    cfg = RunConfig(**CFG)
    seq = [_oracle_run(cfg.with_seed(s), (Xtr, ytr), (Xte, yte)) for s in run_seeds(cfg)]
    for rank, ran, summary in got:
        assert ran == assign_runs(cfg.runs, world, rank)
        if rank == 0:
            for i, s in enumerate(seq):
                assert summary[i] == (list(map(float, s.train_fitness)), list(map(float, s.test_fitness)))
        else:
            assert [i for i, v in enumerate(summary) if v is not None] == ran


def _failing_run(cfg: RunConfig, train, test, **kw):
    if cfg.seed == run_seeds(RunConfig(**CFG))[1]:      # run 1 (rank 1) fails
        from paper_2106_04034_b200.core import GsgpError
        raise GsgpError("injected failure")
    return _oracle_run(cfg, train, test, **kw)


def _fail_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world, timeout=__import__("datetime").timedelta(seconds=60))
    try:
        from paper_2106_04034_b200.core import GsgpError
        from paper_2106_04034_b200.runs import run_many
        Xtr, ytr, Xte, yte = _data()
        try:
            run_many(RunConfig(**CFG), (Xtr, ytr), (Xte, yte), gather="summary", run_fn=_failing_run)
            q.put((rank, "ok"))
        except GsgpError as exc:
            q.put((rank, str(exc)))
    finally:
        td.destroy_process_group()


def test_replica_failure_reaches_every_rank_without_hanging():
    """A run that raises on one rank is reported as GsgpError on that rank and
    on rank 0 (the CLI's clean 'error:' exit) instead of leaving the other
    ranks blocked in the gather until the process-group timeout."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fail_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert "injected failure" in got[0] and "rank 1" in got[0]
    assert "injected failure" in got[1]
