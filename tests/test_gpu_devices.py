"""Single-process multi-GPU (`gsgp_init`, devices.py) and the NCCL transport.

One `run_evolution(cfg, train, test, devices=...)` call drives several GPUs
from one process: one host thread and one rank per device, cases sharded by
device, the canonical-SSE collectives over NCCL (gsgp/evolution.py:115 with
gsgp/backend.py:94-130: the reference's run uses every worker of the host).

On a one-GPU box:
* a device list that repeats GPU 0 runs the same threads with the host
  thread exchange: the result must equal the one-device run bit for bit;
* GSGP_FORCE_COLLECTIVES=1 makes a one-rank job create its NCCL communicator
  (ncclCommInitAll in-process, ncclCommInitRank across processes) and run
  every collective through it, graph-captured — so the NCCL transport itself
  executes here, and must give the same bits;
* a failing device thread aborts its peers (no hang) and the error surfaces.
With two or more GPUs the real multi-device and multi-process NCCL paths run.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as td
import torch.multiprocessing as mp

import paper_2106_04034_b200 as G
from paper_2106_04034_b200 import devices as D

pytestmark = pytest.mark.gpu

N_GPUS = torch.cuda.device_count()


def _case(seed=5, ntr=61_000, nte=29_000, l=6, m=96, g=20):
    """> 12288 cases per shard for up to 4 shards (dist.CASE_ALIGN grid)."""
    rng = np.random.default_rng(seed)
    Xtr, Xte = rng.uniform(-2, 2, (ntr, l)), rng.uniform(-2, 2, (nte, l))
    f = lambda X: X[:, 0] * X[:, 1] + np.sin(X[:, 2]) + X[:, 3] ** 2  # noqa: E731
    cfg = G.RunConfig(population_size=m, random_trees=48, program_size=63, generations=g, seed=seed)
    return cfg, G.Dataset(Xtr, f(Xtr)), G.Dataset(Xte, f(Xte))


def _fingerprint(res):
    plans = b"".join(e.plan.u.tobytes() + e.plan.v.tobytes() + e.plan.ms.tobytes()
                     for e in res.lineage.entries)
    return ([(e.elite.source, e.elite.index, e.elite.slot) for e in res.lineage.entries], plans,
            res.train_fitness.tobytes(), res.test_fitness.tobytes(), res.elite_train_semantics.tobytes(),
            res.overflow_replacements)


@pytest.fixture(autouse=True)
def _single_device_after():
    yield
    D.activate(None)


@pytest.fixture(scope="module")
def reference_run():
    cfg, tr, te = _case()
    return _fingerprint(G.run_evolution(cfg, tr, te, devices=None))


@pytest.mark.parametrize("ids", [(0, 0), (0, 0, 0), (0, 0, 0, 0)])
def test_device_threads_on_one_gpu_equal_single_device(ids, reference_run):
    cfg, tr, te = _case()
    res = G.run_evolution(cfg, tr, te, devices=list(ids))
    assert res.device["devices"] == list(ids)
    assert _fingerprint(res) == reference_run
    assert res.device["shard_train_range"] == (0, tr.n_cases)


def test_device_threads_with_virtual_shards_and_fp64(reference_run):
    cfg, tr, te = _case()
    assert _fingerprint(G.run_evolution(cfg, tr, te, devices=[0, 0], virtual_shards=2)) == reference_run
    a = G.run_evolution(cfg, tr, te, devices=None, storage="fp64")
    b = G.run_evolution(cfg, tr, te, devices=[0, 0, 0], storage="fp64")
    assert _fingerprint(a) == _fingerprint(b)


def test_device_threads_with_empty_ranks():
    """Fewer cases than ranks x 12288: some device threads hold no cases and
    only draw the plan for their lineage record."""
    cfg, tr, te = _case(seed=9, ntr=900, nte=300, g=12)
    a = G.run_evolution(cfg, tr, te, devices=None)
    b = G.run_evolution(cfg, tr, te, devices=[0, 0, 0])
    assert _fingerprint(a) == _fingerprint(b)


def test_forced_nccl_one_rank_in_process(monkeypatch, reference_run):
    """ncclCommInitAll with one device + graph-captured ncclAllReduce of the
    anchors and digits every generation == the collective-free run."""
    monkeypatch.setenv("GSGP_FORCE_COLLECTIVES", "1")
    cfg, tr, te = _case()
    D.activate(None)
    res = G.run_evolution(cfg, tr, te, devices=[0])
    assert _fingerprint(res) == reference_run
    # direct launches (no graph) through NCCL too
    assert _fingerprint(G.run_evolution(cfg, tr, te, devices=[0], use_graph=False)) == reference_run
    assert res.device["loop_launches"] > 2 * cfg.generations     # exp, digits, finish, survive


def test_failing_device_thread_aborts_its_peers(monkeypatch):
    cfg, tr, te = _case(g=3)
    monkeypatch.setenv("GSGP_TEST_FAIL_RANK", "1")
    with pytest.raises(G.GsgpError, match="injected failure"):
        G.run_evolution(cfg, tr, te, devices=[0, 0, 0])
    monkeypatch.delenv("GSGP_TEST_FAIL_RANK")
    # the next run works (device set re-initialised)
    res = G.run_evolution(cfg, tr, te, devices=[0, 0])
    assert res.device["devices"] == [0, 0]


def test_device_argument_validation():
    cfg, tr, te = _case(g=1, ntr=100, nte=20)
    with pytest.raises(G.ConfigError):
        G.run_evolution(cfg, tr, te, devices=0)
    with pytest.raises(G.ConfigError):
        G.run_evolution(cfg, tr, te, devices="most")
    with pytest.raises(G.ConfigError):
        G.run_evolution(cfg, tr, te, devices=[N_GPUS + 3])
    assert D.resolve("auto", 1024, 125_000) is None          # C2 stays on one GPU
    want = min(N_GPUS, 8)
    assert D.resolve("auto", 1024, 12_500_000) == (tuple(range(want)) if want > 1 else None)   # C3


@pytest.mark.skipif(N_GPUS < 2, reason="needs two GPUs")
@pytest.mark.parametrize("n", [2, min(N_GPUS, 8)])
def test_real_multi_gpu_in_process_equals_single_device(n, reference_run):
    cfg, tr, te = _case()
    res = G.run_evolution(cfg, tr, te, devices=n)
    assert res.device["devices"] == list(range(n))
    assert _fingerprint(res) == reference_run


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _nccl_worker(rank, world, port, shared, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if world == 1:
        os.environ["GSGP_FORCE_COLLECTIVES"] = "1"
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2106_04034_b200 import _lib, dist
        _lib.check(_lib.load().gsgp_set_device(0 if shared else rank))
        dist.init_from_torch()
        cfg, tr, te = _case()
        res = G.run_evolution(cfg, tr, te)
        full = dist.gather_elite_semantics(res, tr.n_cases)
        fp = list(_fingerprint(res))
        fp[4] = full.tobytes()
        q.put((rank, fp))
        dist.destroy()
    finally:
        td.destroy_process_group()


def _run_nccl_ranks(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nccl_worker, args=(r, world, port, False, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return got


def test_forced_nccl_one_rank_across_processes(reference_run):
    """dist.init_from_torch (ncclGetUniqueId broadcast, ncclCommInitRank) with
    one rank and forced collectives == the plain run."""
    got = _run_nccl_ranks(1)
    assert tuple(got[0]) == reference_run


@pytest.mark.skipif(N_GPUS < 2, reason="needs two GPUs")
def test_real_nccl_ranks_equal_single_process(reference_run):
    got = _run_nccl_ranks(2)
    for r in range(2):
        assert tuple(got[r]) == reference_run
