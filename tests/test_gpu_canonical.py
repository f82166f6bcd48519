"""The canonical SSE reduction on the B200 (csrc/common.cuh canon_*):

* the device primitive equals its specification (oracle/canon.py) bit for
  bit — fused single-shard path and multi-shard path (anchors, digits,
  finish) alike, for any split of the columns;
* consequently whole runs are bit-identical for any number of case shards:
  virtual shards in one process and real ranks sharing this GPU through the
  host exchange (the NCCL path exchanges the same anchors and digit sums).
  Shards start on the 12288-case grid (dist.CASE_ALIGN), so the datasets
  here are several grid blocks long.
This is the multi-GPU analogue of the reference's backend-invariance tests
(pkg/tests/test_acceptance.py:78, test_evolution.py:169, test_fitness.py:93):
results must not depend on how the work is split."""

from __future__ import annotations

import math
import os
import socket

import numpy as np
import pytest
import torch.distributed as td
import torch.multiprocessing as mp

import paper_2106_04034_b200 as G
from oracle.canon import canonical_rows

pytestmark = pytest.mark.gpu


def _battery():
    rng = np.random.default_rng(7)
    rows = [rng.lognormal(0, 3, 300) * 10.0 ** rng.integers(-40, 40) for _ in range(40)]
    rows += [rng.lognormal(0, 40, 300) for _ in range(10)]            # > 116 binades: truncation
    rows += [np.zeros(300), np.full(300, 5e-324), np.r_[np.full(299, 2.0 ** -1070), 2.0 ** -1022]]
    rows += [np.r_[2.0 ** 53, 1.0, np.zeros(298)], np.r_[2.0 ** 53, 3.0, np.zeros(298)],
             np.r_[2.0 ** 53, 1.0, 2.0 ** -60, np.zeros(297)], np.r_[np.full(2, 1.7e308), np.zeros(298)]]
    inf_row = rng.random(300)
    inf_row[17] = math.inf
    nan_row = rng.random(300)
    nan_row[5], nan_row[6] = math.nan, math.inf
    rows += [inf_row, nan_row]
    return np.array(rows)


@pytest.mark.parametrize("parts", [0, 1, 2, 3, 7, 300])
def test_device_canonical_sum_matches_specification(parts):
    M = _battery()
    got = G.canonical_sum(M, parts=parts)
    want = canonical_rows(M)
    np.testing.assert_array_equal(got, want)          # NaN rows compare equal


def test_device_canonical_sum_is_order_free_at_scale():
    rng = np.random.default_rng(11)
    M = rng.lognormal(0, 6, (64, 20_000))
    ref = G.canonical_sum(M)
    perm = M[:, rng.permutation(M.shape[1])]
    assert np.array_equal(G.canonical_sum(perm), ref)
    assert np.array_equal(G.canonical_sum(perm, parts=13), ref)
    assert np.array_equal(ref, canonical_rows(M))


def _large_case(seed=5, ntr=61_000, nte=29_000, l=6, wide=False):
    rng = np.random.default_rng(seed)
    Xtr = rng.uniform(-2, 2, (ntr, l))
    Xte = rng.uniform(-2, 2, (nte, l))
    if wide:                      # some programs overflow fp32 storage (fp64 SSE slots)
        Xtr[:, 0] *= 1e25
        Xte[:, 0] *= 1e25
    f = lambda X: X[:, 0] * X[:, 1] + np.sin(X[:, 2]) + X[:, 3] ** 2
    cfg = G.RunConfig(population_size=96, random_trees=48, program_size=63, generations=20, seed=seed)
    return cfg, G.Dataset(Xtr, f(Xtr)), G.Dataset(Xte, f(Xte))


def _fingerprint(res):
    plans = b"".join(e.plan.u.tobytes() + e.plan.v.tobytes() + e.plan.ms.tobytes()
                     for e in res.lineage.entries if e.plan is not None)
    return ([(e.elite.source, e.elite.index, e.elite.slot) for e in res.lineage.entries], plans,
            res.train_fitness.tobytes(), res.test_fitness.tobytes(), res.overflow_replacements,
            res.elite_train_semantics.tobytes())


@pytest.mark.parametrize("storage,wide", [("fp32", False), ("fp64", False), ("fp32", True)])
def test_runs_bit_identical_for_any_virtual_shard_count(storage, wide):
    cfg, tr, te = _large_case(wide=wide)
    base = _fingerprint(G.run_evolution(cfg, tr, te, storage=storage))
    for vs in (2, 3, 5, 8):
        assert _fingerprint(G.run_evolution(cfg, tr, te, storage=storage, virtual_shards=vs)) == base, vs


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_worker(rank, world, port, vshards, wide, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2106_04034_b200 as G2
        from paper_2106_04034_b200 import dist
        dist.init_host_exchange()
        cfg, tr, te = _large_case(wide=wide)
        res = G2.run_evolution(cfg, tr, te, virtual_shards=vshards)
        full = dist.gather_elite_semantics(res, tr.n_cases)
        fp = list(_fingerprint(res))
        fp[5] = full.tobytes()
        q.put((rank, fp, res.device["shard_train_range"]))
        dist.destroy()
    finally:
        td.destroy_process_group()


@pytest.mark.parametrize("world,vshards,wide", [(2, 1, False), (3, 1, False), (4, 2, False), (3, 1, True)])
def test_ranks_bit_identical_to_single_process(world, vshards, wide):
    cfg, tr, te = _large_case(wide=wide)
    base = list(_fingerprint(G.run_evolution(cfg, tr, te)))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_worker, args=(r, world, port, vshards, wide, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=900) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    spans = [g[2] for g in got]
    assert sum(1 for lo, hi in spans if hi > lo) >= 2        # the cases really are split
    for rank, fp, _ in got:
        assert fp == base, rank


@pytest.mark.parametrize("ntr,nte,storage", [
    (4096, 4096, "fp32"),            # no tails
    (4096 * 3 + 1, 4095, "fp32"),    # tails 1 + 4095 (do not fit one tile together)
    (12288 * 2 + 4064, 32, "fp32"),  # tails 4064 + 32 fill one tile exactly
    (24576 + 7, 12288 + 9, "fp32"),  # tails on both shard-grid boundaries
    (2048 * 5 + 100, 2048 + 1900, "fp64"),   # fp64 tiles (2048 cases)
    (12288 * 3, 12288, "fp64"),
])
def test_tile_and_shard_boundaries(ntr, nte, storage):
    """Row layouts around the tile and shard-grid boundaries (tails absent,
    merged, too large to merge): every virtual-shard count reproduces the
    one-shard run bit for bit, and the elite trace matches the engine
    restatement (oracle/engine32.py) run on the host."""
    from oracle import engine32, restate as R
    rng = np.random.default_rng(ntr + nte)
    Xtr, Xte = rng.uniform(-1, 1, (ntr, 3)), rng.uniform(-1, 1, (nte, 3))
    f = lambda X: X[:, 0] * X[:, 1] - X[:, 2]
    kw = dict(population_size=12, random_trees=6, program_size=31, generations=6, seed=ntr % 97 + 1)
    cfg = G.RunConfig(**kw)
    tr, te = G.Dataset(Xtr, f(Xtr)), G.Dataset(Xte, f(Xte))
    base = _fingerprint(G.run_evolution(cfg, tr, te, storage=storage))
    for vs in (2, 3, 4):
        assert _fingerprint(G.run_evolution(cfg, tr, te, storage=storage, virtual_shards=vs)) == base, vs
    if storage == "fp32":
        o = engine32.run32(R.Cfg(**kw), Xtr, f(Xtr), Xte, f(Xte))
        assert base[0] == [e[:3] for e in o["elite"]]
