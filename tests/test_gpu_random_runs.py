"""Randomised whole-run parity: random configurations (population, pool and
genome sizes, gene probabilities, ERC range, constant/uniform step, both GSM
signs, eps, case counts, feature widths; a forced small upload chunk and
virtual case shards) through the device `run_evolution`, against

* oracle/engine32.run32 — the op-for-op restatement of the engine's fp32
  storage arithmetic: plans and elite records identical, elite semantics
  bit-identical, traces to 1e-12 (the only difference is the SSE summation
  order, numpy's vs the kernel's fixed tile order);
* oracle/restate.run — the reference loop in fp64, for storage="fp64":
  identical plans and elite records, traces to 1e-12.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import engine32, restate as R

pytestmark = pytest.mark.gpu

import paper_2106_04034_b200 as G  # noqa: E402


def _random_case(seed: int):
    rng = np.random.default_rng(seed)
    p = rng.dirichlet([2.0, 1.0, 1.0]) if rng.random() < 0.8 else np.array([0.5, 0.5, 0.0])
    kw = dict(population_size=int(rng.integers(1, 49)), random_trees=int(rng.integers(2, 49)),
              program_size=int(rng.choice([1, 2, 5, 17, 64, 127, 200, 511, 1024])),
              generations=int(rng.integers(0, 11)), seed=int(rng.integers(-2**40, 2**40)),
              p_function=float(p[0]), p_feature=float(p[1]), p_constant=float(p[2]),
              erc_low=float(rng.uniform(-5, 1)), erc_high=float(rng.uniform(1, 10)),
              mutation_step="uniform" if rng.random() < 0.7 else float(rng.uniform(0.01, 2.0)),
              division_eps=float(10.0 ** rng.uniform(-9, -2)),
              gsm_sign="minus" if rng.random() < 0.6 else "plus")
    l = int(rng.integers(1, 7))
    big = rng.random() < 0.25          # several GSM case tiles (4096 fp32 per tile)
    ntr = int(rng.integers(1, 7000 if big else 400))
    nte = int(rng.integers(1, 2500 if big else 150))
    scale = 10.0 ** rng.uniform(-2, 2)
    Xtr, Xte = rng.uniform(-scale, scale, (ntr, l)), rng.uniform(-scale, scale, (nte, l))
    f = lambda X: X[:, 0] * X[:, -1] - X.sum(axis=1) + 0.5  # noqa: E731
    return kw, Xtr, f(Xtr), Xte, f(Xte)


def _elite(res):
    return [(e.elite.source, e.elite.index, e.elite.slot) for e in res.lineage.entries]


@pytest.mark.parametrize("seed", range(48))
def test_random_run_matches_engine_restatement(seed, monkeypatch):
    kw, Xtr, ytr, Xte, yte = _random_case(seed)
    if seed % 4 == 1:
        monkeypatch.setenv("GSGP_UPLOAD_CHUNK", "3072")
    # every interpreter launch configuration takes part (0 128x4, 2 HBM
    # features, 3 128x2, 4 lean, 5 128x3, 6/7 128x3/128x4 with two genome
    # groups per block, 9 one-warp genome groups on a 128-case tile, 10
    # 128x4 with four genome groups per block)
    monkeypatch.setenv("GSGP_INTERP_CFG", ["0", "5", "2", "3", "4", "6", "7", "9", "10", "5"][seed % 10])
    res = G.run_evolution(G.RunConfig(**kw), G.Dataset(Xtr, ytr), G.Dataset(Xte, yte),
                          virtual_shards=1 + seed % 3)
    o = engine32.run32(R.Cfg(**kw), Xtr, ytr, Xte, yte)
    assert _elite(res) == [e[:3] for e in o["elite"]], kw
    for t, e in enumerate(res.lineage.entries):
        assert np.array_equal(e.plan.u, o["u"][t]) and np.array_equal(e.plan.v, o["v"][t])
        assert np.array_equal(e.plan.ms, o["ms"][t])
    np.testing.assert_allclose(res.train_fitness, o["train"], rtol=1e-12, atol=0)
    np.testing.assert_allclose(res.test_fitness, o["test"], rtol=1e-12, atol=0)
    assert np.array_equal(res.elite_train_semantics, o["elite_train_semantics"])
    assert res.overflow_replacements == o["overflow"]


@pytest.mark.parametrize("seed", range(100, 116))
def test_random_run_fp64_storage_matches_reference_loop(seed):
    kw, Xtr, ytr, Xte, yte = _random_case(seed)
    res = G.run_evolution(G.RunConfig(**kw), G.Dataset(Xtr, ytr), G.Dataset(Xte, yte), storage="fp64")
    o = R.run(R.Cfg(**kw), Xtr, ytr, Xte, yte)
    assert _elite(res) == [e[:3] for e in o["elite"]], kw
    np.testing.assert_allclose(res.train_fitness, o["train"], rtol=1e-12, atol=0)
    np.testing.assert_allclose(res.test_fitness, o["test"], rtol=1e-12, atol=0)
    np.testing.assert_allclose(res.elite_train_semantics, o["elite_train_semantics"], rtol=1e-12, atol=1e-300)


def test_wide_feature_run_matches_engine_restatement(monkeypatch):
    """150 features (features stay in HBM, 3072-case upload chunks) through a
    whole run: plans, elite records and elite semantics exact."""
    rng = np.random.default_rng(77)
    l, ntr, nte = 150, 6000, 1500
    Xtr, Xte = rng.uniform(-1, 1, (ntr, l)), rng.uniform(-1, 1, (nte, l))
    ytr, yte = Xtr[:, 0] * Xtr[:, 7] + Xtr[:, 149], Xte[:, 0] * Xte[:, 7] + Xte[:, 149]
    kw = dict(population_size=40, random_trees=24, program_size=255, generations=6, seed=5)
    monkeypatch.setenv("GSGP_UPLOAD_CHUNK", "3072")
    res = G.run_evolution(G.RunConfig(**kw), G.Dataset(Xtr, ytr), G.Dataset(Xte, yte))
    o = engine32.run32(R.Cfg(**kw), Xtr, ytr, Xte, yte)
    assert _elite(res) == [e[:3] for e in o["elite"]]
    np.testing.assert_allclose(res.train_fitness, o["train"], rtol=1e-12, atol=0)
    assert np.array_equal(res.elite_train_semantics, o["elite_train_semantics"])
