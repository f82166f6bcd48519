"""Operator properties of the reference test suite on the device
(pkg/tests/test_mutation.py, test_population.py, test_fitness.py, same
inputs and assertions); the bit-level parity of the same operators is in
test_gpu_ops.py."""

from __future__ import annotations

import math

import numpy as np
import pytest

import paper_2106_04034_b200 as G
from paper_2106_04034_b200 import ConfigError, GeneTag, MutationPlan, RunConfig, WORST_FITNESS

pytestmark = pytest.mark.gpu


def cfg_with(**kw) -> RunConfig:
    base = dict(population_size=4, random_trees=4, program_size=16, generations=1, seed=3)
    base.update(kw)
    return RunConfig(**base)


# ------------------------------------------------------------------ sigmoid
def test_sigmoid_properties():
    assert G.sigmoid(0.0) == 0.5
    assert abs(G.sigmoid(40.0) - 1.0) < 1e-15
    assert G.sigmoid(-800.0) == 0.0 and G.sigmoid(800.0) == 1.0
    xs = np.linspace(-50, 50, 401)
    s, sm = G.sigmoid_array(xs), G.sigmoid_array(-xs)
    assert np.allclose(s + sm, 1.0, atol=1e-12) and (s >= 0).all() and (s <= 1).all()
    assert ((s > 0) & (s < 1))[np.abs(xs) < 36].all()
    assert (np.diff(G.sigmoid_array(np.linspace(-30, 30, 301))) > 0).all()
    big = np.linspace(-700, 700, 999)
    for x, v in zip(big[::37], G.sigmoid_array(big)[::37]):
        assert v == pytest.approx(G.sigmoid(float(x)), abs=1e-15)


# --------------------------------------------------------------------- plan
def test_plan_properties():
    p = G.build_mutation_plan(200, 2, cfg_with(), generation=1)
    assert set(zip(p.u.tolist(), p.v.tolist())) == {(0, 1), (1, 0)}
    a, b = G.build_mutation_plan(32, 8, cfg_with(), 3), G.build_mutation_plan(32, 8, cfg_with(), 3)
    c = G.build_mutation_plan(32, 8, cfg_with(), 4)
    assert np.array_equal(a.u, b.u) and np.array_equal(a.ms, b.ms)
    assert not (np.array_equal(a.u, c.u) and np.array_equal(a.ms, c.ms))
    for gen in range(1, 30):
        p = G.build_mutation_plan(64, 5, cfg_with(), gen)
        assert (p.u != p.v).all() and p.u.min() >= 0 and p.u.max() < 5 and p.v.max() < 5
        assert (p.ms > 0).all() and (p.ms <= 1.0).all()
    p = G.build_mutation_plan(2000, 4, cfg_with(), 1)
    assert set(zip(p.u.tolist(), p.v.tolist())) == {(u, v) for u in range(4) for v in range(4) if u != v}
    assert abs(G.build_mutation_plan(100_000, 8, cfg_with(), 1).ms.mean() - 0.5) < 0.005
    assert np.array_equal(G.build_mutation_plan(16, 8, cfg_with(mutation_step=0.3), 2).ms, np.full(16, 0.3))
    with pytest.raises(ConfigError):
        G.build_mutation_plan(8, 1, cfg_with(), 1)


# ---------------------------------------------------------------------- gsm
def _state(seed, m=6, r=5, n=9, scale=10.0):
    rng = np.random.default_rng(seed)
    parents, trees = rng.normal(size=(m, n)) * scale, rng.normal(size=(r, n)) * scale
    u = rng.integers(0, r, size=m)
    v = (u + 1 + rng.integers(0, r - 1, size=m)) % r
    return parents, trees, MutationPlan(u, v, rng.uniform(0.01, 1.0, size=m))


def test_gsm_properties():
    cfg = cfg_with()
    parents, trees, plan = _state(1)
    assert np.array_equal(G.gsm(parents, trees, MutationPlan(plan.u, plan.v, np.zeros(6)), cfg), parents)
    same = np.repeat(trees[:1], 5, axis=0)
    assert np.array_equal(G.gsm(parents, same, plan, cfg_with(gsm_sign="minus")), parents)
    one = G.gsm(np.array([[1.0]]), np.array([[math.log(0.8 / 0.2)], [math.log(0.3 / 0.7)]]),
                MutationPlan(np.array([0]), np.array([1]), np.array([0.1])), cfg)
    assert one[0, 0] == pytest.approx(1.05, abs=1e-12)
    parents, trees, plan = _state(4)
    assert G.gsm(parents + 1.0, trees, plan, cfg) == pytest.approx(G.gsm(parents, trees, plan, cfg) + 1.0,
                                                                   abs=1e-12)
    parents, trees, plan = _state(5, scale=3.0)
    assert (np.abs(G.gsm(parents, trees, plan, cfg_with(gsm_sign="minus")) - parents)
            <= plan.ms[:, None]).all()
    d = G.gsm(parents, trees, plan, cfg_with(gsm_sign="plus")) - parents
    assert (d > 0).all() and (d <= 2.0 * plan.ms[:, None]).all()
    with pytest.raises(ConfigError):
        G.gsm(parents[:, :-1], trees, plan, cfg)
    with pytest.raises(ConfigError):
        G.gsm(parents, trees, MutationPlan(plan.u + 100, plan.v, plan.ms), cfg)


def test_gsm_paired_properties():
    cfg = cfg_with()
    parents, trees, plan = _state(8)
    tr, te = G.gsm_paired(parents, parents, trees, trees, plan, cfg)
    assert np.array_equal(tr, te) and np.array_equal(tr, G.gsm(parents, trees, plan, cfg))
    parents, trees, plan = _state(9)
    other = parents[:, :4].copy()
    zero = MutationPlan(plan.u, plan.v, np.zeros(len(plan)))
    a, b = G.gsm_paired(parents, other, trees, trees[:, :4].copy(), zero, cfg)
    assert np.array_equal(a, parents) and np.array_equal(b, other)
    with pytest.raises(ConfigError):
        G.gsm_paired(parents, parents[:-1], trees, trees, plan, cfg)


# --------------------------------------------------------------- population
def test_population_properties():
    pop = G.create_population(3, cfg_with(p_function=1.0, p_feature=0.0, p_constant=0.0), 0, 2)
    assert (pop.tags == GeneTag.FUNCTION).all() and pop.codes.min() >= 0 and pop.codes.max() <= 3
    pop = G.create_population(2, cfg_with(p_function=0.0, p_feature=0.0, p_constant=1.0, program_size=500), 0, 2)
    assert (pop.tags == GeneTag.CONSTANT).all() and pop.consts.min() >= 1.0 and pop.consts.max() <= 10.0
    pop = G.create_population(100, cfg_with(program_size=1000), 0, 5)
    assert abs((pop.tags == GeneTag.FUNCTION).mean() - 0.8 / 0.98) < 0.01
    assert abs((pop.tags == GeneTag.FEATURE).mean() - 0.14 / 0.98) < 0.01
    pop = G.create_population(1, cfg_with(program_size=1), 0, 1)
    assert len(pop) == 1 and pop.genome_length == 1
    big = G.create_population(10240, cfg_with(program_size=127), 0, 1024)
    f = big.codes[big.tags == GeneTag.FEATURE]
    assert big.tags.shape == (10240, 127) and f.min() >= 0 and f.max() < 1024
    small, large = G.create_population(5, cfg_with(), 0, 3), G.create_population(10, cfg_with(), 0, 3)
    shifted = G.create_population(5, cfg_with(), 5, 3)
    assert np.array_equal(small.tags, large.tags[:5]) and np.array_equal(shifted.codes, large.codes[5:])
    pop = G.create_population(8, cfg_with(program_size=40), 0, 3)
    for i in range(8):
        for gene in pop.chromosome(i).genes():
            gene.validate(n_features=3)
    with pytest.raises(ConfigError):
        G.create_population(0, cfg_with(), 0, 2)


# ------------------------------------------------------------------ fitness
def test_fitness_properties():
    row = np.array([1.0, -2.0, 3.5])
    assert G.rmse(row, row) == 0.0
    assert G.rmse([0.0, 0.0], [3.0, 4.0]) == pytest.approx(3.5355339059327378, abs=1e-12)
    assert G.rmse([1.0], [4.0]) == 3.0
    rng = np.random.default_rng(5)
    a, b = rng.normal(size=30), rng.normal(size=30)
    assert G.rmse(a, b) == G.rmse(b, a) >= 0.0
    assert G.rmse(2 * a, 2 * b) == pytest.approx(2 * G.rmse(a, b), abs=1e-12)
    assert G.rmse([1e200, 0.0], [-1e200, 0.0]) == WORST_FITNESS
    assert G.rmse([np.nan], [0.0]) == WORST_FITNESS
    with pytest.raises(ConfigError):
        G.rmse([1.0, 2.0], [1.0])
    with pytest.raises(ConfigError):
        G.compute_fitness(np.zeros((2, 3)), np.zeros(4))
    rng = np.random.default_rng(2)
    sem, tgt = rng.normal(size=(12, 37)), rng.normal(size=37)
    vec = G.compute_fitness(sem, tgt)
    assert all(vec[i] == G.rmse(sem[i], tgt) for i in range(12))
    sem[4] = tgt
    vec = G.compute_fitness(sem, tgt)
    assert vec[4] == 0.0 and (np.delete(vec, 4) > 0.0).all()
    assert np.array_equal(G.compute_fitness(np.zeros((5, 8)), np.ones(8)), np.ones(5))
    s = np.zeros((3, 4))
    s[1] = 1e200
    v = G.compute_fitness(s, np.zeros(4))
    assert v[0] == 0.0 and v[2] == 0.0 and v[1] == WORST_FITNESS
