"""Reference behaviours of the run API, replay and CLI on the device, after
pkg/tests/test_evolution.py:106-260 and pkg/tests/test_io_cli.py:259-345
(same inputs and assertions; `backend` is "cuda")."""

from __future__ import annotations

import dataclasses
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, toy_dataset

import paper_2106_04034_b200 as G
from paper_2106_04034_b200 import ConfigError, LineageError, RunConfig

pytestmark = pytest.mark.gpu


def _ds(n, l, seed):
    X, y = toy_dataset(n, l, seed)
    return G.Dataset(X, y)


def _initial(cfg, train):
    pop = G.create_population(cfg.population_size, cfg, 0, train.n_features)
    trees = G.create_population(cfg.random_trees, cfg, cfg.population_size, train.n_features)
    return G.compute_semantics(pop, train, cfg), G.compute_semantics(trees, train, cfg)


def test_replay_reproduces_live_elite_bitwise_at_scale():
    # pkg/tests/test_evolution.py:207-217 (fp64 storage: the reference's GSM arithmetic)
    cfg = RunConfig(population_size=64, random_trees=32, program_size=63, generations=100, seed=1234)
    train, test = _ds(100, 4, 40), _ds(30, 4, 41)
    res = G.run_evolution(cfg, train, test, storage="fp64")
    replayed = G.replay_lineage(res.lineage, *_initial(cfg, train), cfg)
    assert np.array_equal(replayed, res.elite_train_semantics)
    # the operator rmse sums sequentially like numpy's cumsum; the engine's
    # fitness is the canonical tile sum: equal to the last ulps
    assert G.rmse(replayed, train.target) == pytest.approx(res.train_fitness[-1], rel=1e-14)


def test_replay_with_wrong_seed_detects_mismatch():
    cfg = RunConfig(population_size=4, random_trees=4, program_size=9, generations=5, seed=31)
    train, test = _ds(3, 2, 11), _ds(3, 2, 12)
    res = G.run_evolution(cfg, train, test, storage="fp64")
    replayed = G.replay_lineage(res.lineage, *_initial(cfg.with_seed(32), train), cfg)
    assert not np.array_equal(replayed, res.elite_train_semantics)


def test_replay_empty_and_truncated_logs():
    cfg = RunConfig(population_size=8, random_trees=6, program_size=15, generations=0, seed=3)
    train, test = _ds(10, 3, 13), _ds(5, 3, 14)
    res = G.run_evolution(cfg, train, test, storage="fp64")
    replayed = G.replay_lineage(res.lineage, *_initial(cfg, train), cfg)
    assert np.array_equal(replayed, res.elite_train_semantics)
    assert G.rmse(replayed, train.target) == pytest.approx(res.train_fitness[0], rel=1e-14)
    cfg6 = dataclasses.replace(cfg, generations=6)
    res6 = G.run_evolution(cfg6, train, test)
    truncated = dataclasses.replace(res6.lineage)
    truncated.entries = res6.lineage.entries[:-1]
    with pytest.raises(LineageError):
        G.replay_lineage(truncated, *_initial(cfg6, train), cfg6)


@pytest.mark.parametrize("name", ["plus", "accept", "c1"])
def test_device_replay_reproduces_reference_elite_of_golden_runs(name):
    """gsgp_replay (one device call: plans uploaded once, fp64 GSM and elite
    restores on the device) on the REFERENCE's lineage reproduces the
    reference's final elite semantics bit for bit (the reference's own
    replay contract, pkg/tests/test_evolution.py:197-217)."""
    import ast
    from conftest import golden
    g = golden(f"run_{name}")
    if "u" not in g.files:
        pytest.skip("golden without stored plans")
    cfg = RunConfig(**ast.literal_eval(str(g["cfg"][0])))
    train = G.Dataset(g["Xtr"], g["ytr"])
    log = G.LineageLog(G.EliteRecord("initial", int(g["init"][0]), int(g["init"][0]), float(g["init_fit"][0])))
    for t in range(cfg.generations):
        src = "parent" if g["src"][t] == 0 else "offspring"
        log.entries.append(G.LineageEntry(G.MutationPlan(g["u"][t], g["v"][t], g["ms"][t]),
                                          G.EliteRecord(src, int(g["idx"][t]), int(g["slot"][t]),
                                                        float(g["fit"][t]))))
    init, trees = _initial(cfg, train)
    replayed = G.replay_lineage(log, init, trees, cfg)
    # The replay machinery is exact: the oracle's replay loop (numpy, the
    # reference's op order) fed the device's own sigmoid values reproduces
    # the device replay bit for bit.
    from oracle import restate as R
    sq = G.sigmoid_array(trees)
    cur = init.copy()
    for e in log.entries:
        nxt, _ = R.gsm_squashed(cur, sq, e.plan.u, e.plan.v, e.plan.ms, cfg.gsm_sign)
        if e.elite.source == "parent":
            nxt[e.elite.slot] = cur[e.elite.index]
        cur = nxt
    assert np.array_equal(replayed, cur[log.final_elite().slot])
    # Against the reference's own elite semantics the sigmoid is the one
    # inexact step: numpy's SIMD exp is not correctly rounded (it differs from
    # the correctly rounded exp on ~5 % of inputs in this image) and neither
    # is CUDA's exp (<= 1 ulp), so sigma(tree) can differ in the last bit and
    # the replay agrees to the fp64 tolerance below, not bitwise.
    np.testing.assert_allclose(replayed, g["elite_sem"], rtol=1e-12, atol=1e-12)


def test_device_replay_validates_plans_like_the_reference():
    cfg = RunConfig(population_size=4, random_trees=3, program_size=9, generations=2, seed=3)
    train, test = _ds(6, 2, 21), _ds(3, 2, 22)
    res = G.run_evolution(cfg, train, test, storage="fp64")
    init, trees = _initial(cfg, train)
    bad = dataclasses.replace(res.lineage)
    bad.entries = list(res.lineage.entries)
    e = bad.entries[1]
    bad.entries[1] = G.LineageEntry(G.MutationPlan(e.plan.v, e.plan.v, e.plan.ms), e.elite)   # u == v
    with pytest.raises(ConfigError):
        G.replay_lineage(bad, init, trees, cfg)
    with pytest.raises(ConfigError):
        G.replay_lineage(res.lineage, init, trees[:, :-1], cfg)


def test_gsm_every_slot_mutated_and_timings():
    # pkg/tests/test_evolution.py:180-195 and :256-262
    cfg = RunConfig(population_size=16, random_trees=8, program_size=15, generations=4, seed=9)
    train, test = _ds(15, 2, 15), _ds(6, 2, 16)
    res = G.run_evolution(cfg, train, test)
    t = res.timings
    assert t.create_population_ms >= 0 and t.compute_semantics_ms >= 0 and t.total_ms > 0
    assert t.per_generation_ms >= 0
    with pytest.raises(ConfigError):
        G.run_evolution(cfg, _ds(10, 3, 1), _ds(10, 2, 2))


def _files(tmp_path, runs=1, **extra):
    tr, te = tmp_path / "train.txt", tmp_path / "test.txt"
    G.write_dataset(tr, _ds(20, 3, 1))
    G.write_dataset(te, _ds(8, 3, 2))
    cfg = {"population_size": 12, "random_trees": 6, "program_size": 15, "generations": 5,
           "runs": runs, "seed": 7, **extra}
    c = tmp_path / "run.ini"
    c.write_text("\n".join(f"{k} = {v}" for k, v in cfg.items()) + "\n")
    return tr, te, c


def _cli(tr, te, c, out, *extra):
    return G.run_cli(["-train_file", str(tr), "-test_file", str(te), "-config", str(c),
                      "-output_dir", str(out), *extra])


def test_cli_behaviours(tmp_path, capsys):
    tr, te, c = _files(tmp_path)
    assert _cli(tr, te, c, tmp_path / "a") == 0 and _cli(tr, te, c, tmp_path / "b") == 0
    blob = lambda d: b"".join((d / n).read_bytes() for n in            # noqa: E731
                              ("fitnesstrain.txt", "fitnesstest.txt", "lineage_run000.txt"))
    assert blob(tmp_path / "a") == blob(tmp_path / "b")                # same seed: byte-identical
    vals = [float(x) for x in (tmp_path / "a" / "fitnesstrain.txt").read_text().split()]
    assert len(vals) == 6 and all(b <= a for a, b in zip(vals, vals[1:]))
    assert "train RMSE" in capsys.readouterr().out
    _cli(tr, te, c, tmp_path / "s1", "-seed", "101")
    _cli(tr, te, c, tmp_path / "s2", "-seed", "102")
    assert (tmp_path / "s1" / "fitnesstrain.txt").read_text() != (tmp_path / "s2" / "fitnesstrain.txt").read_text()
    # -backend / -threads change nothing in the results
    _cli(tr, te, c, tmp_path / "t1", "-backend", "sequential")
    _cli(tr, te, c, tmp_path / "t2", "-backend", "threads", "-threads", "4")
    assert (tmp_path / "t1" / "fitnesstrain.txt").read_bytes() == (tmp_path / "t2" / "fitnesstrain.txt").read_bytes()


def test_cli_multiple_runs_and_errors(tmp_path, capsys):
    tr, te, c = _files(tmp_path, runs=3)
    assert _cli(tr, te, c, tmp_path / "o") == 0
    lines = (tmp_path / "o" / "fitnesstrain.txt").read_text().splitlines()
    assert len(lines) == 18 and len({tuple(lines[i:i + 6]) for i in range(0, 18, 6)}) == 3
    assert all((tmp_path / "o" / f"lineage_run{i:03d}.txt").exists() for i in range(3))
    tr, te, c = _files(tmp_path, fitness_cases=9999)
    capsys.readouterr()
    assert _cli(tr, te, c, tmp_path / "x") == 1 and "fitness cases" in capsys.readouterr().err
    assert G.run_cli(["-train_file", str(tmp_path / "nope.txt"),
                      "-test_file", str(tmp_path / "nope.txt")]) == 1
    assert "error" in capsys.readouterr().err


def test_cli_subprocess_runs_are_byte_identical(tmp_path):
    # pkg/tests/test_io_cli.py:345-366: two OS processes, identical files
    tr, te, c = _files(tmp_path)
    outs = []
    for name in ("p", "q"):
        out = tmp_path / name
        subprocess.run([sys.executable, "-m", "paper_2106_04034_b200", "-train_file", str(tr),
                        "-test_file", str(te), "-config", str(c), "-output_dir", str(out)],
                       check=True, cwd=ROOT, capture_output=True)
        outs.append((out / "fitnesstrain.txt").read_bytes() + (out / "lineage_run000.txt").read_bytes())
    assert outs[0] == outs[1]
