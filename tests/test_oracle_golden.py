"""Pin the CPU oracle (oracle/restate.py) to golden vectors produced by the
real reference package (tests/golden/make_golden.py).  CPU only."""

from __future__ import annotations

import ast

import numpy as np
import pytest

from conftest import golden
from oracle import restate as R


def test_rng_bits_units_and_derived_seeds():
    g = golden("rng")
    for s, st, c, b, u in zip(g["seeds"], g["streams"], g["counters"], g["bits"], g["units"]):
        assert R.bits(int(s), int(st), int(c)) == int(b)
        assert R.unit(int(s), int(st), int(c)) == float(u)
    for s, i, d in g["derive"]:
        assert R.run_seed(int(s), int(i)) == int(d)
    assert np.array_equal(R.unit_vec(9, 3, np.arange(4096)), g["vec_seed9_stream3"])


def test_survey_appendix_a_vectors():
    assert R.bits(1, 0, 0) == 0x6E6D5900270F900A
    assert R.bits(-3, 0, 0) == 0x0B01C1CA02803781
    assert R.unit(1, 0, 0) == 0.4313560128567231
    assert R.run_seed(1, 0) == 3140439631417119954
    u, v, ms = R.plan(6, 8, 21, 1)
    assert u.tolist() == [2, 6, 6, 5, 6, 6] and v.tolist() == [3, 1, 1, 6, 2, 1]
    assert ms[0] == 0.830410780131767


def test_population_bit_exact():
    g = golden("population")
    for n, (count, k, l, seed, base, pf, px, pc, lo, hi) in enumerate(g["meta"]):
        tags, codes, consts = R.genomes(int(count), int(k), int(l), int(seed), int(base),
                                        pf, px, pc, lo, hi)
        assert np.array_equal(tags, g[f"tags{n}"])
        assert np.array_equal(codes, g[f"codes{n}"])
        assert np.array_equal(consts.view(np.uint64), g[f"consts{n}"].view(np.uint64))


def test_interpreter_random_genes_bit_exact():
    g = golden("interpreter")
    for i in range(len(g["rand_lens"])):
        n = int(g["rand_lens"][i])
        t, c, v = g["rand_tags"][i, :n], g["rand_codes"][i, :n], g["rand_consts"][i, :n]
        S, _ = R.semantics(t[None], c[None], v[None], g["rand_cases"], 1e-6)
        assert np.array_equal(S[0], g["rand_out"][i])
        for j, x in enumerate(g["rand_cases"][:3]):
            assert R.interpret_one(t, c, v, x, 1e-6) == S[0, j] or (
                not np.isfinite(R.interpret_one(t, c, v, x, 1e-6)))


@pytest.mark.parametrize("name", ["toy", "k127", "k1024", "k255_l100"])
def test_interpreter_sampled_genomes_bit_exact(name):
    g = golden("interpreter")
    S, ovf = R.semantics(g[f"{name}_tags"], g[f"{name}_codes"], g[f"{name}_consts"],
                         g[f"{name}_X"], 1e-6)
    assert np.array_equal(S.view(np.uint64), g[f"{name}_S"].view(np.uint64))
    assert ovf == int(g[f"{name}_overflow"])


def test_interpreter_overflow_kat():
    g = golden("interpreter")
    S, ovf = R.semantics(g["ovf_tags"], g["ovf_codes"], g["ovf_consts"], g["ovf_X"], 1e-6)
    assert np.array_equal(S, g["ovf_S"]) and ovf == int(g["ovf_count"]) == 5


def test_fitness_plan_gsm_survival_bit_exact():
    g = golden("ops")
    assert np.array_equal(R.fitness(g["fit_S"], g["fit_y"]), g["fit_out"])
    for m, r, seed, gen, step in g["plan_meta"]:
        key = f"plan_{m}_{r}_{gen}_{seed % 1000}_{step}"
        u, v, ms = R.plan(int(m), int(r), int(seed), int(gen), step)
        assert np.array_equal(u, g[key + "_u"]) and np.array_equal(v, g[key + "_v"])
        assert np.array_equal(ms, g[key + "_ms"])
    for sign in ("minus", "plus"):
        out, _ = R.gsm_squashed(g[f"gsm_{sign}_P"], R.sigmoid(g[f"gsm_{sign}_T"]),
                                g[f"gsm_{sign}_u"], g[f"gsm_{sign}_v"], g[f"gsm_{sign}_ms"], sign)
        assert np.array_equal(out, g[f"gsm_{sign}_out"])
    for a, b, (src, idx, slot) in zip(g["surv_par"], g["surv_off"], g["surv_dec"]):
        s, i, w = R.survive(a, b)
        assert (0 if s == "parent" else 1, i, w) == (src, idx, slot)
    X, y = R.benchmark_dataset(3, 5, seed=1)
    assert np.array_equal(X, g["bench_X"]) and np.array_equal(y, g["bench_y"])


@pytest.mark.parametrize("name", ["tiny", "small", "plus", "g0", "accept", "c1", "wide", "m1", "k1",
                                  "n1", "const", "funcs", "hugestep", "infstep"])
def test_full_run_bit_exact(name):
    g = golden(f"run_{name}")
    cfg = R.Cfg(**ast.literal_eval(str(g["cfg"][0])))
    out = R.run(cfg, g["Xtr"], g["ytr"], g["Xte"], g["yte"])
    assert np.array_equal(out["train"], g["train"])
    assert np.array_equal(out["test"], g["test"])
    src = np.array([0 if e[0] == "parent" else 1 for e in out["elite"]], np.int8)
    assert np.array_equal(src, g["src"])
    assert [e[1] for e in out["elite"]] == g["idx"].tolist()
    assert [e[2] for e in out["elite"]] == g["slot"].tolist()
    assert np.array_equal(out["elite_train_semantics"], g["elite_sem"])
    assert out["overflow"] == int(g["overflow"][0])
    if "u" in g.files:
        assert np.array_equal(out["u"], g["u"]) and np.array_equal(out["ms"], g["ms"])


def test_split_restatement_matches_reference():
    g = golden("split")
    for key in [k for k in g.files if k.startswith("tr_")]:
        n = int(key[3:])
        frac, seed = g[f"args_{n}"]
        tr, te = R.split_rows(n, float(frac), int(seed))
        assert np.array_equal(tr, g[f"tr_{n}"]) and np.array_equal(te, g[f"te_{n}"]), n


@pytest.mark.parametrize("name", ["mid", "long"])
def test_big_run_restatement_matches_reference(name):
    """Headline-shape goldens (make_golden.py BIG_RUNS, data regenerated from
    make_benchmark_dataset seeds): the restated loop equals the reference's
    traces, elite records, plans and (sampled) elite semantics bit for bit."""
    g = golden(f"big_{name}")
    ntr, l, s1, nte, s2 = (int(x) for x in g["data"])
    Xtr, ytr = R.benchmark_dataset(ntr, l, s1)
    Xte, yte = R.benchmark_dataset(nte, l, s2)
    out = R.run(R.Cfg(**ast.literal_eval(str(g["cfg"][0]))), Xtr, ytr, Xte, yte)
    assert np.array_equal(out["train"], g["train"]) and np.array_equal(out["test"], g["test"])
    assert [e[2] for e in out["elite"]] == g["slot"].tolist()
    assert [e[1] for e in out["elite"]] == g["idx"].tolist()
    assert np.array_equal(out["u"], g["u"]) and np.array_equal(out["v"], g["v"])
    assert np.array_equal(out["ms"], g["ms"])
    assert np.array_equal(out["elite_train_semantics"][::int(g["sample_stride"][0])], g["elite_sem_sample"])
