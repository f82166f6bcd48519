"""Device parity of the hot-path operators against the reference's golden
vectors and the CPU oracle (oracle/).  Integer / index / genome outputs are
bit-exact; fp64 interpreter outputs are bit-exact; fp64 reductions are within
1e-12 relative of the reference's sequential sums.  Runs on a B200."""

from __future__ import annotations

import math
import random

import numpy as np
import pytest

from conftest import golden, toy_dataset
from oracle import engine32, restate as R

pytestmark = pytest.mark.gpu

import paper_2106_04034_b200 as G  # noqa: E402
from paper_2106_04034_b200 import (  # noqa: E402
    Chromosome, ConfigError, FunctionOp, Gene, GeneTag, MutationPlan, Population, RunConfig,
    RunStats,
)


@pytest.fixture(scope="module", autouse=True)
def _device(lib):
    yield


# ------------------------------------------------------------------ rng
def test_rng_bits_and_units_bit_exact():
    g = golden("rng")
    for s, st, c, b, u in zip(g["seeds"], g["streams"], g["counters"], g["bits"], g["units"]):
        assert G.rng_bits(int(s), int(st), int(c)) == int(b)
        assert G.rng_stream(int(s), int(st), int(c)) == float(u)
    assert np.array_equal(G.uniform_array(9, 3, np.arange(4096)), g["vec_seed9_stream3"])
    assert G.rng_bits(-3, 0, 0) == 0x0B01C1CA02803781


def test_rng_bulk_matches_oracle():
    c = np.arange(1_000_003, dtype=np.uint64) * np.uint64(7919)
    assert np.array_equal(G.uniform_array(2**63 + 11, 2**40 + 3, c),
                          R.unit_vec(2**63 + 11, 2**40 + 3, c))


# ------------------------------------------------------------ population
def test_population_bit_exact_against_reference():
    g = golden("population")
    for n, (count, k, l, seed, base, pf, px, pc, lo, hi) in enumerate(g["meta"]):
        cfg = RunConfig(program_size=int(k), seed=int(seed), p_function=pf, p_feature=px,
                        p_constant=pc, erc_low=lo, erc_high=hi)
        pop = G.create_population(int(count), cfg, int(base), int(l))
        assert np.array_equal(pop.tags, g[f"tags{n}"])
        assert np.array_equal(pop.codes, g[f"codes{n}"])
        assert np.array_equal(pop.consts.view(np.uint64), g[f"consts{n}"].view(np.uint64))


def test_population_large_matches_oracle():
    # the paper's benchmark genome shape, 10240 x 127 over 1024 features
    cfg = RunConfig(program_size=127, seed=99)
    pop = G.create_population(10240, cfg, 5, 1024)
    t, c, v = R.genomes(10240, 127, 1024, 99, 5)
    assert np.array_equal(pop.tags, t) and np.array_equal(pop.codes, c)
    assert np.array_equal(pop.consts, v)


def test_sample_gene_matches_rows():
    cfg = RunConfig(program_size=64, seed=3)
    pop = G.create_population(2, cfg, 17, 4)
    for j in (0, 5, 63):
        gene = G.sample_gene(cfg, 18, j, 4)
        assert (gene.tag, gene.code, gene.value) == (pop.tags[1, j], pop.codes[1, j], pop.consts[1, j])


# ------------------------------------------------------------ interpreter
F = lambda op: Gene(GeneTag.FUNCTION, op)  # noqa: E731
X = lambda i: Gene(GeneTag.FEATURE, i)  # noqa: E731
Cst = lambda v: Gene(GeneTag.CONSTANT, 0, v)  # noqa: E731


def run1(genes, case, eps=1e-6):
    return G.interpret(Chromosome.from_genes(genes), case, eps)


def test_interpreter_known_answers():
    # pkg/tests/test_interpreter.py:36-73
    assert run1([X(0), X(1), F(FunctionOp.ADD)], (2.0, 3.0)) == 5.0
    assert run1([F(FunctionOp.ADD), X(0)], (7.0,)) == 7.0
    assert run1([Cst(4.0), Cst(0.0), F(FunctionOp.DIV)], ()) == 1.0
    assert run1([Cst(2.0), Cst(3.0), F(FunctionOp.MUL), Cst(10.0), F(FunctionOp.SUB)], ()) == -4.0
    assert run1([Cst(2.0), Cst(3.0), F(FunctionOp.ADD), Cst(99.0)], ()) == 5.0
    assert run1([F(FunctionOp.MUL)], ()) == 0.0
    assert run1([Cst(1.5), X(0), Cst(-2.5)], (9.0,)) == -2.5
    assert run1([Cst(1.0), Cst(5e-7), F(FunctionOp.DIV)], ()) == 1.0
    assert run1([Cst(1.0), Cst(2e-6), F(FunctionOp.DIV)], ()) == 1.0 / 2e-6
    # operand order with feature operands on both sides and deep spills
    genes = [X(0), X(1), F(FunctionOp.SUB), X(1), X(0), F(FunctionOp.DIV), F(FunctionOp.SUB)]
    assert run1(genes, (3.0, 5.0)) == (3.0 - 5.0) - (5.0 / 3.0)


def test_interpreter_random_genes_bit_exact():
    g = golden("interpreter")
    for i in range(len(g["rand_lens"])):
        n = int(g["rand_lens"][i])
        pop = Population(g["rand_tags"][i:i + 1, :n].copy(), g["rand_codes"][i:i + 1, :n].copy(),
                         g["rand_consts"][i:i + 1, :n].copy())
        S = G.compute_semantics(pop, g["rand_cases"], RunConfig(program_size=n))
        assert np.array_equal(S[0], g["rand_out"][i]), i


@pytest.mark.parametrize("name", ["toy", "k127", "k1024", "k255_l100"])
def test_interpreter_sampled_genomes_bit_exact(name):
    g = golden("interpreter")
    pop = Population(g[f"{name}_tags"], g[f"{name}_codes"], g[f"{name}_consts"])
    stats = RunStats()
    S = G.compute_semantics(pop, g[f"{name}_X"], RunConfig(program_size=pop.genome_length), stats=stats)
    assert np.array_equal(S.view(np.uint64), g[f"{name}_S"].view(np.uint64))
    assert stats.overflow_replacements == int(g[f"{name}_overflow"])


def test_interpreter_overflow_replaced_and_counted():
    g = golden("interpreter")
    stats = RunStats()
    pop = Population(g["ovf_tags"], g["ovf_codes"], g["ovf_consts"])
    S = G.compute_semantics(pop, g["ovf_X"], RunConfig(program_size=3), stats=stats)
    assert np.array_equal(S, g["ovf_S"]) and stats.overflow_replacements == 5


def test_interpreter_hypothesis_style_random_against_oracle():
    pyrng = random.Random(77)
    Xc = np.array([[pyrng.uniform(-3, 3) for _ in range(3)] for _ in range(257)])
    for k in (1, 2, 3, 9, 64, 300):
        tags = np.array([[pyrng.choice([0, 0, 1, 2]) for _ in range(k)] for _ in range(40)], np.uint8)
        codes = np.where(tags == 0, np.random.default_rng(k).integers(0, 4, (40, k)),
                         np.where(tags == 1, np.random.default_rng(k + 1).integers(0, 3, (40, k)), 0)).astype(np.int32)
        consts = np.where(tags == 2, np.random.default_rng(k + 2).uniform(-2, 2, (40, k)), 0.0)
        S = G.compute_semantics(Population(tags, codes, consts), Xc, RunConfig(program_size=k))
        ref, _ = R.semantics(tags, codes, consts, Xc, 1e-6)
        assert np.array_equal(S, ref)


def test_interpreter_feature_range_and_case_permutation():
    pop = Population.from_chromosomes([Chromosome.from_genes([X(5)])])
    Xd, _ = toy_dataset(n_features=3)
    with pytest.raises(ConfigError):
        G.compute_semantics(pop, Xd, RunConfig(program_size=1))
    g = golden("interpreter")
    pop = Population(g["k127_tags"], g["k127_codes"], g["k127_consts"])
    perm = np.random.default_rng(0).permutation(g["k127_X"].shape[0])
    a = G.compute_semantics(pop, g["k127_X"], RunConfig(program_size=127))
    b = G.compute_semantics(pop, g["k127_X"][perm], RunConfig(program_size=127))
    assert np.array_equal(b, a[:, perm])


def _wide_exponent_values(rng, n):
    """fp64 values with exponents spread over the whole range (subnormals,
    the interpreter's fast-division thresholds 2^-500 / 2^501, huge), signed
    zeros and values near the protection threshold eps."""
    v = rng.uniform(1, 2, n) * np.exp2(rng.integers(-1074, 1024, n).astype(np.float64))
    v[rng.random(n) < 0.5] *= -1
    special = np.array([0.0, -0.0, 5e-324, -1e-310, 2.0 ** -500, np.nextafter(2.0 ** -500, 0),
                        2.0 ** 501, np.nextafter(2.0 ** 501, 0), 1e308, -1e308, 1e-6,
                        np.nextafter(1e-6, 0), -1e-6, 1.0, -3.7])
    v[: special.size] = special
    with np.errstate(all="ignore"):
        return np.where(np.isfinite(v), v, 1.0)


def test_interpreter_division_bit_exact_over_the_exponent_range():
    """x0 / x1 and x1 / x0 (both operand roles of the protected division, and
    the leaf-pair, accumulator and reversed forms) on 200k cases whose
    exponents span subnormals to 2^1023: bit-exact with numpy's IEEE
    division (the device uses an interleaved Newton fast path inside
    [2^-500, 2^501) and div.rn elsewhere)."""
    rng = np.random.default_rng(11)
    n = 200_000
    X = np.stack([_wide_exponent_values(rng, n), _wide_exponent_values(rng, n)[rng.permutation(n)],
                  rng.uniform(-1, 1, n)], axis=1)
    F, V, DIV = int(GeneTag.FUNCTION), int(GeneTag.FEATURE), int(FunctionOp.DIV)
    progs = [
        [(V, 0), (V, 1), (F, DIV)],                                  # leaf pair x0 / x1
        [(V, 1), (V, 0), (F, DIV)],                                  # leaf pair x1 / x0
        [(V, 0), (V, 2), (V, 2), (F, 0), (F, DIV)],                  # x0 / acc (reversed)
        [(V, 2), (V, 2), (F, 2), (V, 1), (F, DIV)],                  # acc / x1
        [(V, 0), (V, 2), (F, 0), (V, 1), (V, 2), (F, 1), (F, DIV)],  # stack / acc
        [(V, 0), (V, 1), (F, DIV), (V, 1), (V, 0), (F, DIV), (F, DIV)],
    ]
    k = max(len(p) for p in progs)
    tags = np.full((len(progs), k), int(GeneTag.CONSTANT), np.uint8)
    codes = np.zeros((len(progs), k), np.int32)
    consts = np.zeros((len(progs), k))
    for i, p in enumerate(progs):
        # pad at the front with constants that are dropped (never reach the output)
        off = k - len(p)
        consts[i, :off] = 2.5
        for j, (t, c) in enumerate(p):
            tags[i, off + j], codes[i, off + j] = t, c
    S = G.compute_semantics(Population(tags, codes, consts), X, RunConfig(program_size=k))
    ref, _ = R.semantics(tags, codes, consts, X, 1e-6)
    assert np.array_equal(S.view(np.uint64), ref.view(np.uint64))


def test_interpreter_division_heavy_random_programs_edge_features():
    rng = np.random.default_rng(5)
    X = np.stack([_wide_exponent_values(rng, 4099) for _ in range(4)], axis=1)
    for k in (3, 15, 63, 255, 1024):
        m = 48
        tags = rng.choice([0, 0, 1, 2], size=(m, k), p=[0.4, 0.2, 0.3, 0.1]).astype(np.uint8)
        ops = np.where(rng.random((m, k)) < 0.6, 3, rng.integers(0, 3, (m, k)))
        codes = np.where(tags == 0, ops, np.where(tags == 1, rng.integers(0, 4, (m, k)), 0)).astype(np.int32)
        consts = np.where(tags == 2, _wide_exponent_values(rng, m * k).reshape(m, k), 0.0)
        S = G.compute_semantics(Population(tags, codes, consts), X, RunConfig(program_size=k))
        ref, _ = R.semantics(tags, codes, consts, X, 1e-6)
        assert np.array_equal(S.view(np.uint64), ref.view(np.uint64)), k


def test_interpreter_many_features_global_path():
    # l = 2000 features exceeds the shared-memory feature tile: global path
    cfg = RunConfig(program_size=255, seed=4)
    pop = G.create_population(24, cfg, 0, 2000)
    Xd = np.random.default_rng(1).uniform(-1, 1, (300, 2000))
    S = G.compute_semantics(pop, Xd, cfg)
    ref, _ = R.semantics(pop.tags, pop.codes, pop.consts, Xd, 1e-6)
    assert np.array_equal(S, ref)


# --------------------------------------------------------------- fitness
def test_fitness_against_reference_sequential_sums():
    g = golden("ops")
    got = G.compute_fitness(g["fit_S"], g["fit_y"])
    ref = g["fit_out"]
    assert got[7] == ref[7] == math.inf
    assert got[5] == 0.0
    np.testing.assert_array_equal(got, ref)       # same left-to-right order: bitwise
    assert G.rmse([0.0, 0.0], [3.0, 4.0]) == 3.5355339059327378
    assert G.rmse([1e200, 0.0], [-1e200, 0.0]) == math.inf


@pytest.mark.parametrize("m,n", [(1, 1), (3, 63), (31, 64), (33, 65), (70, 1000), (5, 100_003)])
def test_fitness_is_bitwise_numpy_cumsum_order(m, n):
    """gsgp/fitness.py:43-48: np.cumsum(diff * diff, axis=1)[:, -1] is a
    strictly sequential sum; the operator kernel keeps that order, so the
    RMSE is bitwise the reference's for every shape (rows straddling the
    kernel's 32-row blocks and 64-column tiles)."""
    rng = np.random.default_rng(m * 1000 + n)
    S = rng.lognormal(0, 4, (m, n)) * rng.choice([-1.0, 1.0], (m, n))
    y = rng.normal(0, 3, n)
    with np.errstate(all="ignore"):
        want = np.sqrt(np.cumsum((S - y) * (S - y), axis=1)[:, -1] / n)
    want = np.where(np.isfinite(want), want, math.inf)
    np.testing.assert_array_equal(G.compute_fitness(S, y), want)


# ------------------------------------------------------------------ plan
def test_plans_bit_exact():
    g = golden("ops")
    for m, r, seed, gen, step in g["plan_meta"]:
        key = f"plan_{m}_{r}_{gen}_{seed % 1000}_{step}"
        p = G.build_mutation_plan(int(m), int(r), RunConfig(seed=int(seed), mutation_step=step), int(gen))
        assert np.array_equal(p.u, g[key + "_u"]) and np.array_equal(p.v, g[key + "_v"])
        assert np.array_equal(p.ms, g[key + "_ms"])
    with pytest.raises(ConfigError):
        G.build_mutation_plan(8, 1, RunConfig(), 1)


# ------------------------------------------------------------------- GSM
@pytest.mark.parametrize("sign", ["minus", "plus"])
def test_gsm_fp64_operator_matches_reference(sign):
    g = golden("ops")
    plan = MutationPlan(g[f"gsm_{sign}_u"], g[f"gsm_{sign}_v"], g[f"gsm_{sign}_ms"])
    out = G.gsm(g[f"gsm_{sign}_P"], g[f"gsm_{sign}_T"], plan, RunConfig(gsm_sign=sign))
    np.testing.assert_allclose(out, g[f"gsm_{sign}_out"], rtol=0, atol=1e-12)
    # with the reference's own squashed pool the result is bit-exact
    sq = R.sigmoid(g[f"gsm_{sign}_T"])
    exact = G.ops._gsm_squashed(g[f"gsm_{sign}_P"], sq, plan, sign)
    assert np.array_equal(exact, g[f"gsm_{sign}_out"])


def test_gsm_contract_zero_step_and_validation():
    rng = np.random.default_rng(1)
    P = rng.normal(size=(6, 40)) * 10
    T = rng.normal(size=(5, 40))
    plan = MutationPlan(np.array([0, 1, 2, 3, 4, 0]), np.array([1, 2, 3, 4, 0, 2]), np.zeros(6))
    assert np.array_equal(G.gsm(P, T, plan, RunConfig()), P)
    with pytest.raises(ConfigError):
        G.gsm(P, T, MutationPlan(plan.u + 100, plan.v, plan.ms), RunConfig())
    with pytest.raises(ConfigError):
        G.gsm(P[:, :-1], T, plan, RunConfig())


@pytest.mark.parametrize("ntr,nte", [(1, 1), (31, 0), (500, 200), (2048, 2048), (4099, 1025),
                                     (10_000, 2_500)])
@pytest.mark.parametrize("sign", ["minus", "plus"])
def test_engine_gsm_step_f32_bit_exact(ntr, nte, sign):
    rng = np.random.default_rng(ntr + nte)
    m, r = 19, 7
    Ptr = (rng.normal(size=(m, ntr)) * 30).astype(np.float32)
    Pte = (rng.normal(size=(m, nte)) * 30).astype(np.float32)
    Q = rng.uniform(0, 1, size=(r, ntr + nte)).astype(np.float32)
    ytr, yte = rng.normal(size=ntr), rng.normal(size=nte)
    u = rng.integers(0, r, m)
    v = (u + 1 + rng.integers(0, r - 1, m)) % r
    ms = 1.0 - rng.uniform(size=m)
    plan = MutationPlan(u, v, ms)
    otr, ote, s_tr, s_te = G.gsm_step_f32(Ptr, Pte, Q[:, :ntr], Q[:, ntr:], ytr, yte, plan, sign)
    assert np.array_equal(otr, engine32.gsm_step32(Ptr, Q[:, :ntr], u, v, ms, sign))
    assert np.array_equal(ote, engine32.gsm_step32(Pte, Q[:, ntr:], u, v, ms, sign))
    ref_tr = np.array([math.fsum((otr[i].astype(np.float64) - ytr) ** 2) for i in range(m)])
    np.testing.assert_allclose(s_tr, ref_tr, rtol=1e-12)
    if nte:
        ref_te = np.array([math.fsum((ote[i].astype(np.float64) - yte) ** 2) for i in range(m)])
        np.testing.assert_allclose(s_te, ref_te, rtol=1e-12)
    else:
        assert np.all(s_te == 0.0)


def test_engine_sse_is_bitwise_equal_for_equal_rows():
    # determinism: identical rows -> identical SSE (ties resolve like np.argmin)
    rng = np.random.default_rng(5)
    m, n = 12, 9000
    Ptr = np.repeat((rng.normal(size=(1, n)) * 3).astype(np.float32), m, axis=0)
    Q = np.zeros((2, n), np.float32)
    plan = MutationPlan(np.zeros(m, np.int64), np.ones(m, np.int64), np.full(m, 0.5))
    _, _, s_tr, _ = G.gsm_step_f32(Ptr, Ptr[:, :0], Q, Q[:, :0], rng.normal(size=n), np.zeros(0), plan)
    assert np.all(s_tr == s_tr[0])


# -------------------------------------------------------------- survival
def test_survival_decisions_bit_exact():
    g = golden("ops")
    for a, b, (src, idx, slot) in zip(g["surv_par"], g["surv_off"], g["surv_dec"]):
        s, i, w = G.ops.survive_decision(a, b)
        assert (0 if s == "parent" else 1, i, w) == (src, idx, slot)
    assert G.argmin_fitness(np.array([5.0, 5.0, 5.0])) == 0
    assert G.argmin_fitness(np.full(4, math.inf)) == 0
    assert G.argmax_fitness(np.array([1.0, 2.0, 2.0])) == 1
    assert G.argmax_fitness(np.array([1.0, math.inf, 2.0])) == 1
    with pytest.raises(ConfigError):
        G.argmin_fitness(np.empty(0))


def test_survive_state_copy():
    def st(f, off):
        m = len(f)
        return G.GenerationState(np.arange(m * 3.0).reshape(m, 3) + off, np.array(f, float),
                                 np.arange(m * 2.0).reshape(m, 2) - off)
    parent = st([0.9, 0.5, 0.7, 0.8], 0)
    nxt, e = G.survive(parent, st([1.0, 1.2, 0.9, 3.0], 50))
    assert (e.source, e.index, e.slot) == ("parent", 1, 3)
    assert np.array_equal(nxt.train_semantics[3], parent.train_semantics[1])
    assert nxt.fitness[3] == 0.5


def test_interpreter_lean_configuration_matches(monkeypatch):
    """The lean launch configuration (program and constants read from HBM,
    only spill rows in shared memory: the fallback for programs too large to
    stage) gives bit-identical semantics, with many constants per genome."""
    rng = np.random.default_rng(9)
    X = rng.uniform(-2, 2, (700, 5))
    k, m = 511, 16
    tags = rng.choice([0, 1, 2], size=(m, k), p=[0.5, 0.2, 0.3]).astype(np.uint8)
    codes = np.where(tags == 0, rng.integers(0, 4, (m, k)),
                     np.where(tags == 1, rng.integers(0, 5, (m, k)), 0)).astype(np.int32)
    consts = np.where(tags == 2, rng.uniform(1, 10, (m, k)), 0.0)
    pop = Population(tags, codes, consts)
    ref, _ = R.semantics(tags, codes, consts, X, 1e-6)
    a = G.compute_semantics(pop, X, RunConfig(program_size=k))
    monkeypatch.setenv("GSGP_INTERP_CFG", "4")
    b = G.compute_semantics(pop, X, RunConfig(program_size=k))
    assert np.array_equal(a.view(np.uint64), ref.view(np.uint64))
    assert np.array_equal(b.view(np.uint64), ref.view(np.uint64))


def _hard_division_operands(rng, n):
    """In-range (|v| in [2^-499, 2^499]) operands dominated by near-halfway
    quotients: mantissas 1 - j*2^-53 and 1 + j*2^-52 for small j, powers of
    two, and random mantissas, with random exponents and signs."""
    kind = rng.integers(0, 4, n)
    j = rng.integers(1, 64, n).astype(np.float64)
    mant = np.where(kind == 0, 1.0 - j * 2.0 ** -53,
                    np.where(kind == 1, 1.0 + j * 2.0 ** -52,
                             np.where(kind == 2, 1.0, rng.uniform(1, 2, n))))
    v = mant * np.exp2(rng.integers(-499, 499, n).astype(np.float64))
    return np.where(rng.random(n) < 0.5, -v, v)


def test_interpreter_division_fast_path_near_halfway_quotients():
    """Every case of every group inside the fast-path range, so whole groups
    take the Newton path: x0/x1, x1/x0 and 1/x for near-halfway operands
    (1/nextafter(2^501, 0) misrounded with a zero-low-word reciprocal seed)
    must be bit-exact with numpy's IEEE division, for every tile config."""
    rng = np.random.default_rng(21)
    n = 300_000
    X = np.stack([_hard_division_operands(rng, n), _hard_division_operands(rng, n)], axis=1)
    F, V, DIV = int(GeneTag.FUNCTION), int(GeneTag.FEATURE), int(FunctionOp.DIV)
    progs = [[(V, 0), (V, 1), (F, DIV)],
             [(V, 1), (V, 0), (F, DIV)],
             [(V, 0), (V, 0), (F, DIV), (V, 1), (F, DIV)],            # 1 / x1 (x0/x0 == 1)
             [(V, 1), (V, 1), (F, DIV), (V, 0), (F, DIV), (V, 1), (F, DIV)]]
    k = max(len(p) for p in progs)
    tags = np.full((len(progs), k), int(GeneTag.CONSTANT), np.uint8)
    codes = np.zeros((len(progs), k), np.int32)
    consts = np.full((len(progs), k), 2.5)
    for i, p in enumerate(progs):
        off = k - len(p)
        for jj, (t, c) in enumerate(p):
            tags[i, off + jj], codes[i, off + jj] = t, c
    ref, _ = R.semantics(tags, codes, consts, X, 1e-6)
    pop = Population(tags, codes, consts)
    import os
    for cfg in ("0", "1", "2", "3", "4", "5", "6", "7", "9", "10"):
        os.environ["GSGP_INTERP_CFG"] = cfg
        try:
            S = G.compute_semantics(pop, X, RunConfig(program_size=k))
        finally:
            del os.environ["GSGP_INTERP_CFG"]
        assert np.array_equal(S.view(np.uint64), ref.view(np.uint64)), cfg


def test_dataset_split_matches_reference_golden():
    """Dataset.split (gsgp/core.py:179-192) with device-drawn uniforms: the
    same rows on each side as the reference for several sizes and seeds."""
    g = golden("split")
    for key in [k for k in g.files if k.startswith("tr_")]:
        n = int(key[3:])
        frac, seed = g[f"args_{n}"]
        X = np.stack([np.arange(n, dtype=np.float64), np.ones(n)], axis=1)
        tr, te = G.Dataset(X, np.arange(n, dtype=np.float64)).split(float(frac), int(seed))
        assert np.array_equal(tr.features[:, 0].astype(np.int64), g[f"tr_{n}"]), n
        assert np.array_equal(te.features[:, 0].astype(np.int64), g[f"te_{n}"]), n


@pytest.mark.parametrize("count", [1, 2, 3, 5, 17])
@pytest.mark.parametrize("cfg", ["5", "6", "7", "9", "10"])
def test_interpreter_genome_groups_with_odd_counts(count, cfg, monkeypatch):
    """Grouped interpreter blocks (cfg 6: two genome groups of 128 threads
    per block sharing the feature tile) with genome counts that leave a
    group idle or uneven: bit-identical to the oracle and to one group."""
    from oracle import restate as R
    rng = np.random.default_rng(count)
    X = rng.uniform(-3, 3, (1000, 6))
    cfg_run = RunConfig(program_size=63, seed=count)
    pop = G.create_population(count, cfg_run, 0, 6)
    ref, _ = R.semantics(pop.tags, pop.codes, pop.consts, X, 1e-6)
    monkeypatch.setenv("GSGP_INTERP_CFG", cfg)
    S = G.compute_semantics(pop, X, cfg_run)
    assert np.array_equal(S.view(np.uint64), ref.view(np.uint64))


@pytest.mark.parametrize("cfg", ["5", "7", "9", "10"])
def test_interpreter_divisions_by_and_of_constants_and_spills(cfg, monkeypatch):
    """Divisions by and of constants (in range, and out of the fast path's
    range: 0, subnormal, tiny, huge, inf, near eps) and of spill operands:
    every result bit-exact with numpy, guard included
    (gsgp/interpreter.py:58-65)."""
    rng = np.random.default_rng(21)
    n = 3000
    X = np.stack([_hard_division_operands(rng, n), _hard_division_operands(rng, n),
                  rng.uniform(-3, 3, n)], axis=1)
    X[::17, 0] = 0.0
    X[::23, 1] = 5e-7                      # below eps: guard
    X[::29, 2] = 2e-6                      # just above eps
    F, V, C_, DIV = int(GeneTag.FUNCTION), int(GeneTag.FEATURE), int(GeneTag.CONSTANT), int(FunctionOp.DIV)
    cvals = [0.0, 5e-324, 1e-300, 5e-7, 2e-6, 3.5, -2.0 ** 500, 1e300, float("inf"), -7.25e-151]
    progs = []
    for c in cvals:
        progs.append([(V, 0), (C_, c), (F, DIV)])                      # x0 / c
        progs.append([(C_, c), (V, 1), (F, DIV)])                      # c / x1
        progs.append([(V, 0), (V, 2), (F, int(FunctionOp.MUL)), (C_, c), (F, DIV)])    # (x0*x2) / c
        progs.append([(C_, c), (V, 0), (V, 1), (F, int(FunctionOp.SUB)), (F, DIV)])    # c / (x0-x1)
    # spill operands: (x0/x1) / (x1/x2), (x0*x2 - x1) / (x2 + x0 / x1)
    progs.append([(V, 0), (V, 1), (F, DIV), (V, 1), (V, 2), (F, DIV), (F, DIV)])
    progs.append([(V, 0), (V, 2), (F, int(FunctionOp.MUL)), (V, 1), (F, int(FunctionOp.SUB)),
                  (V, 2), (V, 0), (V, 1), (F, DIV), (F, int(FunctionOp.ADD)), (F, DIV)])
    k = max(len(p) for p in progs)
    tags = np.full((len(progs), k), C_, np.uint8)
    codes = np.zeros((len(progs), k), np.int32)
    consts = np.full((len(progs), k), 1.0)
    for i, p in enumerate(progs):
        off = k - len(p)
        for jj, (t, c) in enumerate(p):
            tags[i, off + jj] = t
            if t == C_:
                consts[i, off + jj] = c
            else:
                codes[i, off + jj] = c
    pop = Population(tags, codes, consts)
    monkeypatch.setenv("GSGP_INTERP_CFG", cfg)
    for eps in (1e-6, 1e-9):
        with np.errstate(all="ignore"):
            ref, _ = R.semantics(tags, codes, consts, X, eps)
        S = G.compute_semantics(pop, X, RunConfig(program_size=k, division_eps=eps))
        ok = np.isfinite(ref)
        assert np.array_equal(S[ok].view(np.uint64), ref[ok].view(np.uint64)), (cfg, eps)
        assert np.all(S[~ok] == 0.0)


def test_interpreter_division_by_constants_hard_operands(monkeypatch):
    """Divisions by constants (acc / c, x / c, spill + x / c) with near-halfway
    numerators and hard constants (in range, tiny, huge, zero, near eps), in
    every configuration: bit-exact with numpy, guard included
    (gsgp/interpreter.py:58-65).  (Precomputing the fast path's reciprocal of
    in-range constants was measured slower and not kept: profiles/r02/README.md.)"""
    rng = np.random.default_rng(33)
    n = 60_000
    X = np.stack([_hard_division_operands(rng, n), _hard_division_operands(rng, n),
                  rng.uniform(-3, 3, n)], axis=1)
    X[::41, 0] = 0.0                      # zero numerators: slow path of the group
    X[::43, 1] = 2.0 ** 600               # numerator out of range
    F, V, C_ = int(GeneTag.FUNCTION), int(GeneTag.FEATURE), int(GeneTag.CONSTANT)
    DIV, MUL, SUB = int(FunctionOp.DIV), int(FunctionOp.MUL), int(FunctionOp.SUB)
    cvals = list(_hard_division_operands(rng, 24)) + [1.0, -1.0, 3.0, 0.1, 7.0 / 3.0,
                                                        np.nextafter(2.0 ** 500, 0), 2.0 ** -499,
                                                        1.0000001e-6, 5e-7, 0.0, 1e300]
    progs = []
    for c in cvals:
        progs.append([(V, 0), (C_, c), (F, DIV)])                          # x0 / c          (LDIVC)
        progs.append([(V, 0), (V, 2), (F, MUL), (C_, c), (F, DIV)])        # (x0*x2) / c     (DIVC)
        progs.append([(V, 1), (V, 2), (F, SUB), (V, 0), (V, 2), (F, MUL),  # (x1-x2) (x0*x2) / ...
                      (V, 1), (C_, c), (F, DIV), (F, MUL), (F, DIV)])       # spill + x1 / c  (PDIVC)
    k = max(len(p) for p in progs)
    tags = np.full((len(progs), k), C_, np.uint8)
    codes = np.zeros((len(progs), k), np.int32)
    consts = np.full((len(progs), k), 1.0)
    for i, p in enumerate(progs):
        off = k - len(p)
        for jj, (t, c) in enumerate(p):
            tags[i, off + jj] = t
            if t == C_:
                consts[i, off + jj] = c
            else:
                codes[i, off + jj] = c
    pop = Population(tags, codes, consts)
    for eps in (1e-6, 1e-9):
        with np.errstate(all="ignore"):
            ref, _ = R.semantics(tags, codes, consts, X, eps)
        ok = np.isfinite(ref)
        for cfg in ("0", "1", "3", "5", "6", "7", "4", "9", "10"):
            monkeypatch.setenv("GSGP_INTERP_CFG", cfg)
            S = G.compute_semantics(pop, X, RunConfig(program_size=k, division_eps=eps))
            assert np.array_equal(S[ok].view(np.uint64), ref[ok].view(np.uint64)), (cfg, eps)


def _chain_genome(n_funcs: int, l: int, rng) -> tuple:
    """A postfix chain f0 f1 op f2 op ... whose compiled program is exactly
    n_funcs instructions (one leaf pair, then one accumulator op per
    function), with every operator kind and feature/constant leaves."""
    tags, codes, consts = [R.FEATURE, R.FEATURE], [0, 1 % l], [0.0, 0.0]
    tags.append(R.FUNCTION)
    codes.append(int(rng.integers(4)))
    consts.append(0.0)
    for _ in range(n_funcs - 1):
        if rng.random() < 0.2:
            tags.append(R.CONSTANT)
            codes.append(0)
            consts.append(float(rng.uniform(1, 10)))
        else:
            tags.append(R.FEATURE)
            codes.append(int(rng.integers(l)))
            consts.append(0.0)
        tags.append(R.FUNCTION)
        codes.append(int(rng.integers(4)))
        consts.append(0.0)
    return tags, codes, consts


@pytest.mark.parametrize("cfg", ["9", "10"])
def test_interpreter_program_ring_chunk_boundaries(cfg, monkeypatch):
    """Programs whose compiled length sits on and around the one-warp groups'
    32-instruction ring chunks (cfg 9 refills chunk c + 1 at the start of
    chunk c) are bit-exact with the oracle; cfg 10 stages whole programs."""
    rng = np.random.default_rng(7)
    lengths = [1, 2, 31, 32, 33, 63, 64, 65, 95, 96, 97, 127, 128, 129, 200]
    l, k = 5, 2 * max(lengths) + 2
    rows = [_chain_genome(n, l, rng) for n in lengths]
    tags = np.full((len(rows), k), R.CONSTANT, np.uint8)   # trailing constants: pushed, never the output
    codes = np.zeros((len(rows), k), np.int32)
    consts = np.ones((len(rows), k))
    for i, (t, c, v) in enumerate(rows):
        # the chain first, padded at the FRONT with constants that stay below
        # the chain on the stack (the output is the last fired function)
        off = k - len(t)
        tags[i, off:], codes[i, off:], consts[i, off:] = t, c, v
    X = rng.uniform(-2, 2, (700, l))
    pop = Population(tags, codes, consts)
    ref, _ = R.semantics(tags, codes, consts, X, 1e-6)
    monkeypatch.setenv("GSGP_INTERP_CFG", cfg)
    S = G.compute_semantics(pop, X, RunConfig(program_size=k))
    assert np.array_equal(S.view(np.uint64), ref.view(np.uint64))
