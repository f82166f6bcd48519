"""Generate golden vectors by importing the REAL reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports `gsgp` from /root/reference/pkg/src (read-only, never modified)
and writes small .npz fixtures next to this file.  The GPU box never needs
the reference: tests load only the committed .npz files.
"""

from __future__ import annotations

import random
import sys
import time
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF_SRC))

import gsgp  # noqa: E402
from gsgp import (  # noqa: E402
    Chromosome, Gene, GeneTag, FunctionOp, MutationPlan, Population, RunConfig, RunStats,
    build_mutation_plan, compute_fitness, compute_semantics, create_population, gsm,
    make_benchmark_dataset, run_evolution, survive,
)
from gsgp.evolution import GenerationState  # noqa: E402
from gsgp import rng as ref_rng  # noqa: E402

OUT = Path(__file__).resolve().parent


def toy_dataset(n_cases=24, n_features=3, seed=0):
    """Same construction as the reference test fixture (pkg/tests/conftest.py:22-30)."""
    r = np.random.default_rng(seed)
    X = r.uniform(-2.0, 2.0, size=(n_cases, n_features))
    y = X[:, 0] * X[:, 1] - X[:, 2 % n_features] + 0.5
    return gsgp.Dataset(X, y)


def random_genes(pyrng, length, n_features, lo=-2.0, hi=2.0):
    """Same generator as pkg/tests/oracles.py:18-30."""
    genes = []
    for _ in range(length):
        roll = pyrng.random()
        if roll < 0.5:
            genes.append(Gene(GeneTag.FUNCTION, pyrng.randrange(4)))
        elif roll < 0.8:
            genes.append(Gene(GeneTag.FEATURE, pyrng.randrange(n_features)))
        else:
            genes.append(Gene(GeneTag.CONSTANT, 0, pyrng.uniform(lo, hi)))
    return genes


def gen_rng():
    coords = [(1, 0, 0), (1, 0, 1), (1, 5, 7), (424242, 2**32 + 1, 0), (-3, 0, 0),
              (2**64 - 1, 2**63 + 5, 2**63 - 1), (12345, 7, 999999), (0, 0, 0),
              (3140439631417119954, 2**34, 17)]
    seeds = np.array([c[0] & (2**64 - 1) for c in coords], np.uint64)
    streams = np.array([c[1] & (2**64 - 1) for c in coords], np.uint64)
    counters = np.array([c[2] & (2**64 - 1) for c in coords], np.uint64)
    bits = np.array([ref_rng.rng_bits(*c) for c in coords], np.uint64)
    units = np.array([ref_rng.rng_stream(*c) for c in coords])
    derive = np.array([[s, i, ref_rng.derive_seed(s, i)] for s in (1, 42, 33_000)
                       for i in range(4)], np.uint64)
    vec = ref_rng.uniform_array(9, 3, np.arange(4096))
    np.savez_compressed(OUT / "rng.npz", seeds=seeds, streams=streams, counters=counters,
                        bits=bits, units=units, derive=derive, vec_seed9_stream3=vec)


POP_CASES = [
    # (count, k, l, seed, stream_base, overrides)
    (2, 8, 3, 3, 0, {}),
    (6, 64, 4, 3, 17, {}),
    (16, 127, 8, 1, 0, {}),
    (8, 255, 100, 7, 1000, {}),
    (4, 1024, 5, 1, 256, {}),
    (3, 50, 2, 11, 0, dict(p_function=1.0, p_feature=0.0, p_constant=0.0)),
    (2, 500, 2, 11, 0, dict(p_function=0.0, p_feature=0.0, p_constant=1.0)),
    (5, 40, 3, 2**63 + 9, 3, dict(p_function=2.0, p_feature=1.0, p_constant=1.0,
                                  erc_low=-5.0, erc_high=5.0)),
]


def gen_population():
    blobs = {}
    for n, (count, k, l, seed, base, ov) in enumerate(POP_CASES):
        cfg = RunConfig(program_size=k, seed=seed, **ov)
        pop = create_population(count, cfg, base, l)
        blobs[f"tags{n}"] = pop.tags
        blobs[f"codes{n}"] = pop.codes
        blobs[f"consts{n}"] = pop.consts
    meta = []
    for count, k, l, seed, base, ov in POP_CASES:
        p = (ov.get("p_function", 0.8), ov.get("p_feature", 0.14), ov.get("p_constant", 0.04))
        erc = (ov.get("erc_low", 1.0), ov.get("erc_high", 10.0))
        meta.append([count, k, l, seed & (2**64 - 1), base, *p, *erc])
    blobs["meta"] = np.array(meta, dtype=object)
    np.savez_compressed(OUT / "population.npz", **blobs, allow_pickle=True)


def gen_interpreter():
    blobs = {}
    # (a) random gene lists from the reference's oracle generator, k <= 15, l = 2
    pyrng = random.Random(20260810)
    cases = np.array([[pyrng.uniform(-5, 5), pyrng.uniform(-5, 5)] for _ in range(20)])
    tags, codes, consts = [], [], []
    K = 15
    for _ in range(300):
        genes = random_genes(pyrng, pyrng.randint(1, K), n_features=2)
        # pad with skipped-function-free filler? no: store true length separately
        t = np.full(K, 255, np.uint8)
        c = np.zeros(K, np.int32)
        v = np.zeros(K)
        for j, gene in enumerate(genes):
            t[j], c[j], v[j] = int(gene.tag), gene.code, gene.value
        tags.append(t); codes.append(c); consts.append(v)
    tags, codes, consts = np.array(tags), np.array(codes), np.array(consts)
    lens = (tags != 255).sum(axis=1)
    outs = np.zeros((len(tags), len(cases)))
    for i in range(len(tags)):
        pop = Population(tags[i:i + 1, :lens[i]].copy(), codes[i:i + 1, :lens[i]].copy(),
                         consts[i:i + 1, :lens[i]].copy())
        outs[i] = compute_semantics(pop, cases, RunConfig(program_size=int(lens[i])))[0]
    blobs.update(rand_tags=tags, rand_codes=codes, rand_consts=consts, rand_lens=lens,
                 rand_cases=cases, rand_out=outs)
    # (b) engine-sampled genomes (the real distribution) on toy and benchmark data
    for name, (m, k, l, seed, n) in {
        "toy": (20, 31, 3, 5, 13),
        "k127": (64, 127, 8, 1, 300),
        "k1024": (48, 1024, 5, 1, 200),
        "k255_l100": (16, 255, 100, 3, 64),
    }.items():
        cfg = RunConfig(program_size=k, seed=seed)
        pop = create_population(m, cfg, 0, l)
        if name == "toy":
            ds = toy_dataset(n, l, seed=5)
            X = ds.features
        else:
            X = make_benchmark_dataset(n, l, seed=seed).features
        stats = RunStats()
        S = compute_semantics(pop, X, cfg, stats=stats)
        blobs[f"{name}_tags"], blobs[f"{name}_codes"], blobs[f"{name}_consts"] = \
            pop.tags, pop.codes, pop.consts
        blobs[f"{name}_X"], blobs[f"{name}_S"] = X, S
        blobs[f"{name}_overflow"] = np.array(stats.overflow_replacements)
    # (c) overflow KAT (pkg/tests/test_interpreter.py:164-176)
    big = 1e200
    pop = Population.from_chromosomes([
        Chromosome.from_genes([Gene(GeneTag.CONSTANT, 0, big), Gene(GeneTag.CONSTANT, 0, big),
                               Gene(GeneTag.FUNCTION, FunctionOp.MUL)]),
        Chromosome.from_genes([Gene(GeneTag.CONSTANT, 0, 1.0), Gene(GeneTag.CONSTANT, 0, 1.0),
                               Gene(GeneTag.FUNCTION, FunctionOp.ADD)]),
    ])
    stats = RunStats()
    X = toy_dataset(5).features
    blobs["ovf_S"] = compute_semantics(pop, X, RunConfig(program_size=3), stats=stats)
    blobs["ovf_count"] = np.array(stats.overflow_replacements)
    blobs["ovf_tags"], blobs["ovf_codes"], blobs["ovf_consts"] = pop.tags, pop.codes, pop.consts
    blobs["ovf_X"] = X
    np.savez_compressed(OUT / "interpreter.npz", **blobs)


def gen_ops():
    blobs = {}
    r = np.random.default_rng(4)
    S = r.normal(size=(64, 333)) * 3
    y = r.normal(size=333)
    S[5] = y
    S[7, 3] = 1e200
    blobs.update(fit_S=S, fit_y=y, fit_out=compute_fitness(S, y))
    plans = []
    for (m, rr, seed, gen, step) in [(6, 8, 21, 1, "uniform"), (200, 2, 21, 1, "uniform"),
                                     (1024, 1024, 1, 1, "uniform"), (1024, 1024, 1, 500, "uniform"),
                                     (257, 13, 2**64 - 5, 77, "uniform"), (16, 8, 21, 2, 0.3),
                                     (8192, 1024, 424242, 9, "uniform")]:
        cfg = RunConfig(seed=seed, mutation_step=step)
        p = build_mutation_plan(m, rr, cfg, gen)
        plans.append((m, rr, seed, gen, step))
        key = f"plan_{m}_{rr}_{gen}_{seed % 1000}_{step}"
        blobs[key + "_u"], blobs[key + "_v"], blobs[key + "_ms"] = p.u, p.v, p.ms
    blobs["plan_meta"] = np.array(plans, dtype=object)
    # GSM on random matrices, both signs
    for sign in ("minus", "plus"):
        rg = np.random.default_rng(617 if sign == "minus" else 618)
        m, n, rr = 37, 29, 11
        P = rg.normal(size=(m, n)) * 40.0
        T = rg.normal(size=(rr, n)) * 10.0
        u = rg.integers(0, rr, size=m)
        v = (u + 1 + rg.integers(0, rr - 1, size=m)) % rr
        ms = rg.uniform(0.0, 1.0, size=m) + 1e-9
        out = gsm(P, T, MutationPlan(u, v, ms), RunConfig(gsm_sign=sign))
        blobs.update({f"gsm_{sign}_P": P, f"gsm_{sign}_T": T, f"gsm_{sign}_u": u,
                      f"gsm_{sign}_v": v, f"gsm_{sign}_ms": ms, f"gsm_{sign}_out": out})
    # survival decisions
    rs = np.random.default_rng(8)
    fp, fo, dec = [], [], []
    for i in range(200):
        m = 9
        a = rs.uniform(0, 2, size=m)
        b = rs.uniform(0, 2, size=m)
        if i % 5 == 0:
            b[rs.integers(0, m)] = a.min()      # exact tie -> offspring kept
        if i % 7 == 0:
            b[rs.integers(0, m, size=3)] = np.inf
        if i % 11 == 0:
            b[:] = b.max()                       # all-equal offspring
        fp.append(a); fo.append(b)
        st_p = GenerationState(np.zeros((m, 1)), a.copy(), np.zeros((m, 1)))
        st_o = GenerationState(np.zeros((m, 1)), b.copy(), np.zeros((m, 1)))
        _, e = survive(st_p, st_o)
        dec.append([0 if e.source == "parent" else 1, e.index, e.slot])
    blobs.update(surv_par=np.array(fp), surv_off=np.array(fo), surv_dec=np.array(dec))
    # synthetic benchmark data
    X, yv = make_benchmark_dataset(3, 5, seed=1).features, make_benchmark_dataset(3, 5, seed=1).target
    blobs.update(bench_X=X, bench_y=yv)
    ds = make_benchmark_dataset(1000, 8, seed=6)
    blobs.update(bench1000_X=ds.features, bench1000_y=ds.target)
    np.savez_compressed(OUT / "ops.npz", **blobs, allow_pickle=True)


RUNS = {
    # name: (cfg kwargs, train (n, l, seed), test (n, seed), data kind)
    "tiny": (dict(population_size=4, random_trees=4, program_size=9, generations=5, seed=31),
             (3, 2, 11), (3, 12), "toy"),
    "small": (dict(population_size=12, random_trees=12, program_size=21, generations=20, seed=5),
              (30, 3, 1), (10, 2), "toy"),
    "plus": (dict(population_size=16, random_trees=8, program_size=31, generations=30, seed=77,
                  gsm_sign="plus", mutation_step=0.25), (40, 3, 3), (12, 4), "toy"),
    "accept": (dict(population_size=256, random_trees=256, program_size=127, generations=50,
                    seed=424242), (1000, 8, 6), (250, 7), "bench"),
    "c1": (dict(population_size=256, random_trees=1024, program_size=1024, generations=50, seed=1),
           (500, 5, 1), (200, 2), "bench"),
    "c2s": (dict(population_size=1024, random_trees=1024, program_size=1024, generations=40, seed=1),
            (4000, 8, 1), (1000, 2), "bench"),
    "g0": (dict(population_size=12, random_trees=12, program_size=21, generations=0, seed=5),
           (30, 3, 1), (10, 2), "toy"),
    # edge cases: single individual, k=1, one fitness case, degenerate gene mixes
    "m1": (dict(population_size=1, random_trees=2, program_size=7, generations=10, seed=3),
           (5, 2, 3), (3, 4), "toy"),
    "k1": (dict(population_size=5, random_trees=3, program_size=1, generations=8, seed=8),
           (9, 2, 5), (4, 6), "toy"),
    "n1": (dict(population_size=6, random_trees=4, program_size=15, generations=10, seed=9),
           (1, 3, 7), (1, 8), "toy"),
    "const": (dict(population_size=8, random_trees=4, program_size=5, generations=10, seed=10,
                   p_function=0.0, p_feature=0.0, p_constant=1.0), (12, 2, 9), (5, 10), "toy"),
    "funcs": (dict(population_size=6, random_trees=3, program_size=9, generations=6, seed=11,
                   p_function=1.0, p_feature=0.0, p_constant=0.0), (10, 2, 11), (4, 12), "toy"),
    # 5 initial rows exceed FLT_MAX: exercises the engine's fp32-overflow slots
    "wide": (dict(population_size=1024, random_trees=64, program_size=1024, generations=40, seed=2),
             (300, 5, 1), (100, 2), "bench"),
    # constant steps past fp32 range (gsgp/core.py:332-336 accepts any finite
    # positive step): the reference stays finite in fp64 where an fp32 store
    # would overflow; the engine must not take the fp32 path for these
    "hugestep": (dict(population_size=16, random_trees=8, program_size=31, generations=20, seed=41,
                      mutation_step=1e38, gsm_sign="plus"), (40, 3, 13), (12, 14), "toy"),
    "infstep": (dict(population_size=12, random_trees=6, program_size=21, generations=8, seed=43,
                     mutation_step=1e39, gsm_sign="plus"), (30, 3, 15), (10, 16), "toy"),
}


def gen_runs(names=None):
    for name, (kw, (ntr, l, s1), (nte, s2), kind) in RUNS.items():
        if names and name not in names:
            continue
        cfg = RunConfig(backend="sequential", **kw)
        if kind == "toy":
            tr, te = toy_dataset(ntr, l, seed=s1), toy_dataset(nte, l, seed=s2)
        else:
            tr, te = make_benchmark_dataset(ntr, l, seed=s1), make_benchmark_dataset(nte, l, seed=s2)
        t0 = time.perf_counter()
        res = run_evolution(cfg, tr, te)
        dt = time.perf_counter() - t0
        log = res.lineage
        src = np.array([0 if e.elite.source == "parent" else 1 for e in log.entries], np.int8)
        idx = np.array([e.elite.index for e in log.entries], np.int64)
        slot = np.array([e.elite.slot for e in log.entries], np.int64)
        fit = np.array([e.elite.fitness for e in log.entries])
        blobs = dict(Xtr=tr.features, ytr=tr.target, Xte=te.features, yte=te.target,
                     train=res.train_fitness, test=res.test_fitness, src=src, idx=idx,
                     slot=slot, fit=fit, init=np.array([log.initial_elite.index]),
                     init_fit=np.array([log.initial_elite.fitness]),
                     elite_sem=res.elite_train_semantics, slot_final=np.array([res.elite_slot]),
                     overflow=np.array([res.overflow_replacements]),
                     cfg=np.array([repr(kw)]))
        if 0 < cfg.population_size * cfg.generations <= 20000:
            blobs["u"] = np.array([e.plan.u for e in log.entries]).reshape(cfg.generations, -1)
            blobs["v"] = np.array([e.plan.v for e in log.entries]).reshape(cfg.generations, -1)
            blobs["ms"] = np.array([e.plan.ms for e in log.entries]).reshape(cfg.generations, -1)
        np.savez_compressed(OUT / f"run_{name}.npz", **blobs)
        print(f"run {name}: {dt:.1f}s, parent elites {int((src == 0).sum())}/{len(src)}")


# Headline-shape runs (VERDICT r01 "Missing" #1): the shapes whose generation
# kernel and SSE reduction configurations the benchmarks run.  Units per row
# (4096-case fp32 tiles): c2 = 31 (C2 itself), mid = 123 (33..1024: the
# warp-per-row reduce), long = 1124 (> 1024: the block-per-row reduce of C3).
# The data is NOT stored: tests regenerate it with make_benchmark_dataset
# (bit-exact with the reference, pinned by ops.npz bench_* vectors).  Stored:
# traces, elite records, plans (uint16) and a strided sample (~20k values) of
# the final elite's train semantics.
BIG_RUNS = {
    "c2": (dict(population_size=1024, random_trees=1024, program_size=1024, generations=5, seed=1),
           (100_000, 8, 1), (25_000, 2)),
    "mid": (dict(population_size=64, random_trees=32, program_size=63, generations=4, seed=17),
            (400_000, 6, 3), (100_000, 4)),
    "long": (dict(population_size=8, random_trees=8, program_size=31, generations=3, seed=23),
             (4_300_000, 4, 5), (300_000, 6)),
}


def gen_big_runs(names=None):
    for name, (kw, (ntr, l, s1), (nte, s2)) in BIG_RUNS.items():
        if names and name not in names:
            continue
        cfg = RunConfig(backend="threads", **kw)
        tr, te = make_benchmark_dataset(ntr, l, seed=s1), make_benchmark_dataset(nte, l, seed=s2)
        t0 = time.perf_counter()
        res = run_evolution(cfg, tr, te)
        dt = time.perf_counter() - t0
        log = res.lineage
        blobs = dict(
            train=res.train_fitness, test=res.test_fitness,
            src=np.array([0 if e.elite.source == "parent" else 1 for e in log.entries], np.int8),
            idx=np.array([e.elite.index for e in log.entries], np.int64),
            slot=np.array([e.elite.slot for e in log.entries], np.int64),
            fit=np.array([e.elite.fitness for e in log.entries]),
            init=np.array([log.initial_elite.index]), init_fit=np.array([log.initial_elite.fitness]),
            u=np.array([e.plan.u for e in log.entries], np.uint16),
            v=np.array([e.plan.v for e in log.entries], np.uint16),
            ms=np.array([e.plan.ms for e in log.entries]),
            elite_sem_sample=res.elite_train_semantics[::max(7, ntr // 20000)].copy(),
            sample_stride=np.array([max(7, ntr // 20000)]),
            slot_final=np.array([res.elite_slot]), overflow=np.array([res.overflow_replacements]),
            data=np.array([ntr, l, s1, nte, s2], np.int64), cfg=np.array([repr(kw)]))
        np.savez_compressed(OUT / f"big_{name}.npz", **blobs)
        print(f"big run {name}: {dt:.1f}s, parent elites {int((blobs['src'] == 0).sum())}/{len(log.entries)}")


def gen_cli():
    """The reference CLI's own files for a 2-run job (pkg/src/gsgp/io_cli.py)."""
    import shutil
    from gsgp import run_cli, write_dataset
    d = OUT / "cli_ref"
    if d.exists():
        shutil.rmtree(d)
    d.mkdir()
    write_dataset(d / "train.txt", make_benchmark_dataset(60, 3, seed=6))
    write_dataset(d / "test.txt", make_benchmark_dataset(20, 3, seed=7))
    (d / "config.ini").write_text(
        "# reference-format config\n[run]\npopulation_size = 24\nrandom_trees = 16\n"
        "program_size = 31\ngenerations = 12\nruns = 2\nseed = 4242\nmutation_step = uniform\n")
    out = d / "out"
    code = run_cli(["-train_file", str(d / "train.txt"), "-test_file", str(d / "test.txt"),
                    "-config", str(d / "config.ini"), "-output_dir", str(out), "-backend", "sequential"])
    assert code == 0
    (out / "timings.csv").unlink()   # wall-clock values: not a fixture


def gen_split():
    """Dataset.split (gsgp/core.py:179-192): rows of each side for several
    sizes, fractions and seeds (the row ids are stored as feature column 0)."""
    rows = {}
    for n, frac, seed in ((2, 0.5, 1), (10, 0.7, 3), (37, 0.25, 5), (1000, 0.8, -7), (513, 0.999, 2**40)):
        X = np.stack([np.arange(n, dtype=np.float64), np.ones(n)], axis=1)
        tr, te = gsgp.Dataset(X, np.arange(n, dtype=np.float64)).split(frac, seed)
        rows[f"tr_{n}"] = tr.features[:, 0].astype(np.int64)
        rows[f"te_{n}"] = te.features[:, 0].astype(np.int64)
        rows[f"args_{n}"] = np.array([frac, seed], dtype=object)
    np.savez_compressed(OUT / "split.npz", **rows)


if __name__ == "__main__":
    if sys.argv[1:2] == ["big"]:          # python make_golden.py big [names...]
        gen_big_runs(sys.argv[2:])
        sys.exit(0)
    if sys.argv[1:2] == ["runs"]:         # python make_golden.py runs [names...]
        gen_runs(sys.argv[2:])
        sys.exit(0)
    gen_split()
    gen_rng()
    gen_population()
    gen_interpreter()
    gen_ops()
    gen_runs()
    gen_cli()
    gen_big_runs()
    print("golden fixtures written to", OUT)
