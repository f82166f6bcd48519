"""Operator API of the hot path, executed on the B200.

Each function has the reference's name, signature, argument meaning and
error behaviour (citations are to /root/reference/pkg/src/gsgp/) and runs its
sm_100a kernel through libgsgp_b200.so.  `backend` arguments are accepted for
signature compatibility and ignored: there is exactly one execution path.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check, ptr, u64
from .core import (
    Chromosome, ConfigError, Dataset, Gene, GeneTag, MutationPlan, Population, RunConfig,
    RunStats,
)

PLAN_STREAM_BASE = 1 << 32     # gsgp/rng.py:27
SPLIT_STREAM = 1 << 33         # gsgp/rng.py:28
HARNESS_STREAM = 1 << 34       # gsgp/harness.py:24


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def config_struct(cfg, *, storage: str = "fp32", use_graph: bool = True,
                  time_kernels: bool = False, virtual_shards: int = 1,
                  window_start: int = 0) -> _lib.GsgpConfig:
    """RunConfig (ours or the reference's: duck-typed) -> gsgp_config."""
    s = _lib.GsgpConfig()
    s.population_size = cfg.population_size
    s.random_trees = cfg.random_trees
    s.program_size = cfg.program_size
    s.generations = cfg.generations
    s.seed = u64(cfg.seed)
    s.p_function, s.p_feature, s.p_constant = cfg.p_function, cfg.p_feature, cfg.p_constant
    s.erc_low, s.erc_high = cfg.erc_low, cfg.erc_high
    uniform = isinstance(cfg.mutation_step, str)
    s.mutation_step_uniform = 1 if uniform else 0
    s.mutation_step = 0.0 if uniform else float(cfg.mutation_step)
    s.gsm_sign = 0 if cfg.gsm_sign == "minus" else 1
    s.division_eps = cfg.division_eps
    if storage not in ("fp32", "fp64"):
        raise ConfigError("storage must be 'fp32' or 'fp64'")
    s.storage_f64 = 1 if storage == "fp64" else 0
    s.use_graph = 1 if use_graph else 0
    s.time_kernels = 1 if time_kernels else 0
    s.virtual_shards = int(virtual_shards)
    s.window_start = int(window_start)
    return s


# ------------------------------------------------------------------ rng.py
def rng_bits(seed: int, stream: int, counter: int) -> int:
    """gsgp/rng.py:43-45 on the device."""
    c = np.array([u64(counter)], np.uint64)
    b = np.empty(1, np.uint64)
    check(_lib.load().gsgp_rng_draw(u64(seed), u64(stream), ptr(c), 1, ptr(b), None))
    return int(b[0])


def rng_stream(seed: int, stream: int, counter: int) -> float:
    """gsgp/rng.py:48-50 on the device."""
    return float(uniform_array(seed, stream, np.array([u64(counter)], np.uint64))[0])


def uniform_array(seed: int, stream: int, counters: np.ndarray) -> np.ndarray:
    """gsgp/rng.py:53-64: U[0,1) for every counter (uint64 wrap semantics)."""
    c = np.ascontiguousarray(np.asarray(counters).astype(np.uint64))
    out = np.empty(c.shape, np.float64)
    check(_lib.load().gsgp_rng_draw(u64(seed), u64(stream), ptr(c.reshape(-1)), c.size, None,
                                    ptr(out.reshape(-1))))
    return out


def release_device_memory() -> None:
    """Hand the engine's cached device memory back to the driver (a run parks
    its device blocks for the next run instead of freeing them)."""
    check(_lib.load().gsgp_trim_device_memory())


def derive_seed(seed: int, index: int) -> int:
    """gsgp/rng.py:67-69."""
    return int(_lib.load().gsgp_derive_seed(u64(seed), u64(index)))


# ------------------------------------------------------------ population.py
def create_population(count: int, cfg: RunConfig, stream_base: int, n_features: int,
                      backend=None) -> Population:
    """gsgp/population.py:73-92: individual i draws from stream stream_base + i."""
    if count < 1:
        raise ConfigError("population count must be >= 1")
    if n_features < 1:
        raise ConfigError("n_features must be >= 1")
    k = cfg.program_size
    tags = np.empty((count, k), np.uint8)
    codes = np.empty((count, k), np.int32)
    consts = np.empty((count, k), np.float64)
    s = config_struct(cfg)
    check(_lib.load().gsgp_create_population(C.byref(s), count, u64(stream_base), n_features,
                                             ptr(tags), ptr(codes), ptr(consts)))
    return Population(tags, codes, consts)


def sample_gene(cfg: RunConfig, stream: int, position: int, n_features: int) -> Gene:
    """gsgp/population.py:27-44: the gene at one genome position (a gene
    depends only on (seed, stream, position), so a 1-row device draw of
    length position+1 yields it)."""
    if n_features < 1:
        raise ConfigError("n_features must be >= 1")
    p = create_population(1, RunConfig(**{**_cfg_dict(cfg), "program_size": position + 1}),
                          stream, n_features)
    return Gene(GeneTag(int(p.tags[0, position])), int(p.codes[0, position]),
                float(p.consts[0, position]))


def _cfg_dict(cfg) -> dict:
    keys = ("population_size", "random_trees", "program_size", "generations", "runs", "seed",
            "p_function", "p_feature", "p_constant", "erc_low", "erc_high", "mutation_step",
            "division_eps", "gsm_sign")
    d = {k: getattr(cfg, k) for k in keys}
    d["backend"] = "cuda"
    return d


# ----------------------------------------------------------- interpreter.py
def compute_semantics(pop: Population, data, cfg: RunConfig, backend=None,
                      stats: RunStats | None = None) -> np.ndarray:
    """gsgp/interpreter.py:122-148: fp64 semantics [count][n]; non-finite
    outputs become 0.0 and are counted into `stats`."""
    X = data.features if isinstance(data, Dataset) else _f64(data)
    if X.ndim != 2:
        raise ConfigError("features must be a 2-D matrix")
    if len(pop) == 0 or X.shape[0] == 0:
        raise ConfigError("compute_semantics needs a nonempty population and dataset")
    feat = pop.codes[pop.tags == GeneTag.FEATURE]
    if feat.size and int(feat.max()) >= X.shape[1]:
        raise ConfigError("genome references a feature beyond the dataset width")
    tags = np.ascontiguousarray(pop.tags, np.uint8)
    codes = np.ascontiguousarray(pop.codes, np.int32)
    consts = _f64(pop.consts)
    X = _f64(X)
    out = np.empty((len(pop), X.shape[0]), np.float64)
    ovf = C.c_int64(0)
    check(_lib.load().gsgp_compute_semantics(ptr(tags), ptr(codes), ptr(consts), len(pop),
                                             pop.genome_length, ptr(X), X.shape[0], X.shape[1],
                                             float(cfg.division_eps), 1, ptr(out), C.byref(ovf)))
    if stats is not None:
        stats.overflow_replacements += int(ovf.value)
    return out


def interpret(chromosome: Chromosome, case_features, eps: float) -> float:
    """gsgp/interpreter.py:45-75: one genome on one fitness case (device)."""
    pop = Population(chromosome.tags[None, :].astype(np.uint8), chromosome.codes[None, :].astype(np.int32),
                     chromosome.consts[None, :].astype(np.float64))
    x = _f64(case_features).reshape(1, -1)
    if x.shape[1] == 0:
        x = np.zeros((1, 1))
    out = np.empty((1, 1), np.float64)
    ovf = C.c_int64(0)
    feat = pop.codes[pop.tags == GeneTag.FEATURE]
    if feat.size and int(feat.max()) >= x.shape[1]:
        raise ConfigError("genome references a feature beyond the case width")
    # raw value: the scalar reference does not replace non-finite results
    check(_lib.load().gsgp_compute_semantics(ptr(pop.tags), ptr(pop.codes), ptr(pop.consts), 1,
                                             pop.genome_length, ptr(x), 1, x.shape[1], float(eps),
                                             0, ptr(out), C.byref(ovf)))
    return float(out[0, 0])


# ---------------------------------------------------------------- fitness.py
def compute_fitness(semantics: np.ndarray, target, backend=None) -> np.ndarray:
    """gsgp/fitness.py:28-51: per-row RMSE, non-finite -> +inf.

    Bitwise the reference's value: the device kernel adds each row's squared
    differences strictly left to right, the order of the reference's
    np.cumsum.  (The engine's in-loop fitness differs from this operator in
    the last bits: it is the canonical tile sum of DESIGN.md §4, which is
    independent of how the cases are split across tiles and GPUs.)"""
    S = _f64(semantics)
    y = _f64(target)
    if S.ndim != 2 or S.shape[1] != y.shape[0]:
        raise ConfigError(f"semantics columns ({S.shape}) must match target length ({y.shape[0]})")
    out = np.empty(S.shape[0], np.float64)
    check(_lib.load().gsgp_compute_fitness(ptr(S), ptr(y), S.shape[0], S.shape[1], ptr(out)))
    return out


def rmse(row, target) -> float:
    """gsgp/fitness.py:11-25 (bitwise; see compute_fitness)."""
    a = _f64(row)
    b = _f64(target)
    if a.shape != b.shape or a.ndim != 1 or a.shape[0] == 0:
        raise ConfigError("rmse needs two equal-length nonempty vectors")
    return float(compute_fitness(a.reshape(1, -1), b)[0])


# --------------------------------------------------------------- mutation.py
def sigmoid_array(x: np.ndarray) -> np.ndarray:
    """gsgp/mutation.py:32-34 (fp64 on the device)."""
    a = _f64(x)
    out = np.empty_like(a)
    check(_lib.load().gsgp_sigmoid(ptr(a.reshape(-1)), a.size, ptr(out.reshape(-1))))
    return out


def canonical_sum(x: np.ndarray, parts: int = 0) -> np.ndarray:
    """Row sums of non-negative fp64 values with the engine's canonical SSE
    reduction (csrc/common.cuh): exact fixed-point digit sums anchored on the
    row's largest exponent, rounded once — independent of the order and
    grouping of the values.  `parts` > 0 runs the multi-shard path over that
    many column pieces (same bits as the fused path by construction)."""
    a = np.ascontiguousarray(np.atleast_2d(np.asarray(x, dtype=np.float64)))
    if a.size == 0:
        raise ConfigError("canonical_sum needs a non-empty matrix")
    out = np.empty(a.shape[0])
    check(_lib.load().gsgp_canonical_sum(ptr(a.reshape(-1)), a.shape[0], a.shape[1], int(parts), ptr(out)))
    return out


def sigmoid(x: float) -> float:
    """gsgp/mutation.py:26-29."""
    return float(sigmoid_array(np.array([float(x)]))[0])


def build_mutation_plan(m: int, r: int, cfg: RunConfig, generation: int) -> MutationPlan:
    """gsgp/mutation.py:37-62: stream 2^32+generation, counters 3i..3i+2."""
    if r < 2:
        raise ConfigError("geometric semantic mutation needs at least 2 random trees")
    if m < 1:
        raise ConfigError("plan length must be >= 1")
    u = np.empty(m, np.int64)
    v = np.empty(m, np.int64)
    ms = np.empty(m, np.float64)
    uniform = isinstance(cfg.mutation_step, str)
    check(_lib.load().gsgp_build_mutation_plan(m, r, u64(cfg.seed), generation, 1 if uniform else 0,
                                               0.0 if uniform else float(cfg.mutation_step),
                                               ptr(u), ptr(v), ptr(ms)))
    return MutationPlan(u, v, ms)


def _gsm_squashed(parent, squashed_trees, plan: MutationPlan, sign: str, backend=None,
                  stats: RunStats | None = None, *, squashed: bool = True) -> np.ndarray:
    """gsgp/mutation.py:65-86 (fp64, the reference's rounding order)."""
    P = _f64(parent)
    T = _f64(squashed_trees)
    if P.ndim != 2 or T.ndim != 2 or P.shape[1] != T.shape[1]:
        raise ConfigError("parent and random-tree matrices must share the case axis")
    if len(plan) != P.shape[0]:
        raise ConfigError("plan length must equal the population size")
    plan.validate(T.shape[0])
    u = np.ascontiguousarray(plan.u, np.int64)
    v = np.ascontiguousarray(plan.v, np.int64)
    ms = _f64(plan.ms)
    out = np.empty_like(P)
    ovf = C.c_int64(0)
    check(_lib.load().gsgp_gsm(ptr(P), P.shape[0], P.shape[1], ptr(T), T.shape[0], ptr(u), ptr(v),
                               ptr(ms), 0 if sign == "minus" else 1, 1 if squashed else 0, ptr(out),
                               C.byref(ovf)))
    if stats is not None:
        stats.overflow_replacements += int(ovf.value)
    return out


def gsm(parent_semantics, tree_semantics, plan: MutationPlan, cfg: RunConfig, backend=None,
        stats: RunStats | None = None) -> np.ndarray:
    """gsgp/mutation.py:89-94: sigmoid of the raw trees fused on the device."""
    return _gsm_squashed(parent_semantics, tree_semantics, plan, cfg.gsm_sign, backend, stats,
                         squashed=False)


def gsm_paired(parent_train, parent_test, tree_train, tree_test, plan: MutationPlan,
               cfg: RunConfig, backend=None, stats: RunStats | None = None):
    """gsgp/mutation.py:97-115: one plan on the train and test sides."""
    if np.shape(parent_train)[0] != np.shape(parent_test)[0]:
        raise ConfigError("train and test parent matrices must have equal row counts")
    if np.shape(tree_train)[0] != np.shape(tree_test)[0]:
        raise ConfigError("train and test tree matrices must have equal row counts")
    return (gsm(parent_train, tree_train, plan, cfg, backend, stats),
            gsm(parent_test, tree_test, plan, cfg, backend, stats))


def gsm_step_f32(parent_tr, parent_te, sq_tr, sq_te, ytr, yte, plan: MutationPlan,
                 sign: str = "minus"):
    """The engine's fused fp32 generation kernel on explicit inputs: returns
    (offspring_train f32, offspring_test f32, sse_train f64, sse_test f64)."""
    Ptr = np.ascontiguousarray(parent_tr, np.float32)
    Pte = np.ascontiguousarray(parent_te, np.float32)
    Qtr = np.ascontiguousarray(sq_tr, np.float32)
    Qte = np.ascontiguousarray(sq_te, np.float32)
    m, ntr = Ptr.shape
    nte = Pte.shape[1]
    r = Qtr.shape[0]
    plan.validate(r)
    otr = np.empty_like(Ptr)
    ote = np.empty_like(Pte)
    s_tr = np.empty(m)
    s_te = np.empty(m)
    u = np.ascontiguousarray(plan.u, np.int64)
    v = np.ascontiguousarray(plan.v, np.int64)
    ms = _f64(plan.ms)
    check(_lib.load().gsgp_gsm_step_f32(ptr(Ptr), ptr(Pte), ptr(Qtr), ptr(Qte), m, r, ntr, nte,
                                        ptr(_f64(ytr)), ptr(_f64(yte)), ptr(u), ptr(v), ptr(ms),
                                        0 if sign == "minus" else 1, ptr(otr), ptr(ote), ptr(s_tr),
                                        ptr(s_te)))
    return otr, ote, s_tr, s_te


# -------------------------------------------------------------- evolution.py
def argmin_fitness(fitness: np.ndarray) -> int:
    """gsgp/evolution.py:36-40: lowest index among the minima."""
    return _argminmax(fitness)[0]


def argmax_fitness(fitness: np.ndarray) -> int:
    """gsgp/evolution.py:43-47: lowest index among the maxima."""
    return _argminmax(fitness)[1]


def _argminmax(fitness) -> tuple[int, int]:
    f = _f64(fitness)
    if f.shape[0] == 0:
        raise ConfigError("empty fitness vector")
    out = np.empty(2, np.int64)
    check(_lib.load().gsgp_argminmax(ptr(f), f.shape[0], ptr(out)))
    return int(out[0]), int(out[1])


def survive_decision(fit_parent, fit_offspring) -> tuple[str, int, int]:
    """gsgp/evolution.py:73-82 decision on the device: (source, index, slot)."""
    a, b = _f64(fit_parent), _f64(fit_offspring)
    if a.shape != b.shape or a.shape[0] == 0:
        raise ConfigError("parent and offspring states must have equal shapes")
    dec = np.empty(3, np.int64)
    check(_lib.load().gsgp_survive(ptr(a), ptr(b), a.shape[0], ptr(dec)))
    return ("parent" if dec[0] == 0 else "offspring"), int(dec[1]), int(dec[2])
