"""numpy restatement of the reference GSGP path (TEST INFRASTRUCTURE ONLY).

Every function cites the reference code it restates; `R:` below abbreviates
`/root/reference/pkg/src/gsgp/`.  The arithmetic is the same sequence of
IEEE-754 binary64 operations as the reference, so on the same inputs the
outputs are bitwise equal (checked by tests/test_oracle_golden.py against
fixtures generated from the reference itself).

Plain tuples/ndarrays are used instead of the reference's dataclasses so the
oracle has no dependency on either the reference or the product package.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

# ---------------------------------------------------------------- RNG (R:rng.py)
M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15          # R:rng.py:17  counter increment
STREAM_MULT = 0xC2B2AE3D27D4EB4F     # R:rng.py:18  stream decorrelation
MIX_A = 0xBF58476D1CE4E5B9           # R:rng.py:19
MIX_B = 0x94D049BB133111EB           # R:rng.py:20
SEED_XOR = 0x8538ECB5BD456EA3        # R:rng.py:21
PLAN_STREAM0 = 1 << 32               # R:rng.py:27
SPLIT_STREAM = 1 << 33               # R:rng.py:28
HARNESS_STREAM = 1 << 34             # R:harness.py:24
TWO_M53 = 1.0 / (1 << 53)            # R:rng.py:23


def finalize(z: int) -> int:
    """splitmix64 output function on a Python int (R:rng.py:31-36)."""
    z &= M64
    z = ((z ^ (z >> 30)) * MIX_A) & M64
    z = ((z ^ (z >> 27)) * MIX_B) & M64
    return z ^ (z >> 31)


def stream_key(seed: int, stream: int) -> int:
    """Per-(seed, stream) base state (R:rng.py:39-40)."""
    return finalize((finalize(seed ^ SEED_XOR) + (stream & M64) * STREAM_MULT) & M64)


def bits(seed: int, stream: int, counter: int) -> int:
    """64 random bits at (seed, stream, counter) (R:rng.py:43-45)."""
    return finalize((stream_key(seed, stream) + (counter & M64) * GOLDEN) & M64)


def unit(seed: int, stream: int, counter: int) -> float:
    """U[0,1) draw = top 53 bits * 2^-53 (R:rng.py:48-50)."""
    return (bits(seed, stream, counter) >> 11) * TWO_M53


def unit_vec(seed: int, stream: int, counters) -> np.ndarray:
    """Vectorised `unit` over an array of counters (R:rng.py:53-64)."""
    z = np.uint64(stream_key(seed, stream)) + np.asarray(counters).astype(np.uint64) * np.uint64(GOLDEN)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(MIX_A)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(MIX_B)
    z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * TWO_M53


def split_rows(n: int, train_fraction: float, seed: int):
    """Row indices of Dataset.split (R:core.py:179-192): stable argsort of the
    split-stream uniforms, first round(n*f) (clamped to [1, n-1]) rows train."""
    order = np.argsort(unit_vec(seed, SPLIT_STREAM, np.arange(n)), kind="stable")
    cut = max(1, min(n - 1, round(n * train_fraction)))
    return order[:cut], order[cut:]


def run_seed(seed: int, index: int) -> int:
    """Seed of sub-run `index` (R:rng.py:67-69)."""
    return finalize((finalize(seed ^ STREAM_MULT) + (index & M64) * GOLDEN) & M64)


# ------------------------------------------------------------ config helpers
def gene_thresholds(p_function: float, p_feature: float, p_constant: float):
    """Renormalised (p_fun, p_fun + p_feat) exactly as R:core.py:338-342 and
    the comparisons at R:population.py:54-56."""
    total = p_function + p_feature + p_constant
    pf = p_function / total
    px = p_feature / total
    return pf, pf + px


# -------------------------------------------------- CreatePopulation (R:population.py)
FUNCTION, FEATURE, CONSTANT = 0, 1, 2     # R:core.py:41-44
ADD, SUB, MUL, DIV = 0, 1, 2, 3           # R:core.py:47-51


def genomes(count: int, k: int, n_features: int, seed: int, stream_base: int,
            p_function=0.8, p_feature=0.14, p_constant=0.04,
            erc_low=1.0, erc_high=10.0):
    """Rows of (tags u8, codes i32, consts f64); gene (i, j) draws counters 2j
    (tag) and 2j+1 (payload) of stream stream_base+i (R:population.py:47-92)."""
    pf = p_function / (p_function + p_feature + p_constant)
    px = p_feature / (p_function + p_feature + p_constant)
    tags = np.empty((count, k), np.uint8)
    codes = np.zeros((count, k), np.int32)
    consts = np.zeros((count, k), np.float64)
    pos = np.arange(k, dtype=np.uint64)
    for i in range(count):
        d_tag = unit_vec(seed, stream_base + i, pos * np.uint64(2))
        d_pay = unit_vec(seed, stream_base + i, pos * np.uint64(2) + np.uint64(1))
        fun = d_tag < pf
        feat = ~fun & (d_tag < pf + px)
        const = ~fun & ~feat
        tags[i] = np.where(fun, FUNCTION, np.where(feat, FEATURE, CONSTANT))
        op = np.minimum((d_pay * 4).astype(np.int32), 3)
        fx = np.minimum((d_pay * n_features).astype(np.int32), n_features - 1)
        codes[i] = np.where(fun, op, np.where(feat, fx, 0))
        consts[i] = np.where(const, erc_low + d_pay * (erc_high - erc_low), 0.0)
    return tags, codes, consts


# ------------------------------------------------ ComputeSemantics (R:interpreter.py)
def interpret_one(tags, codes, consts, x, eps: float) -> float:
    """Scalar postfix scan of one genome on one case (R:interpreter.py:45-75):
    a function fires only when two operands are stacked, left = second pop,
    protected division -> 1.0, result = last fired value else top else 0."""
    stack: list[float] = []
    last = None
    for t, c, v in zip(tags.tolist(), codes.tolist(), consts.tolist()):
        if t == FUNCTION:
            if len(stack) < 2:
                continue
            b = stack.pop()
            a = stack.pop()
            if c == ADD:
                res = a + b
            elif c == SUB:
                res = a - b
            elif c == MUL:
                res = a * b
            else:
                res = 1.0 if abs(b) < eps else a / b
            stack.append(res)
            last = res
        elif t == FEATURE:
            stack.append(float(x[c]))
        else:
            stack.append(v)
    if last is not None:
        return last
    return stack[-1] if stack else 0.0


def interpret_row(tags, codes, consts, cols: np.ndarray, eps: float) -> np.ndarray:
    """One genome over all cases; `cols` is the (l, n) transposed feature
    matrix (R:interpreter.py:78-119).  Stack items are floats or case
    vectors; each fired gene is one elementwise fp64 op."""
    stack: list = []
    last = None
    cl = codes.tolist()
    vl = consts.tolist()
    for j, t in enumerate(tags.tolist()):
        if t == FUNCTION:
            if len(stack) < 2:
                continue
            b = stack.pop()
            a = stack.pop()
            c = cl[j]
            if c == ADD:
                res = a + b
            elif c == SUB:
                res = a - b
            elif c == MUL:
                res = a * b
            elif isinstance(b, float):
                res = 1.0 if abs(b) < eps else a / b
            else:
                res = np.where(np.abs(b) < eps, 1.0, a / b)
            stack.append(res)
            last = res
        elif t == FEATURE:
            stack.append(cols[cl[j]])
        else:
            stack.append(vl[j])
    out = last if last is not None else (stack[-1] if stack else 0.0)
    if isinstance(out, np.ndarray):
        return out
    return np.full(cols.shape[1], float(out))


def zero_nonfinite(a: np.ndarray) -> int:
    """In-place non-finite -> 0.0, returns the count (R:core.py:348-356)."""
    bad = ~np.isfinite(a)
    n = int(bad.sum())
    if n:
        a[bad] = 0.0
    return n


def semantics(tags, codes, consts, X: np.ndarray, eps: float, workers: int = 1):
    """Semantic matrix f64 (count x n) + non-finite count
    (R:interpreter.py:122-148)."""
    X = np.asarray(X, np.float64)
    if int(codes[tags == FEATURE].max(initial=-1)) >= X.shape[1]:
        raise ValueError("genome references a feature beyond the dataset width")
    cols = np.ascontiguousarray(X.T)
    out = np.empty((tags.shape[0], X.shape[0]), np.float64)

    def block(lo, hi):
        with np.errstate(all="ignore"):
            for i in range(lo, hi):
                out[i] = interpret_row(tags[i], codes[i], consts[i], cols, eps)

    row_blocks(tags.shape[0], block, workers)
    return out, zero_nonfinite(out)


# ------------------------------------------------------ ComputeFitness (R:fitness.py)
def rmse(row, target) -> float:
    """Left-to-right cumulative SSE, sqrt(SSE/n), non-finite -> +inf
    (R:fitness.py:11-25)."""
    with np.errstate(all="ignore"):
        d = np.asarray(row, np.float64) - np.asarray(target, np.float64)
        v = float(np.sqrt(np.cumsum(d * d)[-1] / d.shape[0]))
    return v if math.isfinite(v) else math.inf


def fitness(S: np.ndarray, target, workers: int = 1) -> np.ndarray:
    """Per-row RMSE (R:fitness.py:28-51)."""
    target = np.asarray(target, np.float64)
    n = S.shape[1]
    out = np.empty(S.shape[0])

    def block(lo, hi):
        with np.errstate(all="ignore"):
            d = S[lo:hi] - target
            v = np.sqrt(np.cumsum(d * d, axis=1)[:, -1] / n)
            out[lo:hi] = np.where(np.isfinite(v), v, math.inf)

    row_blocks(S.shape[0], block, workers)
    return out


# ------------------------------------------------------------- GSM (R:mutation.py)
def sigmoid(x: np.ndarray) -> np.ndarray:
    """1/(1+exp(-x)) in fp64 (R:mutation.py:32-34)."""
    with np.errstate(all="ignore"):
        return 1.0 / (1.0 + np.exp(-x))


def plan(m: int, r: int, seed: int, generation: int, mutation_step="uniform"):
    """(u, v, ms) for one generation: stream 2^32+gen, counters 3i..3i+2
    (R:mutation.py:37-62)."""
    if r < 2:
        raise ValueError("need at least 2 random trees")
    stream = PLAN_STREAM0 + generation
    base = np.arange(m, dtype=np.uint64) * np.uint64(3)
    du = unit_vec(seed, stream, base)
    dv = unit_vec(seed, stream, base + np.uint64(1))
    u = np.minimum((du * r).astype(np.int64), r - 1)
    v = np.minimum((dv * (r - 1)).astype(np.int64), r - 2)
    v = v + (v >= u)
    if mutation_step == "uniform":
        ms = 1.0 - unit_vec(seed, stream, base + np.uint64(2))
    else:
        ms = np.full(m, float(mutation_step))
    return u, v, ms


def gsm_squashed(parent, sq, u, v, ms, sign="minus", workers: int = 1):
    """offspring = parent + ms*(sq[u] -/+ sq[v]) with the reference's op order
    t=a-b; t*=ms; out=parent+t, then non-finite -> 0 (R:mutation.py:65-86).
    Returns (offspring, n_replaced)."""
    out = np.empty_like(parent)

    def block(lo, hi):
        with np.errstate(all="ignore"):
            a = sq[u[lo:hi]]
            b = sq[v[lo:hi]]
            t = a - b if sign == "minus" else a + b
            np.multiply(t, ms[lo:hi, None], out=t)
            np.add(parent[lo:hi], t, out=out[lo:hi])

    row_blocks(parent.shape[0], block, workers)
    return out, zero_nonfinite(out)


# --------------------------------------------------------- survival (R:evolution.py)
def survive(fit_par, fit_off):
    """Elitist replacement decision (R:evolution.py:65-83): returns
    (source, index, slot) with np.argmin/np.argmax lowest-index ties and a
    strict '<'."""
    bp = int(np.argmin(fit_par))
    bo = int(np.argmin(fit_off))
    if fit_par[bp] < fit_off[bo]:
        return "parent", bp, int(np.argmax(fit_off))
    return "offspring", bo, bo


# ------------------------------------------------------------- backend
def row_blocks(count: int, fn, workers: int = 1) -> None:
    """Even contiguous row chunks over a thread pool (R:backend.py:34-38,
    :115-125); workers == 1 is the sequential backend."""
    if count <= 0:
        return
    if workers <= 1:
        fn(0, count)
        return
    chunk = max(1, -(-count // workers))
    if chunk >= count:
        fn(0, count)
        return
    spans = [(lo, min(lo + chunk, count)) for lo in range(0, count, chunk)]
    with ThreadPoolExecutor(max_workers=workers) as pool:
        for f in [pool.submit(fn, lo, hi) for lo, hi in spans]:
            f.result()


# ------------------------------------------------------- synthetic data (R:harness.py)
def benchmark_dataset(n_cases: int, n_features: int, seed: int = 1):
    """U[-1,1) features from stream 2^34, target x0*x1 + sum(x)
    (R:harness.py:36-41)."""
    d = unit_vec(seed, HARNESS_STREAM, np.arange(n_cases * n_features))
    X = d.reshape(n_cases, n_features) * 2.0 - 1.0
    y = X[:, 0] * X[:, 1 % n_features] + X.sum(axis=1)
    return X, y


# ------------------------------------------------------------------ full run
class Cfg:
    """Plain mirror of the RunConfig fields the path reads (R:core.py:292-309)."""

    def __init__(self, population_size=1024, random_trees=1024, program_size=1024,
                 generations=1024, seed=1, p_function=0.8, p_feature=0.14,
                 p_constant=0.04, erc_low=1.0, erc_high=10.0,
                 mutation_step="uniform", division_eps=1e-6, gsm_sign="minus", **_):
        self.m, self.r, self.k, self.g = population_size, random_trees, program_size, generations
        self.seed = seed
        self.p = (p_function, p_feature, p_constant)
        self.erc = (erc_low, erc_high)
        self.mutation_step = mutation_step
        self.eps = division_eps
        self.sign = gsm_sign


def run(cfg: Cfg, Xtr, ytr, Xte, yte, workers: int = 1, keep_initial: bool = False):
    """The reference loop of R:evolution.py:100-179 in fp64.

    Returns a dict with train/test traces (g+1), per-generation plans and
    elite records, final elite slot and train semantics, overflow count."""
    m, r, g, l = cfg.m, cfg.r, cfg.g, Xtr.shape[1]
    kw = dict(p_function=cfg.p[0], p_feature=cfg.p[1], p_constant=cfg.p[2],
              erc_low=cfg.erc[0], erc_high=cfg.erc[1])
    pop = genomes(m, cfg.k, l, cfg.seed, 0, **kw)
    trees = genomes(r, cfg.k, l, cfg.seed, m, **kw)
    stacked = np.vstack([Xtr, Xte])
    ntr = Xtr.shape[0]
    s_pop, c1 = semantics(*pop, stacked, cfg.eps, workers)
    s_tree, c2 = semantics(*trees, stacked, cfg.eps, workers)
    overflow = c1 + c2
    P_tr = np.ascontiguousarray(s_pop[:, :ntr])
    P_te = np.ascontiguousarray(s_pop[:, ntr:])
    T_tr = np.ascontiguousarray(s_tree[:, :ntr])
    T_te = np.ascontiguousarray(s_tree[:, ntr:])
    F = fitness(P_tr, ytr, workers)
    Q_tr = sigmoid(T_tr)
    Q_te = sigmoid(T_te)
    b0 = int(np.argmin(F))
    out = {
        "initial": ("initial", b0, b0, float(F[b0])),
        "train": np.empty(g + 1), "test": np.empty(g + 1),
        "u": np.empty((g, m), np.int64), "v": np.empty((g, m), np.int64),
        "ms": np.empty((g, m)), "elite": [],
    }
    if keep_initial:
        out["P_tr0"], out["P_te0"], out["F0"] = P_tr.copy(), P_te.copy(), F.copy()
        out["Q_tr"], out["Q_te"], out["T_tr"] = Q_tr, Q_te, T_tr
    out["train"][0] = F[b0]
    out["test"][0] = rmse(P_te[b0], yte)
    for gen in range(1, g + 1):
        u, v, ms = plan(m, r, cfg.seed, gen, cfg.mutation_step)
        O_tr, a = gsm_squashed(P_tr, Q_tr, u, v, ms, cfg.sign, workers)
        O_te, b = gsm_squashed(P_te, Q_te, u, v, ms, cfg.sign, workers)
        overflow += a + b
        Fo = fitness(O_tr, ytr, workers)
        src, idx, slot = survive(F, Fo)
        if src == "parent":
            O_tr[slot] = P_tr[idx]
            O_te[slot] = P_te[idx]
            Fo[slot] = F[idx]
        fit = float(Fo[slot])
        P_tr, P_te, F = O_tr, O_te, Fo
        out["u"][gen - 1], out["v"][gen - 1], out["ms"][gen - 1] = u, v, ms
        out["elite"].append((src, idx, slot, fit))
        out["train"][gen] = fit
        out["test"][gen] = rmse(P_te[slot], yte)
    final = out["elite"][-1] if g else out["initial"]
    out["slot"] = final[2]
    out["elite_train_semantics"] = P_tr[final[2]].copy()
    out["overflow"] = overflow
    return out


def replay(initial_semantics, tree_semantics, plans, elites, sign="minus"):
    """Re-apply recorded plans and survival decisions (R:evolution.py:182-202)."""
    cur = initial_semantics.copy()
    sq = sigmoid(tree_semantics)
    for (u, v, ms), (src, idx, slot, _) in zip(plans, elites):
        nxt, _ = gsm_squashed(cur, sq, u, v, ms, sign)
        if src == "parent":
            nxt[slot] = cur[idx]
        cur = nxt
    return cur


def default_workers() -> int:
    return os.cpu_count() or 1
