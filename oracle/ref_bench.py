"""CPU timing of the REAL reference package (BENCH INFRASTRUCTURE ONLY).

bench.py's `cpu_baseline` leg and `--impl reference` time the reference's
own code — `gsgp` 0.1.0 installed unmodified into `baseline/_ref` (pip
--target; git-ignored, it travels to the GPU box with the
repo snapshot) — on the host cores:

* `ref_generations`: the generation body of `run_evolution`
  (gsgp/evolution.py:146-158) executed with the reference's own functions —
  `build_mutation_plan`, `_gsm_squashed` (train and test), `compute_fitness`,
  `survive`, `rmse` — inside the reference's own backend
  (`get_backend("threads", 0)` = every host core, or "sequential").  The
  state is synthetic fp64 data of the workload's shape: a generation's cost
  does not depend on the values, and the reference's generations/s
  (`StageTimings.per_generation_ms`, evolution.py:145-167) excludes the init
  just like the device number;
* `ref_run`: the whole `run_evolution` call, init included, for workloads
  small enough to run in full (C1).

Nothing here is imported by the product package.  When `baseline/_ref` is
absent, bench.py falls back to the numpy restatement (oracle/cpu_bench.py,
kind "port").
"""

from __future__ import annotations

import importlib
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF_DIR = ROOT / "baseline" / "_ref"


def import_reference():
    """The reference package from baseline/_ref, or (None, reason)."""
    if not (REF_DIR / "gsgp" / "__init__.py").exists():
        return None, f"{REF_DIR} not installed"
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    try:
        mod = importlib.import_module("gsgp")
    except Exception as exc:  # pragma: no cover - broken install
        return None, f"import gsgp failed: {exc!r}"
    if Path(mod.__file__).resolve().parent != (REF_DIR / "gsgp").resolve():
        return None, f"gsgp resolved to {mod.__file__}, not baseline/_ref"
    return mod, ""


class RefLoop:
    """The reference's generation body on synthetic state (evolution.py:146-158)."""

    def __init__(self, gsgp, m, r, ntr, nte, backend="threads", threads=0, seed=1):
        from gsgp.evolution import GenerationState
        from gsgp.mutation import _gsm_squashed
        self.g, self.GS, self.gsm = gsgp, GenerationState, _gsm_squashed
        self.cfg = gsgp.RunConfig(population_size=m, random_trees=r, seed=seed, backend=backend,
                                  threads=threads)
        self.stats = gsgp.RunStats()
        rng = np.random.default_rng(seed)
        self.m, self.r = m, r
        u = lambda *shape: rng.random(shape) * 4.0 - 2.0  # noqa: E731  (values do not matter)
        self.ytr = u(ntr)
        self.yte = u(nte)
        self.sq_tr = gsgp.sigmoid_array(u(r, ntr))
        self.sq_te = gsgp.sigmoid_array(u(r, nte))
        self.backend = gsgp.get_backend(backend, threads)
        self.backend.__enter__()
        P_tr = u(m, ntr)
        self.state = GenerationState(P_tr, gsgp.compute_fitness(P_tr, self.ytr, self.backend), u(m, nte))
        self.workers = getattr(self.backend, "workers", 1)

    def generation(self, gen):
        g, cfg, st, be = self.g, self.cfg, self.state, self.backend
        plan = g.build_mutation_plan(self.m, self.r, cfg, gen)
        off_train = self.gsm(st.train_semantics, self.sq_tr, plan, cfg.gsm_sign, be, self.stats)
        off_test = self.gsm(st.test_semantics, self.sq_te, plan, cfg.gsm_sign, be, self.stats)
        off = self.GS(off_train, g.compute_fitness(off_train, self.ytr, be), off_test)
        self.state, elite = g.survive(st, off)
        g.rmse(self.state.test_semantics[elite.slot], self.yte)

    def close(self):
        self.backend.__exit__(None, None, None)


def ref_generations(m, r, ntr, nte, *, backend="threads", warmup=1, gens=None, budget_s=None,
                    min_gens=2):
    """Seconds per reference generation on an (ntr + nte)-case state; runs
    `gens` generations or until `budget_s` is spent (at least `min_gens`)."""
    gsgp, why = import_reference()
    if gsgp is None:
        raise RuntimeError(why)
    loop = RefLoop(gsgp, m, r, ntr, nte, backend=backend, threads=0)
    try:
        for w in range(warmup):
            loop.generation(w + 1)
        times = []
        t_start = time.perf_counter()
        gen = warmup
        while True:
            gen += 1
            t0 = time.perf_counter()
            loop.generation(gen)
            times.append(time.perf_counter() - t0)
            if gens is not None and len(times) >= gens:
                break
            if budget_s is not None and len(times) >= min_gens and time.perf_counter() - t_start >= budget_s:
                break
        return {"sec_per_gen": float(np.mean(times)), "gens_timed": len(times),
                "workers": loop.workers if backend == "threads" else 1, "backend": backend,
                "times": times}
    finally:
        loop.close()


def ref_run(m, r, k, l, ntr, nte, g, *, backend="threads", seed=1):
    """One whole reference run_evolution on make_benchmark_dataset data
    (train seed 1, test seed 2, gsgp/harness.py:36-41)."""
    gsgp, why = import_reference()
    if gsgp is None:
        raise RuntimeError(why)
    tr = gsgp.make_benchmark_dataset(ntr, l, seed=1)
    te = gsgp.make_benchmark_dataset(nte, l, seed=2)
    cfg = gsgp.RunConfig(population_size=m, random_trees=r, program_size=k, generations=g, seed=seed,
                         backend=backend, threads=0)
    res = gsgp.run_evolution(cfg, tr, te)
    t = res.timings
    return {"per_generation_ms": t.per_generation_ms, "create_ms": t.create_population_ms,
            "semantics_ms": t.compute_semantics_ms, "total_ms": t.total_ms,
            "workers": os.cpu_count() if backend == "threads" else 1, "backend": backend}
