"""CPU timing of the reference generation loop (TEST/BENCH INFRASTRUCTURE ONLY).

Used by bench.py for the `cpu_baseline` leg and for `--impl reference`.  It
times the reference's generation body (gsgp/evolution.py:146-158, restated in
oracle/restate.py with the reference's ThreadBackend row chunking) on the
host cores.  The per-generation cost of that body does not depend on the
semantic values, so the initial state is synthetic fp64 data of the exact
shape (interpreting k=1024 genomes over millions of cases on a CPU would take
hours and is not what generations/s measures — the reference excludes init).
When the configured case count is too large for a bounded CPU sample, the
loop runs on a contiguous case sample and the rate is scaled linearly in the
case count, the reference's own O(m*g*n/t) claim that
pkg/tests/test_acceptance.py:248-257 checks.
"""

from __future__ import annotations

import math
import os
import time

import numpy as np

from . import restate as R


class LoopState:
    def __init__(self, m, r, ntr, nte, seed=1):
        rng = np.random.default_rng(seed)
        self.m, self.r, self.ntr, self.nte = m, r, ntr, nte
        self.P_tr = rng.normal(size=(m, ntr))
        self.P_te = rng.normal(size=(m, nte))
        self.Q_tr = R.sigmoid(rng.normal(size=(r, ntr)))
        self.Q_te = R.sigmoid(rng.normal(size=(r, nte)))
        self.ytr = rng.normal(size=ntr)
        self.yte = rng.normal(size=nte)
        self.F = R.fitness(self.P_tr, self.ytr)

    def generation(self, gen, seed=1, workers=1):
        """One reference generation body (evolution.py:146-158)."""
        u, v, ms = R.plan(self.m, self.r, seed, gen)
        O_tr, _ = R.gsm_squashed(self.P_tr, self.Q_tr, u, v, ms, "minus", workers)
        O_te, _ = R.gsm_squashed(self.P_te, self.Q_te, u, v, ms, "minus", workers)
        Fo = R.fitness(O_tr, self.ytr, workers)
        src, idx, slot = R.survive(self.F, Fo)
        if src == "parent":
            O_tr[slot], O_te[slot], Fo[slot] = self.P_tr[idx], self.P_te[idx], self.F[idx]
        self.P_tr, self.P_te, self.F = O_tr, O_te, Fo
        R.rmse(self.P_te[slot], self.yte)


def time_loop(m, r, ntr, nte, *, budget_s=20.0, max_cases=None, workers=None, min_gens=3,
              max_gens=None, warmup=1):
    """Time the reference generation body; returns a dict with the measured
    seconds per generation on the sample and the rate scaled to (ntr+nte)."""
    workers = workers or os.cpu_count() or 1
    N = ntr + nte
    scale = 1.0
    s_tr, s_te = ntr, nte
    if max_cases is not None and N > max_cases:
        scale = max_cases / N
        s_tr = max(1, int(round(ntr * scale)))
        s_te = max(1, int(round(nte * scale)))
        scale = (s_tr + s_te) / N
    st = LoopState(m, r, s_tr, s_te)
    for w in range(warmup):
        st.generation(w + 1, workers=workers)
    times = []
    gen = warmup
    t_start = time.perf_counter()
    while True:
        gen += 1
        t0 = time.perf_counter()
        st.generation(gen, workers=workers)
        times.append(time.perf_counter() - t0)
        spent = time.perf_counter() - t_start
        if len(times) >= min_gens and (spent >= budget_s or (max_gens and len(times) >= max_gens)):
            break
    sec = float(np.mean(times))
    return {"sec_per_gen_sample": sec, "gens_timed": len(times), "sample_train": s_tr,
            "sample_test": s_te, "case_fraction": scale, "workers": workers,
            "gen_per_s": (1.0 / sec) * scale}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def sample_cases_for(step_seconds: float, m: int, probe=None) -> int:
    """Case count whose generation takes about `step_seconds` (linear model
    from a probe measurement of sec/gen at `probe` cases)."""
    if probe is None:
        return 10_000
    cases, sec = probe
    return max(1000, int(math.floor(cases * step_seconds / max(sec, 1e-9))))
