"""run_evolution and survival on the B200 (gsgp/evolution.py:36-202).

`run_evolution(cfg, train, test)` is the drop-in for the reference's run
API: one call into `gsgp_run` (libgsgp_b200.so, GIL released by ctypes) runs
CreatePopulation, genome compilation, interpretation of population and pool,
and all generations on the device, then returns a `RunResult` with the same
fields as the reference's.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib, devices as _devices, ops
from ._lib import check, ptr
from .core import (
    ConfigError, Dataset, EliteRecord, LineageEntry, LineageError, LineageLog, MutationPlan,
    RunConfig, StageTimings,
)

_SRC = {0: "parent", 1: "offspring", 2: "initial"}


@dataclass
class GenerationState:
    """gsgp/evolution.py:50-62."""

    train_semantics: np.ndarray
    fitness: np.ndarray
    test_semantics: np.ndarray

    def _check_shapes(self, other: "GenerationState") -> None:
        if (self.train_semantics.shape != other.train_semantics.shape
                or self.fitness.shape != other.fitness.shape
                or self.test_semantics.shape != other.test_semantics.shape):
            raise ConfigError("parent and offspring states must have equal shapes")


def survive(parent: GenerationState, offspring: GenerationState):
    """gsgp/evolution.py:65-83: the decision runs on the device; the row copy
    mutates the caller's offspring arrays exactly as the reference does."""
    parent._check_shapes(offspring)
    src, idx, slot = ops.survive_decision(parent.fitness, offspring.fitness)
    if src == "parent":
        offspring.train_semantics[slot] = parent.train_semantics[idx]
        offspring.test_semantics[slot] = parent.test_semantics[idx]
        offspring.fitness[slot] = parent.fitness[idx]
        return offspring, EliteRecord("parent", idx, slot, float(parent.fitness[idx]))
    return offspring, EliteRecord("offspring", idx, slot, float(offspring.fitness[idx]))


@dataclass
class RunResult:
    """gsgp/evolution.py:86-97, plus device-side measurements in `device`."""

    config: RunConfig
    train_fitness: np.ndarray
    test_fitness: np.ndarray
    lineage: LineageLog
    timings: StageTimings
    elite_slot: int
    elite_train_semantics: np.ndarray
    overflow_replacements: int
    device: dict = field(default_factory=dict)


def run_evolution(cfg: RunConfig, train: Dataset, test: Dataset, *, storage: str = "fp32",
                  use_graph: bool = True, time_kernels: bool = False,
                  virtual_shards: int = 1, window_start: int = 0, devices="auto") -> RunResult:
    """gsgp/evolution.py:100-179 on the B200.

    storage: "fp32" (default; semantics stored in fp32, interpreter and SSE in
    fp64 — DESIGN.md §4) or "fp64" (bit-for-bit reference arithmetic for the
    GSM; twice the memory).  virtual_shards > 1 splits the fitness cases into
    that many shards on this device and combines their partial SSEs exactly as
    the multi-GPU path does (single-GPU emulation of case sharding).
    time_kernels records CUDA events around every GSM launch (direct launches
    instead of the replayed graph); window_start opens a device-timed window
    over generations window_start+1..g (`device["window_ms"]`).
    devices: the GPUs this one call drives (devices.py: "auto" = every
    visible GPU the workload can use, one per 2 GiB of population semantics;
    "all"; an int n; a list of ids; None = the current device).  Several
    devices shard the cases by device inside this process (one host thread
    and one NCCL rank per GPU) and give the same bits as one device.
    """
    if train.n_features != test.n_features:
        raise ConfigError(f"train has {train.n_features} features but test has {test.n_features}")
    t0 = time.perf_counter()
    m, g = cfg.population_size, cfg.generations
    # the reference's Dataset may hold strided views (load_dataset slices the
    # target column off): the C ABI takes C-contiguous fp64
    Xtr, ytr = ops._f64(train.features), ops._f64(train.target)
    Xte, yte = ops._f64(test.features), ops._f64(test.target)
    s = ops.config_struct(cfg, storage=storage, use_graph=use_graph, time_kernels=time_kernels,
                          virtual_shards=virtual_shards, window_start=window_start)
    out = _lib.GsgpOutputs()
    arrays = dict(
        train_trace=np.empty(g + 1), test_trace=np.empty(g + 1),
        elite_src=np.empty(g + 1, np.int8), elite_idx=np.empty(g + 1, np.int64),
        elite_slot=np.empty(g + 1, np.int64), elite_fit=np.empty(g + 1),
        plan_u=np.empty((max(g, 1), m), np.int64), plan_v=np.empty((max(g, 1), m), np.int64),
        plan_ms=np.empty((max(g, 1), m)), elite_train_semantics=np.zeros(train.n_cases),
        gsm_ms=np.zeros(max(g, 1)),
    )
    for name, arr in arrays.items():
        setattr(out, name, ptr(arr))
    ids = _devices.resolve(devices, m, train.n_cases + test.n_cases)
    _devices.activate(ids)
    t_call = t_call_start = time.perf_counter()
    rc = _lib.load().gsgp_run(C.byref(s), ptr(Xtr), ptr(ytr), train.n_cases, ptr(Xte), ptr(yte),
                               test.n_cases, train.n_features, C.byref(out))
    if rc and ids is not None and _lib.load().gsgp_device_count_in_use() != len(ids):
        _devices.reset()          # a failed multi-device run dropped its communicators
    check(rc)
    t_call = (time.perf_counter() - t_call) * 1e3
    a = arrays
    log = LineageLog(EliteRecord("initial", int(a["elite_idx"][0]), int(a["elite_slot"][0]),
                                 float(a["elite_fit"][0])))
    for t in range(1, g + 1):
        plan = MutationPlan(a["plan_u"][t - 1], a["plan_v"][t - 1], a["plan_ms"][t - 1])
        log.entries.append(LineageEntry(plan, EliteRecord(
            _SRC[int(a["elite_src"][t])], int(a["elite_idx"][t]), int(a["elite_slot"][t]),
            float(a["elite_fit"][t]))))
    st = list(out.stage_ms)
    total_ms = (time.perf_counter() - t0) * 1e3
    timings = StageTimings(create_population_ms=st[0], compute_semantics_ms=st[1],
                           evolution_ms=st[2], per_generation_ms=st[3], total_ms=total_ms)
    device = {"stage_ms": st, "gsm_kernel_ms": st[5], "gsm_launches": int(st[6]),
              "loop_launches": int(st[7]), "engine_total_ms": st[4], "call_ms": t_call,
              "prep_ms": (t_call_start - t0) * 1e3,
              "window_ms": st[8], "window_gsm_ms": st[9], "window_gsm_launches": int(st[10]),
              "window_loop_launches": int(st[11]),
              "gsm_ms_per_generation": a["gsm_ms"][:g] if time_kernels else None,
              "shard_train_range": (int(out.shard_train_lo), int(out.shard_train_hi)),
              "init_ms": {"upload": st[12], "interpret_population": st[13],
                          "interpret_pool": st[14], "initial_sse": st[15], "compile": st[16],
                          "alloc": st[17]},
              "program_instructions": {"population": int(st[18]), "pool": int(st[19])},
              "program_divisions": {"population": int(out.interp_div[0]), "pool": int(out.interp_div[1])},
              "program_operands": {side: {"vector_loads": int(out.interp_ops[3 * j]),
                                          "constant_loads": int(out.interp_ops[3 * j + 1]),
                                          "spill_stores": int(out.interp_ops[3 * j + 2])}
                                   for j, side in enumerate(("population", "pool"))},
              "devices": list(ids) if ids is not None else None,
              "storage": "fp64" if out.storage_f64_used else "fp32",
              "storage_requested": storage,
              "interpreter": {"config": int(out.interp_info[0]), "max_spill_depth": int(out.interp_info[1]),
                              "max_constants": int(out.interp_info[2]),
                              "max_instructions": int(out.interp_info[3])}}
    return RunResult(
        config=cfg, train_fitness=a["train_trace"], test_fitness=a["test_trace"], lineage=log,
        timings=timings, elite_slot=int(log.final_elite().slot),
        elite_train_semantics=a["elite_train_semantics"],
        overflow_replacements=int(out.overflow), device=device)


def replay_lineage(log: LineageLog, initial_semantics: np.ndarray, tree_semantics: np.ndarray,
                   cfg: RunConfig) -> np.ndarray:
    """gsgp/evolution.py:182-202 in ONE device call (`gsgp_replay`): the
    initial and tree semantics and all plans are uploaded once, every
    generation's fp64 GSM (sigmoid of the trees, as in the reference's gsm)
    and parent-elite restore run on the device, and only the final elite row
    comes back."""
    if log.generations != cfg.generations:
        raise LineageError(
            f"log covers {log.generations} generations, config expects {cfg.generations}")
    cur = np.ascontiguousarray(initial_semantics, dtype=np.float64)
    trees = np.ascontiguousarray(tree_semantics, dtype=np.float64)
    if cur.ndim != 2 or trees.ndim != 2 or cur.shape[1] != trees.shape[1]:
        raise ConfigError("parent and random-tree matrices must share the case axis")
    m, n = cur.shape
    g = len(log.entries)
    for entry in log.entries:
        if len(entry.plan) != m:
            raise LineageError("plan length does not match the population size")
    shape = (max(g, 1), m)
    u, v, ms = np.zeros(shape, np.int64), np.zeros(shape, np.int64), np.zeros(shape)
    src, idx, slot = np.ones(max(g, 1), np.int8), np.zeros(max(g, 1), np.int64), np.zeros(max(g, 1), np.int64)
    for t, e in enumerate(log.entries):
        u[t], v[t], ms[t] = e.plan.u, e.plan.v, e.plan.ms
        src[t] = 0 if e.elite.source == "parent" else 1
        idx[t], slot[t] = e.elite.index, e.elite.slot
    out = np.empty(n)
    check(_lib.load().gsgp_replay(ptr(cur), m, n, ptr(trees), trees.shape[0], g, ptr(u), ptr(v), ptr(ms),
                                  ptr(src), ptr(idx), ptr(slot), int(log.final_elite().slot),
                                  1 if cfg.gsm_sign == "plus" else 0, ptr(out)))
    return out
