"""Multi-run batching: a job's `cfg.runs` independent runs.

The reference executes run i of a job with seed `derive_seed(cfg.seed, i)`,
one after the other (gsgp/io_cli.py:288-289).  Runs share the datasets and
nothing else, so they are replicas: with one process per GPU (torchrun) run
i executes on rank i % world — no collective on the data path, each rank
owns a whole GPU for its runs — and the results (or just their summaries)
are gathered to rank 0 in run order.  Under a single process the runs go
back to back on the one device, exactly as the reference orders them.

Case sharding (one run spread over all ranks, `dist.init_from_torch`) is the
other multi-GPU mode; the two are exclusive: replicas never create the
library's NCCL communicator.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

from .core import ConfigError, GsgpError, RunConfig


def run_seeds(cfg: RunConfig) -> list[int]:
    """Seeds of a job's runs (gsgp/io_cli.py:288-289)."""
    from .ops import derive_seed
    return [derive_seed(cfg.seed, i) for i in range(cfg.runs)]


def assign_runs(runs: int, world: int, rank: int) -> list[int]:
    """Run indices executed by `rank` (round-robin: rank r gets r, r+W, ...)."""
    if world < 1 or not 0 <= rank < world:
        raise ConfigError(f"bad rank {rank} of world {world}")
    return list(range(rank, runs, world))


@dataclass
class RunSummary:
    """What rank 0 needs to report a run it did not execute."""
    index: int
    seed: int
    train_fitness: list
    test_fitness: list
    overflow_replacements: int
    timings: object
    rank: int


def _world(group):
    try:
        import torch.distributed as td
    except ImportError:        # pragma: no cover - torch is in the image
        return 1, 0, None
    if not (td.is_available() and td.is_initialized()):
        return 1, 0, None
    return td.get_world_size(group), td.get_rank(group), td


def select_local_device() -> None:
    """Bind this process to its GPU (LOCAL_RANK) before its first run
    (GSGP_SHARED_GPU=1: every rank on GPU 0, for tests on a one-GPU box)."""
    from . import _lib
    from . import devices
    local = 0 if os.environ.get("GSGP_SHARED_GPU") == "1" else int(os.environ.get("LOCAL_RANK", "0"))
    _lib.check(_lib.load().gsgp_set_device(local))
    devices.reset()


def _device_run(cfg, train, test, **kw):
    from .engine import run_evolution
    return run_evolution(cfg, train, test, **kw)


def run_many(cfg: RunConfig, train, test, *, group=None, gather: str = "results", run_fn=None,
             on_result=None, **engine_kw):
    """Execute the job's cfg.runs runs; returns a list indexed by run.

    gather = "results": rank 0 receives every RunResult (pickled over the
    process group; lineages included), "summary": rank 0 receives a
    RunSummary per foreign run, "none": nothing is exchanged.  Other ranks
    get None for runs they did not execute.  `on_result(index, result)` is
    called on the executing rank right after each run (e.g. to write its
    trace files).  `run_fn` defaults to the device `run_evolution`.
    """
    if gather not in ("results", "summary", "none"):
        raise ConfigError("gather must be 'results', 'summary' or 'none'")
    if run_fn is None:
        run_fn = _device_run
    world, rank, td = _world(group)
    seeds = run_seeds(cfg)
    mine = assign_runs(cfg.runs, world, rank)
    out: list = [None] * cfg.runs
    failure = None
    if world > 1 and run_fn is _device_run:
        engine_kw.setdefault("devices", None)     # replicas: each rank keeps its own GPU
    for i in mine:
        try:
            res = run_fn(cfg.with_seed(seeds[i]), train, test, **engine_kw)
            if on_result is not None:
                on_result(i, res)
        except (GsgpError, OSError) as exc:
            # a failing rank still reaches the gather below, so the other
            # ranks never block in it until the process-group timeout
            if world == 1 or gather == "none":
                raise
            failure = (i, rank, f"{type(exc).__name__}: {exc}")
            break
        out[i] = res
    if world == 1 or gather == "none":
        return out
    if failure is not None:
        payload = {"__failure__": failure}
    elif gather == "summary":
        payload = {i: RunSummary(i, seeds[i], list(map(float, out[i].train_fitness)),
                                 list(map(float, out[i].test_fitness)), int(out[i].overflow_replacements),
                                 out[i].timings, rank) for i in mine}
    else:
        payload = {i: out[i] for i in mine}
    parts = [None] * world if rank == 0 else None
    td.gather_object(payload, parts, dst=0, group=group)
    if failure is not None:
        raise GsgpError(f"run {failure[0]} failed on rank {failure[1]}: {failure[2]}")
    if rank == 0:
        failed = [p["__failure__"] for p in parts if "__failure__" in p]
        if failed:
            i, r, msg = failed[0]
            raise GsgpError(f"run {i} failed on rank {r}: {msg}")
        for part in parts:
            for i, v in part.items():
                if out[i] is None:
                    out[i] = v
    return out
