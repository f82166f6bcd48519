#!/usr/bin/env python
"""GSGP generations/sec on B200 — the BASELINE.json metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

A step is one GSGP generation (plan -> fused GSM+SSE on train and test ->
SSE reduction -> [NCCL allreduce] -> elitist survival) over the configured
synthetic workload.  W warm-up generations run untimed, then exactly K
generations are timed on the device with CUDA events (the engine records
the window events on its stream).  Default workload: C3 = pop 1024, 8
features, 10M train + 2.5M test cases, random-tree pool 1024, k=1024 — the
configuration the metric is quoted on at 1/2/4/8 B200 (cases sharded by
GPU, strong scaling); it fits one GPU (~103 GB).  N > 1 GPUs: under
torchrun one process per GPU; without it, --gpus N drives N GPUs from this
process (gsgp_init: one host thread and one NCCL rank per device).

Printed JSON line (rank 0): value = generations/s of the whole job; e2e =
the same metric through the public `run_evolution` call from host numpy
datasets (H2D, init, loop and D2H inside the timed region); roofline = the
fused GSM+SSE kernel's algorithmic bytes (4*N*(2m+D_g+1) per
generation) over its CUDA-event time; cpu_baseline = the reference's own
generation body (baseline/_ref gsgp 0.1.0, all host cores) on a bounded case
sample.  `--impl reference` times that CPU reference path alone, one
generation per step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "c1": dict(m=256, r=1024, k=1024, l=5, ntr=500, nte=200, g=50,
               desc="C1 synthetic SR, 5 features, 500/200 cases, pop 256, pool 1024, k=1024"),
    "c2": dict(m=1024, r=1024, k=1024, l=8, ntr=100_000, nte=25_000, g=500,
               desc="C2 pop 1024, 8 features, 100k+25k cases, pool 1024, k=1024"),
    "c3": dict(m=1024, r=1024, k=1024, l=8, ntr=10_000_000, nte=2_500_000, g=100,
               desc="C3 pop 1024, 8 features, 10M+2.5M cases sharded by case, pool 1024, k=1024"),
    "c4": dict(m=8192, r=1024, k=255, l=8, ntr=1_000_000, nte=250_000, g=50,
               desc="C4 pop 8192, 1M+250k cases, pool 1024, k=255 (depth-8 trees)"),
    "c5": dict(m=2048, r=1024, k=1024, l=100, ntr=2_000_000, nte=500_000, g=50,
               desc="C5 pop 2048, 100 features, 2M+500k cases, pool 1024, k=1024"),
    # profiling shapes: C4's population/pool ratio on C2's case count, C5's feature count on
    # 200k+50k cases (kernel-replay ncu fits)
    "c5s": dict(m=2048, r=1024, k=1024, l=100, ntr=200_000, nte=50_000, g=50,
                desc="C5-shaped profiling config: pop 2048, 100 features, 200k+50k cases"),
    "c4s": dict(m=8192, r=1024, k=255, l=8, ntr=100_000, nte=25_000, g=50,
                desc="C4-shaped profiling config: pop 8192, pool 1024, k=255, 100k+25k cases"),
}
METRIC = "generations/sec"
L2_BYTES = 126 * 1024 * 1024     # B200 L2 (the timed semantics must not fit in it)
NVML_REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
                0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
                0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
                0x100: "display_clock_setting"}


def peaks():
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler(threading.Thread):
    """nvidia-smi-equivalent sampling (NVML) of SM clock and throttle reasons."""

    def __init__(self, index: int, period: float = 0.02):
        super().__init__(daemon=True)
        self.index, self.period = index, period
        self.samples = []
        self.stop_flag = threading.Event()
        self.max_mhz = None
        self.ok = True

    def run(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            get_reasons = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                N.nvmlDeviceGetCurrentClocksThrottleReasons
            while not self.stop_flag.is_set():
                util = N.nvmlDeviceGetUtilizationRates(h).gpu
                self.samples.append((N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM), int(get_reasons(h)), util,
                                     N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_MEM),
                                     N.nvmlDeviceGetPowerUsage(h) / 1000.0, time.perf_counter()))
                time.sleep(self.period)
        except Exception as exc:  # no NVML: report what we have
            self.ok = False
            self.err = repr(exc)

    def summary(self):
        self.stop_flag.set()
        self.join(timeout=2)
        load = [s for s in self.samples if s[2] >= 30] or self.samples
        reasons = set()
        for s in load:
            for bit, name in NVML_REASONS.items():
                if s[1] & bit and name != "gpu_idle":
                    reasons.add(name)
        med = lambda k: statistics.median([s[k] for s in load]) if load else None  # noqa: E731
        return {"sm_mhz": med(0), "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons),
                "mem_mhz": med(3), "power_w_median": med(4),
                "power_w_max": max((s[4] for s in load), default=None),
                "samples": len(self.samples), "samples_under_load": len(load)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return world, rank, local


def bytes_per_generation(plans, N: int, m: int) -> np.ndarray:
    """4*N*(2m + D_g + 1), D_g = distinct pool rows of the plan."""
    out = []
    for u, v in plans:
        D = len(np.union1d(u, v))
        out.append(4.0 * N * (2 * m + D + 1))
    return np.array(out)


def interp_line(res, c, world: int) -> dict:
    """ComputeSemantics: issue/fp64 bound, reported as function-
    node evaluations per second (one compiled instruction = one function node
    of the dead-code-eliminated, constant-folded tree) with its compulsory
    bytes (features read once, fp32 semantics written)."""
    N = (c["ntr"] + c["nte"]) / world
    ins = res.device["program_instructions"]
    ms = res.device["init_ms"]
    t = (ms["interpret_population"] + ms["interpret_pool"]) / 1e3
    evals = (ins["population"] + ins["pool"]) * N
    byts = N * c["l"] * 8 + (c["m"] + c["r"]) * N * 4
    # fp64 roofline: every instruction is one fp64 op per case, a protected
    # division 8 (the fast path: 5 Newton FMAs, the quotient and its
    # two-FMA correction; + one MUFU.RCP64H on another pipe), against the
    # measured DFMA/DADD/DMUL lane-op rate of this pool's B200s
    div = res.device.get("program_divisions") or {"population": 0, "pool": 0}
    fp64_ops = (ins["population"] + ins["pool"] + 7 * (div["population"] + div["pool"])) * N
    peak = fp64_peak()
    smem = smem_roofline(res, N, t)
    return {"node_evals_per_s": evals / t if t > 0 else None, "unit": "function-node evals/s",
            "seconds": t, "mean_program_instructions": (ins["population"] + ins["pool"]) / (c["m"] + c["r"]),
            "division_share": (div["population"] + div["pool"]) / max(1, ins["population"] + ins["pool"]),
            "compulsory_bytes": byts, "compulsory_GBps": byts / t / 1e9 if t > 0 else None,
            "fp64_roofline": {"achieved": fp64_ops / t if t > 0 else None, "peak": peak["value"],
                              "unit": "fp64 lane-ops/s", "frac": fp64_ops / t / peak["value"] if t > 0 else None,
                              "ops": fp64_ops, "peak_source": peak["source"]},
            "smem_roofline": smem,
            "bound": "shared-memory operand wavefronts + dispatch issue (see DESIGN.md §6)"}


# cases per thread and "features staged in shared memory" of the interpreter
# launch configurations (interp.cu kCfgs; 8 is retired)
INTERP_CFGS = {0: (4, True), 1: (8, True), 2: (4, False), 3: (2, True), 4: (1, False), 5: (3, True),
               6: (3, True), 7: (4, True), 9: (4, True), 10: (4, True)}


def smem_roofline(res, N: float, t: float):
    """Shared-memory wavefronts (128 B each, one per SM per clock) the
    interpreter's operand traffic needs, from the compiled programs' op mix
    (k_compile): per warp-instruction one broadcast LDS.128 program fetch, 2
    wavefronts per case for a per-case operand load (feature or spill row:
    32 lanes x 8 B) or spill store, 1 per case for a broadcast constant load.
    Staging of features/programs/constants and bank conflicts are not
    counted (ncu: the C2 population launch runs at 0.81 of the
    l1tex shared-memory wavefront peak, profiles/r02/ncu_interp_src)."""
    info = res.device.get("interpreter") or {}
    ops = res.device.get("program_operands")
    cfg = INTERP_CFGS.get(info.get("config"))
    if not ops or cfg is None or not cfg[1] or t <= 0:
        return None
    cpt = cfg[0]
    ins = res.device["program_instructions"]
    per_warp = 0.0
    for side in ("population", "pool"):
        o = ops[side]
        per_warp += ins[side] + cpt * (2 * o["vector_loads"] + o["constant_loads"] + 2 * o["spill_stores"])
    wf = per_warp * N / (32 * cpt)
    try:
        mhz = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["sm_max_mhz"])
    except Exception:
        mhz = 1965.0
    peak = 148 * mhz * 1e6
    return {"achieved": wf / t, "peak": peak, "unit": "shared-memory wavefronts/s (128 B)",
            "frac": wf / t / peak, "wavefronts": wf,
            "peak_source": f"1 wavefront per SM per clock at the {mhz:.0f} MHz max SM clock",
            "cases_per_thread": cpt}


def fp64_peak() -> dict:
    """Measured fp64 lane-op rate (tools/fp64_peak.cu on this pool's B200s,
    profiles/r02/fp64_peak.json: DFMA/DADD/DMUL, 8 independent chains per
    thread, all SMs)."""
    try:
        d = json.loads((ROOT / "profiles" / "r02" / "fp64_peak.json").read_text())
        return {"value": float(d["dfma_lane_ops_per_s"]),
                "source": "measured: tools/fp64_peak.cu (profiles/r02/fp64_peak.json)"}
    except Exception:
        return {"value": 148 * 64 * 1.965e9, "source": "fallback: 64 fp64 lanes/SM/clock at 1965 MHz"}


def workload_config(c) -> dict:
    """The `config` object of BOTH arms (identical by construction)."""
    return {"workload": c["desc"], "m": c["m"], "r": c["r"], "k": c["k"], "features": c["l"],
            "n_train": c["ntr"], "n_test": c["nte"],
            "l2": ("inputs larger than L2 (population and pool semantics "
                   f"{4 * c['m'] * (c['ntr'] + c['nte']) / 1e9:.1f} GB each)")
            if 4 * c["m"] * (c["ntr"] + c["nte"]) > L2_BYTES else "small config: L2-resident"}


def ref_sample(c, max_cases=125_000):
    """Case sample of the CPU reference legs: the whole workload when it has
    at most `max_cases` cases, else max_cases in the workload's train:test
    ratio (C3-C5 timed at 100k+25k and scaled linearly in N,
    the reference's O(m*g*n/t))."""
    N = c["ntr"] + c["nte"]
    if N <= max_cases:
        return c["ntr"], c["nte"], 1.0
    s_tr = int(round(max_cases * c["ntr"] / N))
    s_te = max_cases - s_tr
    return s_tr, s_te, max_cases / N


def cpu_leg(c, budget_s: float):
    """cpu_baseline: the reference's own generation body (baseline/_ref,
    oracle/ref_bench.py) on this host — all cores through its ThreadBackend
    (the value) and its SequentialBackend — else the numpy port."""
    from oracle import cpu_bench, ref_bench
    s_tr, s_te, frac = ref_sample(c)
    workers = os.cpu_count() or 1
    gsgp, why = ref_bench.import_reference()
    if gsgp is not None:
        thr = ref_bench.ref_generations(c["m"], c["r"], s_tr, s_te, backend="threads",
                                        budget_s=budget_s * 0.6, min_gens=3)
        seq = ref_bench.ref_generations(c["m"], c["r"], s_tr, s_te, backend="sequential",
                                        budget_s=budget_s * 0.3, min_gens=1, warmup=0)
        sample = (f"reference gsgp 0.1.0 (baseline/_ref, unmodified) generation body "
                  f"(gsgp/evolution.py:146-158: build_mutation_plan, _gsm_squashed x2, compute_fitness, "
                  f"survive, rmse) with get_backend('threads', 0) = {thr['workers']} threads, "
                  f"m={c['m']} r={c['r']} on {s_tr}+{s_te} cases (synthetic fp64 state), "
                  f"{thr['gens_timed']} timed generations")
        if frac < 1.0:
            sample += f", rate scaled linearly from {s_tr + s_te} to {c['ntr'] + c['nte']} cases"
        return {"value": frac / thr["sec_per_gen"], "unit": METRIC, "cores": thr["workers"],
                "kind": "reference", "sample": sample, "cpu": cpu_bench.cpu_model(),
                "sec_per_gen_sample": thr["sec_per_gen"],
                "sequential": {"value": frac / seq["sec_per_gen"], "cores": 1,
                               "sec_per_gen_sample": seq["sec_per_gen"], "gens_timed": seq["gens_timed"]}}
    t = cpu_bench.time_loop(c["m"], c["r"], s_tr, s_te, budget_s=budget_s, workers=workers)
    sample = (f"oracle port of gsgp/evolution.py:146-158 (numpy, {t['workers']} threads; {why}) on "
              f"synthetic fp64 state m={c['m']} r={c['r']} with {s_tr}+{s_te} cases, "
              f"{t['gens_timed']} timed generations")
    if frac < 1.0:
        sample += f", rate scaled linearly from {s_tr + s_te} to {c['ntr'] + c['nte']} cases"
    return {"value": t["sec_per_gen_sample"] and frac / t["sec_per_gen_sample"], "unit": METRIC,
            "cores": t["workers"], "kind": "port", "sample": sample, "cpu": cpu_bench.cpu_model(),
            "sec_per_gen_sample": t["sec_per_gen_sample"]}


def run_ours(args):
    world, rank, local = dist_env()
    if world > 1 and args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but torchrun started {world} ranks")
    td = None
    if world > 1:
        import torch.distributed as td
        td.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2106_04034_b200 as G
    from paper_2106_04034_b200 import _lib, devices, dist
    lib = _lib.load()
    # GSGP_BENCH_HOST_EXCHANGE=1: harness check of the N>1 path with every
    # rank on GPU 0 and the collectives over host memory + gloo (no NCCL);
    # its numbers are not bench values
    host_xchg = world > 1 and os.environ.get("GSGP_BENCH_HOST_EXCHANGE") == "1"
    _lib.check(lib.gsgp_set_device(0 if host_xchg else local))
    devices.reset()
    if world > 1:
        if host_xchg:
            dist.init_host_exchange()
        else:
            dist.init_from_torch()
    # without torchrun, --gpus N > 1 drives N GPUs from this one process
    # (gsgp_init: one host thread and one NCCL rank per device)
    in_proc = args.gpus if world == 1 and args.gpus > 1 else None
    if in_proc is not None and devices.visible_device_count() < in_proc:
        raise SystemExit(f"--gpus {in_proc} but only {devices.visible_device_count()} GPUs are visible")
    n_gpus = world * (in_proc or 1)
    ranks = n_gpus
    shard = rank if world > 1 else 0           # the shard whose kernel time the roofline uses

    def barrier():
        if td:
            td.barrier()

    def max_over_ranks(x: float) -> float:
        if not td:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64)
        td.all_reduce(t, op=td.ReduceOp.MAX)
        return float(t.item())

    c = CONFIGS[args.config]
    K, W = args.steps, args.warmup
    train = G.make_benchmark_dataset(c["ntr"], c["l"], seed=1)
    test = G.make_benchmark_dataset(c["nte"], c["l"], seed=2)
    cfg = G.RunConfig(population_size=c["m"], random_trees=c["r"], program_size=c["k"],
                      generations=W + K, seed=1)

    # ---- device-timed run: W warm-up generations, then exactly K timed
    sampler = ClockSampler(local)
    sampler.start()
    barrier()
    res = G.run_evolution(cfg, train, test, time_kernels=True, window_start=W, devices=in_proc)
    barrier()
    clocks = sampler.summary()
    win_ms = max_over_ranks(res.device["window_ms"])     # engine: max over its device threads
    value = K / (win_ms / 1e3)

    lo, hi = dist.shard_range(c["ntr"], ranks, shard)
    te_lo, te_hi = dist.shard_range(c["nte"], ranks, shard)
    n_local = (hi - lo) + (te_hi - te_lo)     # cases this shard's kernel streams
    plans = [(e.plan.u, e.plan.v) for e in res.lineage.entries[W:]]
    bpg = bytes_per_generation(plans, n_local, c["m"])
    gsm_ms = res.device["window_gsm_ms"]      # shard 0 of this process (rank 0's device thread)
    launches = max(res.device["window_gsm_launches"] // (in_proc or 1), 1)
    achieved = float(bpg.sum() / (gsm_ms / 1e3) / 1e9)
    peak, peak_kind = peaks()
    traffic = None
    tfile = ROOT / "profiles" / "gsm_traffic.json"
    if tfile.exists() and n_gpus == 1:
        try:
            traffic = json.loads(tfile.read_text()).get(args.config)
        except Exception:
            traffic = None

    # ---- end to end through the public API (host datasets, H2D/D2H inside)
    e2e = None
    if not args.no_e2e:
        cfg2 = G.RunConfig(population_size=c["m"], random_trees=c["r"], program_size=c["k"],
                           generations=K, seed=1)
        barrier()
        t0 = time.perf_counter()
        res2 = G.run_evolution(cfg2, train, test, devices=in_proc)
        barrier()
        wall = max_over_ranks(time.perf_counter() - t0)
        h2d = (train.features.nbytes + train.target.nbytes + test.features.nbytes + test.target.nbytes)
        d2h = (K + 1) * (8 + 8 + 1 + 8 + 8 + 8) + K * c["m"] * 24 + 8 * c["ntr"]
        e2e = {"value": K / wall, "unit": METRIC, "h2d_bytes_per_step": h2d / K,
               "d2h_bytes_per_step": d2h / K, "wall_s": wall,
               "init_ms": res2.timings.create_population_ms + res2.timings.compute_semantics_ms,
               "loop_ms": res2.timings.evolution_ms,
               "engine_host_ms": res2.device["engine_total_ms"],
               "engine_call_ms": res2.device["call_ms"], "api_prep_ms": res2.device["prep_ms"],
               "note": "second run_evolution call of the process (after the device-timed run): "
                       "device blocks and pinned staging are reused, the ~20 ms first-run "
                       "cudaMalloc is not in this window",
               "init_phases_ms": res2.device["init_ms"]}

    cpu = None
    if rank == 0 and n_gpus == 1 and not args.no_cpu_baseline:
        cpu = cpu_leg(c, args.cpu_budget)

    # secondary single-GPU line on C2 (configs[1]) for context, same method
    secondary = None
    if n_gpus == 1 and args.config == "c3" and not args.no_secondary:
        c2 = CONFIGS["c2"]
        tr2 = G.make_benchmark_dataset(c2["ntr"], c2["l"], seed=1)
        te2 = G.make_benchmark_dataset(c2["nte"], c2["l"], seed=2)
        K2 = 500
        r2 = G.run_evolution(G.RunConfig(population_size=c2["m"], random_trees=c2["r"],
                                         program_size=c2["k"], generations=W + K2, seed=1),
                             tr2, te2, time_kernels=True, window_start=W, devices=None)
        b2 = bytes_per_generation([(e.plan.u, e.plan.v) for e in r2.lineage.entries[W:]],
                                  c2["ntr"] + c2["nte"], c2["m"])
        a2 = float(b2.sum() / (r2.device["window_gsm_ms"] / 1e3) / 1e9)
        secondary = {"workload": c2["desc"], "steps": K2,
                     "value": K2 / (r2.device["window_ms"] / 1e3), "unit": "generations/s",
                     "roofline": {"achieved": a2, "peak": peak, "unit": "GB/s", "frac": a2 / peak,
                                  "kernel_share_of_step": r2.device["window_gsm_ms"] / r2.device["window_ms"]}}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "generations/s", "n_gpus": n_gpus,
            "steps": K, "warmup": W, "ms_per_step": win_ms / K, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32 storage / f64 interp+SSE",
            "data": "synthetic (make_benchmark_dataset: U[-1,1) features, x0*x1+sum(x) target)",
            "config": workload_config(c),
            "impl": "ours",
            "parallelism": (f"case-shard x{n_gpus}: " +
                            ("one process per GPU (torchrun, NCCL)" if world > 1 else
                             "one process, one host thread + NCCL rank per GPU (gsgp_init)"
                             if in_proc else "single GPU")),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "k_gsm_tma<float> (fused GSM+SSE, train+test)",
                         "peak_kind": peak_kind,
                         "algorithmic_bytes_per_launch": float(bpg.mean()),
                         "avg_launch_ms": gsm_ms / launches,
                         "kernel_share_of_step": gsm_ms / win_ms,
                         "shard": f"{shard} of {ranks} ({n_local} cases)"},
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": res.device["window_loop_launches"] * (world if world > 1 else 1),
            "clocks": clocks,
            "interpreter": interp_line(res, c, ranks),
            "init_ms": {"create_population": res.timings.create_population_ms,
                        "compute_semantics": res.timings.compute_semantics_ms,
                        **res.device["init_ms"]},
            "timing_note": "timed run: direct launches with CUDA events around every GSM launch "
                           "on the engine stream (run_evolution(time_kernels=True)); the default "
                           "API path replays one captured generation as a CUDA graph",
            "secondary": secondary,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy()
        td.destroy_process_group()
    else:
        devices.activate(None)


def run_reference(args):
    """The reference's own CPU code (baseline/_ref gsgp 0.1.0, oracle/ref_bench.py)
    on this host's cores: each step is one generation of the reference's
    generation body with its ThreadBackend over every core, on the workload's
    case sample (ref_sample), value scaled to the full config; the numpy port
    stands in when baseline/_ref is missing."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import cpu_bench, ref_bench
    c = CONFIGS[args.config]
    K, W = args.steps, args.warmup
    N = c["ntr"] + c["nte"]
    s_tr, s_te, frac = ref_sample(c)
    workers = os.cpu_count() or 1
    gsgp, why = ref_bench.import_reference()
    if gsgp is not None:
        kind = "reference"
        r = ref_bench.ref_generations(c["m"], c["r"], s_tr, s_te, backend="threads", warmup=W, gens=K)
        dt = sum(r["times"])
        workers = r["workers"]
        sample = (f"each step = one generation of the reference gsgp 0.1.0 (baseline/_ref, unmodified: "
                  f"gsgp/evolution.py:146-158 with get_backend('threads', 0), {workers} threads) on "
                  f"{s_tr}+{s_te} cases of synthetic fp64 state")
    else:
        kind = "port"
        st = cpu_bench.LoopState(c["m"], c["r"], s_tr, s_te)
        for w in range(W):
            st.generation(w + 1, workers=workers)
        t0 = time.perf_counter()
        for k in range(K):
            st.generation(W + k + 1, workers=workers)
        dt = time.perf_counter() - t0
        sample = (f"each step = one generation of the oracle port of gsgp/evolution.py:146-158 "
                  f"(numpy, {workers} threads; {why}) on {s_tr}+{s_te} cases")
    if frac < 1.0:
        sample += f" of the {N}-case workload; value = steps/s x {frac:.6f} (full-generation equivalents)"
    value = K / dt * frac
    line = {"metric": METRIC, "value": value, "unit": "generations/s", "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": dt / K * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(c),
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": METRIC, "cores": workers, "kind": kind,
                             "sample": sample, "cpu": cpu_bench.cpu_model()},
            "e2e": {"value": value, "unit": METRIC, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-secondary", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
