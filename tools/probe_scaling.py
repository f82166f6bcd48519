"""Probe: per-GPU generation cost of the C3 case shard at N = 1, 2, 4, 8 GPUs,
measured on ONE GPU (gpurun has one), as the ingredients of a strong-scaling
projection.

    python tools/probe_scaling.py [generations]

For each N it runs rank 0's case slice of C3 (dist.shard_range: 12288-case
aligned, the slice the engine gives rank 0 of N) as a one-GPU run and
reports the device-timed generation loop (CUDA-graph replay) and the GSM
kernel time (CUDA events).  It also runs the N = 8 slice as two virtual
shards to measure what the sharded tail (per-shard digits + finish/survive
instead of the fused reduce/survive) costs on the device.  What one GPU
cannot measure — the two NCCL allreduces per generation (8 KB anchors,
64 KB digits at m = 1024) — is printed as an input the projection needs.
"""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2106_04034_b200 as G  # noqa: E402
from paper_2106_04034_b200 import dist  # noqa: E402

gens = int(sys.argv[1]) if len(sys.argv) > 1 else 40
c = bench.CONFIGS["c3"]
tr = G.make_benchmark_dataset(c["ntr"], c["l"], seed=1)
te = G.make_benchmark_dataset(c["nte"], c["l"], seed=2)
cfg = G.RunConfig(population_size=c["m"], random_trees=c["r"], program_size=c["k"], generations=gens, seed=1)
W = 5
for N in (1, 2, 4, 8):
    lo, hi = dist.shard_range(c["ntr"], N, 0)
    tlo, thi = dist.shard_range(c["nte"], N, 0)
    str_, ste = G.Dataset(tr.features[lo:hi], tr.target[lo:hi]), G.Dataset(te.features[tlo:thi], te.target[tlo:thi])
    out = {"N": N, "shard_cases": (hi - lo) + (thi - tlo)}
    for mode, kw in (("graph", {}), ("timed", dict(time_kernels=True))):
        res = G.run_evolution(cfg, str_, ste, window_start=W, devices=None, **kw)
        d = res.device
        if mode == "graph":
            out["loop_ms_per_generation"] = d["window_ms"] / (gens - W)
            out["interpreter_ms"] = d["init_ms"]["interpret_population"] + d["init_ms"]["interpret_pool"]
        else:
            out["gsm_ms_per_generation"] = d["window_gsm_ms"] / (gens - W)
            out["timed_loop_ms_per_generation"] = d["window_ms"] / (gens - W)
    if N == 8:
        res = G.run_evolution(cfg, str_, ste, window_start=W, devices=None, virtual_shards=2, time_kernels=True)
        d = res.device
        out["virtual2_loop_ms_per_generation"] = d["window_ms"] / (gens - W)
        out["virtual2_gsm_ms_per_generation"] = d["window_gsm_ms"] / (gens - W)
    print(json.dumps(out), flush=True)
