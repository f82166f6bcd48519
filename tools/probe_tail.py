"""Probe: per-generation cost of the generation tail by sharding mode on one GPU.

    python tools/probe_tail.py [config] [generations]

Modes (same run, same data; the results are bit-identical by construction,
checked here too):
  * single      one shard: GSM launch + fused reduce/survive kernel (2 launches)
  * virtual2    two case shards on this GPU: 2 GSM + 2 digits + finish/survive
  * threads2    two device threads on this GPU (devices=[0, 0]): the
                multi-device engine with its thread exchange standing in for
                NCCL (allreduce-max of the anchors, allreduce-sum of the digits)
Prints one JSON line per mode: generation-loop ms per generation (device
window), launches per generation, GSM share.
"""
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2106_04034_b200 as G  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
gens = int(sys.argv[2]) if len(sys.argv) > 2 else 200
c = bench.CONFIGS[cfgname]
tr = G.make_benchmark_dataset(c["ntr"], c["l"], seed=1)
te = G.make_benchmark_dataset(c["nte"], c["l"], seed=2)
cfg = G.RunConfig(population_size=c["m"], random_trees=c["r"], program_size=c["k"], generations=gens, seed=1)
ref = None
for mode, kw in (("single", dict(devices=None)), ("virtual2", dict(devices=None, virtual_shards=2)),
                 ("threads2", dict(devices=[0, 0]))):
    G.run_evolution(cfg, tr, te, window_start=10, **kw)          # warm the block cache
    res = G.run_evolution(cfg, tr, te, window_start=10, **kw)
    d = res.device
    fp = (res.train_fitness.tobytes(), res.test_fitness.tobytes(), res.elite_train_semantics.tobytes())
    same = ref is None or fp == ref
    ref = ref or fp
    n = gens - 10
    print(json.dumps({"config": cfgname, "mode": mode, "generations_timed": n,
                      "loop_ms_per_generation": d["window_ms"] / n,
                      "launches_per_generation": d["window_loop_launches"] / n,
                      "gsm_launches_per_generation": d["window_gsm_launches"] / n,
                      "bit_identical_to_single": same}))
