"""Probe: interpreter node-evals/s vs feature count at a fixed launch
configuration (GSGP_INTERP_CFG, default 5 = 128x3).  Shared memory per block
grows by 3 KB per feature, so l <= 6 fits 6 blocks (24 warps) per SM and
l = 8 only 5 (20 warps): the ratio tells whether occupancy limits the
interpreter."""
import json
import os
import sys

sys.path.insert(0, ".")
import paper_2106_04034_b200 as G  # noqa: E402

os.environ.setdefault("GSGP_INTERP_CFG", "5")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 400_000
for l in (4, 6, 7, 8):
    tr = G.make_benchmark_dataset(n, l, seed=1)
    te = G.make_benchmark_dataset(n // 4, l, seed=2)
    cfg = G.RunConfig(population_size=1024, random_trees=1024, program_size=1024, generations=0, seed=1)
    best = None
    for _ in range(3):
        res = G.run_evolution(cfg, tr, te)
        d = res.device
        ms = d["init_ms"]["interpret_population"] + d["init_ms"]["interpret_pool"]
        ins = d["program_instructions"]["population"] + d["program_instructions"]["pool"]
        rate = ins * (n + n // 4) / (ms / 1e3)
        best = max(best or 0, rate)
    print(json.dumps({"l": l, "interp_ms": round(ms, 2), "node_evals_per_s": f"{best:.4g}"}))
