"""Probe: interpreter throughput (run init only) for the C2/C3 population+pool."""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2106_04034_b200 as G  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
c = bench.CONFIGS[cfgname]
tr = G.make_benchmark_dataset(c["ntr"], c["l"], seed=1)
te = G.make_benchmark_dataset(c["nte"], c["l"], seed=2)
cfg = G.RunConfig(population_size=c["m"], random_trees=c["r"], program_size=c["k"], generations=0, seed=1)
out, interp = [], []
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
for rep in range(reps):
    res = G.run_evolution(cfg, tr, te)
    out.append(round(res.timings.compute_semantics_ms, 2))
    im = res.device["init_ms"]
    interp.append(round(im["interpret_population"] + im["interpret_pool"], 2))
print(json.dumps({"config": cfgname, "compute_semantics_ms": out, "interpret_pop_pool_ms": interp,
                  "interpreter": res.device["interpreter"], "train0": float(res.train_fitness[0]),
                  "test0": float(res.test_fitness[0])}))
