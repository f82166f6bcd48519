import time, sys
sys.path.insert(0, '.')
t0=time.perf_counter()
import paper_2106_04034_b200 as G
cfg = G.RunConfig(population_size=64, random_trees=64, program_size=127, generations=2, seed=1)
tr, te = G.make_benchmark_dataset(2048, 4, seed=1), G.make_benchmark_dataset(512, 4, seed=2)
t1=time.perf_counter()
for k in (127, 1023, 2047, 127):
    r = G.run_evolution(G.RunConfig(population_size=64, random_trees=64, program_size=k, generations=2, seed=1), tr, te)
    t2=time.perf_counter()
    print("k", k, "wall ms", round((t2-t1)*1e3,1), "compute_semantics ms", round(r.timings.compute_semantics_ms,2)); t1=t2
