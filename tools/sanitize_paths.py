"""Small workload that drives every device kernel of the library once or a
few times, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck on small configs).

    compute-sanitizer --tool memcheck python tools/sanitize_paths.py

Paths: run_evolution with every interpreter configuration (forced through
GSGP_INTERP_CFG), graph replay and direct launches, fp32 and fp64 storage,
two virtual case shards (sharded SSE tail), the operator entry points
(create_population, compute_semantics, compute_fitness, canonical_sum,
build_mutation_plan, gsm, gsm_paired, gsm_step_f32, survive, argmin/argmax,
sigmoid) and replay_lineage.  Sizes are tiny: a sanitizer run of the whole
script takes minutes, not hours.
"""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2106_04034_b200 as G  # noqa: E402

rng = np.random.default_rng(3)


def data(n, l):
    X = rng.uniform(-1, 1, (n, l))
    return G.Dataset(X, X[:, 0] * X[:, 1] + X.sum(axis=1))


tr, te = data(1500, 5), data(700, 5)
cfg = G.RunConfig(population_size=12, random_trees=8, program_size=63, generations=4, seed=2)
ref = G.run_evolution(cfg, tr, te)
for c in ("0", "1", "2", "3", "4", "5", "6", "7", "9", "10"):
    os.environ["GSGP_INTERP_CFG"] = c
    r = G.run_evolution(cfg, tr, te, use_graph=False)
    assert np.array_equal(r.train_fitness, ref.train_fitness), c
del os.environ["GSGP_INTERP_CFG"]
r = G.run_evolution(cfg, tr, te, time_kernels=True)
r = G.run_evolution(cfg, tr, te, virtual_shards=2)
assert np.array_equal(r.train_fitness, ref.train_fitness)
r64 = G.run_evolution(cfg, tr, te, storage="fp64")
wide = G.run_evolution(G.RunConfig(population_size=6, random_trees=4, program_size=40, generations=2, seed=3),
                       data(300, 100), data(100, 100))

# operators
pop = G.create_population(10, cfg, 0, 5)
S = G.compute_semantics(pop, tr.features, cfg)
F = G.compute_fitness(S, tr.target)
G.canonical_sum(S, 3)
plan = G.build_mutation_plan(10, 8, cfg, 1)
T = G.sigmoid_array(G.compute_semantics(G.create_population(8, cfg, 10, 5), tr.features, cfg))
O = G.gsm(S, T, plan, cfg)
G.gsm_paired(S[:, :1000], S[:, 1000:], T[:, :1000], T[:, 1000:], plan, cfg)
P32 = S.astype(np.float32)
Q32 = T.astype(np.float32)
G.gsm_step_f32(P32[:, :1000], P32[:, 1000:], Q32[:, :1000], Q32[:, 1000:], tr.target[:1000], tr.target[1000:], plan)
G.argmin_fitness(F)
G.argmax_fitness(F)
from paper_2106_04034_b200 import ops  # noqa: E402
ops.survive_decision(F, G.compute_fitness(O, tr.target))
G.sigmoid(0.3)
G.uniform_array(1, 2, np.arange(100, dtype=np.uint64))

# replay of a run's lineage from its initial semantics
r = G.run_evolution(cfg, tr, te, storage="fp64")
G.replay_lineage(r.lineage, G.compute_semantics(G.create_population(12, cfg, 0, 5), tr, cfg),
                 G.compute_semantics(G.create_population(8, cfg, 12, 5), tr, cfg), cfg)
print("sanitize paths ok")
