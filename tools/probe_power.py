"""Probe: per-generation GSM kernel time vs power/clock over a sustained C3 run."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2106_04034_b200 as G  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c3"
gens = int(sys.argv[2]) if len(sys.argv) > 2 else 200
c = bench.CONFIGS[cfgname]
tr = G.make_benchmark_dataset(c["ntr"], c["l"], seed=1)
te = G.make_benchmark_dataset(c["nte"], c["l"], seed=2)
cfg = G.RunConfig(population_size=c["m"], random_trees=c["r"], program_size=c["k"], generations=gens, seed=1)
smp = bench.ClockSampler(0, period=0.01)
smp.start()
t0 = time.perf_counter()
res = G.run_evolution(cfg, tr, te, time_kernels=True)
summ = smp.summary()
ms = res.device["gsm_ms_per_generation"]
loop_start = t0 + (res.timings.create_population_ms + res.timings.compute_semantics_ms) / 1e3
trace = [(round(s[5] - loop_start, 3), s[0], s[3], round(s[4], 1)) for s in smp.samples if s[5] >= loop_start]
out = {"config": cfgname, "gsm_ms_first10": [round(x, 3) for x in ms[:10]],
       "gsm_ms_by_decile": [round(float(np.mean(ch)), 3) for ch in np.array_split(ms, 10)],
       "gsm_ms_min": float(ms.min()), "gsm_ms_median": float(np.median(ms)), "clocks": summ,
       "trace_t_sm_mem_power": trace[:: max(1, len(trace) // 40)]}
print(json.dumps(out))
