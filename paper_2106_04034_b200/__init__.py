"""B200-native GSGP engine: drop-in for the hot path of the reference `gsgp`.

The public names mirror the reference package (`gsgp/__init__.py:12-62`) for
the path this engine owns — the counter RNG, CreatePopulation, the genome
interpreter, fitness, the mutation plan, geometric semantic mutation,
survival and `run_evolution` — and every one of them runs on the B200
through `libgsgp_b200.so`.  Importing the package does not touch the GPU;
the first compute call loads the library and fails loudly if it is missing.
"""

from .backend import BackendDescriptor, get_backend
from .core import (
    BACKENDS, WORST_FITNESS, Chromosome, ConfigError, Dataset, DatasetFormatError, EliteRecord,
    FunctionOp, Gene, GeneTag, GsgpError, LineageEntry, LineageError, LineageLog, MutationPlan,
    Population, RunConfig, RunStats, StageTimings,
)
from .engine import GenerationState, RunResult, replay_lineage, run_evolution, survive
from .ops import (
    argmax_fitness, argmin_fitness, build_mutation_plan, canonical_sum, compute_fitness, compute_semantics,
    create_population, derive_seed, gsm, gsm_paired, gsm_step_f32, interpret,
    release_device_memory, rmse, rng_bits, rng_stream, sample_gene, sigmoid, sigmoid_array,
    uniform_array,
)
from .harness import make_benchmark_dataset, sweep, timed_run
from .runs import RunSummary, assign_runs, run_many, run_seeds
from .io_cli import (
    load_config, load_dataset, read_lineage_sidecar, run_cli, write_dataset,
    write_lineage_sidecar, write_traces,
)

__version__ = "0.1.0"
