/*
 * gsgp_b200.h — C ABI of the B200-native GSGP engine (libgsgp_b200.so).
 *
 * Drop-in boundary for the hot path of the reference package `gsgp` 0.1.0
 * (/root/reference/pkg/src/gsgp, cited as gsgp/X.py:N).  Every entry point
 * replaces one reference function; the Python package
 * `paper_2106_04034_b200` binds them with ctypes and mirrors the reference's
 * Python signatures, argument meaning and exceptions.
 *
 * Conventions
 *   - Return 0 on success; GSGP_ERR_* otherwise, with a thread-local message
 *     from gsgp_last_error().  Python maps 1 -> ConfigError, others -> GsgpError.
 *   - All pointers are HOST pointers owned by the caller and pre-sized; the
 *     library owns all device memory.  Matrices are row-major, C-contiguous.
 *   - Not re-entrant: one call at a time per process.  Multi-GPU runs shard
 *     the fitness cases either across processes (one per GPU, gsgp_comm_init)
 *     or across the devices of one process (gsgp_init).
 *   - There is no CPU fallback: without a CUDA device every compute entry
 *     point fails with GSGP_ERR_CUDA.
 */
#ifndef GSGP_B200_H
#define GSGP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSGP_OK 0
#define GSGP_ERR_CONFIG 1
#define GSGP_ERR_CUDA 2
#define GSGP_ERR_NCCL 3
#define GSGP_ERR_OOM 4

/* Mirrors RunConfig (gsgp/core.py:288-336) minus the CPU-backend knobs. */
typedef struct gsgp_config {
  int64_t population_size;      /* m */
  int64_t random_trees;         /* r */
  int64_t program_size;         /* k */
  int64_t generations;          /* g */
  uint64_t seed;                /* two's complement of the Python int */
  double p_function, p_feature, p_constant;   /* renormalised as core.py:338-342 */
  double erc_low, erc_high;
  int32_t mutation_step_uniform; /* 1: ms = 1 - U[0,1) (mutation.py:48-50) */
  int32_t gsm_sign;              /* 0 "minus", 1 "plus" */
  double mutation_step;          /* constant step when !mutation_step_uniform */
  double division_eps;
  int32_t storage_f64;           /* 0: fp32 semantic storage (default; see storage_f64_used); 1: fp64 */
  int32_t use_graph;             /* 1: replay one captured generation as a CUDA graph */
  int32_t time_kernels;          /* 1: CUDA events around every GSM launch */
  int32_t virtual_shards;        /* case shards per process on its device (>= 1) */
  int64_t window_start;          /* timing window = generations window_start+1 .. g */
} gsgp_config;

/* Outputs of gsgp_run; index 0 of the per-generation arrays is the initial
 * population (evolution.py:138-143), index t the elite after generation t. */
typedef struct gsgp_outputs {
  double* train_trace;           /* [g+1] elite train RMSE */
  double* test_trace;            /* [g+1] same individual's test RMSE */
  int8_t* elite_src;             /* [g+1] 0 parent, 1 offspring, 2 initial */
  int64_t* elite_idx;            /* [g+1] index in the source population */
  int64_t* elite_slot;           /* [g+1] slot in the surviving population */
  double* elite_fit;             /* [g+1] */
  int64_t* plan_u;               /* [g][m] or NULL */
  int64_t* plan_v;               /* [g][m] or NULL */
  double* plan_ms;               /* [g][m] or NULL */
  double* elite_train_semantics; /* [n_train]; this rank's case slice is filled */
  double* gsm_ms;                /* [g] per-generation GSM kernel ms (time_kernels) or NULL */
  int64_t overflow;              /* out: non-finite replacements (RunStats) */
  int64_t shard_train_lo;        /* out: this rank's train case slice */
  int64_t shard_train_hi;
  double stage_ms[20];           /* out: 0 create, 1 semantics, 2 evolution, 3 per_generation,
                                    4 total (host), 5 gsm_kernel_ms_sum, 6 gsm_launches,
                                    7 loop_launches, 8 window_ms, 9 window_gsm_ms,
                                    10 window_gsm_launches, 11 window_loop_launches,
                                    12 upload (H2D + transpose), 13 interpret population,
                                    14 interpret pool, 15 initial SSE (sums over shards),
                                    16 genome compile, 17 device allocation + clears (host
                                    clock), 18 / 19 total compiled instructions (counts, not ms)
                                    of the population / random-tree programs */
  int64_t storage_f64_used;      /* out: 1 if the semantics were stored in fp64 (requested, or
                                    forced by a constant mutation step large enough to leave
                                    fp32 range: step * (1 minus | 2 plus) * g >= 2^70) */
  int64_t interp_info[4];        /* out: interpreter launch configuration, and the compiled
                                    programs' max spill depth, constants, instructions */
  int64_t interp_div[2];         /* out: protected-division instructions of the compiled
                                    population / random-tree programs (fp64 op mix) */
  int64_t interp_ops[6];         /* out: operand traffic of the compiled population (0-2) /
                                    random-tree (3-5) programs: per-case operand loads
                                    (feature and spill rows), constant operand loads, spill
                                    stores (the interpreter's shared-memory roofline) */
} gsgp_outputs;

const char* gsgp_version(void);
const char* gsgp_last_error(void);

/* device count, SM count and name of the current device */
int gsgp_device_info(int* device_count, int* sm_count, char* name, int name_len);
/* one device per process from now on (clears a gsgp_init device set) */
int gsgp_set_device(int device);

/* Single-process multi-GPU (replaces the reference's worker pool behind
 * run_evolution: gsgp/evolution.py:115, gsgp/backend.py:94-130 — one call
 * uses every listed device).  After gsgp_init(n, ids) with n > 1, each
 * gsgp_run drives the n devices from one host thread per device: the cases
 * are sharded by device exactly as across processes, and the per-generation
 * canonical-SSE collectives run over an NCCL communicator created with
 * ncclCommInitAll.  Results are bit-identical to a one-device run.  A list
 * that names a device twice (or GSGP_THREAD_EXCHANGE=1) uses a host thread
 * exchange instead of NCCL (tests on one GPU).  n = 1 selects that device.
 * Cannot be combined with gsgp_comm_init* (one process per GPU). */
int gsgp_init(int n_dev, const int* dev_ids);
/* destroy the device set's communicators; gsgp_run is single-device again */
int gsgp_finalize(void);
/* devices the next gsgp_run drives (0 = the current device, no set) */
int gsgp_device_count_in_use(void);
/* Return the engine's cached device memory (a run parks its device blocks
   for the next run instead of freeing them) and its pinned upload staging
   to the driver.  No reference
   counterpart: the reference allocates with numpy per call. */
int gsgp_trim_device_memory(void);

/* rng_bits / uniform_array (gsgp/rng.py:43-64); either output may be NULL */
int gsgp_rng_draw(uint64_t seed, uint64_t stream, const uint64_t* counters, int64_t n,
                  uint64_t* bits, double* units);
/* derive_seed (gsgp/rng.py:67-69); host-only, needs no device */
uint64_t gsgp_derive_seed(uint64_t seed, uint64_t index);

/* create_population (gsgp/population.py:73-92) */
int gsgp_create_population(const gsgp_config* cfg, int64_t count, uint64_t stream_base,
                           int32_t n_features, uint8_t* tags, int32_t* codes, double* consts);

/* compute_semantics (gsgp/interpreter.py:122-148): out[count][n] fp64,
 * overflow += non-finite replacements.  replace_nonfinite = 0 returns raw
 * values instead (the scalar `interpret`, interpreter.py:45-75). */
int gsgp_compute_semantics(const uint8_t* tags, const int32_t* codes, const double* consts,
                           int64_t count, int64_t k, const double* X, int64_t n, int32_t l,
                           double eps, int32_t replace_nonfinite, double* out,
                           int64_t* overflow);

/* compute_fitness (gsgp/fitness.py:28-51): out[m] RMSE, non-finite -> +inf */
int gsgp_compute_fitness(const double* S, const double* target, int64_t m, int64_t n,
                         double* out);

/* build_mutation_plan (gsgp/mutation.py:37-62) */
int gsgp_build_mutation_plan(int64_t m, int64_t r, uint64_t seed, int64_t generation,
                             int32_t ms_uniform, double ms_const, int64_t* u, int64_t* v,
                             double* ms);

/* gsm / _gsm_squashed (gsgp/mutation.py:65-94), fp64: squashed=0 applies the
 * sigmoid to `trees` first.  overflow += non-finite replacements. */
int gsgp_gsm(const double* parent, int64_t m, int64_t n, const double* trees, int64_t r,
             const int64_t* u, const int64_t* v, const double* ms, int32_t sign,
             int32_t squashed, double* out, int64_t* overflow);

/* replay_lineage (gsgp/evolution.py:182-202) on the device: the initial
 * semantics [m][n] and the raw tree semantics [r][n] are uploaded once, the
 * g plans (u, v, ms: [g][m]) once, the trees squashed once, then every
 * generation's fp64 GSM (mutation.py:65-94) and parent-elite restore run on
 * the device; out[n] = the final elite row (slot final_slot).  elite_src: 0
 * parent, 1 offspring, per generation. */
int gsgp_replay(const double* initial, int64_t m, int64_t n, const double* trees, int64_t r, int64_t g,
                const int64_t* u, const int64_t* v, const double* ms, const int8_t* elite_src,
                const int64_t* elite_idx, const int64_t* elite_slot, int64_t final_slot, int32_t sign,
                double* out);

/* The engine's fused fp32 generation step on explicit inputs (kernel-level
 * parity): offspring (fp32, in the engine's rounding) and per-row fp64 SSE. */
int gsgp_gsm_step_f32(const float* parent_tr, const float* parent_te, const float* sq_tr,
                      const float* sq_te, int64_t m, int64_t r, int64_t ntr, int64_t nte,
                      const double* ytr, const double* yte, const int64_t* u, const int64_t* v,
                      const double* ms, int32_t sign, float* out_tr, float* out_te,
                      double* sse_tr, double* sse_te);

/* survive decision (gsgp/evolution.py:65-83): dec = {src (0 parent,
 * 1 offspring), index, slot} */
int gsgp_survive(const double* fit_parent, const double* fit_offspring, int64_t m, int64_t* dec);

/* sigmoid_array (gsgp/mutation.py:32-34), fp64 */
int gsgp_sigmoid(const double* x, int64_t n, double* out);

/* argmin_fitness / argmax_fitness (gsgp/evolution.py:36-47): out = {argmin,
 * argmax}, ties to the lowest index */
int gsgp_argminmax(const double* fitness, int64_t m, int64_t* out);

/* The engine's canonical SSE sum of non-negative fp64 partials (the
 * reduction behind every fitness of gsgp_run; no reference counterpart —
 * replaces the row sums of gsgp/fitness.py:23 across tiles and ranks):
 * out[i] = sum_j x[i][j], rounded once from an exact fixed-point sum
 * anchored on the row's largest exponent, so the result does not depend on
 * the order or grouping of the x[i][j].  parts = 0 runs the fused
 * single-shard path, parts >= 1 splits the columns into that many pieces
 * and runs the multi-shard path (anchors, digits, finish). */
int gsgp_canonical_sum(const double* x, int64_t rows, int64_t n, int32_t parts, double* out);

/* run_evolution (gsgp/evolution.py:100-179) */
int gsgp_run(const gsgp_config* cfg, const double* Xtr, const double* ytr, int64_t ntr,
             const double* Xte, const double* yte, int64_t nte, int32_t n_features,
             gsgp_outputs* out);

/* Multi-GPU: one process per GPU.  Rank 0 creates the id, every rank calls
 * gsgp_comm_init with it; gsgp_run then shards the cases across ranks
 * (slices aligned to 12288 cases) and allreduces each generation the rows'
 * canonical-SSE anchors (int32 max) and digit sums (uint64 sum) over NCCL:
 * results are bit-identical for any number of ranks. */
int gsgp_comm_unique_id(unsigned char id[128]);
int gsgp_comm_init(int world, int rank, const unsigned char id[128]);
/* Test transport for the same collectives: `allreduce` reduces a HOST
   buffer of `count` elements over the ranks in place (e.g. torch.distributed
   over gloo); dtype 0 = fp64 sum, 1 = int32 sum, 2 = uint64 sum, 3 = int32
   max.  The multi-rank engine path then runs with several processes sharing
   one GPU.  Runs use direct launches (no graph) in this mode. */
int gsgp_comm_init_host(int world, int rank, void (*allreduce)(void* buf, int64_t count, int32_t dtype));
int gsgp_comm_destroy(void);
/* contiguous case slice [lo, hi) of shard `index` out of `count`; interior
 * boundaries are multiples of 12288 cases (the canonical SSE tile grid) */
void gsgp_shard_range(int64_t n, int64_t count, int64_t index, int64_t* lo, int64_t* hi);

#ifdef __cplusplus
}
#endif

#endif /* GSGP_B200_H */
