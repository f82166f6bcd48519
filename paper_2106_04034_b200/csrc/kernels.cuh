// Launchers for the sm_100a kernels.  All launchers are asynchronous on the
// given stream and throw gsgp::Error on launch failure.
#pragma once

#include "common.cuh"

namespace gsgp {

// ------------------------------------------------------------ rng / genomes
void launch_rng_draw(uint64_t seed, uint64_t stream, const uint64_t* counters, int64_t n,
                     uint64_t* bits, double* units, cudaStream_t s);

struct GeneParams {
  uint64_t seed;
  double thr_fun;        // p_fun
  double thr_feat;       // p_fun + p_feat
  double erc_low, erc_high;
  int32_t n_features;
  int32_t k;
};
// gene (i, j) of streams [stream_base, stream_base + count)
void launch_create_population(const GeneParams& p, int64_t count, uint64_t stream_base,
                              uint8_t* tags, int32_t* codes, double* consts, cudaStream_t s);

// ------------------------------------------------------------ plan
struct PlanParams {
  uint64_t seed;
  int64_t m, r;
  int32_t ms_uniform;
  double ms_const;
};
// slot i of a generation's plan (gsgp/mutation.py:37-62): counters 3i, 3i+1,
// 3i+2 of stream 2^32+gen (key); u uniform over [0, r), v uniform over the
// other r-1 indices, ms = 1 - U or the constant step.  All conversions are
// the reference's fp64 product + truncation.
#ifdef __CUDACC__
__device__ __forceinline__ void plan_slot(uint64_t key, int64_t i, int64_t r, int32_t ms_uniform,
                                          double ms_const, int64_t* pu, int64_t* pv, double* pms) {
  const uint64_t c = 3ull * (uint64_t)i;
  int64_t a = (int64_t)__dmul_rn(draw_unit(key, c), (double)r);
  a = a < r - 1 ? a : r - 1;
  int64_t b = (int64_t)__dmul_rn(draw_unit(key, c + 1), (double)(r - 1));
  b = b < r - 2 ? b : r - 2;
  b += (b >= a);
  *pu = a;
  *pv = b;
  *pms = ms_uniform ? __dsub_rn(1.0, draw_unit(key, c + 2)) : ms_const;
}
#endif
// plan for generation `gen` (explicit) or, when gen_ptr != nullptr, for
// generation *gen_ptr read on device (graph-replayable)
void launch_plan(const PlanParams& p, int64_t gen, const int64_t* gen_ptr, int64_t* u, int64_t* v,
                 double* ms, int64_t stride_per_gen, cudaStream_t s);

// ------------------------------------------------------------ compile + interpret
struct Program {
  Ins* code;            // [count][k+1] abstract instructions (k_compile)
  Ins* exe;             // [count][k+1] linked for the launch configuration (k_link)
  int32_t* len;         // [count] instructions
  int32_t* nconst;      // [count] constant-table entries
  double* ctab;         // [count][k] constants referenced by the program
  int32_t* maxima;      // [4] {spill depth, constants, instructions, unused}: max over genomes
  int32_t* scratch;     // [count][4*k] ints
  uint8_t* flags;       // [count][k]
  double* cval;         // [count][k]
  int32_t* ndiv;        // [count][4] op mix (divisions, vector / constant operand loads, spill stores), or null
};
// maxima[] must be zero before the launch (launch_compile clears it)
void launch_compile(const uint8_t* tags, const int32_t* codes, const double* consts, int64_t count,
                    int32_t k, double eps, Program prog, cudaStream_t s);

enum InterpMode : int { INTERP_F64 = 0, INTERP_POP = 1, INTERP_POOL = 2 };
// linked-program scratch of the interpreter launches (relinked per launch):
// `copies` group copies of `count` programs with stride k1 = maxlen + 1
// (callers that allocate before compiling pass maxlen = k), at least 2, at
// most 32, and within ~1 GiB beyond 2
struct LinkedLayout { int64_t k1, ins; int32_t copies; };
inline LinkedLayout linked_layout(int64_t count, int32_t maxlen) {
  LinkedLayout L;
  L.k1 = (maxlen > 0 ? maxlen : 1) + 1;
  const int64_t per = count * L.k1 * 16;
  int64_t c = ((int64_t)1 << 30) / (per > 0 ? per : 1);
  L.copies = (int32_t)(c < 2 ? 2 : (c > 32 ? 32 : c));
  L.ins = L.copies * count * L.k1;
  return L;
}

struct InterpArgs {
  const Ins* code;          // abstract program (count genomes, stride k1)
  Ins* exe;                 // linked copies, rewritten by every launch_interpret (scratch)
  int64_t exe_gstride;      // set by the launch: elements between the per-group linked copies
  int64_t exe_k1;           // linked-program stride per genome (>= maxlen + 1)
  int32_t max_groups;       // linked copies exe holds: max_groups * count * exe_k1 Ins
  const int32_t* len;
  const int32_t* nconst;
  const double* ctab;       // [count][k1 - 1]
  int64_t k1;               // instruction stride per genome (k + 1)
  int64_t count;            // genomes
  int32_t maxdepth, maxconst, maxlen;   // Program::maxima, read back once after compile
  const double* XT;         // [l][xt_pitch] fp64, feature-major: cases q_base .. q_base+nq-1
  int64_t xt_pitch;
  int32_t l;
  int64_t ntr, nte;         // shard case counts (stacked index q < ntr is train)
  int64_t te_q;             // stacked index of test case 0 (>= ntr; [ntr, te_q) is a skipped
                            // gap so the test cases start on a tile: canonical SSE partials)
  int64_t q_base, nq;       // this launch: stacked cases [q_base, q_base + nq) (q_base % tile == 0)
  int64_t part_ntiles;      // row stride of part[] (tiles over all te_q + nte stacked cases)
  double eps;
  // outputs
  double* out64;            // INTERP_F64: [count][ntr+nte]
  void* out;                // INTERP_POP/POOL: [count][pitch] float or double
  int32_t out_is_f64;
  int64_t pitch;            // storage pitch (elements)
  int64_t test_off;         // test case j stored at test_off + j (j < te_full) ...
  int64_t te_full;
  int64_t tail_off;         // ... else at tail_off + (j - te_full) (RowLayout)
  const double* y;          // targets in storage layout (INTERP_POP)
  double* part;             // [count][ntiles][2] SSE partials (INTERP_POP)
  int32_t* wide;            // [count] bit0 train overflowed fp32, bit1 test (INTERP_POP)
  unsigned long long* nonfinite;   // element count replaced by 0.0
  int32_t raw;              // INTERP_F64 only: keep non-finite values (scalar interpret)
};
// case tiles over all te_q + nte stacked cases (the part[] row stride) and the tile size
int64_t interp_tiles(const InterpArgs& a, int* tile_out);
// launch configuration index the interpreter takes for these arguments (a
// function of shared memory only: the same on every rank and every run)
int interp_config(const InterpArgs& a);
void launch_interpret(const InterpArgs& a, int mode, cudaStream_t s);

// ------------------------------------------------------------ storage rows
// One shard's semantics row (pitch elements, fp32 or fp64): the train cases
// [0, ntr) (region padded to ntr_pad), then the test cases.  Generation
// units are `tile`-case tiles anchored on the train region and on the test
// region separately.  When the partial train tail and the partial test tail
// fit in one tile together, the test tail is stored right after the train
// region — [train | test tail | full test tiles] — so the two tails form ONE
// contiguous unit (gsm.cu unit_span); otherwise [train | test].  Test case j
// lives at test_off + j for j < te_full, else at tail_off + (j - te_full).
struct RowLayout {
  int64_t ntr, nte;
  int64_t ntr_pad;          // train region [0, ntr_pad), zero padded
  int64_t tail_off;         // relocated test tail (-1: none), tail_pad elements
  int64_t tail_pad;
  int64_t te_full;          // test cases stored from test_off on
  int64_t test_off;
  int64_t pitch;
  int64_t tile, ttr, tte, ntiles;   // units per row: ttr train units (the last may carry the test tail) + tte
};
RowLayout make_layout(int64_t ntr, int64_t nte, bool f64, bool allow_merge = true);
__host__ __device__ inline int64_t test_col(const RowLayout& L, int64_t j) {
  return j < L.te_full ? L.test_off + j : L.tail_off + (j - L.te_full);
}

// ------------------------------------------------------------ generation
struct GsmArgs {
  const void* pool;         // [r][pitch] squashed trees (float or double)
  void* S;                  // [m][pitch] semantics, updated in place
  const void* elite_prev;   // [pitch] saved parent elite row (redirect target)
  void* elite_cur;          // [pitch] parent row b_p is saved here
  const double* y;          // [pitch] targets in storage layout (0 in padding)
  RowLayout lay;            // storage row layout (units, pitch)
  int64_t m;
  const int64_t* u;         // plan of this generation (or base when gen_ptr != nullptr)
  const int64_t* v;
  const double* ms;
  const int64_t* ctl;       // device control block (see engine.cu), may be nullptr
  int32_t sign;             // 0 minus, 1 plus
  double* part;             // [m][lay.ntiles][2]
  int32_t* emax;            // optional [m][2]: atomicMax of the partials' canon_exp (fused tail);
                            // must hold kExpZero before the launch (the reduce resets it)
  unsigned long long* nonfinite;   // operator mode only
  // {ticket, exited CTAs}: dynamic unit dispatch; zero before the first
  // launch, the last CTA to exit re-zeroes both for the next launch
  unsigned long long* ticket;
  // inline mutation plan (gsgp/mutation.py:37-62): when plan_inline, the
  // producer draws (u, v, ms) of each row itself from the counter RNG and,
  // if write_plan, records them for the lineage into u/v/ms[(gen-1)*m + i]
  int32_t plan_inline;
  int32_t write_plan;
  PlanParams plan;
};
int64_t gsm_tile_cases(bool f64);
void launch_gsm(const GsmArgs& a, bool f64, bool operator_mode, cudaStream_t s);
// SSE of the stored semantics S against y in the generation kernel's exact
// order (no mutation, no stores): part[m][ntiles][2]
void launch_sse_only(const GsmArgs& a, bool f64, cudaStream_t s);
// mode 0 engine, 1 operator (non-finite -> 0), 2 SSE only
void launch_gsm_mode(const GsmArgs& a, bool f64, int mode, cudaStream_t s);

// Canonical SSE (common.cuh canon_*): part[rows][ntiles][2] -> out[rows][2],
// a function of the multiset of tile partials only.  Single part:
void launch_reduce_partials(const double* part, int64_t rows, int64_t ntiles, double* out, cudaStream_t s);
// Several parts (shards, ranks): clear; exp of every part (atomicMax into
// emax[rows][2]); [allreduce max]; digits of every part (atomicAdd into
// digits[rows][2][kLimbs]); [allreduce sum]; finish.
void launch_canon_clear(int64_t rows, int32_t* emax, unsigned long long* digits, cudaStream_t s);
void launch_canon_exp(const double* part, int64_t rows, int64_t ntiles, int32_t* emax, cudaStream_t s);
void launch_canon_digits(const double* part, int64_t rows, int64_t ntiles, const int32_t* emax,
                         unsigned long long* digits, cudaStream_t s);
void launch_canon_finish(const int32_t* emax, const unsigned long long* digits, int64_t rows, double* sse,
                         cudaStream_t s);

// fp64 operator RMSE per row of a dense [m][n] matrix (fitness.py:28-51)
void launch_row_rmse(const double* S, const double* y, int64_t m, int64_t n, double* out,
                     cudaStream_t s);

struct SurviveArgs {
  int64_t m;
  double ntr, nte;
  const double* sse_off;    // [m][2] offspring SSE (train, test), already exchanged
  const double* sse_alt;    // init only: [m][2] fp64-interpreter SSE, used for fp32-overflow slots
  double* F;                // [m] state train fitness (in: parent, out: next)
  double* TS;               // [m] state test SSE
  int32_t* wide;            // [m] slot flags
  int64_t* ctl;             // control block
  // lineage record for this generation (index = ctl[CTL_GEN])
  int8_t* rec_src; int64_t* rec_idx; int64_t* rec_slot; double* rec_fit;
  double* trace_tr; double* trace_te;
};
// per-row canonical SSE into sse (== a.sse_off) fused with survival (single
// shard, single rank); emax = the anchors the GSM launch accumulated (reset
// to kExpZero here; unused when ntiles == 1: the SSE is the partial itself);
// `done` is a zeroed counter, re-zeroed on exit
void launch_reduce_survive(const double* part, int64_t ntiles, int32_t* emax, double* sse,
                           const SurviveArgs& a, unsigned int* done, cudaStream_t s);
// multi-shard / multi-rank tail: sse = canon_finish(digits, emax) per (row,
// train|test), emax re-armed to kExpZero and digits zeroed for the next
// generation, then survival in the last block (`done` as above)
void launch_finish_survive(int32_t* emax, unsigned long long* digits, double* sse, const SurviveArgs& a,
                           unsigned int* done, cudaStream_t s);
// initial elite: fitness from SSE, argmin, trace[0] (evolution.py:132-143)
void launch_init_state(const SurviveArgs& a, cudaStream_t s);
// decision only, for the operator API: out = {src, idx, slot}
void launch_survive_decision(const double* fp, const double* fo, int64_t m, int64_t* out,
                             cudaStream_t s);

// np.argmin / np.argmax of a vector: out = {argmin, argmax}
void launch_argminmax(const double* f, int64_t m, int64_t* out, cudaStream_t s);
// elementwise fp64 sigmoid (mutation.py:32-34)
void launch_sigmoid(const double* x, int64_t n, double* y, cudaStream_t s);

// load the engine's interpreter / generation kernels into the current
// device's context ahead of a run (CUDA lazy module loading)
void interp_preload();
void gsm_preload();

}  // namespace gsgp
