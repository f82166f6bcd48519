// Small kernels of the hot path: counter RNG, CreatePopulation, mutation plan,
// deterministic reductions, RMSE and elitist survival.
//
// Reference citations: gsgp/X.py:N means /root/reference/pkg/src/gsgp/X.py:N.
#include "kernels.cuh"

namespace gsgp {

namespace {

constexpr int kThreads = 256;

inline unsigned blocks_for(int64_t n, int threads = kThreads) {
  int64_t b = (n + threads - 1) / threads;
  return (unsigned)(b < 1 ? 1 : b);
}

inline void check_launch() { GSGP_CUDA(cudaGetLastError()); }

// ---------------------------------------------------------------- rng
__global__ void k_rng_draw(uint64_t key, const uint64_t* __restrict__ counters, int64_t n,
                           uint64_t* bits, double* units) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t b = draw_bits(key, counters[i]);
  if (bits) bits[i] = b;
  if (units) units[i] = (double)(b >> 11) * 0x1p-53;
}

// --------------------------------------------------- CreatePopulation
// gsgp/population.py:47-70: gene (i, j) uses stream base+i, counter 2j for the
// tag and 2j+1 for the payload; non-owning fields are zero.
__global__ void k_create_population(GeneParams p, int64_t count, uint64_t stream_base,
                                    uint8_t* __restrict__ tags, int32_t* __restrict__ codes,
                                    double* __restrict__ consts) {
  int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gid >= count * (int64_t)p.k) return;
  int64_t i = gid / p.k;
  uint64_t j = (uint64_t)(gid - i * p.k);
  uint64_t key = stream_key(p.seed, stream_base + (uint64_t)i);
  double d_tag = draw_unit(key, 2 * j);
  double d_pay = draw_unit(key, 2 * j + 1);
  uint8_t tag;
  int32_t code = 0;
  double c = 0.0;
  if (d_tag < p.thr_fun) {
    tag = TAG_FUNCTION;
    int32_t op = (int32_t)__dmul_rn(d_pay, 4.0);          // population.py:64
    code = op < 3 ? op : 3;
  } else if (d_tag < p.thr_feat) {
    tag = TAG_FEATURE;
    int32_t f = (int32_t)__dmul_rn(d_pay, (double)p.n_features);   // population.py:65
    code = f < p.n_features - 1 ? f : p.n_features - 1;
  } else {
    tag = TAG_CONSTANT;                                    // population.py:70
    c = __dadd_rn(p.erc_low, __dmul_rn(d_pay, __dsub_rn(p.erc_high, p.erc_low)));
  }
  tags[gid] = tag;
  codes[gid] = code;
  consts[gid] = c;
}

// ---------------------------------------------------------------- plan
// gsgp/mutation.py:37-62: stream 2^32 + gen, slot i draws counters 3i, 3i+1,
// 3i+2; u uniform over [0, r), v uniform over the other r-1 indices.
__global__ void k_plan(PlanParams p, int64_t gen, const int64_t* gen_ptr, int64_t* u, int64_t* v,
                       double* ms, int64_t stride) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= p.m) return;
  int64_t g = gen_ptr ? gen_ptr[CTL_GEN] : gen;
  int64_t off = gen_ptr ? (g - 1) * stride : 0;
  const uint64_t key = stream_key(p.seed, kPlanStream0 + (uint64_t)g);
  plan_slot(key, i, p.r, p.ms_uniform, p.ms_const, u + off + i, v + off + i, ms + off + i);
}

// ------------------------------------------------------- reductions
// Canonical SSE of part[row][tile][2] (common.cuh): one warp per row.  The
// anchors are the exact max partial exponents; the digit sums are exact.
__device__ __forceinline__ int2 warp_row_exp(const double* __restrict__ p, int64_t ntiles, int lane) {
  int32_t ex = kExpZero, ez = kExpZero;
  for (int64_t t = lane; t < ntiles; t += 32) {
    const double2 v = *reinterpret_cast<const double2*>(p + 2 * t);
    ex = max(ex, canon_exp(v.x));
    ez = max(ez, canon_exp(v.y));
  }
  return make_int2(__reduce_max_sync(0xffffffffu, ex), __reduce_max_sync(0xffffffffu, ez));
}

// per-row digit sums (train L[0..3], test L[4..7]), complete in every lane
__device__ __forceinline__ void warp_row_digits(const double* __restrict__ p, int64_t ntiles, int lane,
                                                int2 A, unsigned long long L[2 * kLimbs]) {
#pragma unroll
  for (int d = 0; d < 2 * kLimbs; ++d) L[d] = 0;
  const bool fx = A.x < kExpInf, fz = A.y < kExpInf;
  for (int64_t t = lane; t < ntiles; t += 32) {
    const double2 v = *reinterpret_cast<const double2*>(p + 2 * t);
    if (fx) canon_add(v.x, A.x, L);
    if (fz) canon_add(v.y, A.y, L + kLimbs);
  }
#pragma unroll
  for (int d = 0; d < 2 * kLimbs; ++d)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) L[d] += __shfl_xor_sync(0xffffffffu, L[d], o);
}

__device__ __forceinline__ void warp_row_sse(const double* __restrict__ part, int64_t ntiles, int64_t row,
                                             double* __restrict__ sse) {
  const int lane = threadIdx.x & 31;
  const double* p = part + row * ntiles * 2;
  const int2 A = warp_row_exp(p, ntiles, lane);
  unsigned long long L[2 * kLimbs];
  warp_row_digits(p, ntiles, lane, A, L);
  if (lane == 0) {
    sse[2 * row] = canon_finish(L, A.x);
    sse[2 * row + 1] = canon_finish(L + kLimbs, A.y);
  }
}

// the fused generation tail: anchors come from the GSM launch (emax), which
// is reset to kExpZero for the next generation once read
template <int kPer>
__device__ __forceinline__ void warp_row_sse_anchored(const double* __restrict__ part, int64_t ntiles,
                                                      int64_t row, int32_t* emax, double* __restrict__ sse) {
  const int lane = threadIdx.x & 31;
  const double* p = part + row * ntiles * 2;
  // groups of kPer strided loads in flight per lane (1 for rows of <= 32
  // units, else 8); the first group is issued before the anchor load, so the
  // latencies overlap
  auto load = [&](int64_t t0, double2* v) {
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int64_t t = t0 + 32 * j;
      v[j] = t < ntiles ? *reinterpret_cast<const double2*>(p + 2 * t) : make_double2(0.0, 0.0);
    }
  };
  double2 v[kPer];
  load(lane, v);
  const int2 A = *reinterpret_cast<const int2*>(emax + 2 * row);
  __syncwarp();
  if (lane == 0) *reinterpret_cast<int2*>(emax + 2 * row) = make_int2(kExpZero, kExpZero);
  unsigned long long L[2 * kLimbs];
#pragma unroll
  for (int d = 0; d < 2 * kLimbs; ++d) L[d] = 0;
  const bool fx = A.x < kExpInf, fz = A.y < kExpInf;
  for (int64_t t0 = lane;;) {
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      if (fx) canon_add(v[j].x, A.x, L);
      if (fz) canon_add(v[j].y, A.y, L + kLimbs);
    }
    t0 += 32 * kPer;
    if (t0 - lane >= ntiles) break;
    load(t0, v);
  }
#pragma unroll
  for (int d = 0; d < 2 * kLimbs; ++d)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) L[d] += __shfl_xor_sync(0xffffffffu, L[d], o);
  if (lane < 2) sse[2 * row + lane] = canon_finish(lane ? L + kLimbs : L, lane ? A.y : A.x);   // train | test
}

// one 256-thread block per row, for long rows (C3: ~3000 tiles): the same
// anchors and exact digit sums as warp_row_sse, 8x the loads in flight
__device__ void block_row_sse(const double* __restrict__ part, int64_t ntiles, int64_t row,
                              int32_t* emax, double* __restrict__ sse) {
  __shared__ int2 sh_a;
  __shared__ unsigned long long sh_d[8][2 * kLimbs];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const double* p = part + row * ntiles * 2;
  // groups of 4 strided loads in flight per thread; the first group is
  // issued before the anchor handshake
  constexpr int kGrp = 4;
  auto load = [&](int64_t t0, double2* v) {
#pragma unroll
    for (int j = 0; j < kGrp; ++j) {
      const int64_t t = t0 + 256 * j;
      v[j] = t < ntiles ? *reinterpret_cast<const double2*>(p + 2 * t) : make_double2(0.0, 0.0);
    }
  };
  double2 v[kGrp];
  load(tid, v);
  if (tid == 0) {
    sh_a = *reinterpret_cast<int2*>(emax + 2 * row);
    *reinterpret_cast<int2*>(emax + 2 * row) = make_int2(kExpZero, kExpZero);
  }
  __syncthreads();
  const int2 A = sh_a;
  unsigned long long L[2 * kLimbs];
#pragma unroll
  for (int d = 0; d < 2 * kLimbs; ++d) L[d] = 0;
  const bool fx = A.x < kExpInf, fz = A.y < kExpInf;
  for (int64_t t0 = tid;;) {
#pragma unroll
    for (int j = 0; j < kGrp; ++j) {
      if (fx) canon_add(v[j].x, A.x, L);
      if (fz) canon_add(v[j].y, A.y, L + kLimbs);
    }
    t0 += 256 * kGrp;
    if (t0 - tid >= ntiles) break;
    load(t0, v);
  }
#pragma unroll
  for (int d = 0; d < 2 * kLimbs; ++d) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) L[d] += __shfl_xor_sync(0xffffffffu, L[d], o);
    if (lane == 0) sh_d[w][d] = L[d];
  }
  __syncthreads();
  if (tid < 2) {
    unsigned long long T[kLimbs];
#pragma unroll
    for (int d = 0; d < kLimbs; ++d) {
      T[d] = 0;
      for (int i = 0; i < 8; ++i) T[d] += sh_d[i][tid * kLimbs + d];
    }
    sse[2 * row + tid] = canon_finish(T, tid ? A.y : A.x);
  }
}

// multi-shard / multi-rank steps: anchors (atomicMax over shards, then an
// allreduce-max), digits (atomicAdd over shards, then an allreduce-sum), finish
__global__ void k_reduce_partials(const double* __restrict__ part, int64_t ntiles, int64_t rows,
                                  double* __restrict__ out) {
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row < rows) warp_row_sse(part, ntiles, row, out);
}

__global__ void k_canon_exp(const double* __restrict__ part, int64_t ntiles, int64_t rows, int32_t* emax) {
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int lane = threadIdx.x & 31;
  const int2 A = warp_row_exp(part + row * ntiles * 2, ntiles, lane);
  if (lane == 0) {
    atomicMax(emax + 2 * row, A.x);
    atomicMax(emax + 2 * row + 1, A.y);
  }
}

__global__ void k_canon_digits(const double* __restrict__ part, int64_t ntiles, int64_t rows,
                               const int32_t* __restrict__ emax, unsigned long long* digits) {
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int lane = threadIdx.x & 31;
  unsigned long long L[2 * kLimbs];
  warp_row_digits(part + row * ntiles * 2, ntiles, lane, make_int2(emax[2 * row], emax[2 * row + 1]), L);
  if (lane < 2 * kLimbs) {
    unsigned long long mine = 0;
#pragma unroll
    for (int d = 0; d < 2 * kLimbs; ++d) mine = lane == d ? L[d] : mine;
    if (mine) atomicAdd(digits + row * 2 * kLimbs + lane, mine);
  }
}

__global__ void k_canon_finish(const int32_t* __restrict__ emax, const unsigned long long* __restrict__ digits,
                               int64_t n, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;   // (row, train|test)
  if (i >= n) return;
  unsigned long long L[kLimbs];
#pragma unroll
  for (int d = 0; d < kLimbs; ++d) L[d] = digits[(i >> 1) * 2 * kLimbs + (i & 1) * kLimbs + d];
  out[i] = canon_finish(L, emax[i]);
}

// fp64 RMSE of each row (operator API, fitness.py:28-51)
// Operator RMSE (gsgp/fitness.py:11-51): the reference accumulates every row
// strictly left to right (np.cumsum(diff * diff)[-1]), and documents the
// result as bitwise identical across backends, so the operator keeps that
// order: one thread per row adds its squares sequentially.  A block owns 32
// rows; its 256 threads stage a 32 x 64 tile of squared differences in shared
// memory with coalesced loads, then warp 0 folds the tile into the 32 running
// sums in column order.  (The engine's fitness uses the canonical sum
// instead — common.cuh — which is order-free across tiles and ranks.)
constexpr int kRmseRows = 32, kRmseCols = 64;
__global__ void __launch_bounds__(256) k_row_rmse(const double* __restrict__ S, const double* __restrict__ y,
                                                  int64_t m, int64_t n, double* out) {
  __shared__ double sq[kRmseRows][kRmseCols + 1];
  const int64_t r0 = (int64_t)blockIdx.x * kRmseRows;
  const int t = threadIdx.x;
  double acc = 0.0;
  for (int64_t c0 = 0; c0 < n; c0 += kRmseCols) {
    const int64_t w = n - c0 < kRmseCols ? n - c0 : kRmseCols;
    for (int e = t; e < kRmseRows * kRmseCols; e += 256) {
      const int rr = e / kRmseCols, cc = e % kRmseCols;
      if (r0 + rr < m && cc < w) {
        const double d = __dsub_rn(S[(r0 + rr) * n + c0 + cc], y[c0 + cc]);
        sq[rr][cc] = __dmul_rn(d, d);
      }
    }
    __syncthreads();
    if (t < kRmseRows && r0 + t < m)
      for (int cc = 0; cc < w; ++cc) acc = __dadd_rn(acc, sq[t][cc]);
    __syncthreads();
  }
  if (t < kRmseRows && r0 + t < m) out[r0 + t] = rmse_of(acc, (double)n);
}

// ---------------------------------------------------------- arg-min/max
// np.argmin / np.argmax semantics: ties go to the lowest index
// (gsgp/evolution.py:36-47).  Values are never NaN (fitness.py:25 maps
// non-finite RMSE to +inf).
struct ArgVal {
  double v;
  int64_t i;
};

__device__ __forceinline__ ArgVal better_min(ArgVal a, ArgVal b) {
  if (b.v < a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}
__device__ __forceinline__ ArgVal better_max(ArgVal a, ArgVal b) {
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}

template <bool kMin>
__device__ ArgVal block_arg(ArgVal x, ArgVal* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgVal y{__shfl_xor_sync(0xffffffffu, x.v, o), __shfl_xor_sync(0xffffffffu, x.i, o)};
    x = kMin ? better_min(x, y) : better_max(x, y);
  }
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sh[w] = x;
  __syncthreads();
  ArgVal r = sh[0];
  for (int i = 1; i < (int)(blockDim.x >> 5); ++i) r = kMin ? better_min(r, sh[i]) : better_max(r, sh[i]);
  return r;
}

constexpr ArgVal kMinInit{INFINITY, INT64_MAX};
constexpr ArgVal kMaxInit{-INFINITY, INT64_MAX};

// ------------------------------------------------------------- survival
// gsgp/evolution.py:65-83 plus the loop bookkeeping at :146-158.
// Slot flags (wide): a slot whose semantics overflowed fp32 at
// initialisation keeps its (constant) fp64 fitness — see DESIGN.md §4.
// One block of any size: the three arg-reductions share one shared-memory
// exchange, and the next generation's best parent needs no pass at all
// (it is the elite slot: a parent elite is strictly below every offspring,
// an offspring elite is the offspring minimum).
// A candidate with the payload survival needs from its row: the parent
// candidate carries its test SSE and slot flags (moved to the replaced slot
// when a parent survives), the offspring candidate its test SSE (the trace).
struct ArgPay {
  double v;
  int64_t i;
  double ts;
  int32_t fl;
};
template <bool kMin>
__device__ __forceinline__ ArgPay pick(const ArgPay& a, const ArgPay& b) {
  const bool take = kMin ? (b.v < a.v || (b.v == a.v && b.i < a.i)) : (b.v > a.v || (b.v == a.v && b.i < a.i));
  return take ? b : a;
}
template <bool kMin>
__device__ __forceinline__ ArgPay warp_pick(ArgPay x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgPay y{__shfl_xor_sync(0xffffffffu, x.v, o), __shfl_xor_sync(0xffffffffu, x.i, o),
             __shfl_xor_sync(0xffffffffu, x.ts, o), __shfl_xor_sync(0xffffffffu, x.fl, o)};
    x = pick<kMin>(x, y);
  }
  return x;
}

// One pass over the rows: each thread reads its rows' parent state and
// offspring SSE once, writes the next state (F, TS) in place and keeps the
// three candidates (best parent, best and worst offspring) with their
// payloads, so the block's leader finishes the generation from registers and
// shared memory alone (no second pass over the rows; the replaced slot is the
// only row it rewrites).
__device__ void survive_block(const SurviveArgs& a) {
  __shared__ ArgPay sh[3][32];
  const int64_t m = a.m;
  double* __restrict__ F = a.F;
  double* __restrict__ TS = a.TS;
  int32_t* __restrict__ wide = a.wide;
  const double* __restrict__ sse = a.sse_off;
  ArgPay bp{INFINITY, INT64_MAX, 0.0, 0}, bo{INFINITY, INT64_MAX, 0.0, 0}, wo{-INFINITY, INT64_MAX, 0.0, 0};
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    const int32_t fl = wide[i];
    const double fp = F[i], tsp = TS[i];
    const double so = sse[2 * i], to_ = sse[2 * i + 1];
    const double fo = (fl & 1) ? fp : rmse_of(so, a.ntr);
    const double to = (fl & 2) ? tsp : to_;
    bp = pick<true>(bp, ArgPay{fp, i, tsp, fl});
    bo = pick<true>(bo, ArgPay{fo, i, to, 0});
    wo = pick<false>(wo, ArgPay{fo, i, 0.0, 0});
    F[i] = fo;                     // next state (the replaced slot is fixed below)
    TS[i] = to;
  }
  bp = warp_pick<true>(bp);
  bo = warp_pick<true>(bo);
  wo = warp_pick<false>(wo);
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) { sh[0][w] = bp; sh[1][w] = bo; sh[2][w] = wo; }
  __syncthreads();                 // also orders every row's F/TS write before the leader's
  if (threadIdx.x == 0) {
    bp = sh[0][0]; bo = sh[1][0]; wo = sh[2][0];
    for (int k = 1; k < nw; ++k) {
      bp = pick<true>(bp, sh[0][k]);
      bo = pick<true>(bo, sh[1][k]);
      wo = pick<false>(wo, sh[2][k]);
    }
    const int64_t g = a.ctl[CTL_GEN];
    int8_t src;
    int64_t idx, slot;
    double fit, ts;
    if (bp.v < bo.v) {                       // strict: exact ties keep the offspring
      src = 0; idx = bp.i; slot = wo.i; fit = bp.v; ts = bp.ts;
      F[slot] = fit;
      TS[slot] = ts;
      wide[slot] = bp.fl;
      a.ctl[CTL_REDIRECT] = slot;
      a.ctl[CTL_PARENT_ELITES] += 1;
    } else {
      src = 1; idx = bo.i; slot = bo.i; fit = bo.v; ts = bo.ts;
      a.ctl[CTL_REDIRECT] = -1;
    }
    a.rec_src[g] = src;
    a.rec_idx[g] = idx;
    a.rec_slot[g] = slot;
    a.rec_fit[g] = fit;
    a.trace_tr[g] = fit;
    a.trace_te[g] = rmse_of(ts, a.nte);
    a.ctl[CTL_BP] = slot;          // argmin of the surviving fitness vector
    a.ctl[CTL_PARITY] ^= 1;
    a.ctl[CTL_GEN] += 1;
  }
}

// Canonical SSE of every row (one warp per row, warp_row_sse above) fused
// with survival: the last block to finish runs survive_block.
template <int kPer>
__global__ void __launch_bounds__(256) k_reduce_survive(const double* __restrict__ part, int64_t ntiles,
                                                        int32_t* emax, double* __restrict__ sse,
                                                        SurviveArgs a, unsigned int* done) {
  __shared__ int last;
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row < a.m) warp_row_sse_anchored<kPer>(part, ntiles, row, emax, sse);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  survive_block(a);
  if (threadIdx.x == 0) *done = 0;
}

// multi-shard / multi-rank generation tail, after the GSM launches
// accumulated the anchors (emax, allreduce-max over ranks) and k_canon_digits
// the digit sums (allreduce-sum over ranks): one rounding per (row,
// train|test), both accumulators re-armed for the next generation, and the
// last block runs the survival.
__global__ void __launch_bounds__(256) k_finish_survive(int32_t* emax, unsigned long long* digits,
                                                        double* __restrict__ sse, SurviveArgs a,
                                                        unsigned int* done) {
  __shared__ int last;
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;   // (row, train|test)
  if (i < 2 * a.m) {
    unsigned long long L[kLimbs];
    unsigned long long* d = digits + (i >> 1) * 2 * kLimbs + (i & 1) * kLimbs;
#pragma unroll
    for (int j = 0; j < kLimbs; ++j) {
      L[j] = d[j];
      d[j] = 0;
    }
    sse[i] = canon_finish(L, emax[i]);
    emax[i] = kExpZero;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  survive_block(a);
  if (threadIdx.x == 0) *done = 0;
}

// one unit per row (small case counts, e.g. C1): the canonical sum of a
// single partial is that partial, bit for bit (its fixed-point image is
// exact), so the SSE is copied and no anchors are used
__global__ void __launch_bounds__(256) k_reduce_survive_single(const double* __restrict__ part,
                                                               double* __restrict__ sse, SurviveArgs a,
                                                               unsigned int* done) {
  __shared__ int last;
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;   // (row, train|test)
  if (i < 2 * a.m) sse[i] = part[i];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  survive_block(a);
  if (threadIdx.x == 0) *done = 0;
}

__global__ void __launch_bounds__(256) k_reduce_survive_wide(const double* __restrict__ part, int64_t ntiles,
                                                             int32_t* emax, double* __restrict__ sse,
                                                             SurviveArgs a, unsigned int* done) {
  __shared__ int last;
  block_row_sse(part, ntiles, blockIdx.x, emax, sse);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  survive_block(a);
  if (threadIdx.x == 0) *done = 0;
}

// evolution.py:132-143: initial fitness, elite and trace[0].  The fitness
// comes from the stored semantics in the generation kernel's SSE order
// (sse_off), so a later offspring equal to its parent ties with it exactly;
// fp32-overflow slots use the fp64 interpreter SSE (sse_alt).
__global__ void __launch_bounds__(1024) k_init_state(SurviveArgs a) {
  __shared__ ArgVal sh[32];
  ArgVal b = kMinInit;
  for (int64_t i = threadIdx.x; i < a.m; i += blockDim.x) {
    const int32_t fl = a.wide[i];
    double f = rmse_of((fl & 1) ? a.sse_alt[2 * i] : a.sse_off[2 * i], a.ntr);
    a.F[i] = f;
    a.TS[i] = (fl & 2) ? a.sse_alt[2 * i + 1] : a.sse_off[2 * i + 1];
    b = better_min(b, ArgVal{f, i});
  }
  b = block_arg<true>(b, sh);
  if (threadIdx.x == 0) {
    a.rec_src[0] = 2;   // "initial"
    a.rec_idx[0] = b.i;
    a.rec_slot[0] = b.i;
    a.rec_fit[0] = b.v;
    a.trace_tr[0] = b.v;
    a.trace_te[0] = rmse_of(a.TS[b.i], a.nte);
    a.ctl[CTL_GEN] = 1;
    a.ctl[CTL_BP] = b.i;
    a.ctl[CTL_REDIRECT] = -1;
    a.ctl[CTL_PARITY] = 0;
    a.ctl[CTL_PARENT_ELITES] = 0;
  }
}

__global__ void __launch_bounds__(1024) k_survive_decision(const double* fp, const double* fo, int64_t m,
                                                          int64_t* out) {
  __shared__ ArgVal sh[32];
  ArgVal bp = kMinInit, bo = kMinInit, wo = kMaxInit;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    bp = better_min(bp, ArgVal{fp[i], i});
    bo = better_min(bo, ArgVal{fo[i], i});
    wo = better_max(wo, ArgVal{fo[i], i});
  }
  bp = block_arg<true>(bp, sh);
  bo = block_arg<true>(bo, sh);
  wo = block_arg<false>(wo, sh);
  if (threadIdx.x == 0) {
    if (bp.v < bo.v) { out[0] = 0; out[1] = bp.i; out[2] = wo.i; }
    else { out[0] = 1; out[1] = bo.i; out[2] = bo.i; }
  }
}

__global__ void __launch_bounds__(1024) k_argminmax(const double* f, int64_t m, int64_t* out) {
  __shared__ ArgVal sh[32];
  ArgVal lo = kMinInit, hi = kMaxInit;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    lo = better_min(lo, ArgVal{f[i], i});
    hi = better_max(hi, ArgVal{f[i], i});
  }
  lo = block_arg<true>(lo, sh);
  hi = block_arg<false>(hi, sh);
  if (threadIdx.x == 0) { out[0] = lo.i; out[1] = hi.i; }
}

__global__ void k_sigmoid_vec(const double* x, int64_t n, double* y) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] = __ddiv_rn(1.0, __dadd_rn(1.0, exp(-x[i])));   // mutation.py:32-34
}

}  // namespace

// ------------------------------------------------------------- launchers
void launch_argminmax(const double* f, int64_t m, int64_t* out, cudaStream_t s) {
  k_argminmax<<<1, 1024, 0, s>>>(f, m, out);
  check_launch();
}

void launch_sigmoid(const double* x, int64_t n, double* y, cudaStream_t s) {
  if (n <= 0) return;
  k_sigmoid_vec<<<blocks_for(n), kThreads, 0, s>>>(x, n, y);
  check_launch();
}

void launch_rng_draw(uint64_t seed, uint64_t stream, const uint64_t* counters, int64_t n,
                     uint64_t* bits, double* units, cudaStream_t s) {
  if (n <= 0) return;
  k_rng_draw<<<blocks_for(n), kThreads, 0, s>>>(stream_key(seed, stream), counters, n, bits, units);
  check_launch();
}

void launch_create_population(const GeneParams& p, int64_t count, uint64_t stream_base,
                              uint8_t* tags, int32_t* codes, double* consts, cudaStream_t s) {
  int64_t n = count * (int64_t)p.k;
  if (n <= 0) return;
  k_create_population<<<blocks_for(n), kThreads, 0, s>>>(p, count, stream_base, tags, codes, consts);
  check_launch();
}

void launch_plan(const PlanParams& p, int64_t gen, const int64_t* gen_ptr, int64_t* u, int64_t* v,
                 double* ms, int64_t stride_per_gen, cudaStream_t s) {
  k_plan<<<blocks_for(p.m), kThreads, 0, s>>>(p, gen, gen_ptr, u, v, ms, stride_per_gen);
  check_launch();
}

void launch_canon_clear(int64_t rows, int32_t* emax, unsigned long long* digits, cudaStream_t s) {
  GSGP_CUDA(cudaMemsetAsync(emax, 0x80, rows * 2 * 4, s));   // 0x80808080 == kExpZero
  GSGP_CUDA(cudaMemsetAsync(digits, 0, rows * 2 * kLimbs * 8, s));
}

void launch_canon_exp(const double* part, int64_t rows, int64_t ntiles, int32_t* emax, cudaStream_t s) {
  if (rows <= 0 || ntiles <= 0) return;
  k_canon_exp<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(part, ntiles, rows, emax);
  check_launch();
}

void launch_canon_digits(const double* part, int64_t rows, int64_t ntiles, const int32_t* emax,
                         unsigned long long* digits, cudaStream_t s) {
  if (rows <= 0 || ntiles <= 0) return;
  k_canon_digits<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(part, ntiles, rows, emax, digits);
  check_launch();
}

void launch_canon_finish(const int32_t* emax, const unsigned long long* digits, int64_t rows, double* sse,
                         cudaStream_t s) {
  if (rows <= 0) return;
  k_canon_finish<<<blocks_for(rows * 2), kThreads, 0, s>>>(emax, digits, rows * 2, sse);
  check_launch();
}

void launch_reduce_partials(const double* part, int64_t rows, int64_t ntiles, double* out, cudaStream_t s) {
  if (rows <= 0) return;
  k_reduce_partials<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(part, ntiles, rows, out);
  check_launch();
}

void launch_row_rmse(const double* S, const double* y, int64_t m, int64_t n, double* out,
                     cudaStream_t s) {
  if (m <= 0) return;
  k_row_rmse<<<(unsigned)((m + kRmseRows - 1) / kRmseRows), 256, 0, s>>>(S, y, m, n, out);
  check_launch();
}

void launch_reduce_survive(const double* part, int64_t ntiles, int32_t* emax, double* sse,
                           const SurviveArgs& a, unsigned int* done, cudaStream_t s) {
  if (ntiles == 1)     // emax is not used (the generation launch leaves it untouched)
    k_reduce_survive_single<<<(unsigned)((2 * a.m + 255) / 256), 256, 0, s>>>(part, sse, a, done);
  else if (ntiles > 1024)  // long rows (C3 ~3000 units): a block per row; else a warp per row
                           // (C2 31, C4 306, C5 611 units: 8 loads per lane in flight)
    k_reduce_survive_wide<<<(unsigned)a.m, 256, 0, s>>>(part, ntiles, emax, sse, a, done);
  else
    (ntiles <= 32 ? k_reduce_survive<1> : k_reduce_survive<8>)<<<(unsigned)((a.m + 7) / 8), 256, 0, s>>>(
        part, ntiles, emax, sse, a, done);
  check_launch();
}

void launch_finish_survive(int32_t* emax, unsigned long long* digits, double* sse, const SurviveArgs& a,
                           unsigned int* done, cudaStream_t s) {
  k_finish_survive<<<(unsigned)((2 * a.m + 255) / 256), 256, 0, s>>>(emax, digits, sse, a, done);
  check_launch();
}

void launch_init_state(const SurviveArgs& a, cudaStream_t s) {
  k_init_state<<<1, 1024, 0, s>>>(a);
  check_launch();
}

void launch_survive_decision(const double* fp, const double* fo, int64_t m, int64_t* out,
                             cudaStream_t s) {
  k_survive_decision<<<1, 1024, 0, s>>>(fp, fo, m, out);
  check_launch();
}

}  // namespace gsgp
