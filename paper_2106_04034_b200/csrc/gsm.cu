// Fused geometric semantic mutation + SSE, one streaming pass per generation.
//
//   offspring[i, j] = parent[i, j] + ms_i * (sq[u_i, j] -/+ sq[v_i, j])
//
// with the reference's rounding order t = a -/+ b; t = t * ms; out = parent + t
// (gsgp/mutation.py:77-83), applied to train AND test semantics with the same
// plan in one pass (one row of storage = [train cases | pad | test cases | pad]),
// followed by the fp64 squared error against the target (gsgp/fitness.py:23).
// The SSE of each (row, case tile) is reduced in a fixed order —
// thread-sequential -> warp butterfly -> warps in index order — and the tile
// partials are combined by the canonical (exact, order-free) sum of
// common.cuh: a function of case positions only, so equal rows get bit-equal
// SSEs, argmin ties resolve to the lowest index exactly like np.argmin, and
// the result does not depend on how the cases are split over GPUs.
//
// Layout / traffic: row-major [rows][pitch] (pitch % 32 == 0).  Parents are
// updated IN PLACE; the best parent row (ctl[CTL_BP]) is copied aside while
// it streams by, and survival redirects the replaced slot to that copy in the
// next generation (ctl[CTL_REDIRECT]), so no row-copy kernel is needed.
// HBM traffic per generation ~= 4*N*(2m + D + 1) bytes, D = distinct pool
// rows of the plan (each pool tile is read from HBM once, see below).
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "kernels.cuh"

namespace gsgp {

namespace {

template <typename T> struct Vec16;
template <> struct Vec16<float> { using type = float4; static constexpr int n = 4; };
template <> struct Vec16<double> { using type = double2; static constexpr int n = 2; };

template <bool kPlus>
__device__ __forceinline__ float mut(float p, float a, float b, float ms) {
  float t = kPlus ? __fadd_rn(a, b) : __fsub_rn(a, b);
  return __fadd_rn(p, __fmul_rn(t, ms));
}
template <bool kPlus>
__device__ __forceinline__ double mut(double p, double a, double b, double ms) {
  double t = kPlus ? __dadd_rn(a, b) : __dsub_rn(a, b);
  return __dadd_rn(p, __dmul_rn(t, ms));
}

// Units follow the shard's RowLayout (kernels.cuh): tiles anchored on the
// train region and on the test region separately, so no plain tile mixes
// train and test cases and — with shard slices on the kCaseAlign grid
// (engine.cu) — every tile holds the same global cases at the same positions
// for any shard/rank split (canonical partials).  When the two partial tails
// fit in one tile, the layout stores the test tail right after the train
// region, so the train tail + test tail are ONE contiguous unit whose first
// nA elements are train: the unit count of a pitch-wide tiling is kept
// (each unit costs a fixed pipeline round trip; +3 % units measured +2 % time
// at C2) and every unit is a single span.
struct UnitSpan {
  int64_t off;   // storage offset
  int32_t n;     // elements
  int32_t nA;    // the first nA elements are train cases, the rest test
};
__device__ __forceinline__ UnitSpan unit_span(int64_t t, const RowLayout& L) {
  UnitSpan u;
  if (t < L.ttr) {
    u.off = t * L.tile;
    const int64_t end = (t == L.ttr - 1 && L.tail_off >= 0) ? L.tail_off + L.tail_pad : L.ntr_pad;
    u.n = (int32_t)min(L.tile, end - u.off);
    u.nA = (int32_t)min((int64_t)u.n, L.ntr_pad - u.off);
  } else {
    u.off = L.test_off + (t - L.ttr) * L.tile;
    u.n = (int32_t)min(L.tile, L.pitch - u.off);
    u.nA = 0;
  }
  return u;
}

// one work unit = (case tile, population row): 16 KB of each streamed row
#ifndef GSGP_GSM_TILE
#define GSGP_GSM_TILE 16384
#endif
#ifndef GSGP_GSM_STAGES
#define GSGP_GSM_STAGES 4
#endif
#ifndef GSGP_GSM_CWARPS
#define GSGP_GSM_CWARPS 8   // 8 vs 16: C3 +2.7 %, C4 +5 %, C5 +3.6 % (profiles/r02/gsm)
#endif
constexpr int kTileBytes = GSGP_GSM_TILE;

// ===================================================================
// TMA-pipelined persistent kernel (the engine's generation kernel).
//
// Units are numbered tile-major (unit = t*m + i) and handed out from a
// global ticket counter to one persistent CTA per SM, so all CTAs sweep the
// case tiles in lockstep and each pool tile is fetched from HBM once, then
// re-served from L2 to every row that references it (pool copies: L2
// evict_last; parent: evict_first; offspring stores: streaming).
//   warp W  producer (W = kConsumerWarps, 8 by default): claims batches
//           of units, the warp's lanes draw the rows' mutation plans
//           (u, v, ms) from the counter RNG in parallel, and one lane issues
//           3 cp.async.bulk copies (parent row tile, pool[u] tile, pool[v]
//           tile) into a kStages-deep shared-memory ring; completion =
//           mbarrier transaction count.
//   warps 0..W-1 consumers: copy the unit out of shared memory into
//           registers, release the stage at once (so the producer refills it
//           while they compute), mutate, store the offspring with 128-bit
//           streaming stores, save the best parent row, and accumulate the
//           fp64 SSE against the target, which each thread keeps in
//           registers for as long as the CTA stays on the same case tile.
//   warp W+1 finalizer (one lane): folds the W per-warp SSE partials of
//           each unit (fixed warp order) into part[i][t], decoupled from the
//           consumers through a small mbarrier ring.
// ===================================================================
constexpr int kStages = GSGP_GSM_STAGES;
constexpr int kRedStages = 4;
constexpr int kConsumerWarps = GSGP_GSM_CWARPS;
constexpr int kNCT = kConsumerWarps * 32;
constexpr int kTmaThreads = (kConsumerWarps + 2) * 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  const uint32_t a = smem_u32(bar);
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// global -> shared bulk copy on the TMA engine, completion on an mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// kOp: operator mode (gsgp.gsm on arbitrary inputs): non-finite -> 0 with a
// count (mutation.py:86).  In the engine the parent is finite (or an fp32
// overflow slot whose fp64 value the reference keeps constant)
// so no replacement is done there.
// kSseOnly: no mutation and no stores — the SSE of the stored semantics in
// exactly the order a generation uses, for the initial fitness (so an
// offspring that equals its parent bit for bit ties with it, as in numpy).
template <typename T, bool kOp, bool kSseOnly = false, bool kPlus = false>
__global__ void __launch_bounds__(kTmaThreads, 1)
k_gsm_tma(GsmArgs a, int64_t nunits, int kBatch) {
  using Vec = typename Vec16<T>::type;
  constexpr int EV = Vec16<T>::n;
  constexpr int TILE = kTileBytes / (int)sizeof(T);   // elements per unit
  constexpr int VPT = TILE / (kNCT * EV);             // 16-byte vectors per consumer thread
  static_assert(VPT * kNCT * EV == TILE, "tile must split evenly over consumers");
  extern __shared__ __align__(128) unsigned char smem[];
  T* data = reinterpret_cast<T*>(smem);                                   // [S][3][TILE]
  double* red = reinterpret_cast<double*>(smem + kStages * 3 * kTileBytes);  // [RS][W][2]
  uint64_t* full = reinterpret_cast<uint64_t*>(red + kRedStages * kConsumerWarps * 2);
  uint64_t* empty = full + kStages;
  uint64_t* rfull = empty + kStages;
  uint64_t* rempty = rfull + kRedStages;
  int64_t* slot_unit = reinterpret_cast<int64_t*>(rempty + kRedStages);   // [S] unit in stage
  int64_t* red_unit = slot_unit + kStages;                                // [RS] unit in red slot
  double* slot_ms = reinterpret_cast<double*>(red_unit + kRedStages);     // [S] mutation step
  int4* slot_it = reinterpret_cast<int4*>(slot_ms + kStages);             // [S] (row i, tile t, n, nA)
  int64_t* slot_off = reinterpret_cast<int64_t*>(slot_it + kStages);      // [S] storage offset of the unit

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m = a.m;
  const int64_t* u = a.u;
  const int64_t* vv = a.v;
  const double* ms = a.ms;
  int64_t bp = -1, redirect = -1, gen = 0;
  const T* elite_prev = reinterpret_cast<const T*>(a.elite_prev);
  T* elite_cur = reinterpret_cast<T*>(a.elite_cur);
  if (a.ctl) {
    gen = a.ctl[CTL_GEN];
    bp = a.ctl[CTL_BP];
    redirect = a.ctl[CTL_REDIRECT];
    u += (gen - 1) * m;
    vv += (gen - 1) * m;
    ms += (gen - 1) * m;
    if (a.ctl[CTL_PARITY]) {   // ping-pong elite buffers
      const T* t0 = elite_prev;
      elite_prev = elite_cur;
      elite_cur = const_cast<T*>(t0);
    }
  }
  const T* pool = reinterpret_cast<const T*>(a.pool);
  T* S = reinterpret_cast<T*>(a.S);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kConsumerWarps);
    }
    for (int s = 0; s < kRedStages; ++s) {
      mbar_init(rfull + s, kConsumerWarps);
      mbar_init(rempty + s, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // Units are handed out dynamically, in tile-major order, from a global
  // ticket counter: every CTA always works on the globally next units, so
  // the CTAs cannot drift apart over a long kernel and the pool tiles in use
  // stay L2-resident (a static round-robin split drifted by many tiles at
  // 10M cases).  The producer publishes each unit id in slot_unit[stage];
  // -1 terminates the consumers, who forward it to the finalizer.
  if (warp == kConsumerWarps) {
    // ------------------------------------------------------------ producer
    // The whole warp produces: when a batch of units is claimed, lane b
    // draws the plan of unit base + b (the counter RNG makes every draw
    // independent), so the per-unit RNG latency is paid once per batch and in
    // parallel; lane 0 then publishes the units one stage at a time, taking
    // (row, tile, u, v, ms) from the owning lane with shuffles.
    const uint64_t keep = l2_policy_evict_last(), stream = l2_policy_evict_first();
    const uint64_t plan_key = stream_key(a.plan.seed, kPlanStream0 + (uint64_t)gen);
    int64_t* u_out = const_cast<int64_t*>(u);
    int64_t* v_out = const_cast<int64_t*>(vv);
    double* ms_out = const_cast<double*>(ms);
    int s = 0;
    uint32_t j = 0;
    // tickets are claimed kBatch units at a time (launch_gsm_mode sizes the
    // batch to the work per CTA, <= 32), one claim ahead, so the atomic's
    // round trip overlaps the current units' copies.  (Claiming several
    // batches ahead and bulk-prefetching their parent tiles into L2 was
    // measured slower on every config: profiles/r01/README.md.)
    int64_t next = 0;
    if (lane == 0) next = (int64_t)atomicAdd(a.ticket, (unsigned long long)kBatch);
    next = __shfl_sync(0xffffffffu, next, 0);
    int64_t k = 0;
    for (bool done = false; !done;) {
      const int64_t base = next;
      if (base < nunits) {
        if (lane == 0) next = (int64_t)atomicAdd(a.ticket, (unsigned long long)kBatch);
        next = __shfl_sync(0xffffffffu, next, 0);
      }
      // this lane's unit of the batch: (tile tb, row ib), its case span and
      // the three source addresses — all computed here, lane-parallel, so
      // lane 0's per-unit path below is shuffles, slot writes and copies only
      const int64_t ub_unit = base + lane;
      int64_t tb = 0, ib = 0, ub = 0, vb = 0;
      UnitSpan sp{0, 0, 0};
      double msb = 0.0;
      const T *srcb = nullptr, *pub = nullptr, *pvb = nullptr;
      if (lane < kBatch && ub_unit < nunits) {
        tb = ub_unit / m;
        ib = ub_unit - tb * m;
        if (kSseOnly) {
        } else if (a.plan_inline) {
          plan_slot(plan_key, ib, a.plan.r, a.plan.ms_uniform, a.plan.ms_const, &ub, &vb, &msb);
          if (tb == 0 && a.write_plan) { u_out[ib] = ub; v_out[ib] = vb; ms_out[ib] = msb; }
        } else {
          ub = u[ib];
          vb = vv[ib];
          msb = ms[ib];
        }
        sp = unit_span(tb, a.lay);
        srcb = ((ib == redirect) ? elite_prev : S + ib * a.lay.pitch) + sp.off;
        pub = pool + ub * a.lay.pitch + sp.off;
        pvb = pool + vb * a.lay.pitch + sp.off;
      }
      for (int q = 0; q < kBatch; ++q, ++k) {
        const int64_t unit = base + q;
        // packed: (row, tile) in one 64-bit and (n, nA) (<= 8192 each) in one 32-bit shuffle
        const uint64_t ti = __shfl_sync(0xffffffffu, ((uint64_t)tb << 32) | (uint32_t)ib, q);
        const uint32_t nn = __shfl_sync(0xffffffffu, ((uint32_t)sp.n << 16) | (uint32_t)sp.nA, q);
        const int t = (int)(ti >> 32), i = (int)(uint32_t)ti;
        const int n = (int)(nn >> 16), nA = (int)(nn & 0xffffu);
        const int64_t off = __shfl_sync(0xffffffffu, sp.off, q);
        const T* src = reinterpret_cast<const T*>(__shfl_sync(0xffffffffu, (unsigned long long)srcb, q));
        const T* pu = reinterpret_cast<const T*>(__shfl_sync(0xffffffffu, (unsigned long long)pub, q));
        const T* pv = reinterpret_cast<const T*>(__shfl_sync(0xffffffffu, (unsigned long long)pvb, q));
        const double msd = __shfl_sync(0xffffffffu, msb, q);
        if (lane == 0) {
          if (k >= kStages) mbar_wait(empty + s, (j & 1) ^ 1);
          if (unit >= nunits) {
            slot_unit[s] = -1;
            mbar_expect_tx(full + s, 0);   // same completion path as a unit (0 transaction bytes)
          } else {
            const uint32_t bytes = (uint32_t)n * (uint32_t)sizeof(T);
            T* d = data + (int64_t)s * 3 * TILE;
            slot_unit[s] = unit;
            slot_ms[s] = msd;
            slot_it[s] = make_int4(i, t, n, nA);
            slot_off[s] = off;
            mbar_expect_tx(full + s, (kSseOnly ? 1 : 3) * bytes);
            bulk_g2s(d, src, bytes, full + s, stream);
            if (!kSseOnly) {
              bulk_g2s(d + TILE, pu, bytes, full + s, keep);
              bulk_g2s(d + 2 * TILE, pv, bytes, full + s, keep);
            }
          }
        }
        __syncwarp();
        if (unit >= nunits) { done = true; break; }
        if (++s == kStages) { s = 0; ++j; }
      }
    }
    // every claim of this CTA is done; the last CTA out re-arms the ticket
    if (lane == 0) {
      __threadfence();
      if (atomicAdd(a.ticket + 1, 1ull) == (unsigned long long)gridDim.x - 1) {
        atomicExch(a.ticket, 0ull);
        atomicExch(a.ticket + 1, 0ull);
      }
    }
    return;
  }
  if (warp == kConsumerWarps + 1) {
    // ----------------------------------------------------------- finalizer
    if (lane == 0) {
      int rs = 0;
      uint32_t rj = 0;
      for (;;) {
        mbar_wait(rfull + rs, rj & 1);
        const int64_t unit = red_unit[rs];
        if (unit < 0) break;
        const double* r = red + rs * kConsumerWarps * 2;
        double x = 0.0, z = 0.0;
#pragma unroll
        for (int w = 0; w < kConsumerWarps; ++w) {
          x = __dadd_rn(x, r[2 * w]);
          z = __dadd_rn(z, r[2 * w + 1]);
        }
        mbar_arrive(rempty + rs);
        const int64_t t = unit / m, i = unit - t * m;
        a.part[(i * a.lay.ntiles + t) * 2] = x;
        a.part[(i * a.lay.ntiles + t) * 2 + 1] = z;
        if (a.emax) {   // canonical-sum anchors, so the reduce reads the partials once
          if (x != 0.0) atomicMax(a.emax + 2 * i, canon_exp(x));
          if (z != 0.0) atomicMax(a.emax + 2 * i + 1, canon_exp(z));
        }
        if (++rs == kRedStages) { rs = 0; ++rj; }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int ct = threadIdx.x;   // 0 .. kNCT-1
  int64_t cur_t = -1;
  int s = 0, rs = 0;
  uint32_t j = 0, rj = 0;
  double y[VPT][EV];
  unsigned long long nonfinite = 0;
  for (int64_t k = 0;; ++k) {
    mbar_wait(full + s, j & 1);
    // the stage's unit id: read by lane 0 (the lane that releases the stage)
    // and broadcast
    int64_t unit = 0;
    if (lane == 0) unit = slot_unit[s];
    unit = __shfl_sync(0xffffffffu, unit, 0);
    if (unit < 0) {   // no more units: tell the finalizer and stop
      if (lane == 0) {
        if (k >= kRedStages) mbar_wait(rempty + rs, (rj & 1) ^ 1);
        if (warp == 0) red_unit[rs] = -1;
        mbar_arrive(rfull + rs);
      }
      break;
    }
    const int4 it = slot_it[s];
    const int64_t t = it.y, i = it.x;
    const int n = it.z, nA = it.w;                      // elements [0, nA) are train cases
    const int64_t off = slot_off[s];
    if (t != cur_t) {   // target tile: registers, reloaded when the CTA changes tile
#pragma unroll
      for (int q = 0; q < VPT; ++q) {
        const int e = (q * kNCT + ct) * EV;
#pragma unroll
        for (int c = 0; c < EV; ++c) y[q][c] = e < n ? __ldg(a.y + off + e + c) : 0.0;
      }
      cur_t = t;
    }
    const T msv = (T)slot_ms[s];
    const bool save = (i == bp);
    const T* d = data + (int64_t)s * 3 * TILE;
    Vec P[VPT], A[VPT], B[VPT];
#pragma unroll
    for (int q = 0; q < VPT; ++q) {
      const int e = (q * kNCT + ct) * EV;
      P[q] = *reinterpret_cast<const Vec*>(d + e);
      if (!kSseOnly) {
        A[q] = *reinterpret_cast<const Vec*>(d + TILE + e);
        B[q] = *reinterpret_cast<const Vec*>(d + 2 * TILE + e);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + s);   // stage free: the producer refills while we compute
    if (++s == kStages) { s = 0; ++j; }

    T* orow = S + i * a.lay.pitch + off;
    // one 16-byte vector of cases: mutate, store, squared errors summed in
    // element order (thread-sequential part of the fixed SSE order)
    auto vec = [&](int q, int e) -> double {
      const T* pe = reinterpret_cast<const T*>(&P[q]);
      const T* ae = reinterpret_cast<const T*>(&A[q]);
      const T* be = reinterpret_cast<const T*>(&B[q]);
      Vec O;
      T* oe = reinterpret_cast<T*>(&O);
      double sacc = 0.0;
#pragma unroll
      for (int c = 0; c < EV; ++c) {
        T o = kSseOnly ? pe[c] : mut<kPlus>(pe[c], ae[c], be[c], msv);
        if (kOp && !isfinite((double)o)) { o = (T)0; ++nonfinite; }
        oe[c] = o;
        const double dd = __dsub_rn((double)o, y[q][c]);
        sacc = __fma_rn(dd, dd, sacc);   // one fused op: fewer fp64 issues (power-bound)
      }
      if (!kSseOnly) {
        __stcs(reinterpret_cast<Vec*>(orow + e), O);
        if (save) __stcs(reinterpret_cast<Vec*>(elite_cur + off + e), P[q]);
      }
      return sacc;
    };
    double acc_tr = 0.0, acc_te = 0.0;
    if (n == TILE && (nA == 0 || nA == n)) {
      // a full unit of one region (all but the tails): no bounds, one sum
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < VPT; ++q) acc = __dadd_rn(acc, vec(q, (q * kNCT + ct) * EV));
      acc = warp_sum(acc);
      if (nA) acc_tr = acc;
      else acc_te = acc;
    } else {
#pragma unroll
      for (int q = 0; q < VPT; ++q) {
        const int e = (q * kNCT + ct) * EV;
        if (e >= n) continue;
        const double sacc = vec(q, e);
        if (e < nA) acc_tr = __dadd_rn(acc_tr, sacc);
        else acc_te = __dadd_rn(acc_te, sacc);
      }
      // fixed-order warp reduction; a tail unit may hold train and test cases
      if (nA >= n) acc_tr = warp_sum(acc_tr);
      else if (nA == 0) acc_te = warp_sum(acc_te);
      else { acc_tr = warp_sum(acc_tr); acc_te = warp_sum(acc_te); }
    }
    if (lane == 0) {
      if (k >= kRedStages) mbar_wait(rempty + rs, (rj & 1) ^ 1);
      red[(rs * kConsumerWarps + warp) * 2] = acc_tr;
      red[(rs * kConsumerWarps + warp) * 2 + 1] = acc_te;
      if (warp == 0) red_unit[rs] = unit;
      mbar_arrive(rfull + rs);
    }
    if (++rs == kRedStages) { rs = 0; ++rj; }
  }
  if (kOp) {
    for (int o = 16; o > 0; o >>= 1) nonfinite += __shfl_xor_sync(0xffffffffu, nonfinite, o);
    if (lane == 0 && nonfinite) atomicAdd(a.nonfinite, nonfinite);
  }
}

constexpr size_t kTmaSmem = (size_t)kStages * 3 * kTileBytes + (size_t)kRedStages * kConsumerWarps * 2 * 8 +
                            (2 * kStages + 2 * kRedStages) * 8 + (5 * kStages + kRedStages) * 8;
int g_num_sms = 0;

}  // namespace

RowLayout make_layout(int64_t ntr, int64_t nte, bool f64, bool allow_merge) {
  auto pad32 = [](int64_t x) { return (x + 31) / 32 * 32; };
  RowLayout L{};
  L.tile = kTileBytes / (f64 ? 8 : 4);
  L.ntr = ntr;
  L.nte = nte;
  L.ntr_pad = pad32(ntr);
  const int64_t tail_tr = L.ntr_pad % L.tile, tail_te = nte % L.tile;
  const bool merge = allow_merge && tail_tr > 0 && tail_te > 0 && tail_tr + pad32(tail_te) <= L.tile;
  L.ttr = (L.ntr_pad + L.tile - 1) / L.tile;
  if (merge) {   // [train | test tail | full test tiles]
    L.tail_off = L.ntr_pad;
    L.tail_pad = pad32(tail_te);
    L.te_full = nte - tail_te;
    L.test_off = L.tail_off + L.tail_pad;
    L.pitch = L.test_off + L.te_full;
    L.tte = L.te_full / L.tile;
  } else {       // [train | test]
    L.tail_off = -1;
    L.tail_pad = 0;
    L.te_full = nte;
    L.test_off = L.ntr_pad;
    L.pitch = L.test_off + pad32(nte);
    L.tte = (pad32(nte) + L.tile - 1) / L.tile;
  }
  L.ntiles = L.ttr + L.tte;
  return L;
}

int64_t gsm_tile_cases(bool f64) { return kTileBytes / (f64 ? 8 : 4); }

void gsm_preload() {   // see interp_preload
  auto pre = [](auto k) {
    cudaFuncAttributes f{};
    GSGP_CUDA(cudaFuncGetAttributes(&f, k));
  };
  pre(k_gsm_tma<float, false>);
  pre(k_gsm_tma<float, false, false, true>);
  pre(k_gsm_tma<float, false, true>);
  pre(k_gsm_tma<double, false>);
  pre(k_gsm_tma<double, false, false, true>);
  pre(k_gsm_tma<double, false, true>);
}

void launch_gsm(const GsmArgs& a, bool f64, bool operator_mode, cudaStream_t s) {
  launch_gsm_mode(a, f64, operator_mode ? 1 : 0, s);
}

void launch_sse_only(const GsmArgs& a, bool f64, cudaStream_t s) { launch_gsm_mode(a, f64, 2, s); }

void launch_gsm_mode(const GsmArgs& a, bool f64, int mode, cudaStream_t s) {
  if (a.m <= 0 || a.lay.pitch <= 0) return;
  GSGP_REQUIRE(a.lay.pitch % 32 == 0 && a.lay.tile == kTileBytes / (f64 ? 8 : 4), "bad storage layout");
  const int64_t ntiles = a.lay.ntiles;
  if (g_num_sms == 0) {
    int dev = 0;
    GSGP_CUDA(cudaGetDevice(&dev));
    GSGP_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const int64_t nunits = ntiles * a.m;
  const unsigned grid = (unsigned)std::min<int64_t>(g_num_sms, nunits);
  GSGP_REQUIRE(a.ticket != nullptr, "GSM launch needs a ticket counter");
  // claim size: large batches cut ticket atomics and keep a CTA on
  // consecutive rows of one tile (C3 0.91 -> 0.97 of peak at 16), but the
  // last claims of a small launch must still balance across CTAs, so keep
  // >= 48 claims per CTA (profiles/r01/README.md, batch A/B)
  // GSGP_GSM_BATCH (tests, A/B) is read at every launch so one process can
  // exercise several claim sizes
  const char* fb = getenv("GSGP_GSM_BATCH");
  const int forced = fb ? atoi(fb) : 0;
  int batch = 2;
  while (batch < 16 && nunits / ((int64_t)grid * 2 * batch) >= 48) batch *= 2;
  if (forced > 0) batch = forced < 32 ? forced : 32;   // one unit per producer lane
  auto go = [&](auto kern) {
    GSGP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem));
    kern<<<grid, kTmaThreads, kTmaSmem, s>>>(a, nunits, batch);
  };
  // gsm_sign is a kernel parameter of the instantiation: "minus" (the
  // reference default) and "plus" are separate kernels, so the mutation has
  // no per-element select
  const bool plus = a.sign != 0;
  if (f64) {
    if (mode == 2) go(k_gsm_tma<double, false, true>);
    else if (mode == 1) plus ? go(k_gsm_tma<double, true, false, true>) : go(k_gsm_tma<double, true>);
    else plus ? go(k_gsm_tma<double, false, false, true>) : go(k_gsm_tma<double, false>);
  } else {
    if (mode == 2) go(k_gsm_tma<float, false, true>);
    else if (mode == 1) plus ? go(k_gsm_tma<float, true, false, true>) : go(k_gsm_tma<float, true>);
    else plus ? go(k_gsm_tma<float, false, false, true>) : go(k_gsm_tma<float, false>);
  }
  GSGP_CUDA(cudaGetLastError());
}

}  // namespace gsgp
