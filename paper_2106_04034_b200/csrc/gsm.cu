// Fused geometric semantic mutation + SSE, one streaming pass per generation.
//
//   offspring[i, j] = parent[i, j] + ms_i * (sq[u_i, j] -/+ sq[v_i, j])
//
// with the reference's rounding order t = a -/+ b; t = t * ms; out = parent + t
// (gsgp/mutation.py:77-83), applied to train AND test semantics with the same
// plan in one pass (one row of storage = [train cases | pad | test cases | pad]),
// followed by the fp64 squared error against the target (gsgp/fitness.py:23)
// reduced per row: thread-sequential -> warp butterfly -> warps in order ->
// tiles in order (k_reduce_partials).  The order is a function of case
// positions only, so equal rows get bit-equal SSEs and argmin ties resolve to
// the lowest index exactly like np.argmin.
//
// Layout / traffic: row-major [rows][pitch] with pitch % 32 == 0, 128-bit
// loads and stores.  The grid is case-tile-major (blockIdx -> (tile, row
// group)), so all population rows of one case tile are processed close in
// time and each pool row's tile segment is fetched from HBM once and then
// served from L2 to the other rows that reference it: HBM traffic per
// generation ~= 4*N*(2m + D + 1) bytes (D = distinct pool rows in the plan).
// Parents are updated IN PLACE; the best parent row (ctl[CTL_BP]) is copied
// aside while it streams by, and survival redirects the replaced slot to that
// copy in the next generation, so no row copy kernel is needed.
#include "kernels.cuh"

namespace gsgp {

namespace {

template <typename T> struct Vec16;
template <> struct Vec16<float> { using type = float4; static constexpr int n = 4; };
template <> struct Vec16<double> { using type = double2; static constexpr int n = 2; };

__device__ __forceinline__ float mut(float p, float a, float b, float ms, int sign) {
  float t = sign ? __fadd_rn(a, b) : __fsub_rn(a, b);
  return __fadd_rn(p, __fmul_rn(t, ms));
}
__device__ __forceinline__ double mut(double p, double a, double b, double ms, int sign) {
  double t = sign ? __dadd_rn(a, b) : __dsub_rn(a, b);
  return __dadd_rn(p, __dmul_rn(t, ms));
}

template <typename V> __device__ __forceinline__ V ld_stream(const V* p) { return *p; }
template <> __device__ __forceinline__ float4 ld_stream(const float4* p) { return __ldcs(p); }
template <> __device__ __forceinline__ double2 ld_stream(const double2* p) { return __ldcs(p); }

template <typename V> __device__ __forceinline__ V ld_pool(const V* p) { return __ldg(p); }

constexpr int kThreads = 256;

// kOp: operator mode (gsgp.gsm on arbitrary inputs): non-finite -> 0 with a
// count (mutation.py:86).  In the engine the parent is finite (or an fp32
// overflow slot whose fp64 value the reference keeps constant)
// so no replacement is done there.
template <typename T, bool kOp, int V, int R>
__global__ void __launch_bounds__(kThreads, 2)
k_gsm(GsmArgs a, int64_t ntiles, int64_t ngroups) {
  using Vec = typename Vec16<T>::type;
  constexpr int EV = Vec16<T>::n;
  constexpr int TILE = kThreads * V * EV;
  __shared__ double red[kThreads / 32][R][2];

  const int tid = threadIdx.x;
  const int64_t tile = blockIdx.x / ngroups;          // case-tile-major order
  const int64_t grp = blockIdx.x - tile * ngroups;
  const int64_t i0 = grp * R;

  const int64_t* u = a.u;
  const int64_t* vv = a.v;
  const double* ms = a.ms;
  int64_t bp = -1, redirect = -1;
  const T* elite_prev = reinterpret_cast<const T*>(a.elite_prev);
  T* elite_cur = reinterpret_cast<T*>(a.elite_cur);
  if (a.ctl) {
    const int64_t gen = a.ctl[CTL_GEN];
    const int64_t par = a.ctl[CTL_PARITY];
    bp = a.ctl[CTL_BP];
    redirect = a.ctl[CTL_REDIRECT];
    u += (gen - 1) * a.m;
    vv += (gen - 1) * a.m;
    ms += (gen - 1) * a.m;
    if (par) {   // ping-pong elite buffers
      const T* t0 = elite_prev;
      elite_prev = elite_cur;
      elite_cur = const_cast<T*>(t0);
    }
  }

  int64_t e[V];
  bool ok[V], tr[V];
  double y[V][EV];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    e[v] = tile * TILE + ((int64_t)v * kThreads + tid) * EV;
    ok[v] = e[v] < a.pitch;
    tr[v] = e[v] < a.test_off;
#pragma unroll
    for (int c = 0; c < EV; ++c) y[v][c] = ok[v] ? a.y[e[v] + c] : 0.0;
  }

  const T* pool = reinterpret_cast<const T*>(a.pool);
  T* S = reinterpret_cast<T*>(a.S);
  unsigned long long nonfinite = 0;
  double acc_tr[R], acc_te[R];

#pragma unroll
  for (int r = 0; r < R; ++r) {
    acc_tr[r] = 0.0;
    acc_te[r] = 0.0;
    const int64_t i = i0 + r;
    if (i >= a.m) continue;
    const int64_t ui = u[i], vi = vv[i];
    const T msv = (T)ms[i];
    const T* prow = (i == redirect) ? elite_prev : S + i * a.pitch;
    const Vec* pu = reinterpret_cast<const Vec*>(pool + ui * a.pitch);
    const Vec* pv = reinterpret_cast<const Vec*>(pool + vi * a.pitch);
    const Vec* pp = reinterpret_cast<const Vec*>(prow);
    Vec* po = reinterpret_cast<Vec*>(S + i * a.pitch);
    Vec P[V], A[V], Bv[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      if (!ok[v]) continue;
      const int64_t w = e[v] / EV;
      P[v] = ld_stream(pp + w);
      A[v] = ld_pool(pu + w);
      Bv[v] = ld_pool(pv + w);
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      if (!ok[v]) continue;
      const int64_t w = e[v] / EV;
      T* pe = reinterpret_cast<T*>(&P[v]);
      T* ae = reinterpret_cast<T*>(&A[v]);
      T* be = reinterpret_cast<T*>(&Bv[v]);
      Vec O;
      T* oe = reinterpret_cast<T*>(&O);
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < EV; ++c) {
        T o = mut(pe[c], ae[c], be[c], msv, a.sign);
        if (kOp && !isfinite((double)o)) { o = (T)0; ++nonfinite; }
        oe[c] = o;
        double d = __dsub_rn((double)o, y[v][c]);
        s = __dadd_rn(s, __dmul_rn(d, d));
      }
      po[w] = O;
      if (i == bp) reinterpret_cast<Vec*>(elite_cur)[w] = P[v];
      if (tr[v]) acc_tr[r] = __dadd_rn(acc_tr[r], s);
      else acc_te[r] = __dadd_rn(acc_te[r], s);
    }
  }
  // per-row fixed-order block reduction
  const int warp = tid >> 5, lane = tid & 31;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    double x = warp_sum(acc_tr[r]);
    double z = warp_sum(acc_te[r]);
    if (lane == 0) { red[warp][r][0] = x; red[warp][r][1] = z; }
  }
  __syncthreads();
  if (tid < 2 * R) {
    const int r = tid >> 1, w2 = tid & 1;
    const int64_t i = i0 + r;
    if (i < a.m) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) t = __dadd_rn(t, red[w][r][w2]);
      a.part[(i * ntiles + tile) * 2 + w2] = t;
    }
  }
  if (kOp) {
    for (int o = 16; o > 0; o >>= 1) nonfinite += __shfl_xor_sync(0xffffffffu, nonfinite, o);
    if (lane == 0 && nonfinite) atomicAdd(a.nonfinite, nonfinite);
  }
}

constexpr int kRowsPerBlock = 8;
constexpr int kVecF32 = 2;   // 2 x float4 per thread per row: tile = 2048 cases
constexpr int kVecF64 = 4;   // 4 x double2: tile = 2048 cases

}  // namespace

int64_t gsm_tiles(int64_t pitch, bool f64) {
  const int64_t tile = f64 ? kThreads * kVecF64 * 2 : kThreads * kVecF32 * 4;
  return (pitch + tile - 1) / tile;
}

void launch_gsm(const GsmArgs& a, bool f64, bool operator_mode, cudaStream_t s) {
  if (a.m <= 0 || a.pitch <= 0) return;
  GSGP_REQUIRE(a.pitch % 32 == 0, "storage pitch must be a multiple of 32");
  const int64_t ntiles = gsm_tiles(a.pitch, f64);
  const int64_t ngroups = (a.m + kRowsPerBlock - 1) / kRowsPerBlock;
  const int64_t blocks = ntiles * ngroups;
  GSGP_REQUIRE(blocks < (1ll << 31), "generation grid too large");
  if (f64) {
    if (operator_mode)
      k_gsm<double, true, kVecF64, kRowsPerBlock><<<(unsigned)blocks, kThreads, 0, s>>>(a, ntiles, ngroups);
    else
      k_gsm<double, false, kVecF64, kRowsPerBlock><<<(unsigned)blocks, kThreads, 0, s>>>(a, ntiles, ngroups);
  } else {
    if (operator_mode)
      k_gsm<float, true, kVecF32, kRowsPerBlock><<<(unsigned)blocks, kThreads, 0, s>>>(a, ntiles, ngroups);
    else
      k_gsm<float, false, kVecF32, kRowsPerBlock><<<(unsigned)blocks, kThreads, 0, s>>>(a, ntiles, ngroups);
  }
  GSGP_CUDA(cudaGetLastError());
}

}  // namespace gsgp
