// Shared device helpers for the B200 GSGP engine (sm_100a).
//
// Everything here is bit-exact with the reference's numpy arithmetic: the
// counter RNG is integer-only, and every floating-point step that the
// reference rounds separately is written with explicit _rn intrinsics so
// nvcc can never contract it into an FMA (the library is additionally built
// with -fmad=false).
#pragma once

#include <cstdint>
#include <cstdio>
#include <cmath>
#include <string>
#include <cuda_runtime.h>

namespace gsgp {

// ---------------------------------------------------------------- status
enum Status : int { OK = 0, ERR_CONFIG = 1, ERR_CUDA = 2, ERR_NCCL = 3, ERR_OOM = 4 };

void set_error(const std::string& msg);          // thread-local last error (capi.cu)

struct Error {
  int code;
  std::string msg;
};

#define GSGP_CUDA(expr)                                                                  \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess) {                                                             \
      throw ::gsgp::Error{_e == cudaErrorMemoryAllocation ? ::gsgp::ERR_OOM              \
                                                          : ::gsgp::ERR_CUDA,            \
                          std::string(#expr) + ": " + cudaGetErrorString(_e)};           \
    }                                                                                    \
  } while (0)

#define GSGP_REQUIRE(cond, msg)                                                          \
  do {                                                                                   \
    if (!(cond)) throw ::gsgp::Error{::gsgp::ERR_CONFIG, (msg)};                         \
  } while (0)

// ------------------------------------------------------- counter RNG (rng.py)
// splitmix64 constants, reference gsgp/rng.py:16-28
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kStreamMult = 0xC2B2AE3D27D4EB4Full;
constexpr uint64_t kMixA = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kMixB = 0x94D049BB133111EBull;
constexpr uint64_t kSeedXor = 0x8538ECB5BD456EA3ull;
constexpr uint64_t kPlanStream0 = 1ull << 32;

__host__ __device__ __forceinline__ uint64_t sm64_finalize(uint64_t z) {
  z = (z ^ (z >> 30)) * kMixA;
  z = (z ^ (z >> 27)) * kMixB;
  return z ^ (z >> 31);
}

// per-(seed, stream) base state, rng.py:39-40
__host__ __device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t stream) {
  return sm64_finalize(sm64_finalize(seed ^ kSeedXor) + stream * kStreamMult);
}

// 64 bits at (key, counter), rng.py:43-45
__host__ __device__ __forceinline__ uint64_t draw_bits(uint64_t key, uint64_t counter) {
  return sm64_finalize(key + counter * kGolden);
}

// U[0,1) = (bits >> 11) * 2^-53, rng.py:48-50 (both steps exact in fp64)
__host__ __device__ __forceinline__ double draw_unit(uint64_t key, uint64_t counter) {
  return (double)(draw_bits(key, counter) >> 11) * 0x1p-53;
}

// ------------------------------------------------------------ genome coding
enum GeneTag : uint8_t { TAG_FUNCTION = 0, TAG_FEATURE = 1, TAG_CONSTANT = 2 };   // core.py:41-44
enum FunctionOp : int32_t { OP_ADD = 0, OP_SUB = 1, OP_MUL = 2, OP_DIV = 3 };      // core.py:47-51

// One instruction of a compiled (dead-code-eliminated, constant-folded,
// Sethi-Ullman ordered) genome for the accumulator machine of interp.cu.
// Every instruction reads one operand x (a feature, a constant-table entry
// or a static spill-stack slot) and combines it with the accumulator; a
// node with two leaf children reads a second leaf y instead, and when it
// starts the second subtree of a spill (the common case: a spill is always
// followed by such a node) the spill is fused in (P* kinds):
//   ADD acc+x  SUB acc-x  MUL acc*x  DIV |x|<eps ? 1 : acc/x
//   RSUB x-acc RDIV |acc|<eps ? 1 : x/acc  LOAD acc=x  PUSHLOAD slot=acc, acc=x
//   LADD x+y   LSUB x-y   LMUL x*y   LDIV |y|<eps ? 1 : x/y
//   PADD..PDIV slot=acc, then acc = x op y
// k_compile emits the abstract form (operand class + index); k_link rewrites
// it for one interpreter configuration into shared-memory byte offsets, so
// the interpreter fetches x with one address computation and branches once.
enum InsKind : uint32_t { K_ADD = 0, K_SUB = 1, K_MUL = 2, K_DIV = 3, K_RSUB = 4, K_RDIV = 5,
                          K_LOAD = 6, K_PUSHLOAD = 7, K_LADD = 8, K_LSUB = 9, K_LMUL = 10,
                          K_LDIV = 11, K_PADD = 12, K_PSUB = 13, K_PMUL = 14, K_PDIV = 15,
                          K_NUM_KINDS = 16 };
enum InsClass : uint32_t { X_FEAT = 0, X_CONST = 1, X_STACK = 2 };

struct __align__(16) Ins {
  // abstract (compile): a = kind | x class << 8 | y class << 12 | push slot << 16,
  //                     b = x index, c = y index (L*/P* kinds)
  // linked (interpret): a = kind, b = x byte offset, c = y byte offset (L*/P*),
  //                     d = x lane mask (0x3ff vector row, 0 broadcast constant)
  //                         | y-is-vector << 16 | push slot << 20;
  //                     feature offsets carry kFeatGlobal when features stay in HBM,
  //                     constants kConstGlobal in the lean (huge-program) configuration
  uint32_t a, b, c, d;
};
static_assert(sizeof(Ins) == 16, "Ins must be 16 bytes");
constexpr uint32_t kFeatGlobal = 0x80000000u;
constexpr uint32_t kConstGlobal = 0x40000000u;   // lean configuration: constant j read from HBM

// binary op with the reference's protected division (interpreter.py:58-65):
// each case rounds exactly once, as numpy does.
__host__ __device__ __forceinline__ double apply_op(int op, double a, double b, double eps) {
#ifdef __CUDA_ARCH__
  switch (op) {
    case OP_ADD: return __dadd_rn(a, b);
    case OP_SUB: return __dsub_rn(a, b);
    case OP_MUL: return __dmul_rn(a, b);
    default: return fabs(b) < eps ? 1.0 : __ddiv_rn(a, b);
  }
#else
  switch (op) {
    case OP_ADD: return a + b;
    case OP_SUB: return a - b;
    case OP_MUL: return a * b;
    default: return std::fabs(b) < eps ? 1.0 : a / b;
  }
#endif
}

// RMSE from an SSE, fitness.py:11-25 (non-finite -> +inf)
__host__ __device__ __forceinline__ double rmse_of(double sse, double n) {
#ifdef __CUDA_ARCH__
  double v = __dsqrt_rn(__ddiv_rn(sse, n));
#else
  double v = std::sqrt(sse / n);
#endif
  return isfinite(v) ? v : INFINITY;
}

// device control block (int64 words), written by init/survival kernels and
// read by the generation kernels so one captured generation is replayable
enum Ctl : int { CTL_GEN = 0, CTL_BP = 1, CTL_REDIRECT = 2, CTL_PARITY = 3, CTL_PARENT_ELITES = 4,
                 CTL_WORDS = 8 };

__host__ __device__ __forceinline__ int64_t pad32(int64_t n) { return (n + 31) & ~int64_t(31); }

// warp-level fp64 sum with a fixed butterfly order (deterministic)
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ------------------------------------------- canonical (order-free) SSE sums
// The SSE of a row is summed from fp64 tile partials (tiles anchored on
// global case positions, see engine.cu shard_range).  Adding the partials in
// floating point would make the result depend on how the tiles are split
// across shards and ranks; instead every partial v >= 0 is converted to a
// fixed-point integer X = floor(v * 2^(116 - A)) anchored on the row's largest
// partial exponent A (an exact max over all shards/ranks), the integers are
// summed exactly (u64 limbs of 32-bit digits: integer adds, any order, any
// NCCL reduction tree), and the total is rounded once to fp64.  The result is
// therefore a function of the multiset of partials only: bit-identical for
// any number of GPUs and virtual shards.  Truncated bits are < 2^(A-116) per
// partial, i.e. < ntiles * 2^-116 relative to the sum.
constexpr int kLimbs = 4;                      // digits 0..3 of X (X < 2^117)
constexpr int32_t kExpZero = -0x7f7f7f80;      // no non-zero partial (memset 0x80 is below it)
constexpr int32_t kExpInf = 0x7ffffff0;        // some partial is +inf
constexpr int32_t kExpNaN = 0x7fffffff;        // some partial is NaN
constexpr int kAnchor = 116;

__device__ __forceinline__ int32_t canon_exp(double v) {
  if (v != v) return kExpNaN;
  if (v == 0.0) return kExpZero;
  if (isinf(v)) return kExpInf;
  const uint64_t b = (uint64_t)__double_as_longlong(v);
  const int32_t ef = (int32_t)((b >> 52) & 0x7ff);
  if (ef) return ef - 1023;
  return -1074 + 63 - __clzll((long long)(b & ((1ull << 52) - 1)));   // subnormal
}

// add the digits of floor(v * 2^(kAnchor - A)) to L (A = canon_exp max, finite)
__device__ __forceinline__ void canon_add(double v, int32_t A, unsigned long long L[kLimbs]) {
  if (!(v > 0.0)) return;
  const uint64_t b = (uint64_t)__double_as_longlong(v);
  const int32_t ef = (int32_t)((b >> 52) & 0x7ff);
  const uint64_t M = (b & ((1ull << 52) - 1)) | (ef ? (1ull << 52) : 0ull);
  const int32_t sh = (ef ? ef - 1075 : -1074) + kAnchor - A;   // X = M * 2^sh, sh <= 64
  unsigned __int128 X;
  if (sh >= 0) X = (unsigned __int128)M << sh;
  else if (sh > -64) X = M >> (-sh);
  else return;
  L[0] += (uint32_t)X;
  L[1] += (uint32_t)(X >> 32);
  L[2] += (uint32_t)(X >> 64);
  L[3] += (uint32_t)(X >> 96);
}

// round sum(L[d] * 2^(32 d)) * 2^(A - kAnchor) to the nearest fp64 (ties even)
__device__ __forceinline__ double canon_finish(const unsigned long long L[kLimbs], int32_t A) {
  if (A == kExpNaN) return __longlong_as_double(0x7ff8000000000000ll);
  if (A == kExpInf) return __longlong_as_double(0x7ff0000000000000ll);
  if (A < -1100) return 0.0;
  unsigned __int128 acc = (unsigned __int128)L[0] + ((unsigned __int128)L[1] << 32);
  const uint64_t w0 = (uint64_t)acc;
  acc = (acc >> 64) + (unsigned __int128)L[2] + ((unsigned __int128)L[3] << 32);
  const uint64_t w1 = (uint64_t)acc, w2 = (uint64_t)(acc >> 64);
  int h;   // index of the leading bit of the 192-bit integer (w2:w1:w0)
  if (w2) h = 128 + 63 - __clzll((long long)w2);
  else if (w1) h = 64 + 63 - __clzll((long long)w1);
  else if (w0) h = 63 - __clzll((long long)w0);
  else return 0.0;
  // top 64 bits starting at the leading one, and whether anything below is set
  const int lo = h - 63;
  uint64_t top;
  bool below = false;
  if (lo <= 0) {
    top = w0 << (-lo);
  } else {
    const int q = lo >> 6, r = lo & 63;   // q in {0, 1, 2}
    const uint64_t wq = q == 0 ? w0 : (q == 1 ? w1 : w2);
    const uint64_t wn = q == 0 ? w1 : (q == 1 ? w2 : 0ull);
    top = r ? (wq >> r) | (wn << (64 - r)) : wq;
    below = (q >= 1 && w0 != 0) || (q >= 2 && w1 != 0);
    if (r) below |= (wq & ((1ull << r) - 1)) != 0;
  }
  uint64_t mant = top >> 11;
  const bool rnd = (top >> 10) & 1;
  const bool sticky = below || (top & 0x3ff) != 0;
  int e = h - 52;
  if (rnd && (sticky || (mant & 1))) {
    if (++mant == (1ull << 53)) { mant >>= 1; ++e; }
  }
  return ldexp((double)mant, e + A - kAnchor);
}

}  // namespace gsgp
