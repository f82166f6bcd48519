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

}  // namespace gsgp
