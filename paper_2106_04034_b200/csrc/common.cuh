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
// Sethi-Ullman ordered) genome.  The accumulator machine keeps the running
// value in a register; spills go to a per-case stack in shared memory.
enum InsOp : uint8_t { INS_ADD = 0, INS_SUB = 1, INS_MUL = 2, INS_DIV = 3, INS_LOAD = 4, INS_PUSH = 5 };
enum InsSrc : uint8_t { SRC_ACC = 0, SRC_POP = 1, SRC_FEAT = 2, SRC_CONST = 3 };

struct __align__(16) Ins {
  uint8_t op;    // InsOp
  uint8_t ls;    // InsSrc of the left operand (or the LOAD source)
  uint8_t rs;    // InsSrc of the right operand
  uint8_t kind;  // dense dispatch key 0..38, see ins_kind()
  uint16_t lf;   // feature index when ls == SRC_FEAT
  uint16_t rf;   // feature index when rs == SRC_FEAT
  double c;      // constant when ls or rs == SRC_CONST (never both)
};
static_assert(sizeof(Ins) == 16, "Ins must be 16 bytes");
// Dense dispatch keys: the 9 possible operand-source pairs of a binary op
// (index kPair[ls][rs]) x 4 operators = 0..35, LOAD feature 36, LOAD
// constant 37, PUSH 38.  Dense keys let the interpreter's switch compile to
// one jump table.
constexpr int kKindLoadFeat = 36, kKindLoadConst = 37, kKindPush = 38;
__host__ __device__ __forceinline__ int ins_pair(int ls, int rs) {
  // rows: ls = ACC, POP, FEAT, CONST; cols: rs = ACC, POP, FEAT, CONST
  constexpr int8_t kPair[4][4] = {{-1, 0, 2, 3}, {1, -1, -1, -1}, {4, -1, 6, 7}, {5, -1, 8, -1}};
  return kPair[ls][rs];
}
__host__ __device__ __forceinline__ uint8_t ins_kind(const Ins& in) {
  if (in.op == INS_PUSH) return kKindPush;
  if (in.op == INS_LOAD) return in.ls == SRC_FEAT ? kKindLoadFeat : kKindLoadConst;
  return (uint8_t)(ins_pair(in.ls, in.rs) * 4 + in.op);
}

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
