// ComputeSemantics on sm_100a: genome compile + link + case-parallel fp64
// interpreter.
//
// Reference semantics (gsgp/interpreter.py:45-119): postfix scan with a LIFO
// stack; a function fires only when two operands are stacked (else it is
// skipped), left operand = second pop, protected division gives 1.0 when
// |den| < eps, and the program value is the last fired result, else the
// stack top, else 0.0.  Whether a gene fires depends only on the tag
// sequence (interpreter.py:10-15), so each genome is compiled ONCE into the
// expression tree rooted at its output node:
//   * skipped genes and every gene outside that tree are dropped (dead code);
//   * subtrees without a feature are folded to a constant with the same
//     fp64 operations (bit-identical: each node is a pure IEEE function of
//     its children);
//   * children are evaluated in Sethi-Ullman order on a one-operand
//     accumulator machine (common.cuh InsKind): every instruction combines
//     the accumulator with ONE operand x — a feature, a constant-table entry
//     or a spill slot whose index is static — so the interpreter fetches x
//     with a single shared-memory address and branches once, on an 8-way
//     kind.  A node with two leaf children is one L* instruction (x OP y);
//     a spill (PUSH) is always followed by the LOAD that starts the other
//     subtree, so the two fuse into PUSHLOAD (then the leaf pair is
//     PUSHLOAD x + OP y).  ADD/MUL with the accumulator on the
//     right use commutativity (IEEE + and * are commutative bit for bit);
//     SUB/DIV use the reversed kinds RSUB/RDIV, so every operand keeps its
//     role and every node still rounds exactly once.
// k_link rewrites the abstract operands into byte offsets of the chosen
// launch configuration (case tile, shared-memory row layout) once per
// launch.  The evaluator runs one thread per fitness case (CPT cases per
// thread); each block stages a genome's program and constant table in
// shared memory and walks it with broadcast loads.
#include <cstdlib>

#include "kernels.cuh"

namespace gsgp {
namespace {
#include "interp_dispatch.inc"
}  // namespace
}  // namespace gsgp

namespace gsgp {

namespace {

constexpr uint8_t F_EXISTS = 0x80, F_CONST = 0x40, F_FEAT = 0x20, F_NEED = 0x1f;

__device__ __forceinline__ bool is_leaf(uint8_t f) { return (f & (F_CONST | F_FEAT)) != 0; }

__device__ __forceinline__ Ins abstract_ins(uint32_t kind, uint32_t cls, uint32_t idx, uint32_t push,
                                            uint32_t ycls = 0, uint32_t yidx = 0) {
  Ins in;
  in.a = kind | (cls << 8) | (ycls << 12) | (push << 16);
  in.b = idx;
  in.c = yidx;
  in.d = 0;
  return in;
}

// one thread per genome.  Its working arrays (constant values, the stack,
// child links, the emission work stack: 25 B per gene, and the flags) live in
// shared memory when a few genomes' worth fit (k <= ~8k), else in per-genome
// global scratch: the per-thread walks are latency-bound, and global scratch
// went to L2 on every access (C1/C3 compile 1.3-1.4 ms, most of C1's init).
constexpr size_t kCompileSmemCap = 192 * 1024;
constexpr size_t compile_thread_bytes(int32_t k) { return ((size_t)k * (8 + 4 * 4 + 1) + 31) / 16 * 16; }
__global__ void k_compile(const uint8_t* __restrict__ tags, const int32_t* __restrict__ codes,
                          const double* __restrict__ consts, int64_t count, int32_t k, double eps,
                          Program P, bool in_smem) {
  extern __shared__ __align__(16) unsigned char csm[];
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= count) return;
  const uint8_t* T = tags + g * k;
  const int32_t* C = codes + g * k;
  const double* V = consts + g * k;
  double* cv;
  int32_t* stk;
  uint8_t* fl;
  if (in_smem) {
    unsigned char* base = csm + threadIdx.x * compile_thread_bytes(k);
    cv = reinterpret_cast<double*>(base);
    stk = reinterpret_cast<int32_t*>(base + (size_t)k * 8);
    fl = base + (size_t)k * 24;
  } else {
    cv = P.cval + g * (int64_t)k;
    stk = P.scratch + g * 4 * (int64_t)k;
    fl = P.flags + g * (int64_t)k;
  }
  int32_t* Lc = stk + k;
  int32_t* Rc = Lc + k;
  int32_t* work = Rc + k;
  Ins* out = P.code + g * (int64_t)(k + 1);
  double* ctab = P.ctab + g * (int64_t)k;

  // ---- structural scan (interpreter.py:53-70) with attributes in postfix order
  int32_t sp = 0, last = -1;
  for (int32_t j = 0; j < k; ++j) {
    uint8_t t = T[j];
    if (t == TAG_FUNCTION) {
      if (sp < 2) { fl[j] = 0; continue; }          // skipped: operands unavailable
      int32_t r = stk[--sp], l = stk[--sp];
      Lc[j] = l; Rc[j] = r;
      stk[sp++] = j;
      last = j;
      uint8_t fa = fl[l], fb = fl[r];
      if ((fa & F_CONST) && (fb & F_CONST)) {
        cv[j] = apply_op(C[j], cv[l], cv[r], eps);   // constant folding, same IEEE op
        fl[j] = F_EXISTS | F_CONST;
      } else {
        bool la = is_leaf(fa), lb = is_leaf(fb);
        int na = la ? 0 : (fa & F_NEED), nb = lb ? 0 : (fb & F_NEED);
        int need;
        if (la && lb) need = 0;
        else if (lb) need = na;
        else if (la) need = nb;
        else need = (na == nb) ? na + 1 : (na > nb ? na : nb);
        fl[j] = F_EXISTS | (uint8_t)(need < F_NEED ? need : F_NEED);
      }
    } else if (t == TAG_FEATURE) {
      fl[j] = F_EXISTS | F_FEAT;
      stk[sp++] = j;
    } else {
      fl[j] = F_EXISTS | F_CONST;
      cv[j] = V[j];
      stk[sp++] = j;
    }
  }
  int32_t root = last >= 0 ? last : (sp > 0 ? stk[sp - 1] : -1);

  int32_t pc = 0, nc = 0, depth = 0;
  int32_t ssp = 0;            // static spill-stack pointer
  int32_t pending = -1;       // slot of a PUSH waiting for the next LOAD
  // operand class / index of the leaf node n (constants go to the table)
  auto leaf = [&](int32_t n, uint32_t& cls, uint32_t& idx) {
    if (fl[n] & F_CONST) { cls = X_CONST; idx = (uint32_t)nc; ctab[nc++] = cv[n]; }
    else { cls = X_FEAT; idx = (uint32_t)C[n]; }
  };
  // emit an instruction whose operand is the leaf node n
  auto emit_leaf = [&](uint32_t kind, int32_t n) {
    uint32_t cls, idx;
    leaf(n, cls, idx);
    uint32_t push = 0;
    if (pending >= 0) {       // the spill fuses with the LOAD that follows it
      if (kind != K_LOAD) __trap();
      kind = K_PUSHLOAD;
      push = (uint32_t)pending;
      pending = -1;
    }
    out[pc++] = abstract_ins(kind, cls, idx, push);
  };
  // acc = acc OP x  (x is the right operand)
  auto fwd = [](int32_t op) -> uint32_t { return (uint32_t)op; };       // OP_* == K_* for 0..3
  // acc = x OP acc  (x is the left operand)
  auto rev = [](int32_t op) -> uint32_t {
    return op == OP_SUB ? K_RSUB : (op == OP_DIV ? K_RDIV : (uint32_t)op);
  };

  if (root < 0) {
    out[pc++] = abstract_ins(K_LOAD, X_CONST, 0, 0);
    ctab[nc++] = 0.0;
  } else if (is_leaf(fl[root])) {
    emit_leaf(K_LOAD, root);
  } else {
    // ---- iterative Sethi-Ullman emission; frame = node*4 + state
    int32_t top = 0;
    work[top++] = root * 4;
    while (top > 0) {
      const int32_t fr = work[top - 1];
      const int32_t n = fr >> 2, st = fr & 3;
      const int32_t l = Lc[n], r = Rc[n];
      const bool la = is_leaf(fl[l]), lb = is_leaf(fl[r]);
      const bool left_first = (!la && !lb) ? ((fl[l] & F_NEED) >= (fl[r] & F_NEED)) : !la;
      const int32_t op = C[n];
      if (st == 0) {
        if (la && lb) {
          uint32_t xc, xi, yc, yi;
          leaf(l, xc, xi);
          leaf(r, yc, yi);
          if (pending >= 0) {                 // spill, then acc = l OP r
            out[pc++] = abstract_ins(K_PADD + (uint32_t)op, xc, xi, (uint32_t)pending, yc, yi);
            pending = -1;
          } else {                            // acc = l OP r
            out[pc++] = abstract_ins(K_LADD + (uint32_t)op, xc, xi, 0, yc, yi);
          }
          --top;
        } else {
          work[top - 1] = n * 4 + 1;
          work[top++] = (left_first ? l : r) * 4;
        }
      } else if (st == 1) {
        if (lb) { emit_leaf(fwd(op), r); --top; }          // acc = L OP r
        else if (la) { emit_leaf(rev(op), l); --top; }     // acc = l OP R
        else {                                             // spill, evaluate the other child
          pending = ssp++;
          if (ssp > depth) depth = ssp;
          work[top - 1] = n * 4 + 2;
          work[top++] = (left_first ? r : l) * 4;
        }
      } else {                                             // both children non-leaf
        const uint32_t slot = (uint32_t)(--ssp);
        // left evaluated first: stack = L, acc = R -> x OP acc; else stack = R, acc = L
        out[pc++] = abstract_ins(left_first ? rev(op) : fwd(op), X_STACK, slot, 0);
        --top;
      }
    }
  }
  P.len[g] = pc;
  P.nconst[g] = nc;
  if (P.ndiv) {   // op mix for the rooflines (bench.py interp_line)
    // [divisions (8 fp64 ops + MUFU each), per-case operand loads (feature /
    //  spill rows), constant operand loads (broadcast), spill stores]
    int32_t nd = 0, nv = 0, nk = 0, ns = 0;
    for (int32_t i = 0; i < pc; ++i) {
      const uint32_t a = out[i].a, kd = a & 0xff;
      nd += (kd == K_DIV || kd == K_RDIV || kd == K_LDIV || kd == K_PDIV) ? 1 : 0;
      const uint32_t xc = (a >> 8) & 0xf, yc = (a >> 12) & 0xf;
      (xc == X_CONST ? nk : nv) += 1;
      if (kd >= K_LADD) (yc == X_CONST ? nk : nv) += 1;
      ns += (kd == K_PUSHLOAD || kd >= K_PADD) ? 1 : 0;
    }
    P.ndiv[4 * g] = nd;
    P.ndiv[4 * g + 1] = nv;
    P.ndiv[4 * g + 2] = nk;
    P.ndiv[4 * g + 3] = ns;
  }
  atomicMax(P.maxima, depth);
  atomicMax(P.maxima + 1, nc);
  atomicMax(P.maxima + 2, pc);
}

// ---------------------------------------------------------------- configurations
// (threads per block, cases per thread, features in shared memory?)  More
// cases per thread amortise the per-instruction dispatch; shared memory
// holds [features][spill slots][constant rows] of the block's case tile.
struct InterpCfg {
  int nt, cpt;
  bool xsmem;   // features of the tile in shared memory (else read from HBM/L2)
  bool lean;    // program and constants stay in HBM: only the spill rows use
                // shared memory, so any program size fits (huge k fallback)
  int groups = 1;   // genome groups per block sharing one staged feature tile
                    // (each group: nt threads, its own spill/constant rows + program);
                    // 0: as many one-warp groups as shared memory holds (warp_groups)
};
constexpr InterpCfg kCfgs[] = {{128, 4, true, false}, {64, 8, true, false}, {128, 4, false, false},
                               {128, 2, true, false}, {128, 1, false, true}, {128, 3, true, false},
                               {128, 3, true, false, 2}, {128, 4, true, false, 2},
                               {0, 0, false, false, 0},   // 8: retired (register-feature interpreter)
                               {32, 4, true, false, 0},
                               {128, 4, true, false, 4}};
constexpr int kCfgRetired = 8;
constexpr int kCfgWarps = 9;   // one-warp genome groups on a 128-case feature tile
constexpr int kNumCfgs = sizeof(kCfgs) / sizeof(kCfgs[0]);
constexpr size_t kSmemCap = 200 * 1024;

// rows of the case tile + the staged program (16 B per instruction)
// rows of one genome group: spill slots + constant rows
size_t cfg_group_rows(const InterpCfg& c, const InterpArgs& a) {
  const size_t crows = c.lean ? 0 : ((size_t)(a.maxconst > 0 ? a.maxconst : 1) + c.nt - 1) / c.nt;
  return (size_t)a.maxdepth + crows;
}
size_t cfg_rows_bytes(const InterpCfg& c, const InterpArgs& a, int groups) {
  const size_t rowb = (size_t)c.nt * c.cpt * 8;
  return ((c.xsmem ? (size_t)a.l : 0) + groups * cfg_group_rows(c, a)) * rowb;
}
// + 1 instruction per program: the loop prefetches one past the end
size_t cfg_prog_bytes(const InterpArgs& a) { return (size_t)((a.maxlen > 0 ? a.maxlen : 1) + 1) * sizeof(Ins); }
// one-warp genome groups stage their program through a ring of two
// kRingChunk-instruction chunks (+ one mirror slot, so the one-ahead
// instruction fetch never wraps) refilled as the warp walks the program:
// 1 KB per warp instead of the whole program (3.5 KB at k = 1024), so more
// warps fit beside a wide feature tile
constexpr int kRingChunk = 32;
constexpr size_t kRingBytes = (2 * kRingChunk + 1) * sizeof(Ins);
size_t cfg_group_prog_bytes(const InterpCfg& c, const InterpArgs& a) {
  return c.groups == 0 ? kRingBytes : cfg_prog_bytes(a);
}
size_t cfg_smem(const InterpCfg& c, const InterpArgs& a, int groups) {
  if (c.lean) return cfg_rows_bytes(c, a, groups) + 16;
  return cfg_rows_bytes(c, a, groups) + groups * cfg_group_prog_bytes(c, a);
}
// one-warp genome groups: as many as the shared memory (one block per SM)
// and the linked copies hold, at most kMaxWarpGroups warps (the kernel's
// register budget: 80 at 24 warps); 0 if fewer than 8 fit
#ifndef GSGP_WARP_SMEM_KB
#define GSGP_WARP_SMEM_KB 226   // 220: C5 pop+pool 654 ms, 226: 635 ms (profiles/r02/interp/ab_warp_smem_cap.log)
#endif
constexpr size_t kSmemCapWarps = GSGP_WARP_SMEM_KB * 1024;
#ifndef GSGP_WARP_UNROLL
#define GSGP_WARP_UNROLL 2
#endif
#ifndef GSGP_BLOCK_UNROLL
#define GSGP_BLOCK_UNROLL 4
#endif
constexpr int kMaxWarpGroups = 24;
int warp_groups(const InterpArgs& a) {
  const InterpCfg& c = kCfgs[kCfgWarps];
  const size_t base = cfg_smem(c, a, 0), per = cfg_smem(c, a, 1) - base;
  int gmax = base < kSmemCapWarps && per > 0 ? (int)((kSmemCapWarps - base) / per) : 0;
  gmax = std::min(gmax, std::min(kMaxWarpGroups, (int)a.max_groups));
  return gmax >= 8 ? gmax : 0;
}
size_t cfg_smem(const InterpCfg& c, const InterpArgs& a) {
  return cfg_smem(c, a, c.groups ? c.groups : warp_groups(a));
}

int choose_cfg(const InterpArgs& a) {
  const char* env = getenv("GSGP_INTERP_CFG");   // experiments / tests (read per launch)
  const int forced = env ? atoi(env) : -1;
  if (forced == kCfgWarps && warp_groups(a) > 0) return forced;
  if (forced >= 0 && forced < kNumCfgs && forced != kCfgWarps && forced != kCfgRetired &&
      cfg_smem(kCfgs[forced], a) <= kSmemCap && kCfgs[forced].groups <= a.max_groups)
    return forced;
  // two genome groups of 128 x 4 per block (cfg 7, compiled for 3 resident
  // blocks = 24 warps) when shared memory keeps 3 of them per SM: measured
  // 2.8 % faster at C3 than 128 x 3 groups with 32 warps (more cases per
  // dispatched instruction); the decision uses only shared memory, so it is
  // the same for every kernel instance and every rank
  // four genome groups of 128 x 4 per block (cfg 10: 16 warps, compiled
  // for 2 resident blocks = 32 warps at 64 registers, the epilogue state
  // recomputed so the program loop keeps spills to a few words) when shared
  // memory holds 2 of them: C2 20.0 -> 18.4 ms, C3 1770 -> 1688 ms, C4 233 ->
  // 227 ms against cfg 7 (profiles/r02/interp/ab_groups4.log)
  if (a.max_groups >= 4 && 2 * (cfg_smem(kCfgs[10], a) + 2048) <= 228 * 1024) return 10;
  if (a.max_groups >= 2 && 3 * (cfg_smem(kCfgs[7], a) + 2048) <= 228 * 1024) return 7;
  // features in shared memory while the tile keeps >= 3 blocks per SM; the
  // 384-case tile (128 x 3) fits 5 blocks (20 warps) where 128 x 4 fits 4:
  // measured 1-4 % faster (profiles/r01/README.md)
  if (cfg_smem(kCfgs[5], a) <= 45 * 1024) return 5;
  if (cfg_smem(kCfgs[0], a) <= 72 * 1024) return 0;
  // wide datasets (C5: 100 features, 400 KB per 512-case tile): one-warp
  // genome groups on a 128-case tile kept in shared memory, as many warps as
  // fit beside it (C5: 13), instead of feature operands from L2 —
  // C5 pop + pool 800 vs 1095 ms (profiles/r02/README.md)
  if (warp_groups(a) > 0) return kCfgWarps;
  if (cfg_smem(kCfgs[2], a) <= 72 * 1024) return 2;
  if (cfg_smem(kCfgs[2], a) <= kSmemCap) return 2;
  return 4;   // lean: spill rows only (depth <= 31 x 1 KB)
}

// ---------------------------------------------------------------- link
// abstract operand -> byte offset in the block's shared-memory row layout:
// rows [0, l) features (xsmem), then maxdepth spill slots, then constant rows
// (constant j: row j / nt, lane j % nt, replicated for the CPT cases)
// (grouped blocks: group gi's rows start grows * gi rows later; its linked
// copy is written at exe + gi * gstride)
__global__ void k_link(const Ins* __restrict__ code, Ins* __restrict__ exe, const int32_t* __restrict__ len,
                       int64_t count, int64_t k1, int32_t nt, uint32_t rowb, uint32_t frows,
                       uint32_t maxdepth, bool lean, int groups, uint32_t grows, int64_t gstride,
                       int64_t exe_k1) {
  const int64_t g = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;   // one warp per genome
  if (g >= count) return;
  const int32_t n = len[g];
  for (int gi = 0; gi < groups; ++gi) {
  const uint32_t gb = frows + (uint32_t)gi * grows;   // first row of this group
  // byte offset of an operand; vec = 1 for a per-case row, 0 for a constant
  auto off = [&](uint32_t cls, uint32_t idx, uint32_t& vec) -> uint32_t {
    vec = 1;
    if (cls == X_FEAT) return frows ? idx * rowb : (kFeatGlobal | idx);
    if (cls == X_STACK) return (gb + idx) * rowb;
    vec = 0;
    if (lean) return kConstGlobal | idx;
    return (gb + maxdepth + idx / (uint32_t)nt) * rowb + (idx % (uint32_t)nt) * 8u;
  };
  for (int32_t i = threadIdx.x % 32; i < n; i += 32) {
    const Ins in = code[g * k1 + i];
    const uint32_t kind = in.a & 0xff, xcls = (in.a >> 8) & 0xf, ycls = (in.a >> 12) & 0xf;
    const uint32_t push = in.a >> 16;
    uint32_t xvec, yvec = 0;
    Ins o;
    o.b = off(xcls, in.b, xvec);
    o.c = kind >= K_LADD ? off(ycls, in.c, yvec) : 0u;
    o.a = kind;
    // d: x lane mask in the low bits (tid*8 < 1024), y-is-vector bit 16,
    // push slot from bit 20 — so the interpreter uses a as the jump index as is
    o.d = (xvec ? 0x3ffu : 0u) | (yvec << 16) | (push << 20);
    exe[gi * gstride + g * exe_k1 + i] = o;
  }
  // a zero instruction after the program: the interpreter prefetches one
  // instruction past the end, and that read must see written memory
  if (threadIdx.x % 32 == 0) exe[gi * gstride + g * exe_k1 + n] = Ins{0u, 0u, 0u, 0u};
  }
}

// ---------------------------------------------------------------- interpret
// shared-memory accesses at a 32-bit address (the per-case stride becomes the
// instruction's immediate offset), so the base is computed once per instruction
__device__ __forceinline__ double lds_f64(uint32_t p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(p));
  return v;
}
__device__ __forceinline__ uint4 lds_u128(uint32_t p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(p));
  return v;
}


// the grouped launch is compiled for a register budget that lets shared
// memory decide the residency: 4 blocks = 32 warps at 64 registers (a third
// group per block — 36 warps at 56 registers — measured 5 % slower)
#ifndef GSGP_INTERP_MINB2
#define GSGP_INTERP_MINB2 4
#endif
// block barrier of one genome group (GROUPS > 1: named barrier 1 + group)
template <int GROUPS, int NT>
__device__ __forceinline__ void group_sync(int grp) {
  if constexpr (NT == 32) __syncwarp();        // one-warp groups
  else if constexpr (GROUPS == 1) __syncthreads();
  else asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(NT) : "memory");
}

// GROUPS > 1: the block runs GROUPS genome groups of NT threads on the same
// case tile; the staged features are shared, each group has its own spill
// and constant rows (grp_bytes apart) and program slot (prog_bytes apart),
// linked for it by k_link (copy `grp` of the linked programs).  GROUPS == 0:
// blockDim.x / NT groups (one-warp groups, NT == 32, sized at launch).
template <int NT, int CPT, int MODE, typename TOut, bool kXSmem, bool kLean, int GROUPS>
__global__ void __launch_bounds__(GROUPS ? NT * GROUPS : 32 * kMaxWarpGroups,
                                  GROUPS == 2 ? (CPT == 3 ? GSGP_INTERP_MINB2 : 3) : (GROUPS >= 3 ? 2 : 1)) k_interpret(InterpArgs a, int64_t gpb,
                                                           uint32_t stack_off, uint32_t crow_off,
                                                           uint32_t prog_off, uint32_t grp_bytes,
                                                           uint32_t prog_bytes) {
  constexpr int TILE = NT * CPT;
  constexpr uint32_t CSTRIDE = NT * 8;          // bytes between a thread's cases
  extern __shared__ __align__(16) unsigned char smem[];
  static_assert(GROUPS != 0 || NT == 32, "runtime genome groups are one warp each");
  const int ngr = GROUPS ? GROUPS : (int)(blockDim.x / NT);
  const int tid = GROUPS == 1 ? (int)threadIdx.x : (int)threadIdx.x % NT;
  const int grp = GROUPS == 1 ? 0 : (int)threadIdx.x / NT;
  stack_off += grp * grp_bytes;
  crow_off += grp * grp_bytes;
  prog_off += grp * prog_bytes;
  const uint32_t tid8 = (uint32_t)tid * 8u;
  const int64_t tile = blockIdx.x;             // tile of this launch's case range
  const int64_t l0 = tile * TILE;               // first case of the tile, launch-local
  const int64_t q0 = a.q_base + l0;             // ... and as a shard stacked index
  const int64_t N = a.ntr + a.nte;
  __shared__ double red[64];
  // one-warp groups claim genomes dynamically (block-local counter): warps
  // that drew short programs take more, so a block ends within about one
  // genome of its slowest warp (static round-robin left warps idle at the end
  // of every block: one block per SM)
  __shared__ unsigned claim;
  if (GROUPS == 0 && threadIdx.x == 0) claim = 0;
  if (GROUPS == 0) __syncthreads();

  if (kXSmem) {
    double* xs = reinterpret_cast<double*>(smem);
    for (int64_t e = threadIdx.x; e < (int64_t)a.l * TILE; e += NT * ngr) {
      const int64_t f = e / TILE, c = e - f * TILE;
      xs[e] = l0 + c < a.nq ? a.XT[f * a.xt_pitch + l0 + c] : 0.0;
    }
    if (GROUPS != 1) __syncthreads();           // the groups only sync among themselves below
  }
  // per-case bookkeeping of the epilogue, recomputed there (keeping it live
  // through the program loop costs ~20 registers): case c of this thread is
  // stacked case q0 + c * NT + tid; [ntr, te_q) is the test-start gap
  auto is_valid = [&](int c) {
    const int64_t q = q0 + c * NT + tid;
    return l0 + c * NT + tid < a.nq && (q < a.ntr || q >= a.te_q);
  };
  auto column = [&](int c) -> int64_t {     // storage column of case c
    const int64_t q = q0 + c * NT + tid, j = q - a.te_q;
    return q < a.ntr ? q : (j < a.te_full ? a.test_off + j : a.tail_off + (j - a.te_full));
  };
  uint32_t validm = 0;                      // HBM-feature fetches skip the cases past the range
#pragma unroll
  for (int c = 0; c < CPT; ++c) validm |= is_valid(c) ? 1u << c : 0u;
  const double* xg = a.XT + l0 + tid;          // global feature rows (!kXSmem)
  uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("" : "+r"(sbase));              // keep it in a register (no per-iteration remat)
  const uint32_t pbase = sbase + prog_off;
  const uint32_t sp0 = sbase + stack_off + tid8;   // this thread's spill slot 0, case 0
  // division fast path: denominators need |hi word| >= max(2^-500, hi(eps) + 1),
  // compared as f32 bit patterns (interp_dispatch.inc)
  const float dlo = __uint_as_float(max(523u << 20,
      (uint32_t)(__double_as_longlong(fabs(a.eps)) >> 32) + 1u));
  const int64_t cstride = a.k1 - 1;
  unsigned long long nonfinite = 0;

  // operand fetch: a shared-memory row / broadcast constant, or (features
  // left in HBM) a coalesced global row
  const double* cg = nullptr;                  // constants of the genome (kLean)
  auto fetch = [&](uint32_t off, uint32_t mask, double (&v)[CPT]) {
    if (kLean && (off & kConstGlobal)) {
      const double cv = __ldg(cg + (off & ~kConstGlobal));
#pragma unroll
      for (int c = 0; c < CPT; ++c) v[c] = cv;
    } else if (!kXSmem && (off & kFeatGlobal)) {
      const double* p = xg + (int64_t)(off & ~kFeatGlobal) * a.xt_pitch;
#pragma unroll
      for (int c = 0; c < CPT; ++c) v[c] = (validm >> c & 1u) ? __ldg(p + c * NT) : 0.0;
    } else {
      const uint32_t p = sbase + off + (tid8 & mask);
#pragma unroll
      for (int c = 0; c < CPT; ++c) v[c] = lds_f64(p + c * CSTRIDE);
    }
  };

  const int64_t g0 = blockIdx.y * gpb;
  const int64_t g1 = min(a.count, g0 + gpb);
  auto next_genome = [&](int64_t g) -> int64_t {
    if constexpr (GROUPS == 0) {
      unsigned c = 0;
      if (tid == 0) c = atomicAdd(&claim, 1u);
      return g0 + ngr + (int64_t)__shfl_sync(0xffffffffu, c, 0);
    } else {
      return g + ngr;
    }
  };
  for (int64_t g = g0 + grp; g < g1; g = next_genome(g)) {
    // ---- stage genome g: program + constant table (replicated for the CPT
    // cases of a thread) into shared memory
    const int len = a.len[g];
    cg = a.ctab + g * cstride;
    group_sync<GROUPS, NT>(grp);                // previous genome done with both (and red[])
    const uint4* psrc = reinterpret_cast<const uint4*>(a.exe + grp * a.exe_gstride + g * a.exe_k1);
    uint4 pre = make_uint4(0u, 0u, 0u, 0u);   // ring: chunk 2 of the program, staged at chunk 1
    if (!kLean) {
    {
      uint4* dst = reinterpret_cast<uint4*>(smem + prog_off);
      if constexpr (GROUPS == 0) {
        // (instructions 0..len: the program and the zero instruction after it)
        for (int i = tid; i < 2 * kRingChunk; i += NT)
          if (i <= len) dst[i] = __ldg(psrc + i);
        if (2 * kRingChunk + tid <= len) pre = __ldg(psrc + 2 * kRingChunk + tid);
      } else {
        for (int i = tid; i <= len; i += NT) dst[i] = __ldg(psrc + i);
      }
      const int nc = a.nconst[g];
      const double* ct = a.ctab + g * cstride;
      for (int e = tid; e < nc * CPT; e += NT) {
        const int j = e / CPT, c = e - j * CPT;
        *reinterpret_cast<double*>(smem + crow_off + (uint32_t)(j / NT) * (TILE * 8) +
                                   (uint32_t)(j % NT) * 8u + (uint32_t)c * CSTRIDE) = ct[j];
      }
    }
    group_sync<GROUPS, NT>(grp);
    }

    double acc[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) acc[c] = 0.0;
    const uint4* gprog = reinterpret_cast<const uint4*>(a.exe + g * a.exe_k1);   // kLean
    uint4 nxt = kLean ? __ldg(gprog) : lds_u128(pbase);
    // one-warp groups run every warp at its own program point, so the
    // dispatch code is an instruction-cache working set: unrolled 2x there
    // (1x: C3 1965 ms, 2x: 1840, 4x: 2410 — profiles/r02/interp); the
    // block-wide groups keep the compiler's 4x
    constexpr int kUnroll = NT == 32 ? GSGP_WARP_UNROLL : GSGP_BLOCK_UNROLL;
    // one program instruction over the CPT cases of this thread
    auto step = [&](const uint4& in) {
      double x[CPT];
      fetch(in.y, in.w, x);
      const uint32_t kind = in.x;
      // one warp-uniform jump (interp_dispatch.inc); each arm is straight-line
      // code over the CPT cases of this thread, one IEEE rounding per case
      if constexpr (kXSmem && !kLean && CPT != 1) {
        // leaf-pair arms fetch their second operand themselves
        DispatchY<CPT, CSTRIDE>::run(acc, x, kind, in.w, sp0, a.eps, dlo, in.z, sbase, tid8);
      } else {
        double y[CPT];
        if (kind >= K_LADD) fetch(in.z, (in.w & 0x10000u) ? 0xffffffffu : 0u, y);   // second leaf
        Dispatch<CPT, CSTRIDE>::run(acc, x, y, kind, in.w, sp0, a.eps, dlo);
      }
    };
    if constexpr (GROUPS == 0) {
      // program ring: chunk c lives in slot c & 1 (entry 2 * kRingChunk
      // mirrors the first instruction of the even chunk in flight).  At the
      // start of chunk c >= 1 the warp stores chunk c + 1 (loaded into
      // registers one chunk earlier) over chunk c - 1 and loads chunk c + 2.
      for (int i0 = 0; i0 < len; i0 += kRingChunk) {
        if (i0 > 0) {
          const int c = i0 / kRingChunk + 1;
          __syncwarp();                                  // every lane is done with chunk c - 2's slot
          uint4* ring = reinterpret_cast<uint4*>(smem + prog_off);
          ring[(c & 1) * kRingChunk + tid] = pre;
          if ((c & 1) == 0 && tid == 0) ring[2 * kRingChunk] = pre;
          __syncwarp();
          const int64_t nx = (int64_t)(c + 1) * kRingChunk + tid;
          if (nx <= len) pre = __ldg(psrc + nx);
        }
        const int jn = min(kRingChunk, len - i0);
        const uint32_t rbase = pbase + (uint32_t)(i0 & (2 * kRingChunk - 1)) * 16u;
#pragma unroll kUnroll
        for (int j = 0; j < jn; ++j) {
          const uint4 in = nxt;
          nxt = lds_u128(rbase + (uint32_t)(j + 1) * 16u);
          step(in);
        }
      }
    } else {
#pragma unroll kUnroll
    for (int i = 0; i < len; ++i) {
      const uint4 in = nxt;
      // next instruction (smem holds len + 1; the HBM program has k + 1 >= len + 1 slots)
      nxt = kLean ? __ldg(gprog + i + 1) : lds_u128(pbase + (uint32_t)(i + 1) * 16u);
      step(in);
    }
    }
    // ---- epilogue: non-finite -> 0.0 counted (core.py:348-356), then store
    double sse_tr = 0.0, sse_te = 0.0;
    int wide = 0;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      if (!(validm >> c & 1u)) continue;
      double v = acc[c];
      if (!isfinite(v) && !(MODE == INTERP_F64 && a.raw)) { v = 0.0; ++nonfinite; }
      const int64_t q = q0 + c * NT + tid;
      if (MODE == INTERP_F64) {
        a.out64[g * N + q] = v;
      } else if (MODE == INTERP_POP) {
        const int64_t col = column(c);
        const bool train = q < a.ntr;
        TOut o = (TOut)v;
        reinterpret_cast<TOut*>(a.out)[g * a.pitch + col] = o;
        if (isinf((double)o)) wide |= train ? 1 : 2;
        double d = __dsub_rn(v, __ldg(a.y + col));
        if (train) sse_tr = __dadd_rn(sse_tr, __dmul_rn(d, d));
        else sse_te = __dadd_rn(sse_te, __dmul_rn(d, d));
      } else {
        // sigmoid of the pool, once per run (mutation.py:32-34, evolution.py:135-136)
        double sg = __ddiv_rn(1.0, __dadd_rn(1.0, exp(-v)));
        reinterpret_cast<TOut*>(a.out)[g * a.pitch + column(c)] = (TOut)sg;
      }
    }
    if (MODE == INTERP_POP) {
      // fixed-order block reduction of the tile's SSE (train, test)
      sse_tr = warp_sum(sse_tr);
      sse_te = warp_sum(sse_te);
      int wb = __reduce_or_sync(0xffffffffu, wide);
      if constexpr (NT == 32) {   // one warp: the warp sum is the tile partial (0 + s == s)
        if (tid < 2) a.part[(g * a.part_ntiles + a.q_base / TILE + tile) * 2 + tid] = tid ? sse_te : sse_tr;
        if (tid == 0 && wb) atomicOr(a.wide + g, wb);
        continue;
      }
      double* gred = red + grp * (NT / 32) * 2;
      if ((tid & 31) == 0) {
        gred[(tid >> 5) * 2] = sse_tr;
        gred[(tid >> 5) * 2 + 1] = sse_te;
        if (wb) atomicOr(a.wide + g, wb);
      }
      group_sync<GROUPS, NT>(grp);
      if (tid < 2) {
        double t = 0.0;
        for (int w = 0; w < NT / 32; ++w) t = __dadd_rn(t, gred[w * 2 + tid]);
        a.part[(g * a.part_ntiles + a.q_base / TILE + tile) * 2 + tid] = t;
      }
    }
  }
  // block total of replaced elements (integer: order-independent)
  for (int o = 16; o > 0; o >>= 1) nonfinite += __shfl_xor_sync(0xffffffffu, nonfinite, o);
  if ((tid & 31) == 0 && nonfinite) atomicAdd(a.nonfinite, nonfinite);
}

template <int NT, int CPT, int MODE, typename TOut, bool kXSmem, bool kLean = false, int GROUPS = 1>
void launch_cfg(const InterpArgs& a0, cudaStream_t s) {
  constexpr int TILE = NT * CPT;
  constexpr InterpCfg c{NT, CPT, kXSmem, kLean, GROUPS};
  static_assert(GROUPS == 1 || (kXSmem && !kLean), "grouped blocks share a staged feature tile");
  const int G = GROUPS ? GROUPS : warp_groups(a0);
  GSGP_REQUIRE(G >= 1 && G <= a0.max_groups, "not enough linked program copies for the genome groups");
  InterpArgs a = a0;
  a.exe_gstride = a.count * a.exe_k1;   // group copies of this launch's linked programs
  const int64_t ntiles = (a.nq + TILE - 1) / TILE;
  GSGP_REQUIRE(a.te_q >= a.ntr && (a.nte == 0 || a.te_q % TILE == 0 || a.te_q == a.ntr),
               "test cases must start on an interpreter tile");
  GSGP_REQUIRE(a.q_base % TILE == 0 && a.q_base + a.nq <= a.te_q + a.nte, "bad interpreter case range");
  const uint32_t rowb = TILE * 8;
  const uint32_t frows = kXSmem ? (uint32_t)a.l : 0u;
  const size_t smem = cfg_smem(c, a, G);
  GSGP_REQUIRE(smem <= (GROUPS ? kSmemCap : kSmemCapWarps), "interpreter tile does not fit in shared memory");
  // link the programs for this row layout
  const uint32_t grows = (uint32_t)cfg_group_rows(c, a);
  k_link<<<(unsigned)((a.count + 3) / 4), 128, 0, s>>>(a.code, a.exe, a.len, a.count, a.k1, NT, rowb,
                                                      frows, (uint32_t)a.maxdepth, kLean, G, grows,
                                                      a.exe_gstride, a.exe_k1);
  GSGP_CUDA(cudaGetLastError());
  // genomes per block: enough blocks to fill 148 SMs several times over
  // (one-warp groups: one block per SM, genomes per block a multiple of G)
  const int64_t want = GROUPS ? 148 * 8 : 148 * 16;
  int64_t gpb = (a.count * ntiles + want - 1) / want;
  if (GROUPS) {
    gpb = std::max<int64_t>(1, std::min<int64_t>(gpb, 64));
  } else {
    gpb = std::max<int64_t>(gpb, G);
    gpb = std::min<int64_t>((gpb + G - 1) / G * G, (a.count + G - 1) / G * G);
  }
  const int64_t gy = (a.count + gpb - 1) / gpb;
  GSGP_REQUIRE(gy <= 65535, "too many genome groups");
  dim3 grid((unsigned)ntiles, (unsigned)gy);
  auto k = k_interpret<NT, CPT, MODE, TOut, kXSmem, kLean, GROUPS>;
  GSGP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k<<<grid, NT * G, smem, s>>>(a, gpb, frows * rowb, (frows + (uint32_t)a.maxdepth) * rowb,
                               (uint32_t)cfg_rows_bytes(c, a, G), grows * rowb,
                               (uint32_t)cfg_group_prog_bytes(c, a));
  GSGP_CUDA(cudaGetLastError());
}

// 128x3 tiles: 1 or 2 genome groups per block (cfg 5, 6) share the staged
// feature tile; when shared memory limits the resident blocks the grouped
// launch holds more warps per SM.  The occupancy calculator picks the one
// with more resident warps (ties: one group) unless GSGP_INTERP_CFG forces a
// configuration (GSGP_INTERP_TRACE=1 prints the numbers).
template <int MODE, typename TOut, int GROUPS>
int resident_warps(const InterpArgs& a) {
  const InterpCfg& c = kCfgs[4 + GROUPS];
  const size_t sm = cfg_smem(c, a);
  if (sm > kSmemCap || GROUPS > a.max_groups) return 0;
  auto k = k_interpret<128, 3, MODE, TOut, true, false, GROUPS>;
  int b = 0;
  GSGP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  GSGP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, 128 * GROUPS, sm));
  if (getenv("GSGP_INTERP_TRACE")) {
    cudaFuncAttributes f{};
    cudaFuncGetAttributes(&f, k);
    fprintf(stderr, "interp 128x3 x%d groups: %d blocks, %zu B shared, %d regs\n", GROUPS, b, sm, f.numRegs);
  }
  return b * 4 * GROUPS;
}

template <int MODE, typename TOut>
int grouped_or_single(const InterpArgs& a) {
  if (getenv("GSGP_INTERP_CFG")) return 5;
  const int w1 = resident_warps<MODE, TOut, 1>(a), w2 = resident_warps<MODE, TOut, 2>(a);
  return w2 > w1 ? 6 : 5;
}

template <int MODE, typename TOut>
void launch_mode(const InterpArgs& a, cudaStream_t s) {
  int cfg = choose_cfg(a);
  if (cfg == 5) cfg = grouped_or_single<MODE, TOut>(a);
  switch (cfg) {
    case 0: launch_cfg<128, 4, MODE, TOut, true>(a, s); break;
    case 1: launch_cfg<64, 8, MODE, TOut, true>(a, s); break;
    case 2: launch_cfg<128, 4, MODE, TOut, false>(a, s); break;
    case 3: launch_cfg<128, 2, MODE, TOut, true>(a, s); break;
    case 5: launch_cfg<128, 3, MODE, TOut, true>(a, s); break;
    case 6: launch_cfg<128, 3, MODE, TOut, true, false, 2>(a, s); break;
    case 7: launch_cfg<128, 4, MODE, TOut, true, false, 2>(a, s); break;
    case kCfgWarps: launch_cfg<32, 4, MODE, TOut, true, false, 0>(a, s); break;
    case 10: launch_cfg<128, 4, MODE, TOut, true, false, 4>(a, s); break;
    default: launch_cfg<128, 1, MODE, TOut, false, true>(a, s); break;
  }
}

// CUDA loads a kernel lazily at its first launch (milliseconds for the large
// dispatch kernels); interp_preload() loads every interpreter kernel of the
// module up front so no timed stage of a run pays for it
template <typename K>
void preload_fn(K k) {
  cudaFuncAttributes f{};
  GSGP_CUDA(cudaFuncGetAttributes(&f, k));
}
template <int MODE, typename TOut>
void preload_mode() {
  preload_fn(k_interpret<128, 4, MODE, TOut, true, false, 1>);
  preload_fn(k_interpret<64, 8, MODE, TOut, true, false, 1>);
  preload_fn(k_interpret<128, 4, MODE, TOut, false, false, 1>);
  preload_fn(k_interpret<128, 2, MODE, TOut, true, false, 1>);
  preload_fn(k_interpret<128, 3, MODE, TOut, true, false, 1>);
  preload_fn(k_interpret<128, 3, MODE, TOut, true, false, 2>);
  preload_fn(k_interpret<128, 4, MODE, TOut, true, false, 2>);
  preload_fn(k_interpret<128, 4, MODE, TOut, true, false, 4>);
  preload_fn(k_interpret<32, 4, MODE, TOut, true, false, 0>);
  preload_fn(k_interpret<128, 1, MODE, TOut, false, true, 1>);
}

}  // namespace

void interp_preload() {
  preload_fn(k_compile);
  preload_fn(k_link);
  preload_mode<INTERP_F64, double>();
  preload_mode<INTERP_POP, float>();
  preload_mode<INTERP_POP, double>();
  preload_mode<INTERP_POOL, float>();
  preload_mode<INTERP_POOL, double>();
}

void launch_compile(const uint8_t* tags, const int32_t* codes, const double* consts, int64_t count,
                    int32_t k, double eps, Program prog, cudaStream_t s) {
  if (count <= 0) return;
  GSGP_CUDA(cudaMemsetAsync(prog.maxima, 0, 4 * sizeof(int32_t), s));   // all four maxima
  const size_t per = compile_thread_bytes(k);
  const bool in_smem = per <= kCompileSmemCap / 2;
  // shared-memory scratch: as many genomes per block as fit (<= 64), and at
  // least two blocks' worth of genomes spread over the SMs
  const int tpb = in_smem ? (int)std::min<size_t>(64, kCompileSmemCap / per) : 64;
  const size_t smem = in_smem ? (size_t)tpb * per : 0;
  if (in_smem)
    GSGP_CUDA(cudaFuncSetAttribute(k_compile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_compile<<<(unsigned)((count + tpb - 1) / tpb), tpb, smem, s>>>(tags, codes, consts, count, k, eps, prog,
                                                                   in_smem);
  GSGP_CUDA(cudaGetLastError());
}

int interp_config(const InterpArgs& a) { return choose_cfg(a); }

int64_t interp_tiles(const InterpArgs& a, int* tile_out) {
  const InterpCfg c = kCfgs[choose_cfg(a)];
  const int64_t tile = (int64_t)c.nt * c.cpt;
  if (tile_out) *tile_out = (int)tile;
  return (a.te_q + a.nte + tile - 1) / tile;
}

void launch_interpret(const InterpArgs& a, int mode, cudaStream_t s) {
  if (a.count <= 0 || a.nq <= 0) return;
  GSGP_REQUIRE(a.maxdepth <= 31, "spill stack deeper than the compiler's labels");
  if (mode == INTERP_F64) launch_mode<INTERP_F64, double>(a, s);
  else if (mode == INTERP_POP) {
    if (a.out_is_f64) launch_mode<INTERP_POP, double>(a, s);
    else launch_mode<INTERP_POP, float>(a, s);
  } else {
    if (a.out_is_f64) launch_mode<INTERP_POOL, double>(a, s);
    else launch_mode<INTERP_POOL, float>(a, s);
  }
}

}  // namespace gsgp
