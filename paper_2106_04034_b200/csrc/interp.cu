// ComputeSemantics on sm_100a: genome compile + case-parallel fp64 interpreter.
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
//   * children are evaluated in Sethi-Ullman order with terminal operands
//     folded into the instruction, so the spill stack is <= log2(nodes)+1.
// The evaluator then runs one thread per fitness case (CPT cases per thread
// for ILP) over a block-uniform instruction stream — every branch is
// warp-uniform — with the block's feature tile and spill stacks in shared
// memory.
#include <cstdlib>

#include "kernels.cuh"

namespace gsgp {

namespace {

constexpr uint8_t F_EXISTS = 0x80, F_CONST = 0x40, F_FEAT = 0x20, F_NEED = 0x1f;

__device__ __forceinline__ bool is_leaf(uint8_t f) { return (f & (F_CONST | F_FEAT)) != 0; }

// one thread per genome; scratch is per-genome global memory
__global__ void k_compile(const uint8_t* __restrict__ tags, const int32_t* __restrict__ codes,
                          const double* __restrict__ consts, int64_t count, int32_t k, double eps,
                          Program P) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= count) return;
  const uint8_t* T = tags + g * k;
  const int32_t* C = codes + g * k;
  const double* V = consts + g * k;
  int32_t* stk = P.scratch + g * 4 * (int64_t)k;
  int32_t* Lc = stk + k;
  int32_t* Rc = Lc + k;
  int32_t* work = Rc + k;
  uint8_t* fl = P.flags + g * (int64_t)k;
  double* cv = P.cval + g * (int64_t)k;
  Ins* out = P.code + g * (int64_t)(k + 1);

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
        fl[j] = F_EXISTS | (uint8_t)need;
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

  auto leaf_src = [&](int32_t n, uint8_t& src, uint16_t& f, double& c) {
    if (fl[n] & F_CONST) { src = SRC_CONST; c = cv[n]; }
    else { src = SRC_FEAT; f = (uint16_t)C[n]; }
  };

  int32_t pc = 0;
  int depth = 0;
  if (root < 0 || is_leaf(fl[root])) {
    Ins in{};
    in.op = INS_LOAD;
    if (root < 0) { in.ls = SRC_CONST; in.c = 0.0; }
    else leaf_src(root, in.ls, in.lf, in.c);
    in.kind = ins_kind(in);
    out[pc++] = in;
  } else {
    depth = fl[root] & F_NEED;
    // ---- iterative Sethi-Ullman emission; frame = node*4 + state
    int32_t top = 0;
    work[top++] = root * 4;
    while (top > 0) {
      int32_t fr = work[top - 1];
      int32_t n = fr >> 2, st = fr & 3;
      int32_t l = Lc[n], r = Rc[n];
      bool la = is_leaf(fl[l]), lb = is_leaf(fl[r]);
      bool both = !la && !lb;
      bool left_first = both ? ((fl[l] & F_NEED) >= (fl[r] & F_NEED)) : !la;
      int32_t first = left_first ? l : r, second = left_first ? r : l;
      if (st == 0 && !(la && lb)) {
        work[top - 1] = n * 4 + 1;
        work[top++] = first * 4;
        continue;
      }
      if (st == 1 && both) {
        Ins p{};
        p.op = INS_PUSH;
        p.kind = ins_kind(p);
        out[pc++] = p;
        work[top - 1] = n * 4 + 2;
        work[top++] = second * 4;
        continue;
      }
      Ins in{};
      in.op = (uint8_t)C[n];
      if (la && lb) {
        leaf_src(l, in.ls, in.lf, in.c);
        leaf_src(r, in.rs, in.rf, in.c);
      } else if (both) {
        in.ls = left_first ? SRC_POP : SRC_ACC;
        in.rs = left_first ? SRC_ACC : SRC_POP;
      } else if (lb) {                 // right operand is a terminal
        in.ls = SRC_ACC;
        leaf_src(r, in.rs, in.rf, in.c);
      } else {                         // left operand is a terminal
        leaf_src(l, in.ls, in.lf, in.c);
        in.rs = SRC_ACC;
      }
      in.kind = ins_kind(in);
      out[pc++] = in;
      --top;
    }
  }
  P.len[g] = pc;
  P.depth[g] = depth;
  atomicMax(P.maxdepth, depth);
}

// Per-thread evaluation state for CPT cases, with one fully specialised body
// per instruction kind (operator x left source x right source).
template <int NT, int CPT, bool kXSmem>
struct Frame {
  static constexpr int B = NT, TILE = B * CPT;
  double (&acc)[CPT];
  double* stack;               // [depth][TILE] spill stack
  const double* xs;            // [l][TILE] feature tile (kXSmem)
  const double* XT;            // [l][xt_pitch] features in global memory (!kXSmem)
  int64_t xt_pitch, q0;
  const bool (&valid)[CPT];
  int tid;
  double eps;

  // operand base for this instruction: the per-case offsets c*B are then
  // immediates of the shared-memory loads (no per-case address arithmetic)
  template <int S>
  __device__ __forceinline__ const double* base(int sp, int f) const {
    if constexpr (S == SRC_POP) return stack + sp * TILE + tid;
    else if constexpr (S == SRC_FEAT) {
      if constexpr (kXSmem) return xs + f * TILE + tid;
      else return XT + f * xt_pitch + q0 + tid;
    } else return nullptr;
  }
  template <int S>
  __device__ __forceinline__ double get(int c, const double* b, double cst) const {
    if constexpr (S == SRC_ACC) return acc[c];
    else if constexpr (S == SRC_POP) return b[c * B];
    else if constexpr (S == SRC_FEAT) {
      if constexpr (kXSmem) return b[c * B];
      else return valid[c] ? b[c * B] : 0.0;
    } else return cst;
  }
  // the reference's binary op, one IEEE rounding per case (interpreter.py:58-65)
  template <int OP, int LS, int RS>
  __device__ __forceinline__ void op(int& sp, int lf, int rf, double cst) {
    if constexpr (LS == SRC_POP || RS == SRC_POP) --sp;
    const double* lb = base<LS>(sp, lf);
    const double* rb = base<RS>(sp, rf);
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const double l = get<LS>(c, lb, cst), r = get<RS>(c, rb, cst);
      double v;
      if constexpr (OP == OP_ADD) v = __dadd_rn(l, r);
      else if constexpr (OP == OP_SUB) v = __dsub_rn(l, r);
      else if constexpr (OP == OP_MUL) v = __dmul_rn(l, r);
      else v = fabs(r) < eps ? 1.0 : __ddiv_rn(l, r);
      acc[c] = v;
    }
  }
  template <int S>
  __device__ __forceinline__ void load(int& sp, int f, double cst) {
    const double* b = base<S>(sp, f);
#pragma unroll
    for (int c = 0; c < CPT; ++c) acc[c] = get<S>(c, b, cst);
  }
  __device__ __forceinline__ void push(int& sp) {
    double* b = stack + sp * TILE + tid;
#pragma unroll
    for (int c = 0; c < CPT; ++c) b[c * B] = acc[c];
    ++sp;
  }
};

template <int NT, int CPT, int MODE, typename TOut, bool kXSmem>
__global__ void __launch_bounds__(NT) k_interpret(InterpArgs a, int64_t ntiles, int64_t gpb) {
  constexpr int B = NT;
  constexpr int TILE = B * CPT;
  extern __shared__ double smem[];
  const int tid = threadIdx.x;
  const int64_t tile = blockIdx.x;
  const int64_t q0 = tile * TILE;
  const int64_t N = a.ntr + a.nte;
  double* xs = smem;                                  // [l][TILE] when kXSmem
  double* stack = smem + (kXSmem ? (int64_t)a.l * TILE : 0);   // [maxdepth][TILE]
  __shared__ double red[32];

  if (kXSmem) {
    for (int64_t e = tid; e < (int64_t)a.l * TILE; e += B) {
      int64_t f = e / TILE, c = e - f * TILE;
      int64_t q = q0 + c;
      xs[e] = q < N ? a.XT[f * a.xt_pitch + q] : 0.0;
    }
    __syncthreads();
  }
  double ytr[CPT];
  int64_t col[CPT];
  bool valid[CPT], train[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    int64_t q = q0 + c * B + tid;
    valid[c] = q < N;
    train[c] = q < a.ntr;
    col[c] = train[c] ? q : a.test_off + (q - a.ntr);
    ytr[c] = (MODE == INTERP_POP && valid[c]) ? a.y[q] : 0.0;
  }
  unsigned long long nonfinite = 0;

  const int64_t g0 = blockIdx.y * gpb;
  const int64_t g1 = min(a.count, g0 + gpb);
  for (int64_t g = g0; g < g1; ++g) {
    const uint4* code = reinterpret_cast<const uint4*>(a.code + g * a.k1);
    const int len = a.len[g];
    double acc[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) acc[c] = 0.0;
    int sp = 0;
    Frame<NT, CPT, kXSmem> fr{acc, stack, xs, a.XT, a.xt_pitch, q0, valid, tid, a.eps};
    uint4 nxt = len > 0 ? __ldg(code) : make_uint4(0, 0, 0, 0);
    for (int i = 0; i < len; ++i) {
      const uint4 raw = nxt;
      if (i + 1 < len) nxt = __ldg(code + i + 1);   // prefetch the next instruction
      const int kind = raw.x >> 24;
      const int lf = raw.y & 0xffff, rf = raw.y >> 16;
      const double cst = __hiloint2double((int)raw.w, (int)raw.z);
      // one warp-uniform indirect branch per instruction; every case body is
      // straight-line code over the CPT cases of this thread
      switch (kind) {
#define GSGP_K(PAIR, OP, LS, RS) \
  case PAIR * 4 + OP: fr.template op<OP, LS, RS>(sp, lf, rf, cst); break;
#define GSGP_K4(PAIR, LS, RS) \
  GSGP_K(PAIR, 0, LS, RS) GSGP_K(PAIR, 1, LS, RS) GSGP_K(PAIR, 2, LS, RS) GSGP_K(PAIR, 3, LS, RS)
        GSGP_K4(0, SRC_ACC, SRC_POP)
        GSGP_K4(1, SRC_POP, SRC_ACC)
        GSGP_K4(2, SRC_ACC, SRC_FEAT)
        GSGP_K4(3, SRC_ACC, SRC_CONST)
        GSGP_K4(4, SRC_FEAT, SRC_ACC)
        GSGP_K4(5, SRC_CONST, SRC_ACC)
        GSGP_K4(6, SRC_FEAT, SRC_FEAT)
        GSGP_K4(7, SRC_FEAT, SRC_CONST)
        GSGP_K4(8, SRC_CONST, SRC_FEAT)
#undef GSGP_K4
#undef GSGP_K
        case kKindLoadFeat: fr.template load<SRC_FEAT>(sp, lf, cst); break;
        case kKindLoadConst: fr.template load<SRC_CONST>(sp, lf, cst); break;
        case kKindPush: fr.push(sp); break;
        default: __trap();   // the compiler never emits any other kind
      }
    }
    // ---- epilogue: non-finite -> 0.0 counted (core.py:348-356), then store
    double sse_tr = 0.0, sse_te = 0.0;
    int wide = 0;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      if (!valid[c]) continue;
      double v = acc[c];
      if (!isfinite(v) && !(MODE == INTERP_F64 && a.raw)) { v = 0.0; ++nonfinite; }
      const int64_t q = q0 + c * B + tid;
      if (MODE == INTERP_F64) {
        a.out64[g * N + q] = v;
      } else if (MODE == INTERP_POP) {
        TOut o = (TOut)v;
        reinterpret_cast<TOut*>(a.out)[g * a.pitch + col[c]] = o;
        if (isinf((double)o)) wide |= train[c] ? 1 : 2;
        double d = __dsub_rn(v, ytr[c]);
        if (train[c]) sse_tr = __dadd_rn(sse_tr, __dmul_rn(d, d));
        else sse_te = __dadd_rn(sse_te, __dmul_rn(d, d));
      } else {
        // sigmoid of the pool, once per run (mutation.py:32-34, evolution.py:135-136)
        double sg = __ddiv_rn(1.0, __dadd_rn(1.0, exp(-v)));
        reinterpret_cast<TOut*>(a.out)[g * a.pitch + col[c]] = (TOut)sg;
      }
    }
    if (MODE == INTERP_POP) {
      // fixed-order block reduction of the tile's SSE (train, test)
      sse_tr = warp_sum(sse_tr);
      sse_te = warp_sum(sse_te);
      int wb = __reduce_or_sync(0xffffffffu, wide);
      if ((tid & 31) == 0) {
        red[(tid >> 5) * 2] = sse_tr;
        red[(tid >> 5) * 2 + 1] = sse_te;
        if (wb) atomicOr(a.wide + g, wb);
      }
      __syncthreads();
      if (tid < 2) {
        double t = 0.0;
        for (int w = 0; w < B / 32; ++w) t = __dadd_rn(t, red[w * 2 + tid]);
        a.part[(g * ntiles + tile) * 2 + tid] = t;
      }
      __syncthreads();
    }
  }
  // block total of replaced elements (integer: order-independent)
  for (int o = 16; o > 0; o >>= 1) nonfinite += __shfl_xor_sync(0xffffffffu, nonfinite, o);
  if ((tid & 31) == 0 && nonfinite) atomicAdd(a.nonfinite, nonfinite);
}

// (threads per block, cases per thread): more cases per thread amortise the
// per-instruction dispatch; the case tile (features + spill stacks) lives in
// shared memory, so wide feature sets use smaller tiles.
struct InterpCfg {
  int nt, cpt;
};
constexpr InterpCfg kInterpCfgs[] = {{128, 4}, {128, 2}, {128, 1}, {64, 8}};
int choose_cfg(int l) {
  static const int forced = getenv("GSGP_INTERP_CFG") ? atoi(getenv("GSGP_INTERP_CFG")) : -1;
  if (forced >= 0 && forced < 4) return forced;
  return l <= 16 ? 0 : (l <= 48 ? 1 : 2);
}

template <int NT, int CPT, int MODE, typename TOut>
void launch_cpt(const InterpArgs& a, cudaStream_t s) {
  constexpr int TILE = NT * CPT;
  const int64_t N = a.ntr + a.nte;
  const int64_t ntiles = (N + TILE - 1) / TILE;
  const size_t stack_bytes = (size_t)(a.maxdepth > 0 ? a.maxdepth : 1) * TILE * sizeof(double);
  const size_t x_bytes = (size_t)a.l * TILE * sizeof(double);
  const bool xsmem = x_bytes + stack_bytes <= 160 * 1024;
  const size_t smem = (xsmem ? x_bytes : 0) + stack_bytes;
  GSGP_REQUIRE(smem <= 200 * 1024, "interpreter spill stack too deep for shared memory");
  // genomes per block: enough blocks to fill 148 SMs several times over
  int64_t want = 148 * 8;
  int64_t gpb = (a.count * ntiles + want - 1) / want;
  if (gpb < 1) gpb = 1;
  if (gpb > 64) gpb = 64;
  int64_t gy = (a.count + gpb - 1) / gpb;
  GSGP_REQUIRE(gy <= 65535, "too many genome groups");
  dim3 grid((unsigned)ntiles, (unsigned)gy);
  if (xsmem) {
    auto k = k_interpret<NT, CPT, MODE, TOut, true>;
    GSGP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, NT, smem, s>>>(a, ntiles, gpb);
  } else {
    auto k = k_interpret<NT, CPT, MODE, TOut, false>;
    GSGP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, NT, smem, s>>>(a, ntiles, gpb);
  }
  GSGP_CUDA(cudaGetLastError());
}

template <int MODE, typename TOut>
void launch_mode(const InterpArgs& a, cudaStream_t s) {
  switch (choose_cfg(a.l)) {
    case 0: launch_cpt<128, 4, MODE, TOut>(a, s); break;
    case 1: launch_cpt<128, 2, MODE, TOut>(a, s); break;
    case 2: launch_cpt<128, 1, MODE, TOut>(a, s); break;
    default: launch_cpt<64, 8, MODE, TOut>(a, s); break;
  }
}

}  // namespace

void launch_compile(const uint8_t* tags, const int32_t* codes, const double* consts, int64_t count,
                    int32_t k, double eps, Program prog, cudaStream_t s) {
  if (count <= 0) return;
  GSGP_CUDA(cudaMemsetAsync(prog.maxdepth, 0, sizeof(int32_t), s));
  k_compile<<<(unsigned)((count + 63) / 64), 64, 0, s>>>(tags, codes, consts, count, k, eps, prog);
  GSGP_CUDA(cudaGetLastError());
}

int64_t interp_tiles(const InterpArgs& a, int* cpt_out) {
  const InterpCfg c = kInterpCfgs[choose_cfg(a.l)];
  if (cpt_out) *cpt_out = c.cpt;
  const int64_t tile = (int64_t)c.nt * c.cpt;
  return (a.ntr + a.nte + tile - 1) / tile;
}

void launch_interpret(const InterpArgs& a, int mode, cudaStream_t s) {
  if (a.count <= 0 || a.ntr + a.nte <= 0) return;
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
