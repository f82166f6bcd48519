// extern "C" boundary (include/gsgp_b200.h).  Each entry point replaces one
// function of the reference package and runs its sm_100a kernel; errors are
// returned as status codes with a thread-local message.
#include <algorithm>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "gsgp_b200.h"
#include <memory>

#include "kernels.cuh"

namespace gsgp {

thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

void run_engine(const gsgp_config*, const double*, const double*, int64_t, const double*, const double*,
                int64_t, int32_t, gsgp_outputs*);
void comm_unique_id(unsigned char*);
void comm_init(int, int, const unsigned char*);
void comm_destroy();
void comm_init_host(int world, int rank, void (*fn)(void*, int64_t, int32_t));
void trim_device_memory();
void* cache_alloc(size_t bytes, size_t* got);
void cache_park(void* p, size_t bytes);
void devices_init(int, const int*);
void devices_finalize();
int devices_count();
void run_job(const gsgp_config*, const double*, const double*, int64_t, const double*, const double*, int64_t,
             int32_t, gsgp_outputs*);
void shard_range(int64_t, int64_t, int64_t, int64_t*, int64_t*);

namespace {

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return GSGP_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    set_error("host allocation failed");
    return GSGP_ERR_OOM;
  } catch (const std::exception& e) {
    set_error(e.what());
    return GSGP_ERR_CUDA;
  }
}

void require_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw Error{ERR_CUDA, std::string("no CUDA device available: ") + cudaGetErrorString(e)};
  }
}

// RAII device buffer for the operator entry points, taken from the engine's
// device block cache (engine.cu) so repeated operator calls of similar sizes
// neither cudaMalloc nor cudaFree; the operators run on the legacy default
// stream, which is drained before a block is parked again
struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
  explicit Buf(size_t n) { p = cache_alloc(n ? n : 16, &bytes); }
  ~Buf() {
    if (!p) return;
    if (cudaStreamSynchronize(0) == cudaSuccess) {
      cache_park(p, bytes);
    } else {
      cudaGetLastError();
      cudaFree(p);
    }
  }
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
  template <typename T> T* as() const { return reinterpret_cast<T*>(p); }
};

void h2d(void* d, const void* h, size_t n) { if (n) GSGP_CUDA(cudaMemcpy(d, h, n, cudaMemcpyHostToDevice)); }
void d2h(void* h, const void* d, size_t n) { if (n) GSGP_CUDA(cudaMemcpy(h, d, n, cudaMemcpyDeviceToHost)); }

__global__ void k_sigmoid(double* x, int64_t rows, int64_t n, int64_t pitch) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= rows * n) return;
  int64_t i = e / n, j = e - i * n;
  double v = x[i * pitch + j];
  x[i * pitch + j] = __ddiv_rn(1.0, __dadd_rn(1.0, exp(-v)));   // mutation.py:32-34
}

__global__ void k_transpose_op(const double* __restrict__ Xr, int64_t N, int l, double* __restrict__ XT) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= N * l) return;
  int64_t q = e / l, f = e - q * l;
  XT[f * N + q] = Xr[e];
}

inline unsigned nb(int64_t n) { return (unsigned)((n + 255) / 256 > 0 ? (n + 255) / 256 : 1); }

}  // namespace
}  // namespace gsgp

using namespace gsgp;

extern "C" {

const char* gsgp_version(void) { return "gsgp_b200 0.1.0 (sm_100a)"; }

const char* gsgp_last_error(void) { return g_last_error.c_str(); }

int gsgp_device_info(int* device_count, int* sm_count, char* name, int name_len) {
  return guarded([&] {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) { cudaGetLastError(); n = 0; }
    if (device_count) *device_count = n;
    if (n == 0) throw Error{ERR_CUDA, "no CUDA device available"};
    int dev = 0;
    GSGP_CUDA(cudaGetDevice(&dev));
    cudaDeviceProp prop;
    GSGP_CUDA(cudaGetDeviceProperties(&prop, dev));
    if (sm_count) *sm_count = prop.multiProcessorCount;
    if (name && name_len > 0) {
      std::strncpy(name, prop.name, name_len - 1);
      name[name_len - 1] = 0;
    }
  });
}

int gsgp_set_device(int device) {
  return guarded([&] {
    require_device();
    devices_finalize();            // back to one device per process
    GSGP_CUDA(cudaSetDevice(device));
  });
}

int gsgp_trim_device_memory(void) {
  return guarded([&] {
    require_device();
    GSGP_CUDA(cudaDeviceSynchronize());
    trim_device_memory();
  });
}

int gsgp_rng_draw(uint64_t seed, uint64_t stream, const uint64_t* counters, int64_t n, uint64_t* bits,
                  double* units) {
  return guarded([&] {
    require_device();
    GSGP_REQUIRE(n >= 0, "n must be >= 0");
    if (n == 0) return;
    Buf c(n * 8), b(n * 8), u(n * 8);
    h2d(c.p, counters, n * 8);
    launch_rng_draw(seed, stream, c.as<uint64_t>(), n, b.as<uint64_t>(), u.as<double>(), 0);
    if (bits) d2h(bits, b.p, n * 8);
    if (units) d2h(units, u.p, n * 8);
  });
}

uint64_t gsgp_derive_seed(uint64_t seed, uint64_t index) {
  // rng.py:67-69
  return sm64_finalize(sm64_finalize(seed ^ kStreamMult) + index * kGolden);
}

int gsgp_create_population(const gsgp_config* cfg, int64_t count, uint64_t stream_base, int32_t n_features,
                           uint8_t* tags, int32_t* codes, double* consts) {
  return guarded([&] {
    require_device();
    GSGP_REQUIRE(count >= 1, "population count must be >= 1");
    GSGP_REQUIRE(n_features >= 1, "n_features must be >= 1");
    const int64_t k = cfg->program_size;
    GSGP_REQUIRE(k >= 1, "program_size must be >= 1");
    const double total = cfg->p_function + cfg->p_feature + cfg->p_constant;
    GSGP_REQUIRE(total > 0, "gene probabilities must have positive sum");
    GeneParams gp;
    gp.seed = cfg->seed;
    gp.thr_fun = cfg->p_function / total;                       // core.py:338-342
    gp.thr_feat = gp.thr_fun + cfg->p_feature / total;          // population.py:56
    gp.erc_low = cfg->erc_low;
    gp.erc_high = cfg->erc_high;
    gp.n_features = n_features;
    gp.k = (int32_t)k;
    Buf t(count * k), c(count * k * 4), v(count * k * 8);
    launch_create_population(gp, count, stream_base, t.as<uint8_t>(), c.as<int32_t>(), v.as<double>(), 0);
    d2h(tags, t.p, count * k);
    d2h(codes, c.p, count * k * 4);
    d2h(consts, v.p, count * k * 8);
  });
}

int gsgp_compute_semantics(const uint8_t* tags, const int32_t* codes, const double* consts, int64_t count,
                           int64_t k, const double* X, int64_t n, int32_t l, double eps,
                           int32_t replace_nonfinite, double* out, int64_t* overflow) {
  return guarded([&] {
    require_device();
    GSGP_REQUIRE(count >= 1 && n >= 1, "compute_semantics needs a nonempty population and dataset");
    GSGP_REQUIRE(k >= 1 && l >= 1 && l <= 65535, "bad genome length / feature count");
    for (int64_t e = 0; e < count * k; ++e)   // interpreter.py:134-135
      if (tags[e] == TAG_FEATURE && (codes[e] < 0 || codes[e] >= l))
        throw Error{ERR_CONFIG, "genome references a feature beyond the dataset width"};
    Buf dt(count * k), dc(count * k * 4), dv(count * k * 8);
    h2d(dt.p, tags, count * k);
    h2d(dc.p, codes, count * k * 4);
    h2d(dv.p, consts, count * k * 8);
    Buf ins(count * (k + 1) * sizeof(Ins)), len(count * 4),
        nconst(count * 4), ctab(count * k * 8), mx(4 * 4), scr(count * 4 * k * 4), fl(count * k),
        cv(count * k * 8);
    Program prog{ins.as<Ins>(), nullptr, len.as<int32_t>(), nconst.as<int32_t>(),
                 ctab.as<double>(), mx.as<int32_t>(), scr.as<int32_t>(), fl.as<uint8_t>(),
                 cv.as<double>(), nullptr};
    launch_compile(dt.as<uint8_t>(), dc.as<int32_t>(), dv.as<double>(), count, (int32_t)k, eps, prog, 0);
    int32_t maxima[4] = {0, 0, 0, 0};
    d2h(maxima, mx.p, 16);
    const LinkedLayout ll = linked_layout(count, maxima[2]);
    Buf exe(ll.ins * sizeof(Ins));
    Buf xr(n * l * 8), xt(n * l * 8), o(count * n * 8), nf(8);
    h2d(xr.p, X, n * l * 8);
    k_transpose_op<<<nb(n * l), 256>>>(xr.as<double>(), n, l, xt.as<double>());
    GSGP_CUDA(cudaGetLastError());
    GSGP_CUDA(cudaMemset(nf.p, 0, 8));
    InterpArgs a{};
    a.code = ins.as<Ins>();
    a.exe = exe.as<Ins>();
    a.exe_k1 = ll.k1;
    a.max_groups = ll.copies;
    a.len = len.as<int32_t>();
    a.nconst = nconst.as<int32_t>();
    a.ctab = ctab.as<double>();
    a.k1 = k + 1;
    a.count = count;
    a.XT = xt.as<double>();
    a.xt_pitch = n;
    a.l = l;
    a.ntr = n;
    a.nte = 0;
    a.te_q = n;
    a.q_base = 0;
    a.nq = n;
    a.eps = eps;
    a.maxdepth = maxima[0];
    a.maxconst = maxima[1];
    a.maxlen = maxima[2];
    a.out64 = o.as<double>();
    a.nonfinite = nf.as<unsigned long long>();
    a.raw = replace_nonfinite ? 0 : 1;
    launch_interpret(a, INTERP_F64, 0);
    d2h(out, o.p, count * n * 8);
    unsigned long long c = 0;
    d2h(&c, nf.p, 8);
    if (overflow) *overflow += (int64_t)c;
  });
}

int gsgp_compute_fitness(const double* S, const double* target, int64_t m, int64_t n, double* out) {
  return guarded([&] {
    require_device();
    GSGP_REQUIRE(m >= 0 && n >= 1, "fitness needs at least one case");
    if (m == 0) return;
    Buf s(m * n * 8), y(n * 8), o(m * 8);
    h2d(s.p, S, m * n * 8);
    h2d(y.p, target, n * 8);
    launch_row_rmse(s.as<double>(), y.as<double>(), m, n, o.as<double>(), 0);
    d2h(out, o.p, m * 8);
  });
}

int gsgp_build_mutation_plan(int64_t m, int64_t r, uint64_t seed, int64_t generation, int32_t ms_uniform,
                             double ms_const, int64_t* u, int64_t* v, double* ms) {
  return guarded([&] {
    require_device();
    GSGP_REQUIRE(r >= 2, "geometric semantic mutation needs at least 2 random trees");
    GSGP_REQUIRE(m >= 1, "plan length must be >= 1");
    Buf du(m * 8), dv(m * 8), dm(m * 8);
    PlanParams p{seed, m, r, ms_uniform, ms_const};
    launch_plan(p, generation, nullptr, du.as<int64_t>(), dv.as<int64_t>(), dm.as<double>(), m, 0);
    d2h(u, du.p, m * 8);
    d2h(v, dv.p, m * 8);
    d2h(ms, dm.p, m * 8);
  });
}

int gsgp_gsm(const double* parent, int64_t m, int64_t n, const double* trees, int64_t r, const int64_t* u,
             const int64_t* v, const double* ms, int32_t sign, int32_t squashed, double* out,
             int64_t* overflow) {
  return guarded([&] {
    require_device();
    GSGP_REQUIRE(m >= 1 && n >= 1 && r >= 1, "empty GSM operands");
    for (int64_t i = 0; i < m; ++i) {   // MutationPlan.validate, core.py:213-223
      GSGP_REQUIRE(u[i] >= 0 && u[i] < r, "plan index u out of range");
      GSGP_REQUIRE(v[i] >= 0 && v[i] < r, "plan index v out of range");
      GSGP_REQUIRE(u[i] != v[i], "plan requires distinct tree indices per slot");
    }
    const int64_t pitch = pad32(n);
    Buf P(m * pitch * 8), T(r * pitch * 8), y(pitch * 8), du(m * 8), dv(m * 8), dm(m * 8), nf(8),
        e0(pitch * 8), e1(pitch * 8);
    GSGP_CUDA(cudaMemset(P.p, 0, m * pitch * 8));
    GSGP_CUDA(cudaMemset(T.p, 0, r * pitch * 8));
    GSGP_CUDA(cudaMemset(y.p, 0, pitch * 8));
    GSGP_CUDA(cudaMemset(nf.p, 0, 8));
    GSGP_CUDA(cudaMemcpy2D(P.p, pitch * 8, parent, n * 8, n * 8, m, cudaMemcpyHostToDevice));
    GSGP_CUDA(cudaMemcpy2D(T.p, pitch * 8, trees, n * 8, n * 8, r, cudaMemcpyHostToDevice));
    if (!squashed) {
      k_sigmoid<<<nb(r * n), 256>>>(T.as<double>(), r, n, pitch);
      GSGP_CUDA(cudaGetLastError());
    }
    h2d(du.p, u, m * 8);
    h2d(dv.p, v, m * 8);
    h2d(dm.p, ms, m * 8);
    const RowLayout lay = make_layout(n, 0, true);   // [train] = pad32(n) == pitch
    const int64_t ntiles = lay.ntiles;
    Buf part(m * ntiles * 2 * 8);
    GsmArgs a{};
    a.pool = T.p;
    a.S = P.p;
    a.elite_prev = e0.p;
    a.elite_cur = e1.p;
    a.y = y.as<double>();
    a.lay = lay;
    a.m = m;
    a.u = du.as<int64_t>();
    a.v = dv.as<int64_t>();
    a.ms = dm.as<double>();
    a.ctl = nullptr;
    a.sign = sign;
    a.part = part.as<double>();
    a.nonfinite = nf.as<unsigned long long>();
    Buf ticket(16);
    GSGP_CUDA(cudaMemset(ticket.p, 0, 16));
    a.ticket = ticket.as<unsigned long long>();
    launch_gsm(a, true, true, 0);
    GSGP_CUDA(cudaMemcpy2D(out, n * 8, P.p, pitch * 8, n * 8, m, cudaMemcpyDeviceToHost));
    unsigned long long c = 0;
    d2h(&c, nf.p, 8);
    if (overflow) *overflow += (int64_t)c;
  });
}

int gsgp_replay(const double* initial, int64_t m, int64_t n, const double* trees, int64_t r, int64_t g,
                const int64_t* u, const int64_t* v, const double* ms, const int8_t* elite_src,
                const int64_t* elite_idx, const int64_t* elite_slot, int64_t final_slot, int32_t sign,
                double* out) {
  return guarded([&] {
    require_device();
    GSGP_REQUIRE(m >= 1 && n >= 1 && r >= 1 && g >= 0, "empty replay operands");
    GSGP_REQUIRE(final_slot >= 0 && final_slot < m, "final elite slot out of range");
    for (int64_t e = 0; e < g * m; ++e) {   // MutationPlan.validate per generation (core.py:213-223)
      GSGP_REQUIRE(u[e] >= 0 && u[e] < r, "plan index u out of range");
      GSGP_REQUIRE(v[e] >= 0 && v[e] < r, "plan index v out of range");
      GSGP_REQUIRE(u[e] != v[e], "plan requires distinct tree indices per slot");
    }
    for (int64_t t = 0; t < g; ++t)
      if (elite_src[t] == 0)
        GSGP_REQUIRE(elite_idx[t] >= 0 && elite_idx[t] < m && elite_slot[t] >= 0 && elite_slot[t] < m,
                     "elite record index/slot out of range");
    const int64_t pitch = pad32(n);
    Buf P(m * pitch * 8), T(r * pitch * 8), y(pitch * 8), nf(8), e0(pitch * 8), e1(pitch * 8), keep(pitch * 8);
    Buf du(std::max<int64_t>(g, 1) * m * 8), dv(std::max<int64_t>(g, 1) * m * 8), dm(std::max<int64_t>(g, 1) * m * 8);
    GSGP_CUDA(cudaMemset(P.p, 0, m * pitch * 8));
    GSGP_CUDA(cudaMemset(T.p, 0, r * pitch * 8));
    GSGP_CUDA(cudaMemset(y.p, 0, pitch * 8));
    GSGP_CUDA(cudaMemset(nf.p, 0, 8));
    GSGP_CUDA(cudaMemcpy2D(P.p, pitch * 8, initial, n * 8, n * 8, m, cudaMemcpyHostToDevice));
    GSGP_CUDA(cudaMemcpy2D(T.p, pitch * 8, trees, n * 8, n * 8, r, cudaMemcpyHostToDevice));
    // gsm() squashes the raw trees every generation (mutation.py:89-94); the
    // sigmoid is a pure function of the same values, so once is the same bits
    k_sigmoid<<<nb(r * n), 256>>>(T.as<double>(), r, n, pitch);
    GSGP_CUDA(cudaGetLastError());
    if (g > 0) {
      h2d(du.p, u, g * m * 8);
      h2d(dv.p, v, g * m * 8);
      h2d(dm.p, ms, g * m * 8);
    }
    const RowLayout lay = make_layout(n, 0, true);
    Buf part(m * lay.ntiles * 2 * 8), ticket(16);
    GSGP_CUDA(cudaMemset(ticket.p, 0, 16));
    GsmArgs a{};
    a.pool = T.p;
    a.S = P.p;
    a.elite_prev = e0.p;
    a.elite_cur = e1.p;
    a.y = y.as<double>();
    a.lay = lay;
    a.m = m;
    a.ctl = nullptr;
    a.sign = sign;
    a.part = part.as<double>();
    a.nonfinite = nf.as<unsigned long long>();
    a.ticket = ticket.as<unsigned long long>();
    double* S = P.as<double>();
    // evolution.py:195-201 on the device, in place: offspring = gsm(current);
    // a parent-sourced elite puts current[index] into offspring[slot], so
    // that row is saved before the update overwrites it
    for (int64_t t = 0; t < g; ++t) {
      const bool parent = elite_src[t] == 0;
      if (parent)
        GSGP_CUDA(cudaMemcpyAsync(keep.p, S + elite_idx[t] * pitch, n * 8, cudaMemcpyDeviceToDevice, 0));
      a.u = du.as<int64_t>() + t * m;
      a.v = dv.as<int64_t>() + t * m;
      a.ms = dm.as<double>() + t * m;
      launch_gsm(a, true, true, 0);
      if (parent)
        GSGP_CUDA(cudaMemcpyAsync(S + elite_slot[t] * pitch, keep.p, n * 8, cudaMemcpyDeviceToDevice, 0));
    }
    d2h(out, S + final_slot * pitch, n * 8);
  });
}

int gsgp_gsm_step_f32(const float* parent_tr, const float* parent_te, const float* sq_tr, const float* sq_te,
                      int64_t m, int64_t r, int64_t ntr, int64_t nte, const double* ytr, const double* yte,
                      const int64_t* u, const int64_t* v, const double* ms, int32_t sign, float* out_tr,
                      float* out_te, double* sse_tr, double* sse_te) {
  return guarded([&] {
    require_device();
    GSGP_REQUIRE(m >= 1 && r >= 2 && ntr >= 1 && nte >= 0, "bad GSM step shape");
    for (int64_t i = 0; i < m; ++i) {
      GSGP_REQUIRE(u[i] >= 0 && u[i] < r && v[i] >= 0 && v[i] < r && u[i] != v[i], "bad plan");
    }
    const int64_t toff = pad32(ntr), pitch = toff + pad32(nte);
    Buf P(m * pitch * 4), T(r * pitch * 4), y(pitch * 8), du(m * 8), dv(m * 8), dm(m * 8), e0(pitch * 4),
        e1(pitch * 4), sse(m * 2 * 8);
    GSGP_CUDA(cudaMemset(P.p, 0, m * pitch * 4));
    GSGP_CUDA(cudaMemset(T.p, 0, r * pitch * 4));
    GSGP_CUDA(cudaMemset(y.p, 0, pitch * 8));
    GSGP_CUDA(cudaMemcpy2D(P.p, pitch * 4, parent_tr, ntr * 4, ntr * 4, m, cudaMemcpyHostToDevice));
    GSGP_CUDA(cudaMemcpy2D(T.p, pitch * 4, sq_tr, ntr * 4, ntr * 4, r, cudaMemcpyHostToDevice));
    if (nte > 0) {
      GSGP_CUDA(cudaMemcpy2D(P.as<float>() + toff, pitch * 4, parent_te, nte * 4, nte * 4, m,
                             cudaMemcpyHostToDevice));
      GSGP_CUDA(cudaMemcpy2D(T.as<float>() + toff, pitch * 4, sq_te, nte * 4, nte * 4, r,
                             cudaMemcpyHostToDevice));
      h2d(y.as<double>() + toff, yte, nte * 8);
    }
    h2d(y.p, ytr, ntr * 8);
    h2d(du.p, u, m * 8);
    h2d(dv.p, v, m * 8);
    h2d(dm.p, ms, m * 8);
    const RowLayout lay = make_layout(ntr, nte, false, false);   // [train | test], as staged above
    const int64_t ntiles = lay.ntiles;
    Buf part(m * ntiles * 2 * 8);
    GsmArgs a{};
    a.pool = T.p;
    a.S = P.p;
    a.elite_prev = e0.p;
    a.elite_cur = e1.p;
    a.y = y.as<double>();
    a.lay = lay;
    a.m = m;
    a.u = du.as<int64_t>();
    a.v = dv.as<int64_t>();
    a.ms = dm.as<double>();
    a.sign = sign;
    a.part = part.as<double>();
    Buf ticket(16);
    GSGP_CUDA(cudaMemset(ticket.p, 0, 16));
    a.ticket = ticket.as<unsigned long long>();
    launch_gsm(a, false, false, 0);
    launch_reduce_partials(part.as<double>(), m, ntiles, sse.as<double>(), 0);
    GSGP_CUDA(cudaMemcpy2D(out_tr, ntr * 4, P.p, pitch * 4, ntr * 4, m, cudaMemcpyDeviceToHost));
    if (nte > 0)
      GSGP_CUDA(cudaMemcpy2D(out_te, nte * 4, P.as<float>() + toff, pitch * 4, nte * 4, m,
                             cudaMemcpyDeviceToHost));
    std::vector<double> h(m * 2);
    d2h(h.data(), sse.p, m * 16);
    for (int64_t i = 0; i < m; ++i) {
      sse_tr[i] = h[2 * i];
      sse_te[i] = h[2 * i + 1];
    }
  });
}

int gsgp_survive(const double* fit_parent, const double* fit_offspring, int64_t m, int64_t* dec) {
  return guarded([&] {
    require_device();
    GSGP_REQUIRE(m >= 1, "empty fitness vector");
    Buf a(m * 8), b(m * 8), o(3 * 8);
    h2d(a.p, fit_parent, m * 8);
    h2d(b.p, fit_offspring, m * 8);
    launch_survive_decision(a.as<double>(), b.as<double>(), m, o.as<int64_t>(), 0);
    d2h(dec, o.p, 3 * 8);
  });
}

int gsgp_sigmoid(const double* x, int64_t n, double* out) {
  return guarded([&] {
    require_device();
    GSGP_REQUIRE(n >= 0, "n must be >= 0");
    if (n == 0) return;
    Buf a(n * 8), b(n * 8);
    h2d(a.p, x, n * 8);
    launch_sigmoid(a.as<double>(), n, b.as<double>(), 0);
    d2h(out, b.p, n * 8);
  });
}

int gsgp_argminmax(const double* f, int64_t m, int64_t* out) {
  return guarded([&] {
    require_device();
    GSGP_REQUIRE(m >= 1, "empty fitness vector");
    Buf a(m * 8), o(2 * 8);
    h2d(a.p, f, m * 8);
    launch_argminmax(a.as<double>(), m, o.as<int64_t>(), 0);
    d2h(out, o.p, 2 * 8);
  });
}

int gsgp_canonical_sum(const double* x, int64_t rows, int64_t n, int32_t parts, double* out) {
  return guarded([&] {
    require_device();
    GSGP_REQUIRE(rows >= 1 && n >= 1 && parts >= 0, "bad canonical sum shape");
    // x[row][j] -> the engine's partial layout part[row][j][2] (train slot)
    std::vector<double> h(rows * n * 2, 0.0);
    for (int64_t i = 0; i < rows * n; ++i) h[2 * i] = x[i];
    Buf part(rows * n * 16), sse(rows * 16);
    h2d(part.p, h.data(), rows * n * 16);
    if (parts == 0) {   // single part: the fused one-warp-per-row path
      launch_reduce_partials(part.as<double>(), rows, n, sse.as<double>(), 0);
    } else {            // columns split into `parts` pieces: the multi-shard path
      const int64_t w = (n + parts - 1) / parts;
      std::vector<std::unique_ptr<Buf>> pieces;
      Buf cexp(rows * 2 * 4), cdig(rows * 2 * kLimbs * 8);
      launch_canon_clear(rows, cexp.as<int32_t>(), cdig.as<unsigned long long>(), 0);
      for (int64_t c0 = 0; c0 < n; c0 += w) {
        const int64_t nc = std::min(w, n - c0);
        pieces.push_back(std::make_unique<Buf>(rows * nc * 16));
        GSGP_CUDA(cudaMemcpy2D(pieces.back()->p, nc * 16, h.data() + 2 * c0, n * 16, nc * 16, rows,
                               cudaMemcpyHostToDevice));
        launch_canon_exp(pieces.back()->as<double>(), rows, nc, cexp.as<int32_t>(), 0);
      }
      int64_t c0 = 0;
      for (auto& b : pieces) {
        const int64_t nc = std::min(w, n - c0);
        launch_canon_digits(b->as<double>(), rows, nc, cexp.as<int32_t>(), cdig.as<unsigned long long>(), 0);
        c0 += w;
      }
      launch_canon_finish(cexp.as<int32_t>(), cdig.as<unsigned long long>(), rows, sse.as<double>(), 0);
    }
    std::vector<double> r(rows * 2);
    d2h(r.data(), sse.p, rows * 16);
    for (int64_t i = 0; i < rows; ++i) out[i] = r[2 * i];
  });
}

int gsgp_run(const gsgp_config* cfg, const double* Xtr, const double* ytr, int64_t ntr, const double* Xte,
             const double* yte, int64_t nte, int32_t n_features, gsgp_outputs* out) {
  return guarded([&] {
    require_device();
    run_job(cfg, Xtr, ytr, ntr, Xte, yte, nte, n_features, out);
  });
}

int gsgp_init(int n_dev, const int* dev_ids) {
  return guarded([&] {
    require_device();
    devices_init(n_dev, dev_ids);
  });
}

int gsgp_finalize(void) {
  return guarded([&] { devices_finalize(); });
}

int gsgp_device_count_in_use(void) { return devices_count(); }

int gsgp_comm_unique_id(unsigned char id[128]) {
  return guarded([&] { comm_unique_id(id); });
}

int gsgp_comm_init(int world, int rank, const unsigned char id[128]) {
  return guarded([&] {
    require_device();
    comm_init(world, rank, id);
  });
}

int gsgp_comm_init_host(int world, int rank, void (*allreduce)(void* buf, int64_t count, int32_t dtype)) {
  return guarded([&] { comm_init_host(world, rank, allreduce); });
}

int gsgp_comm_destroy(void) {
  return guarded([&] { comm_destroy(); });
}

void gsgp_shard_range(int64_t n, int64_t count, int64_t index, int64_t* lo, int64_t* hi) {
  shard_range(n, count, index, lo, hi);
}

}  // extern "C"
