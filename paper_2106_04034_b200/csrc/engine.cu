// run_evolution on the device (gsgp/evolution.py:100-179).
//
// Host side of the engine: allocation, case sharding, the one-time init
// (CreatePopulation -> compile -> interpret population + pool -> initial
// fitness) and the generation loop, which is a fixed sequence of kernels
//   plan -> GSM+SSE (per shard) -> SSE tile reduction -> [shard sum] ->
//   [NCCL allreduce over ranks] -> survival
// whose every decision lives on the device (control block), so one captured
// generation is replayed g times as a CUDA graph.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <set>
#include <thread>
#include <vector>

#include "gsgp_b200.h"
#include "kernels.cuh"

namespace gsgp {

// ------------------------------------------------------------- device memory
// Engine buffers come from a small process-level cache of device blocks:
// a run's release parks its blocks (after its stream has drained) and the
// next run reuses them, so a job's second run neither allocates nor frees
// its ~100 GB working set (a plain cudaFree of a 51 GB buffer was measured
// at up to 1.6 s; growing the stream-ordered pool at up to 4.8 s).  First
// allocations are plain cudaMalloc; an allocation failure empties the cache
// and retries.  gsgp_trim_device_memory() frees the cache.
struct CachedBlock {
  void* p;
  size_t bytes;
  int dev;          // blocks are only reused on the device that owns them
};
std::mutex g_cache_mu;
std::vector<CachedBlock> g_cache;

int current_device() {
  int d = 0;
  GSGP_CUDA(cudaGetDevice(&d));
  return d;
}

// free the cached blocks of `dev` (-1: of every device)
void cache_trim(int dev = -1) {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  int cur = 0;
  cudaGetDevice(&cur);
  std::vector<CachedBlock> keep;
  for (auto& b : g_cache) {
    if (dev >= 0 && b.dev != dev) {
      keep.push_back(b);
      continue;
    }
    cudaSetDevice(b.dev);
    cudaFree(b.p);
  }
  cudaSetDevice(cur);
  g_cache.swap(keep);
}

void* cache_alloc(size_t bytes, size_t* got) {
  const int dev = current_device();
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    int best = -1;
    for (int i = 0; i < (int)g_cache.size(); ++i)     // smallest block within 1.25x
      if (g_cache[i].dev == dev && g_cache[i].bytes >= bytes && g_cache[i].bytes <= bytes + bytes / 4 &&
          (best < 0 || g_cache[i].bytes < g_cache[best].bytes))
        best = i;
    if (best >= 0) {
      CachedBlock b = g_cache[best];
      g_cache.erase(g_cache.begin() + best);
      *got = b.bytes;
      return b.p;
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    cache_trim(dev);
    e = cudaMalloc(&p, bytes);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error{e == cudaErrorMemoryAllocation ? ERR_OOM : ERR_CUDA,
                "cudaMalloc(" + std::to_string(bytes) + " bytes) on device " + std::to_string(dev) + ": " +
                    cudaGetErrorString(e)};
  }
  *got = bytes;
  return p;
}

// return a block to the cache (its last use must be complete)
void cache_park(void* p, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_cache.push_back({p, bytes, dev});
}

thread_local cudaStream_t g_alloc_stream = nullptr;   // stream a released block may still be used on

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (!p) return;
    // the block is parked for reuse by any stream: drain its stream first
    if (cudaStreamSynchronize(s) == cudaSuccess) {
      int dev = 0;
      cudaGetDevice(&dev);
      std::lock_guard<std::mutex> lk(g_cache_mu);
      g_cache.push_back({p, bytes, dev});
    } else {
      cudaGetLastError();
      cudaFree(p);
    }
    p = nullptr;
  }
  void alloc(size_t n) {
    release();
    s = g_alloc_stream;
    p = cache_alloc(n == 0 ? 16 : n, &bytes);
  }
  template <typename T> T* as() const { return reinterpret_cast<T*>(p); }
};

struct Event {
  cudaEvent_t e = nullptr;
  Event() { GSGP_CUDA(cudaEventCreate(&e)); }
  ~Event() { if (e) cudaEventDestroy(e); }
  Event(const Event&) = delete;
  Event& operator=(const Event&) = delete;
};

float elapsed_ms(const Event& a, const Event& b) {
  float t = 0.f;
  GSGP_CUDA(cudaEventElapsedTime(&t, a.e, b.e));
  return t;
}

// ---------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommInitAll) commInitAll = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclCommAbort) commAbort = nullptr;
  decltype(&ncclGetErrorString) errStr = nullptr;

  void load() {
    if (h) return;
    // prefer an already-loaded libnccl (e.g. torch's); RTLD_NOLOAD first
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw Error{ERR_NCCL, std::string("cannot load libnccl.so.2: ") + dlerror()};
    getUniqueId = (decltype(getUniqueId))dlsym(h, "ncclGetUniqueId");
    commInitRank = (decltype(commInitRank))dlsym(h, "ncclCommInitRank");
    commInitAll = (decltype(commInitAll))dlsym(h, "ncclCommInitAll");
    allReduce = (decltype(allReduce))dlsym(h, "ncclAllReduce");
    commDestroy = (decltype(commDestroy))dlsym(h, "ncclCommDestroy");
    commAbort = (decltype(commAbort))dlsym(h, "ncclCommAbort");
    errStr = (decltype(errStr))dlsym(h, "ncclGetErrorString");
    if (!getUniqueId || !commInitRank || !commInitAll || !allReduce || !commDestroy || !commAbort || !errStr)
      throw Error{ERR_NCCL, "libnccl.so.2 lacks required symbols"};
  }
  void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw Error{ERR_NCCL, std::string(what) + ": " + errStr(r)};
  }
};

NcclApi& nccl() {
  static NcclApi api;
  return api;
}

// GSGP_FORCE_COLLECTIVES=1 (tests): a one-rank job still creates its NCCL
// communicator and runs every collective through it, so the NCCL transport
// (dlopen, allreduce, graph capture of the NCCL kernels) executes on a
// one-GPU box; results must equal the collective-free path bit for bit.
bool force_collectives() {
  const char* e = getenv("GSGP_FORCE_COLLECTIVES");
  return e && e[0] == '1';
}

// Host exchange (tests): the same collectives through a host callback that
// reduces a host buffer over the ranks (e.g. torch.distributed over gloo), so
// the multi-rank engine path runs with several processes on one GPU.  The
// callback's code (HostRed below): 0 fp64 sum, 1 int32 sum, 2 uint64 sum,
// 3 int32 max.  Not graph-capturable: runs use direct launches.
enum HostRed : int32_t { kRedF64Sum = 0, kRedI32Sum = 1, kRedU64Sum = 2, kRedI32Max = 3 };
typedef void (*HostAllreduce)(void* buf, int64_t count, int32_t dtype);

// Thread exchange: the device threads of ONE process (gsgp_init with a
// device list naming a GPU twice, or GSGP_THREAD_EXCHANGE=1) reduce through
// host memory with a barrier, every thread summing the ranks' buffers in
// rank order.  Lets the single-process multi-device driver run on one GPU.
struct ThreadXchg {
  int n = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t phase = 0;
  bool aborted = false;
  std::vector<const unsigned char*> bufs;

  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const int64_t ph = phase;
    if (aborted) throw Error{ERR_CUDA, "another device thread of this run failed"};
    if (++arrived == n) {
      arrived = 0;
      ++phase;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return phase != ph || aborted; });
      if (aborted) throw Error{ERR_CUDA, "another device thread of this run failed"};
    }
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
  }
};

struct CommState {
  ncclComm_t comm = nullptr;
  HostAllreduce host = nullptr;
  ThreadXchg* tx = nullptr;
  int world = 1, rank = 0;
  bool owns_comm = true;   // false: the comm belongs to the device set (gsgp_init)
};
// the process communicator (one process per GPU), or — inside a device
// thread of a single-process multi-device run — that thread's own state
thread_local CommState* t_comm = nullptr;
CommState& comm_state() {
  static CommState c;
  return t_comm ? *t_comm : c;
}

// collectives run when there is more than one rank or a communicator/exchange
// exists (forced one-rank collectives)
bool collective(const CommState& c) { return c.world > 1 || c.comm || c.tx; }

void comm_unique_id(unsigned char* id) {
  nccl().load();
  ncclUniqueId u;
  nccl().check(nccl().getUniqueId(&u), "ncclGetUniqueId");
  std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
}

void comm_reset(CommState& c) {
  if (c.comm && c.owns_comm) nccl().commDestroy(c.comm);
  c.comm = nullptr;
  c.host = nullptr;
  c.tx = nullptr;
  c.world = 1;
  c.rank = 0;
  c.owns_comm = true;
}

void comm_init(int world, int rank, const unsigned char* id) {
  GSGP_REQUIRE(world >= 1 && rank >= 0 && rank < world, "bad world/rank");
  GSGP_REQUIRE(t_comm == nullptr, "comm_init inside a device thread");
  CommState& c = comm_state();
  comm_reset(c);
  c.world = world;
  c.rank = rank;
  if (world == 1 && !force_collectives()) return;
  nccl().load();
  ncclUniqueId u;
  std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
  nccl().check(nccl().commInitRank(&c.comm, world, u, rank), "ncclCommInitRank");
}

void comm_init_host(int world, int rank, HostAllreduce fn) {
  GSGP_REQUIRE(world >= 1 && rank >= 0 && rank < world && fn, "bad world/rank/callback");
  CommState& c = comm_state();
  comm_reset(c);
  c.world = world;
  c.rank = rank;
  c.host = fn;
}

template <typename T, typename Op>
void reduce_ranks(const std::vector<const unsigned char*>& bufs, int64_t count, unsigned char* dst, Op op) {
  T* d = reinterpret_cast<T*>(dst);
  for (int64_t e = 0; e < count; ++e) {
    T a = reinterpret_cast<const T*>(bufs[0])[e];
    for (size_t r = 1; r < bufs.size(); ++r) a = op(a, reinterpret_cast<const T*>(bufs[r])[e]);
    d[e] = a;
  }
}

// in-place reduction over the ranks of a device buffer on stream s (NCCL,
// host callback or thread exchange)
void allreduce(void* dev, int64_t count, HostRed kind, cudaStream_t s, const char* what) {
  CommState& c = comm_state();
  if (!collective(c)) return;
  const bool i32 = kind == kRedI32Sum || kind == kRedI32Max;
  const size_t esz = i32 ? 4 : 8;
  if (c.host || c.tx) {
    std::vector<unsigned char> h(count * esz);
    GSGP_CUDA(cudaMemcpyAsync(h.data(), dev, count * esz, cudaMemcpyDeviceToHost, s));
    GSGP_CUDA(cudaStreamSynchronize(s));
    if (c.host) {
      c.host(h.data(), count, (int32_t)kind);
    } else {
      ThreadXchg& x = *c.tx;
      x.bufs[c.rank] = h.data();
      x.barrier();                                    // every rank's buffer is published
      std::vector<unsigned char> acc(count * esz);
      switch (kind) {
        case kRedF64Sum: reduce_ranks<double>(x.bufs, count, acc.data(), [](double a, double b) { return a + b; }); break;
        case kRedI32Sum: reduce_ranks<int32_t>(x.bufs, count, acc.data(), [](int32_t a, int32_t b) { return a + b; }); break;
        case kRedU64Sum:
          reduce_ranks<uint64_t>(x.bufs, count, acc.data(), [](uint64_t a, uint64_t b) { return a + b; });
          break;
        default: reduce_ranks<int32_t>(x.bufs, count, acc.data(), [](int32_t a, int32_t b) { return a > b ? a : b; });
      }
      x.barrier();                                    // every rank has read every buffer
      h.swap(acc);
    }
    GSGP_CUDA(cudaMemcpyAsync(dev, h.data(), count * esz, cudaMemcpyHostToDevice, s));
    GSGP_CUDA(cudaStreamSynchronize(s));
    return;
  }
  const ncclDataType_t t = kind == kRedF64Sum ? ncclFloat64 : (i32 ? ncclInt32 : ncclUint64);
  const ncclRedOp_t op = kind == kRedI32Max ? ncclMax : ncclSum;
  nccl().check(nccl().allReduce(dev, dev, count, t, op, c.comm, s), what);
}

void comm_destroy() {
  GSGP_REQUIRE(t_comm == nullptr, "comm_destroy inside a device thread");
  comm_reset(comm_state());
}

// Contiguous case slices whose boundaries are multiples of kCaseAlign (the
// lcm of the generation kernel's case tiles, 4096 / 2048, and every
// interpreter tile, 128 x {1,2,3,4,8}): each SSE tile partial then covers the
// same global cases at the same positions for any shard count, and the
// canonical sum (common.cuh) makes the SSE identical across GPU counts.
constexpr int64_t kCaseAlign = 12288;

void shard_range(int64_t n, int64_t count, int64_t index, int64_t* lo, int64_t* hi) {
  auto cut = [&](int64_t i) { return i >= count ? n : (n * i) / count / kCaseAlign * kCaseAlign; };
  *lo = cut(index);
  *hi = cut(index + 1);
}

// ------------------------------------------------------------- small kernels
namespace {

__global__ void k_transpose(const double* __restrict__ Xr, int64_t N, int l, double* __restrict__ XT) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= N * l) return;
  int64_t q = e / l, f = e - q * l;
  XT[f * N + q] = Xr[e];
}

__global__ void k_wide_split(const int32_t* wide, int64_t m, int32_t* bits) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  bits[2 * i] = wide[i] & 1;
  bits[2 * i + 1] = (wide[i] >> 1) & 1;
}

__global__ void k_wide_merge(const int32_t* bits, int64_t m, int32_t* wide) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  wide[i] = (bits[2 * i] > 0 ? 1 : 0) | (bits[2 * i + 1] > 0 ? 2 : 0);
}

inline unsigned nblk(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t > 0 ? (n + t - 1) / t : 1); }

}  // namespace

// --------------------------------------------------------------------- run
// pinned host staging for the chunked case upload, kept for the process
// lifetime (grown on demand): page-locking a fresh buffer per run would cost
// more than the copy it enables
constexpr size_t kUploadChunkBytes = 48u << 20;
constexpr int kMaxDevices = 64;
struct PinnedStage {
  void* p = nullptr;
  size_t bytes = 0;
};
// Pinned staging buffers are pooled for the process lifetime: a run takes
// one (the device threads of a multi-device run each take their own, even
// when they share a GPU), uses it for every chunked upload, and returns it
// at the end, so the next run neither page-locks nor frees ~100 MB again.
std::mutex g_pin_mu;
std::vector<PinnedStage> g_pin_free;

struct PinnedLease {
  PinnedStage st{};
  PinnedLease() = default;
  PinnedLease(const PinnedLease&) = delete;
  PinnedLease& operator=(const PinnedLease&) = delete;
  ~PinnedLease() {
    if (!st.p) return;
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_free.push_back(st);
  }
  // at least `bytes`; a first use above 8 MB takes the full double buffer
  // (page-locking costs ~50 ms per 100 MB, which growing run by run would
  // charge to later runs), small uploads page-lock only what they need
  PinnedStage& get(size_t bytes) {
    const size_t full = 2 * kUploadChunkBytes + (64u << 10);
    if (bytes > (8u << 20) && bytes < full) bytes = full;
    if (st.bytes >= bytes) return st;
    {
      std::lock_guard<std::mutex> lk(g_pin_mu);
      if (st.p) g_pin_free.push_back(st);
      st = PinnedStage{};
      int best = -1;
      for (int i = 0; i < (int)g_pin_free.size(); ++i)
        if (g_pin_free[i].bytes >= bytes && (best < 0 || g_pin_free[i].bytes < g_pin_free[best].bytes)) best = i;
      if (best >= 0) {
        st = g_pin_free[best];
        g_pin_free.erase(g_pin_free.begin() + best);
        return st;
      }
    }
    GSGP_CUDA(cudaHostAlloc(&st.p, bytes, cudaHostAllocPortable));
    st.bytes = bytes;
    return st;
  }
};

void trim_device_memory() {
  cache_trim();
  std::lock_guard<std::mutex> lk(g_pin_mu);
  for (auto& ps : g_pin_free) cudaFreeHost(ps.p);
  g_pin_free.clear();
}

struct Shard {
  int64_t tr_lo = 0, tr_hi = 0, te_lo = 0, te_hi = 0;
  int64_t ntr = 0, nte = 0, pitch = 0, ntiles = 0, itiles = 0;
  RowLayout lay{};
  DevBuf S, pool, elite[2], y_store, part, ipart, ticket;
};

void run_engine(const gsgp_config* cfg, const double* Xtr, const double* ytr, int64_t ntr,
                const double* Xte, const double* yte, int64_t nte, int32_t l, gsgp_outputs* out) {
  auto t_host0 = std::chrono::steady_clock::now();
  GSGP_REQUIRE(cfg && out, "null config/outputs");
  const int64_t m = cfg->population_size, r = cfg->random_trees, k = cfg->program_size,
                g = cfg->generations;
  GSGP_REQUIRE(m >= 1 && r >= 1 && k >= 1, "population_size, random_trees, program_size must be >= 1");
  GSGP_REQUIRE(g >= 0, "generations must be >= 0");
  GSGP_REQUIRE(r >= 2 || g == 0, "geometric semantic mutation needs at least 2 random trees");
  GSGP_REQUIRE(ntr >= 1 && nte >= 1 && l >= 1, "datasets must have at least one row and one feature");
  GSGP_REQUIRE(l <= 65535, "at most 65535 features");
  GSGP_REQUIRE(k < (1ll << 24), "program_size too large");
  const double total = cfg->p_function + cfg->p_feature + cfg->p_constant;
  GSGP_REQUIRE(cfg->p_function >= 0 && cfg->p_feature >= 0 && cfg->p_constant >= 0 && total > 0,
               "gene probabilities must be non-negative with positive sum");
  GSGP_REQUIRE(cfg->division_eps > 0, "division_eps must be > 0");
  GSGP_REQUIRE(cfg->mutation_step_uniform || (std::isfinite(cfg->mutation_step) && cfg->mutation_step > 0),
               "constant mutation_step must be finite and > 0");
  // fp32 storage is only taken when no stored value can leave fp32 range or
  // drift far enough to move an fp32-overflow row's fitness:
  // per generation |t| <= step * (1 or 2), so a cumulative drift below 2^70
  // keeps every finite fp32 value finite (a step < 2^103 cannot round past
  // FLT_MAX) and leaves the squares of overflow rows absorbed.  Larger
  // constant steps (gsgp/core.py:332-336 allows any finite step) run in fp64.
  const double step_bound = (cfg->mutation_step_uniform ? 1.0 : cfg->mutation_step) *
                            (cfg->gsm_sign ? 2.0 : 1.0) * (double)(g > 0 ? g : 1);
  const bool f64 = cfg->storage_f64 != 0 || !(step_bound < 0x1p70);
  out->storage_f64_used = f64 ? 1 : 0;
  for (int q = 0; q < 4; ++q) out->interp_info[q] = -1;
  const size_t esz = f64 ? 8 : 4;
  const int G = cfg->virtual_shards < 1 ? 1 : cfg->virtual_shards;
  GSGP_REQUIRE(G <= 16, "at most 16 virtual shards");
  CommState& cs = comm_state();
  const int W = cs.world;
  const bool coll = collective(cs);   // exchange the per-rank sums (W > 1, or forced one-rank collectives)
  const int64_t nsh_total = (int64_t)W * G;

  cudaStream_t st, up;   // compute stream, host->device upload stream
  GSGP_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } sg{st};
  GSGP_CUDA(cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking));
  StreamGuard sg_up{up};
  struct AllocStream {            // DevBufs of this run drain st before parking their blocks
    cudaStream_t prev;
    explicit AllocStream(cudaStream_t s) : prev(g_alloc_stream) { g_alloc_stream = s; }
    ~AllocStream() { g_alloc_stream = prev; }
  } alloc_stream{st};

  // ---- shards and per-shard device data
  std::vector<std::unique_ptr<Shard>> sh;
  for (int s = 0; s < G; ++s) {
    auto p = std::make_unique<Shard>();
    const int64_t gs = (int64_t)cs.rank * G + s;
    shard_range(ntr, nsh_total, gs, &p->tr_lo, &p->tr_hi);
    shard_range(nte, nsh_total, gs, &p->te_lo, &p->te_hi);
    p->ntr = p->tr_hi - p->tr_lo;
    p->nte = p->te_hi - p->te_lo;
    p->lay = make_layout(p->ntr, p->nte, f64);
    p->pitch = p->lay.pitch;
    p->ntiles = p->lay.ntiles;
    sh.push_back(std::move(p));
  }
  out->shard_train_lo = sh.front()->tr_lo;
  out->shard_train_hi = sh.back()->tr_hi;

  // pinned upload staging, taken before the timed stages (page-locking is a
  // host cost of the first run, not of CreatePopulation / ComputeSemantics):
  // the double buffer of the largest shard's upload chunk (every interpreter
  // tile divides 3072)
  PinnedLease pin_lease;
  {
    size_t upload_bound = 0;
    const size_t row_bytes = (size_t)l * 8 + 8;
    for (auto& p : sh) {
      const int64_t Nq = (p->ntr + p->nte + 3072 + 3071) / 3072 * 3072;   // + the test-start gap
      int64_t chunk = std::max<int64_t>(3072, (int64_t)(kUploadChunkBytes / row_bytes) / 3072 * 3072);
      if (const char* e = getenv("GSGP_UPLOAD_CHUNK")) chunk = std::max<int64_t>(3072, atoll(e) / 3072 * 3072);
      upload_bound = std::max(upload_bound, 2 * (size_t)std::min(chunk, Nq) * row_bytes);
    }
    if (upload_bound) pin_lease.get(upload_bound);
  }
  {   // first run on this device: load the kernels before any timed stage
    static std::mutex mu;
    static std::set<int> loaded;
    std::lock_guard<std::mutex> lk(mu);
    if (loaded.insert(current_device()).second) {
      interp_preload();
      gsm_preload();
    }
  }
  Event ev_begin, ev_created, ev_sem, ev_loop0, ev_loop1;
  GSGP_CUDA(cudaEventRecord(ev_begin.e, st));

  // ---- global (replicated) state
  DevBuf tags, codes, consts, ins, exe, plen, pnconst, ctab, pmax, scratch, flags, cval, pndiv;
  const int64_t ng = m + r;
  tags.alloc(ng * k);
  codes.alloc(ng * k * 4);
  consts.alloc(ng * k * 8);
  ins.alloc(ng * (k + 1) * sizeof(Ins));
  plen.alloc(ng * 4);
  pndiv.alloc(ng * 16);   // [ng][4] op mix
  // linked programs: per-launch scratch, one copy per interpreter genome
  // group, sized for programs of up to k instructions (allocated here, before
  // the timed stages)
  const LinkedLayout ll = linked_layout(std::max(m, r), (int32_t)k);
  exe.alloc(ll.ins * sizeof(Ins));
  pnconst.alloc(ng * 4);
  ctab.alloc(ng * k * 8);
  pmax.alloc(4 * 4);
  scratch.alloc(ng * 4 * k * 4);
  flags.alloc(ng * k);
  cval.alloc(ng * k * 8);
  DevBuf F, TS, wide, ctl, sse_total, nonfinite;
  F.alloc(m * 8); TS.alloc(m * 8);
  wide.alloc(m * 4);
  ctl.alloc(CTL_WORDS * 8);
  sse_total.alloc(m * 2 * 8);
  nonfinite.alloc(8);
  GSGP_CUDA(cudaMemsetAsync(wide.p, 0, m * 4, st));
  GSGP_CUDA(cudaMemsetAsync(ctl.p, 0, CTL_WORDS * 8, st));
  GSGP_CUDA(cudaMemsetAsync(nonfinite.p, 0, 8, st));
  DevBuf pu, pv, pms, rsrc, ridx, rslot, rfit, ttr, tte;
  const int64_t gm = (g > 0 ? g : 1) * m;
  pu.alloc(gm * 8); pv.alloc(gm * 8); pms.alloc(gm * 8);
  rsrc.alloc(g + 1); ridx.alloc((g + 1) * 8); rslot.alloc((g + 1) * 8); rfit.alloc((g + 1) * 8);
  ttr.alloc((g + 1) * 8); tte.alloc((g + 1) * 8);

  // ---- CreatePopulation (population.py:73-92; evolution.py:117-118)
  GeneParams gp;
  gp.seed = cfg->seed;
  gp.thr_fun = cfg->p_function / total;
  gp.thr_feat = gp.thr_fun + cfg->p_feature / total;
  gp.erc_low = cfg->erc_low;
  gp.erc_high = cfg->erc_high;
  gp.n_features = l;
  gp.k = (int32_t)k;
  launch_create_population(gp, m, 0, tags.as<uint8_t>(), codes.as<int32_t>(), consts.as<double>(), st);
  launch_create_population(gp, r, (uint64_t)m, tags.as<uint8_t>() + m * k, codes.as<int32_t>() + m * k,
                           consts.as<double>() + m * k, st);
  GSGP_CUDA(cudaEventRecord(ev_created.e, st));

  // ---- compile all m + r genomes once
  Program prog{ins.as<Ins>(), exe.as<Ins>(), plen.as<int32_t>(), pnconst.as<int32_t>(),
               ctab.as<double>(), pmax.as<int32_t>(), scratch.as<int32_t>(), flags.as<uint8_t>(),
               cval.as<double>(), pndiv.as<int32_t>()};
  Event ev_compile0, ev_compile1;
  GSGP_CUDA(cudaEventRecord(ev_compile0.e, st));
  launch_compile(tags.as<uint8_t>(), codes.as<int32_t>(), consts.as<double>(), ng, (int32_t)k,
                 cfg->division_eps, prog, st);
  GSGP_CUDA(cudaEventRecord(ev_compile1.e, st));
  int32_t maxima[4] = {0, 0, 0, 0};   // {spill depth, constants, instructions, unused}
  GSGP_CUDA(cudaMemcpyAsync(maxima, pmax.p, 16, cudaMemcpyDeviceToHost, st));
  // program lengths: one instruction per function node of the compiled tree
  // (the interpreter's work unit, reported as node evaluations per second)
  std::vector<int32_t> hlen(ng), hdiv(ng * 4);
  GSGP_CUDA(cudaMemcpyAsync(hlen.data(), plen.p, ng * 4, cudaMemcpyDeviceToHost, st));
  GSGP_CUDA(cudaMemcpyAsync(hdiv.data(), pndiv.p, ng * 16, cudaMemcpyDeviceToHost, st));
  GSGP_CUDA(cudaStreamSynchronize(st));

  // pin_lease (this run's pinned upload staging) was taken before the timed
  // stages: see upload_bound
  // ---- per shard: upload the case slice, interpret population and pool
  double init_phase_ms[4] = {0, 0, 0, 0};   // upload, population, pool, initial SSE
  double alloc_ms = 0.0;                     // host clock: device allocations + clears
  for (auto& p : sh) {
    const int64_t N = p->ntr + p->nte;
    const auto t_alloc0 = std::chrono::steady_clock::now();
    p->S.alloc(m * p->pitch * esz);
    p->pool.alloc(r * p->pitch * esz);
    p->elite[0].alloc(p->pitch * esz);
    p->elite[1].alloc(p->pitch * esz);
    p->y_store.alloc(p->pitch * 8);
    p->part.alloc(m * p->ntiles * 2 * 8);
    p->ticket.alloc(16);
    GSGP_CUDA(cudaMemsetAsync(p->ticket.p, 0, 16, st));
    // the interpreter writes every case column of every population and pool
    // row, so only the padding columns are cleared (a full clear of the C3
    // matrices was 102 GB of memset, ~14 ms of every run's init)
    auto clear_padding = [&](void* base, int64_t rows) {
      const RowLayout& L = p->lay;
      auto clr = [&](int64_t c0, int64_t c1) {
        if (c1 > c0 && rows > 0)
          GSGP_CUDA(cudaMemset2DAsync(static_cast<char*>(base) + c0 * esz, (size_t)(L.pitch * esz), 0,
                                      (size_t)((c1 - c0) * esz), (size_t)rows, st));
      };
      clr(L.ntr, L.ntr_pad);                                     // train padding
      if (L.tail_off >= 0) clr(L.tail_off + (L.nte - L.te_full), L.tail_off + L.tail_pad);   // test tail padding
      else clr(L.test_off + L.nte, L.pitch);                     // test padding
    };
    clear_padding(p->S.p, m);
    clear_padding(p->pool.p, r);
    GSGP_CUDA(cudaMemsetAsync(p->elite[0].p, 0, p->pitch * esz, st));
    GSGP_CUDA(cudaMemsetAsync(p->elite[1].p, 0, p->pitch * esz, st));
    GSGP_CUDA(cudaMemsetAsync(p->y_store.p, 0, p->pitch * 8, st));
    GSGP_CUDA(cudaStreamSynchronize(st));
    alloc_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_alloc0).count();
    if (N == 0) continue;
    // Cases are uploaded and interpreted in chunks: the host copies chunk c
    // into a pinned staging buffer while the device interprets chunk c-1, so
    // the feature upload hides behind the (compute-bound) interpreter.
    InterpArgs ia{};
    ia.code = ins.as<Ins>();
    ia.exe = exe.as<Ins>();
    ia.exe_k1 = ll.k1;
    ia.max_groups = ll.copies;
    ia.len = plen.as<int32_t>();
    ia.nconst = pnconst.as<int32_t>();
    ia.ctab = ctab.as<double>();
    ia.k1 = k + 1;
    ia.count = m;
    ia.l = l;
    ia.ntr = p->ntr;
    ia.nte = p->nte;
    ia.te_q = p->ntr;
    ia.eps = cfg->division_eps;
    ia.maxdepth = maxima[0];
    ia.maxconst = maxima[1];
    ia.maxlen = maxima[2];
    ia.out = p->S.p;
    ia.out_is_f64 = f64 ? 1 : 0;
    ia.pitch = p->pitch;
    ia.test_off = p->lay.test_off;
    ia.te_full = p->lay.te_full;
    ia.tail_off = p->lay.tail_off;
    ia.y = p->y_store.as<double>();
    ia.wide = wide.as<int32_t>();
    ia.nonfinite = nonfinite.as<unsigned long long>();
    int itile = 1;
    interp_tiles(ia, &itile);
    out->interp_info[0] = interp_config(ia);
    for (int q = 0; q < 3; ++q) out->interp_info[1 + q] = maxima[q];
    // test cases start on an interpreter tile (stacked index te_q), so no
    // tile mixes train and test cases: canonical partials (see shard_range)
    ia.te_q = (p->ntr + itile - 1) / itile * itile;
    const int64_t itiles = interp_tiles(ia, nullptr);
    const int64_t Nq = ia.te_q + p->nte;                    // stacked cases incl. the gap
    p->itiles = itiles;
    p->ipart.alloc(m * itiles * 2 * 8);
    ia.part = p->ipart.as<double>();
    ia.part_ntiles = itiles;
    // pool: stream base m, same compiled program buffer offset by m genomes
    InterpArgs ip = ia;
    ip.code = ins.as<Ins>() + m * (k + 1);
    ip.exe = exe.as<Ins>();   // relinked by every launch
    ip.len = plen.as<int32_t>() + m;
    ip.nconst = pnconst.as<int32_t>() + m;
    ip.ctab = ctab.as<double>() + m * k;
    ip.count = r;
    ip.out = p->pool.p;
    ip.part = nullptr;
    ip.wide = nullptr;
    ip.y = nullptr;

    const size_t row_bytes = (size_t)l * 8 + 8;             // features + target of one case
    // chunks are multiples of 3072 = lcm of every interpreter tile (128 .. 1024, 384)
    int64_t chunk = (int64_t)(kUploadChunkBytes / row_bytes) / 3072 * 3072;
    if (const char* e = getenv("GSGP_UPLOAD_CHUNK")) chunk = atoll(e) / 3072 * 3072;   // tests
    if (chunk < 3072) chunk = 3072;
    if (chunk > Nq) chunk = (Nq + itile - 1) / itile * itile;
    const int64_t nchunks = (Nq + chunk - 1) / chunk;
    PinnedStage& pin = pin_lease.get(2 * (size_t)chunk * row_bytes);
    DevBuf Xr[2], XT[2];
    for (int b = 0; b < 2 && b < nchunks; ++b) {
      Xr[b].alloc(chunk * l * 8);
      XT[b].alloc(chunk * l * 8);
    }
    Event ev_h2d[2], ev_done[2], e_start, e_first;
    std::vector<std::unique_ptr<Event>> ev_k;
    GSGP_CUDA(cudaEventRecord(e_start.e, st));
    for (int64_t c = 0; c < nchunks; ++c) {
      const int b = (int)(c & 1);
      const int64_t c0 = c * chunk, nq = std::min(chunk, Nq - c0);
      double* hx = reinterpret_cast<double*>(pin.p) + (size_t)b * chunk * (l + 1);
      double* hy = hx + (size_t)chunk * l;
      if (c >= 2) GSGP_CUDA(cudaEventSynchronize(ev_h2d[b].e));   // staging buffer b is free
      // stacked rows [c0, c0 + nq): train rows [c0, ntr), gap rows [ntr, te_q)
      // (zero features, never stored or counted), test rows [te_q, Nq)
      const int64_t tr_end = std::min(c0 + nq, p->ntr);
      const int64_t ntr_part = std::max<int64_t>(0, tr_end - c0);
      const int64_t te_beg = std::max(c0, ia.te_q);
      const int64_t nte_part = std::max<int64_t>(0, c0 + nq - te_beg);
      const int64_t gap0 = std::max(c0, p->ntr), ngap = std::max<int64_t>(0, std::min(c0 + nq, ia.te_q) - gap0);
      if (ntr_part > 0) {
        std::memcpy(hx, Xtr + (p->tr_lo + c0) * l, ntr_part * l * 8);
        std::memcpy(hy, ytr + p->tr_lo + c0, ntr_part * 8);
      }
      if (ngap > 0) std::memset(hx + (gap0 - c0) * l, 0, ngap * l * 8);
      if (nte_part > 0) {
        const int64_t t0 = te_beg - ia.te_q;                // first test row of the chunk
        std::memcpy(hx + (te_beg - c0) * l, Xte + (p->te_lo + t0) * l, nte_part * l * 8);
        std::memcpy(hy + (te_beg - c0), yte + p->te_lo + t0, nte_part * 8);
      }
      if (c >= 2) GSGP_CUDA(cudaStreamWaitEvent(up, ev_done[b].e, 0));   // device buffers free
      GSGP_CUDA(cudaMemcpyAsync(Xr[b].p, hx, nq * l * 8, cudaMemcpyHostToDevice, up));
      if (ntr_part > 0)
        GSGP_CUDA(cudaMemcpyAsync(p->y_store.as<double>() + c0, hy, ntr_part * 8, cudaMemcpyHostToDevice, up));
      if (nte_part > 0) {   // test targets [j0, j0 + nte_part) in storage order (RowLayout)
        const int64_t j0 = te_beg - ia.te_q;
        const int64_t nfull = std::max<int64_t>(0, std::min(j0 + nte_part, p->lay.te_full) - j0);
        const double* src = hy + (te_beg - c0);
        if (nfull > 0)
          GSGP_CUDA(cudaMemcpyAsync(p->y_store.as<double>() + test_col(p->lay, j0), src, nfull * 8,
                                    cudaMemcpyHostToDevice, up));
        if (nte_part > nfull)
          GSGP_CUDA(cudaMemcpyAsync(p->y_store.as<double>() + test_col(p->lay, j0 + nfull), src + nfull,
                                    (nte_part - nfull) * 8, cudaMemcpyHostToDevice, up));
      }
      GSGP_CUDA(cudaEventRecord(ev_h2d[b].e, up));
      GSGP_CUDA(cudaStreamWaitEvent(st, ev_h2d[b].e, 0));
      k_transpose<<<nblk(nq * l), 256, 0, st>>>(Xr[b].as<double>(), nq, l, XT[b].as<double>());
      GSGP_CUDA(cudaGetLastError());
      if (c == 0) GSGP_CUDA(cudaEventRecord(e_first.e, st));
      for (InterpArgs* q : {&ia, &ip}) {
        q->XT = XT[b].as<double>();
        q->xt_pitch = nq;
        q->q_base = c0;
        q->nq = nq;
      }
      ev_k.push_back(std::make_unique<Event>());
      GSGP_CUDA(cudaEventRecord(ev_k.back()->e, st));
      launch_interpret(ia, INTERP_POP, st);
      ev_k.push_back(std::make_unique<Event>());
      GSGP_CUDA(cudaEventRecord(ev_k.back()->e, st));
      launch_interpret(ip, INTERP_POOL, st);
      ev_k.push_back(std::make_unique<Event>());
      GSGP_CUDA(cudaEventRecord(ev_k.back()->e, st));
      GSGP_CUDA(cudaEventRecord(ev_done[b].e, st));
    }
    Event e_sse0, e_sse;
    GSGP_CUDA(cudaEventRecord(e_sse0.e, st));
    // initial SSE of the stored semantics in the generation kernel's order
    GsmArgs ga{};
    ga.pool = p->pool.p;
    ga.S = p->S.p;
    ga.elite_prev = p->elite[0].p;
    ga.elite_cur = p->elite[1].p;
    ga.y = p->y_store.as<double>();
    ga.lay = p->lay;
    ga.m = m;
    ga.part = p->part.as<double>();
    ga.ticket = p->ticket.as<unsigned long long>();
    launch_sse_only(ga, f64, st);
    GSGP_CUDA(cudaEventRecord(e_sse.e, st));
    GSGP_CUDA(cudaEventSynchronize(e_sse.e));   // the shard's temporaries are freed at scope end
    init_phase_ms[0] += elapsed_ms(e_start, e_first);      // exposed upload (first chunk)
    for (size_t q = 0; q + 2 < ev_k.size(); q += 3) {
      init_phase_ms[1] += elapsed_ms(*ev_k[q], *ev_k[q + 1]);
      init_phase_ms[2] += elapsed_ms(*ev_k[q + 1], *ev_k[q + 2]);
    }
    init_phase_ms[3] += elapsed_ms(e_sse0, e_sse);
    GSGP_CUDA(cudaStreamSynchronize(st));   // temporaries (Xr, XT) are freed on scope exit
  }

  // ---- canonical SSE over every shard of every rank (common.cuh canon_*):
  // anchors (max over shards, allreduce-max over ranks), exact digit sums
  // (over shards, allreduce-sum over ranks), one rounding.  Bit-identical
  // for any rank / virtual-shard count.
  DevBuf sse64_total, cexp, cdig;
  sse64_total.alloc(m * 2 * 8);
  cexp.alloc(m * 2 * 4);
  cdig.alloc(m * 2 * kLimbs * 8);
  double* sse_vec = sse_total.as<double>();
  double* sse64_vec = sse64_total.as<double>();
  auto canon_sse = [&](bool interp_parts, double* dst, cudaStream_t s) {
    launch_canon_clear(m, cexp.as<int32_t>(), cdig.as<unsigned long long>(), s);
    for (auto& p : sh) {
      if (p->pitch == 0) continue;
      if (interp_parts) launch_canon_exp(p->ipart.as<double>(), m, p->itiles, cexp.as<int32_t>(), s);
      else launch_canon_exp(p->part.as<double>(), m, p->ntiles, cexp.as<int32_t>(), s);
    }
    if (coll) allreduce(cexp.p, m * 2, kRedI32Max, s, "ncclAllReduce(sse anchors)");
    for (auto& p : sh) {
      if (p->pitch == 0) continue;
      if (interp_parts)
        launch_canon_digits(p->ipart.as<double>(), m, p->itiles, cexp.as<int32_t>(),
                            cdig.as<unsigned long long>(), s);
      else
        launch_canon_digits(p->part.as<double>(), m, p->ntiles, cexp.as<int32_t>(),
                            cdig.as<unsigned long long>(), s);
    }
    if (coll) allreduce(cdig.p, m * 2 * kLimbs, kRedU64Sum, s, "ncclAllReduce(sse digits)");
    launch_canon_finish(cexp.as<int32_t>(), cdig.as<unsigned long long>(), m, dst, s);
  };
  // GSGP_TEST_FAIL_RANK=i (tests): rank i of a multi-rank run fails here,
  // while the other ranks wait in the first exchange, to check that a failed
  // device thread aborts its peers instead of leaving them blocked
  if (const char* f = getenv("GSGP_TEST_FAIL_RANK"))
    if (coll && atoi(f) == cs.rank) throw Error{ERR_CUDA, "injected failure (GSGP_TEST_FAIL_RANK)"};
  canon_sse(false, sse_vec, st);
  canon_sse(true, sse64_vec, st);
  GSGP_CUDA(cudaStreamSynchronize(st));
  for (auto& p : sh) p->ipart.release();
  if (coll) {
    DevBuf bits;
    bits.alloc(m * 2 * 4);
    k_wide_split<<<nblk(m), 256, 0, st>>>(wide.as<int32_t>(), m, bits.as<int32_t>());
    allreduce(bits.p, m * 2, kRedI32Sum, st, "ncclAllReduce(wide)");
    k_wide_merge<<<nblk(m), 256, 0, st>>>(bits.as<int32_t>(), m, wide.as<int32_t>());
    allreduce(nonfinite.p, 1, kRedU64Sum, st, "ncclAllReduce(overflow)");
    GSGP_CUDA(cudaStreamSynchronize(st));
  }

  SurviveArgs sa{};
  sa.m = m;
  sa.ntr = (double)ntr;
  sa.nte = (double)nte;
  sa.sse_off = sse_vec;
  sa.sse_alt = sse64_vec;
  sa.F = F.as<double>();
  sa.TS = TS.as<double>();
  sa.wide = wide.as<int32_t>();
  sa.ctl = ctl.as<int64_t>();
  sa.rec_src = rsrc.as<int8_t>();
  sa.rec_idx = ridx.as<int64_t>();
  sa.rec_slot = rslot.as<int64_t>();
  sa.rec_fit = rfit.as<double>();
  sa.trace_tr = ttr.as<double>();
  sa.trace_te = tte.as<double>();
  launch_init_state(sa, st);
  GSGP_CUDA(cudaEventRecord(ev_sem.e, st));

  // ---- generation loop (evolution.py:146-158)
  PlanParams pp{cfg->seed, m, r, cfg->mutation_step_uniform, cfg->mutation_step};
  const bool timed = cfg->time_kernels != 0;
  std::vector<std::unique_ptr<Event>> tev;
  int64_t launches_per_gen = 0;
  DevBuf done;
  done.alloc(16);
  GSGP_CUDA(cudaMemsetAsync(done.p, 0, 16, st));
  const bool fused_tail = (G == 1 && !coll);
  // fused tail: the GSM launch accumulates the canonical-sum anchors, the
  // reduce reads the partials once and re-arms the anchors (kExpZero)
  DevBuf gemax;
  gemax.alloc(m * 2 * 4);
  GSGP_CUDA(cudaMemsetAsync(gemax.p, 0x80, m * 2 * 4, st));
  GSGP_CUDA(cudaMemsetAsync(cdig.p, 0, m * 2 * kLimbs * 8, st));   // digit sums of the sharded tail
  // one generation: GSM+SSE with the plan drawn inline (per shard; every
  // launch accumulates the canonical-sum anchors), then the canonical SSE and
  // survival — one kernel when there is a single shard, else digits per
  // shard (between the two allreduces) and one finish + survive kernel
  auto enqueue_generation = [&](cudaStream_t s, Event* t0, Event* t1) {
    int64_t n = 0;
    if (t0) GSGP_CUDA(cudaEventRecord(t0->e, s));
    bool plan_written = false;
    for (size_t si = 0; si < sh.size(); ++si) {
      auto& p = sh[si];
      if (p->pitch == 0) continue;
      GsmArgs a{};
      a.pool = p->pool.p;
      a.S = p->S.p;
      a.elite_prev = p->elite[0].p;
      a.elite_cur = p->elite[1].p;
      a.y = p->y_store.as<double>();
      a.lay = p->lay;
      a.m = m;
      a.u = pu.as<int64_t>();
      a.v = pv.as<int64_t>();
      a.ms = pms.as<double>();
      a.ctl = ctl.as<int64_t>();
      a.sign = cfg->gsm_sign;
      a.part = p->part.as<double>();
      a.ticket = p->ticket.as<unsigned long long>();
      // anchors: every shard of the sharded tail; the fused tail only when a
      // row has several units (single unit: SSE = partial)
      a.emax = (!fused_tail || p->ntiles > 1) ? gemax.as<int32_t>() : nullptr;
      a.plan_inline = 1;
      a.write_plan = plan_written ? 0 : 1;   // the first non-empty shard records the plan
      plan_written = true;
      a.plan = pp;
      launch_gsm(a, f64, false, s);
      ++n;
    }
    if (!plan_written) {   // no cases on this rank: draw the plan for the lineage record
      launch_plan(pp, 0, ctl.as<int64_t>(), pu.as<int64_t>(), pv.as<int64_t>(), pms.as<double>(), m, s);
      ++n;
    }
    if (t1) GSGP_CUDA(cudaEventRecord(t1->e, s));
    if (fused_tail) {
      launch_reduce_survive(sh[0]->part.as<double>(), sh[0]->ntiles, gemax.as<int32_t>(), sse_vec, sa,
                            done.as<unsigned int>(), s);
      ++n;
    } else {
      // GSM (anchors) -> allreduce-max -> digits per shard -> allreduce-sum
      // -> finish + survive (re-arms anchors and digits)
      if (coll) allreduce(gemax.p, m * 2, kRedI32Max, s, "ncclAllReduce(sse anchors)");
      for (auto& p : sh) {
        if (p->pitch == 0) continue;
        launch_canon_digits(p->part.as<double>(), m, p->ntiles, gemax.as<int32_t>(),
                            cdig.as<unsigned long long>(), s);
        ++n;
      }
      if (coll) allreduce(cdig.p, m * 2 * kLimbs, kRedU64Sum, s, "ncclAllReduce(sse digits)");
      launch_finish_survive(gemax.as<int32_t>(), cdig.as<unsigned long long>(), sse_vec, sa,
                            done.as<unsigned int>(), s);
      ++n;
    }
    launches_per_gen = n;
  };
  // timing window: generations (w0, g]; ev_win0 is recorded after generation w0
  const int64_t w0 = cfg->window_start < 0 ? 0 : (cfg->window_start > g ? g : cfg->window_start);
  Event ev_win0;
  GSGP_CUDA(cudaEventRecord(ev_loop0.e, st));
  if (w0 == 0) GSGP_CUDA(cudaEventRecord(ev_win0.e, st));
  double gsm_ms = 0.0, win_gsm_ms = 0.0;
  if (g > 0) {
    cudaGraphExec_t exec = nullptr;
    cudaGraph_t graph = nullptr;
    if (!timed && cfg->use_graph && !cs.host && !cs.tx) {
      GSGP_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      enqueue_generation(st, nullptr, nullptr);
      GSGP_CUDA(cudaStreamEndCapture(st, &graph));
      GSGP_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    }
    if (timed)
      for (int64_t t = 0; t < 2 * g; ++t) tev.push_back(std::make_unique<Event>());
    for (int64_t t = 0; t < g; ++t) {
      if (timed) enqueue_generation(st, tev[2 * t].get(), tev[2 * t + 1].get());
      else if (exec) GSGP_CUDA(cudaGraphLaunch(exec, st));
      else enqueue_generation(st, nullptr, nullptr);
      if (t + 1 == w0) GSGP_CUDA(cudaEventRecord(ev_win0.e, st));
    }
    GSGP_CUDA(cudaEventRecord(ev_loop1.e, st));
    GSGP_CUDA(cudaStreamSynchronize(st));
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
  } else {
    GSGP_CUDA(cudaEventRecord(ev_loop1.e, st));
  }
  GSGP_CUDA(cudaStreamSynchronize(st));
  if (timed)
    for (int64_t t = 0; t < g; ++t) {
      const double d = elapsed_ms(*tev[2 * t], *tev[2 * t + 1]);
      if (out->gsm_ms) out->gsm_ms[t] = d;
      gsm_ms += d;
      if (t >= w0) win_gsm_ms += d;
    }

  // ---- results back to the host
  GSGP_CUDA(cudaMemcpyAsync(out->train_trace, ttr.p, (g + 1) * 8, cudaMemcpyDeviceToHost, st));
  GSGP_CUDA(cudaMemcpyAsync(out->test_trace, tte.p, (g + 1) * 8, cudaMemcpyDeviceToHost, st));
  GSGP_CUDA(cudaMemcpyAsync(out->elite_src, rsrc.p, g + 1, cudaMemcpyDeviceToHost, st));
  GSGP_CUDA(cudaMemcpyAsync(out->elite_idx, ridx.p, (g + 1) * 8, cudaMemcpyDeviceToHost, st));
  GSGP_CUDA(cudaMemcpyAsync(out->elite_slot, rslot.p, (g + 1) * 8, cudaMemcpyDeviceToHost, st));
  GSGP_CUDA(cudaMemcpyAsync(out->elite_fit, rfit.p, (g + 1) * 8, cudaMemcpyDeviceToHost, st));
  if (g > 0 && out->plan_u) GSGP_CUDA(cudaMemcpyAsync(out->plan_u, pu.p, g * m * 8, cudaMemcpyDeviceToHost, st));
  if (g > 0 && out->plan_v) GSGP_CUDA(cudaMemcpyAsync(out->plan_v, pv.p, g * m * 8, cudaMemcpyDeviceToHost, st));
  if (g > 0 && out->plan_ms) GSGP_CUDA(cudaMemcpyAsync(out->plan_ms, pms.p, g * m * 8, cudaMemcpyDeviceToHost, st));
  int64_t hctl[CTL_WORDS];
  unsigned long long hnf = 0;
  GSGP_CUDA(cudaMemcpyAsync(hctl, ctl.p, sizeof(hctl), cudaMemcpyDeviceToHost, st));
  GSGP_CUDA(cudaMemcpyAsync(&hnf, nonfinite.p, 8, cudaMemcpyDeviceToHost, st));
  GSGP_CUDA(cudaStreamSynchronize(st));
  out->overflow = (int64_t)hnf;

  // final elite train semantics: slot rec_slot[g]; a parent-sourced elite
  // lives in the elite buffer selected by the final parity (gsm.cu)
  const int64_t slot = out->elite_slot[g];
  const bool redirected = (g > 0 && hctl[CTL_REDIRECT] == slot);
  for (auto& p : sh) {
    if (p->ntr == 0 || !out->elite_train_semantics) continue;
    const char* src = redirected ? (const char*)p->elite[hctl[CTL_PARITY] & 1].p
                                 : (const char*)p->S.p + slot * p->pitch * esz;
    double* dst = out->elite_train_semantics + p->tr_lo;
    if (f64) {
      GSGP_CUDA(cudaMemcpy(dst, src, p->ntr * 8, cudaMemcpyDeviceToHost));
    } else {
      std::vector<float> tmp(p->ntr);
      GSGP_CUDA(cudaMemcpy(tmp.data(), src, p->ntr * 4, cudaMemcpyDeviceToHost));
      for (int64_t j = 0; j < p->ntr; ++j) dst[j] = (double)tmp[j];
    }
  }

  auto t_host1 = std::chrono::steady_clock::now();
  const double evo = elapsed_ms(ev_loop0, ev_loop1);
  out->stage_ms[0] = elapsed_ms(ev_begin, ev_created);
  out->stage_ms[1] = elapsed_ms(ev_created, ev_sem);
  out->stage_ms[2] = evo;
  out->stage_ms[3] = g > 0 ? evo / (double)g : 0.0;
  out->stage_ms[4] = std::chrono::duration<double, std::milli>(t_host1 - t_host0).count();
  out->stage_ms[5] = gsm_ms;
  int64_t gsm_per_gen = 0;
  for (auto& p : sh) gsm_per_gen += p->pitch > 0 ? 1 : 0;
  out->stage_ms[6] = timed ? (double)(g * gsm_per_gen) : 0.0;
  out->stage_ms[7] = (double)(g * launches_per_gen);
  out->stage_ms[8] = elapsed_ms(ev_win0, ev_loop1);
  out->stage_ms[9] = win_gsm_ms;
  out->stage_ms[10] = timed ? (double)((g - w0) * gsm_per_gen) : 0.0;
  out->stage_ms[11] = (double)((g - w0) * launches_per_gen);
  for (int q = 0; q < 4; ++q) out->stage_ms[12 + q] = init_phase_ms[q];
  out->stage_ms[16] = elapsed_ms(ev_compile0, ev_compile1);
  out->stage_ms[17] = alloc_ms;
  double ins_pop = 0, ins_pool = 0;
  for (int64_t i = 0; i < ng; ++i) (i < m ? ins_pop : ins_pool) += hlen[i];
  out->stage_ms[18] = ins_pop;    // instructions (not ms): population programs
  out->stage_ms[19] = ins_pool;   // instructions: random-tree programs
  out->interp_div[0] = out->interp_div[1] = 0;
  for (int q = 0; q < 6; ++q) out->interp_ops[q] = 0;
  for (int64_t i = 0; i < ng; ++i) {
    const int side = i < m ? 0 : 1;
    out->interp_div[side] += hdiv[4 * i];
    for (int q = 0; q < 3; ++q) out->interp_ops[3 * side + q] += hdiv[4 * i + 1 + q];
  }
}

// ------------------------------------------------ single-process multi-GPU
// gsgp_init(n_dev, dev_ids): one gsgp_run drives every listed
// device from this process — one host thread per device, each running the
// rank-sliced engine above as rank i of n with its own stream, and the
// per-generation collectives over an NCCL communicator created with
// ncclCommInitAll (the reference's run_evolution likewise uses every worker
// of the host: gsgp/evolution.py:115, gsgp/backend.py:94-130).  A device list
// that names a GPU twice (or GSGP_THREAD_EXCHANGE=1) runs the same threads
// with the host thread exchange instead of NCCL, so the driver is testable on
// one GPU.  Results equal the one-device run bit for bit (canonical SSE).
struct DeviceSet {
  std::vector<int> devs;
  std::vector<ncclComm_t> comms;   // empty: thread exchange (or a single device)
  bool thread_xchg = false;
};
std::mutex g_devset_mu;
DeviceSet& device_set() {
  static DeviceSet d;
  return d;
}

void devices_release(DeviceSet& d) {
  for (auto c : d.comms)
    if (c) nccl().commDestroy(c);
  d.comms.clear();
  d.devs.clear();
  d.thread_xchg = false;
}

void devices_init(int n, const int* ids) {
  GSGP_REQUIRE(n >= 1 && n <= kMaxDevices && ids, "gsgp_init needs 1..64 device ids");
  GSGP_REQUIRE(comm_state().world == 1 && !comm_state().comm && !comm_state().host,
               "gsgp_init cannot be combined with a multi-process communicator (gsgp_comm_init*)");
  int count = 0;
  GSGP_CUDA(cudaGetDeviceCount(&count));
  std::vector<int> devs(ids, ids + n);
  bool dup = false;
  for (int i = 0; i < n; ++i) {
    GSGP_REQUIRE(devs[i] >= 0 && devs[i] < count,
                 "device id " + std::to_string(devs[i]) + " out of range (" + std::to_string(count) + " devices)");
    for (int j = 0; j < i; ++j) dup |= devs[j] == devs[i];
  }
  std::lock_guard<std::mutex> lk(g_devset_mu);
  DeviceSet& d = device_set();
  devices_release(d);
  d.devs = devs;
  const char* tx = getenv("GSGP_THREAD_EXCHANGE");
  d.thread_xchg = n > 1 && (dup || (tx && tx[0] == '1'));
  if ((n > 1 && !d.thread_xchg) || (n == 1 && force_collectives())) {
    nccl().load();
    d.comms.assign(n, nullptr);
    nccl().check(nccl().commInitAll(d.comms.data(), n, d.devs.data()), "ncclCommInitAll");
  }
  GSGP_CUDA(cudaSetDevice(devs[0]));
}

void devices_finalize() {
  std::lock_guard<std::mutex> lk(g_devset_mu);
  devices_release(device_set());
}

int devices_count() { return (int)device_set().devs.size(); }

void run_job(const gsgp_config* cfg, const double* Xtr, const double* ytr, int64_t ntr, const double* Xte,
             const double* yte, int64_t nte, int32_t l, gsgp_outputs* out) {
  std::unique_lock<std::mutex> lk(g_devset_mu);
  DeviceSet& d = device_set();
  const int n = (int)d.devs.size();
  if (n <= 1 && d.comms.empty()) {              // one device: this thread runs the engine
    if (n == 1) GSGP_CUDA(cudaSetDevice(d.devs[0]));
    lk.unlock();
    run_engine(cfg, Xtr, ytr, ntr, Xte, yte, nte, l, out);
    return;
  }
  GSGP_REQUIRE(cfg && out, "null config/outputs");
  const int64_t g = cfg->generations < 0 ? 0 : cfg->generations;
  // rank 0 writes the caller's outputs; the other ranks compute the same
  // traces and lineage into scratch (checked equal below) and their case
  // slice of the elite train semantics into the caller's buffer
  struct Scratch {
    std::vector<double> tr, te, fit;
    std::vector<int8_t> src;
    std::vector<int64_t> idx, slot;
  };
  std::vector<gsgp_outputs> outs(n, *out);
  std::vector<Scratch> scr(n);
  for (int i = 1; i < n; ++i) {
    Scratch& q = scr[i];
    q.tr.resize(g + 1); q.te.resize(g + 1); q.fit.resize(g + 1);
    q.src.resize(g + 1); q.idx.resize(g + 1); q.slot.resize(g + 1);
    gsgp_outputs& o = outs[i];
    o.train_trace = q.tr.data(); o.test_trace = q.te.data(); o.elite_fit = q.fit.data();
    o.elite_src = q.src.data(); o.elite_idx = q.idx.data(); o.elite_slot = q.slot.data();
    o.plan_u = o.plan_v = nullptr;
    o.plan_ms = nullptr;
    o.gsm_ms = nullptr;
  }
  ThreadXchg tx;
  tx.n = n;
  tx.bufs.assign(n, nullptr);
  std::vector<Error> errs(n, Error{0, ""});
  const std::vector<ncclComm_t> comms = d.comms;
  std::mutex abort_mu;
  bool aborted = false;
  auto abort_all = [&] {       // a failed rank must not leave the others blocked in a collective
    std::lock_guard<std::mutex> g(abort_mu);
    if (aborted) return;
    aborted = true;
    tx.abort();
    for (auto c : comms)
      if (c) nccl().commAbort(c);
  };
  std::vector<std::thread> th;
  for (int i = 0; i < n; ++i)
    th.emplace_back([&, i] {
      CommState cs;
      cs.world = n;
      cs.rank = i;
      cs.owns_comm = false;
      if (comms.empty()) cs.tx = &tx;
      else cs.comm = comms[i];
      t_comm = &cs;
      try {
        GSGP_CUDA(cudaSetDevice(d.devs[i]));
        run_engine(cfg, Xtr, ytr, ntr, Xte, yte, nte, l, &outs[i]);
      } catch (const Error& e) {
        errs[i] = e;
        abort_all();
      } catch (const std::exception& e) {
        errs[i] = Error{ERR_CUDA, e.what()};
        abort_all();
      }
      t_comm = nullptr;
    });
  for (auto& t : th) t.join();
  if (aborted) {                           // the communicators are gone: gsgp_init again
    d.comms.clear();
    d.devs.clear();
  }
  for (int i = 0; i < n; ++i)              // the first failure that is not the abort echo
    if (errs[i].code && errs[i].msg.find("another device thread") == std::string::npos)
      throw Error{errs[i].code, "device " + std::to_string(i) + ": " + errs[i].msg};
  for (int i = 0; i < n; ++i)
    if (errs[i].code) throw Error{errs[i].code, "device " + std::to_string(i) + ": " + errs[i].msg};
  // every rank took the same decisions from the same exchanged sums
  for (int i = 1; i < n; ++i)
    for (int64_t t = 0; t <= g; ++t)
      if (outs[i].elite_slot[t] != out->elite_slot[t] || outs[i].elite_idx[t] != out->elite_idx[t] ||
          std::memcmp(&outs[i].train_trace[t], &out->train_trace[t], 8) != 0)
        throw Error{ERR_CUDA, "device ranks diverged at generation " + std::to_string(t)};
  *out = outs[0];
  out->shard_train_lo = outs[0].shard_train_lo;
  out->shard_train_hi = outs[n - 1].shard_train_hi;
  // device time of the job = the slowest rank; launches = all ranks' kernels
  for (int q : {1, 2, 4, 8, 12, 13, 14, 15})
    for (int i = 1; i < n; ++i) out->stage_ms[q] = std::max(out->stage_ms[q], outs[i].stage_ms[q]);
  out->stage_ms[3] = g > 0 ? out->stage_ms[2] / (double)g : 0.0;
  for (int q : {6, 7, 10, 11})
    for (int i = 1; i < n; ++i) out->stage_ms[q] += outs[i].stage_ms[q];
}


}  // namespace gsgp
