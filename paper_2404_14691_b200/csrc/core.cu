// core.cu — lifecycle, errors, clock, events, the stream ("context") pool,
// pinned host buffers and the CPU_LOAD memcpy fan-out of libsagedp.
//
// Reference seams replaced (paths under /root/reference/pkg/src/gslsim/):
//   Simulation.__init__ device state      simulation.py:99-159
//   Token.subscribe / set_ready          functions.py:281-301  -> events
//   GPU_CTX node (285.1 ms modelled)     functions.py:258-264  -> sage_ctx_*
#include "common.h"

#include <time.h>

#include <cstdio>
#include <mutex>

namespace sage {

State st;
Driver drv;

// ------------------------------------------------------------------ errors --
static thread_local std::string tl_err;
void set_error(const std::string &m) { tl_err = m; }
int fail(int code, const std::string &m) { tl_err = m; return code; }
int cuda_fail(cudaError_t e, const char *what) {
  tl_err = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return SAGE_ECUDA;
}
int cu_fail(CUresult r, const char *what) {
  char buf[64];
  snprintf(buf, sizeof buf, "CUresult %d", (int)r);
  tl_err = std::string(what) + ": " + buf;
  return r == CUDA_ERROR_OUT_OF_MEMORY ? SAGE_ENOMEM : SAGE_ECUDA;
}

// ------------------------------------------------------------------ clock ---
static int64_t g_epoch_ns = 0;
static int64_t mono_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (int64_t)ts.tv_sec * 1000000000ll + ts.tv_nsec;
}
int64_t host_now_us() { return (mono_ns() - g_epoch_ns) / 1000; }
int64_t host_epoch_us() { return g_epoch_ns / 1000; }
int64_t mono_us() { return mono_ns() / 1000; }

// ------------------------------------------------------- driver entry pts ---
template <class F>
static int get_entry(const char *name, F *fp, unsigned ver) {
  cudaDriverEntryPointQueryResult q;
  void *p = nullptr;
  cudaError_t e = cudaGetDriverEntryPointByVersion(name, &p, ver, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !p)
    return fail(SAGE_ECUDA, std::string("driver entry point unavailable: ") + name);
  *fp = reinterpret_cast<F>(p);
  return SAGE_OK;
}
int load_driver() {
  if (drv.MemCreate) return SAGE_OK;
  SAGE_TRY(get_entry("cuMemCreate", &drv.MemCreate, 10020));
  SAGE_TRY(get_entry("cuMemRelease", &drv.MemRelease, 10020));
  SAGE_TRY(get_entry("cuMemAddressReserve", &drv.MemAddressReserve, 10020));
  SAGE_TRY(get_entry("cuMemAddressFree", &drv.MemAddressFree, 10020));
  SAGE_TRY(get_entry("cuMemMap", &drv.MemMap, 10020));
  SAGE_TRY(get_entry("cuMemUnmap", &drv.MemUnmap, 10020));
  SAGE_TRY(get_entry("cuMemSetAccess", &drv.MemSetAccess, 10020));
  SAGE_TRY(get_entry("cuMemGetAllocationGranularity", &drv.MemGetAllocationGranularity, 10020));
  SAGE_TRY(get_entry("cuCtxCreate", &drv.CtxCreate, 3020));
  SAGE_TRY(get_entry("cuCtxDestroy", &drv.CtxDestroy, 4000));
  SAGE_TRY(get_entry("cuCtxSetCurrent", &drv.CtxSetCurrent, 4000));
  SAGE_TRY(get_entry("cuCtxGetCurrent", &drv.CtxGetCurrent, 4000));
  SAGE_TRY(get_entry("cuDevicePrimaryCtxRetain", &drv.DevicePrimaryCtxRetain, 7000));
  SAGE_TRY(get_entry("cuMemExportToShareableHandle", &drv.MemExportToShareableHandle, 10020));
  SAGE_TRY(get_entry("cuMemImportFromShareableHandle", &drv.MemImportFromShareableHandle, 10020));
  return SAGE_OK;
}

int require_up() {
  if (!st.up) return fail(SAGE_ESTATE, "sage_init has not been called");
  return SAGE_OK;
}
Gpu *gpu_get(int g) {
  if (!st.up || g < 0 || g >= st.n_gpus) return nullptr;
  return st.gpus[g].get();
}

// ------------------------------------------------------------ handle table --
// One table per kind; ids are never reused within a process so a stale handle
// is always detected (reference: MemoryLedger.free raises on double/unknown
// free, resources.py:324-326).
struct Table {
  std::mutex mu;
  std::unordered_map<uint64_t, Event *> events;
  std::atomic<uint64_t> next{1};
};
static Table g_ev;
static std::mutex g_evpool_mu;
static std::vector<std::vector<cudaEvent_t>> g_evpool;  // per gpu recycled events

int event_new(int gpu, sage_handle *h, Event **out) {
  Gpu *G = gpu_get(gpu);
  if (!G) return fail(SAGE_ENODEV, "event_new: bad gpu");
  auto *e = new Event();
  e->gpu = gpu;
  {
    std::lock_guard<std::mutex> lk(g_evpool_mu);
    auto &pool = g_evpool[gpu];
    if (!pool.empty()) { e->ev = pool.back(); pool.pop_back(); }
  }
  if (!e->ev) {
    cudaSetDevice(dev_of(gpu));
    cudaError_t err = cudaEventCreate(&e->ev);   // timing enabled: stage times
    if (err != cudaSuccess) { delete e; return cuda_fail(err, "cudaEventCreate"); }
  }
  uint64_t id = g_ev.next++;
  {
    std::lock_guard<std::mutex> lk(g_ev.mu);
    g_ev.events[id] = e;
  }
  *h = make_handle(Kind::Event, id);
  if (out) *out = e;
  return SAGE_OK;
}
int event_new_host(sage_handle *h, Event **out) {
  auto *e = new Event();
  uint64_t id = g_ev.next++;
  {
    std::lock_guard<std::mutex> lk(g_ev.mu);
    g_ev.events[id] = e;
  }
  *h = make_handle(Kind::Event, id);
  if (out) *out = e;
  return SAGE_OK;
}
Event *event_get(sage_handle h) {
  if (handle_kind(h) != Kind::Event) return nullptr;
  std::lock_guard<std::mutex> lk(g_ev.mu);
  auto it = g_ev.events.find(h & ((1ull << 56) - 1));
  return it == g_ev.events.end() ? nullptr : it->second;
}
int event_alias(sage_handle src, sage_handle *out) {
  Event *e = event_get(src);
  if (!e || !out) return fail(SAGE_ESTATE, "event_alias: unknown event");
  e->refs.fetch_add(1);
  uint64_t id = g_ev.next++;
  {
    std::lock_guard<std::mutex> lk(g_ev.mu);
    g_ev.events[id] = e;
  }
  *out = make_handle(Kind::Event, id);
  return SAGE_OK;
}
int event_record(Event *e, cudaStream_t s) {
  SAGE_CUDA(cudaEventRecord(e->ev, s));
  e->done.store(false, std::memory_order_relaxed);
  e->t_cache = INT64_MIN;
  e->recorded.store(true, std::memory_order_release);
  return SAGE_OK;
}

int event_await_recorded(Event *e) {
  if (e->recorded.load(std::memory_order_acquire)) return SAGE_OK;
  if (!e->pending.load(std::memory_order_acquire)) return fail(SAGE_ESTATE, "event was never recorded");
  while (!e->recorded.load(std::memory_order_acquire)) std::this_thread::sleep_for(std::chrono::microseconds(10));
  return SAGE_OK;
}

int event_query(Event *e) {
  if (!e->ev) return e->host_done.load(std::memory_order_acquire) ? SAGE_OK : SAGE_ENOTREADY;
  if (e->done.load(std::memory_order_acquire)) return SAGE_OK;
  if (!e->recorded.load(std::memory_order_acquire))
    return e->pending.load(std::memory_order_acquire) ? SAGE_ENOTREADY : fail(SAGE_ESTATE, "event was never recorded");
  cudaError_t r = cudaEventQuery(e->ev);
  if (r == cudaSuccess) {
    e->done.store(true, std::memory_order_release);
    return SAGE_OK;
  }
  if (r == cudaErrorNotReady) return SAGE_ENOTREADY;
  return cuda_fail(r, "cudaEventQuery");
}

int event_time_us(Event *e, int64_t *t) {
  if (!e->ev) {
    if (!e->host_done.load()) return fail(SAGE_ENOTREADY, "host job not complete");
    *t = e->host_time;
    return SAGE_OK;
  }
  Gpu *G = gpu_get(e->gpu);
  if (!G) return fail(SAGE_ENODEV, "event gpu");
  std::lock_guard<std::mutex> lk(G->anchor_mu);
  if (e->t_cache != INT64_MIN) { *t = e->t_cache; return SAGE_OK; }
  clock_anchor_refresh(G);
  float ms = 0.f;
  SAGE_CUDA(cudaEventElapsedTime(&ms, G->anchor, e->ev));
  *t = e->t_cache = G->anchor_us + (int64_t)llround((double)ms * 1000.0);
  e->done.store(true, std::memory_order_release);
  return SAGE_OK;
}

// Device event times are mapped onto the host clock through an anchor event
// whose host time is the midpoint of record..sync.  That is only accurate if
// the record executes at once: streams alias onto a few hardware queues, so
// an anchor recorded while kernels are queued can complete milliseconds late.
// Re-anchor (every 2 s, keeping float32 elapsed times sub-µs) on a dedicated
// top-priority stream, and accept only a tight round trip; otherwise keep the
// previous anchor (its float32 error grows by ~6e-8 x elapsed only).
void clock_anchor_refresh(Gpu *G, bool force) {
  if (!force && host_now_us() - G->anchor_us <= 2000000) return;
  cudaSetDevice(G->dev);
  cudaEvent_t trial = G->anchor_trial;
  for (int attempt = 0; attempt < 8; ++attempt) {
    int64_t h0 = host_now_us();
    if (cudaEventRecord(trial, G->clock) != cudaSuccess) return;
    if (cudaEventSynchronize(trial) != cudaSuccess) return;
    int64_t h1 = host_now_us();
    if (h1 - h0 <= 60 || (force && attempt == 7)) {
      std::swap(G->anchor, G->anchor_trial);
      G->anchor_us = (h0 + h1) / 2;
      return;
    }
  }
}

// ------------------------------------------------------- memcpy fan-out -----
// CPU_LOAD moves the packed DB record into pinned staging.  One host thread
// is ~3-10 GB/s, far below PCIe Gen5 (~55 GB/s), so every staging memcpy is
// split across a small pool of workers.
namespace {
struct MemcpyPool {
  std::mutex mu;
  std::condition_variable cv, done_cv;
  std::vector<std::thread> th;
  bool stop = false;
  // current job
  uint8_t *dst = nullptr;
  const uint8_t *src = nullptr;
  size_t bytes = 0, piece = 0;
  size_t n_pieces = 0;
  std::atomic<size_t> next{0};
  std::atomic<size_t> finished{0};
  uint64_t gen = 0;
  std::mutex job_mu;  // one job at a time
};
// never destroyed: workers parked on its condition variables at process exit
// (no sage_shutdown) would otherwise block the static destructor / terminate
MemcpyPool &mp = *new MemcpyPool;

void memcpy_worker() {
  pthread_setname_np(pthread_self(), "sage-memcpy");
  uint64_t seen = 0;
  for (;;) {
    {
      std::unique_lock<std::mutex> lk(mp.mu);
      mp.cv.wait(lk, [&] { return mp.stop || mp.gen != seen; });
      if (mp.stop) return;
      seen = mp.gen;
    }
    for (;;) {
      size_t i = mp.next.fetch_add(1);
      if (i >= mp.n_pieces) break;
      size_t off = i * mp.piece;
      size_t len = std::min(mp.piece, mp.bytes - off);
      memcpy(mp.dst + off, mp.src + off, len);
      if (mp.finished.fetch_add(1) + 1 == mp.n_pieces) {
        std::lock_guard<std::mutex> lk(mp.mu);
        mp.done_cv.notify_all();
      }
    }
  }
}
}  // namespace

void pool_threads_start(int n) {
  std::lock_guard<std::mutex> lk(mp.mu);
  if (!mp.th.empty()) return;
  mp.stop = false;
  for (int i = 0; i < n - 1; ++i) mp.th.emplace_back(memcpy_worker);
}
void pool_threads_stop() {
  {
    std::lock_guard<std::mutex> lk(mp.mu);
    mp.stop = true;
    mp.cv.notify_all();
  }
  for (auto &t : mp.th) t.join();
  mp.th.clear();
}

void parallel_memcpy(void *dst, const void *src, size_t bytes) {
  const size_t kPiece = 1 << 20;
  if (bytes <= kPiece || mp.th.empty()) { memcpy(dst, src, bytes); return; }
  std::lock_guard<std::mutex> job(mp.job_mu);
  {
    std::lock_guard<std::mutex> lk(mp.mu);
    mp.dst = (uint8_t *)dst;
    mp.src = (const uint8_t *)src;
    mp.bytes = bytes;
    mp.piece = kPiece;
    mp.n_pieces = (bytes + kPiece - 1) / kPiece;
    mp.next = 0;
    mp.finished = 0;
    mp.gen++;
    mp.cv.notify_all();
  }
  // the calling (CUDA host-function) thread works too
  for (;;) {
    size_t i = mp.next.fetch_add(1);
    if (i >= mp.n_pieces) break;
    size_t off = i * mp.piece;
    memcpy(mp.dst + off, mp.src + off, std::min(mp.piece, mp.bytes - off));
    mp.finished.fetch_add(1);
  }
  std::unique_lock<std::mutex> lk(mp.mu);
  mp.done_cv.wait(lk, [&] { return mp.finished.load() >= mp.n_pieces; });
}

// --------------------------------------------------------- host buffers -----
namespace {
struct HostBuf { void *p; uint64_t bytes; };
std::mutex g_host_mu;
std::unordered_map<uint64_t, HostBuf> g_host;
std::atomic<uint64_t> g_host_next{1};
}  // namespace

// -------------------------------------------------------------- slot table --
namespace {
struct SlotRef { int gpu; int idx; };
std::mutex g_slot_mu;
std::unordered_map<uint64_t, SlotRef> g_slots;
std::atomic<uint64_t> g_slot_next{1};
}  // namespace

static int slot_lookup(sage_handle h, Gpu **G, cudaStream_t *s) {
  if (handle_kind(h) != Kind::Slot) return fail(SAGE_EINVAL, "not a slot handle");
  std::lock_guard<std::mutex> lk(g_slot_mu);
  auto it = g_slots.find(h & ((1ull << 56) - 1));
  if (it == g_slots.end()) return fail(SAGE_ESTATE, "unknown or released slot");
  *G = gpu_get(it->second.gpu);
  *s = (*G)->slots[it->second.idx];
  return SAGE_OK;
}

int slot_stream(sage_handle h, Gpu **G, cudaStream_t *s) { return slot_lookup(h, G, s); }

// ------------------------------------------------------ live kernel timing --
static std::atomic<bool> g_stats{false};
bool stats_on() { return g_stats.load(std::memory_order_relaxed); }

static cudaEvent_t stat_event(Gpu *G) {
  cudaEvent_t e = nullptr;
  {
    std::lock_guard<std::mutex> lk(G->stat_mu);
    if (!G->stat_free.empty()) { e = G->stat_free.back(); G->stat_free.pop_back(); }
  }
  if (!e) cudaEventCreate(&e);
  return e;
}
cudaEvent_t stat_begin(Gpu *G, cudaStream_t s) {
  if (!stats_on()) return nullptr;
  cudaEvent_t b = stat_event(G);
  cudaEventRecord(b, s);
  return b;
}
void stat_end(Gpu *G, cudaStream_t s, int kind, cudaEvent_t b, uint64_t bytes) {
  if (!b) return;
  cudaEvent_t e = stat_event(G);
  cudaEventRecord(e, s);
  std::lock_guard<std::mutex> lk(G->stat_mu);
  G->stat_pending.push_back(Gpu::StatRec{kind, b, e, bytes});
}
static void stats_resolve(Gpu *G) {
  std::lock_guard<std::mutex> lk(G->stat_mu);
  for (auto &r : G->stat_pending) {
    cudaEventSynchronize(r.e);
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, r.b, r.e) == cudaSuccess) {
      G->stat_us[r.kind] += ms * 1000.0;
      G->stat_count[r.kind] += 1;
      G->stat_bytes[r.kind] += r.bytes;
    }
    G->stat_free.push_back(r.b);
    G->stat_free.push_back(r.e);
  }
  G->stat_pending.clear();
}
void stats_clear_gpu(Gpu *G) {
  stats_resolve(G);
  std::lock_guard<std::mutex> lk(G->stat_mu);
  for (int k = 0; k < 8; ++k) { G->stat_count[k] = 0; G->stat_us[k] = 0; G->stat_bytes[k] = 0; }
  for (auto e : G->stat_free) cudaEventDestroy(e);
  G->stat_free.clear();
}

int return_enqueue(Gpu *G, cudaStream_t s, sage_handle prev, uint64_t src, void *dst, uint64_t bytes,
                   bool host_dst, sage_handle *begin_ev, sage_handle *end_ev, sage_handle pre_end) {
  if (bytes && (!dst || !src)) return fail(SAGE_EINVAL, "return: null buffer");
  Event *b, *e;
  std::unique_lock<std::mutex> lk(G->ret_mu, std::defer_lock);
  if (bytes && host_dst && !G->rets.empty()) {
    // the copy leaves the slot stream for a return stream (so it never waits
    // behind, nor holds up, work aliased onto the slot's hardware queue)
    lk.lock();
    SAGE_CUDA(cudaEventRecord(G->ev_ret, s));
    s = G->rets[G->ret_seq++ % G->rets.size()];
    SAGE_CUDA(cudaStreamWaitEvent(s, G->ev_ret, 0));
    prev = 0;
  }
  if (prev) {
    SAGE_TRY(event_alias(prev, begin_ev));    // RETURN begins where COMPUTE ended
  } else {
    SAGE_TRY(event_new(G->id, begin_ev, &b));
    SAGE_TRY(event_record(b, s));
  }
  // UVA: the destination is pinned host memory (D2H) or an HBM buffer (D2D)
  if (bytes) SAGE_CUDA(cudaMemcpyAsync(dst, (const void *)src, bytes, cudaMemcpyDefault, s));
  if (pre_end) {
    e = event_get(pre_end);
    if (!e) return fail(SAGE_ESTATE, "return: unknown pre-created end event");
    SAGE_TRY(event_alias(pre_end, end_ev));
  } else {
    SAGE_TRY(event_new(G->id, end_ev, &e));
  }
  return event_record(e, s);
}

}  // namespace sage

using namespace sage;

// ============================================================== C-ABI =======
extern "C" {

const char *sage_last_error(void) { return tl_err.c_str(); }
int sage_abi_version(void) { return SAGE_ABI_VERSION; }
int64_t sage_now_us(void) { return host_now_us(); }
int64_t sage_clock_epoch_ns(void) { return g_epoch_ns; }

// the physical CUDA device logical GPU g runs on (SAGE_DEVICE_OFFSET and
// SAGE_INIT_SHARE_DEVICE applied): what a framework running a body on the
// invocation's stream (ResNet-50 via PyTorch) must select
int sage_gpu_device(int gpu, int *dev) {
  SAGE_TRY(require_up());
  Gpu *G = gpu_get(gpu);
  if (!G || !dev) return fail(SAGE_ENODEV, "gpu_device: bad logical gpu");
  *dev = G->dev;
  return SAGE_OK;
}
int sage_device_count(int *n) {
  if (!n) return fail(SAGE_EINVAL, "null n");
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) { *n = 0; return fail(SAGE_ENODEV, std::string("no CUDA device: ") + cudaGetErrorString(e)); }
  *n = c;
  return SAGE_OK;
}

int sage_set_host_threads(int n) {
  if (n < 1 || n > 256) return fail(SAGE_EINVAL, "host threads must be in [1, 256]");
  st.host_threads = n;
  if (st.up) { pool_threads_stop(); pool_threads_start(n); }
  return SAGE_OK;
}

int sage_init(int n_gpus, uint64_t pool_bytes_per_gpu, uint64_t staging_bytes, uint64_t chunk_bytes,
              uint32_t flags) {
  if (st.up) return fail(SAGE_ESTATE, "sage_init called twice (sage_shutdown first)");
  if (chunk_bytes == 0) chunk_bytes = 8ull << 20;
  if (chunk_bytes % 256 || chunk_bytes < (64u << 10))
    return fail(SAGE_EINVAL, "chunk_bytes must be a multiple of 256 and >= 64 KiB");
  if (staging_bytes == 0) staging_bytes = 8 * chunk_bytes;
  if (staging_bytes < 2 * chunk_bytes) return fail(SAGE_EINVAL, "staging must hold >= 2 chunks");
  int avail = 0;
  cudaError_t e = cudaGetDeviceCount(&avail);
  if (e != cudaSuccess || avail == 0) return fail(SAGE_ENODEV, "no CUDA device visible");
  if (n_gpus <= 0) n_gpus = avail;
  if (n_gpus > avail && !(flags & SAGE_INIT_SHARE_DEVICE))
    return fail(SAGE_ENODEV, "requested more GPUs than visible");
  st.n_devices = avail;
  SAGE_TRY(load_driver());
  g_epoch_ns = mono_ns();
  st.chunk = chunk_bytes;
  st.flags = flags;
  st.n_gpus = n_gpus;
  st.gpus.clear();
  {
    std::lock_guard<std::mutex> lk(g_evpool_mu);
    g_evpool.assign(n_gpus, {});
  }
  st.up = true;  // gpu_get works during setup
  for (int g = 0; g < n_gpus; ++g) {
    st.gpus.emplace_back(new Gpu());
    int rc = gpu_setup(g, pool_bytes_per_gpu, staging_bytes, chunk_bytes);
    if (rc != SAGE_OK) {
      std::string msg = tl_err;
      sage_shutdown();
      return fail(rc, msg);
    }
  }
  if ((flags & SAGE_INIT_PEER_ACCESS) && n_gpus > 1) {
    for (int a = 0; a < n_gpus; ++a)
      for (int b = 0; b < n_gpus; ++b) {
        const int da = dev_of(a), db = dev_of(b);
        if (da == db) continue;   // logical planes sharing a device need no peer access
        int can = 0;
        cudaDeviceCanAccessPeer(&can, da, db);
        if (!can) continue;
        cudaSetDevice(da);
        cudaError_t pe = cudaDeviceEnablePeerAccess(db, 0);
        if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) {
          std::string m = std::string("peer access ") + cudaGetErrorString(pe);
          sage_shutdown();
          return fail(SAGE_ECUDA, m);
        }
        cudaGetLastError();
      }
  }
  pool_threads_start(st.host_threads);
  return SAGE_OK;
}

int sage_shutdown(void) {
  if (!st.up) return SAGE_OK;
  for (auto &G : st.gpus) {
    cudaSetDevice(G->dev);
    cudaDeviceSynchronize();
  }
  invoke_shutdown();
  pool_threads_stop();
  layouts_destroy_all();
  nets_release_graphs();
  {
    std::lock_guard<std::mutex> lk(g_host_mu);
    for (auto &kv : g_host) cudaFreeHost(kv.second.p);
    g_host.clear();
  }
  {
    std::lock_guard<std::mutex> lk(g_ev.mu);
    for (auto &kv : g_ev.events) {   // aliased events: freed with their last handle
      if (kv.second->refs.fetch_sub(1) != 1) continue;
      if (kv.second->ev) cudaEventDestroy(kv.second->ev);
      delete kv.second;
    }
    g_ev.events.clear();
  }
  {
    std::lock_guard<std::mutex> lk(g_evpool_mu);
    for (auto &p : g_evpool)
      for (auto e : p) cudaEventDestroy(e);
    g_evpool.clear();
  }
  {
    std::lock_guard<std::mutex> lk(g_slot_mu);
    g_slots.clear();
  }
  for (auto &G : st.gpus) gpu_teardown(G.get());
  st.gpus.clear();
  st.up = false;
  st.n_gpus = 0;
  return SAGE_OK;
}

// ------------------------------------------------------------- events -------
int sage_event_alias(sage_handle h, sage_handle *out) {
  if (!out) return fail(SAGE_EINVAL, "event_alias: null out");
  return event_alias(h, out);
}
int sage_event_query(sage_handle h) {
  Event *e = event_get(h);
  if (!e) return fail(SAGE_ESTATE, "unknown event handle");
  return event_query(e);
}
int sage_event_sync(sage_handle h) {
  Event *e = event_get(h);
  if (!e) return fail(SAGE_ESTATE, "unknown event handle");
  if (!e->ev) {
    while (!e->host_done.load(std::memory_order_acquire)) std::this_thread::sleep_for(std::chrono::microseconds(50));
    return SAGE_OK;
  }
  SAGE_TRY(event_await_recorded(e));
  SAGE_CUDA(cudaEventSynchronize(e->ev));
  return SAGE_OK;
}
int sage_event_time(sage_handle h, int64_t *t) {
  Event *e = event_get(h);
  if (!e || !t) return fail(SAGE_ESTATE, "unknown event handle");
  int rc = event_query(e);
  if (rc != SAGE_OK) return rc;
  return event_time_us(e, t);
}
int sage_event_release(sage_handle h) {
  Event *e = nullptr;
  if (handle_kind(h) != Kind::Event) return fail(SAGE_EINVAL, "not an event handle");
  {
    std::lock_guard<std::mutex> lk(g_ev.mu);
    auto it = g_ev.events.find(h & ((1ull << 56) - 1));
    if (it == g_ev.events.end()) return fail(SAGE_ESTATE, "double or unknown event release");
    e = it->second;
    g_ev.events.erase(it);
  }
  if (e->refs.fetch_sub(1) != 1) return SAGE_OK;   // another handle still names it
  if (e->ev && e->ipc) {
    cudaEventDestroy(e->ev);
  } else if (e->ev) {
    std::lock_guard<std::mutex> lk(g_evpool_mu);
    if (e->gpu >= 0 && e->gpu < (int)g_evpool.size()) g_evpool[e->gpu].push_back(e->ev);
    else cudaEventDestroy(e->ev);
  }
  delete e;
  return SAGE_OK;
}
int sage_event_poll(const sage_handle *evs, int n, uint8_t *done, int64_t timeout_us) {
  if (n < 0 || (n > 0 && (!evs || !done))) return fail(SAGE_EINVAL, "bad poll arguments");
  std::vector<Event *> es(n);
  for (int i = 0; i < n; ++i) {
    es[i] = event_get(evs[i]);
    if (!es[i]) return fail(SAGE_ESTATE, "unknown event handle in poll");
  }
  int64_t deadline = host_now_us() + (timeout_us > 0 ? timeout_us : 0);
  for (;;) {
    int cnt = 0;
    for (int i = 0; i < n; ++i) {
      int rc = event_query(es[i]);
      if (rc == SAGE_OK) { done[i] = 1; ++cnt; }
      else if (rc == SAGE_ENOTREADY) done[i] = 0;
      else return rc;
    }
    if (cnt > 0 || n == 0 || host_now_us() >= deadline) return cnt;
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

// ------------------------------------------------------------- slots --------
int sage_ctx_acquire(int gpu, sage_handle *slot) {
  SAGE_TRY(require_up());
  Gpu *G = gpu_get(gpu);
  if (!G || !slot) return fail(SAGE_ENODEV, "ctx_acquire: bad gpu");
  int idx = -1;
  {
    std::lock_guard<std::mutex> lk(G->slot_mu);
    if (!G->slot_free.empty()) { idx = G->slot_free.back(); G->slot_free.pop_back(); }
    else {
      // pool exhausted: grow it (never blocks an admission)
      cudaSetDevice(dev_of(gpu));
      cudaStream_t s;
      SAGE_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      G->slots.push_back(s);
      idx = (int)G->slots.size() - 1;
    }
  }
  uint64_t id = g_slot_next++;
  {
    std::lock_guard<std::mutex> lk(g_slot_mu);
    g_slots[id] = SlotRef{gpu, idx};
  }
  *slot = make_handle(Kind::Slot, id);
  return SAGE_OK;
}

int sage_ctx_release(sage_handle slot) {
  if (handle_kind(slot) != Kind::Slot) return fail(SAGE_EINVAL, "not a slot handle");
  SlotRef r;
  {
    std::lock_guard<std::mutex> lk(g_slot_mu);
    auto it = g_slots.find(slot & ((1ull << 56) - 1));
    if (it == g_slots.end()) return fail(SAGE_ESTATE, "double or unknown slot release");
    r = it->second;
    g_slots.erase(it);
  }
  Gpu *G = gpu_get(r.gpu);
  std::lock_guard<std::mutex> lk(G->slot_mu);
  G->slot_free.push_back(r.idx);
  return SAGE_OK;
}

}  // extern "C"

int sage::wait_events(cudaStream_t s, const sage_handle *w, int n) {
  for (int i = 0; i < n; ++i) {
    Event *e = event_get(w[i]);
    if (!e) return fail(SAGE_ESTATE, "unknown wait event");
    if (!e->ev) {  // host job: block the enqueue until it is done (rare)
      while (!e->host_done.load()) std::this_thread::sleep_for(std::chrono::microseconds(20));
      continue;
    }
    SAGE_TRY(event_await_recorded(e));
    SAGE_CUDA(cudaStreamWaitEvent(s, e->ev, 0));
  }
  return SAGE_OK;
}

extern "C" {

int sage_stream_wait(sage_handle slot, const sage_handle *evs, int n) {
  Gpu *G; cudaStream_t s;
  SAGE_TRY(slot_lookup(slot, &G, &s));
  cudaSetDevice(G->dev);
  return wait_events(s, evs, n);
}

int sage_sync_wait(sage_handle slot, const sage_handle *evs, int n, sage_handle *begin_ev, sage_handle *end_ev) {
  Gpu *G; cudaStream_t s;
  SAGE_TRY(slot_lookup(slot, &G, &s));
  if (!begin_ev || !end_ev) return fail(SAGE_EINVAL, "sync_wait: null out");
  cudaSetDevice(G->dev);
  Event *b, *e;
  SAGE_TRY(event_new(G->id, begin_ev, &b));
  SAGE_TRY(event_record(b, s));
  SAGE_TRY(wait_events(s, evs, n));
  SAGE_TRY(event_new(G->id, end_ev, &e));
  return event_record(e, s);
}

int sage_return_after(sage_handle slot, const sage_handle *wait, int n_wait, uint64_t src, void *dst,
                      uint64_t bytes, sage_handle *begin_ev, sage_handle *end_ev) {
  Gpu *G; cudaStream_t s;
  SAGE_TRY(slot_lookup(slot, &G, &s));
  cudaSetDevice(G->dev);
  SAGE_TRY(wait_events(s, wait, n_wait));
  return sage_return(slot, src, dst, bytes, begin_ev, end_ev);
}

int sage_slot_stream(sage_handle slot, uint64_t *stream) {
  Gpu *G; cudaStream_t s;
  SAGE_TRY(slot_lookup(slot, &G, &s));
  if (!stream) return fail(SAGE_EINVAL, "slot_stream: null out");
  *stream = reinterpret_cast<uint64_t>(s);
  return SAGE_OK;
}

int sage_slot_record(sage_handle slot, sage_handle *ev) {
  Gpu *G; cudaStream_t s;
  SAGE_TRY(slot_lookup(slot, &G, &s));
  cudaSetDevice(G->dev);
  Event *e;
  SAGE_TRY(event_new(G->id, ev, &e));
  return event_record(e, s);
}

int sage_ctx_bind(sage_handle slot, uint64_t ctx_dptr, uint64_t ctx_bytes, const sage_handle *wait,
                  int n_wait, sage_handle *begin_ev, sage_handle *end_ev) {
  Gpu *G; cudaStream_t s;
  SAGE_TRY(slot_lookup(slot, &G, &s));
  cudaSetDevice(G->dev);
  SAGE_TRY(wait_events(s, wait, n_wait));
  Event *b, *e;
  SAGE_TRY(event_new(G->id, begin_ev, &b));
  SAGE_TRY(event_record(b, s));
  // the function context segment: zero its 64 KiB header (descriptor table,
  // scratch counters) on the slot's stream
  if (ctx_dptr && ctx_bytes) SAGE_CUDA(cudaMemsetAsync((void *)ctx_dptr, 0, std::min<uint64_t>(ctx_bytes, 64 << 10), s));
  SAGE_TRY(event_new(G->id, end_ev, &e));
  return event_record(e, s);
}

int sage_return(sage_handle slot, uint64_t src, void *host_dst, uint64_t bytes, sage_handle *begin_ev,
                sage_handle *end_ev) {
  Gpu *G; cudaStream_t s;
  SAGE_TRY(slot_lookup(slot, &G, &s));
  cudaSetDevice(G->dev);
  return return_enqueue(G, s, 0, src, host_dst, bytes, false, begin_ev, end_ev);
}

int sage_d2h_cache(int gpu, uint64_t src, void *host_dst, uint64_t bytes, const sage_handle *wait, int n_wait,
                   sage_handle *end_ev) {
  SAGE_TRY(require_up());
  Gpu *G = gpu_get(gpu);
  if (!G || !host_dst || !src) return fail(SAGE_EINVAL, "d2h_cache: bad argument");
  cudaSetDevice(dev_of(gpu));
  SAGE_TRY(wait_events(G->d2h, wait, n_wait));
  SAGE_CUDA(cudaMemcpyAsync(host_dst, (const void *)src, bytes, cudaMemcpyDeviceToHost, G->d2h));
  Event *e;
  SAGE_TRY(event_new(gpu, end_ev, &e));
  return event_record(e, G->d2h);
}

int sage_fanout(int src_gpu, uint64_t src, int dst_gpu, uint64_t dst, uint64_t bytes, const sage_handle *wait,
                int n_wait, sage_handle *end_ev) {
  SAGE_TRY(require_up());
  Gpu *D = gpu_get(dst_gpu);
  if (!D || !gpu_get(src_gpu)) return fail(SAGE_ENODEV, "fanout: bad gpu");
  cudaSetDevice(dev_of(dst_gpu));
  SAGE_TRY(wait_events(D->copy, wait, n_wait));
  SAGE_CUDA(cudaMemcpyPeerAsync((void *)dst, dev_of(dst_gpu), (const void *)src, dev_of(src_gpu), bytes, D->copy));
  Event *e;
  SAGE_TRY(event_new(dst_gpu, end_ev, &e));
  return event_record(e, D->copy);
}

int sage_stats_enable(int on) {
  g_stats.store(on != 0);
  return SAGE_OK;
}
int sage_stats_reset(void) {
  SAGE_TRY(require_up());
  for (auto &G : st.gpus) {
    cudaSetDevice(G->dev);
    stats_clear_gpu(G.get());
  }
  return SAGE_OK;
}
int sage_stats_get(int gpu, int kind, uint64_t *launches, double *total_us, uint64_t *bytes) {
  SAGE_TRY(require_up());
  Gpu *G = gpu_get(gpu);
  if (!G || kind < 0 || kind >= SAGE_KERNEL_KINDS) return fail(SAGE_EINVAL, "stats_get: bad argument");
  cudaSetDevice(dev_of(gpu));
  stats_resolve(G);
  std::lock_guard<std::mutex> lk(G->stat_mu);
  if (launches) *launches = G->stat_count[kind];
  if (total_us) *total_us = G->stat_us[kind];
  if (bytes) *bytes = G->stat_bytes[kind];
  return SAGE_OK;
}
int sage_device_sync(int gpu) {
  SAGE_TRY(require_up());
  if (!gpu_get(gpu)) return fail(SAGE_ENODEV, "device_sync: bad gpu");
  issuer_drain(gpu);
  SAGE_CUDA(cudaSetDevice(dev_of(gpu)));
  SAGE_CUDA(cudaDeviceSynchronize());
  return SAGE_OK;
}
int sage_mark(int gpu, sage_handle *ev) {
  SAGE_TRY(require_up());
  Gpu *G = gpu_get(gpu);
  if (!G || !ev) return fail(SAGE_EINVAL, "mark: bad argument");
  cudaSetDevice(dev_of(gpu));
  Event *e;
  SAGE_TRY(event_new(gpu, ev, &e));
  return event_record(e, G->aux);
}
int sage_event_elapsed(sage_handle a, sage_handle b, double *us) {
  Event *ea = event_get(a), *eb = event_get(b);
  if (!ea || !eb || !us || !ea->ev || !eb->ev) return fail(SAGE_EINVAL, "event_elapsed: bad events");
  float ms = 0.f;
  SAGE_CUDA(cudaEventElapsedTime(&ms, ea->ev, eb->ev));
  *us = ms * 1000.0;
  return SAGE_OK;
}

int sage_host_register(void *ptr, uint64_t bytes) {
  SAGE_TRY(require_up());
  if (!ptr || !bytes) return fail(SAGE_EINVAL, "host_register: bad argument");
  SAGE_CUDA(cudaHostRegister(ptr, bytes, cudaHostRegisterPortable));
  return SAGE_OK;
}
int sage_host_unregister(void *ptr) {
  if (!ptr) return fail(SAGE_EINVAL, "host_unregister: null");
  SAGE_CUDA(cudaHostUnregister(ptr));
  return SAGE_OK;
}

int sage_host_alloc(uint64_t bytes, sage_handle *h, void **ptr) {
  if (!h || !ptr || bytes == 0) return fail(SAGE_EINVAL, "host_alloc: bad argument");
  void *p = nullptr;
  cudaError_t e = cudaHostAlloc(&p, bytes, cudaHostAllocPortable);
  if (e != cudaSuccess) return cuda_fail(e, "cudaHostAlloc");
  uint64_t id = g_host_next++;
  {
    std::lock_guard<std::mutex> lk(g_host_mu);
    g_host[id] = HostBuf{p, bytes};
  }
  *h = make_handle(Kind::Host, id);
  *ptr = p;
  return SAGE_OK;
}

int sage_host_free(sage_handle h) {
  if (handle_kind(h) != Kind::Host) return fail(SAGE_EINVAL, "not a host buffer handle");
  HostBuf b;
  {
    std::lock_guard<std::mutex> lk(g_host_mu);
    auto it = g_host.find(h & ((1ull << 56) - 1));
    if (it == g_host.end()) return fail(SAGE_ESTATE, "double or unknown host free");
    b = it->second;
    g_host.erase(it);
  }
  SAGE_CUDA(cudaFreeHost(b.p));
  return SAGE_OK;
}

}  // extern "C"

// ------------------------------------------------- cross-process events -----
// A process that lands a segment other processes will read (the home rank of
// a fan-out) hands them an interprocess event recorded after the land; they
// open it and make their own streams wait on it -- a device-side dependency
// across processes, no host round trip.
extern "C" int sage_ipc_event_export(sage_handle after, sage_handle *ev, void *ipc_handle) {
  SAGE_TRY(require_up());
  Event *A = event_get(after);
  if (!A || !A->ev || !ev || !ipc_handle) return fail(SAGE_EINVAL, "ipc_event_export: bad argument");
  SAGE_TRY(event_await_recorded(A));
  Gpu *G = gpu_get(A->gpu);
  if (!G) return fail(SAGE_ENODEV, "ipc_event_export: bad gpu");
  cudaSetDevice(G->dev);
  auto *e = new Event();
  e->gpu = A->gpu;
  e->ipc = true;
  cudaError_t r = cudaEventCreateWithFlags(&e->ev, cudaEventDisableTiming | cudaEventInterprocess);
  if (r != cudaSuccess) { delete e; return cuda_fail(r, "cudaEventCreate(interprocess)"); }
  {
    std::lock_guard<std::mutex> lk(G->ipc_mu);
    if (!G->ipc) r = cudaStreamCreateWithFlags(&G->ipc, cudaStreamNonBlocking);
    if (r == cudaSuccess) r = cudaStreamWaitEvent(G->ipc, A->ev, 0);
    if (r == cudaSuccess) r = cudaEventRecord(e->ev, G->ipc);
  }
  if (r == cudaSuccess) r = cudaIpcGetEventHandle(reinterpret_cast<cudaIpcEventHandle_t *>(ipc_handle), e->ev);
  if (r != cudaSuccess) { cudaEventDestroy(e->ev); delete e; return cuda_fail(r, "ipc_event_export"); }
  e->recorded.store(true);
  uint64_t id = g_ev.next++;
  {
    std::lock_guard<std::mutex> lk(g_ev.mu);
    g_ev.events[id] = e;
  }
  *ev = make_handle(Kind::Event, id);
  return SAGE_OK;
}

extern "C" int sage_ipc_event_open(int gpu, const void *ipc_handle, sage_handle *ev) {
  SAGE_TRY(require_up());
  Gpu *G = gpu_get(gpu);
  if (!G || !ipc_handle || !ev) return fail(SAGE_EINVAL, "ipc_event_open: bad argument");
  cudaSetDevice(G->dev);
  auto *e = new Event();
  e->gpu = gpu;
  e->ipc = true;
  cudaIpcEventHandle_t h;
  memcpy(&h, ipc_handle, sizeof h);
  cudaError_t r = cudaIpcOpenEventHandle(&e->ev, h);
  if (r != cudaSuccess) { delete e; return cuda_fail(r, "cudaIpcOpenEventHandle"); }
  e->recorded.store(true);
  uint64_t id = g_ev.next++;
  {
    std::lock_guard<std::mutex> lk(g_ev.mu);
    g_ev.events[id] = e;
  }
  *ev = make_handle(Kind::Event, id);
  return SAGE_OK;
}
