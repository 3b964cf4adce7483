// pool.cu — per-GPU device state and the VMM segment pool.
//
// Replaces MemoryLedger (resources.py:271-337): a capacity-checked ledger with
// the reference's rounding rule (round_up_umb, resources.py:36-40; 1024 MB for
// FixedGSL, exact otherwise) and its Denied-with-shortfall refusal
// (resources.py:244-257, 309-315).  Unlike the model, every non-account-only
// allocation is real HBM: a cuMemCreate physical allocation mapped with
// cuMemMap/cuMemSetAccess into a reserved VA range.  Physical handles of freed
// segments are cached by size so steady-state churn never calls cuMemCreate.
#include "common.h"

#include <map>

namespace sage {

struct Alloc {
  int gpu = -1;
  uint64_t bytes = 0, eff = 0, phys = 0;
  int cls = 0;
  bool account_only = false;
  bool exported = false;   // pages handed to another process: never recycled through the cache
  bool carved = false;     // a piece of a pool chunk (private writable data): no handle of its own
  CUdeviceptr va = 0;
  CUmemGenericAllocationHandle ph = 0;
};

struct Pool {
  std::mutex mu;
  uint64_t capacity = 0, granularity = 0, usage = 0, by_class[4] = {0, 0, 0, 0};
  uint64_t physical = 0;   // mapped bytes
  uint64_t cached = 0;     // bytes held by the free-handle cache
  uint64_t vmm_gran = 2ull << 20;
  std::multimap<uint64_t, std::pair<CUdeviceptr, CUmemGenericAllocationHandle>> free_mapped;
  std::vector<std::pair<Alloc *, cudaEvent_t>> zombies;  // ledger-freed, pages pending an event
  // private writable segments are carved from chunks mapped once: a fresh
  // segment otherwise costs a cuMemCreate + cuMemSetAccess each (~0.2 ms,
  // ms while the device's pages are first touched), which made the first
  // burst of N concurrent invocations spend ~9 ms of host time per
  // invocation (cfg 5 at N = 512).  Pieces are cached by size when freed and
  // never unmapped; the chunks go at pool teardown.
  struct Chunk {
    CUdeviceptr va = 0;
    CUmemGenericAllocationHandle ph = 0;
    uint64_t live = 0;   // pieces handed out and not freed
    uint64_t used = 0;   // bytes carved (an abandoned tail included)
  };
  std::vector<Chunk> chunks;
  uint64_t chunk_bytes = 1ull << 30, carve_next = 0, carve_left = 0, carved = 0;
  double carve_gb = -1;   // SAGE_POOL_CARVE_GB; < 0: half the budget
  uint64_t carve_cap() const { return carve_gb >= 0 ? (uint64_t)(carve_gb * (1ull << 30)) : capacity / 2; }
  Chunk *chunk_of(CUdeviceptr va) {
    for (auto &c : chunks)
      if (va >= c.va && va < c.va + chunk_bytes) return &c;
    return nullptr;
  }
};

static void unmap_segment(Pool *P, Alloc *A);

// unmap zombies whose last reader finished (called with P->mu held)
static void reap(Pool *P, bool all) {
  auto &Z = P->zombies;
  for (size_t i = 0; i < Z.size();) {
    cudaError_t q = all ? cudaEventSynchronize(Z[i].second) : cudaEventQuery(Z[i].second);
    if (q == cudaSuccess || (q != cudaErrorNotReady)) {
      unmap_segment(P, Z[i].first);
      cudaEventDestroy(Z[i].second);
      delete Z[i].first;
      Z[i] = Z.back();
      Z.pop_back();
    } else {
      ++i;
    }
  }
}

static std::mutex g_alloc_mu;
static std::unordered_map<uint64_t, Alloc *> g_allocs;
static std::atomic<uint64_t> g_alloc_next{1};

static uint64_t round_up(uint64_t v, uint64_t g) { return g ? (v + g - 1) / g * g : v; }

int pool_create(Gpu *G, uint64_t capacity) {
  auto *P = new Pool();
  P->capacity = capacity;
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = G->dev;
  size_t gran = 0;
  SAGE_CU(drv.MemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  if (gran) P->vmm_gran = gran;
  // chunk-carved private segments: at most half the budget (env SAGE_POOL_CARVE_GB)
  const char *e = getenv("SAGE_POOL_CARVE_GB");
  if (e) P->carve_gb = atof(e);
  G->pool = P;
  return SAGE_OK;
}

static void release_chunk(Pool *P, const Pool::Chunk &c) {
  drv.MemUnmap(c.va, P->chunk_bytes);
  drv.MemAddressFree(c.va, P->chunk_bytes);
  drv.MemRelease(c.ph);
}

// unmap every cached segment, and every chunk none of whose pieces is in use
// (its cached pieces leave the cache with it); called under memory pressure
static void release_cache(Pool *P) {
  for (auto it = P->free_mapped.begin(); it != P->free_mapped.end();) {
    if (!it->second.second) { ++it; continue; }   // carved piece: goes with its chunk
    drv.MemUnmap(it->second.first, it->first);
    drv.MemAddressFree(it->second.first, it->first);
    drv.MemRelease(it->second.second);
    P->cached -= it->first;
    it = P->free_mapped.erase(it);
  }
  for (size_t k = 0; k < P->chunks.size();) {
    Pool::Chunk c = P->chunks[k];
    if (c.live) { ++k; continue; }
    for (auto it = P->free_mapped.begin(); it != P->free_mapped.end();) {
      if (it->second.first >= c.va && it->second.first < c.va + P->chunk_bytes) {
        P->cached -= it->first;
        it = P->free_mapped.erase(it);
      } else {
        ++it;
      }
    }
    P->carved -= c.used;
    if (P->carve_left && P->carve_next >= c.va && P->carve_next <= c.va + P->chunk_bytes) {   // being carved
      P->carve_left = 0;
      P->carve_next = 0;
    }
    release_chunk(P, c);
    P->chunks[k] = P->chunks.back();
    P->chunks.pop_back();
  }
}

static void release_chunks(Pool *P) {
  for (auto &c : P->chunks) release_chunk(P, c);
  P->chunks.clear();
}

// map `bytes` (granularity-rounded) of fresh pages at a fresh VA range
static int map_fresh(Gpu *G, Pool *P, uint64_t bytes, CUdeviceptr *va, CUmemGenericAllocationHandle *ph);

void pool_destroy(Gpu *G) {
  Pool *P = G->pool;
  if (!P) return;
  std::vector<uint64_t> mine;
  {
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    for (auto &kv : g_allocs)
      if (kv.second->gpu == G->id) mine.push_back(kv.first);
  }
  for (uint64_t id : mine) sage_pool_free(make_handle(Kind::Alloc, id));
  {
    std::lock_guard<std::mutex> lk(P->mu);
    reap(P, true);
  }
  release_cache(P);
  release_chunks(P);
  delete P;
  G->pool = nullptr;
}

static int map_fresh(Gpu *G, Pool *P, uint64_t bytes, CUdeviceptr *va, CUmemGenericAllocationHandle *ph) {
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = G->dev;
  // exportable as a POSIX file descriptor: function processes map shared
  // segments zero-copy (sage_pool_export / sage_segment_import)
  static const bool shareable = [] { const char *e = getenv("SAGE_POOL_SHAREABLE"); return !(e && atoi(e) == 0); }();
  if (shareable) prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUresult r = drv.MemCreate(ph, bytes, &prop, 0);
  if (r == CUDA_ERROR_OUT_OF_MEMORY && (P->cached || !P->zombies.empty())) {
    reap(P, true);
    release_cache(P);
    r = drv.MemCreate(ph, bytes, &prop, 0);
  }
  if (r != CUDA_SUCCESS) { *ph = 0; return cu_fail(r, "cuMemCreate"); }
  r = drv.MemAddressReserve(va, bytes, P->vmm_gran, 0, 0);
  if (r != CUDA_SUCCESS) { drv.MemRelease(*ph); *ph = 0; return cu_fail(r, "cuMemAddressReserve"); }
  r = drv.MemMap(*va, bytes, 0, *ph, 0);
  if (r != CUDA_SUCCESS) {
    drv.MemAddressFree(*va, bytes); drv.MemRelease(*ph); *ph = 0; *va = 0;
    return cu_fail(r, "cuMemMap");
  }
  std::vector<CUmemAccessDesc> acc;
  int ngpu = (st.flags & SAGE_INIT_PEER_ACCESS) ? st.n_gpus : 1;
  for (int d = 0; d < ngpu; ++d) {
    CUmemAccessDesc a{};
    a.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    a.location.id = (ngpu == 1) ? G->dev : dev_of(d);
    a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    acc.push_back(a);
  }
  r = drv.MemSetAccess(*va, bytes, acc.data(), acc.size());
  if (r != CUDA_SUCCESS) {
    drv.MemUnmap(*va, bytes); drv.MemAddressFree(*va, bytes); drv.MemRelease(*ph);
    *ph = 0; *va = 0;
    return cu_fail(r, "cuMemSetAccess");
  }
  return SAGE_OK;
}

static int map_segment(Gpu *G, Pool *P, Alloc *A) {
  A->phys = round_up(A->bytes, P->vmm_gran);
  // reuse a cached mapped segment of exactly this size: no driver call
  {
    // (a carved piece has no handle of its own: only private writable data reuses one)
    auto rng = P->free_mapped.equal_range(A->phys);
    auto it = rng.first;
    if (A->cls != SAGE_CLASS_WRITABLE)
      while (it != rng.second && !it->second.second) ++it;
    if (it != rng.second) {
      A->va = it->second.first;
      A->ph = it->second.second;
      A->carved = A->ph == 0;
      if (A->carved) {
        if (Pool::Chunk *c = P->chunk_of(A->va)) c->live++;
      }
      P->free_mapped.erase(it);
      P->cached -= A->phys;
      P->physical += A->phys;
      return SAGE_OK;
    }
  }
  // private writable data: a piece of a chunk (see Pool::chunks)
  if (A->cls == SAGE_CLASS_WRITABLE && A->phys <= P->chunk_bytes / 4 && P->carved + A->phys <= P->carve_cap()) {
    if (P->carve_left < A->phys) {
      // (the old chunk's uncarved tail stays unused: at most a quarter chunk)
      Pool::Chunk c;
      if (map_fresh(G, P, P->chunk_bytes, &c.va, &c.ph) == SAGE_OK) {
        if (P->carve_left) {          // the abandoned tail counts as carved
          if (Pool::Chunk *old = P->chunk_of(P->carve_next)) old->used += P->carve_left;
          P->carved += P->carve_left;
        }
        P->chunks.push_back(c);
        P->carve_next = c.va;
        P->carve_left = P->chunk_bytes;
      }
    }
    if (P->carve_left >= A->phys) {
      A->va = P->carve_next;
      A->ph = 0;
      A->carved = true;
      Pool::Chunk *ck = P->chunk_of(A->va);   // the chunk just carved from
      if (ck) { ck->live++; ck->used += A->phys; }
      P->carve_next += A->phys;
      P->carve_left -= A->phys;
      P->carved += A->phys;
      P->physical += A->phys;
      return SAGE_OK;
    }
  }
  SAGE_TRY(map_fresh(G, P, A->phys, &A->va, &A->ph));
  P->physical += A->phys;
  return SAGE_OK;
}

static void unmap_segment(Pool *P, Alloc *A) {
  if (!A->va) return;
  P->physical -= A->phys;
  // keep the segment MAPPED for reuse by the next allocation of this size
  // (per-invocation writable churn then costs no driver call) while mapped +
  // cached pages stay within the budget; otherwise unmap and release them.
  // No separate cap on the cache: with thousands of invocations in flight
  // (offered load above capacity) a 16 GiB cap made every alloc / free a
  // cuMemCreate+Map / Unmap+Release (~150-250 us of host time each), which
  // halved cfg-3 throughput; a cuMemCreate that finds the HBM held by the
  // cache releases it and retries (map_segment)
  if (A->carved) {
    if (Pool::Chunk *c = P->chunk_of(A->va)) c->live--;
  }
  if (A->carved || (!A->exported && P->cached + A->phys + P->physical <= P->capacity + (4ull << 30))) {
    P->free_mapped.emplace(A->phys, std::make_pair(A->va, A->ph));
    P->cached += A->phys;
  } else {
    drv.MemUnmap(A->va, A->phys);
    drv.MemAddressFree(A->va, A->phys);
    drv.MemRelease(A->ph);
  }
  A->va = 0;
  A->ph = 0;
}

// ------------------------------------------------------------- device state -
int gpu_setup(int id, uint64_t pool_bytes, uint64_t staging_bytes, uint64_t chunk) {
  Gpu *G = st.gpus[id].get();
  G->id = id;
  // SAGE_DEVICE_OFFSET: logical GPU 0 is physical device `offset` (one
  // process per GPU with every device visible -- bench.py under torchrun --
  // so peers' exported pages map over NVLink)
  static const int offset = [] { const char *e = getenv("SAGE_DEVICE_OFFSET"); return e ? atoi(e) : 0; }();
  G->dev = (id + std::max(0, offset)) % std::max(1, st.n_devices);
  SAGE_CUDA(cudaSetDevice(G->dev));
  SAGE_CUDA(cudaFree(0));  // create/retain the primary context up front (the pre-created ctx)
  SAGE_CUDA(cudaDeviceGetAttribute(&G->sm_count, cudaDevAttrMultiProcessorCount, G->dev));
  SAGE_CU(drv.CtxGetCurrent(&G->primary));
  int lo = 0, hi = 0;
  SAGE_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  SAGE_CUDA(cudaStreamCreateWithPriority(&G->copy, cudaStreamNonBlocking, hi));
  SAGE_CUDA(cudaStreamCreateWithPriority(&G->direct, cudaStreamNonBlocking, hi));
  SAGE_CUDA(cudaStreamCreateWithPriority(&G->verify, cudaStreamNonBlocking, hi));
  SAGE_CUDA(cudaEventCreateWithFlags(&G->ev_dma, cudaEventDisableTiming));
  SAGE_CUDA(cudaStreamCreateWithPriority(&G->land, cudaStreamNonBlocking, hi));
  SAGE_CUDA(cudaStreamCreateWithFlags(&G->host, cudaStreamNonBlocking));
  SAGE_CUDA(cudaStreamCreateWithFlags(&G->d2h, cudaStreamNonBlocking));
  SAGE_CUDA(cudaStreamCreateWithFlags(&G->aux, cudaStreamNonBlocking));
  {
    // D2H RETURN copy streams (SAGE_RETURN_STREAMS; 0 = on the slot).  Two
    // measured best for the cfg-2 e2e burst (+5% over the slot stream)
    const char *env = getenv("SAGE_RETURN_STREAMS");
    int nret = env ? atoi(env) : 2;
    for (int i = 0; i < nret && i < 16; ++i) {
      cudaStream_t s;
      SAGE_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      G->rets.push_back(s);
    }
    SAGE_CUDA(cudaEventCreateWithFlags(&G->ev_ret, cudaEventDisableTiming));
  }
  const char *slot_env = getenv("SAGE_SLOTS");
  const int kSlots = slot_env ? std::max(4, std::min(256, atoi(slot_env))) : 64;
  for (int i = 0; i < kSlots; ++i) {
    cudaStream_t s;
    SAGE_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    G->slots.push_back(s);
    G->slot_free.push_back(kSlots - 1 - i);
  }
  // staging rings: pinned host + device, `ring` slots of (chunk + 64) bytes
  G->chunk = chunk;
  G->ring = (uint32_t)std::max<uint64_t>(2, staging_bytes / chunk);
  const uint64_t slot_bytes = chunk + 256;
  SAGE_CUDA(cudaHostAlloc((void **)&G->pin, G->ring * slot_bytes, cudaHostAllocPortable));
  SAGE_CUDA(cudaMalloc((void **)&G->dstage, G->ring * slot_bytes));
  G->ev_cpu.resize(G->ring);
  G->ev_h2d.resize(G->ring);
  G->ev_land.resize(G->ring);
  for (uint32_t i = 0; i < G->ring; ++i) {
    SAGE_CUDA(cudaEventCreateWithFlags(&G->ev_cpu[i], cudaEventDisableTiming));
    SAGE_CUDA(cudaEventCreateWithFlags(&G->ev_h2d[i], cudaEventDisableTiming));
    SAGE_CUDA(cudaEventCreateWithFlags(&G->ev_land[i], cudaEventDisableTiming));
  }
  // checksum accumulators: one per in-flight load
  G->scratch.n = 16384;
  G->scratch.busy.assign(G->scratch.n, 0);
  SAGE_CUDA(cudaMalloc((void **)&G->scratch.d_acc, G->scratch.n * sizeof(unsigned long long)));
  SAGE_CUDA(cudaMalloc((void **)&G->scratch.d_done, G->scratch.n * sizeof(unsigned int)));
  SAGE_CUDA(cudaMemset(G->scratch.d_acc, 0, G->scratch.n * sizeof(unsigned long long)));
  SAGE_CUDA(cudaMemset(G->scratch.d_done, 0, G->scratch.n * sizeof(unsigned int)));
  SAGE_CUDA(cudaHostAlloc((void **)&G->scratch.h_res, G->scratch.n * sizeof(unsigned long long),
                          cudaHostAllocPortable | cudaHostAllocMapped));
  SAGE_CUDA(cudaHostGetDevicePointer((void **)&G->scratch.d_res, G->scratch.h_res, 0));
  SAGE_CUDA(cudaMalloc((void **)&G->d_verify, 64));
  // clock anchor on its own top-priority stream (nothing else is queued there)
  SAGE_CUDA(cudaStreamCreateWithPriority(&G->clock, cudaStreamNonBlocking, hi));
  SAGE_CUDA(cudaEventCreate(&G->anchor));
  SAGE_CUDA(cudaEventCreate(&G->anchor_trial));
  {
    std::lock_guard<std::mutex> lk(G->anchor_mu);
    clock_anchor_refresh(G, true);
  }
  if (pool_bytes == 0) {
    size_t fr = 0, tot = 0;
    SAGE_CUDA(cudaMemGetInfo(&fr, &tot));
    pool_bytes = fr > (4ull << 30) ? fr - (4ull << 30) : fr / 2;
  }
  return pool_create(G, pool_bytes);
}

void gpu_teardown(Gpu *G) {
  cudaSetDevice(G->dev);
  stats_clear_gpu(G);
  pool_destroy(G);
  for (auto s : G->slots) cudaStreamDestroy(s);
  G->slots.clear();
  for (auto s : G->rets) cudaStreamDestroy(s);
  G->rets.clear();
  if (G->ev_ret) cudaEventDestroy(G->ev_ret);
  for (cudaStream_t s : {G->copy, G->direct, G->verify, G->land, G->host, G->d2h, G->aux})
    if (s) cudaStreamDestroy(s);
  if (G->ev_dma) cudaEventDestroy(G->ev_dma);
  for (auto e : G->ev_cpu) cudaEventDestroy(e);
  for (auto e : G->ev_h2d) cudaEventDestroy(e);
  for (auto e : G->ev_land) cudaEventDestroy(e);
  if (G->anchor) cudaEventDestroy(G->anchor);
  if (G->anchor_trial) cudaEventDestroy(G->anchor_trial);
  if (G->clock) cudaStreamDestroy(G->clock);
  if (G->ipc) cudaStreamDestroy(G->ipc);
  if (G->pin) cudaFreeHost(G->pin);
  if (G->dstage) cudaFree(G->dstage);
  if (G->scratch.d_acc) cudaFree(G->scratch.d_acc);
  if (G->scratch.d_done) cudaFree(G->scratch.d_done);
  if (G->scratch.h_res) cudaFreeHost(G->scratch.h_res);
  if (G->d_verify) cudaFree(G->d_verify);
}

}  // namespace sage

using namespace sage;

extern "C" {

int sage_pool_configure(int gpu, uint64_t capacity, uint64_t granularity) {
  SAGE_TRY(require_up());
  Gpu *G = gpu_get(gpu);
  if (!G) return fail(SAGE_ENODEV, "pool_configure: bad gpu");
  Pool *P = G->pool;
  std::lock_guard<std::mutex> lk(P->mu);
  if (capacity && capacity < P->usage) return fail(SAGE_EINVAL, "capacity below current usage");
  if (capacity) P->capacity = capacity;
  P->granularity = granularity;
  return SAGE_OK;
}

int sage_pool_trim(int gpu, uint64_t *released) {
  SAGE_TRY(require_up());
  Gpu *G = gpu_get(gpu);
  if (!G) return fail(SAGE_ENODEV, "pool_trim: bad gpu");
  Pool *P = G->pool;
  std::lock_guard<std::mutex> lk(P->mu);
  cudaSetDevice(dev_of(gpu));
  reap(P, false);
  const uint64_t before = P->cached + (uint64_t)P->chunks.size() * P->chunk_bytes;
  release_cache(P);
  const uint64_t after = P->cached + (uint64_t)P->chunks.size() * P->chunk_bytes;
  if (released) *released = before - after;
  return SAGE_OK;
}

int sage_pool_effective(int gpu, uint64_t bytes, uint64_t *effective) {
  SAGE_TRY(require_up());
  Gpu *G = gpu_get(gpu);
  if (!G || !effective) return fail(SAGE_EINVAL, "pool_effective: bad argument");
  *effective = round_up(bytes, G->pool->granularity);
  return SAGE_OK;
}

int sage_pool_alloc(int gpu, uint64_t bytes, int cls, sage_handle *h, uint64_t *dptr, uint64_t *shortfall) {
  SAGE_TRY(require_up());
  Gpu *G = gpu_get(gpu);
  if (!G) return fail(SAGE_ENODEV, "pool_alloc: bad gpu");
  if (!h) return fail(SAGE_EINVAL, "pool_alloc: null handle out");
  if (bytes == 0) return fail(SAGE_EINVAL, "pool_alloc: allocation size must be > 0");
  bool acct = (cls & SAGE_ALLOC_ACCOUNT_ONLY) != 0;
  int c = cls & 0xff;
  if (c < 0 || c > 3) return fail(SAGE_EINVAL, "pool_alloc: bad class");
  if (acct && (cls & SAGE_ALLOC_UNACCOUNTED)) return fail(SAGE_EINVAL, "pool_alloc: account-only and unaccounted");
  Pool *P = G->pool;
  auto *A = new Alloc();
  A->gpu = gpu;
  A->bytes = bytes;
  A->cls = c;
  A->account_only = acct;
  {
    std::lock_guard<std::mutex> lk(P->mu);
    // unaccounted runtime scratch charges nothing (eff = 0) and skips the budget
    A->eff = (cls & SAGE_ALLOC_UNACCOUNTED) ? 0 : round_up(bytes, P->granularity);
    if (A->eff > P->capacity - P->usage) {
      if (shortfall) *shortfall = A->eff - (P->capacity - P->usage);
      delete A;
      return fail(SAGE_ENOMEM, "pool budget exceeded");
    }
    if (!acct) {
      cudaSetDevice(dev_of(gpu));
      if (!P->zombies.empty()) reap(P, false);
      int rc = map_segment(G, P, A);
      if (rc != SAGE_OK) { delete A; return rc; }
    }
    P->usage += A->eff;
    P->by_class[c] += A->eff;
  }
  uint64_t id = g_alloc_next++;
  {
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    g_allocs[id] = A;
  }
  *h = make_handle(Kind::Alloc, id);
  if (dptr) *dptr = (uint64_t)A->va;
  if (shortfall) *shortfall = 0;
  return SAGE_OK;
}

int sage_pool_free(sage_handle h) {
  if (handle_kind(h) != Kind::Alloc) return fail(SAGE_EINVAL, "not a pool handle");
  Alloc *A = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    auto it = g_allocs.find(h & ((1ull << 56) - 1));
    if (it == g_allocs.end()) return fail(SAGE_ESTATE, "double or unknown free");
    A = it->second;
    g_allocs.erase(it);
  }
  Gpu *G = gpu_get(A->gpu);
  Pool *P = G->pool;
  {
    std::lock_guard<std::mutex> lk(P->mu);
    if (!A->account_only) {
      // contract: the caller frees only after the END events of every op that
      // touched the segment completed (the runtime frees on invocation
      // completion / decay), so no device-wide drain is needed here
      cudaSetDevice(dev_of(A->gpu));
      unmap_segment(P, A);
    }
    P->usage -= A->eff;
    P->by_class[A->cls] -= A->eff;
    reap(P, false);
  }
  delete A;
  return SAGE_OK;
}

int sage_pool_free_after_n(sage_handle h, const sage_handle *evs, int n) {
  if (handle_kind(h) != Kind::Alloc) return fail(SAGE_EINVAL, "not a pool handle");
  if (n < 0 || (n > 0 && !evs)) return fail(SAGE_EINVAL, "free_after: bad event list");
  std::vector<Event *> E;
  for (int i = 0; i < n; ++i) {
    if (!evs[i]) continue;
    Event *e = event_get(evs[i]);
    if (!e || !e->ev) return fail(SAGE_ESTATE, "free_after: unknown event");
    SAGE_TRY(event_await_recorded(e));
    E.push_back(e);
  }
  if (E.empty()) return sage_pool_free(h);
  Alloc *A = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    auto it = g_allocs.find(h & ((1ull << 56) - 1));
    if (it == g_allocs.end()) return fail(SAGE_ESTATE, "double or unknown free");
    A = it->second;
    g_allocs.erase(it);
  }
  Gpu *G = gpu_get(A->gpu);
  Pool *P = G->pool;
  std::lock_guard<std::mutex> lk(P->mu);
  P->usage -= A->eff;
  P->by_class[A->cls] -= A->eff;
  if (A->account_only) { delete A; return SAGE_OK; }
  cudaSetDevice(dev_of(A->gpu));
  cudaEvent_t ev;
  SAGE_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  // chain: our private event completes when every reader's event has (the
  // readers may run on other GPUs: a peer land over NVLink)
  for (Event *e : E) SAGE_CUDA(cudaStreamWaitEvent(G->aux, e->ev, 0));
  SAGE_CUDA(cudaEventRecord(ev, G->aux));
  P->zombies.emplace_back(A, ev);
  reap(P, false);
  return SAGE_OK;
}

int sage_pool_free_after(sage_handle h, sage_handle evh) {
  if (!evh) return fail(SAGE_ESTATE, "free_after: unknown event");
  return sage_pool_free_after_n(h, &evh, 1);
}

int sage_pool_usage(int gpu, uint64_t by_class[4], uint64_t *ledger_total, uint64_t *physical_total,
                    uint64_t *capacity) {
  SAGE_TRY(require_up());
  Gpu *G = gpu_get(gpu);
  if (!G) return fail(SAGE_ENODEV, "pool_usage: bad gpu");
  Pool *P = G->pool;
  std::lock_guard<std::mutex> lk(P->mu);
  if (by_class) for (int i = 0; i < 4; ++i) by_class[i] = P->by_class[i];
  if (ledger_total) *ledger_total = P->usage;
  if (physical_total) *physical_total = P->physical;
  if (capacity) *capacity = P->capacity;
  return SAGE_OK;
}

int sage_pool_dptr(sage_handle h, uint64_t *dptr, uint64_t *bytes) {
  if (handle_kind(h) != Kind::Alloc) return fail(SAGE_EINVAL, "not a pool handle");
  std::lock_guard<std::mutex> lk(g_alloc_mu);
  auto it = g_allocs.find(h & ((1ull << 56) - 1));
  if (it == g_allocs.end()) return fail(SAGE_ESTATE, "unknown pool handle");
  if (dptr) *dptr = (uint64_t)it->second->va;
  if (bytes) *bytes = it->second->bytes;
  return SAGE_OK;
}

}  // extern "C"

// the physical pages behind a pool allocation (multicast binding, fanout.cu)
int sage::pool_alloc_phys(sage_handle h, CUmemGenericAllocationHandle *ph, uint64_t *phys, uint64_t *dptr, int *gpu) {
  if (handle_kind(h) != Kind::Alloc) return fail(SAGE_EINVAL, "not a pool handle");
  std::lock_guard<std::mutex> lk(g_alloc_mu);
  auto it = g_allocs.find(h & ((1ull << 56) - 1));
  if (it == g_allocs.end()) return fail(SAGE_ESTATE, "unknown pool handle");
  const Alloc *A = it->second;
  if (A->account_only || !A->ph)
    return fail(SAGE_EINVAL, A->carved ? "allocation is a piece of a pool chunk (private writable data): no pages of its own"
                                       : "allocation has no device pages");
  *ph = A->ph;
  *phys = A->phys;
  *dptr = (uint64_t)A->va;
  *gpu = A->gpu;
  return SAGE_OK;
}

// ------------------------------------------------- cross-process sharing ----
// The paper's memory daemon lands a function's read-only data once and the
// per-function engines (separate processes) map it (PAPER.md:279-281,
// 358-379): the segment's physical handle leaves as a POSIX file descriptor
// and is mapped into the importer's address space -- no copy.
namespace {
struct Import {
  int gpu = -1;
  uint64_t phys = 0;
  CUdeviceptr va = 0;
  CUmemGenericAllocationHandle ph = 0;
};
std::mutex g_imp_mu;
std::unordered_map<uint64_t, Import *> g_imports;
std::atomic<uint64_t> g_imp_next{1};
}  // namespace

extern "C" int sage_pool_export(sage_handle h, int *fd, uint64_t *phys_bytes) {
  SAGE_TRY(require_up());
  if (!fd || !phys_bytes) return fail(SAGE_EINVAL, "pool_export: null argument");
  Alloc *A = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    auto it = g_allocs.find(h & ((1ull << 56) - 1));
    if (handle_kind(h) == Kind::Alloc && it != g_allocs.end()) A = it->second;
  }
  if (A && A->carved) return fail(SAGE_EINVAL, "pool_export: private writable segments are carved from pool chunks");
  if (!A || !A->ph) return fail(SAGE_ESTATE, "pool_export: unknown or unmapped segment");
  int out = -1;
  SAGE_CU(drv.MemExportToShareableHandle(&out, A->ph, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
  A->exported = true;   // importers keep the pages alive; this process must not reuse them
  *fd = out;
  *phys_bytes = A->phys;
  return SAGE_OK;
}

extern "C" int sage_segment_import(int gpu, int fd, uint64_t phys_bytes, sage_handle *h, uint64_t *dptr) {
  SAGE_TRY(require_up());
  Gpu *G = gpu_get(gpu);
  if (!G || fd < 0 || !phys_bytes || !h || !dptr) return fail(SAGE_EINVAL, "segment_import: bad argument");
  auto *I = new Import();
  I->gpu = gpu;
  I->phys = phys_bytes;
  cudaSetDevice(G->dev);
  CUresult r = drv.MemImportFromShareableHandle(&I->ph, reinterpret_cast<void *>(static_cast<uintptr_t>(fd)),
                                                CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
  if (r != CUDA_SUCCESS) { delete I; return cu_fail(r, "cuMemImportFromShareableHandle"); }
  r = drv.MemAddressReserve(&I->va, phys_bytes, G->pool ? G->pool->vmm_gran : 0, 0, 0);
  if (r == CUDA_SUCCESS) r = drv.MemMap(I->va, phys_bytes, 0, I->ph, 0);
  if (r == CUDA_SUCCESS) {
    CUmemAccessDesc a{};
    a.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    a.location.id = G->dev;
    a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    r = drv.MemSetAccess(I->va, phys_bytes, &a, 1);
  }
  if (r != CUDA_SUCCESS) {
    if (I->va) { drv.MemUnmap(I->va, phys_bytes); drv.MemAddressFree(I->va, phys_bytes); }
    drv.MemRelease(I->ph);
    delete I;
    return cu_fail(r, "segment_import map");
  }
  uint64_t id = g_imp_next++;
  {
    std::lock_guard<std::mutex> lk(g_imp_mu);
    g_imports[id] = I;
  }
  *h = make_handle(Kind::Alloc, (1ull << 55) | id);   // import ids live in the upper half of the alloc space
  *dptr = I->va;
  return SAGE_OK;
}

extern "C" int sage_segment_unimport(sage_handle h) {
  Import *I = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_imp_mu);
    auto it = g_imports.find(h & ((1ull << 55) - 1));
    if (handle_kind(h) != Kind::Alloc || !(h & (1ull << 55)) || it == g_imports.end())
      return fail(SAGE_ESTATE, "double or unknown segment unimport");
    I = it->second;
    g_imports.erase(it);
  }
  cudaSetDevice(dev_of(I->gpu));
  // the caller guarantees no device work still reads the mapping
  drv.MemUnmap(I->va, I->phys);
  drv.MemAddressFree(I->va, I->phys);
  drv.MemRelease(I->ph);
  delete I;
  return SAGE_OK;
}
