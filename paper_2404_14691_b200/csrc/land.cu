// land.cu — segment layouts, the chunk planner, the sm_100a `land` kernel and
// the load pipeline (CPU_LOAD memcpy -> H2D on the copy engine -> land).
//
// Replaces the CPU_LOAD -> GPU_LOAD chain of plan_invocation
// (functions.py:257-268) and the fluid Channel it charged
// (resources.py:82-234).  Byte semantics follow oracle/sage_oracle.c
// (oracle_land / oracle_checksum); tests/ check bit-exactness.
//
// Data layout in HBM
//   packed stream  P[0, packed)      tensors back to back (the DB record)
//   landed segment S[0, seg)         tensor i at dst_off[i] (16-B aligned),
//                                    zero padding up to the next extent
//   device staging ring              `ring` slots of (chunk + 256) bytes; slot
//                                    for chunk k holds P[sb_k, se_k) with
//                                    sb_k = c_k - 16 (k > 0) so every 16-B
//                                    destination vector assigned to chunk k
//                                    finds all its source bytes in its slot.
//
// Work assignment: destination vector v (16 B) of tensor i is landed by the
// chunk that holds its LAST source byte (padding vectors go with the tensor's
// last data byte).  Per chunk that is one contiguous run of vectors per
// tensor (an Item); the planner emits Items + a prefix sum of their lengths.
#include "common.h"
#include "checksum.cuh"

#include <algorithm>

namespace sage {

struct __align__(16) LandItem {
  unsigned long long dst_vec0;  // first destination vector (segment relative)
  long long src_rel0;           // source byte of that vector, relative to the slot base
  long long data0;              // data bytes of the tensor from that vector on (<=0: padding)
  unsigned int nvec;
  unsigned int pad_;
};

struct ChunkPlan {
  uint64_t sb = 0, se = 0;       // packed range held by the slot
  uint32_t item_begin = 0, item_end = 0;
  uint32_t prefix_begin = 0;     // index into prefix (item_end - item_begin + 1 entries)
  uint32_t nvec = 0;
};

struct Plan {
  uint64_t chunk = 0;
  std::vector<ChunkPlan> chunks;
  std::vector<LandItem> items;
  std::vector<uint32_t> prefix;
  // device copies per gpu
  std::vector<LandItem *> d_items;
  std::vector<uint32_t *> d_prefix;
};

struct Tensor { uint64_t src, dst, len, ext_end; };

struct Layout {
  std::vector<Tensor> t;
  uint64_t packed = 0, seg = 0;
  Plan chunked, whole;
};

static constexpr uint64_t kWholeChunk = 4ull << 30;   // one launch per segment (<= 4 GiB: 32-bit vector indices)
static std::mutex g_lay_mu;
static std::unordered_map<uint64_t, Layout *> g_layouts;
static std::atomic<uint64_t> g_lay_next{1};

// ------------------------------------------------------------- planner -----
static uint64_t vec_key(const Tensor &T, uint64_t q) {
  // last source byte needed by vector q of tensor T (T.len > 0)
  uint64_t r = 16 * q;
  uint64_t last = (r + 15 < T.len) ? r + 15 : T.len - 1;
  return T.src + last;
}

// first vector q in [0, V) with key(q) >= c
static uint64_t lower_vec(const Tensor &T, uint64_t V, uint64_t c) {
  uint64_t lo = 0, hi = V;
  while (lo < hi) {
    uint64_t mid = (lo + hi) / 2;
    if (vec_key(T, mid) >= c) hi = mid; else lo = mid + 1;
  }
  return lo;
}

static int build_plan(const Layout &L, uint64_t chunk, Plan *P) {
  P->chunk = chunk;
  P->chunks.clear(); P->items.clear(); P->prefix.clear();
  uint64_t nchunks = L.packed == 0 ? 1 : (L.packed + chunk - 1) / chunk;
  P->chunks.resize(nchunks);
  for (uint64_t k = 0; k < nchunks; ++k) {
    ChunkPlan &C = P->chunks[k];
    uint64_t ck = k * chunk;
    C.sb = k == 0 ? 0 : ck - 16;
    C.se = std::min<uint64_t>(L.packed, (k + 1) * chunk);
  }
  // per chunk, collect items of every tensor
  std::vector<std::vector<LandItem>> per(nchunks);
  for (const Tensor &T : L.t) {
    uint64_t V = (T.ext_end - T.dst) / 16;
    if (V == 0) continue;
    if (T.len == 0) {  // pure padding extent: chunk 0
      LandItem I{T.dst / 16, 0, 0, (unsigned)V, 0};
      per[0].push_back(I);
      continue;
    }
    for (uint64_t k = 0; k < nchunks; ++k) {
      uint64_t c0 = k * chunk, c1 = (k + 1 == nchunks) ? ~0ull : (k + 1) * chunk;
      uint64_t qb = k == 0 ? 0 : lower_vec(T, V, c0);
      uint64_t qe = (k + 1 == nchunks) ? V : lower_vec(T, V, c1);
      if (qe <= qb) continue;
      uint64_t sb = P->chunks[k].sb;
      for (uint64_t q = qb; q < qe;) {  // split runs so nvec fits 32 bits
        uint64_t n = std::min<uint64_t>(qe - q, 1u << 30);
        LandItem I;
        I.dst_vec0 = T.dst / 16 + q;
        I.src_rel0 = (long long)(T.src + 16 * q) - (long long)sb;
        I.data0 = (long long)T.len - (long long)(16 * q);
        I.nvec = (unsigned)n;
        I.pad_ = 0;
        per[k].push_back(I);
        q += n;
      }
      (void)c1;
    }
  }
  for (uint64_t k = 0; k < nchunks; ++k) {
    ChunkPlan &C = P->chunks[k];
    C.item_begin = (uint32_t)P->items.size();
    C.prefix_begin = (uint32_t)P->prefix.size();
    uint64_t acc = 0;
    P->prefix.push_back(0);
    for (auto &I : per[k]) {
      P->items.push_back(I);
      acc += I.nvec;
      if (acc > 0xFFFFFFF0ull) return fail(SAGE_EINVAL, "chunk too large for the land planner");
      P->prefix.push_back((uint32_t)acc);
    }
    C.item_end = (uint32_t)P->items.size();
    C.nvec = (uint32_t)acc;
  }
  return SAGE_OK;
}

static int plan_upload(Plan *P, int gpu) {
  if ((int)P->d_items.size() <= gpu) { P->d_items.resize(gpu + 1, nullptr); P->d_prefix.resize(gpu + 1, nullptr); }
  if (P->d_items[gpu]) return SAGE_OK;
  cudaSetDevice(dev_of(gpu));
  size_t ni = std::max<size_t>(1, P->items.size()), np = std::max<size_t>(1, P->prefix.size());
  SAGE_CUDA(cudaMalloc((void **)&P->d_items[gpu], ni * sizeof(LandItem)));
  SAGE_CUDA(cudaMalloc((void **)&P->d_prefix[gpu], np * sizeof(uint32_t)));
  if (!P->items.empty())
    SAGE_CUDA(cudaMemcpy(P->d_items[gpu], P->items.data(), P->items.size() * sizeof(LandItem), cudaMemcpyHostToDevice));
  SAGE_CUDA(cudaMemcpy(P->d_prefix[gpu], P->prefix.data(), P->prefix.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
  return SAGE_OK;
}

static void plan_free(Plan *P) {
  for (size_t g = 0; g < P->d_items.size(); ++g) {
    if (P->d_items[g]) { cudaSetDevice(dev_of((int)g)); cudaFree(P->d_items[g]); }
    if (P->d_prefix[g]) cudaFree(P->d_prefix[g]);
  }
  P->d_items.clear(); P->d_prefix.clear();
}

static int layout_build(const uint64_t *src_off, const uint64_t *dst_off, const uint64_t *len, uint32_t n,
                        uint64_t packed, uint64_t seg, uint64_t chunk, Layout *L) {
  if (seg % 16) return fail(SAGE_EINVAL, "layout: seg_bytes must be a multiple of 16");
  if (n && (!src_off || !dst_off || !len)) return fail(SAGE_EINVAL, "layout: null arrays");
  L->packed = packed;
  L->seg = seg;
  L->t.resize(n);
  for (uint32_t i = 0; i < n; ++i) {
    if (dst_off[i] % 16) return fail(SAGE_EINVAL, "layout: dst_off must be 16-byte aligned");
    if (i == 0 && dst_off[0] != 0) return fail(SAGE_EINVAL, "layout: dst_off[0] must be 0");
    if (src_off[i] + len[i] < src_off[i] || src_off[i] + len[i] > packed)
      return fail(SAGE_EINVAL, "layout: tensor exceeds the packed stream");
    uint64_t lim = (i + 1 < n) ? dst_off[i + 1] : seg;
    if (i + 1 < n && dst_off[i + 1] < dst_off[i]) return fail(SAGE_EINVAL, "layout: dst_off must ascend");
    if (dst_off[i] + len[i] > lim) return fail(SAGE_EINVAL, "layout: tensor overlaps the next extent");
    L->t[i] = Tensor{src_off[i], dst_off[i], len[i], lim};
  }
  if (n == 0 && seg) return fail(SAGE_EINVAL, "layout: empty layout must have seg_bytes == 0");
  SAGE_TRY(build_plan(*L, chunk, &L->chunked));
  // HBM-resident / peer sources need no staging: land straight from the
  // source in one launch per 4 GiB (a 1 GiB segment in 4 x 256 MiB launches
  // measured 391 us vs 361 us in one: ramp and tail per launch)
  SAGE_TRY(build_plan(*L, kWholeChunk, &L->whole));
  return SAGE_OK;
}

static Layout *layout_get(sage_handle h) {
  if (handle_kind(h) != Kind::Layout) return nullptr;
  std::lock_guard<std::mutex> lk(g_lay_mu);
  auto it = g_layouts.find(h & ((1ull << 56) - 1));
  return it == g_layouts.end() ? nullptr : it->second;
}

static void identity_clear();
int layouts_destroy_all() {
  identity_clear();
  std::lock_guard<std::mutex> lk(g_lay_mu);
  for (auto &kv : g_layouts) {
    plan_free(&kv.second->chunked);
    plan_free(&kv.second->whole);
    delete kv.second;
  }
  g_layouts.clear();
  return SAGE_OK;
}

#include "land_kernels.cuh"


// --------------------------------------------------------------- loads -----
struct Load {
  int gpu = -1;
  sage_handle hb = 0, he = 0;                 // pooled begin / end events (internal)
  cudaEvent_t ev_begin = nullptr, ev_end = nullptr;
  Event *eb = nullptr, *ee = nullptr;         // ... as Events (cached times)
  std::atomic<int64_t> cpu_begin{-1}, cpu_end{-1};
  uint64_t host_bytes = 0, link_bytes = 0, landed = 0;
  uint32_t chunks = 0;
  uint32_t acc_idx = UINT32_MAX;   // checksum slot (held until release)
  bool has_gpu_begin = false;
};

static std::mutex g_load_mu;
static std::unordered_map<uint64_t, Load *> g_loads;
static std::atomic<uint64_t> g_load_next{1};

struct HostCopyArg {
  Load *L;
  void *dst;
  const void *src;
  size_t bytes;
};

static void CUDART_CB host_copy_fn(void *p) {
  auto *a = static_cast<HostCopyArg *>(p);
  int64_t t0 = host_now_us();
  int64_t expect = -1;
  a->L->cpu_begin.compare_exchange_strong(expect, t0);
  parallel_memcpy(a->dst, a->src, a->bytes);
  a->L->cpu_end.store(host_now_us());
  delete a;
}

static int wait_list(cudaStream_t s, const sage_handle *w, int n) {
  for (int i = 0; i < n; ++i) {
    Event *e = event_get(w[i]);
    if (!e) return fail(SAGE_ESTATE, "load: unknown wait event");
    if (!e->ev) {
      while (!e->host_done.load()) std::this_thread::sleep_for(std::chrono::microseconds(20));
      continue;
    }
    SAGE_TRY(event_await_recorded(e));
    SAGE_CUDA(cudaStreamWaitEvent(s, e->ev, 0));
  }
  return SAGE_OK;
}

// SAGE_LAND_TMA=1 (opt-in): launches of >= 1 MiB take land_tma_kernel.  Off by
// default: in the bench probe it measured 4.14 TB/s vs land_kernel's 4.80, and
// its one 65 KB-smem CTA per SM keeps concurrent invocations' kernels off the
// SMs (value leg 15.6k vs 20.4k inv/s; profiles/r1_land_tma_ab.txt)
constexpr int kTmaSmem = kTmaStages * kTmaStageBytes + 128;
static bool land_tma_enabled(int dev) {
  static const bool env_on = [] {
    const char *e = getenv("SAGE_LAND_TMA");
    return e && atoi(e) != 0;
  }();
  static std::atomic<int> ok[64];   // per device: 0 unknown, 1 usable, -1 not
  if (!env_on || dev < 0 || dev >= 64) return false;
  int v = ok[dev].load(std::memory_order_acquire);
  if (v == 0) {   // the smem opt-in is per device (current device = dev)
    v = cudaFuncSetAttribute(land_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem) == cudaSuccess
            ? 1 : -1;
    ok[dev].store(v, std::memory_order_release);
  }
  return v > 0;
}

static int enqueue_land(Gpu *G, const Plan &P, const ChunkPlan &C, int gpu, const uint8_t *slot,
                        uint8_t *dst, uint32_t acc_idx, bool final_launch) {
  if (C.nvec == 0 && !final_launch) return SAGE_OK;
  LandArgs a;
  a.acc = G->scratch.d_acc + acc_idx;
  a.done = G->scratch.d_done + acc_idx;
  a.out = final_launch ? G->scratch.d_res + acc_idx : nullptr;
  a.items = P.d_items[gpu] + C.item_begin;
  a.prefix = P.d_prefix[gpu] + C.prefix_begin;
  a.n_items = C.item_end - C.item_begin;
  a.total_vec = C.nvec;
  a.slot = slot;
  a.slot_bytes = C.se - C.sb;
  a.dst = dst;
  cudaEvent_t sb = stat_begin(G, G->land);
  if (C.nvec >= kTmaMinVec && land_tma_enabled(G->dev)) {
    const uint32_t units = (C.nvec + kTmaUnitVec - 1) / kTmaUnitVec;
    const int grid = (int)std::min<uint32_t>(units, (uint32_t)G->sm_count);
    land_tma_kernel<<<grid, kTmaThreads, kTmaSmem, G->land>>>(a);
  } else {
    land_kernel<<<C.nvec ? land_grid(G, C.nvec) : 1, kLandThreads, 0, G->land>>>(a);
  }
  // algorithmic bytes: the packed bytes read + the segment vectors written
  stat_end(G, G->land, SAGE_KERNEL_LAND, sb, (C.se - C.sb) + 16ull * C.nvec);
  SAGE_CUDA(cudaGetLastError());
  return SAGE_OK;
}

int layout_tensors(sage_handle h, std::vector<uint64_t> *src, std::vector<uint64_t> *dst,
                   std::vector<uint64_t> *len, uint64_t *packed, uint64_t *seg) {
  Layout *L = layout_get(h);
  if (!L) return fail(SAGE_ESTATE, "unknown layout");
  for (const Tensor &T : L->t) { src->push_back(T.src); dst->push_back(T.dst); len->push_back(T.len); }
  *packed = L->packed;
  *seg = L->seg;
  return SAGE_OK;
}

// identity layouts (input payloads, cache reloads, fan-out) are cached by size
static std::mutex g_ident_mu;
static std::unordered_map<uint64_t, Layout *> g_ident;
static int identity_layout(uint64_t bytes, Layout **out) {
  std::lock_guard<std::mutex> lk(g_ident_mu);
  auto it = g_ident.find(bytes);
  if (it != g_ident.end()) { *out = it->second; return SAGE_OK; }
  auto *lay = new Layout();
  uint64_t z = 0, n = bytes;
  int rc = layout_build(&z, &z, &n, bytes ? 1u : 0u, bytes, (bytes + 15) & ~15ull, st.chunk, lay);
  for (int g = 0; rc == SAGE_OK && g < st.n_gpus; ++g) {
    rc = plan_upload(&lay->chunked, g);
    if (rc == SAGE_OK) rc = plan_upload(&lay->whole, g);
  }
  if (rc != SAGE_OK) { plan_free(&lay->chunked); plan_free(&lay->whole); delete lay; return rc; }
  g_ident[bytes] = lay;
  *out = lay;
  return SAGE_OK;
}
static void identity_clear() {
  std::lock_guard<std::mutex> lk(g_ident_mu);
  for (auto &kv : g_ident) { plan_free(&kv.second->chunked); plan_free(&kv.second->whole); delete kv.second; }
  g_ident.clear();
}

}  // namespace sage

using namespace sage;

extern "C" {

int sage_layout_create(const uint64_t *src_off, const uint64_t *dst_off, const uint64_t *len, uint32_t n,
                       uint64_t packed_bytes, uint64_t seg_bytes, sage_handle *layout) {
  if (!layout) return fail(SAGE_EINVAL, "layout_create: null out");
  auto *L = new Layout();
  int rc = layout_build(src_off, dst_off, len, n, packed_bytes, seg_bytes, st.up ? st.chunk : (8ull << 20), L);
  if (rc != SAGE_OK) { delete L; return rc; }
  if (st.up) {
    for (int g = 0; g < st.n_gpus; ++g) {
      rc = plan_upload(&L->chunked, g);
      if (rc == SAGE_OK) rc = plan_upload(&L->whole, g);
      if (rc != SAGE_OK) { plan_free(&L->chunked); plan_free(&L->whole); delete L; return rc; }
    }
  }
  uint64_t id = g_lay_next++;
  {
    std::lock_guard<std::mutex> lk(g_lay_mu);
    g_layouts[id] = L;
  }
  *layout = make_handle(Kind::Layout, id);
  return SAGE_OK;
}

int sage_layout_destroy(sage_handle h) {
  if (handle_kind(h) != Kind::Layout) return fail(SAGE_EINVAL, "not a layout handle");
  Layout *L = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_lay_mu);
    auto it = g_layouts.find(h & ((1ull << 56) - 1));
    if (it == g_layouts.end()) return fail(SAGE_ESTATE, "double or unknown layout destroy");
    L = it->second;
    g_layouts.erase(it);
  }
  plan_free(&L->chunked);
  plan_free(&L->whole);
  delete L;
  return SAGE_OK;
}

int sage_layout_chunks(sage_handle h, uint32_t *n) {
  Layout *L = layout_get(h);
  if (!L || !n) return fail(SAGE_ESTATE, "unknown layout");
  *n = (uint32_t)L->chunked.chunks.size();
  return SAGE_OK;
}

int sage_segment_load(const sage_load_desc *d, sage_handle *load_out, sage_handle *end_ev) {
  return segment_load(d, load_out, end_ev, 0);
}

}  // extern "C"

// A staged load being enqueued piece by piece (the issuer interleaves other
// invocations' copies between the pieces of a large cold load).
struct sage::LoadCursor {
  Load *L = nullptr;
  Gpu *G = nullptr;
  const Plan *P = nullptr;
  const uint8_t *src = nullptr;
  uint8_t *dst = nullptr;
  int gpu = -1;
  bool pinned = false;
  bool direct = false;   // unverified identity: H2D from the pinned slot straight into dst, no land
  uint64_t seg = 0;      // landed bytes (direct: zero padding past the packed end)
  size_t next = 0;       // first chunk not yet enqueued
};

// Register a finished load: END on the land stream, handles out.
static int load_finish(Load *L, Gpu *G, sage_handle *load_out, sage_handle *end_ev) {
  if (!L->has_gpu_begin) SAGE_TRY(event_record(L->eb, G->land));
  SAGE_TRY(event_record(L->ee, G->land));
  SAGE_TRY(event_alias(L->he, end_ev));
  uint64_t id = g_load_next++;
  {
    std::lock_guard<std::mutex> lk2(g_load_mu);
    g_loads[id] = L;
  }
  *load_out = make_handle(Kind::Load, id);
  return SAGE_OK;
}

// Enqueue the ring chunks of a staged (packed / pageable) load from
// c->next on until at least `budget` bytes crossed the link or the plan is
// done: CPU_LOAD (pageable only) -> H2D into a ring slot -> land.
static bool staged_land_forced() {
  static const bool v = [] {
    const char *e = getenv("SAGE_STAGED_LAND");
    return e && atoi(e) != 0;
  }();
  return v;
}

static int cursor_advance(LoadCursor *c, uint64_t budget, uint64_t *enq) {
  Gpu *G = c->G;
  Load *L = c->L;
  const Plan &P = *c->P;
  const uint64_t slot_bytes = G->chunk + 256;
  uint64_t moved = 0;
  int rc = SAGE_OK;
  for (; c->next < P.chunks.size() && moved < budget; ++c->next) {
    const size_t k = c->next;
    const ChunkPlan &C = P.chunks[k];
    const uint64_t n = C.se - C.sb;
    const uint32_t r = (uint32_t)(G->chunk_seq++ % G->ring);
    uint8_t *dslot = G->dstage + r * slot_bytes;
    uint8_t *pslot = G->pin + r * slot_bytes;
    const uint8_t *src = c->src + C.sb;
    if (n && !c->pinned) {
      // CPU_LOAD: DB record -> pinned staging, once the slot's last H2D is done
      SAGE_CUDA(cudaStreamWaitEvent(G->host, G->ev_h2d[r], 0));
      SAGE_CUDA(cudaLaunchHostFunc(G->host, host_copy_fn, new HostCopyArg{L, pslot, src, (size_t)n}));
      SAGE_CUDA(cudaEventRecord(G->ev_cpu[r], G->host));
      SAGE_CUDA(cudaStreamWaitEvent(G->copy, G->ev_cpu[r], 0));
      L->host_bytes += n;
    }
    if (!n) {
      if (!L->has_gpu_begin) { SAGE_TRY(event_record(L->eb, G->land)); L->has_gpu_begin = true; }
    } else if (c->direct) {
      // unverified identity: the staged bytes go straight to their place in
      // dst (less the 16 B overlap only the land's funnel shift needs); the
      // device slot is untouched, so ev_land[r] keeps marking its last land
      const uint64_t off = k == 0 ? 0 : C.sb + 16;
      if (!L->has_gpu_begin) { SAGE_TRY(event_record(L->eb, G->copy)); L->has_gpu_begin = true; }
      SAGE_CUDA(cudaMemcpyAsync(c->dst + off, (c->pinned ? src : pslot) + (off - C.sb), C.se - off,
                                cudaMemcpyHostToDevice, G->copy));
      SAGE_CUDA(cudaEventRecord(G->ev_h2d[r], G->copy));
      SAGE_CUDA(cudaStreamWaitEvent(G->land, G->ev_h2d[r], 0));   // END (on land) covers it
      L->link_bytes += C.se - off;
      moved += n;
    } else {
      // GPU_LOAD: H2D into the device slot once its last land is done
      SAGE_CUDA(cudaStreamWaitEvent(G->copy, G->ev_land[r], 0));
      if (!L->has_gpu_begin) { SAGE_TRY(event_record(L->eb, G->copy)); L->has_gpu_begin = true; }
      SAGE_CUDA(cudaMemcpyAsync(dslot, c->pinned ? src : pslot, n, cudaMemcpyHostToDevice, G->copy));
      SAGE_CUDA(cudaEventRecord(G->ev_h2d[r], G->copy));
      SAGE_CUDA(cudaStreamWaitEvent(G->land, G->ev_h2d[r], 0));
      L->link_bytes += n;
      moved += n;
    }
    if (c->direct) {   // no land: zero the padding past the packed end
      if (k + 1 == P.chunks.size() && c->seg > C.se)
        SAGE_CUDA(cudaMemsetAsync(c->dst + C.se, 0, c->seg - C.se, G->land));
      continue;
    }
    if ((rc = enqueue_land(G, P, C, c->gpu, dslot, c->dst, L->acc_idx, k + 1 == P.chunks.size())) != SAGE_OK)
      return rc;
    SAGE_CUDA(cudaEventRecord(G->ev_land[r], G->land));
  }
  if (enq) *enq = moved;
  return SAGE_OK;
}

int sage::segment_load_step(LoadCursor *c, uint64_t budget, uint64_t *bytes, sage_handle *piece_ev, bool *done,
                            sage_handle *load_out, sage_handle *end_ev) {
  Gpu *G = c->G;
  cudaSetDevice(G->dev);
  std::lock_guard<std::mutex> lk(G->load_mu);   // ring order == enqueue order
  uint64_t moved = 0;
  SAGE_TRY(cursor_advance(c, budget, &moved));
  if (bytes) *bytes = moved;
  if (piece_ev) {   // marks the end of this piece's H2D (lookahead accounting)
    Event *e;
    SAGE_TRY(event_new(c->gpu, piece_ev, &e));
    SAGE_TRY(event_record(e, G->copy));
  }
  *done = c->next >= c->P->chunks.size();
  if (*done) SAGE_TRY(load_finish(c->L, G, load_out, end_ev));
  return SAGE_OK;
}

void sage::segment_load_close(LoadCursor *c) { delete c; }

int sage::segment_load(const sage_load_desc *d, sage_handle *load_out, sage_handle *end_ev, sage_handle pre_end) {
  NvtxRange nv("sage.segment_load");
  LoadCursor *c = nullptr;
  SAGE_TRY(segment_load_open(d, pre_end, &c, load_out, end_ev));
  if (!c) return SAGE_OK;
  bool done = false;
  int rc = segment_load_step(c, UINT64_MAX, nullptr, nullptr, &done, load_out, end_ev);
  segment_load_close(c);
  return rc;
}

int sage::segment_load_open(const sage_load_desc *d, sage_handle pre_end, LoadCursor **cur, sage_handle *load_out,
                            sage_handle *end_ev) {
  *cur = nullptr;
  SAGE_TRY(require_up());
  if (!d || !load_out || !end_ev) return fail(SAGE_EINVAL, "segment_load: null argument");
  Gpu *G = gpu_get(d->gpu);
  if (!G) return fail(SAGE_ENODEV, "segment_load: bad gpu");
  if (!d->dst) return fail(SAGE_EINVAL, "segment_load: null dst");
  if (d->src_bytes && !d->src) return fail(SAGE_EINVAL, "segment_load: null src");
  const bool dev_src = (d->flags & (SAGE_LOAD_SRC_DEVICE | SAGE_LOAD_SRC_PEER)) != 0;
  if (dev_src && (reinterpret_cast<uintptr_t>(d->src) & 15))
    return fail(SAGE_EINVAL, "segment_load: device source must be 16-byte aligned");
  if ((d->flags & SAGE_LOAD_SRC_PEER) && !gpu_get(d->src_gpu))
    return fail(SAGE_ENODEV, "segment_load: bad src_gpu");
  if (d->dst & 15) return fail(SAGE_EINVAL, "segment_load: dst must be 16-byte aligned");
  cudaSetDevice(dev_of(d->gpu));

  auto *L = new Load();
  L->gpu = d->gpu;
  Layout *lay = nullptr;
  if (d->layout) {
    lay = layout_get(d->layout);
    if (!lay) { delete L; return fail(SAGE_ESTATE, "segment_load: unknown layout"); }
    if (lay->packed != d->src_bytes) { delete L; return fail(SAGE_EINVAL, "segment_load: src_bytes != layout packed_bytes"); }
  } else {
    // identity layout: dst receives the packed bytes verbatim, padded to 16
    int rc = identity_layout(d->src_bytes, &lay);
    if (rc != SAGE_OK) { delete L; return rc; }
  }
  if (Gpu *G0 = gpu_get(d->gpu); G0 && lay->chunked.chunk != G0->chunk) {
    // planned with another chunk size (created before sage_init picked this
    // plane's): re-plan, or staged chunks would overflow their ring slots
    std::lock_guard<std::mutex> lk(g_lay_mu);
    if (lay->chunked.chunk != G0->chunk) {
      Plan fresh;
      int rc = build_plan(*lay, G0->chunk, &fresh);
      if (rc != SAGE_OK) { delete L; return rc; }
      plan_free(&lay->chunked);
      lay->chunked = std::move(fresh);
    }
  }
  {
    int rc = plan_upload(&lay->chunked, d->gpu);
    if (rc == SAGE_OK) rc = plan_upload(&lay->whole, d->gpu);
    if (rc != SAGE_OK) { delete L; return rc; }
  }
  Event *Eb, *Ee;
  {
    int rc = event_new(d->gpu, &L->hb, &Eb);
    if (rc == SAGE_OK) {
      if (pre_end) {   // the END event was handed out before this load was issued
        Ee = event_get(pre_end);
        rc = Ee ? event_alias(pre_end, &L->he) : fail(SAGE_ESTATE, "segment_load: unknown pre-created end event");
      } else {
        rc = event_new(d->gpu, &L->he, &Ee);
      }
    }
    if (rc != SAGE_OK) { delete L; return rc; }
  }
  L->ev_begin = Eb->ev;
  L->ev_end = Ee->ev;
  L->eb = Eb;
  L->ee = Ee;
  L->landed = lay->seg;
  {
    // a free accumulator slot (owned until sage_load_release)
    ChunkScratch &S = G->scratch;
    std::lock_guard<std::mutex> lk(S.mu);
    uint32_t k = 0;
    for (; k < S.n; ++k) {
      const uint32_t idx = (uint32_t)(S.next++ % S.n);
      if (!S.busy[idx]) {
        S.busy[idx] = 1;
        L->acc_idx = idx;
        break;
      }
    }
    if (k == S.n) { delete L; return fail(SAGE_ENOMEM, "segment_load: every checksum slot is held by an unreleased load"); }
  }
  G->scratch.h_res[L->acc_idx] = 0;   // an empty load publishes nothing
  uint8_t *dst = reinterpret_cast<uint8_t *>(d->dst);

  // the same for an unverified identity load from this GPU's HBM (a private
  // request payload already on the device): one D2D copy, as the e2e path's
  // H2D DMA, instead of a land launch: a 4 MiB land is latency bound at
  // ~8 us under ncu (plan-table lookups, a one-wave grid, the result publish)
  const bool d2d = !d->layout && (d->flags & SAGE_LOAD_SRC_DEVICE) && !(d->flags & SAGE_LOAD_SRC_PEER) &&
                   (d->flags & SAGE_LOAD_NO_VERIFY) && d->src_bytes;
  if (d2d || (!d->layout && !dev_src && (d->flags & SAGE_LOAD_SRC_PINNED) && d->src_bytes &&
              lay->seg / 16 < 0xFFFFFFFFull)) {
    // direct path: an identity load from pinned memory needs no staging or
    // unpack -- one DMA straight into dst on its own stream (so it never
    // queues behind memcpy-gated ring chunks) + a read-only verify pass on a
    // second stream, so the next DMA starts while this one is verified
    cudaStream_t s = G->direct;
    std::lock_guard<std::mutex> lk(G->load_mu);
    SAGE_TRY(wait_list(s, d->wait, d->n_wait));
    SAGE_TRY(event_record(Eb, s));
    L->has_gpu_begin = true;
    const uint64_t n = d->src_bytes, seg = lay->seg;
    if (seg > n) SAGE_CUDA(cudaMemsetAsync(dst + n, 0, seg - n, s));
    SAGE_CUDA(cudaMemcpyAsync(dst, d->src, n, d2d ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    if (!d2d) L->link_bytes = n;
    L->chunks = 1;
    if (!(d->flags & SAGE_LOAD_NO_VERIFY)) {
      SAGE_CUDA(cudaEventRecord(G->ev_dma, s));
      s = G->verify;
      SAGE_CUDA(cudaStreamWaitEvent(s, G->ev_dma, 0));
      LandArgs a{};
      a.dst = dst;
      a.total_vec = (uint32_t)(seg / 16);
      a.acc = G->scratch.d_acc + L->acc_idx;
      a.done = G->scratch.d_done + L->acc_idx;
      a.out = G->scratch.d_res + L->acc_idx;
      const int blocks =
          (int)std::max<uint64_t>(1, std::min<uint64_t>((seg / 16 + 1023) / 1024, G->sm_count * 8ull));
      cudaEvent_t sb = stat_begin(G, s);
      verify_kernel<<<blocks, 256, 0, s>>>(a);
      SAGE_CUDA(cudaGetLastError());
      stat_end(G, s, SAGE_KERNEL_VERIFY, sb, seg);
    }
    SAGE_TRY(event_record(Ee, s));
    SAGE_TRY(event_alias(L->he, end_ev));   // the caller's end handle: same event
    uint64_t id = g_load_next++;
    {
      std::lock_guard<std::mutex> lk2(g_load_mu);
      g_loads[id] = L;
    }
    *load_out = make_handle(Kind::Load, id);
    return SAGE_OK;
  }

  std::lock_guard<std::mutex> lk(G->load_mu);  // ring order == enqueue order
  int rc = SAGE_OK;
  // the land stream owns the accumulator; user waits gate the first copy/land
  if ((rc = wait_list(G->land, d->wait, d->n_wait)) != SAGE_OK) return rc;
  if (dev_src) {
    // HBM-resident (or peer, over NVLink) source: land straight from it
    SAGE_TRY(event_record(Eb, G->land));
    L->has_gpu_begin = true;
    const Plan &P = lay->whole;
    L->chunks = (uint32_t)P.chunks.size();
    if (d->flags & SAGE_LOAD_SRC_PEER) L->link_bytes = d->src_bytes;
    for (size_t k = 0; k < P.chunks.size(); ++k) {
      const ChunkPlan &C = P.chunks[k];
      rc = enqueue_land(G, P, C, d->gpu, static_cast<const uint8_t *>(d->src) + C.sb, dst, L->acc_idx,
                        k + 1 == P.chunks.size());
      if (rc != SAGE_OK) return rc;
    }
  } else {
    const bool pinned = (d->flags & SAGE_LOAD_SRC_PINNED) != 0;
    if ((rc = wait_list(G->copy, d->wait, d->n_wait)) != SAGE_OK) return rc;
    if (!pinned && (rc = wait_list(G->host, d->wait, d->n_wait)) != SAGE_OK) return rc;
    L->chunks = (uint32_t)lay->chunked.chunks.size();
    auto *c = new LoadCursor();
    c->L = L;
    c->G = G;
    c->P = &lay->chunked;
    c->src = static_cast<const uint8_t *>(d->src);
    c->dst = dst;
    c->gpu = d->gpu;
    c->pinned = pinned;
    // an unverified identity load needs no land: each staged chunk is DMA'd
    // into its final place (SAGE_STAGED_LAND=1 keeps the land for A/B runs)
    c->direct = !d->layout && (d->flags & SAGE_LOAD_NO_VERIFY) && !staged_land_forced();
    c->seg = lay->seg;
    *cur = c;   // the chunks are enqueued by segment_load_step
    return SAGE_OK;
  }
  return load_finish(L, G, load_out, end_ev);
}

extern "C" {

int sage_load_info_get(sage_handle h, sage_load_info *out) {
  if (handle_kind(h) != Kind::Load || !out) return fail(SAGE_EINVAL, "not a load handle");
  Load *L;
  {
    std::lock_guard<std::mutex> lk(g_load_mu);
    auto it = g_loads.find(h & ((1ull << 56) - 1));
    if (it == g_loads.end()) return fail(SAGE_ESTATE, "unknown load handle");
    L = it->second;
  }
  cudaSetDevice(dev_of(L->gpu));
  int q = event_query(L->ee);
  if (q != SAGE_OK) return q;
  Gpu *G = gpu_get(L->gpu);
  memset(out, 0, sizeof *out);
  out->cpu_begin_us = L->cpu_begin.load();
  out->cpu_end_us = L->cpu_end.load();
  SAGE_TRY(event_time_us(L->eb, &out->gpu_begin_us));
  SAGE_TRY(event_time_us(L->ee, &out->gpu_end_us));
  out->host_bytes = L->host_bytes;
  out->link_bytes = L->link_bytes;
  out->landed_bytes = L->landed;
  out->checksum = G->scratch.h_res[L->acc_idx];
  out->chunks = L->chunks;
  out->status = SAGE_OK;
  return SAGE_OK;
}

int sage_load_release(sage_handle h) {
  if (handle_kind(h) != Kind::Load) return fail(SAGE_EINVAL, "not a load handle");
  Load *L;
  {
    std::lock_guard<std::mutex> lk(g_load_mu);
    auto it = g_loads.find(h & ((1ull << 56) - 1));
    if (it == g_loads.end()) return fail(SAGE_ESTATE, "double or unknown load release");
    L = it->second;
    g_loads.erase(it);
  }
  cudaSetDevice(dev_of(L->gpu));
  cudaEventSynchronize(L->ev_end);  // host copies reference L until the end
  if (Gpu *G = gpu_get(L->gpu)) {
    std::lock_guard<std::mutex> lk(G->scratch.mu);
    if (L->acc_idx < G->scratch.busy.size()) G->scratch.busy[L->acc_idx] = 0;
  }
  sage_event_release(L->hb);
  sage_event_release(L->he);
  delete L;
  return SAGE_OK;
}

namespace {
struct PlainCopy { void *dst; const void *src; size_t n; };
void CUDART_CB plain_copy_fn(void *p) {
  auto *a = static_cast<PlainCopy *>(p);
  parallel_memcpy(a->dst, a->src, a->n);
  delete a;
}
}  // namespace

int sage_host_load(int gpu, void *dst, const void *src, uint64_t bytes, const sage_handle *wait, int n_wait,
                   sage_handle *begin_ev, sage_handle *end_ev) {
  SAGE_TRY(require_up());
  Gpu *G = gpu_get(gpu);
  if (!G || !begin_ev || !end_ev || (bytes && (!dst || !src))) return fail(SAGE_EINVAL, "host_load: bad argument");
  cudaSetDevice(dev_of(gpu));
  std::lock_guard<std::mutex> lk(G->load_mu);
  SAGE_TRY(wait_list(G->host, wait, n_wait));
  Event *b, *e;
  SAGE_TRY(event_new(gpu, begin_ev, &b));
  SAGE_TRY(event_record(b, G->host));
  if (bytes) SAGE_CUDA(cudaLaunchHostFunc(G->host, plain_copy_fn, new PlainCopy{dst, src, (size_t)bytes}));
  SAGE_TRY(event_new(gpu, end_ev, &e));
  return event_record(e, G->host);
}

int sage_segment_checksum(int gpu, uint64_t dptr, uint64_t bytes, uint64_t *checksum) {
  SAGE_TRY(require_up());
  Gpu *G = gpu_get(gpu);
  if (!G || !checksum) return fail(SAGE_EINVAL, "segment_checksum: bad argument");
  if ((dptr & 15) || (bytes & 15)) return fail(SAGE_EINVAL, "segment_checksum: needs 16-byte alignment");
  cudaSetDevice(dev_of(gpu));
  std::lock_guard<std::mutex> lk(G->load_mu);
  SAGE_CUDA(cudaMemsetAsync(G->d_verify, 0, 8, G->aux));
  uint64_t nvec = bytes / 16;
  if (nvec) {
    int blocks = (int)std::min<uint64_t>((nvec + 1023) / 1024, (uint64_t)G->sm_count * 8);
    checksum_kernel<<<std::max(1, blocks), 256, 0, G->aux>>>(reinterpret_cast<const uint4 *>(dptr), nvec,
                                                             G->d_verify);
    SAGE_CUDA(cudaGetLastError());
  }
  unsigned long long v = 0;
  SAGE_CUDA(cudaMemcpyAsync(&v, G->d_verify, 8, cudaMemcpyDeviceToHost, G->aux));
  SAGE_CUDA(cudaStreamSynchronize(G->aux));
  *checksum = v;
  return SAGE_OK;
}

// Test-only: run the chunk planner and the land semantics on the host, exactly
// as the kernel consumes them (slot conventions included), without a GPU.
int sage_debug_emulate_land(sage_handle h, const void *packed, uint64_t packed_bytes, void *seg_out,
                            uint64_t chunk_bytes, uint64_t *checksum) {
  Layout *L0 = layout_get(h);
  if (!L0 || !seg_out || !checksum) return fail(SAGE_EINVAL, "emulate: bad argument");
  if (packed_bytes != L0->packed) return fail(SAGE_EINVAL, "emulate: packed size mismatch");
  Plan P;
  SAGE_TRY(build_plan(*L0, chunk_bytes ? chunk_bytes : L0->chunked.chunk, &P));
  const uint8_t *pk = static_cast<const uint8_t *>(packed);
  uint8_t *out = static_cast<uint8_t *>(seg_out);
  std::vector<uint8_t> written(L0->seg / 16, 0);
  uint64_t sum = 0;
  std::vector<uint8_t> slot;
  for (const ChunkPlan &C : P.chunks) {
    slot.assign(C.se - C.sb + 32, 0xCD);  // garbage beyond the valid range must never leak
    memcpy(slot.data(), pk + C.sb, C.se - C.sb);
    for (uint32_t i = C.item_begin; i < C.item_end; ++i) {
      const LandItem &I = P.items[i];
      for (uint32_t loc = 0; loc < I.nvec; ++loc) {
        long long s = I.src_rel0 + 16ll * loc, dd = I.data0 - 16ll * loc;
        uint64_t dv = I.dst_vec0 + loc;
        uint8_t v[16] = {0};
        for (int b = 0; b < 16 && b < dd; ++b) {
          long long idx = s + b;
          if (idx < 0 || (uint64_t)idx >= C.se - C.sb) return fail(SAGE_ESTATE, "emulate: slot overrun");
          v[b] = slot[idx];
        }
        if (dv >= written.size() || written[dv]) return fail(SAGE_ESTATE, "emulate: vector landed twice");
        written[dv] = 1;
        memcpy(out + dv * 16, v, 16);
        sum += host_checksum(v, 16, dv * 2);
      }
    }
  }
  for (size_t v = 0; v < written.size(); ++v)
    if (!written[v]) return fail(SAGE_ESTATE, "emulate: vector never landed");
  *checksum = sum;
  return SAGE_OK;
}

// the content checksum the record WILL have once landed (host unpack +
// checksum): a registration-time content key, so a function whose record is
// identical to a resident one can map that segment instead of loading it
int sage_layout_checksum(sage_handle h, const void *packed, uint64_t packed_bytes, uint64_t *checksum) {
  Layout *L = layout_get(h);
  if (!L || !packed || !checksum) return fail(SAGE_EINVAL, "layout_checksum: bad argument");
  if (packed_bytes != L->packed) return fail(SAGE_EINVAL, "layout_checksum: packed size mismatch");
  std::vector<uint8_t> seg(L->seg, 0);
  const uint8_t *pk = static_cast<const uint8_t *>(packed);
  for (const Tensor &T : L->t)
    if (T.len) memcpy(seg.data() + T.dst, pk + T.src, T.len);
  *checksum = host_checksum(seg.data(), L->seg, 0);
  return SAGE_OK;
}

}  // extern "C"
