// invoke.cu — one invocation's Parallel stage DAG in one C-ABI call.
//
// Reference: PlanExecution (functions.py:341-433) starts each node when its
// predecessors finish, on the simulator's event loop.  For the Parallel plan
// (functions.py:258-276) the node set is fixed:
//     GPU_CTX  ‖  CPU_LOAD -> GPU_LOAD   ->  [SYNC_WAIT]  ->  COMPUTE  ->  RETURN
// so the host can enqueue the whole DAG at admission: the context bind and
// compute/return on the invocation's pooled stream, the loads on the copy /
// land / direct streams, joined by cudaStreamWaitEvent on their END events.
// One call replaces ~6 ctypes round trips per invocation; one collect call
// returns every stage time, byte count and checksum at completion.
//
// Issue order (the memory daemon's transfer scheduler).  All host->device
// copies of a GPU execute in the order they were enqueued, whatever stream
// they are on (one H2D copy-engine queue; tools/probe_ce.py).  Enqueued at
// admission, a burst's large cold read-only loads therefore hold the PCIe
// H2D direction for milliseconds while no invocation can compute and the
// D2H direction idles.  sage_invoke hands the invocation to an issuer
// thread instead.  The issuer keeps at most `lookahead` bytes of H2D queued
// per GPU and, whenever there is room, enqueues the ready invocation (every
// event it waits on already recorded) with the smallest H2D - D2H balance,
// FIFO among equals, anything older than `max_defer` first: followers of a
// landed segment (balance ~0: their return traffic overlaps the next loads)
// go before the next cold load.  Optionally (SAGE_ISSUE_PIECE_MB) a large
// cold load staged through the ring is enqueued a piece at a time,
// alternating with those followers.  The events handed back
// are created at submit and recorded when the invocation is issued; waits on
// them block until then.  Off the submitting thread, the ~30 us of CUDA
// enqueue per invocation also overlaps the caller's admission work.
//   SAGE_ISSUER=0              enqueue inline (admission order)
//   SAGE_ISSUE_LOOKAHEAD_MB    H2D bytes kept queued per GPU (default 32)
//   SAGE_ISSUE_MAX_DEFER_US    age that overrides the balance order (3000)
//   SAGE_ISSUE_PIECE_MB        > 0: a staged (ring) RO load is enqueued in
//                              pieces of this many MiB, alternating with the
//                              followers of its GPU (0 = whole loads, default:
//                              on the cfg-2 e2e burst 8 / 16 / 24 MiB pieces
//                              measured 22.4 / 18.9 / 19.0 vs 18.6 ms)
#include "common.h"

namespace sage {

struct Inv {
  int gpu = -1;
  uint64_t id = 0;
  sage_handle slot = 0;
  sage_handle ctx_b = 0, ctx_e = 0, sync_b = 0, sync_e = 0, comp_b = 0, comp_e = 0, ret_b = 0, ret_e = 0;
  sage_handle ro_load = 0, ro_end = 0, in_load = 0, in_end = 0;
  // handed out at submit, recorded at issue: RO landed, context bound, done
  sage_handle pre_ro = 0, pre_ctx = 0, pre_done = 0;
  sage_handle hold[6] = {0, 0, 0, 0, 0, 0};   // retained wait events (released after issue)
  sage_invoke_desc d{};                 // the submitted descriptor (waits -> hold)
  int64_t t_enqueue = 0;
  int64_t h2d = 0, d2h = 0;             // PCIe bytes each way (issue order)
  // issue state across pieces (the RO load of a cold leader may be enqueued
  // in pieces, other invocations' copies in between)
  Gpu *G = nullptr;
  cudaStream_t s = nullptr;
  sage_handle last = 0;                 // the stage boundary most recently recorded on s
  LoadCursor *ro_cur = nullptr;         // staged RO load still being enqueued
  std::atomic<bool> issued{false};
  bool ready = false;                   // issuer only: every held event recorded
  std::string err;                      // issue failure (reported by collect)
  sage_invoke_info info{};
  std::atomic<int> resolved{0};   // 1: `info` computed by the completion thread, 2: done (lazy)
};

static std::mutex g_inv_mu;
static std::unordered_map<uint64_t, Inv *> g_invs;
static std::atomic<uint64_t> g_inv_next{1};

// ---------------------------------------------------------- completions ----
// The device tells the host an invocation is done through a host function
// enqueued on its slot stream after RETURN (no polling of per-invocation
// events).  Host functions may not call CUDA, so they only queue the Inv; a
// completion thread resolves every stage time / byte count / checksum off
// the submitting thread, and sage_invoke_ready hands finished handles out in
// completion order.
namespace {
std::mutex done_mu;
// waitables a parked thread may still wait on at process exit live on the heap
// and are never destroyed: glibc's pthread_cond_destroy blocks on waiters
std::condition_variable &done_cv = *new std::condition_variable;
std::deque<Inv *> done_q;          // device-complete, not yet resolved
bool collector_stop = false;
std::thread *collector = nullptr;   // never destroyed while joinable (exit without shutdown)
std::mutex ready_mu;
std::condition_variable &ready_cv = *new std::condition_variable;
std::deque<uint64_t> ready_q;      // resolved, not yet handed out
}  // namespace

static int resolve_info(Inv *I, sage_invoke_info *out);
static void issuer_shutdown();

static void CUDART_CB on_device_done(void *p) {
  {
    std::lock_guard<std::mutex> lk(done_mu);
    done_q.push_back(static_cast<Inv *>(p));
  }
  done_cv.notify_one();
}

static void collector_main() {
  pthread_setname_np(pthread_self(), "sage-complete");
  int dev = -1;
  // resolve stage times here (default) or lazily on collect (SAGE_EAGER_RESOLVE=0):
  // measured 0.8 vs 2.2 ms of drain per 64-invocation burst
  const char *env = getenv("SAGE_EAGER_RESOLVE");
  const bool eager_resolve = !env || atoi(env) != 0;
  for (;;) {
    Inv *I;
    {
      std::unique_lock<std::mutex> lk(done_mu);
      done_cv.wait(lk, [] { return collector_stop || !done_q.empty(); });
      if (done_q.empty()) return;   // stop requested and drained
      I = done_q.front();
      done_q.pop_front();
    }
    if (eager_resolve) {
      if (dev_of(I->gpu) != dev) cudaSetDevice(dev = dev_of(I->gpu));
      int rc = resolve_info(I, &I->info);
      if (rc != SAGE_OK) I->info.status = rc;
      I->resolved.store(1, std::memory_order_release);
    } else {
      I->resolved.store(2, std::memory_order_release);   // complete; times resolved on collect
    }
    {
      std::lock_guard<std::mutex> lk(ready_mu);
      ready_q.push_back(I->id);
    }
    ready_cv.notify_all();
  }
}

static void collector_start() {
  std::lock_guard<std::mutex> lk(done_mu);
  if (collector) return;
  collector_stop = false;
  collector = new std::thread(collector_main);
}

void invoke_shutdown() {
  issuer_shutdown();   // enqueues everything still queued first
  {
    std::lock_guard<std::mutex> lk(done_mu);
    collector_stop = true;
  }
  done_cv.notify_all();
  if (collector) {
    collector->join();
    delete collector;
    collector = nullptr;
  }
  {
    std::lock_guard<std::mutex> lk(ready_mu);
    ready_q.clear();
  }
  std::lock_guard<std::mutex> lk(g_inv_mu);
  for (auto &kv : g_invs) delete kv.second;   // events / loads / slots die with the plane
  g_invs.clear();
}

static Inv *inv_get(sage_handle h) {
  if (handle_kind(h) != Kind::Inv) return nullptr;
  std::lock_guard<std::mutex> lk(g_inv_mu);
  auto it = g_invs.find(h & ((1ull << 56) - 1));
  return it == g_invs.end() ? nullptr : it->second;
}

static uint32_t load_flags(int kind) {
  switch (kind) {
    case SAGE_SRC_PINNED: return SAGE_LOAD_SRC_PINNED;
    case SAGE_SRC_HBM: return SAGE_LOAD_SRC_DEVICE;
    case SAGE_SRC_PEER: return SAGE_LOAD_SRC_PEER;
    default: return 0;
  }
}

static void inv_free(Inv *I) {
  for (sage_handle h : {I->ctx_b, I->ctx_e, I->sync_b, I->sync_e, I->comp_b, I->comp_e, I->ret_b, I->ret_e,
                        I->ro_end, I->in_end, I->pre_ro, I->pre_ctx, I->pre_done, I->hold[0], I->hold[1],
                        I->hold[2], I->hold[3], I->hold[4], I->hold[5]})
    if (h) sage_event_release(h);
  if (I->ro_load) sage_load_release(I->ro_load);
  if (I->in_load) sage_load_release(I->in_load);
  if (I->slot) sage_ctx_release(I->slot);
  delete I;
}

static int resolve_info(Inv *I, sage_invoke_info *out) {
  for (int i = 0; i < 16; ++i) out->t[i] = -1;
  out->host_bytes = out->link_bytes = out->ro_checksum = out->in_checksum = 0;
  out->ro_landed_us = -1;
  auto both = [&](int stage, sage_handle b, sage_handle e) -> int {
    if (!b) return SAGE_OK;
    SAGE_TRY(sage_event_time(b, &out->t[2 * stage]));
    return sage_event_time(e, &out->t[2 * stage + 1]);
  };
  SAGE_TRY(both(3, I->ctx_b, I->ctx_e));
  SAGE_TRY(both(5, I->sync_b, I->sync_e));
  SAGE_TRY(both(6, I->comp_b, I->comp_e));
  SAGE_TRY(both(7, I->ret_b, I->ret_e));
  int64_t cb = -1, ce = -1, gb = -1, ge = -1;
  for (sage_handle lh : {I->ro_load, I->in_load}) {
    if (!lh) continue;
    sage_load_info li;
    SAGE_TRY(sage_load_info_get(lh, &li));
    if (li.cpu_begin_us >= 0) {
      cb = cb < 0 ? li.cpu_begin_us : std::min(cb, li.cpu_begin_us);
      ce = std::max(ce, li.cpu_end_us);
    }
    gb = gb < 0 ? li.gpu_begin_us : std::min(gb, li.gpu_begin_us);
    ge = std::max(ge, li.gpu_end_us);
    out->host_bytes += li.host_bytes;
    out->link_bytes += li.link_bytes;
    if (lh == I->ro_load) {
      out->ro_checksum = li.checksum;
      out->ro_landed_us = li.gpu_end_us;
    } else {
      out->in_checksum = li.checksum;
    }
  }
  // CPU_LOAD: the staging memcpy, or an empty stage at enqueue when the
  // source needed none (pinned / HBM / peer); GPU_LOAD: first copy .. last land
  out->t[4] = cb >= 0 ? cb : I->t_enqueue;
  out->t[5] = ce >= 0 ? ce : I->t_enqueue;
  out->t[8] = gb >= 0 ? gb : I->t_enqueue;
  out->t[9] = ge >= 0 ? ge : I->t_enqueue;
  out->status = SAGE_OK;
  return SAGE_OK;
}

// ---------------------------------------------------------------- issue ----
static bool pcie_kind(int k) { return k == SAGE_SRC_HOST || k == SAGE_SRC_PINNED; }

// submit side: retain the events the invocation waits on, create the events
// handed back, and size its PCIe traffic
static int submit_prepare(Inv *I) {
  sage_invoke_desc &d = I->d;
  for (int i = 0; i < d.n_wait; ++i) {
    SAGE_TRY(event_alias(d.wait[i], &I->hold[i]));
    d.wait[i] = I->hold[i];
  }
  for (int i = 0; i < d.n_ro_wait; ++i) {
    SAGE_TRY(event_alias(d.ro_wait[i], &I->hold[4 + i]));
    d.ro_wait[i] = I->hold[4 + i];
  }
  Event *e;
  SAGE_TRY(event_new(d.gpu, &I->pre_done, &e));
  e->pending.store(true);
  if (d.flags & SAGE_INV_RO) {
    SAGE_TRY(event_new(d.gpu, &I->pre_ro, &e));
    e->pending.store(true);
  }
  if (d.flags & SAGE_INV_CTX) {
    SAGE_TRY(event_new(d.gpu, &I->pre_ctx, &e));
    e->pending.store(true);
  }
  if ((d.flags & SAGE_INV_RO) && pcie_kind(d.ro_kind)) I->h2d += (int64_t)d.ro_src_bytes;
  if ((d.flags & SAGE_INV_INPUT) && pcie_kind(d.in_kind)) I->h2d += (int64_t)d.in_bytes;
  if (d.flags & SAGE_INV_RET_HOST) I->d2h = (int64_t)d.ret_bytes;
  return SAGE_OK;
}

// Enqueue the Parallel DAG of one invocation in three parts: issue_head
// (GPU_CTX, open the RO load), issue_ro_piece (enqueue the staged RO load's
// chunks, all at once or a piece at a time) and issue_tail (input, SYNC_WAIT,
// COMPUTE, RETURN).  Admission order when inline, the issuer's otherwise.
// Stage boundaries on the slot stream are shared: the event that ends one
// stage also begins the next (one record + one time read instead of two).
static int rec_on(Inv *I, sage_handle *h) {
  Event *e;
  SAGE_TRY(event_new(I->d.gpu, h, &e));
  return event_record(e, I->s);
}
static int rec_pre_on(Inv *I, sage_handle pre, sage_handle *h) {
  SAGE_TRY(event_alias(pre, h));
  return event_record(event_get(pre), I->s);
}

// any failure: waiters on this invocation's events must not hang -- record
// whatever was handed out and never reached (followers then fail their own
// checks); nothing may still reference I afterwards
static void issue_abort(Inv *I) {
  const sage_invoke_desc *d = &I->d;
  if (I->ro_cur) {
    segment_load_close(I->ro_cur);
    I->ro_cur = nullptr;
  }
  Gpu *H = I->G ? I->G : gpu_get(d->gpu);
  cudaSetDevice(dev_of(d->gpu));
  for (sage_handle h : {I->pre_ro, I->pre_ctx, I->pre_done}) {
    Event *e = h ? event_get(h) : nullptr;
    if (e && !e->recorded.load() && H) event_record(e, H->aux);
  }
  cudaDeviceSynchronize();
}

static void issue_release_holds(Inv *I) {
  for (int i = 0; i < 6; ++i)
    if (I->hold[i]) { sage_event_release(I->hold[i]); I->hold[i] = 0; }
  I->issued.store(true, std::memory_order_release);
}

static int issue_head(Inv *I) {
  const sage_invoke_desc *d = &I->d;
  int rc = sage_ctx_acquire(d->gpu, &I->slot);
  if (rc == SAGE_OK) rc = slot_stream(I->slot, &I->G, &I->s);
  if (rc == SAGE_OK) cudaSetDevice(I->G->dev);
  I->last = 0;
  // GPU_CTX: bind the function context on the invocation's pooled stream
  // (zero its 64 KiB header: descriptor table, scratch counters)
  if (rc == SAGE_OK && (d->flags & SAGE_INV_CTX)) {
    rc = rec_on(I, &I->ctx_b);
    if (rc == SAGE_OK && d->ctx_dptr && d->ctx_bytes) {
      cudaError_t e = cudaMemsetAsync((void *)d->ctx_dptr, 0, std::min<uint64_t>(d->ctx_bytes, 64 << 10), I->s);
      if (e != cudaSuccess) rc = cuda_fail(e, "ctx bind memset");
    }
    if (rc == SAGE_OK) rc = rec_pre_on(I, I->pre_ctx, &I->ctx_e);
    I->last = I->ctx_e;
  }
  // CPU_LOAD -> GPU_LOAD: the read-only segment (a staged load stays open)
  if (rc == SAGE_OK && (d->flags & SAGE_INV_RO)) {
    sage_load_desc L{};
    L.gpu = d->gpu;
    L.flags = load_flags(d->ro_kind);
    L.dst = d->ro_dst;
    L.layout = d->ro_layout;
    L.src = d->ro_src;
    L.src_bytes = d->ro_src_bytes;
    L.wait = d->ro_wait;
    L.n_wait = d->n_ro_wait;
    L.src_gpu = d->ro_src_gpu;
    rc = segment_load_open(&L, I->pre_ro, &I->ro_cur, &I->ro_load, &I->ro_end);
  }
  return rc;
}

// enqueue up to `budget` bytes of the open RO load; *done once it is complete
static int issue_ro_piece(Inv *I, uint64_t budget, uint64_t *bytes, sage_handle *piece_ev, bool *done) {
  int rc = segment_load_step(I->ro_cur, budget, bytes, piece_ev, done, &I->ro_load, &I->ro_end);
  if (rc != SAGE_OK || *done) {
    segment_load_close(I->ro_cur);
    I->ro_cur = nullptr;
  }
  return rc;
}

static int issue_tail(Inv *I) {
  const sage_invoke_desc *d = &I->d;
  Gpu *G = I->G;
  cudaStream_t s = I->s;
  cudaSetDevice(G->dev);
  int rc = SAGE_OK;
  // ... and the invocation input (identity layout)
  if (d->flags & SAGE_INV_INPUT) {
    sage_load_desc L{};
    L.gpu = d->gpu;
    L.flags = load_flags(d->in_kind) | ((d->flags & SAGE_INV_VERIFY_INPUT) ? 0u : SAGE_LOAD_NO_VERIFY);
    L.dst = d->in_dst;
    L.src = d->in_src;
    L.src_bytes = d->in_bytes;
    rc = segment_load(&L, &I->in_load, &I->in_end, 0);
  }
  // the join before COMPUTE: loads ran on other streams
  sage_handle deps[8];
  int nd = 0;
  if (I->ro_end) deps[nd++] = I->ro_end;
  if (I->in_end) deps[nd++] = I->in_end;
  // leader tokens (SYNC_WAIT) and the compute-gate predecessor: COMPUTE waits
  // on all of them; only a SYNC_WAIT plan node records the stage
  for (int i = 0; i < d->n_wait && i < 4; ++i) deps[nd++] = d->wait[i];
  sage_handle last = I->last;
  if (rc == SAGE_OK && (d->flags & SAGE_INV_SYNC)) {
    rc = last ? event_alias(last, &I->sync_b) : rec_on(I, &I->sync_b);
    if (rc == SAGE_OK) rc = wait_events(s, deps, nd);
    if (rc == SAGE_OK) rc = rec_on(I, &I->sync_e);
    last = I->sync_e;
  } else if (rc == SAGE_OK && nd) {
    rc = wait_events(s, deps, nd);
    last = 0;  // COMPUTE begins when the joins clear, not at the last boundary
  }
  // COMPUTE
  if (rc == SAGE_OK) rc = last ? event_alias(last, &I->comp_b) : rec_on(I, &I->comp_b);
  if (rc == SAGE_OK) rc = launch_timed(G, s, &d->body);
  if (rc == SAGE_OK) rc = rec_on(I, &I->comp_e);
  // RETURN
  if (rc == SAGE_OK) rc = return_enqueue(G, s, I->comp_e, d->ret_src, d->ret_dst, d->ret_bytes,
                                        (d->flags & SAGE_INV_RET_HOST) != 0, &I->ret_b, &I->ret_e, I->pre_done);
  if (rc == SAGE_OK) {
    // the completion notice waits on RETURN (which may have run on a return
    // stream); issue_notify launches it
    Event *re = event_get(I->ret_e);
    cudaError_t e = re ? cudaStreamWaitEvent(s, re->ev, 0) : cudaErrorInvalidResourceHandle;
    if (e != cudaSuccess) rc = cuda_fail(e, "invoke completion wait");
  }
  return rc;
}

// the whole invocation at once (inline path)
static int issue(Inv *I) {
  int rc = issue_head(I);
  if (rc == SAGE_OK && I->ro_cur) {
    bool done = false;
    rc = issue_ro_piece(I, UINT64_MAX, nullptr, nullptr, &done);
  }
  if (rc == SAGE_OK) rc = issue_tail(I);
  if (rc != SAGE_OK) issue_abort(I);
  issue_release_holds(I);
  return rc;
}

// the device tells the completion thread when the invocation is done: a host
// function on the slot stream.  The last touch of I by the issuing thread --
// after this the caller may collect and release it at any time.
static int issue_notify(Inv *I) {
  Gpu *G;
  cudaStream_t s;
  SAGE_TRY(slot_stream(I->slot, &G, &s));
  SAGE_CUDA(cudaLaunchHostFunc(s, on_device_done, I));
  return SAGE_OK;
}

namespace {
std::mutex iss_mu;
std::condition_variable &iss_cv = *new std::condition_variable;       // work arrived / stop
std::condition_variable &iss_idle_cv = *new std::condition_variable;  // something was issued
std::deque<Inv *> iss_q;              // submitted, not yet issued (submit order)
std::deque<Inv *> iss_open;           // head issued, staged RO load still being enqueued
int iss_busy = 0;                     // being issued right now
bool iss_stop = false;
std::thread *issuer = nullptr;
struct Flight { sage_handle ev; int64_t bytes; int gpu; };
}  // namespace

static bool env_flag(const char *name, bool dflt) {
  const char *e = getenv(name);
  return e ? atoi(e) != 0 : dflt;
}
static int64_t env_i64(const char *name, int64_t dflt) {
  const char *e = getenv(name);
  return e ? atoll(e) : dflt;
}
static bool issuer_enabled() {
  static const bool on = env_flag("SAGE_ISSUER", true);
  return on;
}

static bool inv_ready(Inv *I) {
  if (I->ready) return true;   // readiness never reverts: checked once per hold
  for (sage_handle h : I->hold) {
    if (!h) continue;
    Event *e = event_get(h);
    if (!e) continue;
    if (e->ev ? !e->recorded.load(std::memory_order_acquire) : !e->host_done.load(std::memory_order_acquire))
      return false;
  }
  I->ready = true;
  return true;
}

// an invocation the issuer could not enqueue: complete it as failed
static void complete_failed(Inv *I, int rc, const std::string &msg) {
  for (int i = 0; i < 16; ++i) I->info.t[i] = -1;
  I->info.status = rc;
  I->err = msg;
  I->resolved.store(1, std::memory_order_release);
  {
    std::lock_guard<std::mutex> lk(ready_mu);
    ready_q.push_back(I->id);
  }
  ready_cv.notify_all();
  fprintf(stderr, "sage: invocation %llu failed at issue: %s\n", (unsigned long long)I->id, msg.c_str());
}

// add an H2D flight (bytes in the copy queue until `ev` completes)
static void flight_add(std::deque<Flight> &flights, sage_handle ev_alias_of, int64_t bytes, int gpu) {
  Flight f{0, bytes, gpu};
  if (event_alias(ev_alias_of, &f.ev) == SAGE_OK) flights.push_back(f);
}

// Issue one step of invocation I: a fresh invocation gets its head (and the
// first piece of a staged RO load); an invocation with an open RO load gets
// its next piece.  Returns true when I is fully issued (or failed).
static bool issue_step(Inv *I, int64_t piece, std::deque<Flight> &flights) {
  NvtxRange nv("sage.issue");
  const sage_invoke_desc &d = I->d;
  const bool fresh = I->G == nullptr && !I->ro_cur;
  int rc = SAGE_OK;
  if (fresh) {
    rc = issue_head(I);
    if (rc == SAGE_OK && !I->ro_cur && I->ro_end && (d.flags & SAGE_INV_RO) && pcie_kind(d.ro_kind))
      flight_add(flights, I->ro_end, (int64_t)d.ro_src_bytes, I->gpu);
  }
  if (rc == SAGE_OK && I->ro_cur) {
    uint64_t moved = 0;
    sage_handle pev = 0;
    bool done = false;
    rc = issue_ro_piece(I, piece > 0 ? (uint64_t)piece : UINT64_MAX, &moved, &pev, &done);
    if (pev) {
      if (moved) {
        Flight f{pev, (int64_t)moved, I->gpu};
        flights.push_back(f);
      } else {
        sage_event_release(pev);
      }
    }
    if (rc == SAGE_OK && !done) return false;   // more pieces to come
  }
  if (rc == SAGE_OK) {
    rc = issue_tail(I);
    if (rc == SAGE_OK && I->in_end && (d.flags & SAGE_INV_INPUT) && pcie_kind(d.in_kind))
      flight_add(flights, I->in_end, (int64_t)d.in_bytes, I->gpu);
  }
  if (rc != SAGE_OK) issue_abort(I);
  issue_release_holds(I);
  if (rc == SAGE_OK) rc = issue_notify(I);
  if (rc != SAGE_OK) complete_failed(I, rc, sage_last_error());   // (I may be released from here on)
  return true;
}

static constexpr int kIssueScan = 256;

static void issuer_main() {
  pthread_setname_np(pthread_self(), "sage-issuer");
  const int64_t lookahead = env_i64("SAGE_ISSUE_LOOKAHEAD_MB", 32) << 20;
  const int64_t max_defer = env_i64("SAGE_ISSUE_MAX_DEFER_US", 3000);
  const int64_t piece = env_i64("SAGE_ISSUE_PIECE_MB", 0) << 20;
  const bool tiebreak_d2h = env_i64("SAGE_ISSUE_BIG_RETURN_FIRST", 1) != 0;
  std::deque<Flight> flights;   // H2D queued by this thread, not yet landed
  std::vector<int64_t> pending;
  std::vector<char> piece_turn; // per GPU: the next slot goes to an open staged load
  int rr = 0;                   // GPU the next pick starts looking at
  for (;;) {
    // retire landed H2D (issuer-only state, no lock)
    pending.assign(st.gpus.size() + 1, 0);
    if (piece_turn.size() < pending.size()) piece_turn.resize(pending.size(), 1);
    for (auto it = flights.begin(); it != flights.end();) {
      if (sage_event_query(it->ev) != SAGE_ENOTREADY) {
        sage_event_release(it->ev);
        it = flights.erase(it);
      } else {
        pending[it->gpu] += it->bytes;
        ++it;
      }
    }
    Inv *pick = nullptr;
    {
      std::unique_lock<std::mutex> lk(iss_mu);
      if (iss_q.empty() && iss_open.empty()) {
        if (iss_stop) break;
        if (flights.empty()) {
          iss_cv.wait(lk, [] { return iss_stop || !iss_q.empty(); });
          continue;
        }
        iss_cv.wait_for(lk, std::chrono::microseconds(50));
        continue;
      }
      const int64_t now = host_now_us();
      auto room = [&](int gpu) { return pending[gpu] <= 0 || pending[gpu] < lookahead; };
      // Per GPU, in rotation: an open staged load alternates with the
      // followers (ready invocations whose H2D - D2H balance is within one
      // piece: their returns keep D2H busy while the load crosses H2D);
      // with no open load, the smallest waiting cold load opens next (its
      // followers become ready as soon as it is enqueued), else the
      // follower with the smallest balance (FIFO among equals, overdue first).
      // SAGE_ISSUE_PIECE_MB=0: whole loads, balance order only.
      const int ng = (int)pending.size();
      for (int k = 0; k < ng && !pick; ++k) {
        const int g = (rr + k) % ng;
        // a full PCIe queue holds back everything that adds H2D bytes;
        // invocations without H2D (HBM-resident sources) still go
        const bool has_room = room(g);
        auto open = iss_open.end();
        if (has_room)
          for (auto it = iss_open.begin(); it != iss_open.end(); ++it)
            if ((*it)->gpu == g) { open = it; break; }
        auto fol = iss_q.end(), cold = iss_q.end();
        int64_t fol_key = INT64_MAX, cold_key = INT64_MAX, fol_d2h = -1;
        bool fol_overdue = false;
        // the pick looks at the oldest kIssueScan waiting invocations, and
        // further only until it has a candidate: a backlog of thousands
        // (offered load above capacity) must not make every pick O(backlog)
        // -- that collapsed cfg-3 at 4000/s offered -- while a window of
        // followers whose leader waits further back cannot stall the queue
        int scanned = 0;
        for (auto it = iss_q.begin(); it != iss_q.end(); ++it, ++scanned) {
          if (scanned >= kIssueScan && (fol != iss_q.end() || cold != iss_q.end())) break;
          Inv *I = *it;
          if (I->gpu != g || !inv_ready(I)) continue;
          if (I->h2d > 0 && !has_room) continue;
          const int64_t key = I->h2d - I->d2h;
          if (piece > 0 && key > piece) {
            if (key < cold_key) { cold_key = key; cold = it; }
          } else if (!fol_overdue) {
            if (now - I->t_enqueue >= max_defer) { fol = it; fol_overdue = true; }
            else if (key < fol_key || (key == fol_key && tiebreak_d2h && I->d2h > fol_d2h)) {
              // equal balance: the larger return first, so a burst ends on
              // small returns (a big D2H alone at the end idles the H2D lane)
              fol_key = key; fol_d2h = I->d2h; fol = it;
            }
          }
        }
        if (open != iss_open.end()) {
          if (!piece_turn[g] && fol != iss_q.end()) {
            pick = *fol;
            iss_q.erase(fol);
            piece_turn[g] = 1;
          } else {
            pick = *open;
            iss_open.erase(open);
            piece_turn[g] = 0;
          }
        } else if (cold != iss_q.end()) {
          pick = *cold;
          iss_q.erase(cold);
          piece_turn[g] = 0;
        } else if (fol != iss_q.end()) {
          pick = *fol;
          iss_q.erase(fol);
          piece_turn[g] = 1;
        }
      }
      if (!pick) {
        iss_cv.wait_for(lk, std::chrono::microseconds(20));
        continue;
      }
      rr = (pick->gpu + 1) % ng;
      ++iss_busy;
    }
    const bool finished = issue_step(pick, piece, flights);
    {
      std::lock_guard<std::mutex> lk(iss_mu);
      if (!finished) iss_open.push_back(pick);
      --iss_busy;
    }
    iss_idle_cv.notify_all();
  }
  for (auto &f : flights) sage_event_release(f.ev);
}

static void issuer_submit(Inv *I) {
  {
    std::lock_guard<std::mutex> lk(iss_mu);
    if (!issuer) {
      iss_stop = false;
      issuer = new std::thread(issuer_main);
    }
    iss_q.push_back(I);
  }
  iss_cv.notify_one();
}

void issuer_drain(int gpu) {
  std::unique_lock<std::mutex> lk(iss_mu);
  iss_idle_cv.wait(lk, [gpu] {
    if (iss_busy) return false;
    for (Inv *I : iss_q)
      if (gpu < 0 || I->gpu == gpu) return false;
    for (Inv *I : iss_open)
      if (gpu < 0 || I->gpu == gpu) return false;
    return true;
  });
}

static void issuer_shutdown() {
  {
    std::lock_guard<std::mutex> lk(iss_mu);
    iss_stop = true;
  }
  iss_cv.notify_all();
  if (issuer) {
    issuer->join();
    delete issuer;
    issuer = nullptr;
  }
}

}  // namespace sage

using namespace sage;

extern "C" {

int sage_invoke(const sage_invoke_desc *d, sage_handle *inv_out, sage_handle *done_ev, sage_handle *ro_end,
                sage_handle *ctx_end) {
  SAGE_TRY(require_up());
  if (!d || !inv_out || !done_ev) return fail(SAGE_EINVAL, "invoke: null argument");
  if (!gpu_get(d->gpu)) return fail(SAGE_ENODEV, "invoke: bad gpu");
  if (d->n_wait < 0 || d->n_wait > 4 || d->n_ro_wait < 0 || d->n_ro_wait > 2)
    return fail(SAGE_EINVAL, "invoke: at most four SYNC_WAIT and two RO wait events");
  auto *I = new Inv();
  I->gpu = d->gpu;
  I->id = g_inv_next++;
  I->d = *d;
  I->t_enqueue = host_now_us();
  int rc = submit_prepare(I);
  if (rc != SAGE_OK) {
    std::string msg = sage_last_error();
    inv_free(I);
    return fail(rc, msg);
  }
  {
    std::lock_guard<std::mutex> lk(g_inv_mu);
    g_invs[I->id] = I;
  }
  *inv_out = make_handle(Kind::Inv, I->id);
  *done_ev = I->pre_done;
  if (ro_end) *ro_end = I->pre_ro;
  if (ctx_end) *ctx_end = I->pre_ctx;
  collector_start();
  if (issuer_enabled()) {
    issuer_submit(I);
    return SAGE_OK;
  }
  rc = issue(I);
  if (rc == SAGE_OK) rc = issue_notify(I);
  if (rc != SAGE_OK) {
    std::string msg = sage_last_error();
    {
      std::lock_guard<std::mutex> lk(g_inv_mu);
      g_invs.erase(I->id);
    }
    inv_free(I);
    return fail(rc, msg);
  }
  return SAGE_OK;
}

int sage_invoke_collect(sage_handle h, sage_invoke_info *out) {
  Inv *I = inv_get(h);
  if (!I || !out) return fail(SAGE_ESTATE, "invoke_collect: unknown invocation");
  if (I->resolved.load(std::memory_order_acquire) == 1) {
    *out = I->info;
    if (I->info.status != SAGE_OK && !I->err.empty()) return fail(I->info.status, I->err);
    return I->info.status;
  }
  if (!I->issued.load(std::memory_order_acquire) || !I->ret_e) return SAGE_ENOTREADY;
  int rc = sage_event_query(I->ret_e);
  if (rc != SAGE_OK) return rc;
  return resolve_info(I, out);
}

int sage_invoke_ready(sage_handle *out, int max, int64_t timeout_us) {
  if (max < 0 || (max > 0 && !out)) return fail(SAGE_EINVAL, "invoke_ready: bad arguments");
  std::unique_lock<std::mutex> lk(ready_mu);
  if (ready_q.empty() && timeout_us > 0)
    ready_cv.wait_for(lk, std::chrono::microseconds(timeout_us), [] { return !ready_q.empty(); });
  int n = 0;
  while (n < max && !ready_q.empty()) {
    out[n++] = make_handle(Kind::Inv, ready_q.front());
    ready_q.pop_front();
  }
  return n;
}

int sage_invoke_release(sage_handle h) {
  Inv *I = inv_get(h);
  if (I && !I->resolved.load(std::memory_order_acquire)) {
    // the completion thread still owns I: only a finished invocation may go
    if (!I->issued.load(std::memory_order_acquire) || !I->ret_e || sage_event_query(I->ret_e) != SAGE_OK)
      return fail(SAGE_ESTATE, "invoke_release: still running");
    std::unique_lock<std::mutex> lk(ready_mu);
    ready_cv.wait(lk, [I] { return I->resolved.load(std::memory_order_acquire) != 0; });
  }
  if (I) {   // released without being handed out (collect-by-handle callers)
    std::lock_guard<std::mutex> lk(ready_mu);
    for (auto it = ready_q.begin(); it != ready_q.end(); ++it)
      if (*it == I->id) { ready_q.erase(it); break; }
  }
  {
    std::lock_guard<std::mutex> lk(g_inv_mu);
    auto it = g_invs.find(h & ((1ull << 56) - 1));
    if (handle_kind(h) != Kind::Inv || it == g_invs.end())
      return fail(SAGE_ESTATE, "double or unknown invocation release");
    I = it->second;
    g_invs.erase(it);
  }
  inv_free(I);
  return SAGE_OK;
}

}  // extern "C"
