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
#include "common.h"

namespace sage {

struct Inv {
  int gpu = -1;
  uint64_t id = 0;
  sage_handle slot = 0;
  sage_handle ctx_b = 0, ctx_e = 0, sync_b = 0, sync_e = 0, comp_b = 0, comp_e = 0, ret_b = 0, ret_e = 0;
  sage_handle ro_load = 0, ro_end = 0, in_load = 0, in_end = 0;
  int64_t t_enqueue = 0;
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
std::condition_variable done_cv;
std::deque<Inv *> done_q;          // device-complete, not yet resolved
bool collector_stop = false;
std::thread *collector = nullptr;   // never destroyed while joinable (exit without shutdown)
std::mutex ready_mu;
std::condition_variable ready_cv;
std::deque<uint64_t> ready_q;      // resolved, not yet handed out
}  // namespace

static int resolve_info(Inv *I, sage_invoke_info *out);

static void CUDART_CB on_device_done(void *p) {
  {
    std::lock_guard<std::mutex> lk(done_mu);
    done_q.push_back(static_cast<Inv *>(p));
  }
  done_cv.notify_one();
}

static void collector_main() {
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
                        I->ro_end, I->in_end})
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

}  // namespace sage

using namespace sage;

extern "C" {

int sage_invoke(const sage_invoke_desc *d, sage_handle *inv_out, sage_handle *done_ev, sage_handle *ro_end,
                sage_handle *ctx_end) {
  SAGE_TRY(require_up());
  if (!d || !inv_out || !done_ev) return fail(SAGE_EINVAL, "invoke: null argument");
  if (!gpu_get(d->gpu)) return fail(SAGE_ENODEV, "invoke: bad gpu");
  auto *I = new Inv();
  I->gpu = d->gpu;
  I->id = g_inv_next++;
  {
    std::lock_guard<std::mutex> lk(g_inv_mu);
    g_invs[I->id] = I;
  }
  I->t_enqueue = host_now_us();
  int rc = sage_ctx_acquire(d->gpu, &I->slot);
  Gpu *G = nullptr;
  cudaStream_t s = nullptr;
  if (rc == SAGE_OK) rc = slot_stream(I->slot, &G, &s);
  if (rc == SAGE_OK) cudaSetDevice(G->dev);
  // Stage boundaries on the slot stream are shared: the event that ends one
  // stage also begins the next (one record + one time read instead of two).
  auto rec = [&](sage_handle *h) -> int {
    Event *e;
    SAGE_TRY(event_new(d->gpu, h, &e));
    return event_record(e, s);
  };
  sage_handle last = 0;  // the boundary most recently recorded on s
  // GPU_CTX: bind the function context on the invocation's pooled stream
  // (zero its 64 KiB header: descriptor table, scratch counters)
  if (rc == SAGE_OK && (d->flags & SAGE_INV_CTX)) {
    rc = rec(&I->ctx_b);
    if (rc == SAGE_OK && d->ctx_dptr && d->ctx_bytes) {
      cudaError_t e = cudaMemsetAsync((void *)d->ctx_dptr, 0, std::min<uint64_t>(d->ctx_bytes, 64 << 10), s);
      if (e != cudaSuccess) rc = cuda_fail(e, "ctx bind memset");
    }
    if (rc == SAGE_OK) rc = rec(&I->ctx_e);
    last = I->ctx_e;
  }
  // CPU_LOAD -> GPU_LOAD: the read-only segment ...
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
    rc = sage_segment_load(&L, &I->ro_load, &I->ro_end);
  }
  // ... and the invocation input (identity layout)
  if (rc == SAGE_OK && (d->flags & SAGE_INV_INPUT)) {
    sage_load_desc L{};
    L.gpu = d->gpu;
    L.flags = load_flags(d->in_kind);
    L.dst = d->in_dst;
    L.src = d->in_src;
    L.src_bytes = d->in_bytes;
    rc = sage_segment_load(&L, &I->in_load, &I->in_end);
  }
  // the join before COMPUTE: loads ran on other streams
  sage_handle deps[6];
  int nd = 0;
  if (I->ro_end) deps[nd++] = I->ro_end;
  if (I->in_end) deps[nd++] = I->in_end;
  if (rc == SAGE_OK && (d->flags & SAGE_INV_SYNC)) {
    for (int i = 0; i < d->n_wait && i < 2; ++i) deps[nd++] = d->wait[i];
    rc = last ? event_alias(last, &I->sync_b) : rec(&I->sync_b);
    if (rc == SAGE_OK) rc = wait_events(s, deps, nd);
    if (rc == SAGE_OK) rc = rec(&I->sync_e);
    last = I->sync_e;
  } else if (rc == SAGE_OK && nd) {
    rc = wait_events(s, deps, nd);
    last = 0;  // COMPUTE begins when the joins clear, not at the last boundary
  }
  // COMPUTE
  if (rc == SAGE_OK) rc = last ? event_alias(last, &I->comp_b) : rec(&I->comp_b);
  if (rc == SAGE_OK) rc = launch_timed(G, s, &d->body);
  if (rc == SAGE_OK) rc = rec(&I->comp_e);
  // RETURN
  if (rc == SAGE_OK) rc = return_enqueue(G, s, I->comp_e, d->ret_src, d->ret_dst, d->ret_bytes,
                                        (d->flags & SAGE_INV_RET_HOST) != 0, &I->ret_b, &I->ret_e);
  if (rc == SAGE_OK) {
    // completion notice: on the slot stream, after RETURN (which may have
    // run on a return stream)
    collector_start();
    Event *re = event_get(I->ret_e);
    cudaError_t e = re ? cudaStreamWaitEvent(s, re->ev, 0) : cudaErrorInvalidResourceHandle;
    if (e == cudaSuccess) e = cudaLaunchHostFunc(s, on_device_done, I);
    if (e != cudaSuccess) rc = cuda_fail(e, "invoke completion notice");
  }
  if (rc != SAGE_OK) {
    std::string msg = sage_last_error();
    cudaSetDevice(dev_of(d->gpu));
    cudaDeviceSynchronize();  // error path only: nothing may still reference I
    {
      std::lock_guard<std::mutex> lk(g_inv_mu);
      g_invs.erase(I->id);
    }
    inv_free(I);
    return fail(rc, msg);
  }
  const uint64_t id = I->id;
  *inv_out = make_handle(Kind::Inv, id);
  *done_ev = I->ret_e;
  if (ro_end) *ro_end = I->ro_end;
  if (ctx_end) *ctx_end = I->ctx_e;
  return SAGE_OK;
}

int sage_invoke_collect(sage_handle h, sage_invoke_info *out) {
  Inv *I = inv_get(h);
  if (!I || !out) return fail(SAGE_ESTATE, "invoke_collect: unknown invocation");
  if (I->resolved.load(std::memory_order_acquire) == 1) {
    *out = I->info;
    return I->info.status;
  }
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
    if (sage_event_query(I->ret_e) != SAGE_OK) return fail(SAGE_ESTATE, "invoke_release: still running");
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
