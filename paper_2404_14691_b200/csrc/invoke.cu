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
  sage_handle slot = 0;
  sage_handle ctx_b = 0, ctx_e = 0, sync_b = 0, sync_e = 0, comp_b = 0, comp_e = 0, ret_b = 0, ret_e = 0;
  sage_handle ro_load = 0, ro_end = 0, in_load = 0, in_end = 0;
  int64_t t_enqueue = 0;
};

static std::mutex g_inv_mu;
static std::unordered_map<uint64_t, Inv *> g_invs;
static std::atomic<uint64_t> g_inv_next{1};

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
  if (rc != SAGE_OK) {
    std::string msg = sage_last_error();
    Gpu *G = gpu_get(d->gpu);
    cudaSetDevice(dev_of(d->gpu));
    cudaDeviceSynchronize();  // error path only: nothing may still reference I
    (void)G;
    inv_free(I);
    return fail(rc, msg);
  }
  uint64_t id = g_inv_next++;
  {
    std::lock_guard<std::mutex> lk(g_inv_mu);
    g_invs[id] = I;
  }
  *inv_out = make_handle(Kind::Inv, id);
  *done_ev = I->ret_e;
  if (ro_end) *ro_end = I->ro_end;
  if (ctx_end) *ctx_end = I->ctx_e;
  return SAGE_OK;
}

int sage_invoke_collect(sage_handle h, sage_invoke_info *out) {
  Inv *I = inv_get(h);
  if (!I || !out) return fail(SAGE_ESTATE, "invoke_collect: unknown invocation");
  int rc = sage_event_query(I->ret_e);
  if (rc != SAGE_OK) return rc;
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

int sage_invoke_release(sage_handle h) {
  Inv *I = nullptr;
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
