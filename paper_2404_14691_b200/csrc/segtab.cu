// segtab.cu — the sharing manager's resident table (host code, no device calls
// except token event queries).
//
// The reference keeps one ResidentFunction per (function, GPU) in a Python dict
// and walks it per admission (sharing.py:103-335).  Here the table is native:
// one record per resident holding the refcount, the held resources, the two
// leader tokens, the decay stage and its deadline and the RO content checksum;
// admission, release, the timed decay, victim choice and
// the invariant sweep are single calls.  The caller (sharing.py) owns the
// ledger allocations and the engine timer objects and executes the steps this
// table hands back (allocate the RO cache, free RO after its D2H, free the
// context segment, evict ...).  The behaviour restated here, rule by rule:
//   warmth      held RO (or none needed) + held ctx -> Stage1Hot; ctx -> Stage2;
//               CPU ctx -> Stage3; container -> Stage4; else Cold (sharing.py:115-125)
//   deltas      a shared RO segment is allocated by the admission that finds
//               none (RO sharing on, RO > 0); a shared context likewise (:126-134)
//   leaders     whoever allocates creates the token, not ready until its
//               stage END (or the last release) (:157-172, policies.py:316-320)
//   RO loads    counted per (fn, GPU) unless Stage1Hot, kept across eviction (:174-175)
//   release     refcount; the last one readies both tokens and enters Stage1
//               (multi-stage exit), the flat keep-alive, or evicts (:181-196)
//   decay       Stage1 -> 2 caches RO on the host and frees it on the GPU, 2 -> 3
//               frees the context, 3 -> 4 drops the cache and the CPU ctx,
//               4 -> evicted (:217-246); each step arms the next interval
//   victims     under pressure, Stage2 residents before Stage1 ones (the most
//               decayed first), least recently active first, never an active
//               resident or the admitting function, only holders of GPU
//               segments (:271-298)
// Addition: a content index (checksum -> residents holding landed RO) so a
// function whose record has identical content can map a resident segment
// instead of loading (north_star: "deduplicate and verify shared segments").
#include "common.h"

#include <algorithm>
#include <map>

namespace sage {
namespace {

enum : int { W_COLD = 0, W_STAGE4 = 1, W_STAGE3 = 2, W_STAGE2 = 3, W_STAGE1_HOT = 4 };
enum : int { R_ACTIVE = 0, R_STAGE1 = 1, R_STAGE2 = 2, R_STAGE3 = 3, R_STAGE4 = 4 };

struct Tok {
  bool live = false;     // token exists (the segment is held)
  bool ready = false;
  sage_handle ev = 0;    // leader's stage END event (device); 0 = none attached
  bool is_ready() {
    if (!live) return false;
    if (ready) return true;
    if (ev) {
      Event *e = event_get(ev);   // a released handle only names a finished stage
      if (!e || event_query(e) != SAGE_ENOTREADY) {
        ready = true;             // sticky
        ev = 0;
      }
    }
    return ready;
  }
};

struct Res {
  uint64_t id = 0;
  int32_t fn = -1;
  int gpu = -1;
  int state = R_ACTIVE;
  uint32_t active = 0;
  bool has_ro_fn = false;           // the function has RO data (ro_mem_mb > 0)
  bool ro = false, ctx = false, cache = false, cpu_ctx = true, container = true;
  uint64_t ro_bytes = 0, ctx_bytes = 0;
  Tok ro_tok, ctx_tok;
  int64_t last_activity = 0;
  int64_t deadline = -1;            // armed decay timer
  uint32_t gen = 0;                 // timer generation (bumped on every arm / cancel)
  bool has_cs = false;
  uint64_t cs = 0;
};

struct Table {
  std::mutex mu;
  int n_gpus = 1;
  uint32_t flags = 0;
  int64_t keep_alive = 0, iv[4] = {0, 0, 0, 0};
  uint64_t next_id = 1;
  std::map<std::pair<int32_t, int>, Res *> by_key;
  std::map<uint64_t, Res *> by_id;                      // id order = admission order of first use
  std::map<std::pair<int32_t, int>, uint32_t> ro_loads;
  std::multimap<uint64_t, uint64_t> content;            // checksum -> resident id
};

std::mutex g_tabs_mu;
std::unordered_map<uint64_t, Table *> g_tabs;
uint64_t g_tab_next = 1;
constexpr uint8_t kTabKind = 0x21;

Table *tab_get(sage_handle h) {
  if ((h >> 56) != kTabKind) return nullptr;
  std::lock_guard<std::mutex> lk(g_tabs_mu);
  auto it = g_tabs.find(h & ((1ull << 56) - 1));
  return it == g_tabs.end() ? nullptr : it->second;
}

int warmth_of(Res *r, bool has_ro_fn) {
  if (!r) return W_COLD;
  if ((!has_ro_fn || r->ro) && r->ctx) return W_STAGE1_HOT;
  if (r->ctx) return W_STAGE2;
  if (r->cpu_ctx) return W_STAGE3;
  if (r->container) return W_STAGE4;
  return W_COLD;
}

void fill_grant(Table *T, Res *r, uint64_t ro_bytes, uint64_t ctx_bytes, bool has_ro_fn, sage_share_grant *g) {
  memset(g, 0, sizeof *g);
  g->warmth = warmth_of(r, has_ro_fn);
  const bool ro_held = r && r->ro, ctx_held = r && r->ctx;
  g->shared_ro = ro_held;
  g->shared_ctx = ctx_held;
  g->wait_ro = ro_held && !r->ro_tok.is_ready();
  g->wait_ctx = ctx_held && !r->ctx_tok.is_ready();
  if ((T->flags & SAGE_SHARE_RO) && has_ro_fn && !ro_held) g->alloc_ro = ro_bytes;
  if ((T->flags & SAGE_SHARE_CTX) && !ctx_held) g->alloc_ctx = ctx_bytes;
  g->resident = r ? r->id : 0;
}

void arm(Res *r, int state, int64_t now, int64_t interval, sage_share_step *out) {
  r->state = state;
  r->deadline = now + interval;
  r->gen++;
  out->actions |= SAGE_STEP_ARM;
  out->deadline_us = r->deadline;
  out->timer_gen = r->gen;
}

void cancel_timer(Res *r, uint8_t *cancelled) {
  if (r->deadline >= 0) {
    r->deadline = -1;
    r->gen++;
    if (cancelled) *cancelled = 1;
  }
}

void drop_content(Table *T, Res *r) {
  if (!r->has_cs) return;
  auto range = T->content.equal_range(r->cs);
  for (auto it = range.first; it != range.second; ++it)
    if (it->second == r->id) {
      T->content.erase(it);
      break;
    }
  r->has_cs = false;
}

void drop_ro(Table *T, Res *r) {
  r->ro = false;
  r->ro_tok = Tok{};
  drop_content(T, r);
}

void evict(Table *T, Res *r, sage_share_step *out) {
  cancel_timer(r, nullptr);
  if (r->ro) {
    drop_ro(T, r);
    out->actions |= SAGE_STEP_FREE_RO;
  }
  if (r->ctx) {
    r->ctx = false;
    r->ctx_tok = Tok{};
    out->actions |= SAGE_STEP_FREE_CTX;
  }
  if (r->cache) {
    r->cache = false;
    out->actions |= SAGE_STEP_DROP_CACHE;
  }
  r->cpu_ctx = r->container = false;
  out->actions |= SAGE_STEP_EVICT | SAGE_STEP_GPU_FREED;
  T->by_key.erase({r->fn, r->gpu});
  T->by_id.erase(r->id);
  delete r;
}

// one decay step of a resident that is not active (sharing.py:217-246)
void demote_once(Table *T, Res *r, int64_t now, sage_share_step *out) {
  out->resident = r->id;
  out->state_before = r->state;
  switch (r->state) {
    case R_STAGE1:
      if (!r->cache && r->has_ro_fn) {
        r->cache = true;
        out->actions |= SAGE_STEP_CACHE_RO;   // allocate the host copy (+ D2H while RO is held)
      }
      if (r->ro) {
        drop_ro(T, r);
        out->actions |= SAGE_STEP_FREE_RO | SAGE_STEP_GPU_FREED;
      }
      arm(r, R_STAGE2, now, T->iv[1], out);
      break;
    case R_STAGE2:
      if (r->ctx) {
        r->ctx = false;
        r->ctx_tok = Tok{};
        out->actions |= SAGE_STEP_FREE_CTX | SAGE_STEP_GPU_FREED;
      }
      arm(r, R_STAGE3, now, T->iv[2], out);
      break;
    case R_STAGE3:
      if (r->cache) {
        r->cache = false;
        out->actions |= SAGE_STEP_DROP_CACHE;
      }
      r->cpu_ctx = false;
      arm(r, R_STAGE4, now, T->iv[3], out);
      break;
    case R_STAGE4:
      evict(T, r, out);
      return;
    default:
      break;
  }
  out->state_after = r->state;
}

int check_one(Table *T, Res *r, std::string *why) {
  auto bad = [&](const char *what) {
    *why = "resident fn " + std::to_string(r->fn) + " gpu " + std::to_string(r->gpu) + ": " + what;
    return SAGE_ESTATE;
  };
  const bool ro_expected = (T->flags & SAGE_SHARE_RO) && r->has_ro_fn;
  const bool ctx_expected = (T->flags & SAGE_SHARE_CTX) != 0;
  const bool staged_cache = r->has_ro_fn && (T->flags & SAGE_SHARE_MULTI_STAGE);
  if (r->state == R_ACTIVE) {
    if (r->active < 1 || r->deadline >= 0) return bad("active without users or with a timer");
  } else if (r->active != 0 || r->deadline < 0) {
    return bad("decaying with users or without a timer");
  }
  switch (r->state) {
    case R_ACTIVE:
    case R_STAGE1:
      if (r->ro != ro_expected) return bad("RO segment held/not held against the policy");
      if (r->ctx != ctx_expected) return bad("context segment held/not held against the policy");
      if (!r->cpu_ctx || !r->container) return bad("host state dropped while warm");
      break;
    case R_STAGE2:
      if (r->ro) return bad("Stage2 still holds RO on the GPU");
      if (r->ctx != ctx_expected) return bad("Stage2 context against the policy");
      if (r->cache != staged_cache) return bad("Stage2 host RO cache");
      if (!r->cpu_ctx || !r->container) return bad("Stage2 host state dropped");
      break;
    case R_STAGE3:
      if (r->ro || r->ctx) return bad("Stage3 holds GPU segments");
      if (r->cache != staged_cache) return bad("Stage3 host RO cache");
      if (!r->cpu_ctx || !r->container) return bad("Stage3 host state dropped");
      break;
    case R_STAGE4:
      if (r->ro || r->ctx || r->cache) return bad("Stage4 holds segments");
      if (r->cpu_ctx || !r->container) return bad("Stage4 CPU context / container");
      break;
  }
  if (r->has_cs && !r->ro) return bad("content index names a resident without RO");
  return SAGE_OK;
}

}  // namespace
}  // namespace sage

using namespace sage;

extern "C" int sage_share_create(int n_gpus, uint32_t flags, int64_t keep_alive_us, const int64_t intervals_us[4],
                                 sage_handle *tab) {
  if (n_gpus < 1 || !tab || !intervals_us) return fail(SAGE_EINVAL, "share_create: bad arguments");
  for (int i = 0; i < 4; ++i)
    if (intervals_us[i] < 0) return fail(SAGE_EINVAL, "share_create: negative stage interval");
  auto *T = new Table();
  T->n_gpus = n_gpus;
  T->flags = flags;
  T->keep_alive = keep_alive_us;
  for (int i = 0; i < 4; ++i) T->iv[i] = intervals_us[i];
  std::lock_guard<std::mutex> lk(g_tabs_mu);
  const uint64_t id = g_tab_next++;
  g_tabs[id] = T;
  *tab = ((uint64_t)kTabKind << 56) | id;
  return SAGE_OK;
}

extern "C" int sage_share_destroy(sage_handle tab) {
  Table *T;
  {
    std::lock_guard<std::mutex> lk(g_tabs_mu);
    auto it = g_tabs.find(tab & ((1ull << 56) - 1));
    if ((tab >> 56) != kTabKind || it == g_tabs.end()) return fail(SAGE_ESTATE, "share_destroy: unknown table");
    T = it->second;
    g_tabs.erase(it);
  }
  for (auto &kv : T->by_id) delete kv.second;
  delete T;
  return SAGE_OK;
}

#define TAB_OR_FAIL(T, h)                                              \
  Table *T = tab_get(h);                                               \
  if (!T) return fail(SAGE_ESTATE, "sharing table: unknown handle"); \
  std::lock_guard<std::mutex> lk__(T->mu)

extern "C" int sage_share_preview(sage_handle tab, int32_t fn, int gpu, uint64_t ro_bytes, uint64_t ctx_bytes,
                                  uint32_t fn_flags, sage_share_grant *g) {
  TAB_OR_FAIL(T, tab);
  if (!g || gpu < 0 || gpu >= T->n_gpus) return fail(SAGE_EINVAL, "share_preview: bad arguments");
  auto it = T->by_key.find({fn, gpu});
  fill_grant(T, it == T->by_key.end() ? nullptr : it->second, ro_bytes, ctx_bytes, fn_flags & SAGE_FN_HAS_RO, g);
  return SAGE_OK;
}

static void admit_locked(Table *T, Res *r, int32_t fn, int gpu, bool has_ro, int64_t now_us,
                         sage_share_grant *g) {
  if (!r) {
    r = new Res();
    r->id = T->next_id++;
    r->fn = fn;
    r->gpu = gpu;
    r->has_ro_fn = has_ro;
    T->by_key[{fn, gpu}] = r;
    T->by_id[r->id] = r;
    g->new_resident = 1;
  }
  cancel_timer(r, &g->timer_cancelled);
  r->state = R_ACTIVE;
  r->active++;
  r->cpu_ctx = r->container = true;
  r->last_activity = now_us;
  if (g->alloc_ro) {
    r->ro = true;
    r->ro_bytes = g->alloc_ro;
    r->ro_tok = Tok{true, false, 0};
    drop_content(T, r);
    g->leader_ro = 1;
  }
  if (g->alloc_ctx) {
    r->ctx = true;
    r->ctx_bytes = g->alloc_ctx;
    r->ctx_tok = Tok{true, false, 0};
    g->leader_ctx = 1;
  }
  if (has_ro && g->warmth != W_STAGE1_HOT) T->ro_loads[{fn, gpu}]++;
  g->resident = r->id;
}

extern "C" int sage_share_admit(sage_handle tab, int32_t fn, int gpu, uint64_t ro_bytes, uint64_t ctx_bytes,
                                uint32_t fn_flags, int64_t now_us, sage_share_grant *g) {
  TAB_OR_FAIL(T, tab);
  if (!g || gpu < 0 || gpu >= T->n_gpus) return fail(SAGE_EINVAL, "share_admit: bad arguments");
  const bool has_ro = fn_flags & SAGE_FN_HAS_RO;
  auto it = T->by_key.find({fn, gpu});
  Res *r = it == T->by_key.end() ? nullptr : it->second;
  fill_grant(T, r, ro_bytes, ctx_bytes, has_ro, g);
  admit_locked(T, r, fn, gpu, has_ro, now_us, g);
  return SAGE_OK;
}

// preview + capacity check + admit under one lock: the admission's own
// shared segments plus `extra_bytes` of private ones, rounded up to
// `granularity` as one request, must fit in `avail_bytes` (< 0: unlimited).
// Refused: SAGE_ENOMEM with the preview in *g and no state change.
// SAGE_ADMIT_DEFER_RO_LEADER: an admission that would lead a new RO segment
// returns SAGE_ADMIT_DEFERRED (> 0) with the preview instead (the caller looks
// for identical content first).
extern "C" int sage_share_admit_within(sage_handle tab, int32_t fn, int gpu, uint64_t ro_bytes, uint64_t ctx_bytes,
                                       uint32_t fn_flags, int64_t now_us, int64_t avail_bytes, uint64_t extra_bytes,
                                       uint64_t granularity, uint32_t opts, sage_share_grant *g) {
  TAB_OR_FAIL(T, tab);
  if (!g || gpu < 0 || gpu >= T->n_gpus) return fail(SAGE_EINVAL, "share_admit_within: bad arguments");
  const bool has_ro = fn_flags & SAGE_FN_HAS_RO;
  auto it = T->by_key.find({fn, gpu});
  Res *r = it == T->by_key.end() ? nullptr : it->second;
  fill_grant(T, r, ro_bytes, ctx_bytes, has_ro, g);
  if ((opts & SAGE_ADMIT_DEFER_RO_LEADER) && g->alloc_ro) return SAGE_ADMIT_DEFERRED;
  if (avail_bytes >= 0) {
    uint64_t need = g->alloc_ro + g->alloc_ctx + extra_bytes;
    if (granularity > 1) need = (need + granularity - 1) / granularity * granularity;
    if (need > (uint64_t)avail_bytes) return SAGE_ENOMEM;   // not an error: tl_err untouched
  }
  admit_locked(T, r, fn, gpu, has_ro, now_us, g);
  return SAGE_OK;
}

// attach the leader's stage END event to a token, or mark it ready (ev == 0)
extern "C" int sage_share_token(sage_handle tab, uint64_t resident, int kind, sage_handle ev) {
  TAB_OR_FAIL(T, tab);
  auto it = T->by_id.find(resident);
  if (it == T->by_id.end()) return fail(SAGE_ESTATE, "share_token: unknown resident");
  Tok &t = kind == SAGE_TOKEN_CTX ? it->second->ctx_tok : it->second->ro_tok;
  if (!t.live) return SAGE_OK;   // the segment was freed meanwhile: nothing to wait for
  if (ev) {
    if (!t.ready) t.ev = ev;
  } else {
    t.ready = true;
    t.ev = 0;
  }
  return SAGE_OK;
}

// a token of a resident or segment that is gone names a finished stage: ready
extern "C" int sage_share_token_ready(sage_handle tab, uint64_t resident, int kind, int *ready) {
  TAB_OR_FAIL(T, tab);
  if (!ready) return fail(SAGE_EINVAL, "share_token_ready: null out");
  auto it = T->by_id.find(resident);
  if (it == T->by_id.end()) {
    *ready = 1;
    return SAGE_OK;
  }
  Tok &t = kind == SAGE_TOKEN_CTX ? it->second->ctx_tok : it->second->ro_tok;
  *ready = (!t.live || t.is_ready()) ? 1 : 0;
  return SAGE_OK;
}

extern "C" int sage_share_release(sage_handle tab, int32_t fn, int gpu, int64_t now_us, sage_share_step *out) {
  TAB_OR_FAIL(T, tab);
  if (!out) return fail(SAGE_EINVAL, "share_release: null step");
  memset(out, 0, sizeof *out);
  auto it = T->by_key.find({fn, gpu});
  Res *r = it == T->by_key.end() ? nullptr : it->second;
  if (!r || r->state != R_ACTIVE || r->active < 1)
    return fail(SAGE_ESTATE, "release of a resident that is not active (fn " + std::to_string(fn) + ", gpu" +
                                 std::to_string(gpu) + ")");
  out->resident = r->id;
  out->state_before = R_ACTIVE;
  r->last_activity = now_us;
  if (--r->active > 0) {
    out->state_after = R_ACTIVE;
    return SAGE_OK;
  }
  // the last user: the leader tokens are ready for good
  if (r->ro_tok.live) r->ro_tok.ready = true, r->ro_tok.ev = 0;
  if (r->ctx_tok.live) r->ctx_tok.ready = true, r->ctx_tok.ev = 0;
  if (T->flags & SAGE_SHARE_MULTI_STAGE) {
    arm(r, R_STAGE1, now_us, T->iv[0], out);
  } else if (T->keep_alive > 0) {
    arm(r, R_STAGE1, now_us, T->keep_alive, out);
  } else {
    evict(T, r, out);
    out->actions &= ~SAGE_STEP_GPU_FREED;   // an immediate eviction is not a pressure relief event
    return SAGE_OK;
  }
  out->state_after = r->state;
  return SAGE_OK;
}

// the decay timer (resident, gen) fired at now
extern "C" int sage_share_expire(sage_handle tab, uint64_t resident, uint32_t gen, int64_t now_us,
                                 sage_share_step *out) {
  TAB_OR_FAIL(T, tab);
  if (!out) return fail(SAGE_EINVAL, "share_expire: null step");
  memset(out, 0, sizeof *out);
  auto it = T->by_id.find(resident);
  if (it == T->by_id.end()) return fail(SAGE_ESTATE, "share_expire: unknown resident");
  Res *r = it->second;
  if (r->state == R_ACTIVE || r->deadline < 0 || r->gen != gen)
    return fail(SAGE_ESTATE, "stale decay timer");
  r->deadline = -1;
  if (!(T->flags & SAGE_SHARE_MULTI_STAGE)) {   // flat keep-alive: evict (sharing.py:209-212)
    out->resident = r->id;
    out->state_before = r->state;
    evict(T, r, out);
    return SAGE_OK;
  }
  demote_once(T, r, now_us, out);
  return SAGE_OK;
}

// the pressure victim on gpu, or *resident = 0 (sharing.py:288-298)
extern "C" int sage_share_victim(sage_handle tab, int gpu, int32_t exclude_fn, uint64_t *resident) {
  TAB_OR_FAIL(T, tab);
  if (!resident) return fail(SAGE_EINVAL, "share_victim: null out");
  *resident = 0;
  for (int state : {R_STAGE2, R_STAGE1}) {
    Res *best = nullptr;
    for (auto &kv : T->by_id) {
      Res *r = kv.second;
      if (r->gpu != gpu || r->state != state || r->fn == exclude_fn || !(r->ro || r->ctx)) continue;
      if (!best || r->last_activity < best->last_activity) best = r;   // first minimum (stable)
    }
    if (best) {
      *resident = best->id;
      return SAGE_OK;
    }
  }
  return SAGE_OK;
}

// one forced decay step (the victim's timer is cancelled and re-armed)
extern "C" int sage_share_demote(sage_handle tab, uint64_t resident, int64_t now_us, sage_share_step *out) {
  TAB_OR_FAIL(T, tab);
  if (!out) return fail(SAGE_EINVAL, "share_demote: null step");
  memset(out, 0, sizeof *out);
  auto it = T->by_id.find(resident);
  if (it == T->by_id.end()) return fail(SAGE_ESTATE, "share_demote: unknown resident");
  Res *r = it->second;
  if (r->state == R_ACTIVE) return fail(SAGE_ESTATE, "share_demote: resident is active");
  cancel_timer(r, &out->timer_cancelled);
  demote_once(T, r, now_us, out);
  return SAGE_OK;
}

// evict now (shutdown); the step lists what the caller frees
extern "C" int sage_share_evict(sage_handle tab, uint64_t resident, sage_share_step *out) {
  TAB_OR_FAIL(T, tab);
  if (!out) return fail(SAGE_EINVAL, "share_evict: null step");
  memset(out, 0, sizeof *out);
  auto it = T->by_id.find(resident);
  if (it == T->by_id.end()) return fail(SAGE_ESTATE, "share_evict: unknown resident");
  out->resident = resident;
  out->state_before = it->second->state;
  out->timer_cancelled = it->second->deadline >= 0;
  evict(T, it->second, out);
  return SAGE_OK;
}

extern "C" int sage_share_info(sage_handle tab, uint64_t resident, sage_resident_info *out) {
  TAB_OR_FAIL(T, tab);
  auto it = T->by_id.find(resident);
  if (it == T->by_id.end() || !out) return fail(SAGE_ESTATE, "share_info: unknown resident");
  Res *r = it->second;
  memset(out, 0, sizeof *out);
  out->resident = r->id;
  out->fn = r->fn;
  out->gpu = r->gpu;
  out->state = r->state;
  out->active = r->active;
  out->holds = (r->ro ? SAGE_HOLD_RO : 0) | (r->ctx ? SAGE_HOLD_CTX : 0) | (r->cache ? SAGE_HOLD_CACHE : 0) |
               (r->cpu_ctx ? SAGE_HOLD_CPU_CTX : 0) | (r->container ? SAGE_HOLD_CONTAINER : 0);
  out->ro_bytes = r->ro ? r->ro_bytes : 0;
  out->ctx_bytes = r->ctx ? r->ctx_bytes : 0;
  out->last_activity_us = r->last_activity;
  out->deadline_us = r->deadline;
  out->timer_gen = r->gen;
  out->has_checksum = r->has_cs;
  out->checksum = r->cs;
  return SAGE_OK;
}

extern "C" int sage_share_lookup(sage_handle tab, int32_t fn, int gpu, uint64_t *resident) {
  TAB_OR_FAIL(T, tab);
  if (!resident) return fail(SAGE_EINVAL, "share_lookup: null out");
  auto it = T->by_key.find({fn, gpu});
  *resident = it == T->by_key.end() ? 0 : it->second->id;
  return SAGE_OK;
}

// residents in admission order; *n = count (ids written up to cap)
extern "C" int sage_share_list(sage_handle tab, uint64_t *ids, int cap, int *n) {
  TAB_OR_FAIL(T, tab);
  if (!n) return fail(SAGE_EINVAL, "share_list: null count");
  int k = 0;
  for (auto &kv : T->by_id) {
    if (ids && k < cap) ids[k] = kv.second->id;
    ++k;
  }
  *n = k;
  return SAGE_OK;
}

extern "C" int sage_share_ro_loads(sage_handle tab, int32_t fn, int gpu, uint32_t *n) {
  TAB_OR_FAIL(T, tab);
  if (!n) return fail(SAGE_EINVAL, "share_ro_loads: null out");
  auto it = T->ro_loads.find({fn, gpu});
  *n = it == T->ro_loads.end() ? 0 : it->second;
  return SAGE_OK;
}

// the landed (and verified) content checksum of a resident's RO segment
extern "C" int sage_share_set_checksum(sage_handle tab, uint64_t resident, uint64_t checksum) {
  TAB_OR_FAIL(T, tab);
  auto it = T->by_id.find(resident);
  if (it == T->by_id.end()) return fail(SAGE_ESTATE, "share_set_checksum: unknown resident");
  Res *r = it->second;
  if (!r->ro) return fail(SAGE_ESTATE, "share_set_checksum: resident holds no RO segment");
  if (r->has_cs) {
    if (r->cs != checksum) return fail(SAGE_ECHECKSUM, "share_set_checksum: segment content changed");
    return SAGE_OK;
  }
  r->has_cs = true;
  r->cs = checksum;
  T->content.emplace(checksum, r->id);
  return SAGE_OK;
}

// a resident on gpu (other than exclude_fn's) holding a landed RO segment with
// this content and a ready token; *resident = 0 if none
extern "C" int sage_share_find_content(sage_handle tab, int gpu, uint64_t checksum, int32_t exclude_fn,
                                       uint64_t *resident) {
  TAB_OR_FAIL(T, tab);
  if (!resident) return fail(SAGE_EINVAL, "share_find_content: null out");
  *resident = 0;
  auto range = T->content.equal_range(checksum);
  for (auto it = range.first; it != range.second; ++it) {
    auto f = T->by_id.find(it->second);
    Res *r = f == T->by_id.end() ? nullptr : f->second;
    if (r && r->gpu == gpu && r->fn != exclude_fn && r->ro && r->ro_tok.is_ready()) {
      *resident = r->id;
      return SAGE_OK;
    }
  }
  return SAGE_OK;
}
// the invariant sweep (sharing.py:305-335): SAGE_ESTATE naming the first violation
extern "C" int sage_share_check(sage_handle tab) {
  TAB_OR_FAIL(T, tab);
  std::string why;
  for (auto &kv : T->by_id)
    if (check_one(T, kv.second, &why) != SAGE_OK) return fail(SAGE_ESTATE, why);
  for (auto &kv : T->content) {
    auto it = T->by_id.find(kv.second);
    if (it == T->by_id.end() || !it->second->has_cs || it->second->cs != kv.first)
      return fail(SAGE_ESTATE, "content index out of date");
  }
  return SAGE_OK;
}
