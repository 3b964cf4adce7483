"""The native resident table (csrc/segtab.cu, sage_share_*) driven directly
through the C-ABI on a CPU box: the reference sharing manager's rules
(pkg/src/gslsim/sharing.py) one by one -- warmth, leader election, RO-load
counting, the refcounted release, each decay step and the actions it hands
back, the pressure victim order, the invariant sweep -- and the content
index used to deduplicate identical RO records.  No device is touched."""
import ctypes as C

import pytest

from paper_2404_14691_b200 import _lib

S = 1_000_000
RO, CTX = 100 << 20, 414 << 20


class Table:
    def __init__(self, flags=_lib.SHARE_RO | _lib.SHARE_CTX | _lib.SHARE_MULTI_STAGE, gpus=1, keep_alive=0,
                 iv=(30 * S,) * 4):
        self.L = _lib.lib()
        h = _lib.H(0)
        assert self.L.sage_share_create(gpus, flags, keep_alive, (_lib.i64 * 4)(*iv), C.byref(h)) == 0
        self.h = h.value

    def close(self):
        assert self.L.sage_share_destroy(self.h) == 0

    def admit(self, fn, gpu=0, now=0, has_ro=True, preview=False):
        g = _lib.ShareGrant()
        fl = _lib.FN_HAS_RO if has_ro else 0
        if preview:
            rc = self.L.sage_share_preview(self.h, fn, gpu, RO, CTX, fl, C.byref(g))
        else:
            rc = self.L.sage_share_admit(self.h, fn, gpu, RO, CTX, fl, now, C.byref(g))
        assert rc == 0, _lib.last_error()
        return g

    def step(self, name, *args):
        st = _lib.ShareStep()
        rc = getattr(self.L, name)(self.h, *args, C.byref(st))
        assert rc == 0, _lib.last_error()
        return st

    def info(self, rid):
        out = _lib.ResidentInfo()
        assert self.L.sage_share_info(self.h, rid, C.byref(out)) == 0
        return out

    def check(self):
        assert self.L.sage_share_check(self.h) == 0, _lib.last_error()


@pytest.fixture
def tab(built):
    t = Table()
    yield t
    t.close()


def test_first_admission_leads_both_segments(tab):
    g = tab.admit(7, now=5)
    assert g.warmth == 0 and g.leader_ro and g.leader_ctx and g.new_resident
    assert (g.alloc_ro, g.alloc_ctx) == (RO, CTX)
    f = tab.admit(7, now=6)                        # concurrent follower
    assert f.warmth == 4 and not f.leader_ro and not f.leader_ctx and f.alloc_ro == 0
    assert f.wait_ro and f.wait_ctx and f.resident == g.resident
    # the leader's token (no event attached) readies on demand
    assert tab.L.sage_share_token(tab.h, g.resident, _lib.TOKEN_RO, 0) == 0
    assert not tab.admit(7, preview=True).wait_ro and tab.admit(7, preview=True).wait_ctx
    info = tab.info(g.resident)
    assert info.active == 2 and info.state == 0 and info.last_activity_us == 6
    n = C.c_uint32()
    tab.L.sage_share_ro_loads(tab.h, 7, 0, C.byref(n))
    assert n.value == 1                            # the Stage1Hot follower loads nothing
    tab.check()


def test_release_refcount_then_stage1_timer(tab):
    g = tab.admit(1, now=0)
    tab.admit(1, now=1)
    st = tab.step("sage_share_release", 1, 0, 10)
    assert st.actions == 0 and st.state_after == 0
    st = tab.step("sage_share_release", 1, 0, 20)
    assert st.actions == _lib.STEP_ARM and st.state_after == 1 and st.deadline_us == 20 + 30 * S
    tab.check()
    # a second release of an idle resident is a state error (reference SimulationError)
    assert tab.L.sage_share_release(tab.h, 1, 0, 30, C.byref(_lib.ShareStep())) == _lib.SAGE_ESTATE
    assert tab.info(g.resident).state == 1


def test_decay_steps_and_their_actions(tab):
    g = tab.admit(3, now=0)
    st = tab.step("sage_share_release", 3, 0, 0)
    rid, t = g.resident, st.deadline_us
    want = [
        (1, 2, _lib.STEP_CACHE_RO | _lib.STEP_FREE_RO | _lib.STEP_GPU_FREED | _lib.STEP_ARM, 3),   # -> Stage2
        (2, 3, _lib.STEP_FREE_CTX | _lib.STEP_GPU_FREED | _lib.STEP_ARM, 2),                       # -> Stage3
        (3, 4, _lib.STEP_DROP_CACHE | _lib.STEP_ARM, 1),                                           # -> Stage4
    ]
    for before, after, acts, warmth in want:
        st = tab.step("sage_share_expire", rid, st.timer_gen, t)
        assert (st.state_before, st.state_after, st.actions) == (before, after, acts)
        assert tab.admit(3, preview=True).warmth == warmth
        tab.check()
        t = st.deadline_us
    st = tab.step("sage_share_expire", rid, st.timer_gen, t)
    assert st.actions == _lib.STEP_EVICT | _lib.STEP_GPU_FREED
    assert tab.admit(3, preview=True).warmth == 0
    n = C.c_int()
    tab.L.sage_share_list(tab.h, None, 0, C.byref(n))
    assert n.value == 0


def test_stale_timer_is_refused(tab):
    g = tab.admit(2, now=0)
    st = tab.step("sage_share_release", 2, 0, 0)
    re = tab.admit(2, now=5)                      # rejoin cancels the pending timer
    assert re.timer_cancelled and re.warmth == 4
    rc = tab.L.sage_share_expire(tab.h, g.resident, st.timer_gen, st.deadline_us, C.byref(_lib.ShareStep()))
    assert rc == _lib.SAGE_ESTATE


def test_rejoin_from_stage2_leads_a_new_ro_segment(tab):
    g = tab.admit(4, now=0)
    st = tab.step("sage_share_release", 4, 0, 0)
    st = tab.step("sage_share_expire", g.resident, st.timer_gen, st.deadline_us)   # -> Stage2
    j = tab.admit(4, now=st.deadline_us - 1)
    assert j.warmth == 3 and j.leader_ro and not j.leader_ctx and j.alloc_ro == RO and j.timer_cancelled
    assert tab.info(g.resident).holds & _lib.HOLD_CACHE        # the host copy stays until Stage3 -> 4
    tab.check()


def test_flat_keep_alive_and_immediate_eviction(built):
    t = Table(flags=_lib.SHARE_RO | _lib.SHARE_CTX, keep_alive=5 * S)
    g = t.admit(1)
    st = t.step("sage_share_release", 1, 0, 0)
    assert st.actions == _lib.STEP_ARM and st.deadline_us == 5 * S
    st = t.step("sage_share_expire", g.resident, st.timer_gen, st.deadline_us)
    assert st.actions & _lib.STEP_EVICT and st.actions & _lib.STEP_FREE_RO and st.actions & _lib.STEP_GPU_FREED
    t.close()
    t = Table(flags=_lib.SHARE_CTX)               # SAGE-NR without keep-alive: evict at once, no wake-up
    t.admit(1)
    st = t.step("sage_share_release", 1, 0, 0)
    assert st.actions == _lib.STEP_EVICT | _lib.STEP_FREE_CTX
    t.close()


def test_ro_sharing_off_never_leads_ro(built):
    t = Table(flags=_lib.SHARE_CTX | _lib.SHARE_MULTI_STAGE)
    g = t.admit(1)
    assert g.leader_ctx and not g.leader_ro and g.alloc_ro == 0
    assert t.admit(1, preview=True).warmth == 3   # held ctx but no shared RO: Stage2 (SAGE-NR reloads)
    t.check()
    t.close()


def test_victims_stage2_first_then_least_recent(built):
    t = Table()
    rids = {}
    for k, fn in enumerate((10, 11, 12, 13)):
        rids[fn] = t.admit(fn, now=k).resident
        t.step("sage_share_release", fn, 0, 100 + k)
    v = C.c_uint64()
    assert t.L.sage_share_victim(t.h, 0, 10, C.byref(v)) == 0
    assert v.value == rids[11]                    # 10 excluded; 11 least recently active
    st = t.step("sage_share_demote", rids[11], 200)
    assert st.timer_cancelled and st.state_after == 2
    t.L.sage_share_victim(t.h, 0, 10, C.byref(v))
    assert v.value == rids[11]                    # a Stage2 holder (its context) goes before Stage1 ones
    t.step("sage_share_demote", rids[11], 201)    # -> Stage3: holds no GPU segment any more
    t.L.sage_share_victim(t.h, 0, 10, C.byref(v))
    assert v.value == rids[12]
    t.L.sage_share_victim(t.h, 0, 99, C.byref(v))
    assert v.value == rids[10]
    t.admit(13, now=300)                          # active residents are never victims
    for fn in (10, 12):
        t.step("sage_share_demote", rids[fn], 301)
        t.step("sage_share_demote", rids[fn], 302)
    t.L.sage_share_victim(t.h, 0, 99, C.byref(v))
    assert v.value == 0
    t.check()
    t.close()


def test_content_index_finds_identical_ro_of_another_function(tab):
    a = tab.admit(1, now=0)
    tab.L.sage_share_token(tab.h, a.resident, _lib.TOKEN_RO, 0)
    assert tab.L.sage_share_set_checksum(tab.h, a.resident, 0xABC) == 0
    assert tab.L.sage_share_set_checksum(tab.h, a.resident, 0xABD) == _lib.SAGE_ECHECKSUM
    out = C.c_uint64()
    tab.L.sage_share_find_content(tab.h, 0, 0xABC, 2, C.byref(out))
    assert out.value == a.resident
    tab.L.sage_share_find_content(tab.h, 0, 0xABC, 1, C.byref(out))
    assert out.value == 0                         # never the asking function itself
    tab.L.sage_share_find_content(tab.h, 1 if False else 0, 0xABD, 2, C.byref(out))
    assert out.value == 0
    st = tab.step("sage_share_release", 1, 0, 0)
    tab.step("sage_share_expire", a.resident, st.timer_gen, st.deadline_us)   # RO freed -> out of the index
    tab.L.sage_share_find_content(tab.h, 0, 0xABC, 2, C.byref(out))
    assert out.value == 0
    tab.check()


def test_bad_handles_and_arguments(built):
    L = _lib.lib()
    g = _lib.ShareGrant()
    assert L.sage_share_admit(12345, 0, 0, 1, 1, 1, 0, C.byref(g)) == _lib.SAGE_ESTATE
    h = _lib.H(0)
    assert L.sage_share_create(0, 0, 0, (_lib.i64 * 4)(1, 1, 1, 1), C.byref(h)) == _lib.SAGE_EINVAL
    t = Table(gpus=2)
    assert L.sage_share_admit(t.h, 0, 2, 1, 1, 1, 0, C.byref(g)) == _lib.SAGE_EINVAL
    t.close()
    assert L.sage_share_destroy(t.h) == _lib.SAGE_ESTATE
