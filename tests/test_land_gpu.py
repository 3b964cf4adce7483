"""Parity of the CUDA land path with the oracle (bit-exact bytes + checksum),
through the C-ABI: pageable / pinned / HBM-resident sources, golden vectors,
ragged layouts, ring wrap-around with many loads in flight."""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O
from paper_2404_14691_b200 import device as D
from paper_2404_14691_b200.layout import SegmentLayout

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden" / "land_vectors.json"


def _land_and_read(lay, db, mode="pageable"):
    seg = D.pool_alloc(0, max(16, lay.seg_bytes), D._lib.CLASS_READ_ONLY)
    try:
        if mode == "pageable":
            op = D.load(0, seg.dptr, db, lay)
        elif mode == "pinned":
            pb = D.PinnedBuffer(max(1, db.size))
            pb.view()[:db.size] = db
            op = D.load(0, seg.dptr, db if db.size == 0 else pb, lay) if db.size else D.load(0, seg.dptr, db, lay)
        else:  # device-resident packed source
            src = D.pool_alloc(0, max(16, db.size + 16), D._lib.CLASS_WRITABLE)
            up = D.load(0, src.dptr, db, None)
            up.wait(); up.release()
            op = D.load(0, seg.dptr, None, lay, device_src=src.dptr, device_src_bytes=db.size)
        res = op.wait()
        got = D.read_device(0, seg.dptr, lay.seg_bytes)
        op.release()
        if mode == "device":
            src.free()
        if mode == "pinned":
            pb.free()
        verify = D.segment_checksum(0, seg.dptr, lay.seg_bytes)
        return got, res, verify
    finally:
        seg.free()


@pytest.mark.parametrize("mode", ["pageable", "pinned", "device"])
def test_golden_vectors_gpu(dp, mode):
    data = json.loads(GOLDEN.read_text())
    for case in data["cases"]:
        lay = SegmentLayout(tuple(case["src_off"]), tuple(case["dst_off"]), tuple(case["length"]),
                            case["packed_bytes"], case["seg_bytes"])
        db = O.db_bytes(case["seed"], case["packed_bytes"])
        got, res, verify = _land_and_read(lay, db, mode)
        assert f"{res.checksum:016x}" == case["checksum"], (case["name"], mode)
        assert hashlib.sha256(got.tobytes()).hexdigest() == case["seg_sha256"], (case["name"], mode)
        assert verify == res.checksum
        assert res.landed_bytes == case["seg_bytes"]


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_random_layouts_cross_chunks(dp, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 300))
    total = int(rng.integers(20 << 20, 40 << 20))   # several 8 MiB chunks
    lay = SegmentLayout.packed(O.random_layout_sizes(seed, n, total), align=int(rng.choice([16, 256])),
                               src_order=list(rng.permutation(n)))
    db = O.db_bytes(seed + 50, lay.packed_bytes)
    want_seg, want_cs = O.land_c(db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
    for mode in ("pageable", "device"):
        got, res, verify = _land_and_read(lay, db, mode)
        assert res.checksum == want_cs and verify == want_cs, mode
        assert np.array_equal(got, want_seg), mode
        if mode == "pageable":
            assert res.link_bytes >= lay.packed_bytes and res.host_bytes >= lay.packed_bytes


def test_many_loads_in_flight_wrap_the_ring(dp):
    lays, dbs, segs, ops = [], [], [], []
    for i in range(24):   # 24 x ~3 MiB through an 8-slot ring, all enqueued before any completes
        lay = SegmentLayout.packed(O.random_layout_sizes(i, 7, 3_000_000 + 977 * i), align=256)
        db = O.db_bytes(1000 + i, lay.packed_bytes)
        seg = D.pool_alloc(0, lay.seg_bytes, D._lib.CLASS_READ_ONLY)
        lays.append(lay); dbs.append(db); segs.append(seg)
        ops.append(D.load(0, seg.dptr, db, lay))
    for lay, db, seg, op in zip(lays, dbs, segs, ops):
        res = op.wait()
        _, want = O.land_c(db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
        assert res.checksum == want
        assert D.segment_checksum(0, seg.dptr, lay.seg_bytes) == want
        op.release()
        seg.free()


def test_hundred_mib_segment(dp):
    lay = SegmentLayout.packed(O.random_layout_sizes(77, 161, 100 << 20), align=256)
    db = O.db_bytes(77, lay.packed_bytes)
    _, want = O.land_c(db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
    got, res, verify = _land_and_read(lay, db, "pageable")
    assert res.checksum == want == verify
    assert res.gpu_end_us >= res.gpu_begin_us >= 0
    assert res.cpu_end_us >= res.cpu_begin_us >= 0


def test_pool_denied_and_usage(dp):
    u0 = D.pool_usage(0)
    cap = u0["capacity"]
    with pytest.raises(D.DeniedAlloc) as ei:
        D.pool_alloc(0, cap + 4096, D._lib.CLASS_READ_ONLY, account_only=True)
    assert ei.value.shortfall == cap + 4096 - (cap - u0["ledger"])
    s = D.pool_alloc(0, 10 << 20, D._lib.CLASS_WRITABLE)
    u1 = D.pool_usage(0)
    assert u1["by_class"][2] - u0["by_class"][2] == 10 << 20
    assert u1["physical"] - u0["physical"] >= 10 << 20
    s.free()
    assert D.pool_usage(0)["ledger"] == u0["ledger"]
    with pytest.raises(D._lib.SageError):
        D._lib.check(D.lib().sage_pool_free(s.h or 0x0300000000000001), "double free")


def test_pool_chunk_carving_and_trim(dp):
    """Private writable segments are carved from 1 GiB pool chunks: pieces
    never overlap (each keeps its own bytes), are reused by size once freed,
    cannot be exported (no handle of their own), and sage_pool_trim gives the
    chunks back once no piece is live."""
    import ctypes as Cc
    D.pool_trim(0)
    n, size = 24, 100 << 20                      # 2.4 GB: three chunks
    segs, pats = [], []
    for k in range(n):
        s = D.pool_alloc(0, size, D._lib.CLASS_WRITABLE)
        pat = np.full(size, (37 * k + 11) & 0xFF, dtype=np.uint8)
        op = D.load(0, s.dptr, pat, None)
        op.wait()
        op.release()
        segs.append(s)
        pats.append(pat[0])
    for s, v in zip(segs, pats):
        got = D.read_device(0, s.dptr, size)
        assert got[0] == v and got[-1] == v and np.all(got[::4096] == v)
    fd, ph = Cc.c_int(), D._lib.u64()
    rc = D.lib().sage_pool_export(segs[0].h, Cc.byref(fd), Cc.byref(ph))
    assert rc == D._lib.SAGE_EINVAL           # a carved piece has no pages of its own to export
    ptrs = {s.dptr for s in segs}
    for s in segs:
        s.free()
    again = D.pool_alloc(0, size, D._lib.CLASS_WRITABLE)   # a freed piece of the same size
    assert again.dptr in ptrs
    again.free()
    released = D.pool_trim(0)
    assert released >= n * size                # every chunk idle: unmapped
    assert D.pool_trim(0) == 0


def test_identity_load_from_hbm_verified_and_unverified(dp):
    """An identity load from this GPU's HBM: verified, it is a land with the
    oracle's checksum; unverified (a private payload, SAGE_LOAD_NO_VERIFY),
    it is one D2D copy -- the same bytes, zero padding to 16 B, no checksum."""
    n = 5 * (1 << 20) + 7
    src_bytes = O.db_bytes(21, n)
    src = D.pool_alloc(0, n + 64, D._lib.CLASS_WRITABLE, unaccounted=True)
    op = D.load(0, src.dptr, src_bytes, None)
    op.wait()
    op.release()
    seg = -(-n // 16) * 16
    want_seg, want_sum = O.land_c(src_bytes, np.array([0], np.uint64), np.array([0], np.uint64),
                                  np.array([n], np.uint64), seg)
    for verify in (True, False):
        dst = D.pool_alloc(0, seg + 256, D._lib.CLASS_WRITABLE, unaccounted=True)
        D._lib.check(D.lib().sage_device_sync(0), "sync")
        op = D.load(0, dst.dptr, None, None, device_src=src.dptr, device_src_bytes=n, verify=verify)
        res = op.wait()
        got = D.read_device(0, dst.dptr, seg)
        assert np.array_equal(got, want_seg)
        assert res.checksum == (want_sum if verify else 0)
        op.release()
        dst.free()
    src.free()


def test_staged_identity_unverified_interleaved(dp):
    """Pageable identity loads: verified ones land through the device slot;
    unverified ones (SAGE_LOAD_NO_VERIFY) DMA each staged chunk straight into
    dst, skipping the land. Interleaved through the 8-slot ring, all enqueued
    before any completes, into dirtied destinations: every segment equals the
    oracle's bytes (zero padding to 16 B), checksums only where verified."""
    sizes = [1, 15, 4097, (8 << 20) - 3, (8 << 20) + 16, (21 << 20) + 9, 3 << 20, (17 << 20) + 1]
    jobs = []
    for i, n in enumerate(sizes * 2):
        verify = i % 2 == 0
        db = O.db_bytes(300 + i, n)
        seg_bytes = -(-n // 16) * 16
        seg = D.pool_alloc(0, seg_bytes, D._lib.CLASS_WRITABLE)
        junk = D.PinnedBuffer(seg_bytes)
        junk.view()[:] = 0xCD
        D.load(0, seg.dptr, junk, None).wait()
        junk.free()
        jobs.append((n, db, seg_bytes, seg, verify, D.load(0, seg.dptr, db, None, verify=verify)))
    for n, db, seg_bytes, seg, verify, op in jobs:
        res = op.wait()
        want = np.zeros(seg_bytes, np.uint8)
        want[:n] = db
        assert np.array_equal(D.read_device(0, seg.dptr, seg_bytes), want), (n, verify)
        assert res.checksum == (O.checksum_c(want) if verify else 0), (n, verify)
        assert res.host_bytes >= n and res.landed_bytes == seg_bytes
        op.release()
        seg.free()


def test_direct_path_identity_pinned(dp):
    """Identity loads from pinned memory take the direct DMA + verify path;
    bytes and checksum equal the oracle's (incl. zero padding to 16)."""
    for n in (1, 15, 16, 4097, 3 << 20, (9 << 20) + 5):
        db = O.db_bytes(n, n)
        pb = D.PinnedBuffer(n)
        pb.view()[:] = db
        seg_bytes = (n + 15) // 16 * 16
        seg = D.pool_alloc(0, seg_bytes, D._lib.CLASS_WRITABLE)
        # dirty the destination first: the padding must be re-zeroed
        junk = D.PinnedBuffer(seg_bytes)
        junk.view()[:] = 0xAB
        D.load(0, seg.dptr, junk, None).wait()
        op = D.load(0, seg.dptr, pb, None)
        res = op.wait()
        want_seg = np.zeros(seg_bytes, np.uint8)
        want_seg[:n] = db
        assert res.checksum == O.checksum_c(want_seg), n
        assert np.array_equal(D.read_device(0, seg.dptr, seg_bytes), want_seg), n
        assert res.link_bytes == n and res.host_bytes == 0
        op.release()
        seg.free()
        pb.free()
        junk.free()


def test_two_gib_segment_full_size(dp):
    """BASELINE cfg 4's largest read-only record (2048 MiB, 97 ragged tensors,
    one misaligned every few bytes) at full size: the load's checksum, an
    independent device re-checksum of the landed bytes and the C oracle agree
    (bit-exact), across 256 staging chunks of the ring."""
    total = 2048 << 20
    rng = np.random.default_rng(2048)
    cuts = np.unique(rng.integers(1, total, 96))   # (random_layout_sizes would materialise arange(total))
    sizes = np.diff(np.concatenate([[0], cuts, [total]])).tolist()
    lay = SegmentLayout.packed(sizes, align=256)
    db = O.db_bytes(2048, lay.packed_bytes)
    _, want = O.land_c(db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
    seg = D.pool_alloc(0, lay.seg_bytes, D._lib.CLASS_READ_ONLY)
    try:
        op = D.load(0, seg.dptr, db, lay)
        res = op.wait()
        op.release()
        assert res.chunks >= 256
        assert res.checksum == want
        assert D.segment_checksum(0, seg.dptr, lay.seg_bytes) == want
    finally:
        seg.free()


def test_stage2_cache_round_trip(dp):
    """Stage1 -> Stage2 -> rejoin at full cfg-1 size (100 MiB): D2H of the
    landed segment into a pinned cache, then an identity reload from that
    cache into a fresh segment, is byte-identical (same checksum, same hash)."""
    lay = SegmentLayout.packed(O.random_layout_sizes(5, 64, 100 << 20), align=256)
    db = O.db_bytes(5, lay.packed_bytes)
    want_seg, want = O.land_c(db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
    a = D.pool_alloc(0, lay.seg_bytes, D._lib.CLASS_READ_ONLY)
    b = D.pool_alloc(0, lay.seg_bytes, D._lib.CLASS_READ_ONLY)
    cache = D.PinnedBuffer(lay.seg_bytes)
    try:
        op = D.load(0, a.dptr, db, lay)
        assert op.wait().checksum == want
        ev = D.d2h(0, a.dptr, cache, lay.seg_bytes, wait=[op.end])
        ev.sync()
        op.release()
        ev.release()
        assert hashlib.sha256(cache.view()).digest() == hashlib.sha256(want_seg).digest()
        re = D.load(0, b.dptr, cache, None)
        assert re.wait().checksum == want
        re.release()
        assert hashlib.sha256(D.read_device(0, b.dptr, lay.seg_bytes)).digest() == hashlib.sha256(want_seg).digest()
    finally:
        cache.free()
        a.free()
        b.free()
