"""The oracle's two restatements agree with each other and with the committed
golden vectors (tests/golden/land_vectors.json, made by make_golden.py)."""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O

GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def cbuilt(built):
    return O.c_lib()


def test_checksum_np_matches_c(cbuilt):
    for seed, n in [(1, 0), (2, 8), (3, 16), (4, 1 << 12), (5, (1 << 20) + 8)]:
        b = O.db_bytes(seed, n)
        assert O.checksum_np(b) == O.checksum_c(b)
        assert O.checksum_np(b, word_base=1 << 33) == O.checksum_c(b, word_base=1 << 33)


def test_checksum_is_position_sensitive(cbuilt):
    b = O.db_bytes(7, 64)
    sw = b.copy()
    sw[:4], sw[4:8] = b[4:8], b[:4]
    assert O.checksum_c(b) != O.checksum_c(sw)
    z = np.zeros(64, np.uint8)
    assert O.checksum_c(z) != 0  # padding contributes: the checksum pins the size


def test_checksum_split_additivity(cbuilt):
    # order independence: any split into ranges sums to the whole
    b = O.db_bytes(8, 1 << 16)
    whole = O.checksum_c(b)
    parts = sum(O.checksum_c(b[s:s + 4096], word_base=s // 8) for s in range(0, b.size, 4096))
    assert whole == parts & 0xFFFFFFFFFFFFFFFF


def test_land_np_matches_c(cbuilt):
    from paper_2404_14691_b200.layout import SegmentLayout
    sizes = O.random_layout_sizes(3, 17, 50_001)
    lay = SegmentLayout.packed(sizes, align=256, src_order=list(reversed(range(17))))
    db = O.db_bytes(11, lay.packed_bytes)
    s1, c1 = O.land_np(db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
    s2, c2 = O.land_c(db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
    assert c1 == c2 and np.array_equal(s1, s2)
    assert O.layout_ok_c(lay.src_off, lay.dst_off, lay.length, lay.packed_bytes, lay.seg_bytes)


def test_golden_vectors(cbuilt):
    data = json.loads((GOLDEN / "land_vectors.json").read_text())
    assert len(data["cases"]) >= 8
    for case in data["cases"]:
        db = O.db_bytes(case["seed"], case["packed_bytes"])
        seg, cs = O.land_c(db, case["src_off"], case["dst_off"], case["length"], case["seg_bytes"])
        assert f"{cs:016x}" == case["checksum"], case["name"]
        import hashlib
        assert hashlib.sha256(seg.tobytes()).hexdigest() == case["seg_sha256"], case["name"]
        seg2, cs2 = O.land_np(db, case["src_off"], case["dst_off"], case["length"], case["seg_bytes"])
        assert cs2 == cs


def test_hostpath_matches_land(cbuilt):
    from paper_2404_14691_b200.layout import SegmentLayout
    lay = SegmentLayout.packed(O.random_layout_sizes(4, 9, 300_000))
    db = O.db_bytes(12, lay.packed_bytes)
    _, cs = O.land_c(db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
    sums = O.hostpath_c(db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes, n_inv=5, threads=3)
    assert all(int(s) == cs for s in sums)


def test_body_refs_small():
    rng = np.random.default_rng(0)
    A = rng.standard_normal((8, 4)).astype(np.float32)
    B = rng.standard_normal((4, 3)).astype(np.float32)
    assert np.allclose(O.sgemm_ref(A, B), A @ B, rtol=1e-5)
    rowptr = np.array([0, 2, 2, 3])
    col = np.array([0, 2, 1])
    val = np.array([1.0, 2.0, 3.0], np.float32)
    x = np.array([1.0, 10.0, 100.0], np.float32)
    assert np.allclose(O.spmv_ref(rowptr, col, val, x), [201.0, 0.0, 30.0])


def test_csb_pack_roundtrip_and_oracle_decode():
    """parboil.csb_pack (the product's format builder) against the oracle's
    independent decoder: the same (row, col, val) multiset as the CSR input,
    sub-buckets sorted by row, buckets 16-B padded, and the two spmv
    references agree."""
    from paper_2404_14691_b200.parboil import csb_pack
    rng = np.random.default_rng(5)
    for rows, slices, cw in ((3001, 2, 1024), (4096, 1, 12288), (777, 2, 256)):
        counts = rng.integers(0, 30, rows)
        counts[::5] = 0
        rowptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
        nnz = int(rowptr[-1])
        col = rng.integers(0, rows, nnz, dtype=np.int32)
        val = rng.standard_normal(nnz, dtype=np.float32)
        off, ent, p = csb_pack(rowptr, col, val, rows, slices=slices, chunk_cols=cw)
        assert p["nnz"] == nnz and off[-1] == ent.shape[0] == p["entries"]
        assert np.all(np.diff(off[::O.CSB_W].astype(np.int64)) % 2 == 0)        # 16-B buckets
        r, c, v = O.csb_decode(off, ent, rows, rows, p["R"], p["CW"], p["S"])
        want = np.repeat(np.arange(rows), counts)
        a = np.lexsort((v.view(np.uint32), c, r))
        b = np.lexsort((val.view(np.uint32), col, want))
        assert np.array_equal(r[a], want[b]) and np.array_equal(c[a], col[b])
        assert np.array_equal(v[a].view(np.uint32), val[b].view(np.uint32))
        for k in range(off.size - 1):                                         # rows sorted per sub-bucket
            idx = ent[off[k]:off[k + 1], 0]
            idx = idx[idx != 0xFFFFFFFF] >> 17
            assert np.all(np.diff(idx.astype(np.int64)) >= 0)
        x = rng.standard_normal(rows, dtype=np.float32)
        np.testing.assert_allclose(O.spmv_csb_ref(off, ent, rows, rows, p["R"], p["CW"], p["S"], x),
                                   O.spmv_ref(rowptr, col, val, x), rtol=1e-5, atol=1e-5)
