"""libsagedp.so on a CPU-only box: it loads, exports every symbol the header
declares, validates layouts like the reference validates its inputs
(ValueError-style SAGE_EINVAL), and its chunk planner reproduces the oracle's
bytes and checksum exactly (host emulation of the land kernel's contract)."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O
from paper_2404_14691_b200 import _lib
from paper_2404_14691_b200.layout import SegmentLayout

ROOT = Path(__file__).resolve().parent.parent


def header_symbols():
    text = (ROOT / "include" / "sage_dp.h").read_text()
    return sorted(set(re.findall(r"\b(sage_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol(built):
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 40
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(_lib.exported_symbols()) == syms


def test_abi_and_nodevice(built):
    L = _lib.lib()
    assert L.sage_abi_version() == 1
    from conftest import gpu_available
    if not gpu_available():
        rc = L.sage_init(1, 0, 0, 0, 0)
        assert rc == _lib.SAGE_ENODEV
        assert "device" in _lib.last_error().lower()


@pytest.mark.parametrize("bad", [
    dict(src=[0], dst=[16], ln=[4], packed=4, seg=32),      # dst_off[0] != 0
    dict(src=[0], dst=[0], ln=[5], packed=4, seg=16),       # exceeds packed
    dict(src=[0, 0], dst=[0, 8], ln=[4, 4], packed=4, seg=32),  # unaligned dst
    dict(src=[0, 0], dst=[0, 16], ln=[20, 4], packed=20, seg=32),  # overlap
    dict(src=[0], dst=[0], ln=[4], packed=4, seg=20),       # seg not /16
])
def test_layout_validation(built, bad):
    L = _lib.lib()
    arr = lambda v: (C.c_uint64 * len(v))(*v)
    h = _lib.H()
    rc = L.sage_layout_create(arr(bad["src"]), arr(bad["dst"]), arr(bad["ln"]), len(bad["ln"]),
                              bad["packed"], bad["seg"], C.byref(h))
    assert rc == _lib.SAGE_EINVAL
    assert O.layout_ok_c(bad["src"], bad["dst"], bad["ln"], bad["packed"], bad["seg"]) is False


def _emulate(lay, db, chunk):
    out = np.empty(lay.seg_bytes, np.uint8)
    cs = C.c_uint64()
    rc = _lib.lib().sage_debug_emulate_land(lay.handle(), db.ctypes.data, db.size, out.ctypes.data, chunk,
                                            C.byref(cs))
    assert rc == 0, _lib.last_error()
    return out, cs.value


@pytest.mark.parametrize("seed", range(12))
def test_planner_matches_oracle(built, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 40))
    total = int(rng.integers(n, 400_000))
    sizes = O.random_layout_sizes(seed, n, total, min_size=0)
    order = list(rng.permutation(n)) if seed % 2 else None
    lay = SegmentLayout.packed(sizes, align=int(rng.choice([16, 64, 256])), src_order=order)
    db = O.db_bytes(seed + 100, lay.packed_bytes)
    want_seg, want_cs = O.land_c(db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
    for chunk in (65536, 4096 * 17, 1 << 20, 8 << 20):
        seg, cs = _emulate(lay, db, chunk)
        assert cs == want_cs and np.array_equal(seg, want_seg), (seed, chunk)


def test_planner_golden(built):
    import json
    data = json.loads((ROOT / "tests" / "golden" / "land_vectors.json").read_text())
    for case in data["cases"]:
        lay = SegmentLayout(tuple(case["src_off"]), tuple(case["dst_off"]), tuple(case["length"]),
                            case["packed_bytes"], case["seg_bytes"])
        db = O.db_bytes(case["seed"], case["packed_bytes"])
        for chunk in (65536, 1 << 20):
            seg, cs = _emulate(lay, db, chunk)
            assert f"{cs:016x}" == case["checksum"], case["name"]
