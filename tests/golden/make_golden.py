"""Generate tests/golden/land_vectors.json.

Three restatements must agree before a vector is written: a pure-Python
loop (this file, small cases only), the numpy oracle and the C oracle.  The
committed JSON then pins the byte semantics the CUDA land kernel is tested
against (tests/test_land_gpu.py).  Re-run only when the specification in
oracle/sage_oracle.c changes:   python tests/golden/make_golden.py
"""
import hashlib
import json
import struct
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_2404_14691_b200 import _build  # noqa: E402
from paper_2404_14691_b200.layout import SegmentLayout  # noqa: E402

M64 = (1 << 64) - 1


def py_checksum(seg: bytes) -> int:
    s = 0
    for p in range(len(seg) // 8):
        lo, hi = struct.unpack_from("<II", seg, 8 * p)
        k = ((p & 0xFFFFFFFF) * 0x9E3779B1 ^ (p >> 32) * 0x85EBCA77) & 0xFFFFFFFF
        a = lo ^ k
        b = hi ^ ((k + 0x7F4A7C15) & 0xFFFFFFFF)
        s = (s + a * b + ((b << 32) | a)) & M64
    return s


def py_land(db: bytes, lay) -> bytes:
    seg = bytearray(lay.seg_bytes)
    for s, d, n in zip(lay.src_off, lay.dst_off, lay.length):
        seg[d:d + n] = db[s:s + n]
    return bytes(seg)


def cases():
    yield "empty", 1, SegmentLayout((), (), (), 0, 0)
    yield "one_byte", 2, SegmentLayout.packed([1], align=16)
    yield "three_bytes_pad256", 3, SegmentLayout.packed([3], align=256)
    yield "identity_16", 4, SegmentLayout.identity(16)
    yield "identity_ragged_1001", 5, SegmentLayout.packed([1001], align=16)
    yield "zero_len_tensors", 6, SegmentLayout.packed([0, 5, 0, 0, 33, 0], align=16)
    yield "misaligned_7", 7, SegmentLayout.packed([7] * 23, align=16)
    yield "reversed_src", 8, SegmentLayout.packed(O.random_layout_sizes(8, 12, 4099), align=256,
                                                  src_order=list(reversed(range(12))))
    yield "resnet_like_161", 9, SegmentLayout.packed(O.random_layout_sizes(9, 161, 200_003), align=256)
    yield "big_ragged_3M", 10, SegmentLayout.packed(O.random_layout_sizes(10, 40, 3_000_017), align=256)
    yield "extra_tail_padding", 11, SegmentLayout((0, 5), (0, 256), (5, 17), 22, 1024)


def main():
    _build.build_oracle()
    out = []
    for name, seed, lay in cases():
        db = O.db_bytes(seed, lay.packed_bytes)
        seg_c, cs_c = O.land_c(db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
        seg_n, cs_n = O.land_np(db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
        assert cs_c == cs_n and (seg_c == seg_n).all(), name
        if lay.seg_bytes <= 300_000:
            seg_p = py_land(db.tobytes(), lay)
            assert seg_p == seg_c.tobytes(), name
            assert py_checksum(seg_p) == cs_c, name
        out.append({"name": name, "seed": seed, "packed_bytes": lay.packed_bytes,
                    "src_off": list(lay.src_off), "dst_off": list(lay.dst_off), "length": list(lay.length),
                    "seg_bytes": lay.seg_bytes, "checksum": f"{cs_c:016x}",
                    "seg_sha256": hashlib.sha256(seg_c.tobytes()).hexdigest()})
    path = Path(__file__).with_name("land_vectors.json")
    path.write_text(json.dumps({"spec": "oracle/sage_oracle.c", "cases": out}, indent=1) + "\n")
    print(f"wrote {len(out)} cases to {path}")


if __name__ == "__main__":
    main()
