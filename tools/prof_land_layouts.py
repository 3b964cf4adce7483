"""Land throughput by layout, HBM-resident sources (probe): the bench probe
(spmv, 3 tensors), a 161-tensor ragged 100 MiB record, and ResNet-50's 320
parameter tensors (many of them 1 KB BatchNorm vectors).  20 back-to-back
lands each, CUDA events on the land stream."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import oracle as O  # noqa: E402
from paper_2404_14691_b200 import _lib  # noqa: E402
from paper_2404_14691_b200 import device as D  # noqa: E402
from paper_2404_14691_b200.layout import SegmentLayout  # noqa: E402
from paper_2404_14691_b200.parboil import spmv  # noqa: E402

_lib.init(n_gpus=1, pool_bytes=16 << 30, staging_bytes=64 << 20, chunk_bytes=8 << 20)
L = _lib.lib()
cases = {}
_, fd = spmv()
cases["spmv_3_tensors"] = (fd.layout, fd.db)
lay = SegmentLayout.packed(O.random_layout_sizes(1, 161, 100 << 20), align=256)
cases["ragged_161_tensors"] = (lay, O.db_bytes(1, lay.packed_bytes))
try:
    from paper_2404_14691_b200.dnn import resnet50
    _, rfd = resnet50()
    cases["resnet50_320_tensors"] = (rfd.layout, rfd.db)
except Exception as exc:  # torchvision missing
    print("resnet50 skipped:", exc)
out = {}
for name, (lay, db) in cases.items():
    seg = D.pool_alloc(0, lay.seg_bytes, _lib.CLASS_READ_ONLY)
    src = D.pool_alloc(0, lay.packed_bytes + 64, _lib.CLASS_WRITABLE)
    up = D.load(0, src.dptr, db, None)
    up.wait()
    up.release()
    _lib.check(L.sage_stats_enable(1), "stats")
    _lib.check(L.sage_stats_reset(), "reset")
    ops = [D.load(0, seg.dptr, None, lay, device_src=src.dptr, device_src_bytes=lay.packed_bytes) for _ in range(20)]
    sums = {op.wait().checksum for op in ops}
    for op in ops:
        op.release()
    n, t, b = _lib.u64(), _lib.C.c_double(), _lib.u64()
    _lib.check(L.sage_stats_get(0, 0, _lib.C.byref(n), _lib.C.byref(t), _lib.C.byref(b)), "get")
    out[name] = {"tensors": lay.n, "seg_bytes": lay.seg_bytes, "launches": n.value,
                 "us_per_land": round(t.value / 20, 2), "GBps": round(b.value / t.value / 1e3, 1),
                 "checksums_identical": len(sums) == 1}
    seg.free()
    src.free()
print(json.dumps(out, indent=1))
_lib.shutdown()
