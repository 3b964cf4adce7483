"""Profiling driver for ncu: HBM-resident lands of the bench's probe segment
(spmv, 132 MiB, 3 tensors, packed in reverse order) after one upload.
The upload is an identity load of 132 MiB = 17 chunk launches:
ncu -k regex:land_kernel -s 17 -c 2 python tools/prof_land.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2404_14691_b200 import _lib  # noqa: E402
from paper_2404_14691_b200 import device as D  # noqa: E402
from paper_2404_14691_b200.parboil import spmv  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 5
_lib.init(n_gpus=1, pool_bytes=16 << 30, staging_bytes=64 << 20, chunk_bytes=8 << 20)
spec, fd = spmv()
lay = fd.layout
seg = D.pool_alloc(0, lay.seg_bytes, _lib.CLASS_READ_ONLY)
src = D.pool_alloc(0, lay.packed_bytes + 64, _lib.CLASS_WRITABLE)
up = D.load(0, src.dptr, fd.db, None)
up.wait()
up.release()
for _ in range(iters):
    op = D.load(0, seg.dptr, None, lay, device_src=src.dptr, device_src_bytes=lay.packed_bytes)
    r = op.wait()
    op.release()
print("ok", hex(r.checksum))
_lib.shutdown()
