"""Profiling driver for ncu: one 100 MiB HBM-resident land per iteration
(after a 13-launch upload).  Under ncu use -k regex:land_kernel -s 13."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import oracle as O  # noqa: E402
from paper_2404_14691_b200 import _lib  # noqa: E402
from paper_2404_14691_b200 import device as D  # noqa: E402
from paper_2404_14691_b200.layout import SegmentLayout  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 5
_lib.init(n_gpus=1, pool_bytes=16 << 30, staging_bytes=64 << 20, chunk_bytes=8 << 20)
lay = SegmentLayout.packed(O.random_layout_sizes(1, 161, 100 << 20), align=256)
db = O.db_bytes(1, lay.packed_bytes)
seg = D.pool_alloc(0, lay.seg_bytes, _lib.CLASS_READ_ONLY)
src = D.pool_alloc(0, lay.packed_bytes + 64, _lib.CLASS_WRITABLE)
up = D.load(0, src.dptr, db, None)
up.wait()
up.release()
for _ in range(iters):
    op = D.load(0, seg.dptr, None, lay, device_src=src.dptr, device_src_bytes=lay.packed_bytes)
    r = op.wait()
    op.release()
print("ok", r.checksum)
_lib.shutdown()
