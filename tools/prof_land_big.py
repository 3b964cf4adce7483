"""land of a 1 GiB multi-tensor segment (8x the 126 MB L2) from an
HBM-resident packed record, timed with the load's device events; the
roofline evidence for `land` away from L2 effects.
python tools/prof_land_big.py [GiB] [iters]
ncu: the host upload is 128 staged chunk lands, then one 1 GiB land per
iteration: ncu -k regex:land_kernel -s 128 -c 1 python tools/prof_land_big.py 1 1"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2404_14691_b200 import _lib  # noqa: E402
from paper_2404_14691_b200 import device as D  # noqa: E402
from paper_2404_14691_b200.layout import SegmentLayout  # noqa: E402

gib = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
total = int(gib * (1 << 30)) // 4096 * 4096
sizes = [total // 8 - 37 * k for k in range(8)]          # 8 ragged tensors
lay = SegmentLayout.packed(sizes, align=256)
_lib.init(n_gpus=1, pool_bytes=16 << 30, staging_bytes=64 << 20, chunk_bytes=8 << 20)
db = np.random.default_rng(1).integers(0, 256, lay.packed_bytes, dtype=np.uint8)
src = D.pool_alloc(0, lay.packed_bytes + 64, _lib.CLASS_WRITABLE)
seg = D.pool_alloc(0, lay.seg_bytes, _lib.CLASS_READ_ONLY)
up = D.load(0, src.dptr, db, None)
up.wait()
up.release()
res = []
for _ in range(iters):
    op = D.load(0, seg.dptr, None, lay, device_src=src.dptr, device_src_bytes=lay.packed_bytes)
    r = op.wait()
    res.append(r.gpu_end_us - r.gpu_begin_us)
    op.release()
us = float(np.median(res))
alg = lay.packed_bytes + lay.seg_bytes
print(json.dumps({"segment_bytes": lay.seg_bytes, "tensors": 8, "median_us": us, "alg_bytes": alg,
                  "GBps_alg": round(alg / us / 1e3, 1)}))
_lib.shutdown()
