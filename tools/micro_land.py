"""Microbenchmarks of the load path (not the bench contract; a probe):
land from HBM, H2D pipeline from pageable / pinned sources, checksum verify."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2404_14691_b200 import _lib  # noqa: E402
from paper_2404_14691_b200 import device as D  # noqa: E402
from paper_2404_14691_b200.layout import SegmentLayout  # noqa: E402


def main():
    chunk = int(sys.argv[1]) << 20 if len(sys.argv) > 1 else 8 << 20
    _lib.init(n_gpus=1, pool_bytes=64 << 30, staging_bytes=8 * chunk, chunk_bytes=chunk)
    out = {"chunk_MiB": chunk >> 20}
    S = 100 << 20
    lay = SegmentLayout.packed(O.random_layout_sizes(1, 161, S), align=256)
    db = O.db_bytes(1, lay.packed_bytes)
    _, want = O.land_c(db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
    seg = D.pool_alloc(0, lay.seg_bytes, _lib.CLASS_READ_ONLY)
    src = D.pool_alloc(0, lay.packed_bytes + 64, _lib.CLASS_WRITABLE)
    up = D.load(0, src.dptr, db, None); up.wait(); up.release()
    # land from HBM
    for rep in range(3):
        ops = [D.load(0, seg.dptr, None, lay, device_src=src.dptr, device_src_bytes=lay.packed_bytes)
               for _ in range(20)]
        t0 = time.perf_counter()
        res = [o.wait() for o in ops]
        first, last = res[0], res[-1]
        dt_us = last.gpu_end_us - first.gpu_begin_us
        assert all(r.checksum == want for r in res)
        out[f"land_hbm_rep{rep}"] = {"per_launch_us": dt_us / 20,
                                     "GBps_alg": 20 * (lay.packed_bytes + lay.seg_bytes) / (dt_us * 1e3)}
        for o in ops:
            o.release()
    # H2D pipeline, pageable and pinned
    pb = D.PinnedBuffer(lay.packed_bytes)
    pb.view()[:] = db
    for mode in ("pageable", "pinned"):
        for rep in range(3):
            op = D.load(0, seg.dptr, db if mode == "pageable" else pb, lay)
            r = op.wait()
            assert r.checksum == want
            us = r.gpu_end_us - min(r.gpu_begin_us, r.cpu_begin_us if r.cpu_begin_us >= 0 else 1 << 62)
            out[f"h2d_{mode}_rep{rep}"] = {"us": us, "GBps": lay.packed_bytes / (us * 1e3),
                                          "cpu_us": r.cpu_end_us - r.cpu_begin_us, "chunks": r.chunks}
            op.release()
    # 16 concurrent loads of distinct segments (pageable)
    segs = [D.pool_alloc(0, lay.seg_bytes, _lib.CLASS_READ_ONLY) for _ in range(4)]
    t0 = D.now_us()
    ops = [D.load(0, s.dptr, db, lay) for s in segs]
    rs = [o.wait() for o in ops]
    t1 = max(r.gpu_end_us for r in rs)
    out["h2d_4x_pageable_GBps"] = 4 * lay.packed_bytes / ((t1 - t0) * 1e3)
    for o in ops:
        o.release()
    for s in segs:
        s.free()
    # checksum verify
    t0 = time.perf_counter()
    for _ in range(10):
        assert D.segment_checksum(0, seg.dptr, lay.seg_bytes) == want
    out["verify_GBps_wall"] = 10 * lay.seg_bytes / ((time.perf_counter() - t0) * 1e9)
    print(json.dumps(out, indent=1))
    _lib.shutdown()


if __name__ == "__main__":
    main()
