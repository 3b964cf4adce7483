"""Stencil variant timing at the cfg-2 shape (256 x 256 x 64): 200 launches
back to back on one slot, device time per launch; output hash for parity.
Usage: SAGE_STENCIL=<0|2|4|8|16> python tools/stencil_sweep.py"""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14691_b200 import _lib
from paper_2404_14691_b200 import device as D


def main():
    nx, ny, nz, n = 256, 256, 64, 200
    _lib.init(n_gpus=1, pool_bytes=8 << 30, staging_bytes=64 << 20, chunk_bytes=8 << 20)
    rng = np.random.default_rng(1)
    coef = rng.uniform(0.2, 0.6, (nz, ny, nx)).astype(np.float32)
    grid = rng.standard_normal((nz, ny, nx), dtype=np.float32)
    segs = []
    for a in (coef, grid):
        u = a.view(np.uint8).reshape(-1)
        seg = D.pool_alloc(0, u.size + 256, _lib.CLASS_WRITABLE, unaccounted=True)
        op = D.load(0, seg.dptr, u, None); op.wait(); op.release()
        segs.append(seg)
    out = D.pool_alloc(0, grid.nbytes + 256, _lib.CLASS_WRITABLE, unaccounted=True)
    bits = int(np.float32(0.1).view(np.int32))
    desc = D.body_desc(_lib.BODY_STENCIL, ro=segs[0].dptr, ro_bytes=coef.nbytes, inp=segs[1].dptr,
                       inp_bytes=grid.nbytes, out=out.dptr, out_bytes=grid.nbytes, args=(nx, ny, nz, bits))
    slot = D.Slot(0)
    best = None
    for rep in range(3):
        evs = [slot.launch(desc) for _ in range(n)]
        evs[-1][1].sync()
        t = (evs[-1][1].time_us() - evs[0][0].time_us()) / n
        best = t if best is None else min(best, t)
        for b, e in evs:
            b.release(); e.release()
    got = D.read_device(0, out.dptr, grid.nbytes)
    print(f"SAGE_STENCIL={os.environ.get('SAGE_STENCIL', '0')} us_per_launch={best:.2f} "
          f"GBps={12 * nx * ny * nz / best / 1e3:.0f} sha={hashlib.sha256(got.tobytes()).hexdigest()[:16]}")
    slot.release()
    _lib.shutdown()


if __name__ == "__main__":
    main()
