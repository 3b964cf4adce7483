"""3xTF32 sgemm: one small shape per process (run under `timeout`), prints
max error vs float64 numpy.  python tools/x3_debug.py M N K"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2404_14691_b200 import _lib  # noqa: E402
from paper_2404_14691_b200 import device as D  # noqa: E402

m, n, k = map(int, sys.argv[1:4])
_lib.init(n_gpus=1, pool_bytes=4 << 30)
rng = np.random.default_rng(0)
A = rng.standard_normal((m, k), dtype=np.float32)
BT = rng.standard_normal((n, k), dtype=np.float32)
segs = []
for arr in (A, BT):
    s = D.pool_alloc(0, arr.nbytes + 256, _lib.CLASS_WRITABLE)
    op = D.load(0, s.dptr, arr.view(np.uint8).reshape(-1), None)
    op.wait()
    op.release()
    segs.append(s)
out = D.pool_alloc(0, m * n * 4 + 256, _lib.CLASS_WRITABLE)
slot = D.Slot(0)
b, e = slot.launch(D.body_desc(_lib.BODY_SGEMM, ro=segs[0].dptr, ro_bytes=A.nbytes, inp=segs[1].dptr,
                               inp_bytes=BT.nbytes, out=out.dptr, out_bytes=m * n * 4, args=(m, n, k)))
e.sync()
got = D.read_device(0, out.dptr, m * n * 4).view(np.float32).reshape(m, n)
want = A.astype(np.float64) @ BT.T.astype(np.float64)
print(f"{m}x{n}x{k}: rel err {np.abs(got - want).max() / np.abs(want).max():.3e}", flush=True)
_lib.shutdown()
