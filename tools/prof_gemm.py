"""ncu driver: the cfg-2 sgemm shape (4096 x 256 x 4096, tcgen05; SAGE_SGEMM_PASSES picks 3xTF32 or TF32) launched
back to back.  ncu -k regex:sgemm_tf32 -c 2 python tools/prof_gemm.py"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2404_14691_b200 import _lib  # noqa: E402
from paper_2404_14691_b200 import device as D  # noqa: E402

m, n, k = 4096, 256, 4096
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
_lib.init(n_gpus=1, pool_bytes=8 << 30)
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
out = D.pool_alloc(0, m * n * 4, _lib.CLASS_WRITABLE)
slot = D.Slot(0)
body = D.body_desc(_lib.BODY_SGEMM, ro=segs[0].dptr, ro_bytes=A.nbytes, inp=segs[1].dptr, inp_bytes=BT.nbytes,
                   out=out.dptr, out_bytes=m * n * 4, args=(m, n, k))
t0 = time.perf_counter()
evs = [slot.launch(body) for _ in range(iters)]
host_us = (time.perf_counter() - t0) / iters * 1e6
evs[-1][1].sync()
us = []
for b, e in evs[2:]:
    a_, b_ = D.H(), D.H()
    d = D.C.c_double()
    _lib.check(_lib.lib().sage_event_elapsed(b.h, e.h, D.C.byref(d)), "elapsed")
    us.append(d.value)
import json, os  # noqa: E402
print(json.dumps({"sgemm": f"{m}x{n}x{k}", "passes": os.environ.get("SAGE_SGEMM_PASSES", "3"), "bn": os.environ.get("SAGE_SGEMM_BN", "auto"), "median_us": round(float(np.median(us)), 2), "host_enqueue_us": round(host_us, 2), "tflops_alg": round(2 * m * n * k / np.median(us) / 1e6, 1)}))
_lib.shutdown()
