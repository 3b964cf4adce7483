"""ncu driver: the cfg-2 spmv body (1 Mi rows x 16 nnz, CSR landed from HBM)
launched back to back.  ncu --set full -k regex:spmv4 -s 2 -c 1 python tools/prof_spmv.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2404_14691_b200 import _lib  # noqa: E402
from paper_2404_14691_b200 import device as D  # noqa: E402
from paper_2404_14691_b200.parboil import spmv  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 5
fmt = sys.argv[2] if len(sys.argv) > 2 else "csr"
kw = {}
for a in sys.argv[3:]:                      # csb builder knobs, e.g. chunk_cols=4096 stages=6 slices=2
    k, v = a.split("=")
    kw[k] = int(v)
_lib.init(n_gpus=1, pool_bytes=8 << 30)
spec, fd = spmv(fmt=fmt, csb_opts=kw or None)
seg = D.pool_alloc(0, fd.layout.seg_bytes, _lib.CLASS_READ_ONLY)
op = D.load(0, seg.dptr, fd.db, fd.layout)
op.wait()
op.release()
x = D.pool_alloc(0, fd.input_bytes + 256, _lib.CLASS_WRITABLE)
op = D.load(0, x.dptr, fd.input, None)
op.wait()
op.release()
y = D.pool_alloc(0, fd.out_bytes + 256, _lib.CLASS_WRITABLE)
slot = D.Slot(0)
body = D.body_desc(_lib.BODY_SPMV_CSB if fmt == "csb" else _lib.BODY_SPMV, ro=seg.dptr, ro_bytes=fd.layout.seg_bytes, inp=x.dptr, inp_bytes=fd.input_bytes,
                   out=y.dptr, out_bytes=fd.out_bytes, args=fd.args)
evs = [slot.launch(body) for _ in range(iters)]
evs[-1][1].sync()
us = []
for b, e in evs[1:]:
    d = D.C.c_double()
    _lib.check(_lib.lib().sage_event_elapsed(b.h, e.h, D.C.byref(d)), "elapsed")
    us.append(d.value)
us.sort()
nnz = (fd.args[7] >> 8) if fmt == "csb" else fd.args[1]
alg = 4 * (fd.args[0] + 1) + 12 * nnz + 4 * fd.args[0]      # the CSR algorithmic bytes, both formats
print(f"spmv[{fmt}] {fd.args[0]} rows x {nnz // fd.args[0]} nnz: median {us[len(us) // 2]:.1f} us = "
      f"{alg / us[len(us) // 2] / 1e3:.0f} GB/s algorithmic")
_lib.shutdown()
