"""Native ResNet-50 body alone: one landed BF16 record, K forwards on one
stream (latency) and on S streams at once (throughput), CUDA events.
python tools/prof_resnet_native.py [batch] [streams] [iters]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2404_14691_b200 import _lib, dnn  # noqa: E402
from paper_2404_14691_b200 import device as D  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 8
streams = int(sys.argv[2]) if len(sys.argv) > 2 else 4
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
_lib.init(n_gpus=1, pool_bytes=16 << 30)
spec, fd = dnn.resnet50_native(batch=batch, seed=0)
h = dnn.native_handle(fd)
seg = D.pool_alloc(0, fd.layout.seg_bytes, _lib.CLASS_READ_ONLY)
op = D.load(0, seg.dptr, fd.db, fd.layout)
op.wait()
op.release()
wr = []
for _ in range(streams):
    w = D.pool_alloc(0, spec.writable_bytes, _lib.CLASS_WRITABLE)
    up = D.load(0, w.dptr, fd.input, None)
    up.wait()
    up.release()
    wr.append(w)
in_b = (fd.input_bytes + 16 + 255) // 256 * 256
bodies = [D.body_desc(_lib.BODY_RESNET50, ro=seg.dptr, ro_bytes=fd.layout.seg_bytes, inp=w.dptr,
                      inp_bytes=(fd.input_bytes + 15) // 16 * 16, out=w.dptr + in_b, out_bytes=fd.out_bytes,
                      args=(h, batch)) for w in wr]
slots = [D.Slot(0) for _ in range(streams)]


def run(nst, k):
    evs = []
    for it in range(k):
        for s in range(nst):
            evs.append(slots[s].launch(bodies[s]))
    for b, e in evs:
        e.sync()
    first, last = evs[0][0], evs[-1][1]
    d = D.C.c_double()
    _lib.check(_lib.lib().sage_event_elapsed(first.h, last.h, D.C.byref(d)), "elapsed")
    per = []
    for b, e in evs:
        x = D.C.c_double()
        _lib.lib().sage_event_elapsed(b.h, e.h, D.C.byref(x))
        per.append(x.value)
    for b, e in evs:
        b.release()
        e.release()
    return d.value, per


run(1, 3)
run(streams, 3)
t1, per1 = run(1, iters)
t0 = time.perf_counter()
tS, perS = run(streams, iters)
host = time.perf_counter() - t0
flops = 2 * 4.09e9 * batch
print(json.dumps({"batch": batch, "one_stream_ms_per_forward": round(t1 / iters / 1e3, 3),
                  "one_stream_images_per_s": round(batch * iters / (t1 / 1e6), 1),
                  "streams": streams, "concurrent_images_per_s": round(batch * iters * streams / (tS / 1e6), 1),
                  "concurrent_tflops": round(flops * iters * streams / (tS / 1e6) / 1e12, 1),
                  "host_launch_s": round(host, 3), "median_forward_us_concurrent": round(float(np.median(perS)), 1)}))
_lib.shutdown()
