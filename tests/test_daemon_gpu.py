"""Memory daemon and function engine in separate processes on one GPU
(paper_2404_14691_b200/daemon.py): the daemon
lands a function's read-only segment once, the engine process maps it
zero-copy from a POSIX file descriptor (SageLoadToGPU), reads exactly the
oracle's bytes through the mapping, a second load shares it (Stage1Hot, no
second land), and SageDumpToDB persists the engine's bytes in the daemon."""
import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent

ENGINE = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2404_14691_b200 import _lib
from paper_2404_14691_b200 import device as D
from paper_2404_14691_b200.daemon import SageClient
_lib.init(n_gpus=1, pool_bytes=1 << 30, staging_bytes=16 << 20, chunk_bytes=4 << 20)
want = np.load(sys.argv[3])
cli = SageClient(sys.argv[2])
a = cli.load_to_gpu("fnA")
b = cli.load_to_gpu("fnA")
out = {"warmth": [a.warmth, b.warmth], "checksums": [a.checksum, b.checksum],
       "mapped_checksum": D.segment_checksum(0, a.dptr, a.seg_bytes),
       "bytes_equal": bool(np.array_equal(D.read_device(0, a.dptr, a.seg_bytes), want)),
       "same_pages": D.segment_checksum(0, b.dptr, b.seg_bytes) == D.segment_checksum(0, a.dptr, a.seg_bytes)}
cli.release(b)
cli.release(a)
cli.dump_to_db("result", np.arange(1000, dtype=np.float32))
cli.close()
_lib.shutdown()
print("ENGINE " + json.dumps(out))
"""


def test_daemon_engine_processes_share_a_segment(built, tmp_path):
    from conftest import gpu_available
    from paper_2404_14691_b200.daemon import MemoryDaemon
    from paper_2404_14691_b200.functions import load_spec_table
    from paper_2404_14691_b200.policies import policy_preset
    from paper_2404_14691_b200.runtime import ClusterSpec, Simulation
    if not gpu_available():
        pytest.fail("gpu test run without a visible CUDA device")
    table = load_spec_table({"fnA": {"ro_mem_mb": 64, "writable_mem_mb": 4, "compute_ms": 1}})
    with Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), table, seed=1) as sim:
        fd = sim.dataplane.data_for(table["fnA"])
        lay = fd.layout
        want_seg, want_sum = O.land_c(fd.db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
        np.save(tmp_path / "want.npy", want_seg)
        path = str(tmp_path / "sage.sock")
        daemon = MemoryDaemon(sim, path)
        eng = subprocess.Popen([sys.executable, "-c", ENGINE, str(ROOT), path, str(tmp_path / "want.npy")],
                               stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
        try:
            daemon.serve(clients=1, timeout_s=120)
        finally:
            out, err = eng.communicate(timeout=120)
            daemon.close()
        assert eng.returncode == 0, err[-3000:]
        res = json.loads([ln for ln in out.splitlines() if ln.startswith("ENGINE ")][-1][len("ENGINE "):])
        assert res["warmth"] == ["Cold", "Stage1Hot"]
        assert res["checksums"] == [want_sum, want_sum] and res["mapped_checksum"] == want_sum
        assert res["bytes_equal"] and res["same_pages"]
        assert daemon.loads == 1                                   # landed once for both loads
        assert np.array_equal(np.frombuffer(daemon.store["result"], np.float32), np.arange(1000, dtype=np.float32))
        # the engine released it: an invocation now finds the resident warm
        inv = sim.submit("fnA")
        sim.drain()
        assert inv.outcome == "completed" and inv.warmth.label() == "Stage1Hot"
        sim.sharing.check_consistency()
        sim.check_no_leaks()
