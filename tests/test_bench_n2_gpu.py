"""bench.py's N > 1 path end to end (torchrun, one process per rank, the p2p
fan-out, max-over-ranks timing, cross-rank checksum agreement) with both
ranks on the one GPU of a single-GPU box (SAGE_BENCH_SHARE_GPU=1 -- plumbing,
not a measurement)."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def run_n2(extra_env=None) -> dict:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, SAGE_BENCH_SHARE_GPU="1", **(extra_env or {}))
    res = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"),
                          "--gpus", "2", "--steps", "2", "--warmup", "3", "--burst", "12", "--no-cfg1",
                          "--no-cpu-baseline"], capture_output=True, text=True, env=env, timeout=900, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-4000:]
    return json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1])


def test_bench_two_ranks_shared_gpu(built):
    """The p2p fan-out passes its collective selftest and carries the segments."""
    from conftest import gpu_available
    if not gpu_available():
        pytest.fail("gpu test run without a visible CUDA device")
    line = run_n2()
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["e2e"]["value"] > 0
    f = line["fanout"]
    assert f["ro_checksums_agree"] is True
    assert f["rank0"]["sent"] > 0 and f["rank0"]["received"] > 0 and f["nvlink_bytes_in_all_ranks"] > 0


def test_bench_falls_back_when_a_rank_fails_the_fanout_selftest(built):
    """One rank failing the selftest (injected) makes every rank load over its
    own PCIe; the run still completes and says so."""
    from conftest import gpu_available
    if not gpu_available():
        pytest.fail("gpu test run without a visible CUDA device")
    line = run_n2({"SAGE_FANOUT_SELFTEST_FAIL": "1"})
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["e2e"]["value"] > 0
    assert "fallback" in line["fanout"]
