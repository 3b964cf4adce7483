"""bench.py's N>1 plumbing on CPU: two ranks over gloo (world size 2).

The driver launches `bench.py` under torchrun with one rank per GPU; the
timing contract is barrier + max-over-ranks of device time and a whole-job
sum of invocations.  These helpers are exercised here with the gloo backend
(127.0.0.1 rendezvous), as the GPU runs in this round are single-GPU."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r, w, local = bench._rank_env()
        bench.barrier(dist)
        mx = bench.max_over_ranks(dist, 10.0 + rank)          # per-rank elapsed µs
        sm = bench.sum_over_ranks(dist, 64.0)                 # per-rank invocations
        # box fan-out: every rank derives the same homes; the checksum check
        # agrees when ranks landed identical bytes and not otherwise
        from paper_2404_14691_b200.fanout import BoxFanout

        class _FD:
            def __init__(self, c):
                self.ro_checksum = c
        homes = BoxFanout(rank, world, ["spmv", "sgemm", "stencil"]).homes
        same = bench.ro_checksums_agree(dist, {"a": _FD(0xFEDCBA9876543210), "b": _FD(7)})
        differ = bench.ro_checksums_agree(dist, {"a": _FD(0xFEDCBA9876543210 + rank), "b": _FD(7)})
        q.put((r, w, local, os.environ.get("SAGE_DEVICE_OFFSET"), mx, sm, sorted(homes.items()), same, differ))
    finally:
        dist.destroy_process_group()


def test_two_rank_max_and_sum_over_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [o[0] for o in out] == [0, 1]
    assert all(o[1] == 2 for o in out)
    assert [o[3] for o in out] == ["0", "1"]                  # one GPU per rank (library planes start there)
    assert all(o[4] == 11.0 for o in out)                      # max over ranks
    assert all(o[5] == 128.0 for o in out)                     # whole-job invocations
    assert out[0][6] == out[1][6] == [("sgemm", 0), ("spmv", 1), ("stencil", 0)]   # same homes on every rank
    assert all(o[7] is True and o[8] is False for o in out)


def test_weak_scaling_value_formula():
    # value = invocations of all ranks / max-over-ranks time
    invs_per_rank, ranks, max_us = 64 * 10, 4, 2_000.0
    assert (invs_per_rank * ranks) / (max_us / 1e6) == pytest.approx(1_280_000.0)
