"""PCIe once per box across processes: the segment fan-out of BASELINE.json's
north star for the one-process-per-GPU layout (`bench.py --gpus N` under
torchrun).

The reference has no GPU-to-GPU path at all: every GPU owns an independent
PCIe channel behind one shared host channel (simulation.py:113-115), so in the
model N GPUs pull N copies of a read-only segment across the host
(SURVEY.md §8e).  Here each function has a HOME rank.  On the home rank a
cold leader loads the segment over PCIe as usual (stage → H2D → `land`);
the landed bytes are then broadcast over NVLink/NVSwitch (`ncclBroadcast`
through torch.distributed's NCCL group) into a receive buffer on every other
rank, where the leader's GPU_LOAD becomes an identity `land` from that buffer
(copy + checksum, so every rank verifies what it received).  Followers
everywhere wait on their local leader's RO-landed event as before.

Ordering: a broadcast is a collective, so every rank must issue them in the
same order.  They are issued at admission of a cold leader, from the
admitting thread; with the same burst on every rank (weak scaling) the cold
leaders -- and hence the broadcasts -- come in the same order everywhere.

In the same-process multi-GPU layout (`ClusterSpec(gpus=N)`) the peer `land`
of dataplane._peer_source does this job with direct NVLink loads instead.
"""
from __future__ import annotations

from typing import Callable, Optional

from . import device as D


class BoxFanout:
    """Home assignment + the broadcast step for one rank.

    `homes` maps function name -> home rank (default: position in `names`
    modulo the world size).  `broadcast(tensor, src)` is the collective; the
    default is torch.distributed's (NCCL)."""

    def __init__(self, rank: int, world: int, names, homes: Optional[dict] = None,
                 broadcast: Optional[Callable] = None):
        if world < 1 or not 0 <= rank < world:
            raise ValueError(f"bad rank {rank} / world {world}")
        self.rank, self.world = rank, world
        self.homes = dict(homes) if homes is not None else {n: k % world for k, n in enumerate(sorted(names))}
        self._bcast = broadcast or _torch_broadcast
        self.sent = 0          # segments this rank broadcast (as home)
        self.received = 0      # segments this rank received
        self.bytes_out = 0
        self.bytes_in = 0

    def home(self, name: str) -> int:
        return self.homes.get(name, 0)

    def is_home(self, name: str) -> bool:
        return self.home(name) == self.rank

    def publish(self, gpu: int, dptr: int, nbytes: int, landed: D.Event) -> D.Event:
        """Home side: broadcast the landed segment once `landed` completes.
        Returns the event that ends the send on this GPU."""
        slot = D.Slot(gpu)
        try:
            slot.wait([landed])      # blocks until the issuer has enqueued the load
            self._bcast(gpu, slot.stream(), dptr, nbytes, self.rank)
            ev = slot.record()
        finally:
            slot.release()
        self.sent += 1
        self.bytes_out += nbytes * (self.world - 1)
        return ev

    def receive(self, gpu: int, dptr: int, nbytes: int, name: str) -> D.Event:
        """Receiver side: the segment arrives from its home into dptr.  Returns
        the event after which the bytes are there."""
        slot = D.Slot(gpu)
        try:
            self._bcast(gpu, slot.stream(), dptr, nbytes, self.home(name))
            ev = slot.record()
        finally:
            slot.release()
        self.received += 1
        self.bytes_in += nbytes
        return ev

    def stats(self) -> dict:
        return {"rank": self.rank, "world": self.world, "sent": self.sent, "received": self.received,
                "nvlink_bytes_out": self.bytes_out, "nvlink_bytes_in": self.bytes_in}


def _torch_broadcast(gpu: int, stream: int, dptr: int, nbytes: int, src: int) -> None:
    """ncclBroadcast of nbytes at dptr from rank `src`, ordered on `stream`
    (torch.distributed's NCCL group; the default process group)."""
    import torch
    import torch.distributed as dist

    from .dnn import view
    dev = torch.device("cuda", torch.cuda.current_device())
    t = view(dptr, nbytes, dev)
    ext = torch.cuda.ExternalStream(stream, device=dev)
    with torch.cuda.stream(ext):
        work = dist.broadcast(t, src=src, async_op=True)
        work.wait()              # the slot stream waits for the collective
