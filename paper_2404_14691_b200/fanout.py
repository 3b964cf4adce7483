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

Two exchanges implement it:

  PeerFanout  (default) the home exports the landed segment's pages as a
              POSIX file descriptor and an interprocess event recorded after
              its land; each other rank maps the pages (over NVLink when they
              live on another GPU) and its cold leader's GPU_LOAD is ONE
              `land` launch reading the home's segment peer to peer and
              checksumming it -- transfer and verification fused, no copy
              through an intermediate buffer, device-side wait on the home's
              event.  Descriptors travel over Unix sockets between the ranks.
  BoxFanout   ncclBroadcast into a receive buffer, then a local land (the
              collective-library baseline).

In the same-process multi-GPU layout (`ClusterSpec(gpus=N)`) the peer `land`
of dataplane._peer_source does this job with direct NVLink loads instead.
"""
from __future__ import annotations

import os
import socket
import time
from typing import Callable, Optional

from . import _lib
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

    kind = "nccl"

    def fetch(self, gpu: int, name: str, nbytes: int, scratch: Callable[[int], object]):
        """Receiver side of the common interface: ("copy", buffer, event) --
        the bytes arrive in a scratch buffer from `scratch(nbytes)`."""
        buf = scratch(nbytes)
        return "copy", buf, self.receive(gpu, buf.dptr, nbytes, name)

    def reap(self) -> None:
        pass

    def close(self) -> None:
        pass

    def publish(self, gpu: int, dptr: int, nbytes: int, landed: D.Event, seg_handle: int = 0,
                name: str = "") -> D.Event:
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


# ------------------------------------------------------------ peer mapping ---
def _sock_path(sock_dir: str, job: str, rank: int) -> str:
    return os.path.join(sock_dir, f"sage-fan-{job}-{rank}.sock")


class PeerFanout(BoxFanout):
    """PCIe once per box with the receivers landing the home's segment peer
    to peer (see module docstring).  `barrier()` synchronises the ranks during
    the socket rendezvous (torch.distributed.barrier in bench.py)."""

    kind = "peer"

    def __init__(self, rank: int, world: int, names, homes: Optional[dict] = None, job: str = "sage",
                 sock_dir: str = "/tmp", barrier: Optional[Callable[[], None]] = None, timeout_s: float = 120.0):
        super().__init__(rank, world, names, homes, broadcast=lambda *a: None)
        from .daemon import _recv, _send
        self._recv, self._send = _recv, _send
        self.job, self.sock_dir = job, sock_dir
        self.imports: list = []          # (import handle, ipc event) per received segment
        self._pending: dict = {}         # home rank -> {fn: message, fds}
        path = _sock_path(sock_dir, job, rank)
        if os.path.exists(path):
            os.unlink(path)
        self._lsock = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        self._lsock.bind(path)
        self._lsock.listen(max(1, world))
        self._lsock.settimeout(timeout_s)
        self._barrier = barrier
        if barrier:
            barrier()                                 # everyone listens
        self.to_home: dict[int, socket.socket] = {}
        for h in range(world):                        # every other rank may be a home
            if h == rank:
                continue
            c = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            deadline = time.time() + timeout_s
            while True:
                try:
                    c.connect(_sock_path(sock_dir, job, h))
                    break
                except (FileNotFoundError, ConnectionRefusedError):
                    if time.time() > deadline:
                        raise
                    time.sleep(0.01)
            self._send(c, {"hello": rank})
            self.to_home[h] = c
        self.to_recv: dict[int, socket.socket] = {}
        for _ in range(world - 1):
            conn, _ = self._lsock.accept()
            conn.settimeout(timeout_s)
            self.to_recv[int(self._recv(conn)["hello"])] = conn
        if barrier:
            barrier()

    def publish(self, gpu: int, dptr: int, nbytes: int, landed: D.Event, seg_handle: int = 0,
                name: str = "") -> D.Event:
        """Home: export the segment's pages and an event recorded after its
        land to every other rank.  Returns the interprocess event (kept until
        the resident is evicted)."""
        L = _lib.lib()
        ev, ipc = _lib.H(), (_lib.C.c_ubyte * 64)()
        _lib.check(L.sage_ipc_event_export(landed.h, _lib.C.byref(ev), ipc), "sage_ipc_event_export")
        fd, phys = _lib.C.c_int(), _lib.u64()
        _lib.check(L.sage_pool_export(seg_handle, _lib.C.byref(fd), _lib.C.byref(phys)), "sage_pool_export")
        try:
            msg = {"fn": name, "phys": phys.value, "bytes": nbytes, "ipc": bytes(ipc).hex()}
            for r in sorted(self.to_recv):
                self._send(self.to_recv[r], msg, fds=[fd.value])
        finally:
            os.close(fd.value)
        self.sent += 1
        self.bytes_out += nbytes * (self.world - 1)
        return D.Event(ev.value)

    def _message_for(self, home: int, name: str):
        box = self._pending.setdefault(home, {})
        while name not in box:
            msg, fds = self._recv(self.to_home[home], with_fd=True)
            box[msg["fn"]] = (msg, fds)
        return box.pop(name)

    def fetch(self, gpu: int, name: str, nbytes: int, scratch=None):
        """Receiver: map the home's segment and open its landed event.
        Returns ("peer", device address, event to wait on)."""
        return self._fetch_from(self.home(name), gpu, name, nbytes)

    def _fetch_from(self, home: int, gpu: int, name: str, nbytes: int):
        msg, fds = self._message_for(home, name)
        if msg["bytes"] != nbytes:
            raise RuntimeError(f"{name}: home sent {msg['bytes']} B, expected {nbytes} B")
        L = _lib.lib()
        h, dptr = _lib.H(), _lib.u64()
        try:
            _lib.check(L.sage_segment_import(gpu, fds[0], msg["phys"], _lib.C.byref(h), _lib.C.byref(dptr)),
                       "sage_segment_import")
        finally:
            for f in fds:
                os.close(f)
        ev = _lib.H()
        ipc = (_lib.C.c_ubyte * 64).from_buffer_copy(bytes.fromhex(msg["ipc"]))
        _lib.check(L.sage_ipc_event_open(gpu, ipc, _lib.C.byref(ev)), "sage_ipc_event_open")
        self.imports.append((h.value, ev.value))
        self.received += 1
        self.bytes_in += nbytes
        return "peer", dptr.value, D.Event(ev.value)

    def selftest(self, gpu: int, nbytes: int = 1 << 20) -> bool:
        """Collective check of the whole exchange before any function uses
        it: every rank lands a rank-specific byte pattern and publishes the
        pages; every rank then lands each peer's pages peer to peer (export /
        import / interprocess event / `land` reading the peer) and compares the
        checksum with a local land of the same pattern.  Returns whether this
        rank's checks passed; the caller agrees across ranks and falls back
        when any failed.  `barrier` must be set (peers read this rank's pages
        until every rank is done)."""
        import numpy as np

        def pattern(r: int) -> np.ndarray:
            return np.random.Generator(np.random.PCG64(1000 + r)).integers(0, 256, nbytes, dtype=np.uint8)

        mine = D.pool_alloc(gpu, nbytes, _lib.CLASS_READ_ONLY, unaccounted=True)
        tmp = D.pool_alloc(gpu, nbytes, _lib.CLASS_WRITABLE, unaccounted=True)
        sent, ok = None, True
        stats = (self.sent, self.received, self.bytes_out, self.bytes_in)
        try:
            op = D.load(gpu, mine.dptr, pattern(self.rank))
            op.wait()
            sent = self.publish(gpu, mine.dptr, nbytes, op.end, seg_handle=mine.h, name=f"__selftest_{self.rank}")
            op.release()
            for h in range(self.world):
                if h == self.rank:
                    continue
                _, src, ev = self._fetch_from(h, gpu, f"__selftest_{h}", nbytes)
                got = D.load(gpu, tmp.dptr, None, None, device_src=src, device_src_bytes=nbytes, peer_gpu=gpu,
                             wait=[ev])
                want = D.load(gpu, tmp.dptr, pattern(h), wait=[got.end])
                a, b = got.wait().checksum, want.wait().checksum
                got.release()
                want.release()
                ok = ok and a == b and a != 0
        except Exception as e:   # noqa: BLE001 -- any failure means "do not use this exchange"
            print(f"sage fanout selftest (rank {self.rank}): {e}", flush=True)
            ok = False
        finally:
            if self._barrier:
                self._barrier()                  # peers are done reading `mine`
            try:
                self.reap()
            except Exception:   # noqa: BLE001
                ok = False
            if sent is not None:
                sent.release()
            mine.free()
            tmp.free()
            self.sent, self.received, self.bytes_out, self.bytes_in = stats
        return ok

    def link_probe(self, gpu: int, nbytes: int = 256 << 20, iters: int = 5) -> dict:
        """Collective NVLink measurement of the fan-out step itself: every
        rank lands `nbytes` and publishes the pages; every rank then lands each
        peer's pages `iters` times with the peer-reading `land` (identity
        layout, checksum fused: exactly the receive side of a fan-out) and
        times each with its device events.  Returns this rank's median GB/s
        per peer (segment bytes / land time)."""
        import numpy as np
        mine = D.pool_alloc(gpu, nbytes, _lib.CLASS_READ_ONLY, unaccounted=True)
        tmp = D.pool_alloc(gpu, nbytes, _lib.CLASS_WRITABLE, unaccounted=True)
        stats = (self.sent, self.received, self.bytes_out, self.bytes_in)
        sent, out = None, {}
        try:
            op = D.load(gpu, mine.dptr, np.full(nbytes, self.rank + 1, np.uint8))
            op.wait()
            sent = self.publish(gpu, mine.dptr, nbytes, op.end, seg_handle=mine.h, name=f"__probe_{self.rank}")
            op.release()
            for h in range(self.world):
                if h == self.rank:
                    continue
                _, src, ev = self._fetch_from(h, gpu, f"__probe_{h}", nbytes)
                ev.sync()
                us = []
                for _ in range(iters + 1):
                    ld = D.load(gpu, tmp.dptr, None, None, device_src=src, device_src_bytes=nbytes, peer_gpu=gpu)
                    info = ld.wait()
                    us.append(info.gpu_end_us - info.gpu_begin_us)
                    ld.release()
                t = float(np.median(us[1:]))
                out[h] = round(nbytes / (t * 1e-6) / 1e9, 1) if t > 0 else None
        finally:
            if self._barrier:
                self._barrier()                  # peers are done reading `mine`
            self.reap()
            if sent is not None:
                sent.release()
            mine.free()
            tmp.free()
            self.sent, self.received, self.bytes_out, self.bytes_in = stats
        return out

    def reap(self) -> None:
        """Unmap every received segment; call when no device work reads them
        (after the burst that landed them drained)."""
        L = _lib.lib()
        for h, ev in self.imports:
            _lib.check(L.sage_segment_unimport(h), "sage_segment_unimport")
        self.imports.clear()

    def close(self) -> None:
        self.reap()
        for box in self._pending.values():          # descriptors received but never used
            for _msg, fds in box.values():
                for f in fds:
                    os.close(f)
        self._pending.clear()
        for c in list(self.to_home.values()) + list(self.to_recv.values()):
            c.close()
        self._lsock.close()
        path = _sock_path(self.sock_dir, self.job, self.rank)
        if os.path.exists(path):
            os.unlink(path)
