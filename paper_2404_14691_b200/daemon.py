"""The memory daemon and the function-engine client across processes
(the paper's architecture).

In SAGE a per-GPU unified memory daemon prepares functions' read-only data
and the function engines -- separate processes -- obtain it with
`SageLoadToGPU` (a device pointer to the data, no copy) and persist writable
results with `SageDumpToDB`.  Here the daemon is a Simulation (the B200
plane with the reference's sharing semantics) serving a Unix socket:

  load(fn)     admit fn's resident on the GPU (the same SharingManager admit
               as an invocation: warmth classes, leader election, ledger),
               land its read-only segment if this admission leads (and
               verify its checksum), then export the segment's pages as a
               POSIX file descriptor (SCM_RIGHTS) with its layout; the
               client maps them zero-copy (sage_segment_import)
  release(fn)  the client is done: SharingManager.release (decay timers start
               when the last user leaves, as for invocations)
  dump(key)    bytes the engine persists (SageDumpToDB) into the daemon's
               host store

Messages are length-prefixed JSON; requests are served on the daemon's own
thread (`serve`), never concurrently with its engine loop.
"""
from __future__ import annotations

import json
import os
import socket
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from . import device as D


def _send(sock: socket.socket, obj: dict, fds=()) -> None:
    data = json.dumps(obj).encode()
    msg = struct.pack("<I", len(data)) + data
    if fds:
        socket.send_fds(sock, [msg], list(fds))
    else:
        sock.sendall(msg)


def _recv_exact(sock: socket.socket, n: int) -> bytes:
    buf = b""
    while len(buf) < n:
        part = sock.recv(n - len(buf))
        if not part:
            raise ConnectionError("peer closed")
        buf += part
    return buf


def _recv(sock: socket.socket, with_fd: bool = False):
    fds = []
    if with_fd:
        head, fds, _, _ = socket.recv_fds(sock, 4, 4)
        if len(head) < 4:
            head += _recv_exact(sock, 4 - len(head))
    else:
        head = _recv_exact(sock, 4)
    (n,) = struct.unpack("<I", head)
    obj = json.loads(_recv_exact(sock, n))
    return (obj, fds) if with_fd else obj


class MemoryDaemon:
    """Serves load / release / dump for the functions of one Simulation."""

    def __init__(self, sim, path: str, gpu: int = 0):
        self.sim, self.path, self.gpu = sim, path, gpu
        self.store: dict[str, bytes] = {}
        self.loads = 0
        if os.path.exists(path):
            os.unlink(path)
        self.sock = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        self.sock.bind(path)
        self.sock.listen(8)

    # -- requests --------------------------------------------------------------
    def _attach(self, name: str) -> tuple[dict, int]:
        from .resources import SimulationError
        sim, gpu = self.sim, self.gpu
        spec = sim.spec_table[name]
        fd = sim.dataplane.data_for(spec)
        sharing = sim.sharing
        if sharing is None:
            raise SimulationError("the memory daemon needs a sharing policy (SAGE / SAGE_NR)")
        preview = sharing.preview(spec, gpu)
        ledger = sim.gpu_ledgers[gpu]
        if not ledger.fits(preview.resident_delta) and not sharing.force_demote(gpu, preview.resident_delta, name):
            raise SimulationError(f"{name}: no room for its read-only segment")
        grant = sharing.admit(spec, gpu, preview)
        try:
            return self._land_and_export(name, grant, fd)
        except Exception:
            sharing.release(name, gpu)       # the engine never got it: undo the admission
            raise

    def _land_and_export(self, name: str, grant, fd) -> tuple[dict, int]:
        from .resources import SimulationError
        sim, gpu = self.sim, self.gpu
        r = grant.resident
        if r.gpu_ro is None:
            raise SimulationError(f"{name}: no read-only segment (ro_sharing off?)")
        if grant.leader_ro:
            op = D.load(gpu, r.gpu_ro.dptr, fd.db, fd.layout)
            res = op.wait()
            op.release()
            if fd.ro_checksum is None:
                fd.ro_checksum = res.checksum
            elif fd.ro_checksum != res.checksum:
                raise SimulationError(f"{name}: landed checksum {res.checksum:016x} != {fd.ro_checksum:016x}")
            sim.sharing.record_checksum(r, res.checksum)
            r.ro_token.set_ready(sim.engine.tick())
            self.loads += 1
        elif r.ro_token is not None and not r.ro_token.ready and r.ro_token.event is not None:
            r.ro_token.event.sync()          # an invocation is landing it right now
        if grant.leader_ctx and r.ctx_token is not None:
            r.ctx_token.set_ready(sim.engine.tick())
        fdn, phys = _lib.C.c_int(), _lib.u64()
        _lib.check(_lib.lib().sage_pool_export(r.gpu_ro.segment.h, _lib.C.byref(fdn), _lib.C.byref(phys)),
                   "sage_pool_export")
        lay = fd.layout
        meta = {"ok": True, "fn": name, "gpu": gpu, "phys_bytes": phys.value, "seg_bytes": lay.seg_bytes,
                "checksum": r.ro_checksum if r.ro_checksum is not None else fd.ro_checksum,
                "warmth": grant.warmth.label(), "tensors": [[int(o), int(n)] for o, n in zip(lay.dst_off, lay.length)],
                "names": list(lay.names) if getattr(lay, "names", None) else None}
        return meta, fdn.value

    def _handle(self, conn: socket.socket) -> bool:
        """One request; False when the client closes."""
        try:
            req = _recv(conn)
        except ConnectionError:
            return False
        op = req.get("op")
        try:
            if op == "load":
                meta, fdn = self._attach(req["fn"])
                try:
                    _send(conn, meta, fds=[fdn])
                finally:
                    os.close(fdn)
            elif op == "release":
                self.sim.sharing.release(req["fn"], self.gpu)
                _send(conn, {"ok": True})
            elif op == "dump":
                self.store[req["key"]] = _recv_exact(conn, int(req["nbytes"]))
                _send(conn, {"ok": True, "stored": len(self.store[req["key"]])})
            elif op == "close":
                _send(conn, {"ok": True})
                return False
            else:
                _send(conn, {"ok": False, "error": f"unknown op {op!r}"})
        except Exception as exc:           # report to the client, keep serving
            _send(conn, {"ok": False, "error": f"{type(exc).__name__}: {exc}"})
        return True

    def serve(self, clients: int = 1, timeout_s: float = 60.0) -> None:
        """Serve `clients` connections one after the other, each until it
        closes."""
        self.sock.settimeout(timeout_s)
        for _ in range(clients):
            conn, _ = self.sock.accept()
            with conn:
                conn.settimeout(timeout_s)
                while self._handle(conn):
                    pass

    def close(self) -> None:
        self.sock.close()
        if os.path.exists(self.path):
            os.unlink(self.path)


@dataclass
class SharedSegment:
    """A daemon-landed read-only segment mapped into this process."""
    fn: str
    h: int
    dptr: int
    seg_bytes: int
    checksum: int
    warmth: str
    tensors: list           # [dst_off, length] per tensor

    def tensor_ptr(self, i: int) -> int:
        return self.dptr + self.tensors[i][0]


class SageClient:
    """The function engine's side: SageLoadToGPU / SageDumpToDB.
    The calling process must have initialised its own plane (_lib.init) on
    the same GPU."""

    def __init__(self, path: str, gpu: int = 0):
        self.gpu = gpu
        self.sock = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        self.sock.connect(path)

    def load_to_gpu(self, fn: str) -> SharedSegment:
        _send(self.sock, {"op": "load", "fn": fn})
        meta, fds = _recv(self.sock, with_fd=True)
        if not meta.get("ok"):
            raise RuntimeError(meta.get("error", "load failed"))
        if not fds:
            raise RuntimeError("daemon sent no file descriptor")
        h, dptr = _lib.H(), _lib.u64()
        try:
            _lib.check(_lib.lib().sage_segment_import(self.gpu, fds[0], meta["phys_bytes"], _lib.C.byref(h),
                                                      _lib.C.byref(dptr)), "sage_segment_import")
        finally:
            for f in fds:
                os.close(f)
        return SharedSegment(fn, h.value, dptr.value, meta["seg_bytes"], meta["checksum"], meta["warmth"],
                             meta["tensors"])

    def release(self, seg: SharedSegment) -> None:
        _lib.check(_lib.lib().sage_segment_unimport(seg.h), "sage_segment_unimport")
        _send(self.sock, {"op": "release", "fn": seg.fn})
        if not _recv(self.sock).get("ok"):
            raise RuntimeError("release failed")

    def dump_to_db(self, key: str, data: np.ndarray) -> None:
        raw = np.ascontiguousarray(data).view(np.uint8).tobytes()
        _send(self.sock, {"op": "dump", "key": key, "nbytes": len(raw)})
        self.sock.sendall(raw)
        if not _recv(self.sock).get("ok"):
            raise RuntimeError("dump failed")

    def close(self) -> None:
        try:
            _send(self.sock, {"op": "close"})
            _recv(self.sock)
        finally:
            self.sock.close()
