"""Segment layouts: how a function's read-only data is packed in the "DB"
record and where each tensor lands in its HBM segment.

The reference tracks read-only data only as a byte count (`ro_mem_mb`,
functions.py:49, loaded as one transfer at functions.py:241-268).  The paper's
programming model (ref PAPER.md:345-347, Request/Data with a `key` and a
ReadOnly/Writable type) names the data a function loads; the real plane keeps
each tensor as an extent of a packed stream (arbitrary byte offsets, what a
key-value store returns) and lands it at an aligned offset of the segment so
kernels and PyTorch can use it in place.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib


def _align(v: int, a: int) -> int:
    return (v + a - 1) // a * a


@dataclass(frozen=True)
class SegmentLayout:
    src_off: tuple
    dst_off: tuple
    length: tuple
    packed_bytes: int
    seg_bytes: int
    names: tuple = ()
    _native: dict = field(default_factory=dict, compare=False, repr=False, hash=False)

    @classmethod
    def packed(cls, sizes: Sequence[int], align: int = 256, src_order: Optional[Sequence[int]] = None,
               names: Sequence[str] = ()) -> "SegmentLayout":
        """Tensors of `sizes` bytes: back to back in the packed stream (in
        `src_order`, default the same order) and at `align`-aligned offsets in
        the segment (in index order)."""
        if align % 16:
            raise ValueError("alignment must be a multiple of 16")
        n = len(sizes)
        order = list(range(n)) if src_order is None else list(src_order)
        if sorted(order) != list(range(n)):
            raise ValueError("src_order must be a permutation")
        src = [0] * n
        cur = 0
        for i in order:
            src[i] = cur
            cur += int(sizes[i])
        packed = cur
        dst = []
        d = 0
        for i in range(n):
            dst.append(d)
            d = _align(d + int(sizes[i]), align)
        seg = _align(d, 16) if n else 0
        return cls(tuple(src), tuple(dst), tuple(int(s) for s in sizes), packed, seg, tuple(names))

    @classmethod
    def identity(cls, nbytes: int) -> "SegmentLayout":
        return cls((0,), (0,), (int(nbytes),), int(nbytes), _align(int(nbytes), 16)) if nbytes else \
            cls((), (), (), 0, 0)

    @property
    def n(self) -> int:
        return len(self.length)

    def arrays(self):
        return (np.asarray(self.src_off, dtype=np.uint64), np.asarray(self.dst_off, dtype=np.uint64),
                np.asarray(self.length, dtype=np.uint64))

    def pack(self, tensors: Sequence[np.ndarray]) -> np.ndarray:
        """Serialise tensors into the packed stream (the DB record)."""
        out = np.empty(self.packed_bytes, dtype=np.uint8)
        for i, t in enumerate(tensors):
            b = np.ascontiguousarray(t).view(np.uint8).reshape(-1)
            if b.size != self.length[i]:
                raise ValueError(f"tensor {i}: {b.size} bytes, layout says {self.length[i]}")
            out[self.src_off[i]:self.src_off[i] + b.size] = b
        return out

    def handle(self) -> int:
        """The native layout handle (created once per process / library init)."""
        L = _lib.lib()
        key = _lib.generation()
        h = self._native.get(key)
        if h:
            return h
        s, d, n = self.arrays()
        out = _lib.H()
        P = _lib.C.POINTER(_lib.u64)
        _lib.check(L.sage_layout_create(s.ctypes.data_as(P), d.ctypes.data_as(P), n.ctypes.data_as(P),
                                        self.n, self.packed_bytes, self.seg_bytes, _lib.C.byref(out)),
                   "sage_layout_create")
        self._native[key] = out.value
        return out.value

    def forget_native(self) -> None:
        self._native.clear()
