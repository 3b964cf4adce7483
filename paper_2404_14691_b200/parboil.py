"""Parboil-style GPU functions with real read-only data (BASELINE cfg 2).

The reference calibrates its Parboil functions (lbm / mrif / tpacf, ref
PAPER.md:405-407) as byte counts with a fixed 24.3 ms compute delay
(functions.py:142-160).  cfg 2 asks for sgemm / stencil / spmv with SHARED
read-only segments; sizes are the builder's choice:

  sgemm    RO  A  4096 x 4096 fp32   (64 MiB, the shared weights)
           in  B  4096 x 256  fp32   (4 MiB)      out C 4096 x 256 fp32
  stencil  RO  c  per-cell coefficients 256 x 256 x 64 fp32 (16 MiB)
           in  grid 256 x 256 x 64 fp32 (16 MiB)  out grid (16 MiB)
  spmv     RO  CSR 1 Mi rows x 16 nnz: row_ptr + col + val (132 MiB)
           in  x 1 Mi fp32 (4 MiB)                out y (4 MiB)

Each builder returns (FunctionSpec, FunctionData): the spec's RO footprint
is exactly the landed segment, its writable footprint holds input + output.
"""
from __future__ import annotations

import numpy as np

from .dataplane import FunctionData, synthetic_bytes
from .functions import FunctionSpec
from .layout import SegmentLayout

MIB = 1 << 20


def _mb(nbytes: int) -> float:
    """Smallest µMB-exact MB figure whose byte view (1 MB := 1 MiB) holds nbytes."""
    return -(-nbytes * 1_000_000 // MIB) / 1_000_000


def _writable_mb(*nbytes: int) -> float:
    return _mb(sum((n + 255) // 256 * 256 + 256 for n in nbytes))


def sgemm(m: int = 4096, k: int = 4096, n: int = 256, seed: int = 11, name: str = "sgemm", body: str = "sgemm"):
    """C = A . B with the second operand passed transposed (BT [n, k]), as
    Parboil's sgemm does ("matrix2t"); body "sgemm" runs on tcgen05 (TF32
    MMAs, fp32 accumulate), "sgemm_f32" on the SIMT fp32 cores."""
    rng = np.random.Generator(np.random.PCG64(seed))
    A = rng.standard_normal((m, k), dtype=np.float32)
    BT = rng.standard_normal((n, k), dtype=np.float32)
    layout = SegmentLayout.packed([A.nbytes], align=256, names=("A",))
    data = FunctionData(layout, layout.pack([A]), body=body, args=(m, n, k), input=BT.reshape(-1).view(np.uint8),
                        out_bytes=m * n * 4)
    spec = FunctionSpec(name=name, ro_mem_mb=_mb(layout.seg_bytes), writable_mem_mb=_writable_mb(BT.nbytes, m * n * 4),
                        compute_ms=1.0, input_bytes_host_mb=_mb(BT.nbytes), input_bytes_pcie_mb=_mb(BT.nbytes),
                        body=body)
    return spec, data


def stencil(nx: int = 256, ny: int = 256, nz: int = 64, beta: float = 0.1, seed: int = 12, name: str = "stencil"):
    rng = np.random.Generator(np.random.PCG64(seed))
    coef = rng.uniform(0.2, 0.6, (nz, ny, nx)).astype(np.float32)
    grid = rng.standard_normal((nz, ny, nx), dtype=np.float32)
    layout = SegmentLayout.packed([coef.nbytes], align=256, names=("coef",))
    bits = int(np.float32(beta).view(np.int32))
    data = FunctionData(layout, layout.pack([coef]), body="stencil", args=(nx, ny, nz, bits),
                        input=grid.reshape(-1).view(np.uint8), out_bytes=grid.nbytes)
    spec = FunctionSpec(name=name, ro_mem_mb=_mb(layout.seg_bytes),
                        writable_mem_mb=_writable_mb(grid.nbytes, grid.nbytes), compute_ms=1.0,
                        input_bytes_host_mb=_mb(grid.nbytes), input_bytes_pcie_mb=_mb(grid.nbytes), body="stencil")
    return spec, data


def spmv(rows: int = 1 << 20, nnz_per_row: int = 16, seed: int = 13, name: str = "spmv"):
    rng = np.random.Generator(np.random.PCG64(seed))
    nnz = rows * nnz_per_row
    rowptr = (np.arange(rows + 1, dtype=np.int64) * nnz_per_row).astype(np.int32)
    col = rng.integers(0, rows, nnz, dtype=np.int32)
    val = rng.standard_normal(nnz, dtype=np.float32)
    x = rng.standard_normal(rows, dtype=np.float32)
    # packed DB order: values, columns, row pointers (a different order than
    # the landed layout, so the land kernel really unpacks)
    layout = SegmentLayout.packed([rowptr.nbytes, col.nbytes, val.nbytes], align=256, src_order=[2, 1, 0],
                                  names=("rowptr", "col", "val"))
    data = FunctionData(layout, layout.pack([rowptr, col, val]), body="spmv",
                        args=(rows, nnz, layout.dst_off[0], layout.dst_off[1], layout.dst_off[2]),
                        input=x.view(np.uint8), out_bytes=rows * 4)
    spec = FunctionSpec(name=name, ro_mem_mb=_mb(layout.seg_bytes), writable_mem_mb=_writable_mb(x.nbytes, rows * 4),
                        compute_ms=1.0, input_bytes_host_mb=_mb(x.nbytes), input_bytes_pcie_mb=_mb(x.nbytes),
                        body="spmv")
    return spec, data


def cfg2_functions(scale: int = 1):
    """The cfg-2 mix; scale > 1 shrinks every dimension (tests)."""
    if scale == 1:
        fns = [sgemm(), stencil(), spmv()]
    else:
        fns = [sgemm(m=4096 // scale // 128 * 128 or 128, k=4096 // scale // 8 * 8 or 8, n=256 // scale // 128 * 128 or 128),
               stencil(nx=max(8, 256 // scale), ny=max(8, 256 // scale), nz=max(4, 64 // scale)),
               spmv(rows=max(1024, (1 << 20) // scale))]
    table = {s.name: s for s, _ in fns}
    data = {s.name: d for s, d in fns}
    return table, data


def synthetic_function(name: str, ro_mb: float, writable_mb: float, input_mb: float, tensors: int = 64):
    """A cfg-1 / cfg-4 style synthetic function (TOUCH body) with a ragged
    multi-tensor RO record of exactly ro_mb MiB landed."""
    spec = FunctionSpec(name=name, ro_mem_mb=ro_mb, writable_mem_mb=writable_mb, compute_ms=1.0,
                        input_bytes_host_mb=input_mb, input_bytes_pcie_mb=input_mb)
    from .dataplane import synthetic_data
    return spec, synthetic_data(spec, tensors=tensors)
