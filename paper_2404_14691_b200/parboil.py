"""Parboil-style GPU functions with real read-only data (BASELINE cfg 2).

The reference calibrates its Parboil functions (lbm / mrif / tpacf, ref
PAPER.md:405-407) as byte counts with a fixed 24.3 ms compute delay
(functions.py:142-160).  cfg 2 asks for sgemm / stencil / spmv with SHARED
read-only segments; sizes are the builder's choice:

  sgemm    RO  A  4096 x 4096 fp32   (64 MiB, the shared weights)
           in  B  4096 x 256  fp32   (4 MiB)      out C 4096 x 256 fp32
  stencil  RO  c  per-cell coefficients 256 x 256 x 64 fp32 (16 MiB)
           in  grid 256 x 256 x 64 fp32 (16 MiB)  out grid (16 MiB)
  spmv     RO  1 Mi rows x 16 nnz: CSR row_ptr + col + val (132 MiB), or the
               same matrix column-sliced for shared-memory x (fmt="csb", 128 MiB)
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


def spmv(rows: int = 1 << 20, nnz_per_row: int = 16, seed: int = 13, name: str = "spmv", fmt: str = "csr",
         row_counts: np.ndarray | None = None, csb_opts: dict | None = None):
    """y = A.x with A the function's RO record.  fmt "csr": row_ptr / col /
    val (the scalar and 16-B vector CSR kernels); "csb": the same matrix in
    the column-sliced block format of csrc/spmv_csb.cu (csb_pack), which
    stages x through shared memory instead of gathering it from L2 -- the
    storage choice Parboil itself makes for its GPU spmv (JDS, a
    preprocessed format shipped as the dataset).  `row_counts` overrides the
    uniform nnz_per_row (ragged test matrices); `csb_opts` go to csb_pack."""
    if fmt not in ("csr", "csb"):
        raise ValueError(f"spmv: fmt must be csr or csb, not {fmt!r}")
    rng = np.random.Generator(np.random.PCG64(seed))
    if row_counts is None:
        nnz = rows * nnz_per_row
        rowptr = (np.arange(rows + 1, dtype=np.int64) * nnz_per_row).astype(np.int32)
    else:
        rowptr = np.concatenate([[0], np.cumsum(row_counts)]).astype(np.int32)
        nnz = int(rowptr[-1])
    col = rng.integers(0, rows, nnz, dtype=np.int32)
    val = rng.standard_normal(nnz, dtype=np.float32)
    x = rng.standard_normal(rows, dtype=np.float32)
    if fmt == "csb":
        off, ent, params = csb_pack(rowptr, col, val, rows, **(csb_opts or {}))
        # packed DB order: entries, then offsets (the land kernel unpacks)
        layout = SegmentLayout.packed([off.nbytes, ent.nbytes], align=256, src_order=[1, 0],
                                      names=("offsets", "entries"))
        db = layout.pack([off, ent])
        args = (rows, rows, layout.dst_off[0], layout.dst_off[1], params["R"], params["CW"], params["Emax"],
                params["S"] | params["NS"] << 4 | (int(params["entries"]) << 8))
        body = "spmv_csb"
    else:
        # packed DB order: values, columns, row pointers (a different order than
        # the landed layout, so the land kernel really unpacks)
        layout = SegmentLayout.packed([rowptr.nbytes, col.nbytes, val.nbytes], align=256, src_order=[2, 1, 0],
                                      names=("rowptr", "col", "val"))
        db = layout.pack([rowptr, col, val])
        args = (rows, nnz, layout.dst_off[0], layout.dst_off[1], layout.dst_off[2])
        body = "spmv"
    data = FunctionData(layout, db, body=body, args=args, input=x.view(np.uint8), out_bytes=rows * 4)
    spec = FunctionSpec(name=name, ro_mem_mb=_mb(layout.seg_bytes), writable_mem_mb=_writable_mb(x.nbytes, rows * 4),
                        compute_ms=1.0, input_bytes_host_mb=_mb(x.nbytes), input_bytes_pcie_mb=_mb(x.nbytes),
                        body=body)
    return spec, data


CSB_WARPS = 16               # consumer warps per CTA (kCsbWarps)
CSB_SKIP = 0xFFFFFFFF        # padding entry
CSB_SMEM = 227 * 1024 - 128  # dynamic shared memory per CTA the kernel may use (kCsbSmem)
CSB_STAGES = 4               # x-chunk ring depth


def csb_pack(rowptr: np.ndarray, col: np.ndarray, val: np.ndarray, cols: int, sms: int = 148, slices: int = 2,
             chunk_cols: int = 6144, stages: int = CSB_STAGES):
    """CSR -> the column-sliced block format (layout: csrc/spmv_csb.cu).

    Rows go to G row groups of R rows (G x S CTAs ~ the B200's 148 SMs),
    columns to S slices of SC columns and each slice to CH chunks of CW
    columns (one shared-memory x chunk, `stages` of them in flight); inside
    a chunk each of the 16 consumer warps owns a contiguous row range, its
    entries sorted by row.  Returns (offsets u32,
    entries u32 [n, 2] = (row_local << 17 | col_in_chunk, val bits), params).
    """
    rows = rowptr.size - 1
    nnz = int(rowptr[-1])
    S = max(1, int(slices))
    G = max(1, -(-sms // S))
    R = -(-rows // G)
    if R >= 1 << 14:
        R = (1 << 14) - 1
    G = -(-rows // R)
    SC = -(-(-(-cols // S)) // 4) * 4
    row = np.repeat(np.arange(rows, dtype=np.int64), np.diff(rowptr.astype(np.int64)))
    c64 = col.astype(np.int64)
    g, rl = row // R, row % R
    sl, cc = c64 // SC, c64 % SC
    w = rl * CSB_WARPS // R
    CW = int(chunk_cols)
    while True:
        CH = -(-SC // CW)
        nb = G * S * CH
        c = cc // CW
        sub = (((g * S + sl) * CH + c) * CSB_WARPS + w)
        counts = np.bincount(sub, minlength=nb * CSB_WARPS).reshape(nb, CSB_WARPS)
        per_bucket = counts.sum(1)
        padded = per_bucket + (per_bucket & 1)
        emax = int(padded.max()) if nb else 0
        smem = ((4 * R + 127) // 128 * 128 + (4 * (CH * CSB_WARPS + 1) + 127) // 128 * 128
                + stages * ((4 * CW + 8 * emax + 127) // 128 * 128))
        if smem <= CSB_SMEM or CW <= 1024:
            break
        CW //= 2
    if smem > CSB_SMEM:
        raise ValueError(f"csb_pack: {rows} rows need {smem} B of shared memory")
    # CSR order is row-major, so a stable sort by sub-bucket keeps rows sorted
    # inside each sub-bucket (16-bit keys take numpy's radix sort)
    order = np.argsort(sub.astype(np.uint16) if nb * CSB_WARPS <= 1 << 16 else sub, kind="stable")
    bucket_start = np.concatenate([[0], np.cumsum(padded)])
    sorted_first = np.concatenate([[0], np.cumsum(per_bucket)])
    off = np.empty(nb * CSB_WARPS + 1, np.uint32)
    within = np.concatenate([np.zeros((nb, 1), np.int64), np.cumsum(counts, 1)[:, :-1]], 1)
    off[:-1] = (bucket_start[:-1, None] + within).reshape(-1)
    off[-1] = bucket_start[-1]
    ent = np.empty((int(bucket_start[-1]), 2), np.uint32)
    ent[:, 0] = CSB_SKIP
    ent[:, 1] = 0
    b_sorted = sub[order] // CSB_WARPS
    pos = np.arange(nnz, dtype=np.int64) - sorted_first[b_sorted] + bucket_start[b_sorted]
    ent[pos, 0] = ((rl[order] << 17) | (cc[order] - (cc[order] // CW) * CW)).astype(np.uint32)
    ent[pos, 1] = val[order].view(np.uint32)
    params = {"R": int(R), "S": S, "NS": int(stages), "CW": CW, "CH": int(CH), "G": int(G), "SC": int(SC), "Emax": emax,
              "entries": int(bucket_start[-1]), "nnz": nnz}
    return off, ent, params


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
