"""Function bodies called directly through the C-ABI (sage_launch) against
numpy references: the tcgen05 3xTF32 GEMM over several shapes at the FP32
contract (rtol 1e-3, atol 1e-4 * max|C|), the SIMT fp32 GEMM, stencil and
spmv edge shapes."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2404_14691_b200 import _lib
from paper_2404_14691_b200 import device as D

pytestmark = pytest.mark.gpu


def upload(arr):
    a = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
    seg = D.pool_alloc(0, max(256, a.size + 256), _lib.CLASS_WRITABLE, unaccounted=True)
    op = D.load(0, seg.dptr, a, None)
    op.wait()
    op.release()
    return seg


def run_body(kind, ro, ro_bytes, inp, inp_bytes, out_bytes, args):
    out = D.pool_alloc(0, max(256, out_bytes), _lib.CLASS_WRITABLE, unaccounted=True)
    slot = D.Slot(0)
    b, e = slot.launch(D.body_desc(kind, ro=ro, ro_bytes=ro_bytes, inp=inp, inp_bytes=inp_bytes, out=out.dptr,
                                   out_bytes=out_bytes, args=args))
    e.sync()
    got = D.read_device(0, out.dptr, out_bytes)
    for ev in (b, e):
        ev.release()
    slot.release()
    out.free()
    return got


@pytest.mark.parametrize("m,n,k", [(128, 64, 32), (256, 128, 256), (512, 256, 4096), (4096, 256, 4096),
                                   (1024, 192, 96), (384, 256, 512), (1024, 256, 1024)])
def test_sgemm_tcgen05_fp32(dp, m, n, k):
    rng = np.random.default_rng(m + n + k)
    A = rng.standard_normal((m, k), dtype=np.float32)
    BT = rng.standard_normal((n, k), dtype=np.float32)
    sa, sb = upload(A), upload(BT)
    got = run_body(_lib.BODY_SGEMM, sa.dptr, A.nbytes, sb.dptr, BT.nbytes, m * n * 4, (m, n, k))
    got = got.view(np.float32).reshape(m, n)
    want = O.sgemm_ref(A, BT.T)
    # FP32 contract (north_star): rtol 1e-3 with atol 1e-4 * max|C|.  A
    # single TF32 pass misses it (error ~2^-11 * sqrt(K) per element); the
    # 3xTF32 split is ~2^-21
    np.testing.assert_allclose(got, want, rtol=1e-3, atol=1e-4 * np.abs(want).max())
    # and well inside it: the residual is at fp32 level, not TF32 level
    err = np.abs(got.astype(np.float64) - want).max() / np.abs(want).max()
    assert err < 1e-5, err   # one TF32 pass: ~1e-4
    sa.free()
    sb.free()


def test_sgemm_simt_fp32_strict(dp):
    m, n, k = 256, 128, 512
    rng = np.random.default_rng(3)
    A = rng.standard_normal((m, k), dtype=np.float32)
    BT = rng.standard_normal((n, k), dtype=np.float32)
    sa, sb = upload(A), upload(BT)
    got = run_body(5, sa.dptr, A.nbytes, sb.dptr, BT.nbytes, m * n * 4, (m, n, k)).view(np.float32).reshape(m, n)
    np.testing.assert_allclose(got, O.sgemm_ref(A, BT.T), rtol=1e-3, atol=1e-4)
    sa.free()
    sb.free()


def test_sgemm_rejects_bad_shapes(dp):
    sa = upload(np.zeros(4096, np.float32))
    with pytest.raises(_lib.SageError):
        run_body(_lib.BODY_SGEMM, sa.dptr, 16384, sa.dptr, 16384, 16384, (100, 64, 32))
    sa.free()


# nx % 4 == 0 takes the vectorised slab kernel (partial warps, z not a slab
# multiple); other nx the scalar kernel
@pytest.mark.parametrize("shape", [(8, 8, 4), (33, 17, 9), (256, 64, 16), (12, 10, 11), (260, 7, 5), (256, 256, 64)])
def test_stencil(dp, shape):
    nx, ny, nz = shape
    rng = np.random.default_rng(nx)
    coef = rng.uniform(0.2, 0.6, (nz, ny, nx)).astype(np.float32)
    grid = rng.standard_normal((nz, ny, nx), dtype=np.float32)
    sc, sg = upload(coef), upload(grid)
    bits = int(np.float32(0.1).view(np.int32))
    got = run_body(_lib.BODY_STENCIL, sc.dptr, coef.nbytes, sg.dptr, grid.nbytes, grid.nbytes, (nx, ny, nz, bits))
    np.testing.assert_allclose(got.view(np.float32).reshape(nz, ny, nx), O.stencil_ref(coef, grid, 0.1),
                               rtol=1e-3, atol=1e-5)
    sc.free()
    sg.free()


@pytest.mark.parametrize("misalign", [0, 4])
def test_spmv_ragged_rows(dp, misalign):
    """misalign 0: 16-B aligned col/val (vectorised kernel, unaligned row
    starts); 4: col/val at 4-B offsets (scalar kernel)."""
    rng = np.random.default_rng(9)
    rows = 5000
    counts = rng.integers(0, 40, rows)
    counts[::7] = 0                                     # empty rows
    rowptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    nnz = int(rowptr[-1])
    col = rng.integers(0, rows, nnz, dtype=np.int32)
    val = rng.standard_normal(nnz, dtype=np.float32)
    x = rng.standard_normal(rows, dtype=np.float32)
    o_rp, o_col = 0, (rowptr.nbytes + 255) // 256 * 256 + misalign
    o_val = o_col + (col.nbytes + 255) // 256 * 256
    ro = np.zeros(o_val + val.nbytes, np.uint8)
    ro[o_rp:o_rp + rowptr.nbytes] = rowptr.view(np.uint8)
    ro[o_col:o_col + col.nbytes] = col.view(np.uint8)
    ro[o_val:o_val + val.nbytes] = val.view(np.uint8)
    sr, sx = upload(ro), upload(x)
    got = run_body(_lib.BODY_SPMV, sr.dptr, ro.size, sx.dptr, x.nbytes, rows * 4, (rows, nnz, o_rp, o_col, o_val))
    np.testing.assert_allclose(got.view(np.float32), O.spmv_ref(rowptr, col, val, x), rtol=1e-3, atol=1e-4)
    sr.free()
    sx.free()


def test_gather_ceiling_body(dp):
    """The diagnostic GATHER body (bench.py's spmv gather ceiling) reads the
    input at hashed indices: over an all-ones array warp 0 of block 0 sums
    32 lanes x 4 gathers; bad shapes are refused."""
    seg = upload(np.ones(1 << 12, np.float32))
    got = run_body(_lib.BODY_GATHER, 0, 0, seg.dptr, 4 << 12, 16, (4096,)).view(np.float32)
    assert got[0] == 128.0
    for inp_bytes, n in ((3 << 12, 4096), (4 << 12, 4098), (4 << 12, 0)):
        with pytest.raises(_lib.SageError):
            run_body(_lib.BODY_GATHER, 0, 0, seg.dptr, inp_bytes, 16, (n,))
    seg.free()


def _csb_case(rows, counts, slices, chunk_cols, seed=21):
    from paper_2404_14691_b200.parboil import csb_pack
    rng = np.random.default_rng(seed)
    rowptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    nnz = int(rowptr[-1])
    col = rng.integers(0, rows, nnz, dtype=np.int32)
    val = rng.standard_normal(nnz, dtype=np.float32)
    x = rng.standard_normal(rows, dtype=np.float32)
    off, ent, p = csb_pack(rowptr, col, val, rows, slices=slices, chunk_cols=chunk_cols)
    o_ent = (off.nbytes + 255) // 256 * 256
    ro = np.zeros(o_ent + ent.nbytes, np.uint8)
    ro[:off.nbytes] = off.view(np.uint8)
    ro[o_ent:] = ent.view(np.uint8).reshape(-1)
    args = (rows, rows, 0, o_ent, p["R"], p["CW"], p["Emax"], p["S"] | p["NS"] << 4 | (p["entries"] << 8))
    return rowptr, col, val, x, off, ent, p, ro, args


@pytest.mark.parametrize("rows,kind,slices,chunk_cols", [
    (5000, "ragged", 2, 6144), (5001, "ragged", 1, 1024), (4099, "ragged", 2, 1024), (1 << 16, "uniform", 2, 12288),
    (1 << 20, "uniform", 2, 6144)])
def test_spmv_csb_vs_oracle(dp, rows, kind, slices, chunk_cols):
    """The column-sliced block spmv (TMA-staged x chunks, DSMEM slice sum)
    against the oracle's independent CSB decode AND the CSR reference of the
    same matrix; two launches are bit-identical (fixed summation order)."""
    rng = np.random.default_rng(rows)
    counts = rng.integers(0, 40, rows) if kind == "ragged" else np.full(rows, 16)
    if kind == "ragged":
        counts[::7] = 0
        counts[3] = 300                                     # one long row: runs across warp steps
    rowptr, col, val, x, off, ent, p, ro, args = _csb_case(rows, counts, slices, chunk_cols)
    sr, sx = upload(ro), upload(x)
    got = run_body(_lib.BODY_SPMV_CSB, sr.dptr, ro.size, sx.dptr, x.nbytes, rows * 4, args).view(np.float32)
    again = run_body(_lib.BODY_SPMV_CSB, sr.dptr, ro.size, sx.dptr, x.nbytes, rows * 4, args).view(np.float32)
    assert np.array_equal(got, again)
    want = O.spmv_csb_ref(off, ent, rows, rows, p["R"], p["CW"], p["S"], x)
    np.testing.assert_allclose(got, want, rtol=1e-3, atol=1e-4)
    np.testing.assert_allclose(got, O.spmv_ref(rowptr, col, val, x), rtol=1e-3, atol=1e-4)
    sr.free()
    sx.free()


def test_spmv_csb_rejects_bad_formats(dp):
    rowptr, col, val, x, off, ent, p, ro, args = _csb_case(3000, np.full(3000, 4), 2, 6144)
    sr, sx = upload(ro), upload(x)
    bad = [list(args) for _ in range(5)]
    bad[0][4] = 1 << 15                       # R beyond the 14-bit row field
    bad[1][5] = 1001                          # chunk width not a multiple of 4
    bad[2][6] = 1 << 20                       # entry block larger than shared memory
    bad[3][3] = args[3] + 4                   # entries not 16-B aligned
    bad[4][7] = args[7] & ~0xF0 | 1 << 4      # a 1-deep ring
    for a in bad:
        with pytest.raises(_lib.SageError):
            run_body(_lib.BODY_SPMV_CSB, sr.dptr, ro.size, sx.dptr, x.nbytes, 3000 * 4, tuple(a))
    sr.free()
    sx.free()


_ENV_CHECK = r'''
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from oracle import oracle as O
from paper_2404_14691_b200 import _lib
from paper_2404_14691_b200 import device as D
sys.path.insert(0, sys.argv[1] + "/tests")
from test_bodies_gpu import run_body, upload
_lib.init(n_gpus=1, pool_bytes=4 << 30)
try:
    for m, n, k in [(512, 256, 4096), (4096, 256, 4096), (256, 256, 64)]:
        rng = np.random.default_rng(m + 7 * k)
        A = rng.standard_normal((m, k), dtype=np.float32)
        BT = rng.standard_normal((n, k), dtype=np.float32)
        sa, sb = upload(A), upload(BT)
        got = run_body(_lib.BODY_SGEMM, sa.dptr, A.nbytes, sb.dptr, BT.nbytes, m * n * 4, (m, n, k))
        got = got.view(np.float32).reshape(m, n)
        want = O.sgemm_ref(A, BT.T)
        np.testing.assert_allclose(got, want, rtol=1e-3, atol=1e-4 * np.abs(want).max())
        sa.free(); sb.free()
finally:
    _lib.shutdown()
print("ok")
'''


@pytest.mark.parametrize("env", [{"SAGE_SGEMM_PAIR": "1"}, {"SAGE_SGEMM_CR": "0"}, {"SAGE_SGEMM_MC": "1"},
                                 {"SAGE_SGEMM_SK": "1"}])
def test_sgemm_variants_fp32(env, tmp_path):
    """The opt-in sgemm kernels (CTA pair cta_group::2, split-K by red.add, stream-K,
    B-multicast clusters) hold the same FP32 contract; the variant is chosen
    at library load, so each runs in its own process."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parents[1])
    script = tmp_path / "check.py"
    script.write_text(_ENV_CHECK)
    r = subprocess.run([sys.executable, str(script), root], env={**os.environ, **env}, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-2000:]
