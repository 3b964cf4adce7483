"""Build libsagedp.so (sm_100a) and the CPU oracle library in-tree.

`build()` is what __graft_entry__.build() calls.  nvcc cross-compiles for
sm_100a without a GPU; the products land next to their sources so they travel
to the GPU box with the repo snapshot (they are git-ignored).
"""
from __future__ import annotations

import os
import subprocess
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build"
LIB = PKG / "libsagedp.so"
WORKER = PKG / "sage_instance_worker"      # one FixedGSL instance process (SAGE_INSTANCE_PROCESS)
ORACLE_SRC = ROOT / "oracle" / "sage_oracle.c"
ORACLE_LIB = ROOT / "oracle" / "liboracle.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-v",
              "--expt-relaxed-constexpr", "-I", str(ROOT / "include")]
SOURCES = ["core.cu", "pool.cu", "land.cu", "bodies.cu", "gemm_tc.cu", "spmv_csb.cu", "invoke.cu", "fixedgsl.cu", "segtab.cu", "conv_tc.cu", "resnet.cu", "fanout.cu"]


def _run(cmd: list[str], log: Path | None = None) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        log.write_text(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_lib(force: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "sage_dp.h"]
    objs = []
    jobs = []
    for src in SOURCES:
        s = CSRC / src
        o = BUILD / (s.stem + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append((s, o))

    def compile_one(job):
        s, o = job
        _run([NVCC, *ARCH, *NVCC_FLAGS, "-c", str(s), "-o", str(o)], log=BUILD / (s.stem + ".ptxas.txt"))

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        list(ex.map(compile_one, jobs))
    if force or jobs or _stale(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lpthread"])
    wsrc = CSRC / "instance_worker.cpp"
    if force or _stale(WORKER, [wsrc, LIB]):
        _run(["g++", "-O2", "-o", str(WORKER), str(wsrc), f"-L{PKG}", "-lsagedp", "-Wl,-rpath,$ORIGIN"])
    return LIB


def build_oracle(force: bool = False) -> Path:
    if force or _stale(ORACLE_LIB, [ORACLE_SRC]):
        _run(["gcc", "-O3", "-march=x86-64-v3", "-fPIC", "-shared", "-o", str(ORACLE_LIB), str(ORACLE_SRC),
              "-lpthread"])
    return ORACLE_LIB


def build(force: bool = False) -> None:
    build_oracle(force)
    build_lib(force)


if __name__ == "__main__":
    import sys
    build(force="--force" in sys.argv)
    print(LIB, ORACLE_LIB)
