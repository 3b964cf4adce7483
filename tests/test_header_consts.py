"""The Python binding's body / kernel-kind constants equal include/sage_dp.h's
#defines (CPU: parses the header)."""
import re
from pathlib import Path

from paper_2404_14691_b200 import _lib

HDR = (Path(__file__).resolve().parent.parent / "include" / "sage_dp.h").read_text()


def define(name: str) -> int:
    m = re.search(rf"#define\s+{name}\s+(\d+)", HDR)
    assert m, name
    return int(m.group(1))


def test_body_constants_match_header():
    for n in ("TOUCH", "SGEMM", "STENCIL", "SPMV", "SPIN", "SGEMM_F32", "GATHER"):
        assert getattr(_lib, f"BODY_{n}") == define(f"SAGE_BODY_{n}"), n


def test_bench_kernel_kinds_match_header():
    import bench
    import inspect
    src = inspect.getsource(bench.kernel_stats)
    names = re.search(r"enumerate\(\[([^\]]*)\]\)", src).group(1).replace('"', "").replace(" ", "").split(",")
    for k, n in enumerate(names):
        assert define(f"SAGE_KERNEL_{n.upper()}") == k, n
    assert define("SAGE_KERNEL_KINDS") == len(names)
