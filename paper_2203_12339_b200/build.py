"""Build the sm_100a shared library in-tree (travels to the GPU box).

    python -m paper_2203_12339_b200.build

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3, translation units
compiled in parallel (csrc/abi.cu: every kernel and entry point except the C5
exact pair pass; csrc/abi_exact.cu: its entry point; csrc/abi_exact_part.cu
three times: its 64-material unrolled instantiations), then linked with
-shared into paper_2203_12339_b200/_sss_b200.so.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "_sss_b200.so"
OBJ = PKG / "build"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# (object name, source, extra flags)
UNITS = (("abi", "abi.cu", []), ("abi_exact", "abi_exact.cu", []),
         ("exact_p0", "abi_exact_part.cu", ["-DSSS_EXACT_PART=0"]),
         ("exact_p1", "abi_exact_part.cu", ["-DSSS_EXACT_PART=1"]),
         ("exact_p2", "abi_exact_part.cu", ["-DSSS_EXACT_PART=2"]))
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + \
        [PKG.parent / "include" / "sss_b200.h"]


def up_to_date() -> bool:
    if not OUT.exists():
        return False
    t = OUT.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in sources())


def _run(cmd, what):
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed: {what}")
    return res.stderr


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and up_to_date():
        return OUT
    OBJ.mkdir(exist_ok=True)
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                    "-Xptxas", "-v" if verbose else "-O3"]
    jobs = [([NVCC] + flags + x + ["-c", "-o", str(OBJ / (o + ".o")), str(CSRC / u)], o)
            for o, u, x in UNITS]
    with ThreadPoolExecutor(len(jobs)) as ex:
        logs = list(ex.map(lambda j: _run(*j), jobs))
    _run([NVCC] + ARCH + ["-shared", "-o", str(OUT)] +
         [str(OBJ / (o + ".o")) for o, _, _ in UNITS], "link")
    if verbose:
        sys.stderr.write("".join(logs))
    return OUT


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(OUT)
