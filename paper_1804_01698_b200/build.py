"""Build libspgemm.so (sm_100a) in-tree with nvcc."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libspgemm.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-std=c++17", "-lineinfo", "--extended-lambda",
    "-Xcompiler", "-fPIC", "-shared",
]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + [os.path.join(INCLUDE, "spgemm.h")])


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in _sources())


def build(force: bool = False, verbose: bool = False, out: str | None = None) -> str:
    """Build the library (``out``: another path, for A/B variants built with
    SPG_NVCC_EXTRA defines; the in-tree library is the product)."""
    if out is None and not force and not needs_build():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    extra = os.environ.get("SPG_NVCC_EXTRA", "").split()  # (A/B builds only)
    dst = out or LIB
    cmd = [nvcc, *NVCC_FLAGS, *extra, "-o", dst + ".tmp", os.path.join(CSRC, "spgemm.cu")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    os.replace(dst + ".tmp", dst)
    return dst


if __name__ == "__main__":
    print(build(force=True, verbose=True))
