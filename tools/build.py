"""Build libdi.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery).

    python tools/build.py [--force]
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HERE = os.path.join(ROOT, "paper_1204_6255_b200")
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libdi.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--fmad=false",                 # no FMA contraction: the select arithmetic follows P:258-268 op by op
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
    "-I", os.path.join(ROOT, "include"),
]


def nccl_include():
    """The header of the NCCL torch ships (the library libdi.so dlopens at run time)."""
    try:
        import nvidia.nccl
        for base in nvidia.nccl.__path__:
            inc = os.path.join(base, "include")
            if os.path.exists(os.path.join(inc, "nccl.h")):
                return inc
    except Exception:
        pass
    return "/usr/include"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))


def up_to_date() -> bool:
    if not os.path.exists(SO):
        return False
    t = os.path.getmtime(SO)
    return all(os.path.getmtime(p) <= t for p in deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return SO
    tmp = SO + f".tmp{os.getpid()}"
    # DI_NVCC_DEFS="-DNAME=V ..." (tuning experiments: compile-time knobs of the kernels)
    defs = os.environ.get("DI_NVCC_DEFS", "").split()
    cmd = [NVCC, *FLAGS, *defs, "-I", nccl_include(), "-o", tmp, *sources(), "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libdi.so")
    if verbose:
        sys.stderr.write(res.stderr)
    with open(os.path.join(HERE, "ptxas.log"), "w") as f:
        f.write(res.stderr)
    os.replace(tmp, SO)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(SO)
