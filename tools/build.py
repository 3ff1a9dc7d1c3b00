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
    # one nvcc per translation unit, in parallel, then one link
    objdir = os.path.join(HERE, "build_obj")
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in FLAGS if f != "-shared"]
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + f".{os.getpid()}.o")
        cmd = [NVCC, *cflags, *defs, "-I", nccl_include(), "-c", "-o", obj, src]
        procs.append((obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    log, objs, failed = [], [], False
    for obj, p in procs:
        out, err = p.communicate()
        log.append(err)
        objs.append(obj)
        if p.returncode != 0:
            failed = True
            sys.stderr.write(out + err)
    if failed:
        raise RuntimeError("nvcc failed building libdi.so")
    link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
            "-o", tmp, *objs, "-ldl"]
    res = subprocess.run(link, capture_output=True, text=True)
    for obj in objs:
        os.remove(obj)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking libdi.so")
    if verbose:
        sys.stderr.write("".join(log))
    with open(os.path.join(HERE, "ptxas.log"), "w") as f:
        f.write("".join(log))
    os.replace(tmp, SO)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(SO)
